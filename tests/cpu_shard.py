"""CPU test double of one rank's Lloyd shard — TEST INFRASTRUCTURE ONLY.

Implements the numeric steps of ``engine.ShardSequence`` with numpy (exact f64
distances, lowest-index argmin, f64 sums) so the *shared* iteration sequence
and the multi-rank repair protocol (``distributed.repair_protocol``) can run
under a gloo process group on a machine without a GPU.  The CUDA engine
implements the same methods with the kernels; the gloo tests check that a
sharded run reproduces the single-rank run of this double exactly.
"""
import numpy as np
import torch

from paper_2501_05587_b200.engine import ShardSequence


class LocalComm:
    """world_size 1 stand-in, so single-rank runs use the same repair protocol."""

    rank = 0
    world_size = 1
    multi = False
    offset = 0

    def all_reduce_sum(self, t):
        pass

    def all_gather(self, t):
        return [t.clone()]


class NumpyShard(ShardSequence):
    def __init__(self, P_local, k, n_total, offset, comm, labels0_local, C0, max_iters, dtype=np.float64):
        self.P = np.ascontiguousarray(P_local, dtype=dtype)
        self.P64 = self.P.astype(np.float64)
        self.n, self.d = self.P.shape
        self.k, self.n_total, self.dtype = k, n_total, np.dtype(dtype)
        self.comm = comm
        if comm is not None:
            comm.offset = offset
        self.labels = [torch.from_numpy(np.asarray(labels0_local, dtype=np.int32).copy()),
                       torch.zeros(self.n, dtype=torch.int32)]
        self.acc = torch.zeros(k * self.d + k + 2, dtype=torch.float64)
        self.state = torch.zeros(9, dtype=torch.int64)
        self.C = np.asarray(C0, dtype=dtype).copy()
        self.obj_hist = np.zeros(max_iters)
        self.rep_hist = np.zeros(max_iters, dtype=np.int64)

    def _stopped(self):
        return int(self.state[1]) != 0

    # -- numeric steps ------------------------------------------------------------
    def _assign(self, prev, new, acc, state):
        if self._stopped():
            return
        C64 = self.C.astype(np.float64)
        s = (C64 * C64).sum(1)[None, :] - 2.0 * self.P64 @ C64.T
        lab = np.argmin(s, axis=1).astype(np.int32)
        new.copy_(torch.from_numpy(lab))
        kd = self.k * self.d
        acc[kd:kd + self.k] += torch.from_numpy(np.bincount(lab, minlength=self.k).astype(np.float64))
        acc[kd + self.k + 1] += float(np.count_nonzero(lab != prev.numpy()))

    def _sort_and_sum(self, new, state):
        if self._stopped():
            return
        lab = new.numpy()
        self.perm = np.argsort(lab, kind="stable")
        C64 = self.C.astype(np.float64)
        self.own = ((self.P64[self.perm] - C64[lab[self.perm]]) ** 2).sum(1)
        sums = np.zeros((self.k, self.d))
        np.add.at(sums, lab, self.P64)
        self.acc[:self.k * self.d] += torch.from_numpy(sums.ravel())
        self.acc[self.k * self.d + self.k] += float(self.own.sum())

    def _repair_local(self, prev, new):
        from paper_2501_05587_b200.distributed import repair_protocol
        repair_protocol(self, LocalComm(), prev, new)

    def _finalize(self, check_convergence, tol):
        if self._stopped():
            return
        kd = self.k * self.d
        acc = self.acc.numpy()
        counts = acc[kd:kd + self.k]
        sums = acc[:kd].reshape(self.k, self.d)
        C = np.zeros((self.k, self.d))
        nz = counts > 0
        C[nz] = sums[nz] / counts[nz, None]
        self.C = C.astype(self.dtype)
        it = int(self.state[0])
        self.obj_hist[it] = acc[kd + self.k]
        self.rep_hist[it] = int(self.state[3])
        self.state[3] = 0
        self.state[0] = it + 1
        if check_convergence and acc[kd + self.k + 1] / self.n_total <= tol:
            self.state[1] = 1
            self.state[2] = 1

    # -- multi-rank primitives (same contract as the CUDA engine's) ----------------
    def flag_pending(self):
        if self._stopped():
            return
        kd = self.k * self.d
        if (self.acc[kd:kd + self.k] == 0).any():
            self.acc_saved = self.acc.clone()
            self.state[1] = 2

    def restore_pending(self):
        self.acc.copy_(self.acc_saved)
        self.state[1] = 0

    def snapshot_state(self):
        return self.state[:2].clone()

    @staticmethod
    def read_snapshot(snap):
        return snap.numpy()

    def repair_select(self, offset, E):
        gidx = offset + self.perm
        order = np.lexsort((gidx, -self.own))[:E]
        out = np.full((E, 3), [-np.inf, 9.0e18, -1.0])
        out[:order.size, 0] = self.own[order]
        out[:order.size, 1] = gidx[order]
        out[:order.size, 2] = order
        return torch.from_numpy(out)

    def new_deltas(self, E):
        return torch.zeros((E, self.d + 4), dtype=torch.float64)

    def repair_apply_batch(self, prev, new, pos, js, slots, deltas):
        lab = new.numpy()
        C64 = self.C.astype(np.float64)
        for q, j, e in zip(pos, js, slots):
            donor = int(self.perm[q])
            old = int(lab[donor])
            dnew = float(((self.P64[donor] - C64[j]) ** 2).sum())
            p = int(prev.numpy()[donor])
            deltas[e] = torch.from_numpy(np.concatenate([self.P64[donor], [old, dnew - self.own[q],
                                                                           float((j != p) - (old != p)), 1.0]]))
            lab[donor] = j
            self.own[q] = -np.inf

    def repair_commit_batch(self, js, deltas):
        dl = deltas.numpy()
        d, k = self.d, self.k
        acc = self.acc.numpy()
        for e, j in enumerate(js):
            if dl[e, d + 3] != 1.0:
                continue
            old = int(dl[e, d])
            acc[old * d:(old + 1) * d] -= dl[e, :d]
            acc[j * d:(j + 1) * d] += dl[e, :d]
            acc[k * d + old] -= 1.0
            acc[k * d + j] += 1.0
            acc[k * d + k] += dl[e, d + 1]
            acc[k * d + k + 1] += dl[e, d + 2]
            self.state[3] += 1

    # -- whole fit ------------------------------------------------------------------
    def fit(self, max_iters, check_convergence=False, tol=0.0):
        if self._multi():
            self.run_multi(max_iters, check_convergence, tol)
        else:
            for t in range(max_iters):
                self.iteration(t, check_convergence, tol)
        iters = int(self.state[0])
        return {"labels": self.labels[iters % 2].numpy().copy(), "iters": iters,
                "objective": self.obj_hist[:iters].copy(), "repairs": self.rep_hist[:iters].copy(),
                "centroids": self.C.copy(), "converged": bool(self.state[2])}
