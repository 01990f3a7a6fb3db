"""Kernel K-means drivers on the B200 (the reference's run_popcorn / run_baseline).

``run_popcorn(points, cfg)`` and ``run_baseline(points, cfg)`` keep the
``_ALGORITHMS`` driver contract (clustering.py:165-279): same init stream,
argmin tie-break, repair policy, objective, convergence and result type.
Both formulations compute the same distances — the reference keeps the naive
one as a cross-check — so both run the same device engine (``KernelEngine``):

  K = kernel(P P^T) once in HBM (kernels.kernel_matrix), then per iteration
  counting sort of the labels -> S[j,:] = sum_{m in L_j} K[m,:] (one streaming
  pass over K) -> z, centroid norms -> D = diag(K) - 2 S/|L| + c, argmin ->
  repair -> counts/objective/changed/history, all on the device
  (csrc/kernel_kmeans.cu).  timings.kernel_matrix_seconds is the K build.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from .engine import RunOutput, _p, _stream, h2d_staged, init_labels, require_cuda
from .kernels import GramMethod, KernelSpec, kernel_matrix, padded_ld

_F32 = np.dtype(np.float32)


class KernelEngine:
    """One device holding K (n x ldk) and the per-iteration buffers."""

    def __init__(self, points, k: int, spec: KernelSpec, *, dtype=np.float32, device=None, max_iters: int = 30):
        self.dev = require_cuda(device)
        self.dtype = np.dtype(dtype)
        self.sfx = "f32" if self.dtype == _F32 else "f64"
        td = torch.float32 if self.dtype == _F32 else torch.float64
        self.spec = spec
        with torch.cuda.device(self.dev):
            if isinstance(points, torch.Tensor):
                P = points.to(device=self.dev, dtype=td).contiguous()
            else:
                P = h2d_staged(np.ascontiguousarray(points, dtype=self.dtype), self.dev)
            self.n, self.d = int(P.shape[0]), int(P.shape[1])
            self.k = int(k)
            n, kk, dev = self.n, self.k, self.dev
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            self.K = torch.empty((n, padded_ld(n)), dtype=td, device=dev)  # allocated outside the timing
            t0.record()
            kernel_matrix(P, spec, out=self.K)
            t1.record()
            self._kev = (t0, t1)
            del P
            self.ldk = padded_ld(n)
            self.S = torch.empty((kk, self.ldk), dtype=torch.float64, device=dev)
            self.labels = [torch.zeros(n, dtype=torch.int32, device=dev) for _ in range(2)]
            self.own = torch.empty(n, dtype=torch.float64, device=dev)
            self.perm = torch.empty(n, dtype=torch.int32, device=dev)
            self.offsets = torch.empty(kk + 1, dtype=torch.int32, device=dev)
            self.cursor = torch.empty(kk, dtype=torch.int32, device=dev)
            self.cnt = torch.zeros(kk + 2, dtype=torch.float64, device=dev)  # counts of the current labels
            self.acc = torch.zeros(2 * kk + 2, dtype=torch.float64, device=dev)
            self.icounts = torch.zeros(kk, dtype=torch.int32, device=dev)
            sb = int(L.load().pcb_kk_repair_scratch_bytes(n, kk))
            self.scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
            self.scratch_bytes = sb
            self.state = torch.zeros(L.STATE_WORDS, dtype=torch.int64, device=dev)
            self.max_iters = max(1, int(max_iters))
            self.obj_hist = torch.zeros(self.max_iters, dtype=torch.float64, device=dev)
            self.rep_hist = torch.zeros(self.max_iters, dtype=torch.int64, device=dev)

    def kernel_matrix_seconds(self) -> float:
        self._kev[1].synchronize()
        return self._kev[0].elapsed_time(self._kev[1]) / 1e3

    def init_labels_device(self, seed: int) -> None:
        """init_assignments (clustering.py:91-108) in HBM, then counts."""
        with torch.cuda.device(self.dev):
            init_labels(self.n, self.k, seed, self.dev, out=self.labels[0])
            self._count(self.labels[0])

    def set_labels(self, labels) -> None:
        with torch.cuda.device(self.dev):
            self.labels[0].copy_(torch.from_numpy(np.ascontiguousarray(labels, dtype=np.int32)).to(self.dev))
            self._count(self.labels[0])

    def _count(self, lab) -> None:
        self.cnt.zero_()
        L.call("pcb_count_labels", _p(lab), None, self.n, self.k, 0, _p(self.cnt), None, _stream())

    def iteration(self, t: int, check_convergence: bool = False, tol: float = 0.0, events=None) -> None:
        """One iteration (clustering.py:195-216): labels[t%2] -> labels[(t+1)%2]."""
        prev, new = self.labels[t % 2], self.labels[(t + 1) % 2]
        n, k, sfx = self.n, self.k, self.sfx
        self.acc.zero_()
        if events is not None:
            events[0].record()
        L.call("pcb_sort_by_label", _p(prev), n, k, _p(self.cnt), _p(self.offsets), _p(self.cursor),
               _p(self.perm), _p(self.state), _stream())
        L.call(f"pcb_kk_segment_sums_{sfx}", _p(self.K), self.ldk, n, n, _p(self.perm), _p(self.offsets), k,
               _p(self.S), self.ldk, _p(self.state), _stream())
        L.call(f"pcb_kk_assign_{sfx}", _p(self.K), self.ldk, _p(self.S), self.ldk, n, k, _p(self.cnt),
               _p(self.acc), _p(prev), _p(new), _p(self.own), _p(self.icounts), _p(self.state), _stream())
        if events is not None:
            events[1].record()
        L.call(f"pcb_kk_repair_{sfx}", _p(self.K), self.ldk, _p(self.S), self.ldk, n, k, _p(self.cnt),
               _p(self.acc), _p(new), _p(self.own), _p(self.icounts), _p(self.state), _p(self.scratch),
               self.scratch_bytes, _stream())
        L.call("pcb_kk_finalize", _p(new), _p(prev), _p(self.own), n, k, _p(self.acc), _p(self.cnt),
               _p(self.obj_hist), _p(self.rep_hist), _p(self.state), int(check_convergence), float(tol),
               _stream())
        if events is not None:
            events[2].record()

    def run(self, max_iters: int, tol: float = 0.0, check_convergence: bool = False,
            record_history: bool = True) -> RunOutput:
        if max_iters > self.max_iters:
            raise ValueError("max_iters exceeds the engine's history capacity")
        with torch.cuda.device(self.dev):
            self.state.zero_()
            hist = torch.empty((max_iters, self.n), dtype=torch.int32, pin_memory=True) if record_history else None
            evs = []
            for t in range(max_iters):
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                self.iteration(t, check_convergence, tol, ev)
                evs.append(ev)
                if hist is not None:
                    hist[t].copy_(self.labels[(t + 1) % 2], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            st = self.state.cpu().numpy()
            if st[5] != 0:
                raise ValueError("row_argmin: matrix contains NaN")  # dense.py:66-67
            iters = int(st[0])
            dist_s = sum(e[0].elapsed_time(e[1]) for e in evs[:iters]) / 1e3
            upd_s = sum(e[1].elapsed_time(e[2]) for e in evs[:iters]) / 1e3
            return RunOutput(
                iterations_run=iters, converged=bool(st[2]),
                objective_history=self.obj_hist[:iters].cpu().numpy().astype(np.float64),
                repairs=self.rep_hist[:iters].cpu().numpy().astype(np.int64),
                labels=self.labels[iters % 2].cpu().numpy(),
                label_history=[hist[t].numpy().copy() for t in range(iters)] if hist is not None else [],
                centroids=None, distance_seconds=dist_s, update_seconds=upd_s)

    # -- lockstep (parity harness) ---------------------------------------------------
    def step_from(self, labels_prev) -> dict:
        """One iteration from given previous labels; returns labels, own, objective."""
        self.set_labels(labels_prev)
        with torch.cuda.device(self.dev):
            self.state.zero_()
            self.iteration(0)
            torch.cuda.current_stream().synchronize()
            return {"labels": self.labels[1].cpu().numpy(), "own": self.own.cpu().numpy(),
                    "objective": float(self.obj_hist[0].item()), "moved": int(self.rep_hist[0].item()),
                    "S": self.S[:, :self.n].cpu().numpy(), "nan": bool(self.state[5].item())}

    def cluster_terms(self) -> tuple[np.ndarray, np.ndarray]:
        """(counts, c_j) of the final labels: c_j = sum_{l,m in L_j} K[l,m] / |L_j|^2."""
        with torch.cuda.device(self.dev):
            lab = self.labels[int(self.state[0].item()) % 2]
            self._count(lab)
            self.acc.zero_()
            L.call("pcb_sort_by_label", _p(lab), self.n, self.k, _p(self.cnt), _p(self.offsets), _p(self.cursor),
                   _p(self.perm), None, _stream())
            L.call(f"pcb_kk_segment_sums_{self.sfx}", _p(self.K), self.ldk, self.n, self.n, _p(self.perm),
                   _p(self.offsets), self.k, _p(self.S), self.ldk, None, _stream())
            cnt = self.cnt[:self.k].cpu().numpy()
            S = self.S[:, :self.n]
            labt = lab.long()
            z = S.gather(0, labt.view(1, -1)).view(-1) / self.cnt[:self.k][labt]
            csum = torch.zeros(self.k, dtype=torch.float64, device=self.dev).index_add_(0, labt, z)
            return cnt, (csum / self.cnt[:self.k]).cpu().numpy()


def _driver(points, cfg, name: str):
    from .clustering import ClusteringResult, TimingBreakdown, _prepare_points
    from .validation import normalize_dtype
    dtype = normalize_dtype(cfg.dtype)
    P, n, d = _prepare_points(points, cfg)
    cfg.validate_for(n)
    spec = cfg.kernel if isinstance(cfg.kernel, KernelSpec) else KernelSpec()
    eng = KernelEngine(P, cfg.k, spec, dtype=dtype, device=cfg.device, max_iters=cfg.max_iters)
    eng.init_labels_device(cfg.seed)
    out = eng.run(cfg.max_iters, cfg.tol, cfg.check_convergence, record_history=cfg.record_label_history)
    timings = TimingBreakdown(eng.kernel_matrix_seconds(), out.distance_seconds, out.update_seconds)
    return ClusteringResult(labels=out.labels, iterations_run=out.iterations_run,
                            objective_history=out.objective_history, converged=out.converged,
                            timings=timings, label_history=out.label_history, repairs=out.repairs)


def run_popcorn(points, cfg) -> "ClusteringResult":
    """Matrix-centric kernel K-means (clustering.py:165-218) on the B200."""
    return _driver(points, cfg, "popcorn")


def run_baseline(points, cfg) -> "ClusteringResult":
    """The naive formulation (clustering.py:243-279): same distances, same engine."""
    return _driver(points, cfg, "baseline")


__all__ = ["KernelEngine", "run_popcorn", "run_baseline", "GramMethod"]


def cluster_terms(X_fit, labels, k: int, spec: KernelSpec):
    """(sizes, c_j) for predict: sizes = max(|L_j|, 1) (estimator.py:175),
    c_j = sum_{l,m in L_j} K(x_l, x_m) / sizes_j^2 — from the device K."""
    dt = np.asarray(X_fit).dtype
    eng = KernelEngine(X_fit, k, spec, dtype=dt, max_iters=1)
    eng.set_labels(labels)
    cnt, c = eng.cluster_terms()
    sizes = np.maximum(cnt, 1.0)
    c = np.where(cnt > 0, c * (cnt / sizes) ** 2, 0.0)  # empty cluster: self term 0
    return sizes, c


def predict_labels(X_fit, labels, k: int, spec: KernelSpec, sizes, cself, X) -> np.ndarray:
    """Kernel-trick nearest centroid (estimator.py:137-147) on the device:
    Kx = kernel(X_fit X^T) (n x m, tcgen05 3xTF32 / SIMT f64), per-cluster
    row sums of Kx over the training labels, then argmin of
    self(x) - 2 sum/|L_j| + c_j."""
    from .kernels import FAMILY_CODE
    dev = require_cuda(None)
    dt = np.asarray(X_fit).dtype
    f64 = dt == np.float64
    td = torch.float64 if f64 else torch.float32
    sfx = "f64" if f64 else "f32"
    with torch.cuda.device(dev):
        A = torch.from_numpy(np.ascontiguousarray(X_fit)).to(dev)
        B = torch.from_numpy(np.ascontiguousarray(X, dtype=dt)).to(dev)
        n, d = int(A.shape[0]), int(A.shape[1])
        m = int(B.shape[0])
        ldm = padded_ld(m)
        an = torch.empty(n, dtype=td, device=dev)
        bn = torch.empty(m, dtype=td, device=dev)
        L.call(f"pcb_point_norms_{sfx}", _p(A), n, d, _p(an), _stream())
        L.call(f"pcb_point_norms_{sfx}", _p(B), m, d, _p(bn), _stream())
        Kx = torch.empty((n, ldm), dtype=td, device=dev)
        nonfinite = torch.zeros(1, dtype=torch.int64, device=dev)
        kargs = (FAMILY_CODE[spec.family], float(spec.gamma), float(spec.coef), int(spec.degree),
                 float(spec.sigma))
        if f64:
            L.call("pcb_kernel_cross_f64", _p(A), n, _p(B), m, d, _p(an), _p(bn), _p(Kx), ldm, *kargs,
                   _p(nonfinite), _stream())
        else:
            ld = (d + 31) // 32 * 32
            ah = torch.empty((n, ld), dtype=torch.float32, device=dev)
            al = torch.empty_like(ah)
            bh = torch.empty((m, ld), dtype=torch.float32, device=dev)
            bl = torch.empty_like(bh)
            L.call("pcb_split_tf32", _p(A), n, d, ld, _p(ah), _p(al), _stream())
            L.call("pcb_split_tf32", _p(B), m, d, ld, _p(bh), _p(bl), _stream())
            L.call("pcb_kernel_cross_f32", _p(ah), _p(al), n, _p(bh), _p(bl), m, ld, _p(an), _p(bn), _p(Kx), ldm,
                   *kargs, _p(nonfinite), _stream())
        lab = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.int32)).to(dev)
        cnt = torch.zeros(k + 2, dtype=torch.float64, device=dev)
        L.call("pcb_count_labels", _p(lab), None, n, k, 0, _p(cnt), None, _stream())
        offsets = torch.empty(k + 1, dtype=torch.int32, device=dev)
        cursor = torch.empty(k, dtype=torch.int32, device=dev)
        perm = torch.empty(n, dtype=torch.int32, device=dev)
        L.call("pcb_sort_by_label", _p(lab), n, k, _p(cnt), _p(offsets), _p(cursor), _p(perm), None, _stream())
        S = torch.empty((k, ldm), dtype=torch.float64, device=dev)
        L.call(f"pcb_kk_segment_sums_{sfx}", _p(Kx), ldm, n, m, _p(perm), _p(offsets), k, _p(S), ldm, None,
               _stream())
        sz = torch.from_numpy(np.ascontiguousarray(sizes, dtype=np.float64)).to(dev)
        cs = torch.from_numpy(np.ascontiguousarray(cself, dtype=np.float64)).to(dev)
        out = torch.empty(m, dtype=torch.int32, device=dev)
        L.call(f"pcb_kk_predict_{sfx}", _p(S), ldm, m, k, _p(sz), _p(cs), _p(bn), *kargs, _p(out), _stream())
        if int(nonfinite.item()) != 0:
            raise FloatingPointError(f"kernel_matrix_between[{spec.family}] produced non-finite values")
        return out.cpu().numpy()
