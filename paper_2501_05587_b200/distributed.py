"""Row-sharded multi-GPU Lloyd: one process per GPU, NCCL over NVLink.

Points are split into contiguous row ranges (global index = rank offset +
local index, so the reference's lowest-index tie breaks stay global).
Centroids are replicated.  Each iteration exchanges exactly one buffer: the
fused f64 accumulator [sums k*d | counts k | objective | changed]
(8*(k*(d+1)+2) bytes: 1.06 MB at n=10M/d=128/k=1024) with one in-place
``all_reduce(SUM)``; every rank then runs the identical finalize, so the
centroids stay bitwise identical across ranks.

Empty-cluster repair (clustering.py:111-139) needs global decisions; it is
rare (the first iterations) and host-orchestrated without costing the common
case a host round trip: after the all-reduce a device flag parks an
iteration whose global counts show an empty cluster, the host notices it a
couple of iterations later (ShardSequence.run_multi reads the state with a
lag), and the batched protocol below runs one all_gather + one all_reduce per
pass of the reference's repair loop.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .clustering import ClusteringResult, KKMeansConfig, TimingBreakdown
from .validation import normalize_dtype


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def shard_range(n: int, rank: int, world: int):
    """Contiguous, balanced row range of `rank` (first n % world ranks get one more)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


class Comm:
    """torch.distributed plumbing used by the engine (NCCL on GPU, gloo in CPU tests)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world_size = dist.get_world_size(group) if dist.is_initialized() else 1
        self.offset = 0
        # the multi-rank protocol (collectives, device empty-cluster flags, host
        # repair rounds) runs for world_size > 1; PCB_FORCE_MULTI=1 runs it on a
        # single rank too (diagnostics: NCCL + graph capture on a 1-GPU box)
        self.multi = self.world_size > 1 or os.environ.get("PCB_FORCE_MULTI", "0") == "1"

    def all_reduce_sum(self, t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def all_reduce_max(self, t):
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)

    def all_gather(self, t):
        out = [torch.empty_like(t) for _ in range(self.world_size)]
        dist.all_gather(out, t, group=self.group)
        return out

    def barrier(self):
        dist.barrier(group=self.group)



REPAIR_BATCH = 4096  # repair.cu RP_BATCH: selections per round


def repair_protocol(ops, comm, prev, new) -> None:
    """Global empty-cluster repair across ranks (clustering.py:111-139), batched.

    Same semantics as the single-rank kernel (repair.cu): passes over the
    clusters empty at the start of each pass, ascending; the e-th of them
    receives the e-th unmoved point in (own distance desc, global index asc)
    order.  Every rank holds the same all-reduced accumulator, hence the same
    empty set.  One round per pass (per 4096 empties): each rank ranks its E
    best unmoved points on the device (pcb_repair_select), the keys are
    all-gathered and merged on the host (the global top-E is among the
    per-rank top-E lists), each owner applies its moves and writes their delta
    records into its slots of a zeroed E x (d+4) buffer, one all-reduce
    completes the buffer, and every rank commits all E records in slot order.
    Runs only when a cluster is globally empty (the iteration parked itself,
    ShardSequence.run_multi).
    """
    k, d = ops.k, ops.d
    kd = k * d
    if int(ops.state[1]) != 0:  # stopped (converged): nothing to repair
        return
    while True:
        counts = ops.acc[kd:kd + k]
        empties = torch.nonzero(counts == 0).flatten().tolist()  # host read, rare path
        if not empties:
            return
        for c0 in range(0, len(empties), REPAIR_BATCH):
            J = empties[c0:c0 + REPAIR_BATCH]
            E = len(J)
            keys = ops.repair_select(comm.offset, E)                      # (E, 3) on the device
            allk = torch.stack(comm.all_gather(keys)).cpu().numpy()       # (world, E, 3)
            flat = allk.reshape(-1, 3)
            owner = np.repeat(np.arange(allk.shape[0]), E)
            order = np.lexsort((flat[:, 1], -flat[:, 0]))[:E]             # own desc, global index asc
            mine = [(e, int(flat[i, 2])) for e, i in enumerate(order) if owner[i] == comm.rank]
            deltas = ops.new_deltas(E)
            if mine:
                ops.repair_apply_batch(prev, new, [q for _, q in mine], [J[e] for e, _ in mine],
                                       [e for e, _ in mine], deltas)
            comm.all_reduce_sum(deltas)
            ops.repair_commit_batch(J, deltas)


def run_lloyd_sharded(points_local, cfg: KKMeansConfig, n_total: int, offset: int,
                      comm: Comm | None = None) -> ClusteringResult:
    """Lloyd over a row shard; every rank returns the same global history/centroids
    and its own shard's labels.  Init labels are the reference's global
    PCG64 stream (clustering.py:91-108), sliced to the shard."""
    from .engine import LloydEngine

    comm = comm or Comm()
    comm.offset = offset
    cfg.validate_for(n_total)
    dtype = normalize_dtype(cfg.dtype)
    eng = LloydEngine(points_local, cfg.k, dtype=dtype, device=cfg.device, variant=cfg.variant,
                      comm=comm, n_total=n_total, max_iters=cfg.max_iters)
    eng.init_labels_device(cfg.seed, offset)  # the global stream, sliced to this shard
    if cfg.init is None:
        eng.init_centroids_from_labels()
    else:
        eng.set_centroids(np.asarray(cfg.init))
    out = eng.run(cfg.max_iters, cfg.tol, cfg.check_convergence,
                  record_history=cfg.record_label_history)
    return ClusteringResult(labels=out.labels, iterations_run=out.iterations_run,
                            objective_history=out.objective_history, converged=out.converged,
                            timings=TimingBreakdown(0.0, out.distance_seconds, out.update_seconds),
                            label_history=out.label_history, repairs=out.repairs,
                            centroids=out.centroids)


def init_from_env(backend: str = "nccl"):
    """Initialise torch.distributed from torchrun's env (127.0.0.1 rendezvous)."""
    if dist.is_initialized():
        return
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group(backend=backend, rank=rank, world_size=world)
