"""Device-resident Lloyd engine: buffers, kernel sequencing, collectives.

One ``LloydEngine`` owns one rank's row shard of the points for one fit.
Per iteration it enqueues, on the current CUDA stream and with no host
synchronisation:

    acc <- 0                                   fused f64 accumulator
    assign      (labels, mind, counts, objective, changed)   clustering.py:310-311, 146-149
    sort_by_label + segment_sums (per-cluster f64 row sums)  clustering.py:282-288
    [all_reduce(acc) over NCCL when world_size > 1]
    repair      (empty clusters, on device; no-op normally)  clustering.py:111-139
    finalize    (centroids, cnorm, history, convergence)     clustering.py:316-324

Every kernel checks the device stop flag, so ``check_convergence`` costs no
host round trip; the host syncs once at the end of the fit.  PyTorch is used
only for device memory, streams, pinned host buffers and torch.distributed.
"""
from __future__ import annotations

import ctypes
import os
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

_F32 = np.dtype(np.float32)
_F64 = np.dtype(np.float64)


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_STAGING = {}  # device index -> (pinned buffers, events, copy stream)
_STAGE_CHUNK = 1 << 23  # elements per pinned staging buffer (32 MiB of f32)
_STAGE_BUFS = 4         # measured on the B200 host: 4 x 32 MiB reach ~45 GB/s (scripts/h2d_probe.py)


def _staging(dev: torch.device, dtype: torch.dtype):
    """The device's pinned staging buffers viewed as `dtype` (one set per
    element size: int32 labels reuse the f32 buffers of the point upload)."""
    isz = torch.empty(0, dtype=dtype).element_size()
    key = (dev.index, isz)
    if key not in _STAGING:
        bufs = [torch.empty(_STAGE_CHUNK * isz, dtype=torch.uint8, pin_memory=True) for _ in range(_STAGE_BUFS)]
        _STAGING[key] = (bufs, [torch.cuda.Event() for _ in range(_STAGE_BUFS)], torch.cuda.Stream(dev))
    bufs, evs, cs = _STAGING[key]
    return [b.view(dtype) for b in bufs], evs, cs


def h2d_staged(host: np.ndarray, dev: torch.device) -> torch.Tensor:
    """Host (pageable numpy) -> device copy through reusable pinned staging
    buffers on a side stream: the (multi-threaded) CPU memcpy of chunk i+1
    overlaps the DMA of chunk i, and no per-call pinned allocation of the whole
    array is needed (pageable cudaMemcpy: ~11 GB/s; this: ~45 GB/s)."""
    src = torch.from_numpy(host)
    flat = src.view(-1)
    out = torch.empty(tuple(host.shape), dtype=src.dtype, device=dev)
    if flat.numel() <= _STAGE_CHUNK:
        out.copy_(src)
        return out
    bufs, evs, cs = _staging(dev, src.dtype)
    dflat = out.view(-1)
    cs.wait_stream(torch.cuda.current_stream(dev))
    for i, off in enumerate(range(0, flat.numel(), _STAGE_CHUNK)):
        b = i % len(bufs)
        evs[b].synchronize()            # the DMA that last read this buffer is done
        m = min(_STAGE_CHUNK, flat.numel() - off)
        bufs[b][:m].copy_(flat[off:off + m])
        with torch.cuda.stream(cs):
            dflat[off:off + m].copy_(bufs[b][:m], non_blocking=True)
            evs[b].record(cs)
    torch.cuda.current_stream(dev).wait_stream(cs)
    return out


def d2h_staged(src: torch.Tensor) -> np.ndarray:
    """Device -> host (numpy) copy through the same reusable pinned staging
    buffers: the DMA of chunk i+1 overlaps the CPU copy of chunk i out of
    pinned memory (a plain .cpu() of a large tensor lands in pageable memory
    at a fraction of the bus rate)."""
    src = src.contiguous()
    flat = src.view(-1)
    if flat.numel() <= _STAGE_CHUNK:
        return src.cpu().numpy()
    dev = src.device
    out = np.empty(tuple(src.shape), dtype=torch.empty(0, dtype=src.dtype).numpy().dtype)
    oflat = torch.from_numpy(out).view(-1)
    bufs, evs, cs = _staging(dev, src.dtype)
    cs.wait_stream(torch.cuda.current_stream(dev))
    chunks = list(range(0, flat.numel(), _STAGE_CHUNK))
    def issue(i):
        b = i % len(bufs)
        off = chunks[i]
        m = min(_STAGE_CHUNK, flat.numel() - off)
        with torch.cuda.stream(cs):
            bufs[b][:m].copy_(flat[off:off + m], non_blocking=True)
            evs[b].record(cs)
    for i in range(min(len(bufs), len(chunks))):
        issue(i)
    for i, off in enumerate(chunks):
        b = i % len(bufs)
        m = min(_STAGE_CHUNK, flat.numel() - off)
        evs[b].synchronize()
        oflat[off:off + m].copy_(bufs[b][:m])
        if i + len(bufs) < len(chunks):
            issue(i + len(bufs))
    return out


def require_cuda(device=None) -> torch.device:
    """The CUDA device to run on; RuntimeError if there is none (no CPU fallback)."""
    L.load()
    if not torch.cuda.is_available():
        raise RuntimeError("popcorn_b200 needs a CUDA sm_100 device; none is available "
                           "(there is no CPU fallback)")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       torch.device(device).index or 0)
    sm, mj, mn = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = L.load().pcb_device_info(dev.index, ctypes.byref(sm), ctypes.byref(mj), ctypes.byref(mn))
    if rc != 0:
        raise RuntimeError(f"device {dev} is sm_{mj.value}{mn.value}; popcorn_b200 is built for sm_100a")
    return dev


def resolve_variant(variant: str, dtype: np.dtype, d: int, k: int = 1) -> str:
    if variant not in L.VARIANTS:
        raise ValueError(f"unknown assign variant {variant!r}; expected one of {tuple(L.VARIANTS)}")
    if variant != "auto":
        if dtype == _F64 and variant in ("tc3xtf32", "delta", "deltatc", "tc1xtf32s", "bf16s", "fp8s"):
            raise ValueError(f"variant {variant!r} is float32-only")
        dmax = 1024 if variant == "fp8s" else 512  # 8 operand chunks of 128 bytes
        if variant in ("bf16s", "fp8s") and (d > dmax or k > SCREEN_KMAX):
            raise ValueError(f"variant {variant!r} needs d <= {dmax} and k <= {SCREEN_KMAX}")
        if variant == "rowreg" and d > 32:
            raise ValueError("variant 'rowreg' needs d <= 32")
        if variant == "tc1xtf32s" and k > SCREEN_KMAX:
            raise ValueError(f"variant 'tc1xtf32s' supports k <= {SCREEN_KMAX}")
        return variant
    if d <= 32:
        return "rowreg"
    if dtype != _F32:
        return "tiled"
    if k > SCREEN_KMAX:
        return "tc3xtf32"
    if d > 1024:
        return "tc1xtf32s"
    # E4M3 operands: half the bytes and twice the tensor rate of BF16 (rows of
    # d <= 64 use 64-byte SWIZZLE_64B chunks); the certificate keeps labels exact
    return "fp8s"


SCREEN_KMAX = 6144  # assign_screen.cu SC_KMAX


class HistoryRing:
    """label_history of an eager single-rank fit (clustering.py:320): iteration
    t's labels go D2H into pinned slot t % R and the host copies that slot into
    the result array R iterations later, while the GPU runs ahead, so only R
    rows are pinned — pinning the whole (max_iters x n) staging buffer costs
    ~0.7 s per GB the first time (c3: 1.2 GB)."""

    def __init__(self, n: int, max_iters: int, slots: int = 4):
        self.out = np.empty((max_iters, n), dtype=np.int32)
        self.pin = torch.empty((slots, n), dtype=torch.int32, pin_memory=True)
        self.ev = [None] * slots
        self.pending: list = []

    def push(self, t: int, labels: torch.Tensor) -> None:
        s = t % len(self.ev)
        if self.ev[s] is not None:
            self._drain()
        self.pin[s].copy_(labels, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.ev[s] = ev
        self.pending.append(t)

    def _drain(self) -> None:
        t = self.pending.pop(0)
        s = t % len(self.ev)
        self.ev[s].synchronize()
        torch.from_numpy(self.out[t]).copy_(self.pin[s])
        self.ev[s] = None

    def finish(self, iters: int) -> list:
        while self.pending:
            self._drain()
        return list(self.out[:iters])


@dataclass
class RunOutput:
    iterations_run: int
    converged: bool
    objective_history: np.ndarray
    repairs: np.ndarray
    labels: np.ndarray
    label_history: list
    centroids: np.ndarray
    distance_seconds: float
    update_seconds: float


def init_labels(n: int, k: int, seed: int, device=None, out=None, hollow_fill: bool = True) -> torch.Tensor:
    """Generator(PCG64(seed)).integers(0, k, size=n) on the device as int32,
    followed (hollow_fill) by init_assignments' empty-cluster fill
    (clustering.py:91-108); bit-identical to numpy (init.cu)."""
    seed = int(seed)
    if seed < 0 or seed >= 1 << 64:
        raise ValueError(f"seed must be a non-negative integer below 2**64, got {seed}")
    if hollow_fill and not 1 <= k <= n:
        raise ValueError(f"k must satisfy 1 <= k <= n, got k={k}, n={n}")
    dev = require_cuda(device)
    with torch.cuda.device(dev):
        lab = out if out is not None else torch.empty(n, dtype=torch.int32, device=dev)
        sb = int(L.load().pcb_init_scratch_bytes(n, k))
        scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
        if hollow_fill:
            passes = ctypes.c_int(0)
            L.call("pcb_init_assignments", n, k, seed, _p(lab), _p(scratch), sb, ctypes.byref(passes), _stream())
        else:
            L.call("pcb_bounded_draws", n, k, seed, _p(lab), _p(scratch), sb, _stream())
    return lab


class ShardSequence:
    """The per-rank Lloyd iteration, independent of where the numbers live.

    Subclasses provide the numeric steps (`_assign`, `_sort_and_sum`,
    `_repair_local`, `_finalize`) and the multi-rank primitives
    (`flag_pending`, `restore_pending`, `snapshot_state` / `read_snapshot`,
    `repair_select`, `new_deltas`, `repair_apply_batch`,
    `repair_commit_batch`); the order of operations, the single all-reduce of
    the fused accumulator, the lagged multi-rank loop and the global repair
    protocol live here once, shared by the CUDA engine and the CPU test
    double used by the gloo tests.
    Attributes used: labels[2], acc, state, k, d, comm.
    """

    comm = None

    def iteration(self, t: int, check_convergence: bool = False, tol: float = 0.0,
                  events=None, raw_out=None) -> None:
        """One Lloyd iteration t (reads labels[t%2], writes labels[(t+1)%2]).

        events: optional CUDA events [assign start, assign end, iteration end]
        plus, optionally, [dominant kernel start, dominant kernel end] (recorded
        on the launching stream around the distance+argmin kernel itself).
        """
        prev, new = self.labels[t % 2], self.labels[(t + 1) % 2]
        self._kev = events[3:5] if events is not None and len(events) >= 5 else None
        self.acc.zero_()
        if events is not None:
            events[0].record()
        self._assign(prev, new, self.acc, self.state)           # clustering.py:310-311, 146-149
        if events is not None:
            events[1].record()
        self._update(prev, new)                                 # clustering.py:282-288, 148
        self._after_update(t)
        self._allreduce(self.acc)                               # the one collective per iteration
        if raw_out is not None:
            raw_out.copy_(new)
        if self._multi():
            # a globally empty cluster parks the iteration (state[1] = 2) for the
            # host's repair protocol; no host round trip when none is empty
            self.flag_pending()
        else:
            self._repair_local(prev, new)                       # clustering.py:111-139
        self._finalize(check_convergence, tol)                  # clustering.py:316-324
        if events is not None:
            events[2].record()

    def _multi(self) -> bool:
        return self.comm is not None and self.comm.multi

    # -- multi-rank fit: enqueue ahead, check the repair flag with a lag -----------
    PENDING = 2  # state[1] value of an iteration parked for the host repair

    def run_multi(self, max_iters: int, check_convergence: bool = False, tol: float = 0.0,
                  make_events=None, hist=None, lag: int = 2, t0: int = 0) -> dict:
        """Iterations 0 .. max_iters-1 across ranks with no host synchronisation
        per iteration: each iteration is enqueued, then the device state of the
        iteration `lag` back is read (pinned copy + event).  Empty clusters are
        rare (the first iterations); an iteration that needs the repair parks
        itself on the device, every iteration enqueued after it returns at once,
        and when the host sees the flag it restores the accumulator, runs the
        batched protocol (distributed.repair_protocol) and the finalize, and
        resumes from the next iteration.  Every rank holds the same all-reduced
        accumulator, so every rank takes the same branch at the same iteration.
        Iterations t0 .. max_iters-1; returns {t: events}."""
        from collections import deque
        evs = {}
        queue = deque()
        t = t0
        while t < max_iters:
            ev = make_events() if make_events is not None else None
            self.iteration(t, check_convergence, tol, ev)
            if hist is not None:
                hist[t].copy_(self.labels[(t + 1) % 2], non_blocking=True)
            evs[t] = ev
            queue.append((t, self.snapshot_state()))
            t += 1
            while queue and (len(queue) > lag or t >= max_iters):
                tq, snap = queue.popleft()
                flag = int(self.read_snapshot(snap)[1])
                if flag == self.PENDING:
                    self.resume_after_repair(tq, check_convergence, tol)
                    if hist is not None:
                        hist[tq].copy_(self.labels[(tq + 1) % 2], non_blocking=True)
                    t = tq + 1
                    queue.clear()
                elif flag != 0:  # converged: the rest are no-ops
                    t = max_iters
                    queue.clear()
        return evs

    def resume_after_repair(self, t: int, check_convergence: bool, tol: float) -> None:
        from .distributed import repair_protocol
        prev, new = self.labels[t % 2], self.labels[(t + 1) % 2]
        self.restore_pending()
        repair_protocol(self, self.comm, prev, new)
        self._finalize(check_convergence, tol)

    def _update(self, prev, new) -> None:
        self._sort_and_sum(new, self.state)

    def _after_update(self, t: int) -> None:
        pass

    def _allreduce(self, t) -> None:
        if self.comm is not None and self.comm.multi:
            self.comm.all_reduce_sum(t)


class LloydEngine(ShardSequence):
    """One rank's shard: P (n_local x d) resident in HBM, centroids replicated."""

    def __init__(self, points, k: int, *, dtype=np.float32, device=None, variant: str = "auto",
                 comm=None, n_total: int | None = None, max_iters: int = 30,
                 check_finite: bool = False, update: str = "auto"):
        if update not in ("auto", "full"):
            raise ValueError(f"update must be 'auto' or 'full', got {update!r}")
        self.dev = require_cuda(device)
        self.dtype = np.dtype(dtype)
        self.tdtype = torch.float32 if self.dtype == _F32 else torch.float64
        self.sfx = "f32" if self.dtype == _F32 else "f64"
        self.comm = comm
        with torch.cuda.device(self.dev):
            if isinstance(points, torch.Tensor):
                P = points.to(device=self.dev, dtype=self.tdtype).contiguous()
            else:
                P = h2d_staged(np.ascontiguousarray(points, dtype=self.dtype), self.dev)
            self.P = P
            if check_finite:
                # validation.py:45-46 on the device: ValueError like the reference
                cnt = torch.zeros(1, dtype=torch.int64, device=self.dev)
                L.call(f"pcb_count_nonfinite_{self.sfx}", _p(P), P.numel(), _p(cnt), _stream())
                if int(cnt.item()) != 0:
                    raise ValueError("points contains non-finite entries")
            self.n, self.d = int(P.shape[0]), int(P.shape[1])
            self.k = int(k)
            assert self.k >= 1
            self.n_total = int(n_total if n_total is not None else self.n)
            self.variant = resolve_variant(variant, self.dtype, self.d, self.k)
            self.vcode = L.VARIANTS[self.variant]
            n, d, kk = self.n, self.d, self.k
            dev, td = self.dev, self.tdtype
            self.pnorm = torch.empty(n, dtype=td, device=dev)
            # centroids and their norms in one allocation (C rows, then cnorm):
            # the small-d kernel copies both into the constant bank in one copy
            self._cbuf = torch.zeros(kk * d + kk, dtype=td, device=dev)
            self.C = self._cbuf[: kk * d].view(kk, d)
            self.cnorm = self._cbuf[kk * d:]
            self.labels = [torch.zeros(n, dtype=torch.int32, device=dev) for _ in range(2)]
            self.mind = torch.empty(n, dtype=td, device=dev)
            self.acc_size = kk * d + kk + 2
            self.acc = torch.zeros(self.acc_size, dtype=torch.float64, device=dev)
            # multi-rank: the accumulator of an iteration parked for the host repair
            self.acc_saved = torch.zeros_like(self.acc) if comm is not None and comm.multi else None
            self.perm = torch.empty(n, dtype=torch.int32, device=dev)
            self.own = torch.empty(n, dtype=torch.float64, device=dev)  # own distances, sorted order
            self.offsets = torch.empty(kk + 1, dtype=torch.int32, device=dev)
            self.cursor = torch.empty(kk, dtype=torch.int32, device=dev)
            self.state = torch.zeros(L.STATE_WORDS, dtype=torch.int64, device=dev)
            self.max_iters = max(1, int(max_iters))
            self.obj_hist = torch.zeros(self.max_iters, dtype=torch.float64, device=dev)
            self.rep_hist = torch.zeros(self.max_iters, dtype=torch.int64, device=dev)
            sb = int(L.load().pcb_repair_scratch_bytes(kk))
            self.repair_scratch = torch.empty(sb, dtype=torch.uint8, device=dev)
            self.repair_scratch_bytes = sb
            # delta centroid update (update.cu): persistent local sums S, Q = sum |p|^2
            self.delta_frac = float(os.environ.get("PCB_DELTA_FRAC", "0.05")) if update == "auto" else -1.0
            self.S = torch.zeros(kk * d, dtype=torch.float64, device=dev)
            self.Q = torch.zeros(1, dtype=torch.float64, device=dev)
            self.sums_valid = False
            # split operands for the tensor-core path
            self.ld = 0
            self.P_hi = self.P_lo = self.C_hi = self.C_lo = None
            L.call(f"pcb_point_norms_{self.sfx}", _p(self.P), n, d, _p(self.pnorm), _stream())
            L.call(f"pcb_sum_squares_{self.sfx}", _p(self.P), n * d, _p(self.Q), _stream())
            if self.variant in ("tc3xtf32", "tc1xtf32s", "bf16s", "fp8s"):
                self.ld = (d + 31) // 32 * 32
                self.C_hi = torch.zeros((kk, self.ld), dtype=torch.float32, device=dev)
                self.C_lo = torch.zeros((kk, self.ld), dtype=torch.float32, device=dev)
            if self.variant == "deltatc":
                # delta-chunked ablation on the tensor cores: augmented Q = [1, p] and the
                # centroids' first block column / row (F, G), all split hi/lo (assign_delta_tc.cu)
                self.ldq = int(L.load().pcb_delta_tc_ld(d))
                self.Q_hi = torch.empty((n, self.ldq), dtype=torch.float32, device=dev)
                self.Q_lo = torch.empty((n, self.ldq), dtype=torch.float32, device=dev)
                brows = 8 * int(L.load().pcb_delta_tc_kpad(kk))
                self.FG = [torch.zeros((brows, self.ldq), dtype=torch.float32, device=dev) for _ in range(4)]
                L.call("pcb_delta_tc_prep_points", _p(self.P), n, d, self.ldq, _p(self.Q_hi), _p(self.Q_lo),
                       _stream())
            if self.variant == "tc3xtf32":
                self.P_hi = torch.empty((n, self.ld), dtype=torch.float32, device=dev)
                self.P_lo = torch.empty((n, self.ld), dtype=torch.float32, device=dev)
                L.call("pcb_split_tf32", _p(self.P), n, d, self.ld, _p(self.P_hi), _p(self.P_lo), _stream())
            if self.variant == "tc1xtf32s":
                # certified screening: raw P for the TF32 pass, compact hi/lo for the
                # ambiguous rows (capacity n), truncation norms for the error bound
                self.anorm = torch.empty(n, dtype=torch.float32, device=dev)
                self.danorm = torch.empty(n, dtype=torch.float32, device=dev)
                self.bnorm = torch.empty(kk, dtype=torch.float32, device=dev)
                self.dbnorm = torch.empty(kk, dtype=torch.float32, device=dev)
                self.bstat = torch.zeros(4, dtype=torch.float32, device=dev)
                self.amb_list = torch.empty(n, dtype=torch.int32, device=dev)
                self.amb_count = torch.zeros(1, dtype=torch.int32, device=dev)
                self.sub_hi = torch.empty((n, self.ld), dtype=torch.float32, device=dev)
                self.sub_lo = torch.empty((n, self.ld), dtype=torch.float32, device=dev)
                self.sub_labels = torch.empty(n, dtype=torch.int32, device=dev)
                self.flag_list = torch.empty(n, dtype=torch.int32, device=dev)
                self.flag_count = torch.zeros(1, dtype=torch.int32, device=dev)
                self.exact_scratch = torch.empty(int(L.load().pcb_exact_scratch_bytes()), dtype=torch.uint8,
                                                 device=dev)
                self.P_r = torch.empty((n, self.ld), dtype=torch.float32, device=dev)
                L.call("pcb_screen_prep_points", _p(self.P), n, d, self.ld, _p(self.P_r), _p(self.anorm),
                       _p(self.danorm), _p(self.bstat), _stream())
            if self.variant in ("bf16s", "fp8s"):
                # certified BF16 screening: RN BF16 copy of P, the bound's residual
                # norms, pass-2 buffers for the ambiguous rows (capacity n) and the
                # 3xTF32 resolver's compact hi/lo for rows with too many candidates
                # operand rows: BF16 (ldb elements) or E4M3 (ld8 bytes); ldb is the
                # row length in BF16 units either way (what the tensor maps see)
                self.q8 = self.variant == "fp8s"
                if self.q8:
                    self.ld8 = int(L.load().pcb_screen_fp8_ld(d))
                    self.ldb = self.ld8 // 2
                else:
                    self.ldb = int(L.load().pcb_screen_bf16_ld(d))
                ncand = int(L.load().pcb_screen_bf16_ncand())
                self.P_b = torch.empty((n, self.ldb), dtype=torch.bfloat16, device=dev)  # E4M3 bytes when q8
                kpad = int(L.load().pcb_screen_bf16_kpad(kk))
                self.C_b = torch.zeros((kpad, self.ldb), dtype=torch.bfloat16, device=dev)
                self.C_aug = torch.zeros((kpad, int(L.load().pcb_screen_bf16_aug())), dtype=torch.bfloat16,
                                         device=dev)
                self.anorm = torch.empty(n, dtype=torch.float32, device=dev)
                self.danorm = torch.empty(n, dtype=torch.float32, device=dev)
                self.bnorm = torch.empty(kk, dtype=torch.float32, device=dev)
                self.dbnorm = torch.empty(kk, dtype=torch.float32, device=dev)
                self.bstat = torch.zeros(16, dtype=torch.float32, device=dev)
                self.amb_list = torch.empty(n, dtype=torch.int32, device=dev)
                self.ctr = torch.zeros(2, dtype=torch.int32, device=dev)  # [ambiguous, two-candidate] rows
                self.amb_count = self.ctr[0:1]
                self.amb_thr = torch.empty(n, dtype=torch.float32, device=dev)
                self.two_list = torch.empty(3 * n, dtype=torch.int32, device=dev)  # (row, r1, r2)
                self.two_count = self.ctr[1:2]
                self.sub_b = torch.empty((n, self.ldb), dtype=torch.bfloat16, device=dev)
                self.bypass = max(n // 4, 1)  # more ambiguous rows: straight to 3xTF32
                self.cand = torch.empty((self.bypass, ncand), dtype=torch.int32, device=dev)
                self.cand_n = torch.empty(self.bypass, dtype=torch.int32, device=dev)
                self.ovf_list = torch.empty(n, dtype=torch.int32, device=dev)
                self.ovf_count = torch.zeros(1, dtype=torch.int32, device=dev)
                self.sub_hi = torch.empty((n, self.ld), dtype=torch.float32, device=dev)
                self.sub_lo = torch.empty((n, self.ld), dtype=torch.float32, device=dev)
                self.sub_labels = torch.empty(n, dtype=torch.int32, device=dev)
                self.flag_list = torch.empty(n, dtype=torch.int32, device=dev)
                self.flag_count = torch.zeros(1, dtype=torch.int32, device=dev)
                self.exact_scratch = torch.empty(int(L.load().pcb_exact_scratch_bytes()), dtype=torch.uint8,
                                                 device=dev)
                if self.q8:
                    L.call("pcb_screen_prep_points_fp8", _p(self.P), n, d, self.ld8, _p(self.P_b),
                           _p(self.anorm), _p(self.danorm), _p(self.bstat), _stream())
                else:
                    L.call("pcb_screen_prep_points_bf16", _p(self.P), n, d, self.ldb, _p(self.P_b),
                           _p(self.anorm), _p(self.danorm), _p(self.bstat), _stream())
                self.orig = None  # row layout of P_b / anorm / danorm (None = original order)

    # -- centroid initialisation ------------------------------------------------
    def set_centroids(self, C) -> None:
        """Fixed centroids (additive `init=`), replicated on every rank."""
        self._cold = False
        with torch.cuda.device(self.dev):
            Ct = torch.as_tensor(np.ascontiguousarray(C, dtype=self.dtype).reshape(self.k, self.d))
            self.C.copy_(Ct.to(self.dev))
            self._centroid_norms()

    # Iterations after whose update the bf16 screen's rows are re-laid out by
    # label (the counting sort of that update): labels settle within a few
    # iterations, and a stale layout only costs epilogue skips, never results.
    RELAYOUT_AT = tuple(int(x) for x in os.environ.get("PCB_RELAYOUT_AT", "1,3").split(",") if x)

    def _after_update(self, t: int) -> None:
        if self.variant in ("bf16s", "fp8s") and t in self.RELAYOUT_AT:
            self.relayout()

    # the screen's row layout state (relayout swaps these)
    _LAYOUT_ATTRS = ("orig", "P_b", "anorm", "danorm", "P_b0", "an0", "dan0")

    def relayout(self) -> None:
        """Rebuild P_b / anorm / danorm in the label order of the last update's
        counting sort (self.perm); see pcb_screen_relayout_bf16."""
        if self.orig is None:
            self.orig = torch.empty(self.n, dtype=torch.int32, device=self.dev)
            self.P_b0, self.an0, self.dan0 = self.P_b, self.anorm, self.danorm  # original-order copies
            self.P_b = torch.empty_like(self.P_b0)
            self.anorm = torch.empty_like(self.an0)
            self.danorm = torch.empty_like(self.dan0)
        L.call("pcb_screen_relayout_bf16", _p(self.P_b0), _p(self.an0), _p(self.dan0), self.n, self.ldb,
               _p(self.perm), _p(self.P_b), _p(self.anorm), _p(self.danorm), _p(self.orig), _stream())

    def _screen_centroid_stats(self) -> None:
        if self.variant in ("bf16s", "fp8s"):
            L.call("pcb_screen_prep_centroids_fp8" if self.q8 else "pcb_screen_prep_centroids_bf16", _p(self.C),
                   _p(self.cnorm), self.k, self.d, self.ld8 if self.q8 else self.ldb, _p(self.C_b), _p(self.C_aug),
                   _p(self.bnorm), _p(self.dbnorm), _p(self.bstat), _stream())
        if self.variant == "deltatc":
            L.call("pcb_delta_tc_prep_centroids", _p(self.C), _p(self.cnorm), self.k, self.d, self.ldq,
                   *[_p(t) for t in self.FG], _stream())
        if self.variant == "tc1xtf32s":
            L.call("pcb_screen_prep_centroids", _p(self.C), self.k, self.d, _p(self.bnorm),
                   _p(self.dbnorm), _p(self.bstat), _stream())

    def _centroid_norms(self) -> None:
        if self.dtype == _F32:
            L.call("pcb_centroid_norms_f32", _p(self.C), self.k, self.d, _p(self.cnorm),
                   _p(self.C_hi), _p(self.C_lo), self.ld, _stream())
            self._screen_centroid_stats()
        else:
            L.call("pcb_centroid_norms_f64", _p(self.C), self.k, self.d, _p(self.cnorm), _stream())

    def set_labels(self, labels_local: np.ndarray, counts_global: np.ndarray | None = None) -> None:
        """Labels of this shard (clustering.py:298); previous labels of iteration 1."""
        self.sums_valid = False
        with torch.cuda.device(self.dev):
            lab = torch.from_numpy(np.ascontiguousarray(labels_local, dtype=np.int32))
            self.labels[0].copy_(lab.to(self.dev))

    def init_labels_device(self, seed: int, offset: int = 0) -> None:
        """init_assignments (clustering.py:91-108) generated in HBM.

        The global label vector of all n_total points is drawn on this device
        (numpy's PCG64 stream, bit-identical; see init.cu) and this shard's
        rows [offset, offset + n) become the labels of iteration 0.
        """
        self.sums_valid = False
        with torch.cuda.device(self.dev):
            if self.n_total == self.n:
                init_labels(self.n, self.k, seed, self.dev, out=self.labels[0])
            else:
                full = init_labels(self.n_total, self.k, seed, self.dev)
                self.labels[0].copy_(full[offset:offset + self.n])

    def init_centroids_from_labels(self, labels_local: np.ndarray | None = None) -> None:
        """Initial means over the init labels (clustering.py:298-300), on device.

        labels_local: this shard's init labels on the host; None = the labels
        already on the device (init_labels_device).
        """
        if labels_local is not None:
            self.set_labels(labels_local)
        with torch.cuda.device(self.dev):
            self.acc.zero_()
            L.call("pcb_count_labels", _p(self.labels[0]), None, self.n, self.k, self.d, _p(self.acc), None,
                   _stream())
            self._sort_and_sum(self.labels[0], None)
            self._allreduce(self.acc)
            if self.dtype == _F32:
                L.call("pcb_centroids_from_acc_f32", _p(self.acc), self.k, self.d, _p(self.C),
                       _p(self.cnorm), _p(self.C_hi), _p(self.C_lo), self.ld, _stream())
                self._screen_centroid_stats()
            else:
                L.call("pcb_centroids_from_acc_f64", _p(self.acc), self.k, self.d, _p(self.C),
                       _p(self.cnorm), _stream())
        # means of random labels all sit near the global mean: the next assignment
        # goes straight to 3xTF32 (see _assign)
        self._cold = self.variant in ("bf16s", "fp8s") and os.environ.get("PCB_COLD_START", "1") != "0"

    # -- building blocks ---------------------------------------------------------
    def _sort_and_sum(self, labels, state) -> None:
        counts = self.acc[self.k * self.d:]
        L.call("pcb_sort_by_label", _p(labels), self.n, self.k, _p(counts), _p(self.offsets),
               _p(self.cursor), _p(self.perm), _p(state), _stream())
        L.call(f"pcb_segment_sums_{self.sfx}", _p(self.P), self.n, self.d, _p(self.perm),
               _p(self.offsets), self.k, _p(self.C), _p(self.own), _p(self.acc), _p(state), _stream())

    def _update(self, prev, new) -> None:
        """Centroid sums of the new labels: full counting sort + segmented sums,
        or the delta update over the changed rows (decided on the device,
        pcb_update_mode; see update.cu)."""
        if self.delta_frac < 0:
            self._sort_and_sum(new, self.state)
            return
        L.call("pcb_update_mode", _p(self.acc), self.k, self.d, self.n, self.delta_frac,
               int(not self.sums_valid), _p(self.state), _stream())
        self._sort_and_sum(new, self.state)  # no-ops in delta mode
        L.call(f"pcb_delta_update_{self.sfx}", _p(self.P), self.n, self.d, _p(prev), _p(new), _p(self.C),
               self.k, _p(self.S), _p(self.Q), _p(self.acc), _p(self.state), _stream())
        self.sums_valid = True

    _cold = False

    def _assign(self, prev, new, acc, state) -> None:
        if self.variant in ("bf16s", "fp8s") and self._cold:
            # First assignment after the random init (clustering.py:298-300): every
            # centroid is a mean of ~n/k random rows, near the global mean, and the
            # low-precision screen certifies almost no row (100 % ambiguous at c3),
            # so its resolver would bypass to 3xTF32 for every row anyway.  Run that
            # resolver on all rows directly (identity list) and skip the screen.
            self._cold = False
            torch.arange(self.n, dtype=torch.int32, device=self.dev, out=self.ovf_list)
            self.ovf_count.fill_(self.n)
            self._kmark(0)
            self._resolve(self.ovf_list, self.ovf_count, new, state)
            self._kmark(1)
            if acc is not None:
                self._count_labels(new, prev, acc, state)
            return
        if self.variant in ("bf16s", "fp8s"):
            self.ctr.zero_()  # both counters, one fill
            self._kmark(0)
            ldq = self.ld8 if self.q8 else self.ldb
            L.call("pcb_assign_screen_fp8" if self.q8 else "pcb_assign_screen_bf16", _p(self.P_b), self.n, ldq,
                   _p(self.C_b), self.k,
                   _p(self.C_aug), _p(self.anorm), _p(self.danorm), _p(self.bstat), _p(new),
                   _p(self.amb_list), _p(self.amb_count), _p(self.amb_thr), _p(self.orig), _p(prev),
                   _p(self.two_list), _p(self.two_count), _p(state), _stream())
            self._kmark(1)
            L.call("pcb_resolve_screen_fp8" if self.q8 else "pcb_resolve_screen_bf16", _p(self.P), self.n,
                   self.d, _p(self.P_b), ldq,
                   _p(self.C_b), _p(self.C), self.k, _p(self.C_aug), _p(self.bstat), _p(self.amb_list),
                   _p(self.amb_count), _p(self.amb_thr), self.bypass, _p(self.sub_b), _p(self.cand),
                   _p(self.cand_n), _p(new), _p(self.ovf_list), _p(self.ovf_count), _p(self.orig),
                   _p(self.two_list), _p(self.two_count), _p(state), _stream())
            self._resolve(self.ovf_list, self.ovf_count, new, state)
            if acc is not None:
                self._count_labels(new, prev, acc, state)
            return
        if self.variant == "tc1xtf32s":
            self.amb_count.zero_()
            self._kmark(0)
            L.call("pcb_assign_screen_f32", _p(self.P_r), self.n, self.ld, _p(self.C_hi), self.k,
                   _p(self.cnorm), _p(self.anorm), _p(self.danorm), _p(self.bstat), _p(new),
                   _p(self.amb_list), _p(self.amb_count), _p(state), _stream())
            self._kmark(1)
            self._resolve(self.amb_list, self.amb_count, new, state)
            if acc is not None:
                self._count_labels(new, prev, acc, state)
            return
        self._kmark(0)
        if self.variant == "deltatc":
            L.call("pcb_assign_delta_tc_f32", _p(self.Q_hi), _p(self.Q_lo), self.ldq, self.n, self.d,
                   *[_p(t) for t in self.FG], self.k, _p(prev), _p(new), _p(self.mind), _p(acc), _p(state),
                   _stream())
        elif self.variant == "tc3xtf32":
            L.call("pcb_assign_tc_f32", _p(self.P_hi), _p(self.P_lo), self.ld, _p(self.pnorm), self.n,
                   self.d, _p(self.C_hi), _p(self.C_lo), _p(self.cnorm), self.k, _p(prev), _p(new),
                   _p(self.mind), _p(acc), _p(state), _stream())
        else:
            if self.delta_frac >= 0 and self.dtype == _F32 and acc is not None:
                # the small-d kernel applies the changed rows to S itself (update mode 3)
                L.call("pcb_assign_spec_f32", _p(self.P), _p(self.pnorm), self.n, self.d, _p(self.C),
                       _p(self.cnorm), self.k, _p(prev), _p(new), _p(self.mind), _p(acc), _p(state),
                       _p(self.S), self.vcode, _stream())
            else:
                L.call(f"pcb_assign_{self.sfx}", _p(self.P), _p(self.pnorm), self.n, self.d, _p(self.C),
                       _p(self.cnorm), self.k, _p(prev), _p(new), _p(self.mind), _p(acc), _p(state),
                       self.vcode, _stream())
        self._kmark(1)

    def _count_labels(self, new, prev, acc, state) -> None:
        """counts / changed of the new labels (clustering.py:146-149); with the delta
        update on, fused with its changed-row sums when the previous iteration was a
        delta one (pcb_count_labels_delta_f32; delta_sums then has nothing left to do)."""
        if self.delta_frac >= 0 and self.dtype == _F32:
            L.call("pcb_count_labels_delta_f32", _p(new), _p(prev), self.n, self.k, self.d, _p(acc), _p(state),
                   _p(self.P), _p(self.S), _stream())
        else:
            L.call("pcb_count_labels", _p(new), _p(prev), self.n, self.k, self.d, _p(acc), _p(state), _stream())

    def _resolve(self, rows, count, new, state) -> None:
        """3xTF32 labels of the listed rows, made exact (pcb_resolve_ambiguous_f32
        with the flag list: near-ties re-evaluated over all centroids)."""
        L.call("pcb_resolve_ambiguous_f32", _p(self.P), self.n, self.d, _p(rows), _p(count), self.ld,
               _p(self.sub_hi), _p(self.sub_lo), _p(self.sub_labels), _p(self.pnorm), _p(self.C), _p(self.C_hi),
               _p(self.C_lo), _p(self.cnorm), self.k, _p(new), _p(self.flag_list), _p(self.flag_count),
               _p(self.exact_scratch), self.exact_scratch.numel(), _p(state), _stream())

    _kev = None

    def _kmark(self, i: int) -> None:
        if self._kev is not None:
            self._kev[i].record()

    def _repair_local(self, prev, new) -> None:
        L.call(f"pcb_repair_{self.sfx}", _p(self.P), self.n, self.d, _p(self.C), self.k, _p(self.perm),
               _p(prev), _p(new), _p(self.own), _p(self.acc), _p(self.state), _p(self.repair_scratch),
               self.repair_scratch_bytes, _p(self.S) if self.delta_frac >= 0 else None, _stream())

    def _finalize(self, check_convergence: bool, tol: float) -> None:
        if self.dtype == _F32:
            L.call("pcb_finalize_f32", _p(self.acc), self.k, self.d, self.n_total, _p(self.C),
                   _p(self.cnorm), _p(self.C_hi), _p(self.C_lo), self.ld, _p(self.obj_hist),
                   _p(self.rep_hist), _p(self.state), int(check_convergence), float(tol), _stream())
            self._screen_centroid_stats()
        else:
            L.call("pcb_finalize_f64", _p(self.acc), self.k, self.d, self.n_total, _p(self.C),
                   _p(self.cnorm), _p(self.obj_hist), _p(self.rep_hist), _p(self.state),
                   int(check_convergence), float(tol), _stream())

    # -- multi-rank repair primitives (distributed.repair_protocol) ---------------
    def flag_pending(self) -> None:
        L.call("pcb_flag_global_empty", _p(self.acc), self.k, self.d, _p(self.acc_saved), _p(self.state),
               _stream())

    def restore_pending(self) -> None:
        self.acc.copy_(self.acc_saved)
        self.state[1] = 0

    def snapshot_state(self):
        """Asynchronous copy of the loop state words (pinned) + its event."""
        if not hasattr(self, "_snap_ring"):
            self._snap_ring = torch.zeros((8, 2), dtype=torch.int64, pin_memory=True)
            self._snap_i = 0
        slot = self._snap_ring[self._snap_i % 8]
        self._snap_i += 1
        slot.copy_(self.state[:2], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return slot, ev

    @staticmethod
    def read_snapshot(snap):
        slot, ev = snap
        ev.synchronize()
        return slot.numpy().copy()

    def repair_select(self, offset: int, E: int):
        out = torch.empty((E, 3), dtype=torch.float64, device=self.dev)
        L.call("pcb_repair_select", _p(self.own), _p(self.perm), self.n, int(offset), int(E), _p(out),
               _p(self.repair_scratch), self.repair_scratch_bytes, _stream())
        return out

    def new_deltas(self, E: int):
        return torch.zeros((E, self.d + 4), dtype=torch.float64, device=self.dev)

    def repair_apply_batch(self, prev, new, pos, js, slots, deltas) -> None:
        t = torch.tensor([pos, js, slots], dtype=torch.int32).to(self.dev)
        L.call(f"pcb_repair_apply_batch_{self.sfx}", _p(self.P), self.d, _p(self.C), _p(self.perm), _p(prev),
               _p(new), _p(self.own), _p(t[0]), _p(t[1]), _p(t[2]), len(pos), _p(deltas), _stream())

    def repair_commit_batch(self, js, deltas) -> None:
        t = torch.tensor(js, dtype=torch.int32).to(self.dev)
        L.call("pcb_repair_commit_batch", _p(self.acc), self.k, self.d, len(js), _p(t), _p(deltas),
               _p(self.state), _stream())

    # -- whole fit -----------------------------------------------------------------
    def run(self, max_iters: int, tol: float = 0.0, check_convergence: bool = False,
            record_history: bool = True, timing: bool = True, graph: bool = True) -> RunOutput:
        """The whole fit.  Small single-rank fits are recorded once into a CUDA
        graph and replayed (every decision inside an iteration is taken on the
        device, and the host-side schedule — full update at the start,
        relayouts — is known in advance), which removes the launch gaps between
        the ~30 small kernels of an iteration; large fits are GPU-bound and run
        eagerly.  Multi-rank fits are enqueued ahead with a lagged check of the
        repair flag (run_multi): no host synchronisation per iteration."""
        if max_iters > self.max_iters:
            raise ValueError("max_iters exceeds the engine's history capacity")
        with torch.cuda.device(self.dev):
            self.state.zero_()
            # graphs pay off where launches dominate (small n k d); a large fit
            # is GPU-bound and instantiating ~1000 nodes would only add latency
            small = 2.0 * self.n * self.k * self.d < 1e11
            use_graph = graph and small and not self._multi()
            hist = None
            if record_history:
                # eager single-rank fits stream the history through a few pinned slots
                hist = (HistoryRing(self.n, max_iters) if not use_graph and not self._multi() else
                        torch.empty((max_iters, self.n), dtype=torch.int32, pin_memory=True))
            if self._multi():
                mk = (lambda: [torch.cuda.Event(enable_timing=True) for _ in range(3)]) if timing else None
                evd = self.run_multi(max_iters, check_convergence, tol, mk, hist)
                torch.cuda.current_stream().synchronize()
                return self.collect(hist, [evd[t] for t in sorted(evd)] if timing else ())
            evs = self.iterations(0, max_iters, check_convergence, tol, timing, hist, use_graph)
            torch.cuda.current_stream().synchronize()
            return self.collect(hist, evs)

    def iterations(self, t0: int, count: int, check_convergence: bool = False, tol: float = 0.0,
                   timing: bool = True, hist=None, graph: bool = True, nev: int = 3):
        """Iterations t0 .. t0+count-1, eagerly or as one captured CUDA graph
        (replayed once).  Returns the per-iteration timing events (nev each)."""
        def body(external):
            evs = []
            for t in range(t0, t0 + count):
                ev = ([torch.cuda.Event(enable_timing=True, external=external) for _ in range(nev)]
                      if timing else None)
                self.iteration(t, check_convergence, tol, ev)
                if ev is not None:
                    evs.append(ev)
                if isinstance(hist, HistoryRing):
                    hist.push(t, self.labels[(t + 1) % 2])
                elif hist is not None:
                    hist[t].copy_(self.labels[(t + 1) % 2], non_blocking=True)
            return evs
        if graph and not isinstance(hist, HistoryRing):
            saved, cold = self.sums_valid, self._cold
            # relayout() (captured at t in RELAYOUT_AT) swaps in new operand buffers whose
            # fill kernels only run on replay: keep the current ones to restore on failure
            layout = {a: getattr(self, a, None) for a in self._LAYOUT_ATTRS}
            try:
                g = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream(self.dev)
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
                    evs = body(True)
                torch.cuda.current_stream().wait_stream(cs)
                g.replay()
                self._graph = g  # kept alive until the next run (its nodes reference our buffers)
                return evs
            except RuntimeError as e:  # capture unsupported here: run the same kernels eagerly
                warnings.warn(f"CUDA graph capture failed ({e}); running the iterations eagerly")
                self.sums_valid, self._cold = saved, cold
                for a, v in layout.items():
                    setattr(self, a, v)
                self._graph = None
                torch.cuda.synchronize()
        return body(False)

    @staticmethod
    def _history_arrays(hist, iters: int) -> list:
        """label_history (clustering.py:320): one int32[n] array per iteration, as
        rows of one host array filled by a single (multi-threaded) copy out of the
        pinned staging rows — 30 separate single-threaded copies cost ~10x more."""
        if isinstance(hist, HistoryRing):
            return hist.finish(iters)
        if hist is None or iters == 0:
            return []
        out = np.empty((iters, hist.shape[1]), dtype=np.int32)
        torch.from_numpy(out).copy_(hist[:iters])
        return list(out)

    def collect(self, hist=None, evs=()) -> RunOutput:
        st = self.state.cpu().numpy()
        if st[5] != 0:
            raise ValueError("row_argmin: matrix contains NaN")  # dense.py:66-67 semantics
        iters = int(st[0])
        labels = d2h_staged(self.labels[iters % 2])
        dist_s = upd_s = 0.0
        for ev in list(evs)[:iters]:
            dist_s += ev[0].elapsed_time(ev[1]) / 1e3
            upd_s += ev[1].elapsed_time(ev[2]) / 1e3
        return RunOutput(
            iterations_run=iters, converged=bool(st[2]),
            objective_history=self.obj_hist[:iters].cpu().numpy().astype(np.float64),
            repairs=self.rep_hist[:iters].cpu().numpy().astype(np.int64),
            labels=labels,
            label_history=self._history_arrays(hist, iters),
            centroids=self.C.cpu().numpy(), distance_seconds=dist_s, update_seconds=upd_s)

    # -- lockstep / predict -----------------------------------------------------------
    def step_from(self, centroids, labels_prev) -> dict:
        """One iteration from given centroids and previous labels (parity harness)."""
        self.set_centroids(centroids)
        self.set_labels(labels_prev)
        with torch.cuda.device(self.dev):
            self.state.zero_()
        return self.traced_iteration(0)

    def traced_iteration(self, t: int) -> dict:
        """Iteration t of the ongoing fit (same kernels, relayouts and update
        mode as run()), synchronised, with everything the lockstep checker
        needs: the input centroids / previous labels, raw (pre-repair) and
        final labels, objective, changed, moved, new centroids and, for the
        screening variants, how many rows the certificate settled."""
        with torch.cuda.device(self.dev):
            c_in = self.C.cpu().numpy()
            prev = self.labels[t % 2].cpu().numpy()
            raw = torch.empty_like(self.labels[1])
            self.iteration(t, raw_out=raw)
            torch.cuda.current_stream().synchronize()
            acc = self.acc.cpu().numpy()
            st = self.state.cpu().numpy()
            kd = self.k * self.d
            out = {
                "centroids_in": c_in,
                "labels_prev": prev,
                "labels": self.labels[(t + 1) % 2].cpu().numpy(),
                "raw_labels": raw.cpu().numpy(),
                "mind": self.mind.cpu().numpy(),
                "objective": float(self.obj_hist[max(int(st[0]) - 1, 0)].item()),  # finalize's history slot
                "changed": float(acc[kd + self.k + 1]) / self.n_total,
                "moved": int(self.rep_hist[max(int(st[0]) - 1, 0)].item()),
                "centroids": self.C.cpu().numpy(),
                "counts": acc[kd:kd + self.k].copy(),
                "nan": bool(st[5]),
                "update_mode": "delta" if int(st[6]) & 1 else "full",
            }
            if self.variant in ("bf16s", "fp8s"):
                amb, two, ovf = int(self.amb_count.item()), int(self.two_count.item()), int(self.ovf_count.item())
                out["screen"] = {"ambiguous": amb, "two_candidate": two, "to_3xtf32": ovf,
                                 "certified": self.n - amb - two, "relayout": self.orig is not None}
            return out

    def predict(self, X) -> np.ndarray:
        """Nearest centroid for new points (estimator.py:131-136) — the same
        assignment kernel with the bookkeeping disabled."""
        with torch.cuda.device(self.dev):
            Xt = (X.to(self.dev, self.tdtype) if isinstance(X, torch.Tensor) else
                  torch.from_numpy(np.ascontiguousarray(X, dtype=self.dtype)).to(self.dev))
            m = int(Xt.shape[0])
            xn = torch.empty(m, dtype=self.tdtype, device=self.dev)
            out = torch.empty(m, dtype=torch.int32, device=self.dev)
            L.call(f"pcb_point_norms_{self.sfx}", _p(Xt), m, self.d, _p(xn), _stream())
            if self.variant in ("tc3xtf32", "tc1xtf32s", "bf16s", "fp8s"):
                # 3xTF32 over every row, near-ties re-evaluated exactly: the exact argmin
                xh = torch.empty((m, self.ld), dtype=torch.float32, device=self.dev)
                xl = torch.empty_like(xh)
                rows = torch.arange(m, dtype=torch.int32, device=self.dev)
                cnt = torch.full((1,), m, dtype=torch.int32, device=self.dev)
                sub = torch.empty(m, dtype=torch.int32, device=self.dev)
                fl = torch.empty(m, dtype=torch.int32, device=self.dev)
                fc = torch.zeros(1, dtype=torch.int32, device=self.dev)
                xs = torch.empty(int(L.load().pcb_exact_scratch_bytes()), dtype=torch.uint8, device=self.dev)
                L.call("pcb_resolve_ambiguous_f32", _p(Xt), m, self.d, _p(rows), _p(cnt), self.ld, _p(xh), _p(xl),
                       _p(sub), _p(xn), _p(self.C), _p(self.C_hi), _p(self.C_lo), _p(self.cnorm), self.k, _p(out),
                       _p(fl), _p(fc), _p(xs), xs.numel(), None, _stream())
            else:
                L.call(f"pcb_assign_{self.sfx}", _p(Xt), _p(xn), m, self.d, _p(self.C), _p(self.cnorm),
                       self.k, None, _p(out), None, None, None, self.vcode if self.variant not in ("delta", "deltatc") else 0,
                       _stream())
            return out.cpu().numpy()
