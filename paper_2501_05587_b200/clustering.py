"""Lloyd driver with the reference's contract, running on the B200 engine.

Mirrors ``popcorn.clustering`` (/root/reference/pkg/src/popcorn/clustering.py)
for the classical Lloyd path:

* ``KKMeansConfig``      clustering.py:43-68  (+ additive: init, record_label_history,
                                               variant, device)
* ``ClusteringResult``   clustering.py:71-88  (+ additive: centroids)
* ``TimingBreakdown``    clustering.py:34-40
* ``init_assignments``   clustering.py:91-108 (host mirror; drivers draw it on the device)
* ``run_lloyd``          clustering.py:291-325 — same signature
  ``driver(points, cfg) -> ClusteringResult`` as the `_ALGORITHMS` plugins.

Validation happens on the host first so errors match the reference
(ValueError for bad config / non-finite input); device failures surface as
RuntimeError.  Everything numeric runs in the CUDA library; there is no CPU
fallback.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from time import perf_counter
from typing import Any

import numpy as np

from .kernels import GramMethod, KernelSpec
from .validation import as_float_matrix, normalize_dtype

LABEL_DTYPE = np.int32


@dataclass
class TimingBreakdown:
    """Seconds per phase, accumulated across iterations (clustering.py:34-40).

    On the GPU path these are CUDA-event times: pairwise_distances_seconds is
    the fused distance+argmin kernel, argmin_update_seconds the centroid
    update, repair and finalize; kernel_matrix_seconds stays 0 for Lloyd.
    """

    kernel_matrix_seconds: float = 0.0
    pairwise_distances_seconds: float = 0.0
    argmin_update_seconds: float = 0.0


@dataclass
class KKMeansConfig:
    """Driver settings (clustering.py:43-68).

    ``kernel``/``gram`` (KernelSpec/GramMethod, kernels.py) drive run_popcorn
    and run_baseline; Lloyd ignores them (clustering.py:292).
    Additive fields (defaults reproduce the reference exactly):
      init                 None -> random labels + means (clustering.py:298-300);
                           an array (k, d) -> fixed initial centroids.
      record_label_history keep per-iteration labels (4n bytes D2H per iteration).
      variant              assignment kernel: 'auto', 'rowreg', 'tiled', 'tc3xtf32', 'tc1xtf32s', 'bf16s',
                           'fp8s', or the delta-chunked ablations 'delta' (FFMA) / 'deltatc' (tcgen05).
      device               CUDA device index (None = current).
    """

    k: int
    max_iters: int = 30
    tol: float = 0.0
    check_convergence: bool = False
    seed: int = 0
    kernel: Any = field(default_factory=KernelSpec)
    gram: Any = field(default_factory=GramMethod)
    dtype: object = np.float32
    init: Any = None
    record_label_history: bool = True
    variant: str = "auto"
    device: Any = None

    def validate_for(self, n: int) -> None:
        if not 1 <= self.k <= n:
            raise ValueError(f"k must satisfy 1 <= k <= n, got k={self.k}, n={n}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if not 0.0 <= self.tol <= 1.0:
            raise ValueError("tol must lie in [0, 1]")


@dataclass
class ClusteringResult:
    """Outcome of one driver call (clustering.py:71-88) + final centroids."""

    labels: np.ndarray
    iterations_run: int
    objective_history: np.ndarray
    converged: bool
    timings: TimingBreakdown
    label_history: list
    repairs: np.ndarray
    centroids: np.ndarray | None = field(default=None)


def init_assignments(n: int, k: int, seed: int) -> np.ndarray:
    """Seeded PCG64 labels with no empty cluster (clustering.py:91-108).

    The host-returning mirror of the reference function (numpy's own PCG64).
    The drivers (run_lloyd, run_lloyd_sharded, bench) draw the same stream on
    the device instead: LloydEngine.init_labels_device / pcb_init_assignments.
    """
    if not 1 <= k <= n:
        raise ValueError(f"k must satisfy 1 <= k <= n, got k={k}, n={n}")
    rng = np.random.Generator(np.random.PCG64(seed))
    labels = rng.integers(0, k, size=n).astype(LABEL_DTYPE)
    while True:
        empty = np.flatnonzero(np.bincount(labels, minlength=k) == 0)
        if empty.size == 0:
            return labels
        labels[empty] = empty.astype(LABEL_DTYPE)


def _prepare_points(points, cfg: KKMeansConfig):
    try:
        import torch
        if isinstance(points, torch.Tensor):
            if points.ndim != 2 or points.shape[0] < 1 or points.shape[1] < 1:
                raise ValueError(f"points must be a non-empty 2-D matrix, got shape {tuple(points.shape)}")
            if not bool(torch.isfinite(points).all()):
                raise ValueError("points contains non-finite entries")
            return points, int(points.shape[0]), int(points.shape[1])
    except ImportError:  # pragma: no cover
        pass
    # Small inputs are scanned for non-finite values on the host; large ones
    # (> 16M values) on the device right after the copy (same ValueError).
    A = np.asarray(points)
    host_check = A.size <= (1 << 24)
    P = as_float_matrix(points, dtype=normalize_dtype(cfg.dtype), name="points", check_finite=host_check)
    return P, P.shape[0], P.shape[1]


def run_lloyd(points, cfg: KKMeansConfig) -> ClusteringResult:
    """Classical Lloyd iteration on the B200 (clustering.py:291-325).

    Same loop semantics as the reference: labels from init_assignments,
    initial mean centroids, then per iteration distance + lowest-index argmin,
    empty-cluster repair, objective (sum of own distances, f64), mean update
    and the fraction-changed convergence test.  Accepts a numpy array (copied
    once to HBM) or a CUDA tensor (used in place, additive).
    """
    from .engine import LloydEngine  # torch is imported lazily

    dtype = normalize_dtype(cfg.dtype)
    P, n, d = _prepare_points(points, cfg)
    cfg.validate_for(n)
    if cfg.init is not None:
        init = np.asarray(cfg.init)
        if init.shape != (cfg.k, d):
            raise ValueError(f"init centroids must have shape ({cfg.k}, {d}), got {init.shape}")
        if not np.isfinite(init).all():
            raise ValueError("init contains non-finite entries")
    eng = LloydEngine(P, cfg.k, dtype=dtype, device=cfg.device, variant=cfg.variant,
                      max_iters=cfg.max_iters, check_finite=isinstance(P, np.ndarray) and P.size > (1 << 24))
    eng.init_labels_device(cfg.seed)  # init_assignments, clustering.py:91-108, in HBM
    if cfg.init is None:
        eng.init_centroids_from_labels()
    else:
        eng.set_centroids(init)
    out = eng.run(cfg.max_iters, cfg.tol, cfg.check_convergence,
                  record_history=cfg.record_label_history)
    timings = TimingBreakdown(0.0, out.distance_seconds, out.update_seconds)
    return ClusteringResult(labels=out.labels, iterations_run=out.iterations_run,
                            objective_history=out.objective_history, converged=out.converged,
                            timings=timings, label_history=out.label_history,
                            repairs=out.repairs, centroids=out.centroids)


def lloyd_step(points, centroids, labels_prev, k: int, dtype=np.float32, variant: str = "auto"):
    """One Lloyd iteration from given centroids (lockstep parity API).

    Returns a dict with labels, mind (own distances), objective, changed,
    moved (repairs) and the new centroids — the quantities of
    clustering.py:310-317 for a single pass.
    """
    from .engine import LloydEngine

    P = as_float_matrix(points, dtype=normalize_dtype(dtype), name="points")
    eng = LloydEngine(P, k, dtype=normalize_dtype(dtype), variant=variant, max_iters=1)
    return eng.step_from(centroids, labels_prev)
