"""CPU oracle for the Lloyd hot path — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The shipped path
(``paper_2501_05587_b200``) never imports it and has no CPU fallback.

It restates, with plain numpy, the classical Lloyd driver of the reference
package ``popcorn`` (``/root/reference/pkg/src/popcorn``):

* ``run_lloyd``            -> clustering.py:291-325
* ``init_assignments``     -> clustering.py:91-108   (PCG64 labels + empty fix)
* ``repair_empty_clusters``-> clustering.py:111-139  (farthest-point donation)
* ``assignment_step``      -> clustering.py:142-150  (argmin, repair, objective)
* ``mean_centroids``       -> clustering.py:282-288  (per-cluster mean in dtype)
* ``distance_matrix``      -> clustering.py:310-311  (pn - 2 P C^T + cn)
* ``row_argmin``           -> dense.py:56-68         (lowest index on ties)
* ``as_float_matrix`` / ``normalize_dtype`` -> validation.py:18-47
* ``augmented_distance``   -> analysis.py:83-102     (q C q^T, f64)

The arithmetic is the same sequence of numpy calls as the reference, so on the
same numpy/OpenBLAS build the outputs are bit-identical; that is pinned by
``tests/test_oracle.py`` against fixtures generated from the reference itself
(``tests/golden/make_golden.py``).  Parity status: PINNED (golden vectors from
the reference run in the authoring container).

On top of the restatement it offers the lockstep helpers the parity harness
needs: one Lloyd step from given centroids, f64 top-2
distance gaps for the label exemption, and f64 centroid means.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from time import perf_counter

import numpy as np

LABEL_DTYPE = np.int32
_FLOAT_DTYPES = (np.float32, np.float64)
_ALIASES = {"f32": np.float32, "f64": np.float64, "float32": np.float32,
            "float64": np.float64, "single": np.float32, "double": np.float64}


# -- validation (validation.py:18-47) ---------------------------------------
def normalize_dtype(dtype) -> np.dtype:
    if isinstance(dtype, str):
        if dtype.lower() not in _ALIASES:
            raise ValueError(f"unsupported dtype {dtype!r}")
        return np.dtype(_ALIASES[dtype.lower()])
    dt = np.dtype(dtype)
    if dt not in (np.dtype(np.float32), np.dtype(np.float64)):
        raise ValueError(f"unsupported dtype {dtype!r}")
    return dt


def as_float_matrix(X, dtype=None, name: str = "X") -> np.ndarray:
    if dtype is None:
        src = np.asarray(X)
        dtype = src.dtype if src.dtype in _FLOAT_DTYPES else np.float32
    A = np.ascontiguousarray(X, dtype=normalize_dtype(dtype))
    if A.ndim != 2 or A.shape[0] < 1 or A.shape[1] < 1:
        raise ValueError(f"{name} must be a non-empty 2-D matrix, got shape {A.shape}")
    if not np.isfinite(A).all():
        raise ValueError(f"{name} contains non-finite entries")
    return A


# -- init (clustering.py:91-108) --------------------------------------------
def init_assignments(n: int, k: int, seed: int) -> np.ndarray:
    if not 1 <= k <= n:
        raise ValueError(f"k must satisfy 1 <= k <= n, got k={k}, n={n}")
    gen = np.random.Generator(np.random.PCG64(seed))
    labels = gen.integers(0, k, size=n).astype(LABEL_DTYPE)
    while True:
        hollow = np.flatnonzero(np.bincount(labels, minlength=k) == 0)
        if hollow.size == 0:
            return labels
        labels[hollow] = hollow.astype(LABEL_DTYPE)


# -- argmin (dense.py:56-68) --------------------------------------------------
def row_argmin(D) -> np.ndarray:
    A = np.asarray(D)
    if A.ndim != 2 or A.shape[0] < 1 or A.shape[1] < 1:
        raise ValueError(f"row_argmin expects a non-empty 2-D matrix, got {A.shape}")
    if np.isnan(A).any():
        raise ValueError("row_argmin: matrix contains NaN")
    return np.argmin(A, axis=1).astype(LABEL_DTYPE)


# -- repair (clustering.py:111-139) ------------------------------------------
def repair_empty_clusters(labels, D, k: int) -> np.ndarray:
    lab = np.asarray(labels).astype(LABEL_DTYPE)
    n = lab.size
    if k > n:
        raise ValueError(f"cannot fill {k} clusters with {n} points")
    Dm = np.asarray(D)
    if Dm.shape != (n, k):
        raise ValueError(f"distance matrix shape {Dm.shape} != ({n}, {k})")
    lab = lab.copy()
    taken = np.zeros(n, dtype=bool)
    rows = np.arange(n)
    while True:
        hollow = np.flatnonzero(np.bincount(lab, minlength=k) == 0)
        if hollow.size == 0:
            return lab
        for j in hollow:
            own = Dm[rows, lab].astype(np.float64)
            own[taken] = -np.inf
            donor = int(np.argmax(own))
            lab[donor] = j
            taken[donor] = True


# -- one assignment (clustering.py:142-150) ----------------------------------
def assignment_step(D, labels_prev, k: int):
    n = D.shape[0]
    raw = row_argmin(D)
    if np.bincount(raw, minlength=k).min() == 0:
        labels = repair_empty_clusters(raw, D, k)
    else:
        labels = raw
    moved = int(np.count_nonzero(labels != raw))
    objective = float(D[np.arange(n), labels].sum(dtype=np.float64))
    changed = float(np.count_nonzero(labels != labels_prev)) / n
    return labels, moved, objective, changed


# -- centroids (clustering.py:282-288) ----------------------------------------
def mean_centroids(P: np.ndarray, labels: np.ndarray, k: int) -> np.ndarray:
    C = np.zeros((k, P.shape[1]), dtype=P.dtype)
    for j in range(k):
        idx = np.flatnonzero(labels == j)
        if idx.size:
            C[j] = P[idx].mean(axis=0)
    return C


def mean_centroids_f64(P: np.ndarray, labels: np.ndarray, k: int) -> np.ndarray:
    """Exact-ish (f64-accumulated) means; the tolerance anchor for centroids."""
    P64 = np.asarray(P, dtype=np.float64)
    sums = np.zeros((k, P.shape[1]), dtype=np.float64)
    np.add.at(sums, labels, P64)
    counts = np.bincount(labels, minlength=k).astype(np.float64)
    out = np.zeros_like(sums)
    nz = counts > 0
    out[nz] = sums[nz] / counts[nz, None]
    return out


# -- distances (clustering.py:302, 310-311) ----------------------------------
def point_norms(P: np.ndarray) -> np.ndarray:
    return (P * P).sum(axis=1)


def distance_matrix(P: np.ndarray, pnorm: np.ndarray, centroids: np.ndarray) -> np.ndarray:
    cn = (centroids * centroids).sum(axis=1)
    return pnorm[:, None] - 2.0 * (P @ centroids.T) + cn[None, :]


def augmented_distance(p, c) -> float:
    """q . C . q^T with q=[1,p], C=[[|c|^2,-c^T],[-c,I]] (analysis.py:83-102)."""
    pv = np.asarray(p, dtype=np.float64).ravel()
    cv = np.asarray(c, dtype=np.float64).ravel()
    if pv.size != cv.size:
        raise ValueError("dimension mismatch")
    M = np.eye(pv.size + 1)
    M[0, 0] = cv @ cv
    M[0, 1:] = -cv
    M[1:, 0] = -cv
    q = np.concatenate(([1.0], pv))
    return float(q @ M @ q)


# -- lockstep step ------------------------------------------------------------
@dataclass
class StepResult:
    labels: np.ndarray          # post-repair labels of this iteration
    raw_labels: np.ndarray      # pre-repair argmin
    moved: int                  # repair count
    objective: float            # sum D[i, label_i] in f64
    changed: float              # fraction of labels != previous labels
    centroids: np.ndarray       # mean centroids over the new labels (dtype of P)


def lloyd_step(P, pnorm, centroids, labels_prev, k: int) -> StepResult:
    """One iteration of the loop body at clustering.py:309-317."""
    D = distance_matrix(P, pnorm, centroids)
    raw = row_argmin(D)
    labels, moved, objective, changed = assignment_step(D, labels_prev, k)
    return StepResult(labels=labels, raw_labels=raw, moved=moved, objective=objective,
                      changed=changed, centroids=mean_centroids(P, labels, k))


def top2_gap_f64(P, centroids, chunk: int = 16384):
    """Relative top-2 gap (d2-d1)/|d1| per point, in f64.

    The exemption of the north-star tolerance: labels may differ where this is
    below 1e-5.  Returns (d1, gap_rel) arrays.
    """
    P64 = np.asarray(P, dtype=np.float64)
    C64 = np.asarray(centroids, dtype=np.float64)
    n = P64.shape[0]
    d1 = np.empty(n)
    gap = np.empty(n)
    cn = (C64 * C64).sum(1)
    for s in range(0, n, chunk):
        blk = P64[s:s + chunk]
        # difference form in f64 (accurate to ~1e-16 relative)
        D = (blk * blk).sum(1)[:, None] - 2.0 * blk @ C64.T + cn[None, :]
        if C64.shape[0] == 1:
            d1[s:s + chunk] = D[:, 0]
            gap[s:s + chunk] = np.inf
            continue
        part = np.partition(D, 1, axis=1)[:, :2]
        a, b = part[:, 0], part[:, 1]
        d1[s:s + chunk] = a
        gap[s:s + chunk] = (b - a) / np.maximum(np.abs(a), 1e-300)
    return d1, gap


def top2_gap_abs_f64(P, centroids, chunk: int = 16384):
    """Absolute top-2 gap d2 - d1 per point in f64 (inf for k = 1): compared with
    the reference's own f32 expansion error in the parity checker."""
    P64 = np.asarray(P, dtype=np.float64)
    C64 = np.asarray(centroids, dtype=np.float64)
    n = P64.shape[0]
    out = np.full(n, np.inf)
    if C64.shape[0] == 1:
        return out
    cn = (C64 * C64).sum(1)
    for s in range(0, n, chunk):
        blk = P64[s:s + chunk]
        D = (blk * blk).sum(1)[:, None] - 2.0 * blk @ C64.T + cn[None, :]
        part = np.partition(D, 1, axis=1)[:, :2]
        out[s:s + chunk] = part[:, 1] - part[:, 0]
    return out


# -- full driver (clustering.py:291-325) ---------------------------------------
@dataclass
class OracleTimings:
    kernel_matrix_seconds: float = 0.0
    pairwise_distances_seconds: float = 0.0
    argmin_update_seconds: float = 0.0


@dataclass
class OracleResult:
    labels: np.ndarray
    iterations_run: int
    objective_history: np.ndarray
    converged: bool
    timings: OracleTimings
    label_history: list = field(default_factory=list)
    repairs: np.ndarray = None
    centroids: np.ndarray = None
    centroid_history: list = field(default_factory=list)


def run_lloyd(points, k: int, max_iters: int = 30, tol: float = 0.0,
              check_convergence: bool = False, seed: int = 0, dtype=np.float32,
              init_centroids=None, record_centroids: bool = False) -> OracleResult:
    """Lloyd's loop exactly as clustering.py:291-325 sequences it.

    ``init_centroids`` (additive, not in the reference) replaces the
    random-label init + initial means (clustering.py:298-300) with fixed
    centroids; the initial "previous labels" are then the init labels
    anyway, so ``changed`` of iteration 1 is measured against them.
    """
    P = as_float_matrix(points, dtype=normalize_dtype(dtype), name="points")
    n = P.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"k must satisfy 1 <= k <= n, got k={k}, n={n}")
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    if not 0.0 <= tol <= 1.0:
        raise ValueError("tol must lie in [0, 1]")
    t = OracleTimings()
    labels = init_assignments(n, k, seed)
    t0 = perf_counter()
    if init_centroids is None:
        C = mean_centroids(P, labels, k)
    else:
        C = np.ascontiguousarray(init_centroids, dtype=P.dtype).reshape(k, P.shape[1])
    t.argmin_update_seconds += perf_counter() - t0
    pn = point_norms(P)

    hist, lhist, reps, chist = [], [], [], []
    converged = False
    for _ in range(max_iters):
        t0 = perf_counter()
        D = distance_matrix(P, pn, C)
        t.pairwise_distances_seconds += perf_counter() - t0
        t0 = perf_counter()
        labels, moved, objective, changed = assignment_step(D, labels, k)
        C = mean_centroids(P, labels, k)
        t.argmin_update_seconds += perf_counter() - t0
        hist.append(objective)
        lhist.append(labels.copy())
        reps.append(moved)
        if record_centroids:
            chist.append(C.copy())
        if check_convergence and changed <= tol:
            converged = True
            break
    return OracleResult(labels=labels, iterations_run=len(hist),
                        objective_history=np.asarray(hist, dtype=np.float64),
                        converged=converged, timings=t, label_history=lhist,
                        repairs=np.asarray(reps, dtype=np.int64), centroids=C,
                        centroid_history=chist)


# -- synthetic workloads --------------------------------------
def make_blobs(n: int, d: int, k: int, seed: int = 0, spread: float = 10.0,
               sigma: float = 1.0) -> np.ndarray:
    """PCG64 blobs: centers ~ U(-spread, spread)^{k x d}, P = centers[true] + N(0, sigma)."""
    gen = np.random.Generator(np.random.PCG64(seed))
    centers = gen.uniform(-spread, spread, size=(k, d))
    true = gen.integers(0, k, size=n)
    P = centers[true] + gen.normal(0.0, sigma, size=(n, d))
    return P.astype(np.float32)
