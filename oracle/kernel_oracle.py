"""CPU oracle for the kernel K-means path (f4) — TEST INFRASTRUCTURE ONLY.

Like lloyd_oracle.py this is the checker, never the product: only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import it.  It restates
with plain numpy the matrix-centric driver of the reference package
(/root/reference/pkg/src/popcorn):

* ``compute_gram``            -> kernels.py:85-89 (+ select_gram_algorithm :72-82,
                                 gemm_gram dense.py:20-29, syrk_gram dense.py:32-46)
* ``apply_kernel``            -> kernels.py:111-131 (+ _int_pow :96-108)
* ``build_selection_matrix``  -> sparse.py:101-118 (as dense counts/order arrays)
* ``spmm_neg2_kvt``           -> sparse.py:121-142
* ``spmv_scaled``             -> sparse.py:145-160
* ``run_popcorn``             -> clustering.py:165-218
* ``kernel_trick_distances``  -> clustering.py:221-240 (run_baseline's distances)
* ``run_baseline``            -> clustering.py:243-279

The assignment step, repair and init are shared with lloyd_oracle.  The same
numpy calls in the same order make the outputs bit-identical to the reference
on the same numpy build; tests/test_oracle_kernel.py pins that against
fixtures produced by the reference itself (tests/golden/make_kernel_golden.py).
Parity status: PINNED.
"""
from __future__ import annotations

import numpy as np

from .lloyd_oracle import (LABEL_DTYPE, OracleResult, OracleTimings, as_float_matrix, assignment_step,
                           init_assignments, normalize_dtype)

KERNEL_FAMILIES = ("linear", "polynomial", "gaussian", "sigmoid")
GAUSSIAN_EXP_FLOOR = -88.0


def select_gram_algorithm(n: int, d: int, variant: str = "auto", threshold: float = 100.0) -> str:
    if variant != "auto":
        return variant
    return "gemm" if n / d > threshold else "syrk"


def compute_gram(P, variant: str = "auto", threshold: float = 100.0) -> np.ndarray:
    P = np.ascontiguousarray(P)
    n = P.shape[0]
    if select_gram_algorithm(n, P.shape[1], variant, threshold) == "gemm":
        return P @ P.T
    out = np.zeros((n, n), dtype=P.dtype)
    for i in range(n):
        out[i, i:] = P[i:, :] @ P[i, :]
    for i in range(n):
        out[i + 1:, i] = out[i, i + 1:]
    return out


def _int_pow(base, exponent: int):
    result = None
    acc = base
    e = exponent
    while e:
        if e & 1:
            result = acc if result is None else result * acc
        e >>= 1
        if e:
            acc = acc * acc
    return result


def apply_kernel(B, family="polynomial", gamma=1.0, coef=1.0, degree=2, sigma=1.0) -> np.ndarray:
    Bd = np.asarray(B)
    with np.errstate(over="ignore", invalid="ignore"):
        if family == "linear":
            K = Bd.copy()
        elif family == "polynomial":
            K = _int_pow(gamma * Bd + coef, degree)
        elif family == "sigmoid":
            K = np.tanh(gamma * Bd + coef)
        else:
            dvec = Bd.diagonal()
            expo = (-gamma / (sigma * sigma)) * (-2.0 * Bd + dvec[:, None] + dvec[None, :])
            np.maximum(expo, GAUSSIAN_EXP_FLOOR, out=expo)
            K = np.exp(expo)
            np.fill_diagonal(K, 1.0)
    K = np.ascontiguousarray(K, dtype=Bd.dtype)
    if not np.isfinite(K).all():
        raise FloatingPointError(f"apply_kernel[{family}] produced non-finite values")
    return K


def selection(labels, k: int, dtype=np.float32):
    """CSR arrays of build_selection_matrix: rowptrs, colinds (stable order), values."""
    labels = np.asarray(labels).astype(LABEL_DTYPE)
    counts = np.bincount(labels, minlength=k)
    rowptrs = np.zeros(k + 1, dtype=np.int32)
    np.cumsum(counts, out=rowptrs[1:])
    order = np.argsort(labels, kind="stable").astype(np.int32)
    values = (1.0 / counts[labels[order]]).astype(dtype)
    return rowptrs, order, values


def spmm_neg2_kvt(K, rowptrs, colinds, values) -> np.ndarray:
    n = K.shape[0]
    k = rowptrs.size - 1
    E = np.empty((n, k), dtype=K.dtype)
    for j in range(k):
        lo, hi = int(rowptrs[j]), int(rowptrs[j + 1])
        cols, vals = colinds[lo:hi], values[lo:hi]
        if cols.size == 0:
            E[:, j] = 0.0
            continue
        E[:, j] = K[:, cols] @ vals.astype(K.dtype, copy=False)
    np.multiply(E, -2.0, out=E)
    return E


def spmv_scaled(alpha, rowptrs, colinds, values, z) -> np.ndarray:
    zv = np.asarray(z)
    k = rowptrs.size - 1
    products = values.astype(np.float64) * zv[colinds].astype(np.float64)
    row_ids = np.repeat(np.arange(k), np.diff(rowptrs))
    out = np.bincount(row_ids, weights=products, minlength=k)
    return (float(alpha) * out).astype(zv.dtype)


def popcorn_distances(K, labels, k: int) -> np.ndarray:
    """D of one run_popcorn iteration (clustering.py:197-204)."""
    n = K.shape[0]
    rowptrs, colinds, values = selection(labels, k, dtype=K.dtype)
    E = spmm_neg2_kvt(K, rowptrs, colinds, values)
    z = -0.5 * E[np.arange(n), labels]
    cn = spmv_scaled(1.0, rowptrs, colinds, values, z)
    D = E
    D += np.ascontiguousarray(K.diagonal())[:, None]
    D += cn[None, :]
    return D


def kernel_trick_distances(K, labels, k: int) -> np.ndarray:
    n = K.shape[0]
    dk = K.diagonal()
    D = np.empty((n, k), dtype=K.dtype)
    for j in range(k):
        members = np.flatnonzero(labels == j)
        m = members.size
        if m == 0:
            D[:, j] = np.inf
            continue
        cluster_sum = K[:, members].sum(axis=1)
        self_term = float(K[np.ix_(members, members)].sum())
        D[:, j] = dk - (2.0 / m) * cluster_sum + self_term / (m * m)
    return D


def kernel_matrix(P, family="polynomial", gamma=1.0, coef=1.0, degree=2, sigma=1.0, gram="auto",
                  threshold=100.0, dtype=np.float32) -> np.ndarray:
    P = as_float_matrix(P, dtype=normalize_dtype(dtype))
    return apply_kernel(compute_gram(P, gram, threshold), family, gamma, coef, degree, sigma)


def _run(P, k, dist_fn, max_iters=30, tol=0.0, check_convergence=False, seed=0, dtype=np.float32, K=None,
         **kernel):
    P = as_float_matrix(P, dtype=normalize_dtype(dtype))
    n = P.shape[0]
    if K is None:
        K = kernel_matrix(P, dtype=dtype, **kernel)
    labels = init_assignments(n, k, seed)
    hist, lab_hist, reps = [], [], []
    converged = False
    for _ in range(max_iters):
        D = dist_fn(K, labels, k)
        labels, moved, objective, changed = assignment_step(D, labels, k)
        hist.append(objective)
        lab_hist.append(labels.copy())
        reps.append(moved)
        if check_convergence and changed <= tol:
            converged = True
            break
    return OracleResult(labels=labels, iterations_run=len(hist),
                        objective_history=np.asarray(hist, dtype=np.float64), converged=converged,
                        timings=OracleTimings(), label_history=lab_hist,
                        repairs=np.asarray(reps, dtype=np.int64))


def run_popcorn(P, k, **kw):
    return _run(P, k, popcorn_distances, **kw)


def run_baseline(P, k, **kw):
    return _run(P, k, kernel_trick_distances, **kw)


def top2_gap(D) -> np.ndarray:
    """Per row: second smallest minus smallest entry (f64)."""
    Ds = np.sort(np.asarray(D, dtype=np.float64), axis=1)
    return Ds[:, 1] - Ds[:, 0] if Ds.shape[1] > 1 else np.full(Ds.shape[0], np.inf)


def kernel_matrix_between(X, Y, family="polynomial", gamma=1.0, coef=1.0, degree=2, sigma=1.0):
    """kernels.py:143-166."""
    B = X @ Y.T
    if family == "linear":
        K = B
    elif family == "polynomial":
        K = _int_pow(gamma * B + coef, degree)
    elif family == "sigmoid":
        K = np.tanh(gamma * B + coef)
    else:
        xn = (X * X).sum(axis=1)
        yn = (Y * Y).sum(axis=1)
        expo = (-gamma / (sigma * sigma)) * (-2.0 * B + xn[:, None] + yn[None, :])
        np.maximum(expo, GAUSSIAN_EXP_FLOOR, out=expo)
        K = np.exp(expo)
    return np.ascontiguousarray(K, dtype=X.dtype)


def predict_kernel(X_fit, labels, k, X, family="polynomial", gamma=1.0, coef=1.0, degree=2, sigma=1.0):
    """KernelKMeans.predict for the kernel drivers (estimator.py:137-147, 163-181);
    also returns D for gap checks."""
    kw = dict(family=family, gamma=gamma, coef=coef, degree=degree, sigma=sigma)
    X = np.asarray(X, dtype=X_fit.dtype)
    cross = kernel_matrix_between(X, X_fit, **kw)
    sq = (X * X).sum(axis=1)
    if family == "linear":
        self_terms = sq
    elif family == "polynomial":
        self_terms = (gamma * sq + coef) ** degree
    elif family == "sigmoid":
        self_terms = np.tanh(gamma * sq + coef)
    else:
        self_terms = np.ones_like(sq)
    members = [np.flatnonzero(labels == j) for j in range(k)]
    sizes = np.array([max(m.size, 1) for m in members])
    cluster_self = np.array([float(kernel_matrix_between(X_fit[m], X_fit[m], **kw).sum()) if m.size else 0.0
                             for m in members])
    D = np.empty((X.shape[0], k), dtype=X.dtype)
    for j in range(k):
        m = sizes[j]
        D[:, j] = self_terms - (2.0 / m) * cross[:, members[j]].sum(axis=1) + cluster_self[j] / (m * m)
    return np.argmin(D, axis=1).astype(LABEL_DTYPE), D
