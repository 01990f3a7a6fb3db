"""Certificate audit of the screening variants (test infrastructure).

For every iteration of a real fit (same kernels, relayouts, delta updates and
two-candidate shortcut as the benchmark), compare the screen's pre-repair
labels of ALL rows with the exact argmin (row_argmin, dense.py:56-68: lowest
index on ties) of the iteration's input centroids:

* exact argmin = f64 expansion |p|^2 - 2 p.c + |c|^2 on the device (the
  library's f64 SIMT kernel, pcb_assign_f64 / tiled, over row chunks of P
  converted to f64), re-checked on the host with direct f64 sums
  sum_t (p_t - c_t)^2 for every row where it disagrees with the screen;
* a row is a VIOLATION when the screen's label is farther (direct f64) than
  the exact argmin, or equally far with a higher index.

Rows the certificate passes on to the 3xTF32 resolver (more than 64
candidates; everything at the cold start) are only f32-faithful: a mismatch
there is reported separately with its relative top-2 gap (the north star
exempts gaps below 1e-5), so ``violations`` counts certificate failures and
``resolver_mismatches`` the rest.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from paper_2501_05587_b200 import _lib as L


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def exact_argmin_device(P: torch.Tensor, C: np.ndarray, chunk: int = 2_000_000) -> torch.Tensor:
    """Lowest-index argmin of the f64 expansion for every row of P (device)."""
    n, d = P.shape
    k = C.shape[0]
    dev = P.device
    C64 = torch.from_numpy(np.ascontiguousarray(C, dtype=np.float64)).to(dev)
    cn = torch.empty(k, dtype=torch.float64, device=dev)
    L.call("pcb_centroid_norms_f64", _p(C64), k, d, _p(cn), _stream())
    out = torch.empty(n, dtype=torch.int32, device=dev)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        X = P[s:e].double().contiguous()
        xn = torch.empty(e - s, dtype=torch.float64, device=dev)
        L.call("pcb_point_norms_f64", _p(X), e - s, d, _p(xn), _stream())
        L.call("pcb_assign_f64", _p(X), _p(xn), e - s, d, _p(C64), _p(cn), k, None, _p(out[s:]), None, None,
               None, L.ASSIGN_TILED, _stream())
        del X
    return out


def direct_f64(P_rows: np.ndarray, C: np.ndarray, labels: np.ndarray) -> np.ndarray:
    P64 = P_rows.astype(np.float64)
    return ((P64 - C.astype(np.float64)[labels]) ** 2).sum(1)


def top2_rel_gap(P_rows: np.ndarray, C: np.ndarray) -> np.ndarray:
    P64 = P_rows.astype(np.float64)
    D = ((P64[:, None, :] - C.astype(np.float64)[None, :, :]) ** 2).sum(-1)
    part = np.partition(D, 1, axis=1)
    return (part[:, 1] - part[:, 0]) / np.maximum(np.abs(part[:, 0]), 1e-300)


def audit_fit(eng, iters: int, chunk: int = 2_000_000, log=None) -> list:
    """Run iterations 0 .. iters-1 of eng's fit (already initialised) and audit
    each one.  Returns one dict per iteration."""
    P = eng.P
    rows = []
    raw = torch.empty(eng.n, dtype=torch.int32, device=eng.dev)
    for t in range(iters):
        C_in = eng.C.cpu().numpy()
        cold = bool(getattr(eng, "_cold", False))
        eng.iteration(t, raw_out=raw)
        torch.cuda.synchronize()
        scr = {}
        if eng.variant in ("bf16s", "fp8s"):
            scr = {"ambiguous": int(eng.amb_count.item()), "two_candidate": int(eng.two_count.item()),
                   "to_3xtf32": int(eng.ovf_count.item())}
        ex = exact_argmin_device(P, C_in, chunk)
        mism = torch.nonzero(ex != raw).flatten().cpu().numpy()
        viol = res_mis = 0
        max_gap_mis = 0.0
        if mism.size:
            Pr = P[torch.from_numpy(mism).to(P.device)].cpu().numpy()
            sl = raw[torch.from_numpy(mism).to(P.device)].cpu().numpy()
            xl = ex[torch.from_numpy(mism).to(P.device)].cpu().numpy()
            ds, dx = direct_f64(Pr, C_in, sl), direct_f64(Pr, C_in, xl)
            # the device f64 expansion can itself mis-rank a near-tie: trust direct sums
            worse = (ds > dx) | ((ds == dx) & (sl > xl))
            gaps = top2_rel_gap(Pr[worse], C_in) if worse.any() else np.zeros(0)
            # rows that reached the 3xTF32 resolver are f32-faithful, not certified:
            # with the cold start every row does; afterwards only the overflow list
            if cold or scr.get("to_3xtf32", 0) > 0:
                ovf = set()
                if not cold:
                    ovf = set(eng.ovf_list[: scr["to_3xtf32"]].cpu().numpy().tolist())
                in_res = np.array([cold or int(r) in ovf for r in mism[worse]], dtype=bool)
            else:
                in_res = np.zeros(int(worse.sum()), dtype=bool)
            viol = int((~in_res).sum())
            res_mis = int(in_res.sum())
            max_gap_mis = float(gaps.max()) if gaps.size else 0.0
        r = {"iteration": t, "rows": eng.n, "cold_start_3xtf32": cold, "mismatch_vs_f64_expansion": int(mism.size),
             "violations": viol, "resolver_mismatches": res_mis, "max_rel_gap_of_mismatch": max_gap_mis, **scr}
        rows.append(r)
        if log is not None:
            log(r)
    return rows
