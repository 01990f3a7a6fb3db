"""Lockstep parity checker (SURVEY.md Appendix B / BASELINE.json north_star).

Given the reference step (oracle, same inputs) and the GPU step, assert:

* labels identical except rows whose f64 top-2 relative gap (d2-d1)/|d1|
  at the step's input centroids is below GAP_EXEMPT = 1e-5, or whose absolute
  gap is below the reference's own f32 expansion error, ABS_EXEMPT = 2^-20 of
  |p|^2 + |c|^2 (the reference ranks pn - 2 p.c + cn in f32: below that gap its
  label is rounding noise, e.g. when points coincide with centroids);
* objective within OBJ_RTOL = 1e-6 relative of the reference's objective
  formula evaluated on the GPU labels (= the reference objective whenever the
  labels agree; differs only through exempt rows), plus an f32
  rounding allowance for the reference's own expansion
  (2^-22 * sum_i (pn_i + cn_label_i)), which only matters when the
  objective is tiny compared with the norms (cancellation);
* centroids within CEN_RTOL = 1e-5 (per centroid, inf-norm relative) of the
  f64 means over the GPU's own labels, and of the reference's centroids
  whenever the labels agree;
* moved (repairs) and changed identical whenever the labels agree;
* empty-cluster repair: donors are the points with the largest own distance;
  when two candidates' own distances agree to DONOR_RTOL = 1e-6 (the
  reference ranks f32 expansion values, we rank exact ones) the donor order
  may swap — rows whose mismatch is explained by such a swap are exempt.
"""
import numpy as np

import oracle

GAP_EXEMPT = 1e-5
ABS_EXEMPT = 2.0 ** -20
OBJ_RTOL = 1e-6
CEN_RTOL = 1e-5
DONOR_RTOL = 1e-6


def _donor_swap_exempt(P, C, gpu, ref, diff):
    """Rows differing only because repair picked a near-tied donor."""
    if "raw_labels" not in gpu:
        return np.zeros_like(diff)
    P64 = np.asarray(P, dtype=np.float64)
    C64 = np.asarray(C, dtype=np.float64)
    ref_don = ref.labels != ref.raw_labels
    gpu_don = gpu["labels"] != gpu["raw_labels"]
    cand = diff & (ref_don | gpu_don)
    if not cand.any():
        return cand
    raw = ref.raw_labels
    own = ((P64 - C64[raw]) ** 2).sum(1)
    scale = (P64 ** 2).sum(1) + (C64[raw] ** 2).sum(1)  # the reference's f32 expansion error scale
    # every donor-related mismatch must have a swap partner: another mismatched
    # donor (in either run) whose own distance ties with it to DONOR_RTOL (or
    # to the reference's f32 expansion error)
    pool = np.flatnonzero(cand)
    ok = np.zeros_like(diff)
    for x in pool:
        others = pool[pool != x]
        tol = DONOR_RTOL * abs(own[x]) + ABS_EXEMPT * scale[x]
        if others.size and np.min(np.abs(own[others] - own[x])) <= tol:
            ok[x] = True
    return ok


def centroid_rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    num = np.abs(a - b).max(axis=1)
    den = np.maximum(np.abs(b).max(axis=1), 1e-30)
    return float((num / den).max())


def check_step(P, C_in, labels_prev, k, gpu, ref=None, *, dtype=np.float32, what=""):
    """Compare one GPU step (dict from LloydEngine.step_from) with the oracle."""
    Pd = np.ascontiguousarray(P, dtype=dtype)
    Cd = np.ascontiguousarray(C_in, dtype=dtype)
    if ref is None:
        ref = oracle.lloyd_step(Pd, oracle.point_norms(Pd), Cd, labels_prev, k)
    _, gap = oracle.top2_gap_f64(Pd, Cd)
    gap_abs = oracle.top2_gap_abs_f64(Pd, Cd)
    P64 = Pd.astype(np.float64)
    cmax = float((Cd.astype(np.float64) ** 2).sum(1).max())
    noise = ABS_EXEMPT * ((P64 ** 2).sum(1) + cmax)
    diff = gpu["labels"] != ref.labels
    # a repaired row can legitimately differ only through a different donor,
    # which itself requires a near-tie; treat donors like exempt rows
    exempt = (gap < GAP_EXEMPT) | (gap_abs <= noise) | _donor_swap_exempt(Pd, Cd, gpu, ref, diff)
    bad = diff & ~exempt
    assert not bad.any(), (f"{what}: {int(bad.sum())} non-exempt label mismatches "
                           f"(first rows {np.flatnonzero(bad)[:8].tolist()}, gaps {gap[bad][:8]})")
    pn = oracle.point_norms(Pd.astype(np.float64))
    cn = (Cd.astype(np.float64) ** 2).sum(1)
    allowance = 2.0 ** -22 * float((pn + cn[ref.labels]).sum())
    ref_obj = ref.objective
    if diff.any():
        # the reference's D (clustering.py:311) summed over the GPU's labels
        D = oracle.distance_matrix(Pd, oracle.point_norms(Pd), Cd)
        ref_obj = float(D[np.arange(Pd.shape[0]), gpu["labels"]].sum(dtype=np.float64))
    dobj = abs(gpu["objective"] - ref_obj)
    assert dobj <= OBJ_RTOL * abs(ref_obj) + allowance, (
        f"{what}: objective {gpu['objective']!r} vs ref {ref_obj!r} (|d|={dobj:.3e})")
    exact = oracle.mean_centroids_f64(Pd, gpu["labels"], k)
    err = centroid_rel_err(gpu["centroids"], exact)
    assert err <= CEN_RTOL, f"{what}: centroids vs f64 means rel err {err:.3e}"
    if not diff.any():
        assert gpu["moved"] == ref.moved, f"{what}: moved {gpu['moved']} vs {ref.moved}"
        assert abs(gpu["changed"] - ref.changed) <= 1e-12, f"{what}: changed"
        # the reference's mean is an f32 running sum (clustering.py:287); on
        # adversarial inputs (thousands of identical rows) its own error vs the
        # exact mean exceeds CEN_RTOL — ours is within CEN_RTOL of the exact
        # mean (above), so the distance to the reference may add the reference's
        err_ref = centroid_rel_err(gpu["centroids"], ref.centroids)
        ref_self = centroid_rel_err(ref.centroids, exact)
        assert err_ref <= CEN_RTOL + ref_self, (f"{what}: centroids vs reference rel err {err_ref:.3e} "
                                                f"(reference vs exact means {ref_self:.3e})")
    return {"mismatches": int(diff.sum()), "exempt": int(exempt.sum()),
            "obj_rel": dobj / max(abs(ref_obj), 1e-300), "cen_rel": err}


def exact_rank_check(P, C, rows, lab_a, lab_b):
    """Direct f64 distances sum_t (p_t - c_t)^2 of `rows` to labels a and b:
    returns (da, db)."""
    P64 = np.asarray(P, dtype=np.float64)[rows]
    C64 = np.asarray(C, dtype=np.float64)
    da = ((P64 - C64[lab_a]) ** 2).sum(1)
    db = ((P64 - C64[lab_b]) ** 2).sum(1)
    return da, db


def check_step_strict(P, k, gpu, ref, *, what=""):
    """The north-star bar with no allowances beyond the stated one.

    * labels identical except rows whose f64 top-2 relative gap is below
      GAP_EXEMPT; any other mismatch must be a row the reference itself
      mis-ranks in its f32 expansion (clustering.py:311): the GPU label is
      the exact f64 argmin (direct sum of squares, lowest index on ties) and
      the reference's label is not — counted and returned as ``ref_f32_flips``;
    * objective within OBJ_RTOL of the reference's objective, no allowance;
    * centroids within CEN_RTOL of the f64 means of the GPU labels, and of
      the reference's centroids for every cluster no mismatched row touches.
    """
    C_in = gpu["centroids_in"]
    Pd = np.ascontiguousarray(P, dtype=np.float32)
    _, gap = oracle.top2_gap_f64(Pd, C_in)
    diff = gpu["labels"] != ref.labels
    gap_ex = diff & (gap < GAP_EXEMPT)
    rest = np.flatnonzero(diff & ~gap_ex)
    flips = 0
    if rest.size:
        g_lab, r_lab = gpu["labels"][rest], ref.labels[rest]
        dg, dr = exact_rank_check(Pd, C_in, rest, g_lab, r_lab)
        gpu_exact = (dg < dr) | ((dg == dr) & (g_lab < r_lab))
        # the reference's own f32 values rank its label first
        D32 = oracle.distance_matrix(Pd[rest], oracle.point_norms(Pd[rest]), np.asarray(C_in, np.float32))
        ref_f32 = D32[np.arange(rest.size), r_lab] <= D32[np.arange(rest.size), g_lab]
        moved = gpu["labels"][rest] != gpu["raw_labels"][rest]
        bad = ~(gpu_exact & ref_f32) & ~moved
        assert not bad.any(), (f"{what}: {int(bad.sum())} non-exempt label mismatches not explained by the "
                               f"reference's f32 rounding (rows {rest[bad][:8].tolist()}, gaps {gap[rest][bad][:8]})")
        flips = int(rest.size)
    obj_rel = abs(gpu["objective"] - ref.objective) / max(abs(ref.objective), 1e-300)
    assert obj_rel <= OBJ_RTOL, f"{what}: objective {gpu['objective']!r} vs ref {ref.objective!r} rel {obj_rel:.3e}"
    exact = oracle.mean_centroids_f64(Pd, gpu["labels"], k)
    cen_rel = centroid_rel_err(gpu["centroids"], exact)
    assert cen_rel <= CEN_RTOL, f"{what}: centroids vs f64 means rel err {cen_rel:.3e}"
    touched = np.zeros(k, dtype=bool)
    if diff.any():
        touched[gpu["labels"][diff]] = True
        touched[ref.labels[diff]] = True
    keep = ~touched
    cen_ref = centroid_rel_err(gpu["centroids"][keep], ref.centroids[keep]) if keep.any() else 0.0
    ref_self = centroid_rel_err(ref.centroids[keep], exact[keep]) if keep.any() else 0.0
    assert cen_ref <= CEN_RTOL + ref_self, (f"{what}: centroids vs reference rel err {cen_ref:.3e} "
                                            f"(reference vs exact means {ref_self:.3e})")
    if not diff.any():
        assert gpu["moved"] == ref.moved, f"{what}: moved {gpu['moved']} vs {ref.moved}"
        assert abs(gpu["changed"] - ref.changed) <= 1e-12, f"{what}: changed"
    return {"mismatches": int(diff.sum()), "gap_exempt": int(gap_ex.sum()), "ref_f32_flips": flips,
            "obj_rel": obj_rel, "cen_rel": cen_rel, "cen_ref_rel": cen_ref, "ref_mean_self_err": ref_self}
