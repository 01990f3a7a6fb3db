"""Certified BF16 screening (variant "bf16s", assign_screen_bf16.cu).

The screen must never certify a wrong argmin, the candidate pass must contain
the exact argmin, and the exact resolution must pick the f64 argmin with the
lowest index on ties (dense.py:56-68).  Parity bar as everywhere else
(tests/parity.py): labels equal except rows whose f64 top-2 gap is < 1e-5.
"""
import numpy as np
import pytest

import oracle
from conftest import make_rng
from parity import check_step

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(params=["bf16s", "fp8s"])
def screen_variant(request):
    """Both certified screens: BF16 (kind::f16) and E4M3 (kind::f8f6f4)."""
    return request.param


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _exact(P, C):
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    D = ((P64[:, None, :] - C64[None, :, :]) ** 2).sum(-1) if P.shape[0] * C.shape[0] * P.shape[1] < 4e8 else \
        (P64 * P64).sum(1)[:, None] - 2 * P64 @ C64.T + (C64 * C64).sum(1)[None, :]
    srt = np.sort(D, 1)
    gap = (srt[:, 1] - srt[:, 0]) / np.maximum(np.abs(srt[:, 0]), 1e-300)
    return D.argmin(1), gap


@pytest.mark.parametrize("n,d,k", [(1000, 40, 17), (777, 100, 300), (4096, 64, 64), (300, 33, 1),
                                   (5000, 128, 1024), (1500, 96, 129), (5000, 64, 4096),
                                   (3000, 256, 200), (2500, 200, 77), (20000, 128, 1024)])
def test_bf16_lockstep_ragged_shapes(n, d, k, screen_variant):
    from paper_2501_05587_b200.engine import LloydEngine
    P = oracle.make_blobs(n, d, max(k, 1), seed=n + d)
    lab = oracle.init_assignments(n, k, 1)
    C = oracle.mean_centroids(P, lab, k)
    eng = LloydEngine(P, k, variant=screen_variant, max_iters=1)
    pn = oracle.point_norms(P)
    for t in range(4):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        gpu = eng.step_from(C, lab)
        check_step(P, C, lab, k, gpu, ref=ref, what=f"bf16s n={n} d={d} k={k} it{t}")
        C, lab = ref.centroids, ref.labels


@pytest.mark.parametrize("spread", [3.0, 0.3])
def test_bf16_labels_are_exact_argmin(spread, screen_variant):
    """Certified rows and candidate-resolved rows carry the exact f64 argmin;
    only rows sent on to the 3xTF32 resolver may differ, and only inside the
    1e-5 gap exemption."""
    from paper_2501_05587_b200.engine import LloydEngine
    rng = make_rng(21)
    n, d, k = 6000, 128, 512
    P = rng.normal(0, 3, size=(n, d)).astype(np.float32)
    C = (rng.normal(0, spread, size=(k, d)) + 1.0).astype(np.float32)
    eng = LloydEngine(P, k, variant=screen_variant, max_iters=1)
    out = eng.step_from(C, np.zeros(n, dtype=np.int32))
    amb, ovf = int(eng.amb_count.item()), int(eng.ovf_count.item())
    exact, gap = _exact(P, C)
    bad = (out["raw_labels"] != exact) & (gap >= 1e-5)
    assert not bad.any(), f"{int(bad.sum())} wrong labels (ambiguous {amb}, overflow {ovf})"
    if ovf == 0:
        # no 3xTF32 rows: every label is exact, ties included
        np.testing.assert_array_equal(out["raw_labels"], exact)
    print(f"spread {spread}: ambiguous {amb}/{n}, overflow {ovf}")


def test_bf16_duplicate_centroids_tie_to_lowest_index(screen_variant):
    from paper_2501_05587_b200.engine import LloydEngine
    rng = make_rng(22)
    n, d, k = 3000, 64, 64
    P = rng.normal(0, 1, size=(n, d)).astype(np.float32)
    C = rng.normal(0, 1, size=(k, d)).astype(np.float32)
    C[40] = C[7]
    C[63] = C[7]
    eng = LloydEngine(P, k, variant=screen_variant, max_iters=1)
    out = eng.step_from(C, np.zeros(n, dtype=np.int32))
    assert not np.any(out["raw_labels"] == 40)
    assert not np.any(out["raw_labels"] == 63)
    exact, _ = _exact(P, C)
    np.testing.assert_array_equal(out["raw_labels"], exact)


def test_bf16_candidate_overflow_goes_to_3xtf32(screen_variant):
    """A cluster of 70 near-identical centroids gives its points more
    candidates than the pass-2 list holds (64): those rows take the 3xTF32
    path, the rest stay exact."""
    from paper_2501_05587_b200.engine import LloydEngine
    rng = make_rng(23)
    n, d, k = 4000, 96, 200
    C = rng.uniform(-10, 10, size=(k, d)).astype(np.float32)
    C[:70] = C[0] + rng.normal(0, 1e-3, size=(70, d)).astype(np.float32)
    true = np.where(rng.random(n) < 0.1, 0, rng.integers(70, k, size=n))
    P = (C[true] + rng.normal(0, 1, size=(n, d))).astype(np.float32)
    eng = LloydEngine(P, k, variant=screen_variant, max_iters=1)
    out = eng.step_from(C, np.zeros(n, dtype=np.int32))
    ovf = int(eng.ovf_count.item())
    assert ovf > 0
    assert ovf < n // 4
    exact, gap = _exact(P, C)
    ovf_rows = np.zeros(n, dtype=bool)
    ovf_rows[eng.ovf_list[:ovf].cpu().numpy()] = True
    raw = out["raw_labels"]
    # candidate-resolved and certified rows: exact argmin
    np.testing.assert_array_equal(raw[~ovf_rows], exact[~ovf_rows])
    # 3xTF32 rows: f32-faithful expansion (|p|^2 - 2<p,c> + |c|^2), so the
    # chosen distance is within a few f32 ulps of |p|^2 + |c|^2 of the minimum
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    Dg = ((P64 - C64[raw]) ** 2).sum(1)
    De = ((P64 - C64[exact]) ** 2).sum(1)
    scale = (P64 ** 2).sum(1) + (C64 ** 2).sum(1).max()
    assert np.all(Dg - De <= 2.0 ** -20 * scale)


def test_bf16_bypass_when_most_rows_ambiguous(screen_variant):
    """Centroids bunched near the global mean (as right after a random-label
    init at large n): most rows are ambiguous, the candidate pass is bypassed
    and every ambiguous row goes to the 3xTF32 resolver."""
    from paper_2501_05587_b200.engine import LloydEngine
    rng = make_rng(24)
    n, d, k = 8000, 128, 256
    P = oracle.make_blobs(n, d, k, seed=5)
    C = (P.mean(0)[None, :] + rng.normal(0, 1e-2, size=(k, d))).astype(np.float32)
    lab = rng.integers(0, k, size=n).astype(np.int32)
    eng = LloydEngine(P, k, variant=screen_variant, max_iters=1)
    ref = oracle.lloyd_step(P, oracle.point_norms(P), C, lab, k)
    gpu = eng.step_from(C, lab)
    assert int(eng.amb_count.item()) > n // 4
    assert int(eng.ovf_count.item()) == int(eng.amb_count.item())
    check_step(P, C, lab, k, gpu, ref=ref, what="bf16s bypass")


def test_bf16_full_run_matches_reference(screen_variant):
    import paper_2501_05587_b200 as pcb
    P = oracle.make_blobs(20000, 128, 64, seed=4)
    a = pcb.run_lloyd(P, pcb.KKMeansConfig(k=64, max_iters=8, variant=screen_variant))
    ref = oracle.run_lloyd(P, 64, max_iters=8)
    np.testing.assert_allclose(a.objective_history, ref.objective_history, rtol=1e-6)
    np.testing.assert_array_equal(a.labels, ref.labels)


def test_bf16_predict_matches_assignment(screen_variant):
    import paper_2501_05587_b200 as pcb
    P = oracle.make_blobs(5000, 64, 32, seed=9)
    est = pcb.KernelKMeans(n_clusters=32, algorithm="lloyd", max_iter=5, variant=screen_variant).fit(P)
    np.testing.assert_array_equal(est.predict(P[:1000]), est.labels_[:1000])


def test_bf16_relayout_keeps_results(screen_variant):
    """Labels, objective and centroids do not depend on the screen's row
    layout (pcb_screen_relayout_bf16): lockstep steps before and after the
    rows are re-laid out by label agree bit for bit."""
    from paper_2501_05587_b200.engine import LloydEngine
    n, d, k = 30000, 128, 256
    P = oracle.make_blobs(n, d, k, seed=6)
    lab = oracle.init_assignments(n, k, 0)
    C = oracle.mean_centroids(P, lab, k)
    pn = oracle.point_norms(P)
    for _ in range(3):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        C, lab = ref.centroids, ref.labels
    eng = LloydEngine(P, k, variant=screen_variant, max_iters=1)
    a = eng.step_from(C, lab)
    eng.relayout()  # perm of the step just taken: rows grouped by label
    assert eng.orig is not None
    orig = eng.orig.cpu().numpy()
    assert np.array_equal(np.sort(orig), np.arange(n))
    assert np.all(np.diff(a["labels"][orig]) >= 0)  # grouped by label
    b = eng.step_from(C, lab)
    np.testing.assert_array_equal(a["raw_labels"], b["raw_labels"])
    np.testing.assert_array_equal(a["labels"], b["labels"])
    assert abs(a["objective"] - b["objective"]) <= 1e-12 * abs(a["objective"])  # f64 atomics order
    np.testing.assert_allclose(a["centroids"], b["centroids"], rtol=1e-6)
    ref = oracle.lloyd_step(P, pn, C, lab, k)
    check_step(P, C, lab, k, b, ref=ref, what="bf16s after relayout")


@pytest.mark.parametrize("variant,n,d,k", [("fp8s", 3000, 784, 256), ("fp8s", 1500, 1000, 60),
                                           ("fp8s", 2000, 300, 129), ("bf16s", 2000, 400, 100),
                                           ("bf16s", 1200, 512, 64)])
def test_long_rows_one_resident_tile(variant, n, d, k):
    """Rows of 5-8 operand chunks run with one resident row tile of 128 and
    the warp-per-row exact resolver (d > 256)."""
    from paper_2501_05587_b200.engine import LloydEngine
    P = oracle.make_blobs(n, d, k, seed=d)
    lab = oracle.init_assignments(n, k, 2)
    C = oracle.mean_centroids(P, lab, k)
    eng = LloydEngine(P, k, variant=variant, max_iters=1)
    pn = oracle.point_norms(P)
    for t in range(4):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        gpu = eng.step_from(C, lab)
        check_step(P, C, lab, k, gpu, ref=ref, what=f"{variant} n={n} d={d} k={k} it{t}")
        C, lab = ref.centroids, ref.labels


@pytest.mark.parametrize("case", ["wide_range", "identical", "integer_grid"])
def test_screen_hard_inputs(case, screen_variant):
    """Inputs that stress the low-precision screen: a wide dynamic range across
    columns (E4M3 scale set by the largest entry, small entries subnormal),
    all points identical (every key tied), small integers (exact ties between
    centroids).  Labels must still match the reference step."""
    from paper_2501_05587_b200.engine import LloydEngine
    rng = make_rng(41)
    n, d, k = 3000, 48, 24
    if case == "wide_range":
        P = (rng.normal(size=(n, d)) * np.logspace(-3, 3, d)[None, :]).astype(np.float32)
    elif case == "identical":
        P = np.repeat(rng.normal(size=(1, d)), n, axis=0).astype(np.float32)
    else:
        P = rng.integers(0, 4, size=(n, d)).astype(np.float32)
    lab = oracle.init_assignments(n, k, 3)
    C = oracle.mean_centroids(P, lab, k)
    eng = LloydEngine(P, k, variant=screen_variant, max_iters=1)
    pn = oracle.point_norms(P)
    for t in range(3):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        gpu = eng.step_from(C, lab)
        check_step(P, C, lab, k, gpu, ref=ref, what=f"{screen_variant} {case} it{t}")
        C, lab = ref.centroids, ref.labels
