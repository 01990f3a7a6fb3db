"""The tcgen05 3xTF32 assignment kernel: numerics probes and ragged shapes."""
import ctypes

import numpy as np
import pytest

import oracle
from conftest import make_rng
from parity import check_step

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _tc_raw(Phi, Plo, Chi, Clo, pnorm, cnorm, d):
    from paper_2501_05587_b200 import _lib
    n, ld = Phi.shape
    k = Chi.shape[0]
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    mind = torch.empty(n, dtype=torch.float32, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.call("pcb_assign_tc_f32", _p(Phi), _p(Plo), ld, _p(pnorm), n, d, _p(Chi), _p(Clo), _p(cnorm), k,
              None, _p(lab), _p(mind), None, None, st)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), mind.cpu().numpy()


def test_tf32_operand_conversion_probe():
    """How does kind::tf32 read an f32 operand whose low 13 bits are set?
    x = 1 + 2^-11 + 2^-12: truncation gives 1, round-to-nearest 1 + 2^-10.
    Either is fine for the 3xTF32 split (hi is pre-rounded); recorded for DESIGN.md."""
    n, ld, k = 128, 32, 1
    x = np.float32(1.0 + 2.0 ** -11 + 2.0 ** -12)
    Phi = torch.zeros((n, ld), device="cuda")
    Phi[:, 0] = float(x)
    Plo = torch.zeros_like(Phi)
    Chi = torch.zeros((k, ld), device="cuda")
    Chi[0, 0] = 1.0
    Clo = torch.zeros_like(Chi)
    _, mind = _tc_raw(Phi, Plo, Chi, Clo, torch.zeros(n, device="cuda"), torch.zeros(k, device="cuda"), 32)
    seen = -mind / 2.0
    assert np.all(seen == seen[0])
    print(f"tf32 conversion of {x!r}: hardware used {seen[0]!r} "
          f"({'truncation' if seen[0] == 1.0 else 'round-to-nearest' if seen[0] == 1 + 2**-10 else 'other'})")
    assert seen[0] in (np.float32(1.0), np.float32(1 + 2.0 ** -10), x)


def test_3xtf32_dot_products_fp32_faithful():
    """Split-precision products vs f64: error ~2^-21 relative to sum |p||c|."""
    from paper_2501_05587_b200 import _lib
    rng = make_rng(3)
    n, d, k = 1000, 128, 300
    P = rng.uniform(-10, 10, size=(n, d)).astype(np.float32)
    C = rng.uniform(-10, 10, size=(k, d)).astype(np.float32)
    from paper_2501_05587_b200.engine import LloydEngine
    eng = LloydEngine(P, k, variant="tc3xtf32", max_iters=1)
    eng.set_centroids(C)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    lab = torch.empty(n, dtype=torch.int32, device="cuda")
    mind = torch.empty(n, dtype=torch.float32, device="cuda")
    _lib.call("pcb_assign_tc_f32", _p(eng.P_hi), _p(eng.P_lo), eng.ld, _p(eng.pnorm), n, d, _p(eng.C_hi),
              _p(eng.C_lo), _p(eng.cnorm), k, None, _p(lab), _p(mind), None, None, st)
    torch.cuda.synchronize()
    lab = lab.cpu().numpy()
    mind = mind.cpu().numpy().astype(np.float64)
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    D = ((P64[:, None, :] - C64[None, :, :]) ** 2).sum(-1)
    scale = (np.abs(P64) @ np.abs(C64).T)
    own_true = D[np.arange(n), lab]
    err = np.abs(mind - own_true) / scale[np.arange(n), lab]
    assert err.max() < 2.0 ** -18, err.max()
    d1 = D.min(1)
    gap_ok = (np.sort(D, 1)[:, 1] - d1) > 1e-5 * d1
    assert np.all(lab[gap_ok] == D.argmin(1)[gap_ok])


@pytest.mark.parametrize("n,d,k", [(1000, 40, 17), (777, 100, 300), (4096, 64, 64), (300, 33, 1),
                                   (5000, 128, 1024), (2000, 784, 256), (1500, 96, 129), (5000, 64, 4096)])
def test_tc_lockstep_ragged_shapes(n, d, k):
    from paper_2501_05587_b200.engine import LloydEngine
    P = oracle.make_blobs(n, d, max(k, 1), seed=n + d)
    lab = oracle.init_assignments(n, k, 1)
    C = oracle.mean_centroids(P, lab, k)
    eng = LloydEngine(P, k, variant="tc3xtf32", max_iters=1)
    gpu = eng.step_from(C, lab)
    check_step(P, C, lab, k, gpu, what=f"tc n={n} d={d} k={k}")


def test_tc_full_run_matches_ffma_run():
    import paper_2501_05587_b200 as pcb
    P = oracle.make_blobs(20000, 128, 64, seed=4)
    a = pcb.run_lloyd(P, pcb.KKMeansConfig(k=64, max_iters=8, variant="tc3xtf32"))
    b = pcb.run_lloyd(P, pcb.KKMeansConfig(k=64, max_iters=8, variant="tiled"))
    ref = oracle.run_lloyd(P, 64, max_iters=8)
    for r in (a, b):
        np.testing.assert_allclose(r.objective_history, ref.objective_history, rtol=1e-6)
    np.testing.assert_array_equal(a.labels, ref.labels)


# ---------------------------------------------------------------------------
# certified 1xTF32 screening (variant tc1xtf32s)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,d,k", [(1000, 40, 17), (777, 100, 300), (4096, 64, 64), (300, 32, 1),
                                   (5000, 128, 1024), (2000, 784, 256), (1500, 96, 129), (5000, 64, 4096),
                                   (20000, 128, 1024)])
def test_screen_lockstep_ragged_shapes(n, d, k):
    from paper_2501_05587_b200.engine import LloydEngine
    P = oracle.make_blobs(n, d, max(k, 1), seed=n + d)
    lab = oracle.init_assignments(n, k, 1)
    C = oracle.mean_centroids(P, lab, k)
    eng = LloydEngine(P, k, variant="tc1xtf32s", max_iters=1)
    pn = oracle.point_norms(P)
    for t in range(3):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        gpu = eng.step_from(C, lab)
        check_step(P, C, lab, k, gpu, ref=ref, what=f"screen n={n} d={d} k={k} it{t}")
        C, lab = ref.centroids, ref.labels


def test_screen_certified_labels_are_exact_argmin():
    """Rows not sent to the fallback must carry the exact (f64) argmin."""
    from paper_2501_05587_b200.engine import LloydEngine
    rng = make_rng(11)
    n, d, k = 6000, 128, 512
    P = rng.normal(0, 3, size=(n, d)).astype(np.float32)
    C = rng.normal(0, 3, size=(k, d)).astype(np.float32)
    eng = LloydEngine(P, k, variant="tc1xtf32s", max_iters=1)
    eng.set_centroids(C)
    out = eng.step_from(C, np.zeros(n, dtype=np.int32))
    amb = int(eng.amb_count.item())
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    D = (P64 * P64).sum(1)[:, None] - 2 * P64 @ C64.T + (C64 * C64).sum(1)[None, :]
    exact = D.argmin(1)
    srt = np.sort(D, 1)
    gap = (srt[:, 1] - srt[:, 0]) / np.abs(srt[:, 0])
    bad = (out["raw_labels"] != exact) & (gap >= 1e-5)
    assert not bad.any(), f"{int(bad.sum())} wrong certified labels"
    print(f"ambiguous rows: {amb}/{n}")
    assert amb < n


def test_screen_duplicate_centroids_tie_to_lowest_index():
    from paper_2501_05587_b200.engine import LloydEngine
    rng = make_rng(12)
    n, d, k = 3000, 64, 64
    P = rng.normal(0, 1, size=(n, d)).astype(np.float32)
    C = rng.normal(0, 1, size=(k, d)).astype(np.float32)
    C[40] = C[7]  # exact duplicate: every row nearest to it must pick 7
    eng = LloydEngine(P, k, variant="tc1xtf32s", max_iters=1)
    out = eng.step_from(C, np.zeros(n, dtype=np.int32))
    assert not np.any(out["raw_labels"] == 40)
    assert eng.amb_count.item() >= np.sum(out["raw_labels"] == 7)


def test_screen_full_run_matches_reference():
    import paper_2501_05587_b200 as pcb
    P = oracle.make_blobs(20000, 128, 64, seed=4)
    a = pcb.run_lloyd(P, pcb.KKMeansConfig(k=64, max_iters=8, variant="tc1xtf32s"))
    ref = oracle.run_lloyd(P, 64, max_iters=8)
    np.testing.assert_allclose(a.objective_history, ref.objective_history, rtol=1e-6)
    np.testing.assert_array_equal(a.labels, ref.labels)


# ---------------------------------------------------------------------------
# delta-chunked P.C.P^T ablation
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("variant", ["delta", "deltatc"])
@pytest.mark.parametrize("n,d,k", [(500, 2, 7), (1000, 16, 40), (1500, 100, 33), (600, 784, 20), (700, 7, 17),
                                   (300, 8, 16), (1000, 31, 129)])
def test_delta_chunked_lockstep(variant, n, d, k):
    from paper_2501_05587_b200.engine import LloydEngine
    P = oracle.make_blobs(n, d, k, seed=d)
    lab = oracle.init_assignments(n, k, 2)
    C = oracle.mean_centroids(P, lab, k)
    eng = LloydEngine(P, k, variant=variant, max_iters=1)
    pn = oracle.point_norms(P)
    for t in range(3):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        gpu = eng.step_from(C, lab)
        check_step(P, C, lab, k, gpu, ref=ref, what=f"{variant} n={n} d={d} k={k} it{t}")
        C, lab = ref.centroids, ref.labels


@pytest.mark.parametrize("variant", ["delta", "deltatc"])
def test_delta_chunked_worked_examples(variant):
    """The attachment's worked values via the chunked kernel (analysis.py oracle)."""
    from paper_2501_05587_b200.engine import LloydEngine
    for p, c, want in (([3.0], [7.0], 16.0), ([1.0], [7.0], 36.0), ([5.0, 2.0], [1.0, 4.0], 20.0),
                       ([4.0, 3.0, 2.0], [5.0, 2.0, 3.0], 3.0)):
        P = np.array([p], dtype=np.float32)
        eng = LloydEngine(P, 1, variant=variant, max_iters=1)
        eng.set_centroids(np.array([c], dtype=np.float32))
        out = eng.step_from(np.array([c], dtype=np.float32), np.zeros(1, dtype=np.int32))
        assert out["mind"][0] == pytest.approx(want, abs=1e-5)
        assert out["mind"][0] == pytest.approx(oracle.augmented_distance(p, c), abs=1e-5)


def test_delta_tc_full_distances():
    """Every (point, centroid) value of the tensor-core chunked form against the
    f64 distance, through predict-free single-centroid runs: k = 1 makes mind the
    chunked D of that centroid, for d spanning partial blocks and chunks."""
    from paper_2501_05587_b200.engine import LloydEngine
    rng = np.random.default_rng(5)
    for d in (1, 7, 8, 9, 31, 32, 33, 100):
        P = rng.normal(size=(300, d)).astype(np.float32) * 3
        c = rng.normal(size=(1, d)).astype(np.float32)
        eng = LloydEngine(P, 1, variant="deltatc", max_iters=1)
        out = eng.step_from(c, np.zeros(300, dtype=np.int32))
        exact = ((P.astype(np.float64) - c.astype(np.float64)) ** 2).sum(1)
        scale = (P.astype(np.float64) ** 2).sum(1) + (c.astype(np.float64) ** 2).sum()
        assert np.all(np.abs(out["mind"] - exact) <= 1e-5 * scale + 1e-6), d


def test_delta_tc_ablation_matches_fused():
    """The chunked tensor-core form and the fused 3xTF32 GEMM agree on a fit
    (both exact up to the f32 expansion's near-ties)."""
    import paper_2501_05587_b200 as pcb
    P = oracle.make_blobs(20000, 64, 48, seed=3)
    a = pcb.run_lloyd(P, pcb.KKMeansConfig(k=48, max_iters=6, variant="deltatc"))
    ref = oracle.run_lloyd(P, 48, max_iters=6)
    np.testing.assert_allclose(a.objective_history, ref.objective_history, rtol=1e-6)
    np.testing.assert_array_equal(a.labels, ref.labels)


# ---------------------------------------------------------------------------
# small-d FFMA2 kernel (assign_rowpair) vs the scalar FFMA kernel (assign_rowreg)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("d", [1, 2, 3, 5, 8, 13, 16, 17, 32])
@pytest.mark.parametrize("k", [1, 7, 64, 1001])
def test_rowpair_bit_identical_to_rowreg(d, k, monkeypatch):
    """Same per-pair f32 arithmetic in the same order: labels and own distances
    are bit-identical (odd k pads a +inf centroid; k = 1001 spans several
    shared-memory chunks for d = 32), and both match the oracle step."""
    from paper_2501_05587_b200.engine import LloydEngine
    n = 5000 + 37
    P = oracle.make_blobs(n, d, min(k, 50), seed=d + k)
    lab = oracle.init_assignments(n, k, 1) if k <= n else np.zeros(n, np.int32)
    C = oracle.make_blobs(k, d, min(k, 50), seed=d * 7 + 1)
    outs = []
    for scalar in (False, True):
        if scalar:
            monkeypatch.setenv("PCB_ROWREG_SCALAR", "1")
        else:
            monkeypatch.delenv("PCB_ROWREG_SCALAR", raising=False)
        eng = LloydEngine(P, k, variant="rowreg", max_iters=1)
        outs.append(eng.step_from(C, lab))
    np.testing.assert_array_equal(outs[0]["raw_labels"], outs[1]["raw_labels"])
    np.testing.assert_array_equal(outs[0]["mind"].view(np.uint32), outs[1]["mind"].view(np.uint32))


@pytest.mark.parametrize("d,k", [(2, 10), (16, 64), (16, 7), (8, 40), (5, 33),
                                 (16, 120), (16, 121), (8, 227), (8, 228)])
@pytest.mark.parametrize("n", [400_003, 1_000_000])
def test_small_d_full_size_bit_identical_to_rowreg(n, d, k, monkeypatch):
    """The default small-d kernel at c2's size (several rounds per block, a
    ragged last round; assign_rowcst for d in {8, 16}, the ragged k = 7 / 33
    tails of its centroid blocks, the constant bank's capacity edge k (d + 1)
    = 2048 / 2049 -> assign_rowpair, assign_rowpair for d = 2, 5): labels and
    own distances bit-identical to the scalar kernel."""
    from paper_2501_05587_b200.engine import LloydEngine
    P = oracle.make_blobs(n, d, min(k, 50), seed=n % 97 + d)
    lab = oracle.init_assignments(n, k, 1)
    C = oracle.make_blobs(k, d, min(k, 50), seed=d * 3 + 5)
    outs = []
    for scalar in (False, True):
        if scalar:
            monkeypatch.setenv("PCB_ROWREG_SCALAR", "1")
        else:
            monkeypatch.delenv("PCB_ROWREG_SCALAR", raising=False)
        eng = LloydEngine(P, k, variant="rowreg", max_iters=1)
        outs.append(eng.step_from(C, lab))
    np.testing.assert_array_equal(outs[0]["raw_labels"], outs[1]["raw_labels"])
    np.testing.assert_array_equal(outs[0]["mind"].view(np.uint32), outs[1]["mind"].view(np.uint32))
