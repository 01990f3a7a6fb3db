"""Delta centroid update (update.cu): per-cluster f64 sums maintained over the
changed rows, objective from sum |p|^2 - 2 <c, S> + n |c|^2.  Must agree with
the full counting-sort update to f64 rounding, on every variant, and fall
back to the full update when rows churn or clusters empty out."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(P, k, update, variant="auto", iters=20, dtype=np.float32):
    from paper_2501_05587_b200.engine import LloydEngine
    eng = LloydEngine(P, k, variant=variant, dtype=dtype, max_iters=iters, update=update)
    eng.init_labels_device(0)
    eng.init_centroids_from_labels()
    eng.state.zero_()
    modes, objs, cents = [], [], []
    for t in range(iters):
        eng.iteration(t)
        torch.cuda.synchronize()
        modes.append(int(eng.state[6].item()))
        cents.append(eng.C.cpu().numpy().copy())
    out = eng.collect()
    return out, modes, cents, eng


@pytest.mark.parametrize("variant,n,d,k", [("bf16s", 40000, 128, 64), ("fp8s", 40000, 128, 64), ("rowreg", 30000, 16, 32),
                                           ("rowreg", 30000, 8, 40), ("rowreg", 30000, 12, 32),
                                           ("tiled", 20000, 48, 40), ("tc3xtf32", 20000, 64, 50)])
def test_delta_matches_full_update(variant, n, d, k):
    P = oracle.make_blobs(n, d, k, seed=3)
    a, modes, ca, _ = _run(P, k, "auto", variant)
    b, _, cb, _ = _run(P, k, "full", variant)
    assert any(m & 1 for m in modes), "the delta update never ran"
    assert modes[0] == 0  # sums not valid yet: full
    if variant in ("fp8s", "bf16s") or (variant == "rowreg" and d in (8, 16)):
        # delta after delta: the count pass (screens) or the constant-bank
        # small-d kernel applied the changed-row sums (mode 3)
        assert 3 in modes, modes
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_allclose(a.objective_history, b.objective_history, rtol=1e-10)
    for x, y in zip(ca, cb):
        np.testing.assert_allclose(x, y, rtol=1e-6, atol=1e-6)


def test_delta_matches_full_update_f64():
    P = oracle.make_blobs(20000, 24, 30, seed=8).astype(np.float64)
    a, modes, _, _ = _run(P, 30, "auto", dtype=np.float64)
    b, _, _, _ = _run(P, 30, "full", dtype=np.float64)
    assert any(m & 1 for m in modes)
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_allclose(a.objective_history, b.objective_history, rtol=1e-10)
    np.testing.assert_allclose(a.centroids, b.centroids, rtol=1e-12, atol=1e-12)


def test_delta_run_matches_reference():
    """Free-running Lloyd against the reference restatement (f64 exact sums
    vs the reference's f32 expansion: labels equal on well-separated blobs)."""
    import paper_2501_05587_b200 as pcb
    P = oracle.make_blobs(30000, 64, 48, seed=12)
    res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=48, max_iters=15))
    ref = oracle.run_lloyd(P, 48, max_iters=15)
    np.testing.assert_array_equal(res.labels, ref.labels)
    np.testing.assert_allclose(res.objective_history, ref.objective_history, rtol=1e-6)


def test_repair_keeps_delta_sums():
    """Duplicate points empty clusters out: the repair moves points and the
    delta update's sums S with them, so later delta iterations still match
    the full update bit for bit (labels, repairs) and the objective."""
    from paper_2501_05587_b200.engine import LloydEngine
    rng = np.random.default_rng(4)
    base = rng.normal(size=(5, 8)).astype(np.float32)
    P = np.repeat(base, 400, axis=0) + rng.normal(0, 1e-3, size=(2000, 8)).astype(np.float32)
    k = 12
    a, modes, _, _ = _run(P, k, "auto", "tiled", iters=10)
    b, _, _, _ = _run(P, k, "full", "tiled", iters=10)
    rep = np.flatnonzero(np.asarray(a.repairs) > 0)
    assert rep.size, "no repair ran"
    assert any(modes[t] == 1 for t in range(int(rep[0]) + 1, len(modes))), modes
    np.testing.assert_array_equal(a.labels, b.labels)
    np.testing.assert_array_equal(a.repairs, b.repairs)
    np.testing.assert_allclose(a.objective_history, b.objective_history, rtol=1e-9)
    ref = oracle.run_lloyd(P, k, max_iters=10)
    np.testing.assert_array_equal(a.repairs, ref.repairs)


def test_history_ring_matches_pinned_history():
    """label_history of an eager fit (streamed through the pinned slot ring)
    equals the graph-replayed fit's (one pinned buffer), iteration by iteration,
    including a fit that converges early (the ring drops the no-op iterations)."""
    from paper_2501_05587_b200.engine import LloydEngine
    P = oracle.make_blobs(30000, 48, 20, seed=12)
    outs = []
    for graph in (True, False):
        eng = LloydEngine(P, 20, max_iters=12)
        eng.init_labels_device(0)
        eng.init_centroids_from_labels()
        outs.append(eng.run(12, check_convergence=True, tol=0.0, record_history=True, graph=graph))
    a, b = outs
    assert a.iterations_run == b.iterations_run and len(a.label_history) == a.iterations_run
    for x, y in zip(a.label_history, b.label_history):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(a.labels, b.labels)
