"""GPU parity of the Lloyd path against the reference (golden) and the oracle.

All tests call through the C ABI (ctypes -> libpopcorn_b200.so) on cuda:0.
Tolerances are those of BASELINE.json's north star, stated in tests/parity.py.
"""
import numpy as np
import pytest

import oracle
from conftest import golden_runs, make_rng
from parity import check_step, centroid_rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _engine(P, k, dtype=np.float32, variant="auto"):
    from paper_2501_05587_b200.engine import LloydEngine
    return LloydEngine(P, k, dtype=dtype, variant=variant, max_iters=1)


def _run_meta(golden, name):
    k, seed, cc, mi, dtc = (int(x) for x in golden[f"run_{name}_meta"])
    return k, seed, bool(cc), mi, (np.float32 if dtc == 1 else np.float64)


# --------------------------------------------------------------------------
# lockstep against the reference's own per-iteration centroids and labels
# --------------------------------------------------------------------------
@pytest.mark.parametrize("variant", ["auto", "tiled"])
def test_lockstep_against_golden(golden, variant):
    checked = 0
    for name in golden_runs(golden):
        k, seed, cc, mi, dtype = _run_meta(golden, name)
        P = golden[f"run_{name}_P"]
        labs = golden[f"run_{name}_labels"]
        cents = golden[f"run_{name}_centroids"]
        lab0 = oracle.init_assignments(P.shape[0], k, seed)
        C0 = oracle.mean_centroids(np.ascontiguousarray(P, dtype=dtype), lab0, k)
        eng = _engine(P, k, dtype, variant)
        prevs = [lab0] + [labs[t] for t in range(labs.shape[0] - 1)]
        cins = [C0] + [cents[t] for t in range(cents.shape[0] - 1)]
        for t, (lp, cin) in enumerate(zip(prevs, cins)):
            gpu = eng.step_from(cin, lp)
            check_step(P, cin, lp, k, gpu, dtype=dtype, what=f"{name} it{t} {variant}")
            checked += 1
    assert checked > 300


def test_free_running_f64_identical_to_reference(golden):
    """f64 is the reference's oracle precision: full label sequences must match."""
    import paper_2501_05587_b200 as pcb
    for name in golden_runs(golden):
        k, seed, cc, mi, dtype = _run_meta(golden, name)
        if dtype != np.float64:
            continue
        P = golden[f"run_{name}_P"]
        res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=k, seed=seed, max_iters=mi, check_convergence=cc,
                                                 tol=float(golden[f"run_{name}_tol"]), dtype=np.float64))
        ref_l = golden[f"run_{name}_labels"]
        assert res.iterations_run == ref_l.shape[0], name
        np.testing.assert_array_equal(np.stack(res.label_history), ref_l, err_msg=name)
        np.testing.assert_allclose(res.objective_history, golden[f"run_{name}_objective"],
                                   rtol=1e-12, atol=1e-12, err_msg=name)
        np.testing.assert_array_equal(res.repairs, golden[f"run_{name}_repairs"], err_msg=name)
        assert res.converged == bool(golden[f"run_{name}_converged"])


def test_free_running_f32_small_instances(golden):
    """f32 free-running runs: identical label sequences on every golden
    instance whose top-2 gaps stay above the exemption (most of them), and
    the reference's final objective within 1e-6 otherwise."""
    import paper_2501_05587_b200 as pcb
    identical = 0
    total = 0
    for name in golden_runs(golden):
        k, seed, cc, mi, dtype = _run_meta(golden, name)
        if dtype != np.float32:
            continue
        total += 1
        P = golden[f"run_{name}_P"]
        res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=k, seed=seed, max_iters=mi, check_convergence=cc,
                                                 tol=float(golden[f"run_{name}_tol"])))
        ref_l = golden[f"run_{name}_labels"]
        if res.iterations_run == ref_l.shape[0] and np.array_equal(np.stack(res.label_history), ref_l):
            identical += 1
            np.testing.assert_array_equal(res.repairs, golden[f"run_{name}_repairs"])
    assert identical >= total - 2, f"only {identical}/{total} f32 runs identical"


def test_reference_lloyd_examples():
    """The reference's own Lloyd tests (test_clustering.py:139-151)."""
    import paper_2501_05587_b200 as pcb
    P = make_rng(5).random((4, 2))
    res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=4, check_convergence=True))
    assert res.iterations_run == 1
    assert res.objective_history[-1] == pytest.approx(0.0, abs=1e-6)
    P = np.array([[0.0], [0.1], [10.0], [10.1]])
    res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=2, seed=1, dtype=np.float64, check_convergence=True))
    groups = {frozenset(np.flatnonzero(res.labels == j).tolist()) for j in range(2)}
    assert groups == {frozenset({0, 1}), frozenset({2, 3})}
    assert res.objective_history[-1] == pytest.approx(0.01, rel=1e-9)


def test_convergence_semantics():
    import paper_2501_05587_b200 as pcb
    P = make_rng(16).random((60, 4))
    res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=4, check_convergence=True, tol=1.0))
    assert res.converged and res.iterations_run == 1
    res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=4, check_convergence=False, max_iters=7))
    assert not res.converged and res.iterations_run == 7
    assert len(res.label_history) == 7 and res.repairs.shape == (7,)
    assert res.timings.pairwise_distances_seconds > 0 and res.timings.argmin_update_seconds > 0


# --------------------------------------------------------------------------
# benchmark-config shapes (subsampled) against the oracle, lockstep
# --------------------------------------------------------------------------
SHAPES = {
    "c1_full": (100_000, 2, 10),
    "c2_sub": (200_000, 16, 64),
    "c3_sub": (30_000, 128, 1024),
    "c4_sub": (8_000, 784, 256),
    "c5_sub": (12_000, 64, 4096),
}


@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_lockstep_config_shapes(shape):
    n, d, k = SHAPES[shape]
    P = oracle.make_blobs(n, d, k, seed=0)
    lab = oracle.init_assignments(n, k, 0)
    C = oracle.mean_centroids(P, lab, k)
    eng = _engine(P, k)
    pn = oracle.point_norms(P)
    for t in range(3):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        gpu = eng.step_from(C, lab)
        check_step(P, C, lab, k, gpu, ref=ref, what=f"{shape} it{t}")
        C, lab = ref.centroids, ref.labels


def test_predict_matches_assignment():
    from paper_2501_05587_b200 import KernelKMeans
    rng = make_rng(5)
    X = np.vstack([rng.normal(loc=c, scale=0.4, size=(20, 3)) for c in (0.0, 5.0, 10.0)])
    est = KernelKMeans(n_clusters=3, algorithm="lloyd", random_state=3, check_convergence=True,
                       max_iter=100).fit(X)
    np.testing.assert_array_equal(est.predict(X), est.labels_)
    assert est.score() == -est.inertia_
    assert est.cluster_centers_.shape == (3, 3)


def test_repair_path_device():
    """Many duplicate points: clusters empty out and the device repair runs."""
    import paper_2501_05587_b200 as pcb
    g = make_rng(101)
    P = np.vstack([np.zeros((400, 3)), g.normal(0.0, 5.0, size=(40, 3))])
    g.shuffle(P)
    ref = oracle.run_lloyd(P, 30, max_iters=6, seed=2, dtype=np.float64)
    res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=30, max_iters=6, seed=2, dtype=np.float64))
    assert ref.repairs.sum() > 0
    np.testing.assert_array_equal(res.repairs, ref.repairs)
    np.testing.assert_array_equal(np.stack(res.label_history), np.stack(ref.label_history))


def test_device_side_finiteness_check():
    """Large inputs are validated on the device after the copy: same ValueError."""
    import paper_2501_05587_b200 as pcb
    P = np.zeros((1 << 19, 33), dtype=np.float32)  # > 16M values
    P[12345, 7] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        pcb.run_lloyd(P, pcb.KKMeansConfig(k=3, max_iters=1))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_repair_many_empty_clusters(dtype):
    """Hundreds of clusters empty at once (duplicate centroids): the batched
    top-E donor selection must pick the reference's donors, in order
    (repair_empty_clusters applied to the device's own raw labels with exact
    distances)."""
    rng = make_rng(31)
    n, d, k = 40000, 8, 300
    P = rng.normal(0, 1, size=(n, d)).astype(dtype)
    C = np.repeat(rng.normal(0, 1, size=(1, d)), k, axis=0).astype(dtype)
    C[:10] = rng.normal(0, 1, size=(10, d)).astype(dtype)  # 10 live centroids, 290 duplicates
    lab = np.zeros(n, dtype=np.int32)
    eng = _engine(P, k, dtype, "tiled" if dtype == np.float64 else "auto")
    gpu = eng.step_from(C, lab)
    raw = gpu["raw_labels"]
    assert np.bincount(raw, minlength=k).min() == 0
    P64, C64 = P.astype(np.float64), C.astype(np.float64)
    D = ((P64[:, None, :] - C64[None, :, :]) ** 2).sum(-1)
    ref = oracle.repair_empty_clusters(raw, D, k)
    assert int((ref != raw).sum()) >= 280
    assert gpu["moved"] == int((ref != raw).sum())
    np.testing.assert_array_equal(gpu["labels"], ref)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("d", [1536, 2048])
def test_wide_rows_lockstep(d, dtype):
    """d > 1024: the segmented sums run in 1024-column slabs (update.cu);
    run_lloyd and the lockstep step must work for any d, like the reference."""
    import paper_2501_05587_b200 as pcb
    n, k = 3000, 16
    P = oracle.make_blobs(n, d, k, seed=4).astype(dtype)
    lab = oracle.init_assignments(n, k, 0)
    C = oracle.mean_centroids(P, lab, k)
    eng = _engine(P, k, dtype)
    pn = oracle.point_norms(P)
    for t in range(3):
        ref = oracle.lloyd_step(P, pn, C, lab, k)
        gpu = eng.step_from(C, lab)
        check_step(P, C, lab, k, gpu, ref=ref, dtype=dtype, what=f"d={d} it{t}")
        C, lab = ref.centroids, ref.labels
    res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=k, max_iters=5, dtype=dtype))
    refr = oracle.run_lloyd(P, k, max_iters=5, dtype=dtype)
    assert res.iterations_run == 5
    np.testing.assert_allclose(res.objective_history, refr.objective_history, rtol=1e-6)
