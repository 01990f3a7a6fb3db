"""Pin the CPU oracle against golden vectors produced by the reference itself."""
import numpy as np
import pytest

import oracle
from conftest import golden_runs, make_rng


def test_init_golden(golden):
    for i, (n, k, s) in enumerate(golden["init_cases"]):
        np.testing.assert_array_equal(oracle.init_assignments(int(n), int(k), int(s)),
                                      golden[f"init_{i}"])


def test_init_reference_fixture():
    # GOLDEN_INIT_100_10_42 of the reference's test_clustering.py:13-18 (first row)
    first = [0, 7, 6, 4, 4, 8, 0, 6, 2, 0, 5, 9, 7, 7, 7, 7, 5, 1, 8, 4, 5, 3, 1, 9, 7]
    assert oracle.init_assignments(100, 10, 42)[:25].tolist() == first


def test_repair_golden(golden):
    for i in range(int(golden["repair_count"])):
        out = oracle.repair_empty_clusters(golden[f"repair_{i}_labels"], golden[f"repair_{i}_D"],
                                           int(golden[f"repair_{i}_k"]))
        np.testing.assert_array_equal(out, golden[f"repair_{i}_out"])


def test_augmented_worked_values(golden):
    got = [oracle.augmented_distance([3.0], [7.0]), oracle.augmented_distance([1.0], [7.0]),
           oracle.augmented_distance([5.0, 2.0], [1.0, 4.0]),
           oracle.augmented_distance([4.0, 3.0, 2.0], [5.0, 2.0, 3.0])]
    assert got == [16.0, 36.0, 20.0, 3.0]
    np.testing.assert_array_equal(got, golden["aug_cases"])


@pytest.mark.parametrize("idx", range(63))
def test_run_lloyd_bit_identical_to_reference(golden, idx):
    names = golden_runs(golden)
    if idx >= len(names):
        pytest.skip("fewer runs")
    name = names[idx]
    k, seed, cc, mi, dtc = (int(x) for x in golden[f"run_{name}_meta"])
    dtype = np.float32 if dtc == 1 else np.float64
    res = oracle.run_lloyd(golden[f"run_{name}_P"], k, max_iters=mi,
                           tol=float(golden[f"run_{name}_tol"]), check_convergence=bool(cc),
                           seed=seed, dtype=dtype, record_centroids=True)
    np.testing.assert_array_equal(np.stack(res.label_history), golden[f"run_{name}_labels"])
    np.testing.assert_array_equal(res.objective_history, golden[f"run_{name}_objective"])
    np.testing.assert_array_equal(res.repairs, golden[f"run_{name}_repairs"])
    assert res.converged == bool(golden[f"run_{name}_converged"])
    np.testing.assert_array_equal(np.stack(res.centroid_history), golden[f"run_{name}_centroids"])


def test_lockstep_step_matches_driver(golden):
    name = "blob_c3"
    P = golden[f"run_{name}_P"]
    k = int(golden[f"run_{name}_meta"][0])
    labs = golden[f"run_{name}_labels"]
    cents = golden[f"run_{name}_centroids"]
    pn = oracle.point_norms(P)
    for t in range(1, labs.shape[0]):
        st = oracle.lloyd_step(P, pn, cents[t - 1], labs[t - 1], k)
        np.testing.assert_array_equal(st.labels, labs[t])
        np.testing.assert_array_equal(st.centroids, cents[t])


def test_top2_gap_and_f64_means():
    P = make_rng(3).random((200, 4)).astype(np.float32)
    C = P[:5].copy()
    d1, gap = oracle.top2_gap_f64(P, C)
    assert np.all(gap >= 0)
    assert np.allclose(d1[:5], 0.0, atol=1e-12)
    lab = oracle.row_argmin(oracle.distance_matrix(P.astype(np.float64),
                                                   oracle.point_norms(P.astype(np.float64)),
                                                   C.astype(np.float64)))
    m = oracle.mean_centroids_f64(P, lab, 5)
    m32 = oracle.mean_centroids(P, lab, 5)
    assert np.max(np.abs(m - m32)) < 1e-5


def test_validation_errors():
    with pytest.raises(ValueError):
        oracle.run_lloyd(np.zeros((4, 2)), 5)
    with pytest.raises(ValueError):
        oracle.run_lloyd(np.array([[np.nan, 0.0]]), 1)
    with pytest.raises(ValueError):
        oracle.row_argmin(np.array([[1.0, np.nan]]))
    with pytest.raises(ValueError):
        oracle.normalize_dtype("f16")
