"""Host-side contract of the drop-in API (no GPU needed).

Mirrors the reference tests that pin the Lloyd driver's host logic:
test_clustering.py (init golden, config validation) and test_estimator.py
(sklearn contract, error types).
"""
import numpy as np
import pytest

import paper_2501_05587_b200 as pcb
from conftest import has_cuda

GOLDEN_INIT_100_10_42 = [
    0, 7, 6, 4, 4, 8, 0, 6, 2, 0, 5, 9, 7, 7, 7, 7, 5, 1, 8, 4, 5, 3, 1, 9, 7,
    6, 4, 8, 5, 4, 4, 2, 0, 5, 8, 0, 8, 8, 2, 6, 1, 7, 7, 3, 0, 9, 4, 8, 6, 7,
    7, 1, 3, 4, 4, 0, 5, 1, 7, 6, 9, 7, 3, 9, 4, 3, 9, 3, 0, 4, 7, 1, 4, 1, 6,
    4, 3, 2, 5, 6, 9, 4, 1, 8, 6, 7, 0, 3, 7, 8, 4, 8, 8, 3, 8, 2, 2, 6, 6, 1,
]


def test_init_golden():
    np.testing.assert_array_equal(pcb.init_assignments(100, 10, 42), GOLDEN_INIT_100_10_42)


def test_init_matches_golden_cases(golden):
    for i, (n, k, s) in enumerate(golden["init_cases"]):
        np.testing.assert_array_equal(pcb.init_assignments(int(n), int(k), int(s)), golden[f"init_{i}"])


def test_init_rejects_k_gt_n():
    with pytest.raises(ValueError):
        pcb.init_assignments(3, 4, 0)


@pytest.mark.parametrize("cfg", [dict(k=5), dict(k=0), dict(k=2, tol=1.5), dict(k=2, max_iters=0)])
def test_config_validation_raises_value_error(cfg):
    P = np.zeros((4, 2)) + 0.5
    with pytest.raises(ValueError):
        pcb.run_lloyd(P, pcb.KKMeansConfig(**cfg))


def test_non_finite_points_rejected():
    with pytest.raises(ValueError):
        pcb.run_lloyd(np.array([[np.nan, 0.0], [1.0, 2.0]]), pcb.KKMeansConfig(k=1))


def test_dtype_aliases():
    assert pcb.normalize_dtype("f64") == np.float64
    assert pcb.normalize_dtype("single") == np.float32
    with pytest.raises(ValueError):
        pcb.normalize_dtype("f16")


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    P = np.random.Generator(np.random.PCG64(0)).random((50, 3))
    with pytest.raises(RuntimeError, match="no CPU fallback|CUDA"):
        pcb.run_lloyd(P, pcb.KKMeansConfig(k=3))


class TestEstimatorContract:
    def test_get_set_params_round_trip(self):
        est = pcb.KernelKMeans(n_clusters=4, max_iter=7)
        params = est.get_params()
        clone = pcb.KernelKMeans(**params)
        assert clone.get_params() == params
        clone.set_params(n_clusters=7)
        assert clone.n_clusters == 7

    def test_set_params_rejects_unknown(self):
        with pytest.raises(ValueError):
            pcb.KernelKMeans().set_params(bogus=1)

    def test_sklearn_clone_compatible(self):
        sklearn_base = pytest.importorskip("sklearn.base")
        est = pcb.KernelKMeans(n_clusters=3, max_iter=12)
        assert sklearn_base.clone(est).get_params() == est.get_params()

    def test_repr_mentions_params(self):
        assert "n_clusters=5" in repr(pcb.KernelKMeans(n_clusters=5))

    def test_unknown_algorithm_rejected(self):
        with pytest.raises(ValueError):
            pcb.KernelKMeans(algorithm="spectral").fit(np.zeros((6, 2)))

    def test_unfitted_predict_raises(self):
        with pytest.raises(RuntimeError):
            pcb.KernelKMeans().predict(np.zeros((3, 2)))

    def test_registry_has_lloyd_driver(self):
        assert pcb._ALGORITHMS["lloyd"] is pcb.run_lloyd
