"""On-device init_assignments (f2): bit-identical to the reference's numpy stream.

The reference draws Generator(PCG64(seed)).integers(0, k, size=n) and fills
empty clusters (clustering.py:91-108); the device path (init.cu) must give the
same labels, including the rare Lemire rejections (forced here with k just above
a power of two, where ~25 % of the 32-bit draws are rejected).
"""
import numpy as np
import pytest

import oracle
from conftest import has_cuda

pytestmark = pytest.mark.gpu


def _dev_init(n, k, seed, fill=True):
    from paper_2501_05587_b200.engine import init_labels
    return init_labels(n, k, seed, hollow_fill=fill).cpu().numpy()


@pytest.mark.parametrize("k", [1, 2, 10, 1000, 1024, 4097, 65537, (1 << 30) + 1, (1 << 31) - 1])
@pytest.mark.parametrize("n", [1, 7, 1000, 100_003])
def test_bounded_draws_match_numpy(n, k):
    for seed in (0, 42):
        ref = np.random.Generator(np.random.PCG64(seed)).integers(0, k, size=n)
        np.testing.assert_array_equal(_dev_init(n, k, seed, fill=False), ref.astype(np.int32))


def test_init_golden_cases(golden):
    for i, (n, k, s) in enumerate(golden["init_cases"]):
        np.testing.assert_array_equal(_dev_init(int(n), int(k), int(s)), golden[f"init_{i}"])


@pytest.mark.parametrize("n,k,seed", [(100, 90, 0), (500, 400, 3), (50, 50, 1), (2000, 1999, 5),
                                      (1_000_000, 1024, 0), (3_000_001, 4095, 17)])
def test_init_matches_oracle(n, k, seed):
    np.testing.assert_array_equal(_dev_init(n, k, seed), oracle.init_assignments(n, k, seed))


def test_large_seed_and_errors():
    n, k = 10_000, 13
    for seed in (2**32 + 7, 2**63 + 5, 2**64 - 1):
        np.testing.assert_array_equal(_dev_init(n, k, seed), oracle.init_assignments(n, k, seed))
    with pytest.raises(ValueError):
        _dev_init(10, 11, 0)
    with pytest.raises(ValueError):
        _dev_init(10, 3, -1)


def test_sharded_engine_takes_its_slice():
    import torch
    from paper_2501_05587_b200.engine import LloydEngine
    n, d, k = 10_001, 8, 37
    P = torch.randn(4000, d, device="cuda")
    eng = LloydEngine(P, k, n_total=n)
    eng.init_labels_device(9, 3000)
    np.testing.assert_array_equal(eng.labels[0].cpu().numpy(), oracle.init_assignments(n, k, 9)[3000:7000])


@pytest.mark.parametrize("n,d,seed", [(1, 1, 0), (50, 3, 9), (1000, 17, 123), (100_000, 64, 2**40 + 3)])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_synthesize_points_matches_reference(n, d, seed, dt):
    """cli.synthesize_points (cli.py:102-105): Generator(PCG64(seed)).random((n, d)).astype(dtype)."""
    from paper_2501_05587_b200.io import synthesize_points
    got = synthesize_points(n, d, seed, dtype=dt)
    ref = np.random.Generator(np.random.PCG64(seed)).random((n, d)).astype(dt)
    assert got.dtype == ref.dtype
    np.testing.assert_array_equal(got, ref)
