"""Tensor-core accumulation probe: the screens' error model, measured.

The certified E4M3 / BF16 screens (assign_screen_bf16.cu:435-437,
screen_common.cuh:39-45) are exact only if every tcgen05.mma adds at most
``acc_rel`` of the sum of |terms| it combines.  These tests run adversarial
K groups through ``pcb_mma_probe`` (one dominant product plus many tiny ones,
cancelling pairs, a dominant or cancelled accumulator, exponents over the
whole E4M3 range, long chains, the screen's own operand pattern) and compare
with exactly rounded sums (tests/mma_probe_cases.py).
"""
import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs a B200")]

import mma_probe_cases as M  # noqa: E402


@pytest.mark.parametrize("case", M.all_cases(), ids=lambda c: c[0])
def test_accumulation_within_certificate_budget(case):
    name, steps, init, m = case
    r = M.measure(name, steps, init, m)
    assert r["worst_units"] <= r["budget_units"], r


def test_probe_reproduces_exact_small_sums():
    # integers: every product and partial sum is exact in f32 -> D must be exact
    rng = np.random.Generator(np.random.PCG64(5))
    ints = np.array([M.e4m3_code(float(v)) for v in range(-8, 9)], np.uint8)
    steps = [M.e4m3_step(rng.choice(ints, 4096), rng.choice(ints, 4096)) for _ in range(3)]
    D = M.run_device(steps)
    ex, _ = M.exact(steps)
    assert np.array_equal(D, ex)


def test_probe_bf16_and_tf32_exact_on_integers():
    rng = np.random.Generator(np.random.PCG64(6))
    a = rng.integers(-64, 65, (128, 16)).astype(np.float32)
    b = rng.integers(-64, 65, (128, 16)).astype(np.float32)
    steps = [M.bf16_step(a, b), M.tf32_step(a[:, :8], b[:, :8])]
    D = M.run_device(steps)
    ex, _ = M.exact(steps)
    assert np.array_equal(D, ex)
