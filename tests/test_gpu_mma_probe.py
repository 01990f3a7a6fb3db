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


def test_f16acc_layout_and_exact_integers():
    """E4M3 into an F16 accumulator: small integer sums are exact; the packed
    readout puts column 2i in the low half of register i; the unpacked cell of
    column j holds D[:, j] as an f16 in its low 16 bits (recorded, not assumed)."""
    rng = np.random.Generator(np.random.PCG64(7))
    ints = np.array([M.e4m3_code(float(v)) for v in range(-4, 5)], np.uint8)
    steps = [M.e4m3_step(rng.choice(ints, 4096), rng.choice(ints, 4096)) for _ in range(2)]
    D, raw = M.run_device_f16acc(steps)
    ex, _ = M.exact(steps)
    assert np.array_equal(D, ex)
    lo = (raw & 0xFFFF).astype(np.uint16).view(np.float16).astype(np.float64)
    print("raw low-half == D:", bool(np.array_equal(lo, ex)), "high halves zero:", bool(((raw >> 16) == 0).all()))


@pytest.mark.parametrize("case", M.f16acc_cases(), ids=lambda c: c[0])
def test_f16acc_error_model(case):
    name, steps, init = case
    r = M.measure_f16acc(name, steps, init)
    print(r)
    assert r["nonfinite"] == 0, r
    # budget of the F16-key screen: 2 units of 2^-11 (one RN rounding of the
    # result plus alignment) per MMA of (sum |terms| + |result|)
    assert r["worst_units"] <= 2.0 * r["n_mma"], r
