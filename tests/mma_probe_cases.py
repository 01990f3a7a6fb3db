"""Adversarial operand sets for the tensor-core accumulation probe
(``pcb_mma_probe``, csrc/mma_probe.cu) and their exactly rounded results.

The certified screens (assign_screen_bf16.cu) charge the f32 accumulation
inside tcgen05.mma as ``acc_rel`` of the sum of |terms| (products, augmented
columns and the running accumulator): ``(#MMA + 3) * 2^-18`` for E4M3 chains
(``kind::f8f6f4``, K = 32) and ``(#MMA + 3) * 2^-19`` for BF16 chains
(``kind::f16``, K = 16) — i.e. 32 / 16 units of 2^-23 per MMA.  Each case here
measures ``|D - exact| / (sum |terms| + |init|)`` in units of 2^-23; the
budget is met when the worst case of a chain of m MMAs stays below
``(m + 3) * unit``.

Used by tests/test_gpu_mma_probe.py and scripts/mma_accum_probe.py (which
records the table under profiles/).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

E4M3, BF16, TF32 = 0, 1, 2
K_OF = {E4M3: 32, BF16: 16, TF32: 8}
NAME = {E4M3: "e4m3", BF16: "bf16", TF32: "tf32"}
# per-MMA budget of the certificates, in units of 2^-23 of sum |terms|
BUDGET_UNITS = {E4M3: 32.0, BF16: 16.0, TF32: 16.0}


def _e4m3_table() -> np.ndarray:
    v = np.zeros(256)
    for c in range(256):
        s = -1.0 if c & 0x80 else 1.0
        e, m = (c >> 3) & 0xF, c & 7
        if e == 15 and m == 7:
            v[c] = np.nan
        elif e == 0:
            v[c] = s * m / 8.0 * 2.0 ** -6
        else:
            v[c] = s * (1.0 + m / 8.0) * 2.0 ** (e - 7)
    return v


E4M3_VAL = _e4m3_table()
E4M3_FINITE = np.array([c for c in range(256) if np.isfinite(E4M3_VAL[c])], dtype=np.uint8)


def e4m3_code(x: float) -> int:
    """Code of an exactly representable E4M3 value."""
    hits = np.nonzero(E4M3_VAL == x)[0]
    assert hits.size, f"{x} is not an E4M3 value"
    return int(hits[0])


class Step:
    """One MMA step: operand values (128 x K each) of one kind, as bytes."""

    def __init__(self, kind: int, a_bytes: np.ndarray, b_bytes: np.ndarray):
        assert a_bytes.shape == (128, 32) and b_bytes.shape == (128, 32)
        self.kind, self.a, self.b = kind, a_bytes, b_bytes

    def values(self):
        if self.kind == E4M3:
            return E4M3_VAL[self.a], E4M3_VAL[self.b]
        if self.kind == BF16:
            f = lambda u8: (u8.view(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
            return f(np.ascontiguousarray(self.a)), f(np.ascontiguousarray(self.b))
        f = lambda u8: (u8.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
        return f(np.ascontiguousarray(self.a)), f(np.ascontiguousarray(self.b))


def e4m3_step(a_codes, b_codes) -> Step:
    return Step(E4M3, np.asarray(a_codes, np.uint8).reshape(128, 32), np.asarray(b_codes, np.uint8).reshape(128, 32))


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """RN-even BF16 bit patterns of f32 values."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def bf16_step(a_vals, b_vals) -> Step:
    a = bf16_bits(np.asarray(a_vals, np.float32).reshape(128, 16)).view(np.uint8).reshape(128, 32)
    b = bf16_bits(np.asarray(b_vals, np.float32).reshape(128, 16)).view(np.uint8).reshape(128, 32)
    return Step(BF16, a, b)


def tf32_step(a_vals, b_vals) -> Step:
    m = np.uint32(0xFFFFE000)
    a = (np.asarray(a_vals, np.float32).reshape(128, 8).view(np.uint32) & m).view(np.uint8).reshape(128, 32)
    b = (np.asarray(b_vals, np.float32).reshape(128, 8).view(np.uint32) & m).view(np.uint8).reshape(128, 32)
    return Step(TF32, a, b)


def exact(steps, init=None):
    """Exactly rounded init + sum of every step's products, and sum |terms|.
    Products of E4M3/BF16/TF32 values are exact in f64; math.fsum rounds the
    sum of each (row, column) once."""
    terms = []
    for s in steps:
        a, b = s.values()
        k = K_OF[s.kind]
        a, b = a[:, :k], b[:, :k]
        terms.append(a[:, None, :] * b[None, :, :])  # (128, 128, K)
    T = np.concatenate(terms, axis=2)
    if init is not None:
        T = np.concatenate([T, np.asarray(init, np.float64)[:, :, None]], axis=2)
    flat = T.reshape(128 * 128, -1)
    ex = np.array([math.fsum(r) for r in flat]).reshape(128, 128)
    mag = np.abs(T).sum(axis=2)
    return ex, mag


def run_device(steps, init=None) -> np.ndarray:
    """D = init + sum of the steps on the tensor core (pcb_mma_probe)."""
    import torch

    from paper_2501_05587_b200 import _lib as L

    n = len(steps)
    A = np.concatenate([s.a for s in steps], axis=1)
    B = np.concatenate([s.b for s in steps], axis=1)
    kinds = np.array([s.kind for s in steps], np.int32)
    dev = torch.device("cuda", 0)
    tA = torch.from_numpy(np.ascontiguousarray(A)).to(dev)
    tB = torch.from_numpy(np.ascontiguousarray(B)).to(dev)
    tk = torch.from_numpy(kinds).to(dev)
    ti = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.float32)).to(dev)
    tD = torch.empty((128, 128), dtype=torch.float32, device=dev)
    p = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
    L.call("pcb_mma_probe", p(tA), p(tB), p(tk), n, p(ti), p(tD),
           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return tD.cpu().numpy().astype(np.float64)


def measure(name, steps, init=None, n_mma=None):
    """Worst |D - exact| / (sum |terms|) of the case, in units of 2^-23."""
    D = run_device(steps, init)
    ex, mag = exact(steps, init)
    err = np.abs(D - ex)
    units = err / np.maximum(mag, 1e-300) / 2.0 ** -23
    signed = (D - ex) / np.maximum(mag, 1e-300) / 2.0 ** -23
    main = [s.kind for s in steps if s.kind != BF16] or [BF16]
    kind = main[0]
    m = n_mma if n_mma is not None else len(steps)
    return {
        "case": name, "kind": NAME[kind], "n_mma": m, "worst_units": float(units.max()),
        "mean_signed_units": float(signed.mean()), "frac_exact": float((err == 0).mean()),
        "budget_units": float((m + 3) * BUDGET_UNITS[kind]),
        "worst_over_budget": float(units.max() / ((m + 3) * BUDGET_UNITS[kind])),
        "per_mma_worst_units": float(units.max() / m),
    }


# ---- the cases ------------------------------------------------------------------

def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def e4m3_cases(seed=0):
    rng = _rng(seed)
    out = []
    # (a) random finite codes, one MMA
    out.append(("e4m3 random codes", [e4m3_step(rng.choice(E4M3_FINITE, 4096), rng.choice(E4M3_FINITE, 4096))], None, 1))
    # (b) one dominant product + 31 tiny ones; the ratio sweeps 2^-4 .. 2^-30 over the rows
    a = np.zeros((128, 32), np.uint8)
    b = np.zeros((128, 32), np.uint8)
    big = e4m3_code(448.0)
    for i in range(128):
        a[i, 0] = big
        e = -(i % 10) - 1          # tiny exponents 2^-1 .. 2^-10 (normal) and subnormals below
        tiny = [c for c in E4M3_FINITE if 0 < E4M3_VAL[c] <= 2.0 ** e] or [1]
        a[i, 1:] = rng.choice(np.array(tiny, np.uint8), 31)
    for j in range(128):
        b[j, 0] = e4m3_code(float(rng.choice([256.0, 448.0, 1.0, 2.0 ** -3])))
        b[j, 1:] = rng.choice(np.array([c for c in E4M3_FINITE if 0 < E4M3_VAL[c] < 8], np.uint8), 31)
    out.append(("e4m3 dominant + 31 tiny", [e4m3_step(a, b)], None, 1))
    # (c) cancelling pairs with one small survivor
    a = rng.choice(E4M3_FINITE, (128, 32)).astype(np.uint8)
    b = rng.choice(E4M3_FINITE, (128, 32)).astype(np.uint8)
    a[:, 1::2] = a[:, 0::2]
    b[:, 1::2] = b[:, 0::2] ^ 0x80  # -b: products cancel pairwise
    a[:, 31] = rng.choice(E4M3_FINITE, 128)
    out.append(("e4m3 cancelling pairs", [e4m3_step(a, b)], None, 1))
    # (d) large accumulator + small products (the running sum dominates)
    init = (rng.choice([-1.0, 1.0], (128, 128)) * 2.0 ** rng.integers(8, 24, (128, 128))
            * (1 + rng.integers(0, 2 ** 23, (128, 128)) / 2.0 ** 23)).astype(np.float32)
    small = np.array([c for c in E4M3_FINITE if abs(E4M3_VAL[c]) < 4], np.uint8)
    out.append(("e4m3 large accumulator + small products", [e4m3_step(rng.choice(small, 4096), rng.choice(small, 4096))],
                init, 1))
    # (e) accumulator cancelled by the products (result << |init|)
    a = np.full((128, 32), e4m3_code(448.0), np.uint8)
    b = np.full((128, 32), e4m3_code(448.0), np.uint8)
    a[:, 16:] = rng.choice(small, (128, 16))
    tot = (E4M3_VAL[a][:, None, :] * E4M3_VAL[b][None, :, :]).sum(axis=2)
    init = (-tot[:, :] * (1 + rng.uniform(-2 ** -10, 2 ** -10, (128, 128)))).astype(np.float32)
    out.append(("e4m3 accumulator cancelled", [e4m3_step(a, b)], init, 1))
    # (f) chains of m random MMAs with a moderate accumulator (exponents spread)
    for m in (4, 8, 32):
        steps = [e4m3_step(rng.choice(E4M3_FINITE, 4096), rng.choice(E4M3_FINITE, 4096)) for _ in range(m)]
        init = rng.normal(0, 1e5, (128, 128)).astype(np.float32)
        out.append((f"e4m3 chain of {m} random", steps, init, m))
    return out


def bf16_cases(seed=1):
    rng = _rng(seed)
    out = []
    spread = lambda shape, lo, hi: (rng.choice([-1.0, 1.0], shape) * 2.0 ** rng.integers(lo, hi, shape)
                                    * (1 + rng.integers(0, 128, shape) / 128.0)).astype(np.float32)
    out.append(("bf16 random, exponents 2^-20..2^20", [bf16_step(spread((128, 16), -20, 20), spread((128, 16), -20, 20))],
                None, 1))
    a = spread((128, 16), -12, -2)
    b = spread((128, 16), -12, -2)
    a[:, 0] = 2.0 ** 10
    b[:, 0] = 2.0 ** 10
    out.append(("bf16 dominant + 15 tiny", [bf16_step(a, b)], None, 1))
    init = spread((128, 128), 10, 24)
    out.append(("bf16 large accumulator + small products", [bf16_step(spread((128, 16), -4, 2), spread((128, 16), -4, 2))],
                init, 1))
    for m in (4, 16):
        steps = [bf16_step(spread((128, 16), -8, 8), spread((128, 16), -8, 8)) for _ in range(m)]
        out.append((f"bf16 chain of {m}", steps, spread((128, 128), 0, 16), m))
    return out


def tf32_cases(seed=2):
    rng = _rng(seed)
    spread = lambda shape, lo, hi: (rng.choice([-1.0, 1.0], shape) * 2.0 ** rng.integers(lo, hi, shape)
                                    * (1 + rng.integers(0, 1024, shape) / 1024.0)).astype(np.float32)
    out = [("tf32 random, exponents 2^-20..2^20", [tf32_step(spread((128, 8), -20, 20), spread((128, 8), -20, 20))],
            None, 1)]
    a = spread((128, 8), -12, -2)
    b = spread((128, 8), -12, -2)
    a[:, 0] = 2.0 ** 10
    b[:, 0] = 2.0 ** 10
    out.append(("tf32 dominant + 7 tiny", [tf32_step(a, b)], None, 1))
    out.append(("tf32 large accumulator + small products",
                [tf32_step(spread((128, 8), -4, 2), spread((128, 8), -4, 2))], spread((128, 128), 10, 24), 1))
    return out


def screen_pattern_case(seed=3, d=128):
    """The E4M3 screen's own MMA chain: d/32 E4M3 steps over blob-like scaled
    operands, then the BF16 augmented step [1 1 1 0..] x [h1 h2 h3 0..]
    adding S (|c|^2 + OFF) (assign_screen_bf16.cu, centroid_aug_kernel)."""
    rng = _rng(seed)
    centers = rng.uniform(-10, 10, (8, d))
    P = (centers[rng.integers(0, 8, 128)] + rng.normal(0, 1, (128, d))).astype(np.float32)
    C = (centers[rng.integers(0, 8, 128)] + rng.normal(0, 0.05, (128, d))).astype(np.float32)
    sp = 2.0 ** math.floor(math.log2(448.0 / np.abs(P).max()))
    sc = 2.0 ** math.floor(math.log2(448.0 / (2 * np.abs(C).max())))
    enc = lambda x: np.array([int(np.abs(E4M3_VAL[E4M3_FINITE] - v).argmin()) for v in x.ravel()], np.uint8)
    codes = E4M3_FINITE
    qa = codes[enc(P * sp)].reshape(128, d)
    qb = codes[enc(-2.0 * C * sc)].reshape(128, d)
    steps = [e4m3_step(qa[:, 32 * s:32 * s + 32], qb[:, 32 * s:32 * s + 32]) for s in range(d // 32)]
    off = 1.01 * float((P.astype(np.float64) ** 2).sum(1).max()) + 1.0
    cn = (C.astype(np.float64) ** 2).sum(1)
    cp = ((cn + off) * sp * sc).astype(np.float32)
    h1 = np.float32(cp)
    h1b = (bf16_bits(h1).astype(np.uint32) << 16).view(np.float32)
    r1 = (h1 - h1b).astype(np.float32)
    h2b = (bf16_bits(r1).astype(np.uint32) << 16).view(np.float32)
    h3b = (bf16_bits((r1 - h2b).astype(np.float32)).astype(np.uint32) << 16).view(np.float32)
    a_aug = np.zeros((128, 16), np.float32)
    a_aug[:, :3] = 1.0
    b_aug = np.zeros((128, 16), np.float32)
    b_aug[:, 0], b_aug[:, 1], b_aug[:, 2] = h1b, h2b, h3b
    steps.append(bf16_step(a_aug, b_aug))
    return ("screen pattern: %d E4M3 steps + BF16 augmented step" % (d // 32), steps, None, d // 32)


def all_cases():
    return e4m3_cases() + bf16_cases() + tf32_cases() + [screen_pattern_case()]


def half_ulp_cases():
    """Tiny products just below the f32 ulp of one dominant product: a
    per-term truncation shows up as (K - 1) / 2 units, one final rounding as
    <= 0.5 unit."""
    out = []
    a = np.full((128, 32), e4m3_code(0.125), np.uint8)
    b = np.full((128, 32), e4m3_code(2.0 ** -5), np.uint8)   # 2^-8 = ulp(2^16) / 2
    b[64:, 1:] = e4m3_code(0.09375)                         # 0.75 * 2^-7 on half the rows
    a[:, 0] = e4m3_code(256.0)
    b[:, 0] = e4m3_code(256.0)                              # 2^16
    out.append(("e4m3 2^16 + 31 half-ulp products", [e4m3_step(a, b)], None, 1))
    a = np.full((128, 16), 2.0 ** -4, np.float32)
    b = np.full((128, 16), 2.0 ** -4, np.float32)
    a[:, 0] = b[:, 0] = 2.0 ** 8
    out.append(("bf16 2^16 + 15 half-ulp products", [bf16_step(a, b)], None, 1))
    init = np.full((128, 128), 2.0 ** 16, np.float32)
    a = np.full((128, 32), e4m3_code(0.125), np.uint8)
    b = np.full((128, 32), e4m3_code(2.0 ** -5), np.uint8)
    out.append(("e4m3 accumulator 2^16 + 32 half-ulp products", [e4m3_step(a, b)], init, 1))
    return out


_all_cases_base = all_cases


def all_cases():  # noqa: F811
    return _all_cases_base() + half_ulp_cases()


# ---- F16 accumulator (E4M3 into kind::f8f6f4 with D = F16) ------------------------

def run_device_f16acc(steps, init=None):
    """(D as f64, raw 32-bit TMEM cells) of an E4M3 chain into an F16 accumulator."""
    import torch

    from paper_2501_05587_b200 import _lib as L

    n = len(steps)
    A = np.concatenate([s.a for s in steps], axis=1)
    B = np.concatenate([s.b for s in steps], axis=1)
    dev = torch.device("cuda", 0)
    tA = torch.from_numpy(np.ascontiguousarray(A)).to(dev)
    tB = torch.from_numpy(np.ascontiguousarray(B)).to(dev)
    tk = torch.zeros(n, dtype=torch.int32, device=dev)
    ti = None if init is None else torch.from_numpy(np.ascontiguousarray(init, np.float32)).to(dev)
    tD = torch.empty((128, 128), dtype=torch.float32, device=dev)
    tR = torch.empty((128, 128), dtype=torch.int32, device=dev)
    p = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())
    L.call("pcb_mma_probe_f16acc", p(tA), p(tB), p(tk), n, p(ti), p(tD), p(tR),
           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return tD.cpu().numpy().astype(np.float64), tR.cpu().numpy().view(np.uint32)


def measure_f16acc(name, steps, init=None):
    """Worst |D - exact| in units of 2^-11 of (sum |terms| + |exact|) per MMA."""
    D, _ = run_device_f16acc(steps, init)
    init16 = None if init is None else np.asarray(init, np.float32).astype(np.float16).astype(np.float64)
    ex, mag = exact(steps, init16)
    err = np.abs(D - ex)
    finite = np.isfinite(D)
    scale = np.maximum(mag + np.abs(ex), 1e-300)
    units = np.where(finite, err / scale / 2.0 ** -11, np.inf)
    m = len(steps)
    return {"case": name, "kind": "e4m3->f16", "n_mma": m, "worst_units": float(units.max()),
            "per_mma_worst_units": float(units.max() / m), "frac_exact": float((err == 0).mean()),
            "nonfinite": int((~finite).sum())}


def f16acc_cases(seed=11):
    """E4M3 chains into an F16 accumulator, sized so no partial sum overflows f16."""
    rng = _rng(seed)
    small = np.array([c for c in E4M3_FINITE if abs(E4M3_VAL[c]) <= 4], np.uint8)
    mid = np.array([c for c in E4M3_FINITE if abs(E4M3_VAL[c]) <= 16], np.uint8)
    out = []
    out.append(("f16acc random |x| <= 4", [e4m3_step(rng.choice(small, 4096), rng.choice(small, 4096))], None))
    out.append(("f16acc random |x| <= 16", [e4m3_step(rng.choice(mid, 4096), rng.choice(mid, 4096))], None))
    out.append(("f16acc chain of 4 |x| <= 4", [e4m3_step(rng.choice(small, 4096), rng.choice(small, 4096))
                                               for _ in range(4)], None))
    # dominant product + tiny ones
    a = rng.choice(small, (128, 32)).astype(np.uint8)
    b = rng.choice(small, (128, 32)).astype(np.uint8)
    a[:, 0] = e4m3_code(16.0)
    b[:, 0] = e4m3_code(16.0)
    tiny = np.array([c for c in E4M3_FINITE if 0 < abs(E4M3_VAL[c]) <= 2.0 ** -4], np.uint8)
    a[:, 1:] = rng.choice(tiny, (128, 31))
    out.append(("f16acc dominant + 31 tiny", [e4m3_step(a, b)], None))
    # large accumulator (init) + small products
    init = (rng.choice([-1.0, 1.0], (128, 128)) * rng.uniform(1000, 30000, (128, 128))).astype(np.float32)
    out.append(("f16acc large accumulator + small products", [e4m3_step(rng.choice(small, 4096),
                                                                         rng.choice(small, 4096))], init))
    # the screen pattern: 4 E4M3 K steps of -2 p.c then the augmented step adding |c|^2 + OFF pieces
    out.append(("f16acc chain of 4 + init 2^14", [e4m3_step(rng.choice(small, 4096), rng.choice(small, 4096))
                                                  for _ in range(4)],
                np.full((128, 128), 16384.0, np.float32)))
    return out
