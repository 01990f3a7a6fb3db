"""The C-ABI library loads and exports every symbol include/popcorn_b200.h declares.

CPU-only: nothing here launches a kernel.
"""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "popcorn_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pcb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("pcb_assign_f32", "pcb_assign_f64", "pcb_segment_sums_f32", "pcb_repair_f32",
                 "pcb_finalize_f32", "pcb_sort_by_label", "pcb_point_norms_f32"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2501_05587_b200 import _lib
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, f"declared but not exported: {missing}"


def test_ctypes_signatures_cover_header():
    from paper_2501_05587_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_abi_version_and_errors():
    from paper_2501_05587_b200 import _lib
    lib = _lib.load()
    assert lib.pcb_abi_version() == 1
    assert b"invalid argument" in lib.pcb_error_string(-1)
    assert b"unsupported" in lib.pcb_error_string(-2)
    assert lib.pcb_repair_scratch_bytes(1024) > 1024 * 4


def test_argument_errors_without_gpu():
    """Bad sizes are rejected before any CUDA call (no device needed)."""
    from paper_2501_05587_b200 import _lib
    lib = _lib.load()
    assert lib.pcb_assign_f32(None, None, 0, 2, None, None, 3, None, None, None, None, None, 0, None) == -1
    assert lib.pcb_segment_sums_f32(None, 10, 2, None, None, 3, None, None, None, None, None) == -1
    assert lib.pcb_split_tf32(None, 4, 8, 4, None, None, None) == -1


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2501_05587_b200", "lib", "libpopcorn_b200.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_pcg64_seed_state_matches_numpy():
    """pcb_pcg64_seed_state restates numpy's SeedSequence -> PCG64 seeding
    (the first step of init_assignments, clustering.py:101) on the host."""
    import numpy as np
    from paper_2501_05587_b200 import _lib
    lib = _lib.load()
    seeds = [0, 1, 42, 2**32 - 1, 2**32, 2**64 - 1] + [int(s) for s in np.random.default_rng(1).integers(0, 2**63, 50)]
    for seed in seeds:
        out = (ctypes.c_uint64 * 4)()
        assert lib.pcb_pcg64_seed_state(seed, out) == 0
        st = np.random.PCG64(seed).state["state"]
        assert (out[0] << 64 | out[1], out[2] << 64 | out[3]) == (st["state"], st["inc"]), seed
    assert lib.pcb_init_scratch_bytes(0, 3) == -1
    assert lib.pcb_init_assignments(5, 6, 0, None, None, 0, None, None) == -1
