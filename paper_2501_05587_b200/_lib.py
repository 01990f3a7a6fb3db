"""ctypes binding of the C-ABI library ``lib/libpopcorn_b200.so``.

The library is the product: there is no CPU fallback.  If it is missing or
cannot be loaded, every entry point raises ``RuntimeError`` at call time (the
import itself succeeds so that CPU-only tooling can introspect the package).
Signatures mirror ``include/popcorn_b200.h``.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCB_LIB_PATH", os.path.join(_HERE, "lib", "libpopcorn_b200.so"))

P = ctypes.c_void_p
I32 = ctypes.c_int
I64 = ctypes.c_int64
F64 = ctypes.c_double

# name -> (restype, argtypes); kept in sync with include/popcorn_b200.h
SIGNATURES = {
    "pcb_abi_version": (I32, []),
    "pcb_launch_count": (ctypes.c_longlong, []),
    "pcb_error_string": (ctypes.c_char_p, [I32]),
    "pcb_device_info": (I32, [I32, P, P, P]),
    "pcb_count_nonfinite_f32": (I32, [P, I64, P, P]),
    "pcb_count_nonfinite_f64": (I32, [P, I64, P, P]),
    "pcb_init_scratch_bytes": (I64, [I64, I32]),
    "pcb_pcg64_seed_state": (I32, [ctypes.c_uint64, P]),
    "pcb_init_assignments": (I32, [I64, I32, ctypes.c_uint64, P, P, I64, P, P]),
    "pcb_bounded_draws": (I32, [I64, I32, ctypes.c_uint64, P, P, I64, P]),
    "pcb_synthesize_uniform": (I32, [I64, ctypes.c_uint64, I32, P, P]),
    "pcb_load_libsvm": (I32, [ctypes.c_char_p, I64, I32, I32, P, P, P, I64, I32]),
    "pcb_load_csv": (I32, [ctypes.c_char_p, I64, I32, I32, P, P, P, I64, I32]),
    "pcb_point_norms_f32": (I32, [P, I64, I32, P, P]),
    "pcb_point_norms_f64": (I32, [P, I64, I32, P, P]),
    "pcb_split_tf32": (I32, [P, I64, I32, I32, P, P, P]),
    "pcb_assign_f32": (I32, [P, P, I64, I32, P, P, I32, P, P, P, P, P, I32, P]),
    "pcb_assign_f64": (I32, [P, P, I64, I32, P, P, I32, P, P, P, P, P, I32, P]),
    "pcb_assign_spec_f32": (I32, [P, P, I64, I32, P, P, I32, P, P, P, P, P, P, I32, P]),
    "pcb_assign_tc_f32": (I32, [P, P, I32, P, I64, I32, P, P, P, I32, P, P, P, P, P, P]),
    "pcb_screen_prep_points": (I32, [P, I64, I32, I32, P, P, P, P, P]),
    "pcb_screen_prep_centroids": (I32, [P, I32, I32, P, P, P, P]),
    "pcb_assign_screen_f32": (I32, [P, I64, I32, P, I32, P, P, P, P, P, P, P, P, P]),
    "pcb_resolve_ambiguous_f32": (I32, [P, I64, I32, P, P, I32, P, P, P, P, P, P, P, P, I32, P, P, P, P, I64, P,
                                        P]),
    "pcb_exact_scratch_bytes": (I64, []),
    "pcb_update_mode": (I32, [P, I32, I32, I64, F64, I32, P, P]),
    "pcb_delta_update_f32": (I32, [P, I64, I32, P, P, P, I32, P, P, P, P, P]),
    "pcb_delta_update_f64": (I32, [P, I64, I32, P, P, P, I32, P, P, P, P, P]),
    "pcb_sum_squares_f32": (I32, [P, I64, P, P]),
    "pcb_sum_squares_f64": (I32, [P, I64, P, P]),
    "pcb_screen_fp8_ld": (I32, [I32]),
    "pcb_screen_prep_points_fp8": (I32, [P, I64, I32, I32, P, P, P, P, P]),
    "pcb_screen_prep_centroids_fp8": (I32, [P, P, I32, I32, I32, P, P, P, P, P, P]),
    "pcb_assign_screen_fp8": (I32, [P, I64, I32, P, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "pcb_resolve_screen_fp8": (I32, [P, I64, I32, P, I32, P, P, I32, P, P, P, P, P, I64, P, P, P, P, P, P, P, P, P,
                                     P, P]),
    "pcb_screen_bf16_ld": (I32, [I32]),
    "pcb_screen_bf16_ncand": (I32, []),
    "pcb_screen_prep_points_bf16": (I32, [P, I64, I32, I32, P, P, P, P, P]),
    "pcb_screen_prep_centroids_bf16": (I32, [P, P, I32, I32, I32, P, P, P, P, P, P]),
    "pcb_screen_bf16_kpad": (I32, [I32]),
    "pcb_screen_bf16_aug": (I32, []),
    "pcb_assign_screen_bf16": (I32, [P, I64, I32, P, I32, P, P, P, P, P, P, P, P, P, P, P, P, P, P]),
    "pcb_resolve_screen_bf16": (I32, [P, I64, I32, P, I32, P, P, I32, P, P, P, P, P, I64, P, P, P, P, P, P, P, P, P,
                                      P, P]),
    "pcb_screen_relayout_bf16": (I32, [P, P, P, I64, I32, P, P, P, P, P, P]),
    "pcb_count_labels": (I32, [P, P, I64, I32, I32, P, P, P]),
    "pcb_count_labels_delta_f32": (I32, [P, P, I64, I32, I32, P, P, P, P, P]),
    "pcb_sort_by_label": (I32, [P, I64, I32, P, P, P, P, P, P]),
    "pcb_segment_sums_f32": (I32, [P, I64, I32, P, P, I32, P, P, P, P, P]),
    "pcb_segment_sums_f64": (I32, [P, I64, I32, P, P, I32, P, P, P, P, P]),
    "pcb_repair_scratch_bytes": (I64, [I32]),
    "pcb_repair_f32": (I32, [P, I64, I32, P, I32, P, P, P, P, P, P, P, I64, P, P]),
    "pcb_repair_f64": (I32, [P, I64, I32, P, I32, P, P, P, P, P, P, P, I64, P, P]),
    "pcb_repair_select": (I32, [P, P, I64, I64, I32, P, P, I64, P]),
    "pcb_repair_apply_batch_f32": (I32, [P, I32, P, P, P, P, P, P, P, P, I32, P, P]),
    "pcb_repair_apply_batch_f64": (I32, [P, I32, P, P, P, P, P, P, P, P, I32, P, P]),
    "pcb_repair_commit_batch": (I32, [P, I32, I32, I32, P, P, P, P]),
    "pcb_flag_global_empty": (I32, [P, I32, I32, P, P, P]),
    "pcb_finalize_f32": (I32, [P, I32, I32, I64, P, P, P, P, I32, P, P, P, I32, F64, P]),
    "pcb_finalize_f64": (I32, [P, I32, I32, I64, P, P, P, P, P, I32, F64, P]),
    "pcb_centroids_from_acc_f32": (I32, [P, I32, I32, P, P, P, P, I32, P]),
    "pcb_centroids_from_acc_f64": (I32, [P, I32, I32, P, P, P]),
    "pcb_centroid_norms_f32": (I32, [P, I32, I32, P, P, P, I32, P]),
    "pcb_centroid_norms_f64": (I32, [P, I32, I32, P, P]),
    "pcb_kernel_gram_f32": (I32, [P, P, I32, I64, P, P, I64, I32, F64, F64, I32, F64, P, P]),
    "pcb_kernel_gram_f64": (I32, [P, I64, I32, P, P, I64, I32, F64, F64, I32, F64, P, P]),
    "pcb_kk_segment_sums_f32": (I32, [P, I64, I64, I64, P, P, I32, P, I64, P, P]),
    "pcb_kk_segment_sums_f64": (I32, [P, I64, I64, I64, P, P, I32, P, I64, P, P]),
    "pcb_kernel_cross_f32": (I32, [P, P, I64, P, P, I64, I32, P, P, P, I64, I32, F64, F64, I32, F64, P, P]),
    "pcb_kernel_cross_f64": (I32, [P, I64, P, I64, I32, P, P, P, I64, I32, F64, F64, I32, F64, P, P]),
    "pcb_kk_predict_f32": (I32, [P, I64, I64, I32, P, P, P, I32, F64, F64, I32, F64, P, P]),
    "pcb_kk_predict_f64": (I32, [P, I64, I64, I32, P, P, P, I32, F64, F64, I32, F64, P, P]),
    "pcb_kk_assign_f32": (I32, [P, I64, P, I64, I64, I32, P, P, P, P, P, P, P, P]),
    "pcb_kk_assign_f64": (I32, [P, I64, P, I64, I64, I32, P, P, P, P, P, P, P, P]),
    "pcb_kk_repair_scratch_bytes": (I64, [I64, I32]),
    "pcb_kk_repair_f32": (I32, [P, I64, P, I64, I64, I32, P, P, P, P, P, P, P, I64, P]),
    "pcb_kk_repair_f64": (I32, [P, I64, P, I64, I64, I32, P, P, P, P, P, P, P, I64, P]),
    "pcb_kk_finalize": (I32, [P, P, P, I64, I32, P, P, P, P, P, I32, F64, P]),
    "pcb_mma_probe": (I32, [P, P, P, I32, P, P, P]),
    "pcb_mma_probe_f16acc": (I32, [P, P, P, I32, P, P, P, P]),
    "pcb_delta_tc_ld": (I32, [I32]),
    "pcb_delta_tc_kpad": (I32, [I32]),
    "pcb_delta_tc_prep_points": (I32, [P, I64, I32, I32, P, P, P]),
    "pcb_delta_tc_prep_centroids": (I32, [P, P, I32, I32, I32, P, P, P, P, P]),
    "pcb_assign_delta_tc_f32": (I32, [P, P, I32, I64, I32, P, P, P, P, I32, P, P, P, P, P, P]),
}

ASSIGN_AUTO, ASSIGN_ROWREG, ASSIGN_TILED, ASSIGN_TC3XTF32, ASSIGN_DELTA, ASSIGN_SCREEN = 0, 1, 2, 3, 4, 5
ASSIGN_SCREEN_BF16 = 6
ASSIGN_SCREEN_FP8 = 7
ASSIGN_DELTA_TC = 8
VARIANTS = {"auto": ASSIGN_AUTO, "rowreg": ASSIGN_ROWREG, "tiled": ASSIGN_TILED,
            "tc3xtf32": ASSIGN_TC3XTF32, "delta": ASSIGN_DELTA, "tc1xtf32s": ASSIGN_SCREEN,
            "bf16s": ASSIGN_SCREEN_BF16, "fp8s": ASSIGN_SCREEN_FP8,
            "deltatc": ASSIGN_DELTA_TC}
STATE_WORDS = 9

_lib = None
_load_error = None


def load():
    """Load (once) and return the library; raise RuntimeError if unavailable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise RuntimeError(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = (f"popcorn_b200 CUDA library not built: {LIB_PATH} is missing "
                       "(run `make` or __graft_entry__.build()); there is no CPU fallback")
        raise RuntimeError(_load_error)
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        _load_error = f"cannot load {LIB_PATH}: {e}"
        raise RuntimeError(_load_error) from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pcb_abi_version() != 1:
        raise RuntimeError("popcorn_b200 ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().pcb_error_string(rc).decode()
        raise RuntimeError(f"{what} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
