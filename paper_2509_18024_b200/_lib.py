"""ctypes binding of libcoreals_b200.so (the C ABI in include/coreals_b200.h).

There is no CPU fallback: importing the product path on a machine without the
built library or without a CUDA device raises loudly.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcoreals_b200.so")

CALS_OK = 0
CALS_ROW_OK, CALS_ROW_JITTERED, CALS_ROW_SINGULAR = 0, 1, 2
CALS_MAX_NF = 128

P = ctypes.c_void_p
i64, i32, f64, sz = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t


class cals_side(ctypes.Structure):
    _fields_ = [("ptr", P), ("idx", P), ("val", P), ("n_rows", i64), ("nnz", i64)]


class cals_plan(ctypes.Structure):
    _fields_ = [
        ("budget", P), ("small_rows", P), ("n_small", i64),
        ("small_seg", i64 * 4), ("small_seg_maxn", ctypes.c_int32 * 3), ("small_seg_maxs", ctypes.c_int32 * 3),
        ("big_rows", P), ("n_big", i64), ("big_tile_ptr", P), ("n_big_tiles", i64),
        ("big_cand_ptr", P), ("big_cand_total", i64), ("item_rows", ctypes.c_int32),
        ("n_f", ctypes.c_int32),
        ("big_tile_ptr_host", P), ("big_cand_ptr_host", P), ("big_tile_row", P), ("n_rows", i64),
    ]


class cals_tuning(ctypes.Structure):
    _fields_ = [("item_rows", ctypes.c_int32), ("ill_ratio", ctypes.c_float), ("rf_slice_max", ctypes.c_int32),
                ("gram_path", ctypes.c_int32), ("calib_samples", ctypes.c_int32), ("calib_z", ctypes.c_float),
                ("fold_chunks", ctypes.c_int32), ("serial_tiers", ctypes.c_int32),
                ("tc_debug", ctypes.c_int32), ("qtab_min_nnz", ctypes.c_int64), ("staged_max_rows", ctypes.c_int32)]


TUNING_DEFAULTS = dict(item_rows=0, ill_ratio=-1.0, rf_slice_max=-1, gram_path=0, calib_samples=0, calib_z=0.0,
                       fold_chunks=0, serial_tiers=0, tc_debug=0, qtab_min_nnz=0, staged_max_rows=0)


def set_tuning(**fields):
    """Explicit tuning of the native path (cals_set_tuning); unnamed fields take the
    defaults.  Returns the previous settings as a dict (pass them back to restore)."""
    L = load()
    prev = cals_tuning()
    L.cals_get_tuning(ctypes.byref(prev))
    old = {f: getattr(prev, f) for f, _ in cals_tuning._fields_}
    t = cals_tuning(**{**TUNING_DEFAULTS, **fields})
    L.cals_set_tuning(ctypes.byref(t))
    return old


# name -> (restype, argtypes): every symbol include/coreals_b200.h declares
SIGNATURES = {
    "cals_budget_host": (i32, [P, i64, f64, P]),
    "cals_plan_build": (i32, [P, i64, i32, f64, P, P, P, P, P, ctypes.POINTER(cals_plan)]),
    "cals_workspace_bytes": (sz, [ctypes.POINTER(cals_plan)]),
    "cals_core_half_sweep": (i32, [ctypes.POINTER(cals_side), ctypes.POINTER(cals_plan), P, i64, i32, i32, f64,
                                   P, i32, P, i32, P, P, P, P, P, P, sz, P]),
    "cals_residual": (i32, [ctypes.POINTER(cals_side), P, i32, i32, P, i32, P, P]),
    "cals_plan_build_fast": (i32, [P, i64, i32, i32, P, P, P, P, ctypes.POINTER(cals_plan)]),
    "cals_fast_sketch_workspace_bytes": (ctypes.c_size_t, [i32]),
    "cals_fast_sketch": (i32, [P, i64, i32, i32, i64, P, P, P, ctypes.c_size_t, P]),
    "cals_fast_half_sweep": (i32, [ctypes.POINTER(cals_side), ctypes.POINTER(cals_plan), P, i64, i32, i32, f64, P, P,
                                   i32, P, i32, P, P, P, P, P, ctypes.c_size_t, P]),
    "cals_sum_f64": (i32, [P, i64, P, P, sz, P]),
    "cals_weighted_sqnorm": (i32, [P, i64, i32, i32, P, P, P, sz, P]),
    "cals_ces_sketch": (i32, [P, i64, i32, ctypes.c_int32, P, P, P, sz, P]),
    "cals_ces_sketch_workspace_bytes": (sz, [i64, i32]),
    "cals_ces_sketch_f64": (i32, [P, i64, i32, ctypes.c_int32, P, P, sz, P]),
    "cals_update_core": (i32, [P, i64, i32, P, P, P, f64, i32, P, P, P]),
    "cals_predict_entries": (i32, [P, P, i32, i32, i32, P, P, i64, P, P]),
    "cals_predict_entries_f64": (i32, [P, P, i32, i32, i32, P, P, i64, P, P]),
    "cals_predict_full_f64": (i32, [P, P, i64, i64, i32, i32, i32, P, i64, P]),
    "cals_rank_metrics": (i32, [P, i64, P, P, P, i32, f64, i32, P, P, P, P, P]),
    "cals_index_workspace_bytes": (sz, [i64, i64, i64]),
    "cals_coo_to_csr": (i32, [P, P, P, i64, i64, i64, P, P, P, P, P, sz, P]),
    "cals_csr_to_csc": (i32, [P, P, P, i64, i64, i64, P, P, P, P, sz, P]),
    "cals_profile_enable": (None, [i32]),
    "cals_profile_enabled": (i32, []),
    "cals_debug_stats": (None, [P]),
    "cals_debug_big_batch": (None, [ctypes.c_int64, ctypes.c_int64]),
    "cals_set_tuning": (None, [P]),
    "cals_get_tuning": (None, [P]),
    "cals_profile_collect": (i32, [ctypes.c_char_p, sz]),
    "cals_strerror": (ctypes.c_char_p, [i32]),
    "cals_build_info": (ctypes.c_char_p, []),
}

_lib = None


def load(build_if_missing: bool = True):
    """Load (building first if needed and possible) the native library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if not build_if_missing:
            raise RuntimeError(f"{LIB_PATH} is missing; run __graft_entry__.build()")
        from . import build as _build
        _build.build()
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != CALS_OK:
        msg = load().cals_strerror(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} (status {rc})")


def profile_enable(on: bool) -> None:
    load().cals_profile_enable(1 if on else 0)


def profile_enabled() -> bool:
    return bool(load().cals_profile_enabled())


# the standalone selection kernels of a half-sweep (FitReport.sketch_time); the staged
# tier selects inside its Gram kernel and is not separable
SELECTION_KERNELS = ("quantile_table_kernel", "big_calib_kernel", "big_scan2_kernel", "big_resolve_kernel",
                     "tc_scales_kernel", "fast_sketch_kernels")


def profile_collect() -> dict:
    """{kernel name: (launches, total ms)} since the last collect."""
    buf = ctypes.create_string_buffer(1 << 16)
    load().cals_profile_collect(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


def require_cuda():
    """The product path runs on the GPU only; fail loudly otherwise."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_18024_b200 requires a CUDA device (sm_100a); there is no CPU fallback")
    load()
    return torch
