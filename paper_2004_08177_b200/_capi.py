"""ctypes binding of the C ABI declared in ``include/gdvfs.h``.

The shared library is the in-tree ``lib/libgdvfs.so`` (built by
``paper_2004_08177_b200._build``).  There is no fallback: if the library is
missing or the device is not a Blackwell GPU, calls raise ``GdError``.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# GDVFS_LIB selects another build of the same library (A/B experiments).
LIB_PATH = Path(os.environ.get("GDVFS_LIB", Path(__file__).resolve().parent / "lib" / "libgdvfs.so"))

GD_OK = 0
GD_ERR_INVALID_ARGUMENT = 1
GD_ERR_DATA = 2
GD_ERR_MISSING_ARTIFACT = 3
GD_ERR_IO = 4
GD_ERR_CUDA = 5
GD_ERR_UNSUPPORTED = 6


class ForestView(C.Structure):
    _fields_ = [
        ("n_trees", C.c_int32),
        ("tree_offsets", C.c_void_p),
        ("feature", C.c_void_p),
        ("threshold", C.c_void_p),
        ("left", C.c_void_p),
        ("right", C.c_void_p),
        ("leaf_value", C.c_void_p),
    ]


class ModelInfo(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("target", C.c_int32),
        ("n_cols", C.c_int32),
        ("n_trees", C.c_int32),
        ("n_nodes", C.c_int64),
        ("max_depth", C.c_int32),
        ("pad", C.c_int32),
        ("base_prediction", C.c_double),
        ("learning_rate", C.c_double),
    ]


class Grid(C.Structure):
    _fields_ = [
        ("rows", C.c_void_p),
        ("n_records", C.c_int64),
        ("n_cols", C.c_int32),
        ("n_cat", C.c_int32),
        ("cat_t", C.c_void_p),
        ("cat_cols", C.c_void_p),
        ("rec_of_clock", C.c_void_p),
        ("n_apps", C.c_int64),
        ("sm_clock", C.c_void_p),
        ("mem_clock", C.c_void_p),
        ("n_clocks", C.c_int32),
        ("sm_col", C.c_int32),
        ("mem_col", C.c_int32),
        ("pad", C.c_int32),
        ("budgets", C.c_void_p),
    ]


class SelectOpts(C.Structure):
    _fields_ = [("mode", C.c_int32), ("objective", C.c_int32), ("best_effort", C.c_int32), ("pad", C.c_int32)]


class GbtConfig(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("depth", C.c_int32), ("learning_rate", C.c_double),
                ("l2_leaf_reg", C.c_double), ("seed", C.c_uint64)]


class Job(C.Structure):
    _fields_ = [
        ("arrival_s", C.c_double),
        ("deadline_s", C.c_double),
        ("app_rank", C.c_int64),
        ("app_index", C.c_int32),
        ("pad", C.c_int32),
    ]


EXEC_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_int64, C.c_int32)

# Every symbol include/gdvfs.h declares, with its ctypes signature.
_P = C.c_void_p
SIGNATURES = {
    "gd_last_error": (C.c_char_p, []),
    "gd_version": (C.c_char_p, []),
    "gd_ctx_create": (C.c_int, [C.c_int32, C.POINTER(_P)]),
    "gd_ctx_destroy": (C.c_int, [_P]),
    "gd_ctx_set_stream": (C.c_int, [_P, _P]),
    "gd_ctx_synchronize": (C.c_int, [_P]),
    "gd_ctx_launch_count": (C.c_int64, [_P]),
    "gd_ctx_set_timing": (C.c_int, [_P, C.c_int]),
    "gd_ctx_kernel_times": (C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_char_p), C.c_int32,
                                      C.POINTER(C.c_int32)]),
    "gd_model_upload_gbt": (C.c_int, [_P, C.POINTER(ForestView), C.c_double, C.c_double, C.c_int32, C.c_int32,
                                      C.POINTER(_P)]),
    "gd_model_upload_linear": (C.c_int, [_P, _P, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "gd_model_load_file": (C.c_int, [_P, C.c_char_p, C.POINTER(_P)]),
    "gd_model_info_get": (C.c_int, [_P, C.POINTER(ModelInfo)]),
    "gd_model_column": (C.c_char_p, [_P, C.c_int32]),
    "gd_model_export": (C.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "gd_model_free": (C.c_int, [_P]),
    "gd_predict_rows": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int32, _P, _P]),
    "gd_predict_rows_device": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int32, _P, _P]),
    "gd_grid_select": (C.c_int, [_P, _P, _P, C.POINTER(Grid), C.POINTER(SelectOpts), _P, _P, _P]),
    "gd_grid_select_device": (C.c_int, [_P, _P, _P, C.POINTER(Grid), C.POINTER(SelectOpts), _P, _P, _P]),
    "gd_select": (C.c_int, [_P, _P, _P, C.c_int64, _P, C.c_int32, _P, C.POINTER(SelectOpts), _P]),
    "gd_microbench_dadd": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "gd_schedule_edf": (C.c_int, [_P, C.c_int64, _P, _P, _P, C.c_int32, C.c_int32, C.POINTER(SelectOpts), _P,
                                  EXEC_FN, _P, _P, _P]),
    "gd_frontier": (C.c_int, [_P, _P, _P, C.c_int64, _P, C.c_int32, C.c_int32, _P, _P, _P]),
    "gd_schedule_edf_frontier": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, _P, C.c_int32, C.c_int32,
                                           C.POINTER(SelectOpts), _P, EXEC_FN, _P, _P, _P]),
    "gd_fit_gbt": (C.c_int, [_P, _P, C.c_int64, C.c_int32, _P, C.POINTER(GbtConfig), C.c_int32, C.POINTER(_P)]),
    "gd_comm_unique_id": (C.c_int, [_P]),
    "gd_comm_init_rank": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.POINTER(_P)]),
    "gd_comm_destroy": (C.c_int, [_P]),
    "gd_gather_decisions": (C.c_int, [_P, _P, _P, _P, C.c_int32]),
    "gd_multi_create": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "gd_multi_destroy": (C.c_int, [_P]),
    "gd_multi_size": (C.c_int32, [_P]),
    "gd_multi_ctx": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "gd_multi_model_replicate": (C.c_int, [_P, _P, _P]),
    "gd_multi_grid_select": (C.c_int, [_P, _P, _P, C.POINTER(Grid), C.POINTER(SelectOpts), _P, _P, _P]),
}


class GdError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """Load (once) the native library; raise if it was never built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise GdError(GD_ERR_CUDA, f"native library {LIB_PATH} is missing; run "
                                       "`python -m paper_2004_08177_b200._build` (no CPU fallback exists)")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != GD_OK:
        msg = lib().gd_last_error()
        raise GdError(rc, msg.decode() if msg else f"gdvfs error {rc}")
