"""ctypes binding of ``libcmlb.so`` (the C ABI in ``include/cmlb.h``).

This is the reference-side FFI for a Python reference: plain ctypes over
``extern "C"`` entry points.  The library is REQUIRED: there is no CPU
fallback anywhere in the package, so a missing or stale build raises
immediately with the build command in the message.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceError, error_for_status

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcmlb.so")

ABI_VERSION = 3  # CMLB_ABI_VERSION in include/cmlb.h

c_i32, c_i64, c_f32, c_f64, c_vp = C.c_int32, C.c_int64, C.c_float, C.c_double, C.c_void_p
P = C.POINTER


class ColumnOp(C.Structure):
    _fields_ = [("src", c_i32), ("op", c_i32), ("a", c_f32), ("b", c_f32)]


class ForestDesc(C.Structure):
    _fields_ = [
        ("n_trees", c_i32), ("n_features", c_i32), ("n_outputs", c_i32),
        ("node_offset", P(c_i64)), ("leaf_offset", P(c_i64)),
        ("feature", P(c_i32)), ("threshold", P(c_f32)), ("left", P(c_i32)), ("right", P(c_i32)),
        ("payload", P(c_f32)),
        ("aggregation", c_i32), ("tail", c_i32), ("learning_rate", c_f32), ("base_score", c_f32),
        ("classes", P(c_f64)), ("n_classes", c_i32), ("out_dtype", c_i32),
        ("dense_selector", c_i32), ("variant", c_i32),
        ("prologue", c_vp), ("n_inputs", c_i32), ("n_trees_total", c_i32),
    ]


class LinearDesc(C.Structure):
    _fields_ = [
        ("n_features", c_i32), ("n_outputs", c_i32), ("coef", P(c_f32)), ("intercept", P(c_f32)),
        ("tail", c_i32), ("classes", P(c_f64)), ("n_classes", c_i32), ("out_dtype", c_i32),
        ("sparse_coef", c_i32), ("prologue", c_vp), ("n_inputs", c_i32),
    ]


class ScalerDesc(C.Structure):
    _fields_ = [
        ("kind", c_i32), ("n_features", c_i32), ("threshold", c_f32), ("a", P(c_f32)), ("b", P(c_f32)),
    ]


class SVMDesc(C.Structure):
    _fields_ = [
        ("n_features", c_i32), ("n_sv", c_i32), ("kernel", c_i32), ("degree", c_i32),
        ("gamma", c_f64), ("coef0", c_f64), ("support_vectors", P(c_f32)), ("dual_coef", P(c_f32)),
        ("intercept", P(c_f32)), ("n_support", P(c_i32)), ("n_classes", c_i32), ("classes", P(c_f64)),
        ("out_dtype", c_i32), ("prologue", c_vp), ("n_inputs", c_i32),
    ]


class ColumnsDesc(C.Structure):
    _fields_ = [
        ("n_inputs", c_i32), ("n_outputs", c_i32), ("ops", c_vp), ("n_checks", c_i32),
        ("check_col", P(c_i32)), ("check_offset", P(c_i64)), ("check_values", P(c_f32)),
    ]


# enum values (cmlb.h)
AGG_NONE, AGG_MEAN, AGG_SUM = 0, 1, 2
TAIL_VALUES, TAIL_ARGMAX, TAIL_SIGMOID = 0, 1, 2
FOREST_AUTO, FOREST_PERFECT, FOREST_GENERAL, FOREST_RANKED, FOREST_MMA, FOREST_SKEW = 0, 1, 2, 3, 4, 5
LIN_VALUES, LIN_ARGMAX, LIN_SOFTMAX_ARGMAX, LIN_SIGMOID, LIN_SIGN = 0, 1, 2, 3, 4
(SCALER_BINARIZER, SCALER_NORM_L1, SCALER_NORM_L2, SCALER_NORM_MAX, SCALER_MINMAX,
 SCALER_SUB_DIV, SCALER_DIV) = range(7)
SVM_KERNEL = {"linear": 0, "poly": 1, "rbf": 2, "sigmoid": 3}

_lock = threading.Lock()
_lib = None

# name -> (restype, argtypes); every declaration of include/cmlb.h
SIGNATURES = {
    "cmlb_last_error": (C.c_char_p, []),
    "cmlb_abi_version": (C.c_int, []),
    "cmlb_launch_count": (c_i64, []),
    "cmlb_forest_create": (C.c_int, [P(ForestDesc), C.c_int, P(c_vp)]),
    "cmlb_forest_run": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "cmlb_forest_partial": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "cmlb_forest_finish": (C.c_int, [c_vp, c_vp, c_i32, P(c_i32), c_i32, c_i64, c_vp, c_vp]),
    "cmlb_forest_merge": (C.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "cmlb_forest_info": (C.c_int, [c_vp, P(c_i32), P(c_i32), P(c_i32), P(c_i32)]),
    "cmlb_forest_destroy": (None, [c_vp]),
    "cmlb_linear_create": (C.c_int, [P(LinearDesc), C.c_int, P(c_vp)]),
    "cmlb_linear_run": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "cmlb_linear_destroy": (None, [c_vp]),
    "cmlb_scaler_create": (C.c_int, [P(ScalerDesc), C.c_int, P(c_vp)]),
    "cmlb_scaler_run": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "cmlb_scaler_destroy": (None, [c_vp]),
    "cmlb_svm_create": (C.c_int, [P(SVMDesc), C.c_int, P(c_vp)]),
    "cmlb_svm_run": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "cmlb_svm_destroy": (None, [c_vp]),
    "cmlb_svm_debug_fast": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "cmlb_columns_create": (C.c_int, [P(ColumnsDesc), C.c_int, P(c_vp)]),
    "cmlb_columns_run": (C.c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "cmlb_columns_destroy": (None, [c_vp]),
    "cmlb_debug_pairwise_schedule": (C.c_int, [c_i64, P(C.c_uint32)]),
    "cmlb_debug_sums_order_free": (C.c_int, [P(ForestDesc)]),
    "cmlb_debug_linear_queued": (C.c_int64, []),
}


def lib():
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"native library {LIB_PATH} is missing; build it with "
                    "`python -m paper_2301_13441_b200.build` (no CPU fallback exists)")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            if handle.cmlb_abi_version() != ABI_VERSION:
                raise DeviceError(f"{LIB_PATH} has ABI {handle.cmlb_abi_version()}, this package needs "
                                  f"{ABI_VERSION}; rebuild with `python -m paper_2301_13441_b200.build`")
            _lib = handle
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().cmlb_last_error().decode("utf-8", "replace")
        raise error_for_status(status, msg)


def ptr(arr, ctype):
    """ctypes pointer into a C-contiguous numpy array (caller keeps it alive)."""
    return arr.ctypes.data_as(P(ctype))
