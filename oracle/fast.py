"""ctypes wrapper of oracle/liboracle.so (the multi-threaded C oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Builds the library on
first use when gcc is available.  Works on the reference's forest/tree models
and on ours (node arrays read through :func:`oracle.semantics.node_arrays`).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from . import semantics as sem

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        srcs = [os.path.join(HERE, f) for f in ("cml_oracle.c", "svm_oracle.c")]
        if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(s) for s in srcs):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        _lib = C.CDLL(LIB)
        _lib.oracle_forest.restype = C.c_int
        _lib.oracle_svm.restype = C.c_int
        _lib.oracle_svm.argtypes = [C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_void_p, C.c_int32,
                                    C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                    C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32]
    return _lib


class PackedForest:
    """Concatenated original node arrays + in-order leaf positions."""

    def __init__(self, model):
        trees = model.trees if hasattr(model, "trees") else (model,)
        parts = [sem.node_arrays(t) for t in trees]
        self.T = len(trees)
        self.C = parts[0][5].shape[1]
        self.F = model.n_features
        self.offsets = np.zeros(self.T + 1, np.int64)
        for i, p in enumerate(parts):
            self.offsets[i + 1] = self.offsets[i] + len(p[0])
        cat = lambda k, dt: np.ascontiguousarray(np.concatenate([p[k] for p in parts]).astype(dt))
        self.is_leaf = cat(0, np.uint8)
        self.feature = cat(1, np.int32)
        self.threshold = cat(2, np.float32)
        self.left = cat(3, np.int32)
        self.right = cat(4, np.int32)
        self.value = np.ascontiguousarray(np.concatenate([p[5] for p in parts]).astype(np.float32))
        self.leaf_pos = np.ascontiguousarray(np.concatenate(
            [sem.inorder_leaf_position(p[0], p[3], p[4]) for p in parts]).astype(np.int32))
        mt = model.model_type
        self.model = model
        if mt in ("random_forest_classifier", "random_forest_regressor"):
            self.agg, self.tail = 1, (1 if model.classes is not None else 0)
            self.lr, self.base = 1.0, 0.0
        elif mt in ("gbdt_regressor", "gbdt_binary_classifier"):
            self.agg, self.tail = 2, (2 if model.classes is not None else 0)
            self.lr, self.base = float(model.learning_rate), float(model.base_score)
        else:
            raise ValueError(f"C oracle covers ensembles, not {mt}")
        self.classes = np.ascontiguousarray(np.asarray(model.classes or (0.0,), np.float64))


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def forest_predict(packed: PackedForest, x: np.ndarray, dense_selector: bool = False,
                   want_leaves: bool = False, threads: int | None = None):
    x = np.ascontiguousarray(x, np.float32)
    n = x.shape[0]
    k = packed.C if packed.tail == 0 else 1
    out = np.zeros((n, k), np.float64)
    leaves = np.zeros((n, packed.T), np.int32) if want_leaves else None
    threads = threads or os.cpu_count() or 1
    st = lib().oracle_forest(
        _p(packed.offsets, C.c_int64), _p(packed.is_leaf, C.c_uint8), _p(packed.feature, C.c_int32),
        _p(packed.threshold, C.c_float), _p(packed.left, C.c_int32), _p(packed.right, C.c_int32),
        _p(packed.value, C.c_float), _p(packed.leaf_pos, C.c_int32), C.c_int32(packed.T),
        C.c_int32(packed.C), C.c_int32(packed.F), _p(x, C.c_float), C.c_int64(n), C.c_int64(x.shape[1]),
        C.c_int32(packed.agg), C.c_int32(packed.tail), C.c_float(packed.lr), C.c_float(packed.base),
        _p(packed.classes, C.c_double), C.c_int32(int(dense_selector)), _p(out, C.c_double),
        _p(leaves, C.c_int32) if leaves is not None else None, C.c_int32(threads))
    if st != 0:
        raise RuntimeError("oracle_forest failed")
    return out, leaves
