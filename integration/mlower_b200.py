"""Reference-side binding: what a maintainer adds next to ``mlower/runtime.py``.

    # mlower/runtime.py (reference), after the existing execute():
    from mlower_b200 import make_execute
    execute = make_execute(execute)          # forest plans on the B200, the rest interpreted

This is the ctypes FFI a Python reference binds.  It
uses no PyTorch: device memory comes from the CUDA runtime through ctypes, and
the plan -> descriptor step is the pure-Python half of paper_2301_13441_b200
(``lower.lower_plan`` inverts the plan's W1/W2/W3 tensors into canonical trees,
``descs.forest_desc`` packs ``cmlb_forest_desc``).  A plan whose lowering is a
single fused forest (every tree / forest / GBDT plan ``compile_model`` emits)
runs through ``cmlb_forest_create`` + ``cmlb_forest_run``; everything else
(linear models, scalers, hand-built graphs) stays on the reference interpreter.
Device programs are cached per plan, like the package's own executor.

Exercised by tests/test_gpu_reference_swap.py: the reference's own test suite
runs with ``mlower.runtime.execute`` replaced by ``make_execute(execute)``.
"""

from __future__ import annotations

import ctypes as C
import ctypes.util
import functools
import os
import threading
import weakref

import numpy as np

from paper_2301_13441_b200 import _native as N
from paper_2301_13441_b200.descs import forest_desc
from paper_2301_13441_b200.errors import UnresolvedKernel
from paper_2301_13441_b200.lower import ForestSpec, lower_plan

_NP = {"bool": np.uint8, "int8": np.int8, "int16": np.int16, "int32": np.int32, "float32": np.float32}


@functools.lru_cache(maxsize=None)
def _cudart():
    for name in ("libcudart.so.12", ctypes.util.find_library("cudart") or "", "/usr/local/cuda/lib64/libcudart.so"):
        if not name:
            continue
        try:
            lib = C.CDLL(name)
        except OSError:
            continue
        lib.cudaMalloc.argtypes = [C.POINTER(C.c_void_p), C.c_size_t]
        lib.cudaFree.argtypes = [C.c_void_p]
        lib.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        return lib
    raise OSError("CUDA runtime library not found")


_H2D, _D2H = 1, 2


class _DeviceForest:
    """One plan's forest program on device 0 (freed with the plan)."""

    def __init__(self, spec: ForestSpec, n_in: int, out_cols: int, out_dtype: str):
        self.lib = N.lib()
        d, keep = forest_desc(spec)
        h = C.c_void_p()
        N.check(self.lib.cmlb_forest_create(C.byref(d), 0, C.byref(h)))
        del keep
        self.h, self.n_in, self.out_cols, self.out_dtype = h, n_in, out_cols, out_dtype
        self.lock = threading.Lock()
        self.dx, self.dy, self.cap_x, self.cap_y = C.c_void_p(), C.c_void_p(), 0, 0  # grow-only device buffers

    def _ensure(self, rt, nx: int, ny: int):
        if nx > self.cap_x:
            if self.cap_x:
                rt.cudaFree(self.dx)
            self.cap_x = 0
            if rt.cudaMalloc(C.byref(self.dx), nx):
                raise MemoryError("cudaMalloc failed")
            self.cap_x = nx
        if ny > self.cap_y:
            if self.cap_y:
                rt.cudaFree(self.dy)
            self.cap_y = 0
            if rt.cudaMalloc(C.byref(self.dy), ny):
                raise MemoryError("cudaMalloc failed")
            self.cap_y = ny

    def run(self, x: np.ndarray) -> np.ndarray:
        rt = _cudart()
        n = x.shape[0]
        y = np.empty((n, self.out_cols), _NP[self.out_dtype])
        if n == 0:
            return y
        with self.lock:  # one call at a time per plan: the device buffers are the plan's
            self._ensure(rt, x.nbytes, y.nbytes)
            if rt.cudaMemcpy(self.dx, x.ctypes.data, x.nbytes, _H2D):
                raise RuntimeError("cudaMemcpy H2D failed")
            N.check(self.lib.cmlb_forest_run(self.h, self.dx, n, x.shape[1], self.dy, None, None))  # legacy stream
            if rt.cudaMemcpy(y.ctypes.data, self.dy, y.nbytes, _D2H):  # synchronizes with the kernel
                raise RuntimeError("cudaMemcpy D2H failed")
        return y

    def __del__(self):
        try:
            rt = _cudart()
            if self.cap_x:
                rt.cudaFree(self.dx)
            if self.cap_y:
                rt.cudaFree(self.dy)
            self.lib.cmlb_forest_destroy(self.h)
        except Exception:
            pass


_lock = threading.Lock()
_cache: dict = {}
STATS = {"b200": 0, "interpreted": 0}


def _program(plan):
    key = id(plan)
    with _lock:
        if key in _cache:
            return _cache[key]
    try:
        spec = lower_plan(plan)
        st = spec.stages[0] if len(spec.stages) == 1 else None
        prog = _DeviceForest(st, spec.n_features, st.out_cols, st.out_dtype) if isinstance(st, ForestSpec) else None
    except UnresolvedKernel:
        prog = None
    with _lock:
        _cache[key] = prog
    weakref.finalize(plan, lambda k=key: _cache.pop(k, None))
    return prog


def make_execute(interpret):
    """Wrap the reference's ``execute(plan, x)``: same signature, same checks
    (``runtime.py:200-205``, done by the interpreter's own code path for the
    plans it keeps), same output ``Tensor`` type and dtype."""
    from mlower.dtypes import DType
    from mlower.errors import InputMismatch
    from mlower.tensor import Tensor

    def execute(plan, x):
        if x.rank != 2 or x.shape[1] != plan.n_features:
            raise InputMismatch(f"input shape {x.shape} does not match (batch, {plan.n_features})")
        if x.dtype != plan.input_dtype:
            raise InputMismatch(f"input dtype {x.dtype} != {plan.input_dtype}")
        prog = _program(plan) if os.environ.get("MLOWER_B200", "1") != "0" else None
        if prog is None:
            STATS["interpreted"] += 1
            return interpret(plan, x)
        y = prog.run(np.ascontiguousarray(x.to_numpy(), np.float32))
        STATS["b200"] += 1
        return Tensor.from_dense(y, DType(prog.out_dtype))

    execute.__wrapped__ = interpret
    return execute
