"""Element types at the boundary.

Only what the inference path needs: the seven dtype names of the reference
lattice (``pkg/src/mlower/dtypes.py:23-36``), their host storage (BOOL is one
byte, ``dtypes.py:51-59``), dispatch promotion (``dtypes.py:112-118``) and the
smallest-exact-dtype scan that fixes the dtype of class-label outputs
(``dtypes.py:128-147``, consumed through ``gather_rows``, ``kernels.py:217``).

The DType enum is value-compatible with the reference's: ``DType("int8")``
here and ``mlower.DType("int8")`` carry the same ``.value``, which is what the
executor keys on when it receives reference objects.
"""

from __future__ import annotations

import enum

import numpy as np


class DType(enum.Enum):
    BOOL = "bool"
    INT4 = "int4"
    INT8 = "int8"
    INT16 = "int16"
    INT32 = "int32"
    FLOAT16 = "float16"
    FLOAT32 = "float32"

    def __str__(self) -> str:
        return self.value


# host numpy storage per dtype name
STORAGE = {
    "bool": np.uint8,
    "int4": np.int8,
    "int8": np.int8,
    "int16": np.int16,
    "int32": np.int32,
    "float16": np.float16,
    "float32": np.float32,
}

# integer range per dtype name (bool holds 0/1)
INT_RANGE = {
    "bool": (0, 1),
    "int4": (-8, 7),
    "int8": (-128, 127),
    "int16": (-32768, 32767),
    "int32": (-(2**31), 2**31 - 1),
}

# the native library's output element codes (include/cmlb.h: CMLB_OUT_*)
OUT_CODE = {"bool": 0, "int8": 1, "int16": 2, "int32": 3, "float32": 4}


def name_of(d) -> str:
    """Accept our DType, the reference's DType, or a plain string."""
    return d if isinstance(d, str) else d.value


def dispatch_name(d) -> str:
    """int4 runs as int8 and float16 as float32 (no native kernels for them)."""
    n = name_of(d)
    return {"int4": "int8", "float16": "float32"}.get(n, n)


def _fits(values: np.ndarray, name: str) -> bool:
    if values.size == 0:
        return True
    if name in INT_RANGE:
        lo, hi = INT_RANGE[name]
        if not np.all(np.isfinite(values)):
            return False
        return bool(np.all(values == np.floor(values)) and values.min() >= lo and values.max() <= hi)
    back = values.astype(STORAGE[name]).astype(np.float64)
    return bool(np.array_equal(back, values, equal_nan=True))


def smallest_name(values) -> str:
    """Narrowest lattice dtype that holds every value exactly."""
    v = np.asarray(values, dtype=np.float64)
    for name in ("bool", "int4", "int8", "int16", "int32"):
        if _fits(v, name):
            return name
    return "float32"


def to_enum(name: str, like=None):
    """Materialize a dtype name in the caller's enum class (ours by default)."""
    cls = type(like) if like is not None and isinstance(like, enum.Enum) else DType
    return cls(name)
