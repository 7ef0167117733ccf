"""Host value type for inputs and outputs that live in CPU memory.

Mirrors the parts of the reference ``Tensor`` (``pkg/src/mlower/tensor.py:35-153``)
a caller of ``execute``/``predict`` touches: ``from_dense``, ``shape``,
``dtype``, ``rank``, ``to_numpy``, ``rows``.  Buffers are read-only, as in the
reference (``tensor.py:19-23``).  Device-resident data does not use this class:
``execute`` takes and returns CUDA ``torch.Tensor`` objects directly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dtypes import DType, STORAGE, _fits, name_of
from .errors import ValidationError


@dataclass(frozen=True)
class Tensor:
    shape: tuple
    dtype: DType
    dense: np.ndarray

    @staticmethod
    def from_dense(values, dtype) -> "Tensor":
        arr = np.asarray(values)
        name = name_of(dtype)
        if not _fits(arr.astype(np.float64, copy=False), name):
            raise ValidationError(f"values not representable in {name}")
        out = np.array(arr, dtype=STORAGE[name], copy=True, order="C")
        out.flags.writeable = False
        return Tensor(tuple(int(s) for s in out.shape), DType(name), out)

    @property
    def rank(self) -> int:
        return len(self.shape)

    @property
    def size(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    @property
    def is_csr(self) -> bool:
        return False

    def to_numpy(self) -> np.ndarray:
        return self.dense

    def rows(self) -> list:
        if self.rank != 2:
            raise ValidationError(f"rows() requires rank 2, got {self.shape}")
        return [[float(v) for v in r] for r in self.dense]


def wrap_like(template, values: np.ndarray, dtype_name: str):
    """Build an output tensor of the same family as the caller's input.

    A reference ``Tensor`` in gives a reference ``Tensor`` out (its
    ``from_dense`` re-validates representability exactly as the reference
    executor does for every kernel output), otherwise ours.
    """
    cls = type(template)
    if cls is not Tensor and hasattr(cls, "from_dense") and hasattr(template, "dtype"):
        enum_cls = type(template.dtype)
        return cls.from_dense(values, enum_cls(dtype_name))
    return Tensor.from_dense(values, DType(dtype_name))
