"""Serialized ``KernelPlan`` objects (JSON) for environments without the reference.

A plan written by ``tools/make_golden.py`` (from the reference's own
``translate``, ``pkg/src/mlower/runtime.py:88-144``) loads back into
lightweight objects exposing exactly the attributes the reference's
``KernelPlan`` / ``Invocation`` / ``WeightBinding`` / ``Tensor`` expose and
that :func:`lower.lower_plan` reads, so the ``execute(plan, x)`` drop-in route
is testable on the GPU box where the reference is not installed.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from .dtypes import STORAGE, DType


@dataclass(frozen=True, eq=False)
class PlanTensor:
    shape: tuple
    dtype: DType
    dense: np.ndarray | None = None
    csr: tuple | None = None  # (offsets, cols, values)

    @property
    def is_csr(self) -> bool:
        return self.csr is not None

    @property
    def rank(self) -> int:
        return len(self.shape)

    def to_numpy(self) -> np.ndarray:
        if self.csr is None:
            return self.dense
        off, cols, vals = self.csr
        out = np.zeros(self.shape, dtype=STORAGE[self.dtype.value])
        rows = np.repeat(np.arange(self.shape[0]), np.diff(off))
        out[rows, cols] = vals
        return out


@dataclass(frozen=True, eq=False)
class PlanWeight:
    name: str
    tensor: PlanTensor
    cast_to: DType | None


@dataclass(frozen=True, eq=False)
class PlanInvocation:
    node_id: int
    kernel: str
    variant: DType
    use_sparse: bool
    weights: tuple
    inputs: tuple
    output: int
    attrs: tuple

    def attr(self, name, default=None):
        for k, v in self.attrs:
            if k == name:
                return v
        return default


@dataclass(frozen=True, eq=False)
class LoadedPlan:
    invocations: tuple
    slot_shapes: tuple
    slot_dtypes: tuple
    input_slot: int
    output_slot: int
    n_features: int
    input_dtype: DType


def _dec_attr(v):
    if isinstance(v, dict) and "__dtype__" in v:
        return DType(v["__dtype__"])
    if isinstance(v, list):
        return tuple(_dec_attr(e) for e in v)
    return v


def _dec_tensor(d) -> PlanTensor:
    dt = DType(d["dtype"])
    shape = tuple(d["shape"])
    if "csr" in d:
        c = d["csr"]
        return PlanTensor(shape, dt, csr=(np.asarray(c["offsets"], np.int64), np.asarray(c["cols"], np.int64),
                                          np.asarray(c["values"], np.float64).astype(STORAGE[dt.value])))
    arr = np.asarray(d["dense"], np.float64).astype(STORAGE[dt.value]).reshape(shape)
    return PlanTensor(shape, dt, dense=arr)


def load_plan(text: str) -> LoadedPlan:
    obj = json.loads(text)
    invs = []
    for i in obj["invocations"]:
        invs.append(PlanInvocation(
            node_id=i["node_id"], kernel=i["kernel"], variant=DType(i["variant"]),
            use_sparse=bool(i["use_sparse"]),
            weights=tuple(PlanWeight(w["name"], _dec_tensor(w["tensor"]),
                                     DType(w["cast_to"]) if w["cast_to"] else None) for w in i["weights"]),
            inputs=tuple(i["inputs"]), output=i["output"],
            attrs=tuple((k, _dec_attr(v)) for k, v in i["attrs"]),
        ))
    return LoadedPlan(
        invocations=tuple(invs),
        slot_shapes=tuple(tuple(s) for s in obj["slot_shapes"]),
        slot_dtypes=tuple(DType(d) for d in obj["slot_dtypes"]),
        input_slot=obj["input_slot"], output_slot=obj["output_slot"],
        n_features=obj["n_features"], input_dtype=DType(obj["input_dtype"]),
    )


def load_plan_file(path: str) -> LoadedPlan:
    with open(path) as fh:
        return load_plan(fh.read())
