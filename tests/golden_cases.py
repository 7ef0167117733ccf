"""Loader for the golden vectors written by tools/make_golden.py (reference run)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

from paper_2301_13441_b200.models import parse_model

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def _index():
    with open(os.path.join(GOLDEN, "index.json")) as fh:
        return json.load(fh)["cases"]


@functools.lru_cache(maxsize=1)
def _arrays():
    return dict(np.load(os.path.join(GOLDEN, "arrays.npz")))


class Case:
    def __init__(self, entry: dict):
        self.entry = entry
        self.name = entry["name"]
        self.profile = entry["profile"]
        self.passes = tuple(entry["passes"])
        arr = _arrays()
        self.x = arr[f"{self.name}__x"]
        self.want = arr[f"{self.name}__want"]
        self.leaves = arr.get(f"{self.name}__leaves")
        self.want_dtype = entry["want_dtype"]

    @functools.cached_property
    def model(self):
        return parse_model(self.entry["model_json"])

    @property
    def plan_path(self):
        p = self.entry.get("plan")
        return os.path.join(GOLDEN, p) if p else None

    def oracle_flags(self) -> dict:
        """How this case's profile/passes shape the reference semantics."""
        sor = "sor" in self.passes and self.profile == "cpu-avx2"
        m = self.model
        flags = {"dense_selector": not (sor and 1.0 / m.n_features < 0.3)}
        if hasattr(m, "coef"):
            w = np.asarray(m.coef, np.float64)
            flags["sparse_coef"] = sor and np.count_nonzero(w) / w.size < 0.3
            flags["softmax"] = "re" not in self.passes
        return flags

    @property
    def is_classifier(self) -> bool:
        return getattr(self.model, "classes", None) is not None


def all_cases():
    return [Case(e) for e in _index()]


def case_names():
    return [e["name"] for e in _index()]


def get(name: str) -> Case:
    for e in _index():
        if e["name"] == name:
            return Case(e)
    raise KeyError(name)


def agrees(case: Case, got: np.ndarray, tol: float = 1e-5) -> bool:
    """Reference acceptance rule (helpers.py:336-339): classes exact, floats 1e-5 rel."""
    want = case.want
    if got.shape != want.shape:
        return False
    if case.is_classifier:
        return bool(np.array_equal(got, want))
    both_nan = np.isnan(got) & np.isnan(want)
    same = (got == want) | both_nan
    close = np.abs(got - want) <= tol * np.maximum(np.abs(want), 1.0)
    return bool(np.all(same | close))


# -- extended families (tools/make_golden_ext.py: scikit-learn + reference steps) --


@functools.lru_cache(maxsize=1)
def _ext_index():
    with open(os.path.join(GOLDEN, "ext_index.json")) as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=1)
def _ext_arrays():
    return dict(np.load(os.path.join(GOLDEN, "ext_arrays.npz")))


class ExtCase:
    def __init__(self, entry: dict):
        self.entry = entry
        self.name = entry["name"]
        self.kind = entry["kind"]          # svm | transform | pipeline
        arr = _ext_arrays()
        self.x = arr[f"{self.name}__x"]
        self.want = arr[f"{self.name}__want"]
        self.dec = arr.get(f"{self.name}__dec")
        self.sk_pred = arr.get(f"{self.name}__sk_pred")
        self.model_json = bytes(arr[f"{self.name}__model"]).decode()
        self.want_dtype = entry["want_dtype"]

    @functools.cached_property
    def model(self):
        return parse_model(self.model_json)

    @property
    def is_classifier(self) -> bool:
        return bool(getattr(self.model, "is_classifier", False))


def ext_case_names():
    return [e["name"] for e in _ext_index()]


def ext_get(name: str) -> ExtCase:
    for e in _ext_index():
        if e["name"] == name:
            return ExtCase(e)
    raise KeyError(name)
