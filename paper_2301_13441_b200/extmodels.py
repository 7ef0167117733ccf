"""Model families beyond the reference schema: kernel SVMs, one-hot encoding,
column transformers and pipelines (BASELINE configs 4b/5).

The reference (``mlower``) stops at separate single models: its exporter
rejects ``Pipeline`` / ``OneHotEncoder`` (``exporter/export.py:245-246``) and
it has no kernel SVM (``SPEC.md:9``).  These families follow the reference's
JSON conventions -- one object per model discriminated by ``model_type``,
``format_version`` 1, every number rounded to float32 on the way in
(``pkg/src/mlower/models.py:201-206``) -- and their semantics are
scikit-learn's (the only oracle, "parity unpinned" against the reference):

* ``svc`` / ``svr``: libsvm's dense ``svm_predict_values`` as shipped in
  scikit-learn 1.9 -- per pair (i, j) of classes the sequential float64 sum
  over class i's support vectors with ``dual_coef[j-1]`` then class j's with
  ``dual_coef[i]``, minus rho (= -intercept); one-vs-one votes, first max.
  Binary SVC predicts ``classes[0]`` iff that decision value is > 0.
* ``one_hot_encoder``: ``OneHotEncoder.transform`` with numeric categories,
  optional ``drop`` index per input column, ``handle_unknown`` error|ignore.
* ``column_transformer``: ``ColumnTransformer`` with scaler / one-hot /
  passthrough blocks, outputs concatenated in transformer order, remainder
  columns (drop|passthrough) last in ascending index order.
* ``pipeline``: steps applied in order; every step but the last is a
  transformer.  Each step keeps its own semantics: a scaler step computes
  exactly what the reference scaler computes (float32, pinned rounding).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import SchemaError, ValidationError

SVM_TYPES = ("svc", "svr")
SVM_KERNELS = ("linear", "poly", "rbf", "sigmoid")
EXT_TYPES = SVM_TYPES + ("one_hot_encoder", "column_transformer", "pipeline")


@dataclass(frozen=True, eq=False)
class SVMModel:
    model_type: str            # "svc" | "svr"
    n_features: int
    kernel: str
    gamma: float
    coef0: float
    degree: int
    support_vectors: np.ndarray   # float32 (n_sv, F), grouped by class (svc)
    dual_coef: np.ndarray         # float32 (C - 1, n_sv) for svc, (1, n_sv) for svr
    intercept: np.ndarray         # float32 (C (C - 1) / 2,) for svc, (1,) for svr
    n_support: tuple              # per class (svc); (n_sv,) for svr
    classes: tuple | None

    @property
    def is_classifier(self) -> bool:
        return self.classes is not None

    @property
    def n_sv(self) -> int:
        return int(self.support_vectors.shape[0])

    def thresholds(self) -> list:
        return []


@dataclass(frozen=True, eq=False)
class OneHotModel:
    model_type: str
    n_features: int
    categories: tuple             # per input column: float32 array, sorted, unique
    drop: tuple                   # per input column: dropped category index or None
    handle_unknown: str           # "error" | "ignore"

    is_classifier = False

    @property
    def out_width(self) -> int:
        return sum(len(c) - (d is not None) for c, d in zip(self.categories, self.drop))

    def thresholds(self) -> list:
        return []


@dataclass(frozen=True, eq=False)
class ColumnTransformerModel:
    model_type: str
    n_features: int
    transformers: tuple           # ((columns tuple, model | "passthrough" | "drop"), ...)
    remainder: str                # "drop" | "passthrough"

    is_classifier = False

    def remainder_columns(self) -> tuple:
        used = {c for cols, _ in self.transformers for c in cols}
        if self.remainder != "passthrough":
            return ()
        return tuple(c for c in range(self.n_features) if c not in used)

    @property
    def out_width(self) -> int:
        w = 0
        for cols, m in self.transformers:
            if m == "drop":
                continue
            w += len(cols) if m == "passthrough" else out_width(m)
        return w + len(self.remainder_columns())

    def thresholds(self) -> list:
        return []


@dataclass(frozen=True, eq=False)
class PipelineModel:
    model_type: str
    n_features: int
    steps: tuple

    @property
    def is_classifier(self) -> bool:
        return bool(getattr(self.steps[-1], "is_classifier", False))

    def thresholds(self) -> list:
        return []


def is_transformer(m) -> bool:
    mt = getattr(m, "model_type", None)
    from .models import SCALER_TYPES
    return mt in SCALER_TYPES or mt in ("one_hot_encoder", "column_transformer") or (
        mt == "pipeline" and is_transformer(m.steps[-1]))


def out_width(m) -> int:
    """Output columns of a transformer (scaler, one-hot, column transformer, pipeline)."""
    mt = m.model_type
    if mt in ("one_hot_encoder", "column_transformer"):
        return m.out_width
    if mt == "pipeline":
        return out_width(m.steps[-1])
    return m.n_features


# -- parsing ---------------------------------------------------------------------


def _list(v, where):
    if not isinstance(v, list):
        raise SchemaError(f"{where}: expected list")
    return v


def _parse_svm(obj, mtype, nf):
    from .models import _classes, _field, _int, _num, _nums
    kernel = obj.get("kernel", "rbf")
    if kernel not in SVM_KERNELS:
        raise SchemaError(f"$.kernel: expected one of {SVM_KERNELS}, got {kernel!r}")
    gamma = _num(obj.get("gamma", 1.0 / nf), "$.gamma")
    coef0 = _num(obj.get("coef0", 0.0), "$.coef0")
    degree = _int(obj.get("degree", 3), "$.degree")
    if degree < 0:
        raise ValidationError("$.degree: must be >= 0")
    raw_sv = _list(_field(obj, "support_vectors", "$"), "$.support_vectors")
    if not raw_sv:
        raise ValidationError("$.support_vectors: must be non-empty")
    sv = np.array([_nums(r, f"$.support_vectors[{i}]") for i, r in enumerate(raw_sv)], dtype=np.float32)
    if sv.ndim != 2 or sv.shape[1] != nf:
        raise ValidationError(f"$.support_vectors: rows must have n_features = {nf} values")
    n_sv = sv.shape[0]
    raw_dc = _list(_field(obj, "dual_coef", "$"), "$.dual_coef")
    dc = np.array([_nums(r, f"$.dual_coef[{i}]") for i, r in enumerate(raw_dc)], dtype=np.float32)
    intercept = np.array(_nums(_field(obj, "intercept", "$"), "$.intercept"), dtype=np.float32)
    if dc.ndim != 2 or dc.shape[1] != n_sv:
        raise ValidationError(f"$.dual_coef: rows must have {n_sv} values (one per support vector)")
    if mtype == "svr":
        if dc.shape[0] != 1 or intercept.shape != (1,):
            raise ValidationError("$.dual_coef/$.intercept: svr needs one row and one intercept")
        return SVMModel(mtype, nf, kernel, gamma, coef0, degree, sv, dc, intercept, (n_sv,), None)
    classes = _classes(obj, True)
    C = len(classes)
    if C < 2:
        raise ValidationError("$.classes: classifiers need at least 2 classes")
    n_support = tuple(_int(v, f"$.n_support[{i}]") for i, v in
                      enumerate(_list(_field(obj, "n_support", "$"), "$.n_support")))
    if len(n_support) != C or any(v < 0 for v in n_support) or sum(n_support) != n_sv:
        raise ValidationError(f"$.n_support: need {C} non-negative counts summing to {n_sv}")
    if dc.shape[0] != C - 1:
        raise ValidationError(f"$.dual_coef: svc with {C} classes needs {C - 1} rows")
    if intercept.shape != (C * (C - 1) // 2,):
        raise ValidationError(f"$.intercept: svc with {C} classes needs {C * (C - 1) // 2} values")
    return SVMModel(mtype, nf, kernel, gamma, coef0, degree, sv, dc, intercept, n_support, classes)


def _parse_onehot(obj, nf):
    from .models import _int, _nums
    cats = []
    for i, c in enumerate(_list(obj.get("categories"), "$.categories")):
        v = np.array(_nums(c, f"$.categories[{i}]"), dtype=np.float32)
        if v.size == 0:
            raise ValidationError(f"$.categories[{i}]: must be non-empty")
        if np.any(np.diff(v.astype(np.float64)) <= 0):
            raise ValidationError(f"$.categories[{i}]: must be sorted and unique")
        cats.append(v)
    if len(cats) != nf:
        raise ValidationError(f"$.categories: {len(cats)} lists != n_features {nf}")
    drop_raw = obj.get("drop")
    if drop_raw is None:
        drop = (None,) * nf
    else:
        drop = tuple(None if d is None else _int(d, f"$.drop[{i}]") for i, d in enumerate(_list(drop_raw, "$.drop")))
        if len(drop) != nf:
            raise ValidationError(f"$.drop: {len(drop)} entries != n_features {nf}")
        for i, (d, c) in enumerate(zip(drop, cats)):
            if d is not None and not 0 <= d < len(c):
                raise ValidationError(f"$.drop[{i}]: index {d} out of range")
    hu = obj.get("handle_unknown", "error")
    if hu not in ("error", "ignore"):
        raise SchemaError(f"$.handle_unknown: expected error|ignore, got {hu!r}")
    return OneHotModel("one_hot_encoder", nf, tuple(cats), drop, hu)


def _sub_model(raw, where):
    from .models import model_from_obj
    if not isinstance(raw, dict):
        raise SchemaError(f"{where}: expected model object")
    raw = dict(raw)
    raw.setdefault("format_version", 1)
    try:
        return model_from_obj(raw)
    except (SchemaError, ValidationError) as e:
        raise type(e)(f"{where}: {e}") from None


def _parse_column_transformer(obj, nf):
    from .models import _int
    trs = []
    for i, t in enumerate(_list(obj.get("transformers"), "$.transformers")):
        w = f"$.transformers[{i}]"
        if not isinstance(t, dict):
            raise SchemaError(f"{w}: expected object")
        cols = tuple(_int(c, f"{w}.columns[{k}]") for k, c in enumerate(_list(t.get("columns"), f"{w}.columns")))
        if any(not 0 <= c < nf for c in cols):
            raise ValidationError(f"{w}.columns: index out of range for {nf} input columns")
        m = t.get("model")
        if m not in ("passthrough", "drop"):
            m = _sub_model(m, f"{w}.model")
            if not is_transformer(m) or m.model_type in ("pipeline", "column_transformer"):
                raise ValidationError(f"{w}.model: {m.model_type} is not a column transformer block")
            if m.n_features != len(cols):
                raise ValidationError(f"{w}.model: n_features {m.n_features} != {len(cols)} columns")
        trs.append((cols, m))
    rem = obj.get("remainder", "drop")
    if rem not in ("drop", "passthrough"):
        raise SchemaError(f"$.remainder: expected drop|passthrough, got {rem!r}")
    return ColumnTransformerModel("column_transformer", nf, tuple(trs), rem)


def _parse_pipeline(obj):
    steps = [_sub_model(s, f"$.steps[{i}]") for i, s in enumerate(_list(obj.get("steps"), "$.steps"))]
    if not steps:
        raise ValidationError("$.steps: must be non-empty")
    for i, s in enumerate(steps[:-1]):
        if not is_transformer(s):
            raise ValidationError(f"$.steps[{i}]: {s.model_type} is not a transformer")
        if out_width(s) != steps[i + 1].n_features:
            raise ValidationError(f"$.steps[{i + 1}]: n_features {steps[i + 1].n_features} != "
                                  f"{out_width(s)} columns produced by step {i}")
    return PipelineModel("pipeline", steps[0].n_features, tuple(steps))


def ext_model_from_obj(obj, mtype: str):
    if mtype == "pipeline":
        return _parse_pipeline(obj)
    from .models import _field, _int
    nf = _int(_field(obj, "n_features", "$"), "$.n_features")
    if nf <= 0:
        raise ValidationError("$.n_features: must be positive")
    if mtype in SVM_TYPES:
        return _parse_svm(obj, mtype, nf)
    if mtype == "one_hot_encoder":
        return _parse_onehot(obj, nf)
    return _parse_column_transformer(obj, nf)


# -- serialization (the inverse of parsing; used by the exporter) -----------------


def _fl(a) -> list:
    return [float(v) for v in np.asarray(a, np.float32).ravel()]


def to_obj(m) -> dict:
    """Model -> JSON object for the extended families (reference families are
    emitted by :mod:`.export`)."""
    mt = m.model_type
    if mt in SVM_TYPES:
        o = {"model_type": mt, "format_version": 1, "n_features": m.n_features, "kernel": m.kernel,
             "gamma": float(m.gamma), "coef0": float(m.coef0), "degree": int(m.degree),
             "support_vectors": [_fl(r) for r in m.support_vectors],
             "dual_coef": [_fl(r) for r in m.dual_coef], "intercept": _fl(m.intercept)}
        if mt == "svc":
            o["n_support"] = [int(v) for v in m.n_support]
            o["classes"] = [float(c) for c in m.classes]
        return o
    if mt == "one_hot_encoder":
        return {"model_type": mt, "format_version": 1, "n_features": m.n_features,
                "categories": [_fl(c) for c in m.categories],
                "drop": [None if d is None else int(d) for d in m.drop], "handle_unknown": m.handle_unknown}
    raise ValidationError(f"to_obj: {mt} is serialized by export.py")
