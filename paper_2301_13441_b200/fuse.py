"""Lowering of composite models (pipelines, column transformers, one-hot
encoders) with preprocessing fused into the consumer's row load.

The reference runs separate models only (``convert.py:255-284`` lowers each
scaler to its own kernel chain; its exporter rejects ``Pipeline`` and
``OneHotEncoder``, ``exporter/export.py:245-246``).  Here a pipeline

    ColumnTransformer(StandardScaler | OneHotEncoder | passthrough) -> model

becomes ONE kernel reading the raw rows: every model input column f is
``op_f(x[src_f])`` (``cmlb_column_op``: the reference scalers' float32
rounding, or a one-hot indicator ``x == category``), evaluated inside the
forest / linear / SVM kernel's X load.  What cannot be expressed per column
stays a stage of its own: a Normalizer (row norm) runs the scaler kernel, a
chain of two arithmetic transforms on one column materialises the first, and
a pipeline ending in a transformer runs the standalone column kernel.
``OneHotEncoder(handle_unknown='error')`` adds a membership check of its raw
columns (a small kernel); the executor raises ``ValidationError`` with
scikit-learn's message when a row holds an unknown category.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import UnresolvedKernel
from .extmodels import out_width
from .models import family_of

COL_DTYPE = np.dtype([("src", "<i4"), ("op", "<i4"), ("a", "<f4"), ("b", "<f4")])
COPY, SUB_DIV, DIV, MUL_ADD, GREATER, EQUAL = range(6)


@dataclass(eq=False)
class ColumnsSpec:
    """y[:, f] = op_f(x[:, src_f]) plus one-hot membership checks."""

    ops: np.ndarray                  # COL_DTYPE [n_out]
    n_inputs: int
    checks: list = field(default_factory=list)   # [(raw column, ascending float32 categories)]
    emit: bool = True                # False: check-only stage (ops fused downstream)
    out_dtype: str = "float32"

    @property
    def n_features(self) -> int:
        return self.n_inputs

    @property
    def out_cols(self) -> int:
        return int(self.ops.shape[0])


def _ops(rows) -> np.ndarray:
    return np.array([tuple(r) for r in rows], dtype=COL_DTYPE).reshape(-1)


def identity_ops(n: int) -> np.ndarray:
    return _ops([(i, COPY, 0.0, 0.0) for i in range(n)])


def _scaler_ops(m):
    """Per-column ops of an elementwise reference scaler, or None (Normalizer)."""
    kind, F = m.model_type, m.n_features
    v = lambda name: np.asarray(m.vector(name), np.float32)
    if kind == "normalizer":
        return None
    if kind == "binarizer":
        t = np.float32(m.threshold)
        return _ops([(i, GREATER, t, 0.0) for i in range(F)])
    if kind == "minmax_scaler":
        s, mn = v("scale"), v("min")
        return _ops([(i, MUL_ADD, s[i], mn[i]) for i in range(F)])
    if kind in ("standard_scaler", "robust_scaler"):
        c, s = v("mean" if kind == "standard_scaler" else "center"), v("scale")
        return _ops([(i, SUB_DIV, c[i], s[i]) for i in range(F)])
    if kind == "maxabs_scaler":
        s = v("scale")
        return _ops([(i, DIV, s[i], 0.0) for i in range(F)])
    raise UnresolvedKernel(f"no column lowering for {kind}")


def _onehot_ops(m):
    rows, checks = [], []
    for i, (cats, d) in enumerate(zip(m.categories, m.drop)):
        for k, c in enumerate(np.asarray(cats, np.float32)):
            if d is not None and k == d:
                continue
            rows.append((i, EQUAL, c, 0.0))
        if m.handle_unknown == "error":
            checks.append((i, np.asarray(cats, np.float32)))
    return _ops(rows), checks


def columns_of(m) -> ColumnsSpec | None:
    """ColumnsSpec of a per-column transformer, or None if it needs its own kernel."""
    mt = m.model_type
    if mt == "one_hot_encoder":
        ops, checks = _onehot_ops(m)
        return ColumnsSpec(ops, m.n_features, checks)
    if mt == "column_transformer":
        rows, checks = [], []
        for cols, sub in m.transformers:
            if sub == "drop":
                continue
            if sub == "passthrough":
                rows += [(c, COPY, 0.0, 0.0) for c in cols]
                continue
            inner = columns_of(sub)
            if inner is None:
                return None  # e.g. a Normalizer block: not per-column
            for o in inner.ops:
                rows.append((cols[int(o["src"])], int(o["op"]), o["a"], o["b"]))
            checks += [(cols[c], v) for c, v in inner.checks]
        rows += [(c, COPY, 0.0, 0.0) for c in m.remainder_columns()]
        return ColumnsSpec(_ops(rows), m.n_features, checks)
    ops = _scaler_ops(m)
    return None if ops is None else ColumnsSpec(ops, m.n_features)


def compose(first: ColumnsSpec, second: ColumnsSpec) -> ColumnsSpec | None:
    """second(first(x)) as one column map, or None when a column would need two
    arithmetic ops (the first result must then be materialised)."""
    out = []
    for o in second.ops:
        p = first.ops[int(o["src"])]
        if int(p["op"]) == COPY:
            out.append((int(p["src"]), int(o["op"]), o["a"], o["b"]))
        elif int(o["op"]) == COPY:
            out.append(tuple(p))
        else:
            return None
    checks = list(first.checks)
    for c, v in second.checks:
        p = first.ops[c]
        if int(p["op"]) != COPY:
            return None
        checks.append((int(p["src"]), v))
    return ColumnsSpec(_ops(out), first.n_inputs, checks)


def _model_stage(m, profile, passes):
    from .lower import lower_model
    return lower_model(m, profile, passes).stages


def lower_composite(model, profile=None, passes=("re", "dr", "sor")):
    """Pipeline / column transformer / one-hot encoder -> ProgramSpec with the
    per-column preprocessing fused into the consumer."""
    from .lower import ForestSpec, LinearSpec, ProgramSpec, ScalerSpec, SVMSpec, lower_scaler_model
    steps = list(model.steps) if model.model_type == "pipeline" else [model]
    stages = []
    for s in steps:
        fam = family_of(s)
        if fam in ("scaler", "columns"):
            cs = columns_of(s)
            if cs is None:
                if fam == "scaler":
                    stages.append(lower_scaler_model(s))
                    continue
                raise UnresolvedKernel(f"{s.model_type}: block needs a row-wise kernel inside a column transformer")
            if stages and isinstance(stages[-1], ColumnsSpec):
                merged = compose(stages[-1], cs)
                if merged is not None:
                    stages[-1] = merged
                    continue
            stages.append(cs)
        elif fam == "pipeline":
            stages += lower_composite(s, profile, passes).stages
        else:
            stages += _model_stage(s, profile, passes)
    # fuse a column map into the consumer that follows it
    fused = []
    for st in stages:
        prev = fused[-1] if fused else None
        if isinstance(prev, ColumnsSpec) and prev.emit and isinstance(st, (ForestSpec, LinearSpec, SVMSpec)):
            st.prologue = prev.ops
            st.n_inputs = prev.n_inputs
            if prev.checks:
                prev.emit = False      # membership check only
            else:
                fused.pop()
        fused.append(st)
    return ProgramSpec(fused, model.n_features)
