"""CPU restatement of the families beyond the reference (kernel SVMs, one-hot,
column transformers, pipelines).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  These families are
not in the reference (``SPEC.md:9``; ``exporter/export.py:245-246``), so
scikit-learn 1.9 is the oracle ("parity unpinned" against the reference):
this restatement is pinned to golden vectors produced by scikit-learn itself
(``tools/make_golden_ext.py`` -> ``tests/golden/ext_*``), and pipeline steps
that ARE reference families (scalers, trees, forests, linear) use the
reference semantics of :mod:`oracle.semantics` (pinned to ``mlower``).

* SVM: libsvm's dense ``svm_predict_values`` -> ``oracle/svm_oracle.c``.
* ``OneHotEncoder.transform`` (sklearn/preprocessing/_encoders.py,
  ``_transform`` + ``_compute_transformed_categories``): column i's value is
  looked up in ``categories_[i]``; the matching indicator is 1.0; unknown
  values raise (handle_unknown='error') or give all zeros ('ignore'); the
  ``drop_idx_`` category's column is removed.
* ``ColumnTransformer.transform`` (sklearn/compose/_column_transformer.py):
  blocks in transformer order, remainder passthrough columns last.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import semantics as sem

KERNEL_CODE = {"linear": 0, "poly": 1, "rbf": 2, "sigmoid": 3}


class UnknownCategory(ValueError):
    pass


def svm_decision(m, x: np.ndarray, threads: int = 0):
    """(decision values float64 [n][pairs or 1], class index int32 [n] or None)."""
    from .fast import lib
    import os
    x = np.ascontiguousarray(x, np.float32)
    n = x.shape[0]
    sv = np.ascontiguousarray(m.support_vectors, np.float32)
    coef = np.ascontiguousarray(m.dual_coef, np.float32)
    ic = np.ascontiguousarray(m.intercept, np.float32)
    if m.model_type == "svr":
        Ccls, npairs, ns = 0, 1, np.zeros(1, np.int32)
    else:
        Ccls = len(m.classes)
        npairs = Ccls * (Ccls - 1) // 2
        ns = np.ascontiguousarray(m.n_support, np.int32)
    dec = np.zeros((n, npairs), np.float64)
    vote = np.zeros(n, np.int32)
    st = lib().oracle_svm(KERNEL_CODE[m.kernel], float(m.gamma), float(m.coef0), int(m.degree),
                          sv.ctypes.data, sv.shape[0], sv.shape[1], coef.ctypes.data, ic.ctypes.data,
                          ns.ctypes.data, Ccls, x.ctypes.data, n, x.shape[1] if n else m.n_features,
                          dec.ctypes.data, vote.ctypes.data, threads or os.cpu_count() or 1)
    if st != 0:
        raise RuntimeError("oracle_svm failed")
    return dec, (vote if Ccls else None)


def predict_svm(m, x):
    dec, vote = svm_decision(m, x)
    if m.model_type == "svr":
        return dec[:, :1].astype(np.float32).astype(np.float64), "float32"
    labels = np.asarray(m.classes, np.float64)[vote].reshape(-1, 1)
    return labels, sem.smallest_dtype(m.classes)


def onehot(m, x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, np.float32)
    blocks = []
    for i, (cats, d) in enumerate(zip(m.categories, m.drop)):
        col = x[:, i]
        hit = col[:, None] == cats[None, :]
        unknown = ~hit.any(axis=1)
        if unknown.any() and m.handle_unknown == "error":
            raise UnknownCategory(f"Found unknown categories in column {i} during transform")
        if d is not None:
            hit = np.delete(hit, d, axis=1)
        blocks.append(hit.astype(np.float32))
    return np.concatenate(blocks, axis=1) if blocks else np.zeros((x.shape[0], 0), np.float32)


def transform(m, x: np.ndarray) -> np.ndarray:
    """Transformer output (float32)."""
    x = np.asarray(x, np.float32)
    mt = m.model_type
    if mt == "one_hot_encoder":
        return onehot(m, x)
    if mt == "column_transformer":
        out = []
        for cols, sub in m.transformers:
            if sub == "drop":
                continue
            part = x[:, list(cols)]
            out.append(part if sub == "passthrough" else transform(sub, part))
        rem = m.remainder_columns()
        if rem:
            out.append(x[:, list(rem)])
        return np.concatenate(out, axis=1).astype(np.float32) if out else np.zeros((x.shape[0], 0), np.float32)
    if mt == "pipeline":
        for s in m.steps:
            x = transform(s, x)
        return x
    vals, _ = sem.predict_scaler(m, x)
    return vals.astype(np.float32)


def predict(model, x, **flags):
    """Output of the full model on host rows: (float64 values, dtype name)."""
    mt = model.model_type
    x = np.asarray(x, np.float32)
    if mt in ("svc", "svr"):
        return predict_svm(model, x)
    if mt == "pipeline":
        for s in model.steps[:-1]:
            x = transform(s, x)
        return predict(model.steps[-1], x, **flags)
    if mt in ("one_hot_encoder", "column_transformer"):
        return transform(model, x).astype(np.float64), "float32"
    return sem.predict(model, x, **flags)
