"""scikit-learn estimators -> model JSON objects, including the families the
reference exporter rejects (``Pipeline``, ``ColumnTransformer``,
``OneHotEncoder``: ``exporter/export.py:245-246``; kernel SVMs: ``SPEC.md:9``).

For the reference families the emitted object is the one the reference
exporter produces (``pkg/exporter/export.py:56-193``; equality is checked in
``tests/test_ext_models.py`` when the reference is importable): node indices
kept verbatim, classifier trees carry raw class weights, random-forest
classifier leaves are normalised to probabilities, GBDT base score is the
estimator's raw init prediction, every number float32-rounded.  Extended
families are documented in :mod:`.extmodels`.

Host-side ingestion only: nothing here runs at predict time.
"""

from __future__ import annotations

import json

import numpy as np

from .errors import ValidationError
from .extmodels import to_obj as _ext_obj

FORMAT_VERSION = 1


class UnsupportedEstimator(ValidationError):
    """Estimator family outside the supported export surface."""


def _f32(v) -> float:
    return float(np.float32(v))


def _vec(a) -> list:
    return np.asarray(a, dtype=np.float64).astype(np.float32).ravel().tolist()


def _labels(est) -> list:
    c = np.asarray(est.classes_)
    if not np.issubdtype(c.dtype, np.number):
        raise UnsupportedEstimator(f"{type(est).__name__}: class labels must be numeric")
    return _vec(c)


def _nodes(tree, leaf_rows: np.ndarray) -> list:
    """sklearn ``Tree`` arrays -> node objects; ``leaf_rows[i]`` is node i's leaf vector."""
    cl, cr = tree.children_left, tree.children_right
    feat, thr = tree.feature, np.asarray(tree.threshold, np.float64).astype(np.float32)
    out = []
    for i in range(tree.node_count):
        if cl[i] < 0:
            out.append({"leaf": leaf_rows[i].tolist()})
        else:
            out.append({"feature": int(feat[i]), "threshold": float(thr[i]), "left": int(cl[i]),
                        "right": int(cr[i])})
    return out


def _leaf_values(tree, mode: str) -> np.ndarray:
    v = np.asarray(tree.value, np.float64)[:, 0, :]       # (nodes, outputs)
    if mode == "proba":
        tot = v.sum(axis=1, keepdims=True)
        v = np.divide(v, tot, out=v.copy(), where=tot != 0)
    elif mode == "scalar":
        v = v[:, :1]
    return v.astype(np.float32)


def _tree_obj(est, clf: bool) -> dict:
    o = {"model_type": "decision_tree_classifier" if clf else "decision_tree_regressor",
         "n_features": int(est.n_features_in_),
         "nodes": _nodes(est.tree_, _leaf_values(est.tree_, "raw" if clf else "scalar"))}
    if clf:
        o["classes"] = _labels(est)
    return o


def _forest_obj(est, clf: bool) -> dict:
    mode = "proba" if clf else "scalar"
    o = {"model_type": "random_forest_classifier" if clf else "random_forest_regressor",
         "n_features": int(est.n_features_in_), "aggregation": "mean_probability",
         "trees": [{"nodes": _nodes(e.tree_, _leaf_values(e.tree_, mode))} for e in est.estimators_]}
    if clf:
        o["classes"] = _labels(est)
    return o


def _gbdt_obj(est, clf: bool) -> dict:
    if clf and est.n_classes_ != 2:
        raise UnsupportedEstimator("multi-class GradientBoosting is not supported")
    init = est._raw_predict_init(np.zeros((1, est.n_features_in_)))
    o = {"model_type": "gbdt_binary_classifier" if clf else "gbdt_regressor",
         "n_features": int(est.n_features_in_), "aggregation": "sum",
         "learning_rate": _f32(est.learning_rate), "base_score": _f32(init[0][0]),
         "trees": [{"nodes": _nodes(st[0].tree_, _leaf_values(st[0].tree_, "scalar"))} for st in est.estimators_]}
    if clf:
        o["classes"] = _labels(est)
    return o


_LINEAR = {"LinearRegression": ("linear_regression", False), "Ridge": ("linear_regression", False),
           "SGDRegressor": ("linear_regression", False), "LinearSVR": ("linear_svr", False),
           "LogisticRegression": ("logistic_regression", True), "SGDClassifier": ("sgd_classifier", True),
           "RidgeClassifier": ("ridge_classifier", True), "Perceptron": ("perceptron", True),
           "LinearSVC": ("linear_svc", True)}


def _linear_obj(est, mtype: str, clf: bool) -> dict:
    coef = np.atleast_2d(np.asarray(est.coef_, np.float64))
    b = np.atleast_1d(np.asarray(est.intercept_, np.float64))
    if b.shape[0] != coef.shape[0]:
        b = np.full(coef.shape[0], b[0])
    o = {"model_type": mtype, "n_features": int(est.n_features_in_), "coef": [_vec(r) for r in coef],
         "intercept": _vec(b)}
    if clf:
        o["classes"] = _labels(est)
    return o


_SCALERS = {"Binarizer": "binarizer", "Normalizer": "normalizer", "MinMaxScaler": "minmax_scaler",
            "RobustScaler": "robust_scaler", "StandardScaler": "standard_scaler", "MaxAbsScaler": "maxabs_scaler"}


def _scaler_obj(est, kind: str) -> dict:
    n = int(est.n_features_in_)
    o = {"model_type": kind, "n_features": n}
    fill = lambda v, d: [d] * n if v is None else _vec(v)
    if kind == "binarizer":
        o["threshold"] = _f32(est.threshold)
    elif kind == "normalizer":
        o["norm"] = str(est.norm)
    elif kind == "minmax_scaler":
        o["scale"], o["min"] = _vec(est.scale_), _vec(est.min_)
    elif kind == "robust_scaler":
        o["center"] = fill(getattr(est, "center_", None), 0.0)
        o["scale"] = fill(getattr(est, "scale_", None), 1.0)
    elif kind == "standard_scaler":
        o["mean"] = fill(getattr(est, "mean_", None), 0.0)
        o["scale"] = fill(getattr(est, "scale_", None), 1.0)
    else:
        o["scale"] = _vec(est.scale_)
    return o


# -- extended families ------------------------------------------------------------


def _svm_obj(est) -> dict:
    from .extmodels import SVMModel
    name = type(est).__name__
    kernel = est.kernel
    if not isinstance(kernel, str) or kernel not in ("linear", "poly", "rbf", "sigmoid"):
        raise UnsupportedEstimator(f"{name}: kernel {kernel!r} is not supported")
    if getattr(est, "_sparse", False):
        raise UnsupportedEstimator(f"{name}: fitted on sparse input")
    sv = np.asarray(est.support_vectors_, np.float64).astype(np.float32)
    # libsvm's own coefficients and intercepts (sklearn flips the public
    # attributes' sign for binary SVC; predict uses these)
    dc = np.asarray(est._dual_coef_, np.float64).astype(np.float32)
    ic = np.asarray(est._intercept_, np.float64).astype(np.float32)
    F = int(est.n_features_in_)
    if name in ("SVR", "NuSVR"):
        m = SVMModel("svr", F, kernel, _f32(est._gamma), _f32(est.coef0), int(est.degree), sv, dc, ic,
                     (sv.shape[0],), None)
    else:
        m = SVMModel("svc", F, kernel, _f32(est._gamma), _f32(est.coef0), int(est.degree), sv, dc, ic,
                     tuple(int(v) for v in est._n_support), tuple(_labels(est)))
    return _ext_obj(m)


def _onehot_obj(est) -> dict:
    from .extmodels import OneHotModel
    if est.handle_unknown not in ("error", "ignore"):
        raise UnsupportedEstimator(f"OneHotEncoder: handle_unknown={est.handle_unknown!r} is not supported")
    if getattr(est, "_infrequent_enabled", False):
        raise UnsupportedEstimator("OneHotEncoder: infrequent categories are not supported")
    cats = []
    for c in est.categories_:
        c = np.asarray(c)
        if not np.issubdtype(c.dtype, np.number) or not np.all(np.isfinite(c.astype(np.float64))):
            raise UnsupportedEstimator("OneHotEncoder: categories must be finite numbers")
        cats.append(c.astype(np.float32))
    di = getattr(est, "drop_idx_", None)
    drop = tuple(None if di is None or di[i] is None else int(di[i]) for i in range(len(cats)))
    return _ext_obj(OneHotModel("one_hot_encoder", int(est.n_features_in_), tuple(cats), drop, est.handle_unknown))


def _cols(spec, n: int) -> list:
    idx = np.arange(n)[spec]
    return [int(i) for i in np.atleast_1d(idx)]


def _column_transformer_obj(est) -> dict:
    n = int(est.n_features_in_)
    trs = []
    for name, tr, cols in est.transformers_:
        if name == "remainder":
            continue
        cols = _cols(cols, n)
        if isinstance(tr, str):
            trs.append({"columns": cols, "model": tr})
        else:
            trs.append({"columns": cols, "model": to_model_object(tr)})
    rem = est.remainder if isinstance(est.remainder, str) else None
    if rem not in ("drop", "passthrough"):
        raise UnsupportedEstimator("ColumnTransformer: remainder must be 'drop' or 'passthrough'")
    return {"model_type": "column_transformer", "format_version": FORMAT_VERSION, "n_features": n,
            "transformers": trs, "remainder": rem}


def to_model_object(est) -> dict:
    """Fitted estimator -> model JSON object (reference families byte-compatible)."""
    name = type(est).__name__
    if name == "Pipeline":
        steps = [s for _, s in est.steps if s not in (None, "passthrough")]
        return {"model_type": "pipeline", "format_version": FORMAT_VERSION,
                "steps": [to_model_object(s) for s in steps]}
    if name == "ColumnTransformer":
        return _column_transformer_obj(est)
    if name == "OneHotEncoder":
        return _onehot_obj(est)
    if name in ("SVC", "NuSVC", "SVR", "NuSVR"):
        return _svm_obj(est)
    if name in ("DecisionTreeClassifier", "ExtraTreeClassifier", "DecisionTreeRegressor", "ExtraTreeRegressor"):
        o = _tree_obj(est, name.endswith("Classifier"))
    elif name in ("RandomForestClassifier", "ExtraTreesClassifier", "RandomForestRegressor", "ExtraTreesRegressor"):
        o = _forest_obj(est, name.endswith("Classifier"))
    elif name in ("GradientBoostingClassifier", "GradientBoostingRegressor"):
        o = _gbdt_obj(est, name.endswith("Classifier"))
    elif name in _LINEAR:
        o = _linear_obj(est, *_LINEAR[name])
    elif name in _SCALERS:
        o = _scaler_obj(est, _SCALERS[name])
    else:
        raise UnsupportedEstimator(f"no exporter for estimator kind {name!r}")
    o["format_version"] = FORMAT_VERSION
    return o


def to_model(est):
    """Fitted estimator -> parsed model object ready for ``compile_model``."""
    from .models import parse_model
    return parse_model(json.dumps(to_model_object(est)))
