"""Golden vectors for the families beyond the reference (kernel SVMs, one-hot,
column transformers, pipelines) -> tests/golden/ext_index.json + ext_arrays.npz
(inputs, expected outputs, decision values and the model JSON bytes).

Run in the build container (needs scikit-learn and, for pipeline steps that
are reference families, the reference package at /root/reference):

    python tools/make_golden_ext.py

Oracles:
* SVC / NuSVC / SVR: scikit-learn itself.  The fitted estimator's libsvm
  parameters are first rounded to float32 exactly as the model JSON stores
  them (support vectors, dual coefficients, intercepts, gamma, coef0), so
  scikit-learn's predict / decision_function ARE the semantics of the JSON.
* OneHotEncoder / ColumnTransformer: scikit-learn ``transform``.
* Pipelines: each step by its own oracle -- the reference (``mlower``
  compile_model + execute) for scaler / tree / forest / linear steps,
  scikit-learn for one-hot and SVM steps -- composed step by step.
  scikit-learn's own ``Pipeline.predict`` is also stored (``sk_pred``) for an
  agreement statistic only: its scalers compute in float64, the reference's
  in float32.
"""

from __future__ import annotations

import copy
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
OUT = os.path.join(ROOT, "tests", "golden")

from paper_2301_13441_b200.export import to_model_object  # noqa: E402


def f32r(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def round_svm(est):
    """Copy of a fitted libsvm estimator whose parameters are float32-exact."""
    e = copy.deepcopy(est)
    e.support_vectors_ = np.ascontiguousarray(f32r(e.support_vectors_))
    e._dual_coef_ = np.ascontiguousarray(f32r(e._dual_coef_))
    e._intercept_ = np.ascontiguousarray(f32r(e._intercept_))
    if hasattr(e, "dual_coef_"):
        e.dual_coef_ = -e._dual_coef_ if _binary_svc(e) else e._dual_coef_
        e.intercept_ = -e._intercept_ if _binary_svc(e) else e._intercept_
    e._gamma = float(np.float32(e._gamma))
    e.coef0 = float(np.float32(e.coef0))
    return e


def _binary_svc(e):
    return type(e).__name__ in ("SVC", "NuSVC") and len(e.classes_) == 2


def svm_golden(est, x):
    e = round_svm(est)
    name = type(e).__name__
    if name in ("SVR", "NuSVR"):
        want = e.predict(x.astype(np.float64)).astype(np.float32).astype(np.float64).reshape(-1, 1)
        dec = e._decision_function(x.astype(np.float64)).reshape(-1, 1)
        return e, want, dec
    want = e.predict(x.astype(np.float64)).astype(np.float64).reshape(-1, 1)
    e.decision_function_shape = "ovo"
    dec = e.decision_function(x.astype(np.float64))
    if _binary_svc(e):
        dec = -dec.reshape(-1, 1)  # libsvm sign (sklearn flips it for binary)
    return e, want, dec


def ref_step(step, x):
    """Reference semantics of one pipeline step on float32 rows."""
    import mlower
    from mlower.tensor import Tensor
    from mlower.dtypes import DType
    name = type(step).__name__
    if name == "OneHotEncoder":
        return step.transform(x.astype(np.float32)).astype(np.float32), None
    if name == "ColumnTransformer":
        parts = []
        n = x.shape[1]
        for tname, tr, cols in step.transformers_:
            if tname == "remainder" and tr == "drop":
                continue
            idx = np.arange(n)[cols]
            if tr == "drop" or len(np.atleast_1d(idx)) == 0:
                continue
            sub = x[:, idx]
            parts.append(sub if tr == "passthrough" else ref_step(tr, sub)[0])
        return np.concatenate(parts, axis=1).astype(np.float32), None
    if name in ("SVC", "NuSVC", "SVR", "NuSVR"):
        _, want, _ = svm_golden(step, x)
        return want, ("float32" if name.endswith("SVR") else None)
    m = mlower.parse_model(json.dumps(to_model_object(step)))
    res = mlower.execute(mlower.compile_model(m).plan, Tensor.from_dense(x.astype(np.float32), DType.FLOAT32))
    return res.to_numpy().astype(np.float64 if res.dtype.value != "float32" else np.float32), res.dtype.value


def pipeline_golden(pipe, x):
    cur = x.astype(np.float32)
    steps = [s for _, s in pipe.steps]
    for s in steps[:-1]:
        cur = ref_step(s, cur)[0].astype(np.float32)
    out, dt = ref_step(steps[-1], cur)
    return np.asarray(out, np.float64), dt


def main():
    from sklearn.compose import ColumnTransformer
    from sklearn.datasets import make_classification, make_regression
    from sklearn.ensemble import RandomForestClassifier
    from sklearn.linear_model import LogisticRegression
    from sklearn.pipeline import Pipeline
    from sklearn.preprocessing import MinMaxScaler, OneHotEncoder, StandardScaler
    from sklearn.svm import SVC, SVR, NuSVC

    rng = np.random.default_rng(20261017)
    cases = []  # (name, estimator, x, kind)

    def special(n, F, base):
        rows = base[rng.integers(0, len(base), n)].copy()
        return rows

    # ---- kernel SVMs -----------------------------------------------------------
    X, y = make_classification(n_samples=600, n_features=12, n_informative=6, n_classes=4, random_state=0)
    X = X.astype(np.float32)
    xt = np.concatenate([rng.standard_normal((250, 12)).astype(np.float32) * 1.5, X[:50]])
    for kern, kw in (("rbf", {}), ("poly", {"degree": 3, "coef0": 0.5}), ("sigmoid", {"coef0": 0.1}),
                     ("linear", {})):
        cases.append((f"svc4_{kern}", SVC(kernel=kern, gamma=0.05, **kw).fit(X, y), xt, "svm"))
    yb = (y % 2).astype(np.float64) * 3.0 - 1.0   # labels {-1, 2}
    cases.append(("svc2_rbf", SVC(kernel="rbf", gamma="scale").fit(X, yb), xt, "svm"))
    cases.append(("svc2_poly2", SVC(kernel="poly", degree=2, gamma=0.1, coef0=1.0).fit(X, yb), xt, "svm"))
    cases.append(("nusvc3_rbf", NuSVC(nu=0.3, gamma=0.08).fit(X, y % 3), xt, "svm"))
    Xr, yr = make_regression(n_samples=500, n_features=10, n_informative=6, noise=0.2, random_state=1)
    Xr = Xr.astype(np.float32)
    yr = yr / np.abs(yr).max()
    cases.append(("svr_rbf", SVR(kernel="rbf", gamma=0.1, C=2.0, epsilon=0.01).fit(Xr, yr),
                  rng.standard_normal((300, 10)).astype(np.float32), "svm"))
    # config 4b scaled down: 784 features, 10 classes
    Xl, yl = make_classification(n_samples=1500, n_features=784, n_informative=50, n_classes=10,
                                 random_state=0)
    Xl = Xl.astype(np.float32)
    cases.append(("svc10_rbf_784", SVC(kernel="rbf").fit(Xl[:700], yl[:700]),
                  np.concatenate([rng.standard_normal((200, 784)).astype(np.float32), Xl[:56]]), "svm"))

    # ---- one-hot / column transformer / pipelines ------------------------------
    n = 3000
    num = rng.standard_normal((n, 10)).astype(np.float32)
    cat = np.stack([rng.integers(0, k, n) for k in (3, 5, 8, 16)], axis=1).astype(np.float32)
    cat[:, 2] = cat[:, 2] * 0.5 - 1.0  # non-integer category codes
    Xm = np.concatenate([num[:, :5], cat[:, :2], num[:, 5:], cat[:, 2:]], axis=1)  # 14 columns, cats at 5,6,12,13
    ym = ((num[:, 0] + cat[:, 1] * 0.3 + (cat[:, 3] > 7)) > 0.8).astype(np.int64)
    cat_cols, num_cols = [5, 6, 12, 13], [0, 1, 2, 3, 4, 7, 8, 9, 10, 11]
    xm_test = Xm[:400].copy()
    oh = OneHotEncoder(handle_unknown="ignore", sparse_output=False).fit(Xm[:, cat_cols])
    xo = Xm[:300, cat_cols].copy()
    xo[:20, 1] = 99.0  # unknown category -> all zeros under 'ignore'
    cases.append(("onehot_ignore", oh, xo, "transform"))
    oh_drop = OneHotEncoder(drop="first", sparse_output=False).fit(Xm[:, cat_cols])
    cases.append(("onehot_drop_first", oh_drop, Xm[:300, cat_cols], "transform"))
    ct = ColumnTransformer([("num", StandardScaler(), num_cols),
                            ("cat", OneHotEncoder(sparse_output=False), cat_cols)]).fit(Xm)
    cases.append(("ct_std_onehot", ct, xm_test, "transform"))
    ct2 = ColumnTransformer([("mm", MinMaxScaler(), [0, 1, 2]), ("cat", OneHotEncoder(sparse_output=False), [5, 6])],
                            remainder="passthrough").fit(Xm)
    cases.append(("ct_minmax_onehot_rem", ct2, xm_test, "transform"))
    pipe_rf = Pipeline([("pre", ColumnTransformer([("num", StandardScaler(), num_cols),
                                                   ("cat", OneHotEncoder(sparse_output=False), cat_cols)])),
                        ("rf", RandomForestClassifier(n_estimators=16, max_depth=7, random_state=0))]).fit(Xm, ym)
    cases.append(("pipe_ct_rf16", pipe_rf, xm_test, "pipeline"))
    pipe_lr = Pipeline([("ss", StandardScaler()), ("lr", LogisticRegression(max_iter=300))]).fit(Xl[:800], yl[:800])
    cases.append(("pipe_ss_logreg_784", pipe_lr, Xl[800:1000], "pipeline"))
    pipe_svc = Pipeline([("pre", ColumnTransformer([("num", StandardScaler(), num_cols),
                                                    ("cat", OneHotEncoder(sparse_output=False), cat_cols)])),
                         ("svc", SVC(kernel="rbf", gamma=0.1))]).fit(Xm[:1000], ym[:1000])
    cases.append(("pipe_ct_svc", pipe_svc, xm_test, "pipeline"))

    index, arrays = [], {}
    for name, est, x, kind in cases:
        x = np.ascontiguousarray(x, np.float32)
        entry = {"name": name, "kind": kind}
        if kind == "svm":
            e, want, dec = svm_golden(est, x)
            entry["model_json"] = json.dumps(to_model_object(e))
            entry["want_dtype"] = "float32" if type(e).__name__.endswith("SVR") else None
            arrays[f"{name}__dec"] = dec
        elif kind == "transform":
            want = est.transform(x).astype(np.float64)
            entry["model_json"] = json.dumps(to_model_object(est))
            entry["want_dtype"] = "float32"
        else:
            steps = [s for _, s in est.steps]
            last = steps[-1]
            if type(last).__name__ in ("SVC", "NuSVC", "SVR", "NuSVR"):
                est = copy.deepcopy(est)
                est.steps[-1] = (est.steps[-1][0], round_svm(last))
            want, dt = pipeline_golden(est, x)
            entry["model_json"] = json.dumps(to_model_object(est))
            entry["want_dtype"] = dt
            arrays[f"{name}__sk_pred"] = np.asarray(est.predict(x), np.float64)
        # model JSON rides in the compressed npz (the 784-feature models are MBs of text)
        arrays[f"{name}__model"] = np.frombuffer(entry.pop("model_json").encode(), np.uint8)
        arrays[f"{name}__x"] = x
        arrays[f"{name}__want"] = np.asarray(want, np.float64).reshape(len(x), -1)
        index.append(entry)
        print(name, "rows", len(x), "want", arrays[f"{name}__want"].shape, flush=True)
    with open(os.path.join(OUT, "ext_index.json"), "w") as fh:
        json.dump(index, fh, indent=0)
    np.savez_compressed(os.path.join(OUT, "ext_arrays.npz"), **arrays)


if __name__ == "__main__":
    main()
