"""Pin the extended-family oracle (kernel SVMs, one-hot, column transformers,
pipelines) to golden vectors from scikit-learn and the reference.

These families are not in the reference (exporter/export.py:245-246);
scikit-learn 1.9 is their oracle.  The C restatement of libsvm must reproduce
scikit-learn's decision values BIT-EXACTLY; pipeline outputs must equal the
step-by-step composition of the reference (scalers, forests, linear) and
scikit-learn (one-hot, SVM) bit-exactly.
"""

import json

import numpy as np
import pytest

import golden_cases as gc
from oracle import ext_semantics as ext
from paper_2301_13441_b200.extmodels import to_obj
from paper_2301_13441_b200.models import parse_model


@pytest.mark.parametrize("name", gc.ext_case_names())
def test_ext_oracle_matches_golden_bitwise(name):
    case = gc.ext_get(name)
    got, dtype = ext.predict(case.model, case.x)
    assert got.shape == case.want.shape
    np.testing.assert_array_equal(got, case.want)
    if case.want_dtype is not None:
        assert dtype == case.want_dtype


@pytest.mark.parametrize("name", [n for n in gc.ext_case_names() if gc.ext_get(n).kind == "svm"])
def test_svm_decision_values_bitwise(name):
    case = gc.ext_get(name)
    dec, _ = ext.svm_decision(case.model, case.x)
    np.testing.assert_array_equal(dec, case.dec)


@pytest.mark.parametrize("name", [n for n in gc.ext_case_names() if gc.ext_get(n).kind == "pipeline"])
def test_pipeline_agrees_with_sklearn_predict_mostly(name):
    """Informational bound: scikit-learn's own Pipeline.predict computes its
    scalers in float64, so a few rows near a boundary may differ."""
    case = gc.ext_get(name)
    agree = np.mean(case.want.ravel() == case.sk_pred.ravel())
    assert agree >= 0.97, agree


@pytest.mark.parametrize("name", [n for n in gc.ext_case_names() if gc.ext_get(n).kind == "svm"])
def test_svm_json_round_trip(name):
    m = gc.ext_get(name).model
    m2 = parse_model(json.dumps(to_obj(m)))
    assert np.array_equal(m.support_vectors, m2.support_vectors)
    assert np.array_equal(m.dual_coef, m2.dual_coef) and np.array_equal(m.intercept, m2.intercept)
    assert (m.gamma, m.coef0, m.degree, m.kernel, m.n_support) == (m2.gamma, m2.coef0, m2.degree, m2.kernel,
                                                                    m2.n_support)


def test_onehot_unknown_raises():
    case = gc.ext_get("onehot_drop_first")
    x = case.x.copy()
    x[3, 2] = 12345.0
    with pytest.raises(ext.UnknownCategory):
        ext.transform(case.model, x)


def test_export_matches_reference_exporter():
    """Our exporter emits the reference exporter's objects for its families
    (pkg/exporter/export.py); checked here where the reference is present."""
    import sys
    sys.path.insert(0, "/root/reference/pkg/exporter")
    ref = pytest.importorskip("export")
    from sklearn.datasets import make_classification, make_regression
    from sklearn.ensemble import GradientBoostingRegressor, RandomForestClassifier
    from sklearn.linear_model import LogisticRegression, LinearRegression
    from sklearn.preprocessing import MinMaxScaler, Normalizer, StandardScaler
    from sklearn.tree import DecisionTreeClassifier
    from paper_2301_13441_b200.export import to_model_object
    X, y = make_classification(n_samples=300, n_features=6, n_classes=3, n_informative=4, random_state=0)
    Xr, yr = make_regression(n_samples=200, n_features=5, random_state=0)
    ests = [DecisionTreeClassifier(max_depth=4, random_state=0).fit(X, y),
            RandomForestClassifier(n_estimators=3, max_depth=3, random_state=0).fit(X, y),
            GradientBoostingRegressor(n_estimators=3, max_depth=2, random_state=0).fit(Xr, yr),
            LogisticRegression(max_iter=200).fit(X, y), LinearRegression().fit(Xr, yr),
            StandardScaler().fit(X), MinMaxScaler().fit(X), Normalizer().fit(X)]
    for e in ests:
        assert json.dumps(to_model_object(e), sort_keys=True) == json.dumps(ref.to_model_object(e), sort_keys=True), \
            type(e).__name__
