"""The C oracle (full-size checker / CPU baseline) equals the numpy oracle,
which is itself pinned bit-exactly to the reference (test_oracle_golden.py)."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import fast, semantics as sem

FOREST_CASES = [n for n in gc.case_names()
                if gc.get(n).entry["model_type"] in sem._FORESTS]


@pytest.mark.parametrize("name", FOREST_CASES)
def test_c_oracle_matches_golden(name):
    case = gc.get(name)
    packed = fast.PackedForest(case.model)
    got, leaves = fast.forest_predict(packed, case.x, case.oracle_flags()["dense_selector"], want_leaves=True,
                                      threads=3)
    np.testing.assert_array_equal(got, case.want)
    np.testing.assert_array_equal(leaves, case.leaves)


def test_c_oracle_adversarial_sums():
    """Leaf values spanning 80 binades: summation order is observable."""
    rng = np.random.default_rng(5)
    case = gc.get("family_gbdt_regressor_0")
    m = case.model
    for t in m.trees:
        a = t.arrays
        e = rng.integers(-40, 40, size=a.value.shape).astype(float)
        a.value[:] = (rng.standard_normal(a.value.shape) * 2.0 ** e).astype(np.float32)
    x = rng.uniform(-10, 10, size=(3000, m.n_features)).astype(np.float32)
    want, _ = sem.predict_forest(m, x)
    got, _ = fast.forest_predict(fast.PackedForest(m), x, threads=4)
    np.testing.assert_array_equal(got, want)
