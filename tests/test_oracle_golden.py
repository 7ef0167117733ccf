"""Pin the numpy oracle to golden vectors produced by the reference itself.

The oracle must reproduce the reference output BIT-EXACTLY (not merely within
tolerance) on every golden case -- including NaN/inf/-0.0 rows, boundary rows
(feature == threshold) and the profile/pass variants -- before any GPU result
is compared against it.
"""

import numpy as np
import pytest

import golden_cases as gc
from oracle import semantics as sem


@pytest.mark.parametrize("name", gc.case_names())
def test_oracle_matches_reference_bitwise(name):
    case = gc.get(name)
    got, dtype = sem.predict(case.model, case.x, **case.oracle_flags())
    assert dtype == case.want_dtype
    assert got.shape == case.want.shape
    np.testing.assert_array_equal(got, case.want)


@pytest.mark.parametrize("name", [n for n in gc.case_names() if gc.get(n).leaves is not None])
def test_oracle_leaf_indices_match_reference(name):
    case = gc.get(name)
    m = case.model
    dense = case.oracle_flags()["dense_selector"]
    if hasattr(m, "trees"):
        got = sem.forest_leaf_indices(m, case.x, dense)
    else:
        xs = sem.poison_dense_selector(case.x) if dense and m.internal_count() else case.x
        got = sem.tree_leaf_index(m, xs).reshape(-1, 1)
    np.testing.assert_array_equal(got, case.leaves)
