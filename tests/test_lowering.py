"""CPU tests of the lowering (no GPU): both routes agree on every golden case.

Route 1 lowers the model arrays directly; route 2 inverts the reference's own
tensor encoding from a KernelPlan (serialized fixtures, and -- when the
reference is importable in this container -- freshly compiled plans for every
profile / pass subset the golden set covers).
"""

import os
import sys

import numpy as np
import pytest

import golden_cases as gc
from paper_2301_13441_b200 import lower
from paper_2301_13441_b200.errors import UnresolvedKernel
from paper_2301_13441_b200.planio import load_plan_file
from paper_2301_13441_b200.trees import canon_from_arrays, canon_from_encoding, routes_matrix
from paper_2301_13441_b200.models import tree_arrays_of

REF_SRC = "/root/reference/pkg/src"


def _ref():
    if not os.path.isdir(REF_SRC):
        return None
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    import mlower
    return mlower


PLAN_CASES = [n for n in gc.case_names() if gc.get(n).plan_path]


@pytest.mark.parametrize("name", PLAN_CASES)
def test_fixture_plan_lowers_like_model(name):
    case = gc.get(name)
    plan = load_plan_file(case.plan_path)
    a = lower.lower_plan(plan)
    b = lower.lower_model(case.model, case.profile, case.passes)
    assert lower.specs_equal(a, b)
    assert a.out_dtype == case.want_dtype


@pytest.mark.parametrize("name", gc.case_names())
def test_reference_plan_lowers_like_model(name):
    mlower = _ref()
    if mlower is None:
        pytest.skip("reference not present")
    case = gc.get(name)
    m = mlower.parse_model(case.entry["model_json"])
    compiled = mlower.compile_model(m, profile=mlower.BUILTIN_PROFILES[case.profile], passes=case.passes)
    a = lower.lower_plan(compiled.plan)
    b = lower.lower_model(case.model, case.profile, case.passes)
    c = lower.lower_model(m, case.profile, case.passes)  # reference model objects lower too
    assert lower.specs_equal(a, b)
    assert lower.specs_equal(b, c)
    assert a.out_dtype == case.want_dtype
    assert a.out_cols == case.want.shape[1]


def test_routes_matrix_matches_reference_kats():
    # test_convert.py:109-120 known answers for tree_a / tree_b
    want = {"fixture_tree_a": [[0, 1, 1], [1, 0, 1]], "fixture_tree_b": [[0, 0, 1], [0, 1, 1]]}
    for name, w3 in want.items():
        m = gc.get(name).model
        t = canon_from_arrays(tree_arrays_of(m))
        np.testing.assert_array_equal(routes_matrix(t), np.asarray(w3, np.uint8))


def test_encoding_round_trip_all_small_shapes():
    """Every full binary tree shape up to 7 internal nodes: encode -> decode."""
    from paper_2301_13441_b200.models import TreeArrays

    def shapes(n):
        if n == 0:
            yield None
            return
        for k in range(n):
            for l in shapes(k):
                for r in shapes(n - 1 - k):
                    yield (l, r)

    count = 0
    for n in range(1, 8):
        for shp in shapes(n):
            nodes = []

            def build(s):
                i = len(nodes)
                nodes.append(None)
                if s is None:
                    nodes[i] = ("leaf", float(i))
                else:
                    left = build(s[0])
                    right = build(s[1])
                    nodes[i] = ("node", i % 3, float(i) + 0.5, left, right)
                return i

            build(shp)
            k = len(nodes)
            a = TreeArrays(
                is_leaf=np.array([x[0] == "leaf" for x in nodes]),
                feature=np.array([x[1] if x[0] == "node" else 0 for x in nodes], np.int32),
                threshold=np.array([x[2] if x[0] == "node" else 0 for x in nodes], np.float32),
                left=np.array([x[3] if x[0] == "node" else -1 for x in nodes], np.int32),
                right=np.array([x[4] if x[0] == "node" else -1 for x in nodes], np.int32),
                value=np.array([[x[1]] if x[0] == "leaf" else [0.0] for x in nodes], np.float32),
            )
            t = canon_from_arrays(a)
            w1 = np.zeros((3, t.n_internal))
            w1[t.feature, np.arange(t.n_internal)] = 1
            back = canon_from_encoding(w1, t.threshold, routes_matrix(t), t.payload)
            assert back.same_as(t)
            count += 1
    assert count == 1 + 2 + 5 + 14 + 42 + 132 + 429


def test_bad_encoding_is_rejected():
    t = canon_from_arrays(tree_arrays_of(gc.get("fixture_tree_a").model))
    w3 = routes_matrix(t).copy()
    w3[0] = 1 - w3[0]  # no longer a left-prefix
    w1 = np.zeros((2, t.n_internal))
    w1[t.feature, np.arange(t.n_internal)] = 1
    with pytest.raises(UnresolvedKernel):
        canon_from_encoding(w1, t.threshold, w3, t.payload)
