"""The SKEW variant's precondition (cmlb_debug_sums_order_free): a forest's
float64 sums over trees are certified exact in ANY order.  Checked against a
Python restatement of the certificate, and -- the property it promises -- by
summing the payloads of random paths in shuffled orders (every order must give
numpy's sequential and pairwise results bit for bit).  Host only (no GPU)."""

import ctypes as C
import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2301_13441_b200 import _native as N, lower  # noqa: E402
from paper_2301_13441_b200.runtime import forest_desc  # noqa: E402


def certified(spec) -> bool:
    d, keep = forest_desc(spec)
    r = N.lib().cmlb_debug_sums_order_free(C.byref(d))
    assert r in (0, 1)
    return r == 1


def restated(spec) -> bool:
    q, bound = -2000, 0.0
    for t in spec.trees:
        p = np.asarray(t.payload, np.float32)
        if not np.all(np.isfinite(p)):
            return False
        nz = p[p != 0]
        if nz.size:
            m, e = np.frexp(nz.astype(np.float64))
            qv = np.where(np.abs(nz) >= np.finfo(np.float32).tiny, 24 - e, 149)
            q = max(q, int(qv.max()))
            bound += float(np.abs(nz).max())
    return bound == 0 or math.ldexp(bound * (1 + 1e-12), q) < 2.0 ** 53


def _forest(rng, T, scale_exp):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from bench_configs import perfect_gbdt
    g = perfect_gbdt(T=T, depth=4, F=6, seed=int(rng.integers(1 << 30)))
    from paper_2301_13441_b200.models import ForestModel, TreeArrays, TreeModel
    trees = []
    for t in g.trees:
        a = t.arrays
        v = a.value.copy()
        leaf = a.is_leaf
        # RF-like probabilities with a controllable smallest magnitude
        p = rng.random(leaf.sum()).astype(np.float64) * 2.0 ** -rng.integers(0, scale_exp, leaf.sum())
        v2 = np.zeros((len(leaf), 2), np.float32)
        v2[leaf, 0] = p.astype(np.float32)
        v2[leaf, 1] = (1 - p).astype(np.float32)
        trees.append(TreeModel("decision_tree_regressor", 6,
                               TreeArrays(leaf, a.feature, a.threshold, a.left, a.right, v2), None))
    return ForestModel("random_forest_classifier", 6, tuple(trees), "mean_probability", 1.0, 0.0, (0.0, 1.0))


def test_bench_model_is_certified():
    import bench
    model, _, _ = bench.load_model()
    spec = lower.lower_model(model).stages[0]
    assert restated(spec) and certified(spec)


@pytest.mark.parametrize("scale_exp", [4, 12, 20, 40])
def test_certificate_matches_restatement_and_promise(scale_exp):
    rng = np.random.default_rng(scale_exp)
    m = _forest(rng, 200, scale_exp)
    spec = lower.lower_model(m).stages[0]
    ok = certified(spec)
    assert ok == restated(spec)
    if not ok:
        return
    # the promise: any order of any path's payloads sums to the same float64
    for _ in range(50):
        vals = np.array([t.payload[rng.integers(t.payload.shape[0])] for t in spec.trees], np.float64)
        for c in range(vals.shape[1]):
            col = vals[:, c]
            seq = 0.0
            for v in col:
                seq += v
            pw = col.reshape(1, -1, 1).sum(axis=1)[0, 0]
            assert seq == pw
            for _ in range(5):
                s = 0.0
                for v in rng.permutation(col):
                    s += v
                assert s == seq


def test_tiny_payloads_are_not_certified():
    rng = np.random.default_rng(0)
    m = _forest(rng, 64, 4)
    t0 = m.trees[0]
    v = t0.arrays.value.copy()
    v[np.flatnonzero(t0.arrays.is_leaf)[0], 0] = np.float32(1e-30)
    from paper_2301_13441_b200.models import ForestModel, TreeArrays, TreeModel
    a = t0.arrays
    trees = (TreeModel(t0.model_type, 6, TreeArrays(a.is_leaf, a.feature, a.threshold, a.left, a.right, v), None),) + m.trees[1:]
    spec = lower.lower_model(ForestModel(m.model_type, 6, trees, m.aggregation, 1.0, 0.0, m.classes)).stages[0]
    assert not certified(spec) and not restated(spec)
