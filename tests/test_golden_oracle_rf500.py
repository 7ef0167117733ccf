"""Pin the oracles to the reference on the NORTH-STAR model itself
(tests/golden/rf500_ref.npz, made by tools/make_golden_rf500.py from
mlower.execute): the C oracle and the numpy restatement must give the
reference's class of every row and its per-tree leaf indices."""

import os
import sys

import numpy as np

from oracle import fast, semantics as sem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden", "rf500_ref.npz")


def test_c_oracle_matches_reference_on_rf500():
    import bench
    model, _, _ = bench.load_model()
    z = np.load(GOLD)
    got, leaves = fast.forest_predict(fast.PackedForest(model), z["x"], want_leaves=True)
    assert np.array_equal(got.ravel(), z["want"])
    assert np.array_equal(leaves, z["leaves"].astype(np.int32))


def test_numpy_oracle_matches_reference_on_rf500():
    import bench
    model, _, _ = bench.load_model()
    z = np.load(GOLD)
    got, dtype = sem.predict(model, z["x"][:1500])
    assert dtype == str(z["want_dtype"])
    assert np.array_equal(np.asarray(got, np.float64).ravel(), z["want"][:1500])
