"""Synthetic workloads of the BASELINE configs that have no shipped model
(shared by tests/ and tools/bench_configs.py).  Test/bench infrastructure."""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def config5_pipeline(rows: int = 5_000_000, seed: int = 4):
    """Config 5: ColumnTransformer(StandardScaler on 56 numeric columns,
    OneHotEncoder(handle_unknown='error') on 8 categorical columns with 16
    categories each, stored as float codes) -> the RF500 depth-8 bench forest,
    its 28 features re-pointed onto the 56 + 128 = 184 transformed columns
    (20 onto scaled numeric columns, 8 onto one-hot indicators at 0.5).
    Returns (PipelineModel, x float32 [rows, 64])."""
    import bench
    from paper_2301_13441_b200.extmodels import ColumnTransformerModel, OneHotModel, PipelineModel
    from paper_2301_13441_b200.models import ForestModel, ScalerModel, TreeArrays, TreeModel
    rng = np.random.default_rng(seed)
    n_num, n_cat, k = 56, 8, 16
    mu = rng.standard_normal(n_num).astype(np.float32)
    sd = rng.uniform(0.5, 2.0, n_num).astype(np.float32)
    ss = ScalerModel("standard_scaler", n_num, vectors=(("mean", tuple(float(v) for v in mu)),
                                                         ("scale", tuple(float(v) for v in sd))))
    oh = OneHotModel("one_hot_encoder", n_cat, tuple(np.arange(k, dtype=np.float32) for _ in range(n_cat)),
                     (None,) * n_cat, "error")
    ct = ColumnTransformerModel("column_transformer", n_num + n_cat,
                                ((tuple(range(n_num)), ss), (tuple(range(n_num, n_num + n_cat)), oh)), "drop")
    rf, _, _ = bench.load_model()
    F2 = n_num + n_cat * k
    fmap = np.array([(f * 3) % n_num if f < 20 else n_num + ((f - 20) * k + (f * 5) % k) for f in range(28)])
    trees = []
    for t in rf.trees:
        a = t.arrays
        internal = ~a.is_leaf
        feat = np.where(internal, fmap[a.feature], 0).astype(np.int32)
        thr = np.where(internal & (feat >= n_num), np.float32(0.5), a.threshold).astype(np.float32)
        trees.append(TreeModel("decision_tree_regressor", F2, TreeArrays(a.is_leaf, feat, thr, a.left, a.right,
                                                                          a.value), None))
    forest = ForestModel("random_forest_classifier", F2, tuple(trees), "mean_probability", 1.0, 0.0, rf.classes)
    model = PipelineModel("pipeline", n_num + n_cat, (ct, forest))
    x = np.empty((rows, n_num + n_cat), np.float32)
    x[:, :n_num] = rng.standard_normal((rows, n_num), dtype=np.float32) * sd + mu
    x[:, n_num:] = rng.integers(0, k, (rows, n_cat)).astype(np.float32)
    return model, x
