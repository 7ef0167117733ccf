"""The headline roofline's algorithmic count (bench.forest_wavefronts_row)
on the bench's own RF500 model: per tree 2 x depth + 2 payload wavefronts per
32 rows over 512 padded trees, plus the rank pass's bucket-table search (one
start lookup + T_f binary-lifting steps per feature, T_f from the same
bucketing as forest.cu build_rank_tables).  Pins the figure DESIGN.md quotes."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools")]


def test_rf500_algorithmic_wavefronts():
    import bench
    from paper_2301_13441_b200 import lower
    model, _, _ = bench.load_model()
    spec = lower.lower_model(model).stages[0]
    wf = bench.forest_wavefronts_row(spec, {"variant": "skew", "depth": 8})
    assert wf["trees_walked"] == 512 and wf["walk"] == 512 * 18 / 32
    assert 3.0 < wf["rank"] < 6.0
    assert abs(wf["total"] - 292.15625) < 1e-9


def test_bucket_steps_cover_the_largest_bucket():
    import bench
    rng = np.random.default_rng(0)
    for n in (0, 1, 2, 7, 1000, 5000):
        u = np.unique(rng.standard_normal(n).astype(np.float32))
        t = bench._bucket_steps(u)
        assert t >= 0 and (n == 0 or (1 << t) - 1 >= 1)
    # all thresholds in one tiny interval: one bucket holds them all
    u = np.unique((np.float32(1.0) + np.arange(300, dtype=np.float32) * np.float32(1e-7)).astype(np.float32))
    u = np.concatenate([u, np.float32([1e6])]).astype(np.float32)
    assert (1 << bench._bucket_steps(u)) - 1 >= u.size - 1
