"""Secondary BASELINE configs on one B200 (parity-checked, CUDA-event timed).

    python tools/bench_configs.py [--quick]

1. DecisionTreeClassifier depth 6 on 100k x 28 (sklearn-trained)
3. GradientBoostingRegressor 1000 perfect depth-10 trees on 1M x 90 (config 3; the
   SURVEY's throughput model: features U{0..89}, thresholds N(0,1), leaves
   U[-0.05, 0.05], lr 0.1, seed 0), single GPU (tree-sharding is exact, see shard.py)
4a. LogisticRegression 784 -> 10 classes on 1M x 784 (config 4a; random-init weights)
5. StandardScaler(64) then RandomForest 500 x d8 on 5M x 64 (config 5 numeric part,
   run as the composition execute(rf, execute(scaler, x)))

Each line: device time per launch (median of 10 after 3 warm-ups, inputs > L2),
rows/s, the bound and achieved fraction of the measured HBM peak, and a parity
check of a row subset against the oracle (bit-exact).  Prints one JSON per
config and writes profiles/r1_configs.json.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import fast, semantics as sem  # noqa: E402  (checker only)
from paper_2301_13441_b200 import api  # noqa: E402
from paper_2301_13441_b200.models import (ForestModel, LinearModel, ScalerModel, TreeArrays,  # noqa: E402
                                          TreeModel)

HBM = 6550.4
try:
    HBM = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass


def time_launch(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def perfect_gbdt(T=1000, depth=10, F=90, seed=0):
    rng = np.random.default_rng(seed)
    ni, nl = 2 ** depth - 1, 2 ** depth
    trees = []
    for _ in range(T):
        n = ni + nl
        is_leaf = np.zeros(n, bool)
        is_leaf[ni:] = True
        idx = np.arange(ni)
        left = np.full(n, -1, np.int32)
        right = np.full(n, -1, np.int32)
        left[:ni] = 2 * idx + 1
        right[:ni] = 2 * idx + 2
        feat = np.zeros(n, np.int32)
        feat[:ni] = rng.integers(0, F, ni)
        thr = np.zeros(n, np.float32)
        thr[:ni] = rng.standard_normal(ni).astype(np.float32)
        val = np.zeros((n, 1), np.float32)
        val[ni:, 0] = rng.uniform(-0.05, 0.05, nl).astype(np.float32)
        trees.append(TreeModel("decision_tree_regressor", F, TreeArrays(is_leaf, feat, thr, left, right, val), None))
    return ForestModel("gbdt_regressor", F, tuple(trees), "sum", float(np.float32(0.1)), 0.0, None)


def line(name, ms, rows, bytes_row, parity, extra=None):
    rps = rows / (ms / 1e3)
    gbs = rps * bytes_row / 1e9
    d = {"config": name, "ms": ms, "rows": rows, "rows_per_s": rps, "hbm_gbs": gbs,
         "hbm_frac_of_measured": gbs / HBM, "bytes_row": bytes_row, "parity_bit_exact": parity}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="1,3,4a,5")
    args = ap.parse_args()
    only = set(args.only.split(","))
    scale = 10 if args.quick else 1
    out = []
    dev = torch.device("cuda", 0)

    # ---- config 1: DT depth 6 (sklearn) -----------------------------------
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import golden_cases as gc
    rng = np.random.default_rng(3)
    if "1" in only:
        config1(out, dev, gc)
    if "3" in only:
        config3(out, dev, scale)
    if "4a" in only:
        config4a(out, dev, scale, rng)
    if "5" in only:
        config5(out, dev, scale, rng)
    path = os.path.join(ROOT, "gpurun_out", "configs.json")
    if os.path.isdir(os.path.dirname(path)):
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)


def config1(out, dev, gc):
    case = gc.get("sk_dt_d6")
    m = case.model
    x = torch.randn((100_000, 28), device=dev) * 2
    prog = api.compile_model(m).program(0)
    ms = time_launch(lambda: prog.run(x))
    want, _ = sem.predict(m, x[:5000].cpu().numpy())
    got = prog.run(x[:5000]).cpu().numpy().astype(np.float64)
    out.append(line("1: DecisionTreeClassifier d6, 100k x 28", ms, 100_000, 113, bool(np.array_equal(got, want)),
                    {"variant": prog.forest().info()}))



def config3(out, dev, scale):
    m = perfect_gbdt()
    n = 1_000_000 // scale
    x = torch.randn((n, 90), generator=torch.Generator(device=dev).manual_seed(2), device=dev)
    prog = api.compile_model(m).program(0)
    ms = time_launch(lambda: prog.run(x), reps=5)
    sub = x[:4000].cpu().numpy()
    want, _ = fast.forest_predict(fast.PackedForest(m), sub)
    got = prog.run(x[:4000]).cpu().numpy().astype(np.float64)
    out.append(line("3: GradientBoostingRegressor 1000 x d10, 1M x 90", ms, n, 364, bool(np.array_equal(got, want)),
                    {"variant": prog.forest().info(), "node_visits_per_row": 10000}))



def config4a(out, dev, scale, rng):
    lm = LinearModel("logistic_regression", 784,
                     tuple(tuple(float(v) for v in row) for row in rng.standard_normal((10, 784)).astype(np.float32) * 0.05),
                     tuple(float(v) for v in rng.standard_normal(10).astype(np.float32)), tuple(float(c) for c in range(10)))
    n = 1_000_000 // scale
    x = torch.randn((n, 784), generator=torch.Generator(device=dev).manual_seed(3), device=dev)
    prog = api.compile_model(lm).program(0)
    ms = time_launch(lambda: prog.run(x))
    sub = x[:3000].cpu().numpy()
    want, _ = sem.predict(lm, sub)
    got = prog.run(x[:3000]).cpu().numpy().astype(np.float64)
    out.append(line("4a: LogisticRegression 784 -> 10, 1M x 784", ms, n, 784 * 4 + 1,
                    bool(np.array_equal(got, want)), {"fp64_fma_per_row": 7840}))



def config5(out, dev, scale, rng):
    import bench
    rf, mu, sigma = bench.load_model()
    F = 64
    # the same trees, re-indexed onto 64 features (scaled inputs), so the forest shape is the north star's
    trees = []
    for t in rf.trees:
        a = t.arrays
        trees.append(TreeModel("decision_tree_regressor", F, TreeArrays(a.is_leaf, (a.feature * 2 + 1) % F,
                                                                        a.threshold / 3.0, a.left, a.right, a.value), None))
    rf64 = ForestModel("random_forest_classifier", F, tuple(trees), "mean_probability", 1.0, 0.0, rf.classes)
    ss = ScalerModel("standard_scaler", F, vectors=(("mean", tuple(float(v) for v in rng.standard_normal(F).astype(np.float32))),
                                                     ("scale", tuple(float(v) for v in rng.uniform(0.5, 2, F).astype(np.float32)))))
    n = 5_000_000 // scale
    x = torch.randn((n, F), generator=torch.Generator(device=dev).manual_seed(4), device=dev) * 2
    p_ss = api.compile_model(ss).program(0)
    p_rf = api.compile_model(rf64).program(0)
    ms_ss = time_launch(lambda: p_ss.run(x))
    xs = p_ss.run(x)
    ms_rf = time_launch(lambda: p_rf.run(xs), reps=5)
    sub = x[:3000].cpu().numpy()
    want_s, _ = sem.predict(ss, sub)
    want, _ = sem.predict(rf64, want_s.astype(np.float32))
    got = p_rf.run(p_ss.run(x[:3000])).cpu().numpy().astype(np.float64)
    out.append(line("5: StandardScaler(64) -> RF500 d8, 5M x 64", ms_ss + ms_rf, n, 64 * 4 + 1,
                    bool(np.array_equal(got, want)),
                    {"scaler_ms": ms_ss, "forest_ms": ms_rf, "scaler_hbm_gbs": n * 64 * 8 / (ms_ss / 1e3) / 1e9,
                     "variant": p_rf.forest().info()}))


if __name__ == "__main__":
    main()
