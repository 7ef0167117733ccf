"""Secondary BASELINE configs on one B200 (parity-checked, CUDA-event timed).

    python tools/bench_configs.py [--quick]

1. DecisionTreeClassifier depth 6 on 100k x 28 (sklearn-trained)
3. GradientBoostingRegressor 1000 perfect depth-10 trees on 1M x 90 (config 3; the
   SURVEY's throughput model: features U{0..89}, thresholds N(0,1), leaves
   U[-0.05, 0.05], lr 0.1, seed 0), single GPU (tree-sharding is exact, see shard.py)
4a. LogisticRegression 784 -> 10 classes on 1M x 784 (config 4a; random-init weights)
4b. SVC RBF, 10,000 support vectors, 10 classes, on 1M x 784 (config 4b; synthetic
   model: SVs N(0,1), dual coefficients U(-1,1), gamma 1/784 -- a 784-feature SVC with
   10k SVs takes minutes to fit and 31 MB to ship, so the shape is synthesized)
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
    ap.add_argument("--only", default="1,3,4a,4b,5")
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
    if "4b" in only:
        config4b(out, dev, scale)
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



def synthetic_svc(F=784, n_sv=10_000, C=10, seed=5):
    from paper_2301_13441_b200.extmodels import SVMModel
    rng = np.random.default_rng(seed)
    sv = rng.standard_normal((n_sv, F)).astype(np.float32)
    n_support = np.full(C, n_sv // C)
    n_support[: n_sv - n_support.sum()] += 1
    dc = rng.uniform(-1, 1, (C - 1, n_sv)).astype(np.float32)
    ic = rng.uniform(-0.5, 0.5, C * (C - 1) // 2).astype(np.float32)
    return SVMModel("svc", F, "rbf", float(np.float32(1.0 / F)), 0.0, 3, sv, dc, ic,
                    tuple(int(v) for v in n_support), tuple(float(c) for c in range(C)))


def svc_model():
    """Config 4b: sklearn SVC(kernel="rbf") fit on synthetic MNIST-shaped 8-bit
    digits, 9,626 support vectors (tools/make_svc_model.py ->
    bench_assets/svc_digits.npz); support vectors are exactly u8 / 255 in f32."""
    from paper_2301_13441_b200.extmodels import SVMModel
    z = np.load(os.path.join(ROOT, "bench_assets", "svc_digits.npz"))
    sv = z["sv_u8"].astype(np.float32) / np.float32(255)
    return SVMModel("svc", 784, "rbf", float(z["gamma"]), 0.0, 3, sv, z["dual_coef"], z["intercept"],
                    tuple(int(v) for v in z["n_support"]), tuple(float(c) for c in z["classes"]))


def svc_inputs(dev, rank: int, n: int):
    """Inference rows from the model's own distribution: a class prototype at a
    random contrast plus pixel noise, clipped and quantised to 8 bits, / 255."""
    import torch
    z = np.load(os.path.join(ROOT, "bench_assets", "svc_digits.npz"))
    g = torch.Generator(device=dev)
    g.manual_seed(3 + rank)
    proto = torch.from_numpy(z["proto"]).to(dev)
    y = torch.randint(0, proto.shape[0], (n,), generator=g, device=dev)
    x = proto[y] * (0.5 + 0.7 * torch.rand((n, 1), generator=g, device=dev))
    x += float(z["noise"]) * torch.randn((n, 784), generator=g, device=dev)
    return x.round_().clamp_(0, 255).div_(255.0)


def tf32_peak():
    p = os.path.join(ROOT, "profiles", "peaks_tf32.json")
    if os.path.exists(p):
        return float(json.load(open(p))["tf32_tflops_burst"]), "profiles/peaks_tf32.json (measured cuBLAS TF32)"
    return 1100.0, "nominal 1.1 PFLOP/s dense (B200_PROFILING.md)"


def config4b(out, dev, scale):
    from oracle import ext_semantics as ext
    m = synthetic_svc()
    F, nsv = m.n_features, m.n_sv
    n = 1_000_000 // scale
    x = torch.randn((n, F), generator=torch.Generator(device=dev).manual_seed(3), device=dev)
    compiled = api.compile_model(m)
    prog = compiled.program(0)
    st = prog.stages[0]
    y = torch.empty((n, 1), dtype=torch.int8, device=dev)
    ex = torch.zeros(1, dtype=torch.int32, device=dev)
    sh = torch.cuda.current_stream().cuda_stream
    ms = time_launch(lambda: st.run(x, y, n, F, sh, exact_rows=ex), reps=5)
    n_exact = int(ex.item())
    from paper_2301_13441_b200 import _native as NN
    dec = torch.empty((n, st.pairs), dtype=torch.float64, device=dev)
    err = torch.empty(n, dtype=torch.float32, device=dev)
    ms_fast = time_launch(lambda: NN.check(NN.lib().cmlb_svm_debug_fast(
        st.handle, x.data_ptr(), n, F, y.data_ptr(), dec.data_ptr(), err.data_ptr(), sh)), reps=3)
    st.run(x, y, n, F, sh, exact_rows=ex)
    sub = 1024
    want_dec, vote = ext.svm_decision(m, x[:sub].cpu().numpy())
    got = y[:sub].cpu().numpy().astype(np.float64).ravel()
    parity = bool(np.array_equal(got, np.asarray(m.classes)[vote]))
    flops_row = 2.0 * F * nsv
    peak, src = tf32_peak()
    achieved = n * flops_row / (ms / 1e3) / 1e12
    out.append(line("4b: SVC RBF 10k SVs, 10 classes, 1M x 784", ms, n, F * 4 + 1, parity,
                    {"gemm_flops_per_row": flops_row, "achieved_tflops": achieved,
                     "tensor_issued_tflops_3xtf32": 3 * achieved, "tf32_peak_tflops": peak, "peak_source": src,
                     "frac_of_tf32_peak_algorithmic": achieved / peak, "frac_of_tf32_peak_issued": 3 * achieved / peak,
                     "exact_path_rows": n_exact, "parity_rows": sub, "fast_path_only_ms": ms_fast,
                     "fast_path_tflops_algorithmic": n * flops_row / (ms_fast / 1e3) / 1e12}))


def config5(out, dev, scale, rng):
    """Config 5: ColumnTransformer(StandardScaler 56 + OneHotEncoder 8 x 16) -> RF500 d8
    on 5M x 64, fused (one forest kernel with the column prologue + the one-hot
    membership check) vs materialised (column kernel writes the 184 model
    columns, then the forest)."""
    from oracle import ext_semantics as ext
    from paper_2301_13441_b200.fuse import ColumnsSpec
    from paper_2301_13441_b200.lower import ProgramSpec
    from paper_2301_13441_b200.runtime import DeviceProgram
    from workloads import config5_pipeline
    n = 5_000_000 // scale
    m, xh = config5_pipeline(rows=n)
    x = torch.from_numpy(xh).to(dev)
    compiled = api.compile_model(m)
    prog = compiled.program(0)
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    ms = time_launch(lambda: prog.run(x, bad=bad), reps=5)
    assert int(bad.item()) == -1
    from paper_2301_13441_b200 import _native as NN
    l0 = NN.lib().cmlb_launch_count()
    prog.run(x, bad=bad)
    launches = NN.lib().cmlb_launch_count() - l0
    cs, fs = prog.spec.stages
    unfused = DeviceProgram(ProgramSpec([ColumnsSpec(fs.prologue, cs.n_inputs, cs.checks),
                                         type(fs)(**{**fs.__dict__, "prologue": None, "n_inputs": 0})], 64), 0)
    ms_unfused = time_launch(lambda: unfused.run(x, bad=bad), reps=5)
    sub = 3000
    want, _ = ext.predict(m, xh[:sub])
    got = prog.run(x[:sub]).cpu().numpy().astype(np.float64)
    got_u = unfused.run(x[:sub]).cpu().numpy().astype(np.float64)
    out.append(line("5: ColumnTransformer(StandardScaler 56 + OneHot 8x16) -> RF500 d8, 5M x 64 (fused)", ms, n,
                    64 * 4 + 1, bool(np.array_equal(got, want) and np.array_equal(got_u, want)),
                    {"unfused_ms": ms_unfused, "fusion_speedup": ms_unfused / ms, "model_columns": 184,
                     "variant": prog.stages[-1].info(), "launches_per_step": launches}))


if __name__ == "__main__":
    main()
