"""Small-shape runs of every TMA / mbarrier / tcgen05 kernel, for
compute-sanitizer (tests/test_gpu_sanitizer.py):

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py forest
    compute-sanitizer --tool synccheck python tools/sanitize_driver.py svm

Each family runs a few hundred rows (sanitizers serialize and instrument every
access, so shapes stay tiny) and checks the result against the oracle, so a
silent corruption under instrumentation also fails.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tools"), os.path.join(ROOT, "tests")]


def forest():
    import torch

    import bench
    from oracle import fast
    from paper_2301_13441_b200 import _native as N, lower
    from paper_2301_13441_b200.models import ForestModel
    from paper_2301_13441_b200.runtime import DeviceProgram
    model, mu, sigma = bench.load_model()
    small = ForestModel(model.model_type, model.n_features, model.trees[:160], model.aggregation, 1.0, 0.0,
                        model.classes)
    x = (np.random.default_rng(0).standard_normal((300, 28)) * sigma + mu).astype(np.float32)
    want, _ = fast.forest_predict(fast.PackedForest(small), x)
    spec = lower.lower_model(small)
    for v in (N.FOREST_SKEW, N.FOREST_RANKED, N.FOREST_PERFECT, N.FOREST_MMA):
        prog = DeviceProgram(spec, 0, forest_variant=v)
        got = prog.run(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
        assert np.array_equal(got, want), f"variant {v} differs"
        prog.close()
    from bench_configs import perfect_gbdt
    g = perfect_gbdt(T=130, depth=6, F=20)
    xg = np.random.default_rng(1).standard_normal((200, 20)).astype(np.float32)
    want, _ = fast.forest_predict(fast.PackedForest(g), xg)
    prog = DeviceProgram(lower.lower_model(g), 0, forest_variant=N.FOREST_RANKED)
    assert np.array_equal(prog.run(torch.from_numpy(xg).cuda()).cpu().numpy().astype(np.float64), want)


def svm():
    import torch

    from oracle import ext_semantics as ext
    from paper_2301_13441_b200 import api
    from bench_configs import synthetic_svc
    m = synthetic_svc(F=64, n_sv=300, C=4, seed=2)
    x = np.random.default_rng(3).standard_normal((160, 64)).astype(np.float32)
    got = api.predict(api.compile_model(m), torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64).ravel()
    _, vote = ext.svm_decision(m, x)
    assert np.array_equal(got, np.asarray(m.classes, np.float64)[vote])
    # rows on a linear SVC's hyperplane: every row takes the pair tier (scatter,
    # SV-split units, finish), the full certifying tier and the exact kernel
    from paper_2301_13441_b200.extmodels import SVMModel
    m2 = synthetic_svc(F=16, n_sv=96, C=2, seed=21)
    m2 = SVMModel(m2.model_type, m2.n_features, "linear", m2.gamma, m2.coef0, m2.degree, m2.support_vectors,
                  m2.dual_coef, m2.intercept, m2.n_support, m2.classes)
    sv = np.asarray(m2.support_vectors, np.float64)
    w = (np.asarray(m2.dual_coef, np.float64)[0][:, None] * sv).sum(0)
    b = float(np.asarray(m2.intercept, np.float64)[0])
    x2 = np.random.default_rng(5).standard_normal((200, 16))
    x2 = (x2 - ((x2 @ w + b) / (w @ w))[:, None] * w[None, :]).astype(np.float32)
    got = api.predict(api.compile_model(m2), torch.from_numpy(x2).cuda()).cpu().numpy().astype(np.float64).ravel()
    _, vote = ext.svm_decision(m2, x2)
    assert np.array_equal(got, np.asarray(m2.classes, np.float64)[vote])


def linear():
    import torch

    from oracle import semantics as sem
    from paper_2301_13441_b200 import api
    from paper_2301_13441_b200.models import LinearModel
    rng = np.random.default_rng(4)
    lm = LinearModel("logistic_regression", 96,
                     tuple(tuple(float(v) for v in r) for r in rng.standard_normal((10, 96)).astype(np.float32)),
                     tuple(float(v) for v in rng.standard_normal(10).astype(np.float32)), tuple(float(c) for c in range(10)))
    x = rng.standard_normal((700, 96)).astype(np.float32)
    got = api.predict(api.compile_model(lm), torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    want, _ = sem.predict(lm, x)
    assert np.array_equal(got, want)


if __name__ == "__main__":
    {"forest": forest, "svm": svm, "linear": linear}[sys.argv[1]]()
    print("ok", sys.argv[1])
