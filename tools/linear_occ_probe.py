import os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2301_13441_b200 import api
from paper_2301_13441_b200.models import LinearModel
rng = np.random.default_rng(3)
for C in (1, 10):
    k = "logistic_regression"
    cls = (0.0, 1.0) if C == 1 else tuple(float(c) for c in range(C))
    m = LinearModel(k, 784, tuple(tuple(float(v) for v in r) for r in (rng.standard_normal((C, 784)) * 0.05).astype(np.float32)),
                    tuple(float(v) for v in rng.standard_normal(C).astype(np.float32)), cls)
    p = api.compile_model(m).program(0)
    x = torch.randn((1_000_000, 784), device="cuda")
    ts = []
    for i in range(15):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); p.run(x); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print("C", C, "median ms", sorted(ts[3:])[len(ts[3:]) // 2])
