"""Drive the HBM-bound kernels once each for an ncu metrics pass:
linear (LR 784->10, 1M rows), the column transform (config 5 columns
materialised, 5M x 64 -> 184) and its membership check, and the standalone
StandardScaler (5M x 64)."""
import os
import sys

import numpy as np
import torch

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
from paper_2301_13441_b200 import api  # noqa: E402
from paper_2301_13441_b200.fuse import ColumnsSpec  # noqa: E402
from paper_2301_13441_b200.lower import ProgramSpec  # noqa: E402
from paper_2301_13441_b200.models import LinearModel, ScalerModel  # noqa: E402
from paper_2301_13441_b200.runtime import DeviceProgram  # noqa: E402
from workloads import config5_pipeline  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(3)
lm = LinearModel("logistic_regression", 784,
                 tuple(tuple(float(v) for v in r) for r in rng.standard_normal((10, 784)).astype(np.float32) * 0.05),
                 tuple(float(v) for v in rng.standard_normal(10).astype(np.float32)), tuple(float(c) for c in range(10)))
c_lm = api.compile_model(lm)
p_lm = c_lm.program(0)
x = torch.randn((1_000_000, 784), device=dev)
for _ in range(3):
    p_lm.run(x)
m5, xh = config5_pipeline(rows=5_000_000)
x5 = torch.from_numpy(xh).to(dev)
c5 = api.compile_model(m5)
cs, fs = c5.spec.stages
cols = DeviceProgram(ProgramSpec([ColumnsSpec(fs.prologue, cs.n_inputs, cs.checks)], 64), 0)
bad = torch.empty(1, dtype=torch.int64, device=dev)
for _ in range(3):
    cols.run(x5, bad=bad)
ss = ScalerModel("standard_scaler", 64, vectors=(("mean", tuple(float(v) for v in rng.standard_normal(64))),
                                                 ("scale", tuple(float(v) for v in rng.uniform(0.5, 2, 64)))))
c_ss = api.compile_model(ss)
p_ss = c_ss.program(0)
for _ in range(3):
    p_ss.run(x5)
torch.cuda.synchronize()
print("ok")
