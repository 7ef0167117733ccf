"""Drive the LR 784->10 certified linear path (1M rows) for ncu / timing
probes: prints per-launch CUDA-event times of the whole program run."""
import os
import sys

import numpy as np
import torch

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__)))]
from paper_2301_13441_b200 import api  # noqa: E402
from paper_2301_13441_b200.models import LinearModel  # noqa: E402

dev = torch.device("cuda", 0)
rng = np.random.default_rng(3)
C = int(os.environ.get("PROBE_C", "10"))
lm = LinearModel("logistic_regression", 784,
                 tuple(tuple(float(v) for v in r) for r in rng.standard_normal((C, 784)).astype(np.float32) * 0.05),
                 tuple(float(v) for v in rng.standard_normal(C).astype(np.float32)), tuple(float(c) for c in range(C)))
c_lm = api.compile_model(lm)
p_lm = c_lm.program(0)
x = torch.randn((1_000_000, 784), device=dev)
n = int(os.environ.get("PROBE_ITERS", "20"))
ts = []
for i in range(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p_lm.run(x)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("impl", os.environ.get("CMLB_LINEAR_IMPL", "1"), "median ms", sorted(ts[3:])[len(ts[3:]) // 2], "min", min(ts[3:]))
if os.environ.get("CMLB_LINEAR_QSTAT"):
    from paper_2301_13441_b200 import _native as N  # noqa: E402
    print("queued rows (float64 recompute)", N.lib().cmlb_debug_linear_queued(), "of", x.shape[0])
if os.environ.get("PROBE_GAPS"):
    xh = x.cpu().numpy().astype(np.float64)
    W = np.array(lm.coef, dtype=np.float64)
    z = xh @ W.T + np.array(lm.intercept, dtype=np.float64)
    nu = (784 + 2) * 2.0 ** -24
    e = nu * np.sqrt((xh * xh).sum(1))[:, None] * 1.0625 * np.sqrt((W * W).sum(1))[None, :]
    t = z.argmax(1)
    zt = z[np.arange(len(z)), t]
    et = e[np.arange(len(z)), t]
    gap = zt[:, None] - z
    need = 2 * (et[:, None] + e)
    gap[np.arange(len(z)), t] = np.inf
    print("uncertified rows (estimate):", int((gap <= need).any(1).sum()))
