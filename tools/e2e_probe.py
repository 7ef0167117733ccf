"""Host-streaming (run_host) throughput vs chunk size and stream count, RF500 d8
on 10M x 28 pinned rows (H2D of X + D2H of labels inside the timed region)."""
import itertools
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2301_13441_b200 import api  # noqa: E402
from paper_2301_13441_b200.runtime import run_host  # noqa: E402

model, mu, sigma = bench.load_model()
compiled = api.compile_model(model)
prog = compiled.program(0)
n = 10_000_000
x = (torch.randn((n, 28)) * torch.from_numpy(sigma) + torch.from_numpy(mu)).float().pin_memory()
y = torch.empty((n, 1), dtype=torch.uint8).pin_memory()
# raw H2D copy rate for reference
d = torch.empty((n, 28), device="cuda")
for _ in range(2):
    d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); d.copy_(x, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(json.dumps({"h2d_gbs": n * 112 / (e0.elapsed_time(e1) / 1e3) / 1e9}), flush=True)
CH = tuple(int(v) for v in os.environ.get("E2E_CHUNKS", str((1 << 19, 1 << 20, 1 << 21, 1 << 22))).strip("()").split(",") if v.strip())
for chunk, ns in itertools.product(CH, (2, 3, 4)):
    run_host(prog, x[: chunk * ns], out_host=y[: chunk * ns], chunk_rows=chunk, n_streams=ns)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        run_host(prog, x, out_host=y, chunk_rows=chunk, n_streams=ns)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"chunk_rows": chunk, "streams": ns, "M_rows_per_s": 2 * n / (e0.elapsed_time(e1) / 1e3) / 1e6}),
          flush=True)
