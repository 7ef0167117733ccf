"""Small SVC run for ncu: 10k SVs x 784 features, 10 classes, N rows (fast path + exact path)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import synthetic_svc  # noqa: E402
from paper_2301_13441_b200 import api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
m = synthetic_svc()
compiled = api.compile_model(m)
prog = compiled.program(0)
st = prog.stages[0]
x = torch.randn((n, m.n_features), device="cuda")
y = torch.empty((n, 1), dtype=torch.int8, device="cuda")
for _ in range(2):
    st.run(x, y, n, m.n_features, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
