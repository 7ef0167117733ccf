"""Which stage of the SVM fast-path pipeline binds?  Times cmlb_svm_debug_fast
on 262,144 rows x 10k SVs x 784 with parts switched off (CMLB_SVM_PROBE bits:
1 = no X loads, 2 = no B copies, 4 = no epilogue math).  Results are garbage
by design; only the times matter."""
import json
import os
import subprocess
import sys

CODE = r'''
import os, sys, torch
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from bench_configs import synthetic_svc, time_launch
from paper_2301_13441_b200 import api, _native as N
m = synthetic_svc(); c = api.compile_model(m); p = c.program(0); st = p.stages[0]
n = 262144
x = torch.randn((n, 784), device="cuda"); y = torch.empty((n, 1), dtype=torch.int8, device="cuda")
dec = torch.empty((n, st.pairs), dtype=torch.float64, device="cuda"); err = torch.empty(n, device="cuda")
sh = torch.cuda.current_stream().cuda_stream
ms = time_launch(lambda: N.check(N.lib().cmlb_svm_debug_fast(st.handle, x.data_ptr(), n, 784, y.data_ptr(), dec.data_ptr(), err.data_ptr(), sh)), reps=3)
print(ms)
'''
for probe in (0, 1, 2, 4, 3, 7):
    env = dict(os.environ, CMLB_SVM_PROBE=str(probe))
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    ms = float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else None
    print(json.dumps({"probe": probe, "ms_262k_rows": ms, "err": out.stderr[-300:] if out.returncode else ""}), flush=True)
