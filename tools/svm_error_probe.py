"""Calibrate the SVM fast path's error bound on the GPU: fast-path decision
values (every row, no exact path) vs the libsvm C oracle, in units of the
epilogue's per-row bound E.  Prints one JSON line per configuration."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import ext_semantics as ext  # noqa: E402
from paper_2301_13441_b200 import _native as N, api  # noqa: E402
from test_gpu_svm import _synthetic_svc  # noqa: E402


def probe(F, n_sv, C, kernel, rows=4096, seed=0):
    m = _synthetic_svc(F, n_sv, C, kernel, seed=seed)
    x = np.random.default_rng(seed + 1).standard_normal((rows, F)).astype(np.float32)
    compiled = api.compile_model(m)
    prog = compiled.program(0)
    st = prog.stages[0]
    xd = torch.from_numpy(x).cuda()
    y = torch.empty((rows, 1), dtype=torch.int8, device="cuda")
    dec = torch.empty((rows, st.pairs), dtype=torch.float64, device="cuda")
    err = torch.empty(rows, dtype=torch.float32, device="cuda")
    N.check(N.lib().cmlb_svm_debug_fast(st.handle, xd.data_ptr(), rows, F, y.data_ptr(), dec.data_ptr(),
                                        err.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want, _ = ext.svm_decision(m, x)
    d, e = dec.cpu().numpy(), err.cpu().numpy().astype(np.float64)[:, None]
    ratio = np.abs(d - want) / e
    near = (np.abs(want) <= 4 * e).any(axis=1).mean()
    out = {"F": F, "n_sv": n_sv, "C": C, "kernel": kernel, "max_err_over_E": float(ratio.max()),
           "p99_err_over_E": float(np.quantile(ratio, 0.99)), "median_E": float(np.median(e)),
           "max_abs_err": float(np.abs(d - want).max()), "frac_rows_within_4E": float(near)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for cfg in [(784, 1000, 10, "rbf"), (784, 2000, 2, "rbf"), (100, 600, 3, "rbf"), (64, 513, 4, "poly"),
                (50, 257, 5, "sigmoid"), (33, 100, 2, "linear"), (784, 500, 4, "linear")]:
        probe(*cfg)
