"""Full-size parity of the BASELINE workloads (every row, not a sample):
the north-star RF500 d8 on the bench's own 10M x 28 input and the config-5
fused pipeline on 5M x 64, against the multi-threaded C oracle (which is
itself pinned to the reference in tests/test_c_oracle.py).  Slow (~1 min)."""

import os
import sys

import numpy as np
import pytest
import torch

from oracle import ext_semantics as ext, fast

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def test_rf500_d8_all_10m_rows_bit_exact():
    import bench
    from paper_2301_13441_b200 import api
    model, mu, sigma = bench.load_model()
    compiled = api.compile_model(model)
    prog = compiled.program(0)
    n = 10_000_000
    g = torch.Generator(device="cuda").manual_seed(1)          # bench.py's rank-0 input
    x = torch.randn((n, 28), generator=g, device="cuda")
    x.mul_(torch.from_numpy(sigma).cuda()).add_(torch.from_numpy(mu).cuda())
    got = prog.run(x).cpu().numpy().astype(np.float64).ravel()
    want, _ = fast.forest_predict(fast.PackedForest(model), x.cpu().numpy())
    mism = np.flatnonzero(got != want.ravel())
    assert mism.size == 0, f"{mism.size} of {n} rows differ, first {mism[:5]}"


def test_config5_pipeline_all_5m_rows_bit_exact():
    from workloads import config5_pipeline
    from paper_2301_13441_b200 import api
    m, xh = config5_pipeline(rows=5_000_000)
    compiled = api.compile_model(m)
    got = compiled.program(0).run(torch.from_numpy(xh).cuda()).cpu().numpy().astype(np.float64).ravel()
    ct, forest = m.steps
    xt = ext.transform(ct, xh)                                   # reference scaler + sklearn one-hot semantics
    want, _ = fast.forest_predict(fast.PackedForest(forest), xt)
    mism = np.flatnonzero(got != want.ravel())
    assert mism.size == 0, f"{mism.size} of {len(xh)} rows differ"


def test_config3_gbr_all_1m_rows_bit_exact():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from bench_configs import perfect_gbdt
    from paper_2301_13441_b200 import api
    m = perfect_gbdt()
    x = torch.randn((1_000_000, 90), generator=torch.Generator(device="cuda").manual_seed(2), device="cuda")
    got = api.compile_model(m).program(0).run(x).cpu().numpy().astype(np.float64).ravel()
    want, _ = fast.forest_predict(fast.PackedForest(m), x.cpu().numpy())
    mism = np.flatnonzero(got != want.ravel())
    assert mism.size == 0, f"{mism.size} rows differ"


def test_config4a_logreg_all_1m_rows_bit_exact():
    from oracle import semantics as sem
    from paper_2301_13441_b200 import api
    from paper_2301_13441_b200.models import LinearModel
    rng = np.random.default_rng(3)
    lm = LinearModel("logistic_regression", 784,
                     tuple(tuple(float(v) for v in r) for r in rng.standard_normal((10, 784)).astype(np.float32) * 0.05),
                     tuple(float(v) for v in rng.standard_normal(10).astype(np.float32)), tuple(float(c) for c in range(10)))
    x = torch.randn((1_000_000, 784), generator=torch.Generator(device="cuda").manual_seed(3), device="cuda")
    got = api.compile_model(lm).program(0).run(x).cpu().numpy().astype(np.float64).ravel()
    xh = x.cpu().numpy()
    want = np.concatenate([sem.predict(lm, xh[i:i + 100_000])[0].ravel() for i in range(0, len(xh), 100_000)])
    mism = np.flatnonzero(got != want)
    assert mism.size == 0, f"{mism.size} rows differ"
