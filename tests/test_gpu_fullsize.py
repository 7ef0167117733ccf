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
