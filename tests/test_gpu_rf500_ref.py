"""The north-star model itself against the REFERENCE (tests/golden/rf500_ref.npz,
made by tools/make_golden_rf500.py from mlower.execute): class labels and the
per-tree in-order leaf index of every row, under every forest variant, plus
per-tree leaves at scale (1M rows of the bench input against the C oracle)
for RF500 and for config 3's GBR 1000 x d10."""

import os
import sys

import numpy as np
import pytest
import torch

from oracle import fast

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
GOLD = os.path.join(ROOT, "tests", "golden", "rf500_ref.npz")

pytestmark = pytest.mark.gpu

from paper_2301_13441_b200 import _native as N, api, lower  # noqa: E402
from paper_2301_13441_b200.errors import UnresolvedKernel  # noqa: E402
from paper_2301_13441_b200.runtime import DeviceProgram  # noqa: E402

VARIANTS = {"auto": N.FOREST_AUTO, "skew": N.FOREST_SKEW, "ranked": N.FOREST_RANKED, "perfect": N.FOREST_PERFECT,
            "general": N.FOREST_GENERAL, "mma": N.FOREST_MMA}


@pytest.fixture(scope="module")
def rf500():
    import bench
    model, mu, sigma = bench.load_model()
    return model, mu, sigma, lower.lower_model(model)


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_rf500_classes_and_leaves_match_reference(rf500, variant):
    model, _, _, spec = rf500
    z = np.load(GOLD)
    x = torch.from_numpy(z["x"]).cuda()
    prog = DeviceProgram(spec, 0, forest_variant=VARIANTS[variant])
    leaves = torch.full((x.shape[0], len(model.trees)), -1, dtype=torch.int32, device="cuda")
    y = prog.run(x, leaf_out=leaves)
    assert str(z["want_dtype"]) == "bool" and y.dtype == torch.uint8
    got = y.cpu().numpy().astype(np.float64).ravel()
    bad = np.flatnonzero(got != z["want"])
    assert bad.size == 0, f"{variant}: {bad.size} class mismatches, first rows {bad[:5]}"
    lv = leaves.cpu().numpy()
    bad = np.argwhere(lv != z["leaves"].astype(np.int32))
    assert bad.size == 0, f"{variant}: {len(bad)} leaf mismatches, first (row, tree) {bad[:5].tolist()}"
    y2 = prog.run(x)  # the path without leaf output
    assert torch.equal(y2, y)
    prog.close()


def _leaves_vs_oracle(prog, model, x, chunk=100_000):
    packed = fast.PackedForest(model)
    T = len(model.trees)
    for r0 in range(0, x.shape[0], chunk):
        xs = x[r0:r0 + chunk]
        leaves = torch.empty((xs.shape[0], T), dtype=torch.int32, device="cuda")
        y = prog.run(xs, leaf_out=leaves)
        want, want_leaves = fast.forest_predict(packed, xs.cpu().numpy(), want_leaves=True)
        lv = leaves.cpu().numpy()
        bad = np.argwhere(lv != want_leaves)
        assert bad.size == 0, f"rows {r0}+: {len(bad)} leaf mismatches, first {bad[:3].tolist()}"
        got = y.cpu().numpy().astype(np.float64)
        assert np.array_equal(got, want), f"rows {r0}+: outputs differ"


def test_rf500_leaves_1m_rows_of_bench_input(rf500):
    model, mu, sigma, spec = rf500
    g = torch.Generator(device="cuda").manual_seed(1)  # bench.py's rank-0 input, first 1M rows
    x = torch.randn((10_000_000, 28), generator=g, device="cuda")[:1_000_000]
    x.mul_(torch.from_numpy(sigma).cuda()).add_(torch.from_numpy(mu).cuda())
    prog = api.compile_model(model).program(0)
    _leaves_vs_oracle(prog, model, x)


def test_gbr1000_d10_leaves_1m_rows():
    from bench_configs import perfect_gbdt
    m = perfect_gbdt()
    x = torch.randn((1_000_000, 90), generator=torch.Generator(device="cuda").manual_seed(2), device="cuda")
    prog = api.compile_model(m).program(0)
    _leaves_vs_oracle(prog, m, x)
