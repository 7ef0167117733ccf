"""The certified float32 linear path (class tails) must give the reference's
classes bit-exactly, falling back to the float64 recompute on near-ties."""

import numpy as np
import pytest
import torch

from oracle import semantics as sem
from paper_2301_13441_b200 import api
from paper_2301_13441_b200.models import LinearModel

pytestmark = pytest.mark.gpu


def lm(kind, coef, b, classes):
    return LinearModel(kind, coef.shape[1], tuple(tuple(float(v) for v in r) for r in coef.astype(np.float32)),
                       tuple(float(v) for v in np.asarray(b, np.float32)), tuple(float(c) for c in classes))


def check(m, x):
    got = api.predict(api.compile_model(m), torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    want, _ = sem.predict(m, x)
    np.testing.assert_array_equal(got, want)


def test_logreg_784x10_random():
    rng = np.random.default_rng(0)
    m = lm("logistic_regression", rng.standard_normal((10, 784)) * 0.05, rng.standard_normal(10), range(10))
    check(m, rng.standard_normal((40_000, 784)).astype(np.float32))


def test_exact_ties_take_first_max():
    rng = np.random.default_rng(1)
    w = rng.standard_normal((6, 50)).astype(np.float32)
    w[4] = w[1]                                  # classes 1 and 4 always tie
    m = lm("linear_svc", w, np.zeros(6), range(6))
    check(m, rng.standard_normal((5000, 50)).astype(np.float32))


def test_sigmoid_window_rows():
    """0 < z <= 2^-23 rounds sigmoid to exactly 0.5 -> class 0."""
    rng = np.random.default_rng(2)
    w = np.zeros((1, 8), np.float32)
    w[0, 0] = 1.0
    m = lm("logistic_regression", w, [0.0], (0.0, 1.0))
    x = np.zeros((4000, 8), np.float32)
    x[:, 0] = np.concatenate([rng.uniform(-1e-6, 1e-6, 2000), np.float32(2.0) ** -np.arange(2000) % 1e-5])
    x[:, 1:] = rng.standard_normal((4000, 7))
    check(m, x.astype(np.float32))


def test_sign_tail_and_nonfinite_rows():
    rng = np.random.default_rng(3)
    w = rng.standard_normal((1, 30)).astype(np.float32)
    w[0, 5] = 0.0
    m = lm("perceptron", w, [0.1], (-1.0, 1.0))
    x = rng.standard_normal((3000, 30)).astype(np.float32)
    x[0, 5] = np.inf   # meets a zero weight: CSR semantics skip it, dense gives NaN
    x[1, 3] = np.nan
    x[2, :] = 0.0
    check(m, x)


# --- the cp.async-tiled kernel (F % 4 == 0, aligned rows) and the per-(row,
# output) float64 recompute: ragged tiles, strides, ties, non-finite values

@pytest.mark.parametrize("n_rows", [1, 255, 256, 257, 4099])
@pytest.mark.parametrize("C", [3, 10, 16])
def test_tile_ragged_rows(n_rows, C):
    rng = np.random.default_rng(10 + C)
    m = lm("logistic_regression", rng.standard_normal((C, 64)) * 0.2, rng.standard_normal(C), range(C))
    check(m, rng.standard_normal((n_rows, 64)).astype(np.float32))


def test_tile_binary_sigmoid_and_tail_slice():
    rng = np.random.default_rng(20)
    m = lm("logistic_regression", rng.standard_normal((1, 36)) * 0.3, [0.05], (0.0, 1.0))
    x = rng.standard_normal((3001, 36)).astype(np.float32)   # 36 = two 16-feature slices + 4
    x[:50] *= 1e-7                                           # sigmoid-window rows -> recompute
    check(m, x)


def test_tile_strided_rows():
    rng = np.random.default_rng(21)
    m = lm("linear_svc", rng.standard_normal((7, 48)), rng.standard_normal(7), range(7))
    big = rng.standard_normal((2000, 56)).astype(np.float32)
    x = torch.from_numpy(big).cuda()[:, :48]                  # ldx = 56, 16-byte aligned rows
    got = api.predict(api.compile_model(m), x).cpu().numpy().astype(np.float64)
    want, _ = sem.predict(m, np.ascontiguousarray(big[:, :48]))
    np.testing.assert_array_equal(got, want)


def test_tile_ties_go_to_recompute_first_max():
    rng = np.random.default_rng(22)
    w = rng.standard_normal((12, 52)).astype(np.float32)
    w[9] = w[2]                                               # classes 2 and 9 always tie
    m = lm("linear_svc", w, np.zeros(12), range(12))
    check(m, rng.standard_normal((5000, 52)).astype(np.float32))


def test_tile_nonfinite_and_sparse_zero_weight():
    rng = np.random.default_rng(23)
    w = rng.standard_normal((4, 32)).astype(np.float32)
    w[:, 7] = 0.0
    m = lm("linear_svc", w, rng.standard_normal(4), range(4))
    x = rng.standard_normal((1000, 32)).astype(np.float32)
    x[0, 7] = np.inf     # only meets zero weights
    x[1, 3] = np.nan
    x[2, 0] = -np.inf
    x[3, :] = 0.0
    check(m, x)
