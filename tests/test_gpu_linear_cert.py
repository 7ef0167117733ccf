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
