"""Fit the config-4b model once and store it compactly (bench_assets/svc_digits.npz).

    python tools/make_svc_model.py        # ~1 min (libsvm, one core)

SURVEY 8d config 4b asks for ``SVC(kernel="rbf")`` fit so that n_SV ~ 10,000 on
784 features.  The data are synthetic MNIST-shaped digits (no network for the
real set): ten smooth random 28 x 28 class prototypes, each sample a prototype
at a random contrast plus heavy pixel noise, clipped and quantised to 8 bits,
scaled by 1/255 in float32 -- so every support vector is an 8-bit image and the
model ships as uint8 (the float32 values are exactly u8 / 255 in float32, the
values libsvm was trained on).  The class-prototype parameters are stored too,
so bench.py draws its 1M inference rows from the same distribution on the GPU.
"""

from __future__ import annotations

import os
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "bench_assets", "svc_digits.npz")
F, K = 784, 10
N_TRAIN = 12_300
NOISE = 200.0


def prototypes(seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    proto = np.clip(rng.normal(0, 1, (K, 28, 28)).cumsum(1).cumsum(2), 0, None)
    proto = proto / proto.max(axis=(1, 2), keepdims=True) * 255
    return proto.reshape(K, F).astype(np.float32)


def digits(proto: np.ndarray, n: int, rng) -> tuple[np.ndarray, np.ndarray]:
    y = rng.integers(0, K, n)
    x = proto[y] * rng.uniform(0.5, 1.2, (n, 1)) + rng.normal(0, NOISE, (n, F))
    return np.clip(np.round(x), 0, 255).astype(np.uint8), y


def main() -> None:
    from sklearn.svm import SVC
    proto = prototypes(0)
    x8, y = digits(proto, N_TRAIN, np.random.default_rng(1))
    X = x8.astype(np.float32) / np.float32(255)
    t = time.time()
    m = SVC(kernel="rbf").fit(X, y)
    print(f"fit {time.time() - t:.1f} s, n_SV {m.support_vectors_.shape[0]}, per class {m.n_support_.tolist()}")
    sv8 = x8[m.support_]
    assert np.array_equal((sv8.astype(np.float32) / np.float32(255)).astype(np.float64), m.support_vectors_)
    np.savez_compressed(
        OUT, sv_u8=sv8, dual_coef=m.dual_coef_.astype(np.float32), intercept=m.intercept_.astype(np.float32),
        n_support=m.n_support_.astype(np.int32), gamma=np.float32(m._gamma), classes=m.classes_.astype(np.float64),
        proto=proto, noise=np.float32(NOISE))
    print(OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()
