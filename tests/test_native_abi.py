"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/cmlb.h declares, and its host-only helpers behave (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2301_13441_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "cmlb.h")).read()
    return sorted(set(re.findall(r"\b(cmlb_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(N.LIB_PATH):
        from paper_2301_13441_b200.build import build
        build()
    return N.lib()


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} has no ctypes signature"


def test_abi_version(lib):
    assert lib.cmlb_abi_version() == 3
    assert lib.cmlb_launch_count() >= 0


def test_create_rejects_bad_descriptors_without_gpu(lib):
    d = N.ForestDesc()
    d.n_trees = 0
    h = N.c_vp()
    st = lib.cmlb_forest_create(ctypes.byref(d), 0, ctypes.byref(h))
    assert st == 1  # CMLB_E_VALIDATION, raised as ValidationError
    from paper_2301_13441_b200.errors import ValidationError
    with pytest.raises(ValidationError):
        N.check(st)


# -- numpy pairwise-sum replay ---------------------------------------------------

def _replay(codes, vals):
    """Python replay of the kernel's accumulate() on float64 values."""
    r = [0.0] * 8
    res = 0.0
    st = []
    fold = lambda: ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    for t, (c, v) in enumerate(zip(codes, vals)):
        c = int(c)
        if c & 4:
            res = fold()
        op = c & 3
        if op == 0:
            r[t % 8] = v
        elif op == 1:
            r[t % 8] += v
        elif op == 2:
            res = 0.0 + v
        else:
            res += v
        if c & 8:
            res = fold()
        if c & 16:
            st.append(res)
            for _ in range(c >> 8):
                hi = st.pop()
                lo = st.pop()
                st.append(lo + hi)
    assert len(st) == 1
    return 0.0 + st[0]


@pytest.mark.parametrize("T", [1, 2, 7, 8, 9, 15, 16, 17, 127, 128, 129, 255, 256, 300, 500, 1000, 1023,
                               2049, 5000])
def test_pairwise_schedule_reproduces_numpy(lib, T):
    codes = (ctypes.c_uint32 * T)()
    depth = lib.cmlb_debug_pairwise_schedule(T, codes)
    assert depth <= 10
    rng = np.random.default_rng(T)
    for _ in range(5):
        e = rng.integers(-40, 40, size=T).astype(float)
        a = (rng.standard_normal(T) * 2.0 ** e).astype(np.float32).astype(np.float64)
        want = a.reshape(1, T, 1).sum(axis=1)[0, 0]  # the reference reduce layout
        assert _replay(list(codes), list(a)) == want
