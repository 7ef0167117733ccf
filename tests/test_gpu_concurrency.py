"""Programs are immutable and reentrant across streams (reference runtime.py:199,
SPEC.md:574): the same program run concurrently on two streams gives the
sequential results bit-for-bit -- forest, certified linear (fixup queue) and
SVM (exact-path queue) all keep their scratch stream-ordered."""

import numpy as np
import pytest
import torch

import golden_cases as gc
from paper_2301_13441_b200 import api

pytestmark = pytest.mark.gpu


def _concurrent(prog, xs):
    want = [prog.run(x).clone() for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in xs]
    outs = [None] * len(xs)
    for _ in range(3):
        for i, (s, x) in enumerate(zip(streams, xs)):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                outs[i] = prog.run(x, stream=s)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        for o, w in zip(outs, want):
            assert torch.equal(o, w)


def test_forest_two_streams():
    case = gc.get("sk_rf24_d8")
    prog = api.compile_model(case.model).program(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    xs = [torch.randn((300_000, 28), generator=g, device="cuda") * 3 for _ in range(2)]
    _concurrent(prog, xs)


def test_linear_certified_two_streams():
    case = gc.get("sk_logreg_784x10")
    prog = api.compile_model(case.model).program(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = [torch.randn((100_000, 784), generator=g, device="cuda") for _ in range(2)]
    _concurrent(prog, xs)


def test_svm_two_streams():
    case = gc.ext_get("svc10_rbf_784")
    compiled = api.compile_model(case.model)
    prog = compiled.program(0)
    g = torch.Generator(device="cuda").manual_seed(2)
    xs = [torch.randn((20_000, 784), generator=g, device="cuda") for _ in range(2)]
    _concurrent(prog, xs)
