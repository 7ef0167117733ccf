"""Config 3 (GBR 1000 x d10, 1M x 90) under each forest variant that fits."""
import json
import os
import sys

import torch

sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__))]
from bench_configs import perfect_gbdt, time_launch  # noqa: E402
from paper_2301_13441_b200 import _native as N, api  # noqa: E402
from paper_2301_13441_b200.errors import UnresolvedKernel  # noqa: E402
from paper_2301_13441_b200.runtime import DeviceProgram  # noqa: E402

m = perfect_gbdt()
spec = api.compile_model(m).spec
x = torch.randn((1_000_000, 90), generator=torch.Generator(device="cuda").manual_seed(2), device="cuda")
ref = None
for name, v in (("ranked", N.FOREST_RANKED), ("perfect", N.FOREST_PERFECT), ("general", N.FOREST_GENERAL)):
    try:
        prog = DeviceProgram(spec, 0, forest_variant=v)
    except UnresolvedKernel as e:
        print(json.dumps({"variant": name, "unresolved": str(e)}))
        continue
    ms = time_launch(lambda: prog.run(x), reps=5)
    y = prog.run(x[:20000])
    ref = y if ref is None else ref
    print(json.dumps({"variant": name, "ms": ms, "M_rows_per_s": 1e3 / ms, "info": prog.forest().info(),
                      "agrees_with_first": bool(torch.equal(y, ref))}), flush=True)
