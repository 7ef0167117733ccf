import sys, os, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import golden_cases as gc
from oracle import semantics as sem
from paper_2301_13441_b200 import lower, _native as N
from paper_2301_13441_b200.runtime import DeviceProgram
for name in ["fixture_forest", "sk_rf24_d8", "family_gbdt_regressor_0", "sk_gbr12_d6"]:
    case = gc.get(name)
    spec = lower.lower_model(case.model, case.profile, case.passes)
    prog = DeviceProgram(spec, 0, forest_variant=N.FOREST_MMA)
    x = torch.from_numpy(case.x).cuda()
    leaves = torch.full((x.shape[0], len(spec.stages[0].trees)), -7, dtype=torch.int32, device="cuda")
    y = prog.run(x, leaf_out=leaves); torch.cuda.synchronize()
    ok_l = np.array_equal(leaves.cpu().numpy(), case.leaves)
    got = y.cpu().numpy().astype(np.float64)
    ok = np.array_equal(got, case.want) or np.all((got == case.want) | (np.isnan(got) & np.isnan(case.want)))
    print(name, prog.forest().info(), "leaves", ok_l, "out", ok, flush=True)
