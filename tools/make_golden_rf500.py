"""Golden vectors for the NORTH-STAR model, produced by the reference itself
(this container only; ~3 min of ``mlower.execute``).

    python tools/make_golden_rf500.py      # writes tests/golden/rf500_ref.npz

The bench model (``bench_assets/rf500_d8.npz``: sklearn RandomForestClassifier
500 trees, max_depth 8, on make_classification 200k x 28) is written out in
the reference's model-JSON schema (``pkg/exporter/export.py:56-116``) and
compiled by ``mlower.compile_model`` with the default profile.  Rows:

* 2,000 rows drawn like the bench input (``randn * sigma + mu``, seed 101);
* 1,000 reference boundary rows (``helpers.boundary_inputs``: zeros with one
  feature exactly at one of the model's thresholds, ``cli.py:61-68``), for a
  random sample of the 123,934 (feature, threshold) pairs;
* 1,000 bench-like rows with one feature set exactly to a threshold of that
  feature (ties deep inside the trees, not just at zero rows);
* 48 rows with NaN / +-inf / -0 / +-FLT_MAX / denormal features.

Recorded: the reference ``execute`` output (class labels, BOOL dtype) and the
per-tree in-order leaf index of every row (the plan's per-tree
``argmax`` slots).  The plan is executed ONCE with the reference's own
``_run_invocation`` (``runtime.py:147-195``) keeping every slot, instead of
once per tree with ``output_slot`` replaced (500 x slower, same values).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = ["/root/reference/pkg/src", "/root/reference/pkg/tests", ROOT]
sys.dont_write_bytecode = True

OUT = os.path.join(ROOT, "tests", "golden", "rf500_ref.npz")
SPECIAL = np.float32([np.nan, np.inf, -np.inf, -0.0, 3.4028235e38, -3.4028235e38, 1e-45, 1.17549435e-38])


def reference_json(z) -> str:
    offs = z["offsets"]
    trees = []
    for t in range(len(offs) - 1):
        lo, hi = int(offs[t]), int(offs[t + 1])
        nodes = []
        for i in range(lo, hi):
            if z["is_leaf"][i]:
                nodes.append({"leaf": [float(v) for v in z["value"][i]]})
            else:
                nodes.append({"feature": int(z["feature"][i]), "threshold": float(z["threshold"][i]),
                              "left": int(z["left"][i]), "right": int(z["right"][i])})
        trees.append({"nodes": nodes})
    from mlower.models import FORMAT_VERSION
    return json.dumps({"format_version": FORMAT_VERSION, "model_type": "random_forest_classifier", "n_features": int(z["n_features"]),
                       "trees": trees, "aggregation": "mean_probability",
                       "classes": [float(c) for c in z["classes"]]})


def rows(z, rng):
    mu, sigma = z["mu"], z["sigma"]
    F = int(z["n_features"])
    inner = ~z["is_leaf"]
    pairs = np.stack([z["feature"][inner], z["threshold"][inner].view(np.int32)], axis=1)
    pairs = np.unique(pairs, axis=0)
    bench = (rng.standard_normal((2000, F)) * sigma + mu).astype(np.float32)
    pick = pairs[rng.choice(len(pairs), 1000, replace=False)]
    zeros = np.zeros((1000, F), np.float32)
    zeros[np.arange(1000), pick[:, 0]] = pick[:, 1].view(np.float32)
    pick = pairs[rng.choice(len(pairs), 1000, replace=False)]
    tie = (rng.standard_normal((1000, F)) * sigma + mu).astype(np.float32)
    tie[np.arange(1000), pick[:, 0]] = pick[:, 1].view(np.float32)
    special = (rng.standard_normal((48, F)) * sigma + mu).astype(np.float32)
    for i in range(48):
        cols = rng.choice(F, size=1 + i % 3, replace=False)
        special[i, cols] = rng.choice(SPECIAL, size=len(cols))
    return np.concatenate([bench, zeros, tie, special]).astype(np.float32)


def main() -> None:
    from mlower import compile_model
    from mlower.dtypes import DType
    from mlower.models import parse_model
    from mlower.runtime import _run_invocation
    from mlower.tensor import Tensor

    z = dict(np.load(os.path.join(ROOT, "bench_assets", "rf500_d8.npz")))  # NpzFile re-reads per access
    model = parse_model(reference_json(z))
    compiled = compile_model(model)
    plan = compiled.plan
    x = rows(z, np.random.default_rng(101))
    xt = Tensor.from_dense(x, DType.FLOAT32)
    t0 = time.time()
    slots = [None] * len(plan.slot_shapes)
    slots[plan.input_slot] = xt
    for inv in plan.invocations:
        slots[inv.output] = _run_invocation(inv, [slots[s] for s in inv.inputs], x.shape[0])
    out = slots[plan.output_slot]
    argmax = [inv.output for inv in plan.invocations if inv.kernel == "argmax"]
    assert len(argmax) == len(model.trees) + 1  # per-tree argmax slots + the class argmax
    leaves = np.stack([slots[s].to_numpy() for s in argmax[:-1]], axis=1)
    assert leaves.max() < 256
    np.savez_compressed(OUT, x=x, want=out.to_numpy().astype(np.float64).ravel(),
                        want_dtype=np.array(out.dtype.value), leaves=leaves.astype(np.uint8),
                        rows_note=np.array("0:2000 bench-like, 2000:3000 boundary (zeros + one threshold), "
                                           "3000:4000 bench-like with one feature at a threshold, "
                                           "4000:4048 non-finite/extreme"))
    print(f"{OUT}: {x.shape[0]} rows, dtype {out.dtype.value}, {time.time() - t0:.0f} s of mlower execute")


if __name__ == "__main__":
    main()
