"""Generate golden vectors by running the REFERENCE itself (this container only).

    python tools/make_golden.py            # writes tests/golden/

Imports ``mlower`` from ``/root/reference/pkg/src`` (read-only; never copied)
and its test helpers from ``/root/reference/pkg/tests`` to build the
reference's own fixture models and random model families, then records, per
case: the canonical model JSON (``serialize_model``), the input rows, the
reference ``execute`` output and its dtype, per-tree in-order leaf indices
(extracted from the plan's per-tree ``argmax`` slots), and for a
few cases the serialized ``KernelPlan`` so the GPU suite can exercise the
``execute(plan, x)`` drop-in route without the reference installed.

Seeds are fixed; ``PYTHONHASHSEED`` does not matter (unlike the reference's
own 19-family sweep, ``test_acceptance.py:113``).
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

sys.path[:0] = [REF_SRC, REF_TESTS]
sys.dont_write_bytecode = True

import helpers  # noqa: E402  (reference test helpers: fixtures + generators)
from mlower import BUILTIN_PROFILES, compile_model, serialize_model  # noqa: E402
from mlower.dtypes import DType  # noqa: E402
from mlower.runtime import execute  # noqa: E402
from mlower.tensor import Tensor  # noqa: E402

SPECIAL = np.float32([np.nan, np.inf, -np.inf, -0.0, 0.0, 3.4028235e38, -3.4028235e38, 1e-45])


def special_rows(rng, n_features: int, n: int = 24) -> np.ndarray:
    rows = rng.uniform(-10, 10, size=(n, n_features)).astype(np.float32)
    for i in range(n):
        k = 1 + (i % 3)  # one, two or three special features per row
        cols = rng.choice(n_features, size=min(k, n_features), replace=False)
        rows[i, cols] = rng.choice(SPECIAL, size=len(cols))
    return rows


def inputs_for(model, rng, n_random: int) -> np.ndarray:
    parts = [helpers.random_inputs(rng, n_random, model.n_features).to_numpy(),
             helpers.boundary_inputs(model).to_numpy(),
             special_rows(rng, model.n_features)]
    return np.concatenate(parts).astype(np.float32)


def _is_tree_chain_argmax(plan):
    """node ids of per-tree argmax invocations, in tree order."""
    return [inv for inv in plan.invocations if inv.kernel == "argmax"]


def tree_reps(model):
    """(base node id, has_argmax) per tree in converter order (convert.py:287-311)."""
    trees = model.trees if hasattr(model, "trees") else (model,)
    out, base = [], 0
    for t in trees:
        if t.internal_count() == 0:
            out.append((base, False))
            base += 1
        else:
            out.append((base, True))
            base += 5
    return out


def leaf_indices(compiled, x_t: Tensor):
    plan = compiled.plan
    slot_of_node = {inv.node_id: inv.output for inv in plan.invocations}
    cols = []
    for base, has in tree_reps(compiled.model):
        if not has:
            cols.append(np.zeros(x_t.shape[0], np.int32))
            continue
        slot = slot_of_node[base + 3]  # matmul, greater, matmul, argmax, gather
        cols.append(execute(dataclasses.replace(plan, output_slot=slot), x_t).to_numpy().astype(np.int32))
    return np.stack(cols, axis=1)


# -- plan serialization (mirrors paper_2301_13441_b200/planio.py) --------------


def _enc_attr(v):
    if isinstance(v, DType):
        return {"__dtype__": v.value}
    if isinstance(v, (list, tuple)):
        return [_enc_attr(e) for e in v]
    return v


def _enc_tensor(t: Tensor):
    d = {"dtype": t.dtype.value, "shape": list(t.shape)}
    if t.is_csr:
        d["csr"] = {"offsets": t.csr.row_offsets.tolist(), "cols": t.csr.col_indices.tolist(),
                    "values": t.csr.values.astype(np.float64).tolist()}
    else:
        d["dense"] = t.dense.astype(np.float64).reshape(-1).tolist()
    return d


def plan_to_json(plan) -> str:
    invs = []
    for inv in plan.invocations:
        invs.append({
            "node_id": inv.node_id, "kernel": inv.kernel, "variant": inv.variant.value,
            "use_sparse": inv.use_sparse,
            "weights": [{"name": b.name, "tensor": _enc_tensor(b.tensor),
                         "cast_to": b.cast_to.value if b.cast_to else None} for b in inv.weights],
            "inputs": list(inv.inputs), "output": inv.output,
            "attrs": [[k, _enc_attr(v)] for k, v in inv.attrs],
        })
    return json.dumps({
        "invocations": invs,
        "slot_shapes": [list(s) for s in plan.slot_shapes],
        "slot_dtypes": [d.value for d in plan.slot_dtypes],
        "input_slot": plan.input_slot, "output_slot": plan.output_slot,
        "n_features": plan.n_features, "input_dtype": plan.input_dtype.value,
    })


# -- sklearn-trained models (scaled down) ----------


def sklearn_models():
    sys.path.insert(0, "/root/reference/pkg/exporter")
    from export import to_model_object  # reference exporter (ingestion only)
    from sklearn.datasets import make_classification, make_regression
    from sklearn.ensemble import GradientBoostingRegressor, RandomForestClassifier
    from sklearn.linear_model import LogisticRegression
    from sklearn.tree import DecisionTreeClassifier
    from sklearn.preprocessing import StandardScaler

    from mlower.models import parse_model

    out = {}
    X, y = make_classification(n_samples=120_000, n_features=28, n_informative=20, random_state=0)
    X = X.astype(np.float32)
    dt = DecisionTreeClassifier(max_depth=6, random_state=0).fit(X[:100_000], y[:100_000])
    out["sk_dt_d6"] = (parse_model(json.dumps(to_model_object(dt))), X[100_000:102_000])
    rf = RandomForestClassifier(n_estimators=24, max_depth=8, random_state=0, n_jobs=-1).fit(X[:20_000], y[:20_000])
    out["sk_rf24_d8"] = (parse_model(json.dumps(to_model_object(rf))), X[100_000:101_500])
    Xr, yr = make_regression(n_samples=4_000, n_features=90, n_informative=40, random_state=0)
    yr = yr / np.abs(yr).max()
    gbr = GradientBoostingRegressor(n_estimators=12, max_depth=6, random_state=0).fit(Xr, yr)
    out["sk_gbr12_d6"] = (parse_model(json.dumps(to_model_object(gbr))),
                          np.random.default_rng(2).standard_normal((800, 90)).astype(np.float32))
    Xl, yl = make_classification(n_samples=3_000, n_features=784, n_informative=50, n_classes=10,
                                 random_state=0)
    lr = LogisticRegression(max_iter=60).fit(Xl, yl)
    out["sk_logreg_784x10"] = (parse_model(json.dumps(to_model_object(lr))),
                               np.random.default_rng(3).standard_normal((300, 784)).astype(np.float32))
    ss = StandardScaler().fit(X[:5000])
    out["sk_standard_scaler"] = (parse_model(json.dumps(to_model_object(ss))), X[:400])
    return out


def main() -> None:
    os.makedirs(os.path.join(OUT, "plans"), exist_ok=True)
    rng = np.random.default_rng(20261017)
    cases = []  # (name, model, x, profile_name, passes, save_plan)
    for name, build in helpers.FIXTURE_MODELS.items():
        m = build()
        x = inputs_for(m, rng, 120)
        cases.append((f"fixture_{name}", m, x, "cpu-avx2", ("re", "dr", "sor"), True))
        cases.append((f"fixture_{name}_plain", m, x, "plain", ("re", "dr", "sor"), False))
        cases.append((f"fixture_{name}_nopass", m, x, "cpu-avx2", (), False))
    from test_acceptance import FAMILIES  # the reference's 19-family table
    for fam_i, (family, make) in enumerate(FAMILIES):
        frng = np.random.default_rng(1000 + fam_i)
        for k in range(4):
            m = make(frng)
            x = inputs_for(m, frng, 150)
            cases.append((f"family_{family}_{k}", m, x, "cpu-avx2", ("re", "dr", "sor"), k == 0))
        m = make(frng)
        cases.append((f"family_{family}_nore", m, inputs_for(m, frng, 100), "cpu-avx2", ("dr", "sor"), False))
    for name, (m, x) in sklearn_models().items():
        x = np.concatenate([x, special_rows(rng, m.n_features, 16)])
        cases.append((name, m, x.astype(np.float32), "cpu-avx2", ("re", "dr", "sor"), name not in ("sk_logreg_784x10", "sk_rf24_d8")))

    index, arrays = [], {}
    for name, m, x, prof, passes, save_plan in cases:
        compiled = compile_model(m, profile=BUILTIN_PROFILES[prof], passes=passes)
        xt = Tensor.from_dense(x, DType.FLOAT32)
        out = execute(compiled.plan, xt)
        entry = {"name": name, "model_type": m.model_type, "profile": prof, "passes": list(passes),
                 "model_json": serialize_model(m), "want_dtype": out.dtype.value,
                 "want_shape": list(out.shape), "has_leaves": False, "plan": None}
        arrays[f"{name}__x"] = x
        arrays[f"{name}__want"] = out.to_numpy().astype(np.float64)
        if hasattr(m, "nodes") or hasattr(m, "trees"):
            arrays[f"{name}__leaves"] = leaf_indices(compiled, xt)
            entry["has_leaves"] = True
        if save_plan:
            entry["plan"] = f"plans/{name}.json"
            with open(os.path.join(OUT, entry["plan"]), "w") as fh:
                fh.write(plan_to_json(compiled.plan))
        index.append(entry)
    with open(os.path.join(OUT, "index.json"), "w") as fh:
        json.dump({"generator": "tools/make_golden.py", "reference": "mlower (pkg/src)",
                   "cases": index}, fh, indent=0)
    np.savez_compressed(os.path.join(OUT, "arrays.npz"), **arrays)
    print(f"wrote {len(index)} cases to {OUT}")


if __name__ == "__main__":
    main()
