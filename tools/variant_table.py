"""Measure every forest variant over (depth, trees) on one B200: the table the
AUTO variant choice is based on (north star: "the variant is picked per
(depth, tree count) from measurement").

    python tools/variant_table.py [--rows N]

Forests: near-perfect random trees, 28 features, 2 classes (RF-shaped), rows
N(0,1).  Each variant is parity-checked against the ranked result (bit-exact)
and timed with CUDA events (median of 5 after 2 warm-ups).  Writes
gpurun_out/variant_table.json.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

from paper_2301_13441_b200 import _native as N, lower  # noqa: E402
from paper_2301_13441_b200.errors import UnresolvedKernel  # noqa: E402
from paper_2301_13441_b200.models import ForestModel, TreeArrays, TreeModel  # noqa: E402

VARIANTS = {"ranked": N.FOREST_RANKED, "perfect": N.FOREST_PERFECT, "general": N.FOREST_GENERAL,
            "mma": N.FOREST_MMA}


def forest(rng, T, depth, F=28, C=2):
    trees = []
    for _ in range(T):
        ni, nl = 2 ** depth - 1, 2 ** depth
        n = ni + nl
        is_leaf = np.zeros(n, bool)
        is_leaf[ni:] = True
        idx = np.arange(ni)
        left = np.full(n, -1, np.int32)
        right = np.full(n, -1, np.int32)
        left[:ni], right[:ni] = 2 * idx + 1, 2 * idx + 2
        feat = np.zeros(n, np.int32)
        feat[:ni] = rng.integers(0, F, ni)
        thr = np.zeros(n, np.float32)
        thr[:ni] = rng.standard_normal(ni).astype(np.float32)
        val = np.zeros((n, C), np.float32)
        p = rng.random((nl, C)).astype(np.float32)
        val[ni:] = p / p.sum(axis=1, keepdims=True)
        trees.append(TreeModel("decision_tree_regressor", F, TreeArrays(is_leaf, feat, thr, left, right, val), None))
    return ForestModel("random_forest_classifier", F, tuple(trees), "mean_probability", 1.0, 0.0,
                       tuple(float(c) for c in range(C)))


def main():
    from paper_2301_13441_b200.runtime import DeviceProgram
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=2_000_000)
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    out = []
    x = torch.randn((args.rows, 28), device="cuda")
    for depth in (2, 4, 6, 8, 10):
        for T in (16, 128, 500):
            m = forest(rng, T, depth)
            spec = lower.lower_model(m)
            ref = None
            row = {"depth": depth, "trees": T, "rows": args.rows}
            for name, v in VARIANTS.items():
                try:
                    prog = DeviceProgram(spec, 0, forest_variant=v)
                except UnresolvedKernel as e:
                    row[name] = None
                    continue
                y = prog.run(x)
                if ref is None:
                    ref = y
                ok = bool(torch.equal(y, ref))
                ts = []
                for i in range(7):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    prog.run(x, out=y)
                    b.record()
                    torch.cuda.synchronize()
                    if i >= 2:
                        ts.append(a.elapsed_time(b))
                ms = statistics.median(ts)
                row[name] = {"ms": ms, "rows_per_s": args.rows / ms * 1e3, "parity": ok}
                prog.close()
            best = max((k for k in VARIANTS if row.get(k)), key=lambda k: row[k]["rows_per_s"])
            row["best"] = best
            print(json.dumps(row), flush=True)
            out.append(row)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "variant_table.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
