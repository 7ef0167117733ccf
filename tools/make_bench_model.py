"""Train the north-star model once and store it compactly (bench_assets/).

    python tools/make_bench_model.py      # ~1 min on 8 cores

SURVEY 8d config 2: RandomForestClassifier(n_estimators=500, max_depth=8,
random_state=0, n_jobs=-1) fit on make_classification(n_samples=200_000,
n_features=28, n_informative=20, n_classes=2, random_state=0), exported with
the reference exporter's rules (``pkg/exporter/export.py:56-116``: float32
thresholds, leaf rows = per-class counts normalised to probabilities, node ids
verbatim).  Stored as concatenated node arrays plus the per-feature training
mean/std used to synthesise 10M x 28 inputs (randn * sigma + mu).
"""

from __future__ import annotations

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "bench_assets", "rf500_d8.npz")


def main() -> None:
    from sklearn.datasets import make_classification
    from sklearn.ensemble import RandomForestClassifier

    X, y = make_classification(n_samples=200_000, n_features=28, n_informative=20, n_classes=2,
                               random_state=0)
    X = X.astype(np.float32)
    rf = RandomForestClassifier(n_estimators=500, max_depth=8, random_state=0, n_jobs=-1).fit(X, y)
    offs = [0]
    parts = {k: [] for k in ("is_leaf", "feature", "threshold", "left", "right", "value")}
    for est in rf.estimators_:
        t = est.tree_
        leaf = t.children_left == -1
        counts = t.value[:, 0, :].astype(np.float64)
        tot = counts.sum(axis=1, keepdims=True)
        prob = np.where(tot > 0, counts / np.where(tot > 0, tot, 1), counts)
        parts["is_leaf"].append(leaf)
        parts["feature"].append(np.where(leaf, 0, t.feature).astype(np.int32))
        parts["threshold"].append(np.where(leaf, 0, t.threshold).astype(np.float32))
        parts["left"].append(np.where(leaf, -1, t.children_left).astype(np.int32))
        parts["right"].append(np.where(leaf, -1, t.children_right).astype(np.int32))
        parts["value"].append(prob.astype(np.float32))
        offs.append(offs[-1] + t.node_count)
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(
        OUT, offsets=np.asarray(offs, np.int64),
        **{k: np.concatenate(v) for k, v in parts.items()},
        classes=rf.classes_.astype(np.float64), n_features=np.int64(28),
        mu=X.mean(axis=0).astype(np.float32), sigma=X.std(axis=0).astype(np.float32))
    print(OUT, os.path.getsize(OUT))


if __name__ == "__main__":
    main()
