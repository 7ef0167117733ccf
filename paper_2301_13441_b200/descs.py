"""Descriptor builders for the C ABI (``include/cmlb.h``), numpy + ctypes only.

No torch here: a reference-side binding builds the
same ``cmlb_forest_desc`` from a lowered plan without pulling in PyTorch.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .dtypes import OUT_CODE
from .lower import ForestSpec


def compact_features(spec: ForestSpec, feature: np.ndarray):
    """Rank / stage only the features the trees test.

    A one-hot-widened input (config 5: 184 model columns, 28 tested) would
    otherwise make every kernel variant stage and rank 156 dead columns per
    row.  The used columns become the forest's features through a prologue
    (a COPY gather of the raw column, or the subset of the fused
    preprocessing ops).  Not with a dense selector: there a non-finite value
    in ANY column poisons the row.  Returns (n_features,
    prologue ops or None, n_inputs)."""
    from .fuse import identity_ops
    F = spec.n_features
    if spec.dense_selector or feature.size == 0:
        return F, spec.prologue, spec.n_inputs
    used = np.unique(feature)
    if used.size == F or (spec.prologue is None and used.size > 0.75 * F):
        return F, spec.prologue, spec.n_inputs
    base = spec.prologue if spec.prologue is not None else identity_ops(F)
    n_in = spec.n_inputs if spec.prologue is not None else F
    return int(used.size), np.ascontiguousarray(base[used]), n_in


def forest_desc(spec: ForestSpec, variant: int = N.FOREST_AUTO):
    """cmlb_forest_desc for a lowered forest; returns (desc, buffers to keep
    alive until the C call that reads it returns)."""
    trees = spec.trees
    T = len(trees)
    node_off = np.zeros(T + 1, np.int64)
    leaf_off = np.zeros(T + 1, np.int64)
    for i, t in enumerate(trees):
        node_off[i + 1] = node_off[i] + t.n_internal
        leaf_off[i + 1] = leaf_off[i] + t.n_leaves
    cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs).astype(dt)) if xs else np.zeros(0, dt)
    feature = cat([t.feature for t in trees], np.int32)
    threshold = cat([t.threshold for t in trees], np.float32)
    left = cat([t.left for t in trees], np.int32)
    right = cat([t.right for t in trees], np.int32)
    payload = np.ascontiguousarray(np.concatenate([t.payload for t in trees]).astype(np.float32))
    classes = np.ascontiguousarray(np.asarray(spec.classes, np.float64))
    n_features, prologue, n_inputs = compact_features(spec, feature)
    if prologue is not spec.prologue:
        feature = np.ascontiguousarray(np.searchsorted(np.unique(feature), feature).astype(np.int32))
    keep = [node_off, leaf_off, feature, threshold, left, right, payload, classes]
    d = N.ForestDesc()
    d.n_trees, d.n_features, d.n_outputs = T, n_features, spec.n_outputs
    d.node_offset = N.ptr(node_off, N.c_i64)
    d.leaf_offset = N.ptr(leaf_off, N.c_i64)
    d.feature = N.ptr(feature, N.c_i32)
    d.threshold = N.ptr(threshold, N.c_f32)
    d.left = N.ptr(left, N.c_i32)
    d.right = N.ptr(right, N.c_i32)
    d.payload = N.ptr(payload, N.c_f32)
    d.aggregation, d.tail = spec.aggregation, spec.tail
    d.learning_rate, d.base_score = spec.learning_rate, spec.base_score
    d.classes = N.ptr(classes, N.c_f64)
    d.n_classes = len(spec.classes)
    d.out_dtype = OUT_CODE[spec.out_dtype]
    d.dense_selector = int(spec.dense_selector)
    d.variant = variant
    d.n_trees_total = int(spec.n_trees_total)
    if prologue is not None:
        pro = np.ascontiguousarray(prologue)
        keep.append(pro)
        d.prologue, d.n_inputs = pro.ctypes.data, int(n_inputs)
    return d, keep
