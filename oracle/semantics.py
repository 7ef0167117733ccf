"""numpy restatement of ``mlower.runtime.execute`` for every model family.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Each function follows the reference kernel it names and uses the same numpy
reductions, so float summation order and rounding match by construction:

* tree chain (``convert.py:192-204``): the selector matmul + ``greater`` +
  route matmul + first-max ``argmax`` select the traversal leaf with the
  strict ``x > t`` test (``oracle.py:52-56``); the leaf index
  is the in-order position (``convert.py:122-135``).  With a *dense* selector
  (``kernels.py:95-100``, profile ``plain`` / SOR off) ``0 * inf = NaN``
  poisons the row; ``dense_selector=True`` reproduces that.
* ensembles (``convert.py:287-311``): ``np.stack(axis=1)`` then
  ``astype(float64).mean|sum(axis=1)`` then float32 (``kernels.py:180-190``),
  then float32 ``* lr`` and ``+ base`` (``kernels.py:162-166``), sigmoid in
  float64 (``kernels.py:234-235``) rounded to float32 before ``> 0.5``.
* linear (``convert.py:230-252``): ascending-k float64 ``acc += x_k * w_k``
  (``kernels.py:95-100``; CSR skips zero weights, ``kernels.py:115-123``),
  float32 round, float32 ``+ b``; tails as above; softmax (when RE did not
  remove it) in float64 then float32 before ``argmax`` (``kernels.py:227-233``).
* scalers (``convert.py:255-284``): float32 elementwise, ``row_norm`` in
  float64 with the zero-row guard (``kernels.py:245-261``).

Output: ``(values, dtype_name)`` where ``values`` is a float64 array of the
reference output shape and ``dtype_name`` the reference output dtype.
"""

from __future__ import annotations

import numpy as np


# -- model access (works on the reference's models and on ours) ----------------


def node_arrays(tree):
    """(is_leaf, feature, threshold, left, right, value) for either model type."""
    a = getattr(tree, "arrays", None)
    if a is not None:
        return a.is_leaf, a.feature, a.threshold, a.left, a.right, a.value
    nodes = tree.nodes
    n = len(nodes)
    width = next(len(nd.value) for nd in nodes if hasattr(nd, "value"))
    is_leaf = np.zeros(n, bool)
    feat = np.zeros(n, np.int64)
    thr = np.zeros(n, np.float32)
    left = np.zeros(n, np.int64)
    right = np.zeros(n, np.int64)
    val = np.zeros((n, width), np.float32)
    for i, nd in enumerate(nodes):
        if hasattr(nd, "value"):
            is_leaf[i] = True
            val[i] = nd.value
        else:
            feat[i], thr[i], left[i], right[i] = nd.feature, nd.threshold, nd.left, nd.right
    return is_leaf, feat, thr, left, right, val


def inorder_leaf_position(is_leaf, left, right) -> np.ndarray:
    """node id -> in-order leaf position (-1 for internal nodes)."""
    pos = np.full(len(is_leaf), -1, np.int64)
    k = 0
    stack = [0]
    while stack:
        i = stack.pop()
        if is_leaf[i]:
            pos[i] = k
            k += 1
        else:
            stack.append(int(right[i]))
            stack.append(int(left[i]))
    return pos


def poison_dense_selector(x: np.ndarray) -> np.ndarray:
    """Row transform equivalent to the dense selector's 0*inf contamination.

    select_j = sum_k x_k * W1[k, j] (float64, ascending k) is NaN as soon as a
    non-finite x_k meets a zero weight.  One non-finite feature: every other
    node sees NaN, nodes testing that feature see it; two or more: all NaN.
    """
    x = np.array(x, dtype=np.float32, copy=True)
    bad = ~np.isfinite(x)
    nbad = bad.sum(axis=1)
    one = nbad == 1
    x[one[:, None] & ~bad] = np.nan
    x[nbad >= 2] = np.nan
    return x


# -- trees -------------------------------------------------------------------


def tree_leaf_nodes(tree, x: np.ndarray) -> np.ndarray:
    """Node id reached by every row (strict ``x > t`` goes right, NaN left)."""
    is_leaf, feat, thr, left, right, _ = node_arrays(tree)
    n = x.shape[0]
    node = np.zeros(n, np.int64)
    live = np.flatnonzero(~is_leaf[node]) if n else np.zeros(0, np.int64)
    while live.size:
        nd = node[live]
        go_right = x[live, feat[nd]] > thr[nd]
        node[live] = np.where(go_right, right[nd], left[nd])
        live = live[~is_leaf[node[live]]]
    return node


def tree_leaf_index(tree, x: np.ndarray) -> np.ndarray:
    is_leaf, _, _, left, right, _ = node_arrays(tree)
    return inorder_leaf_position(is_leaf, left, right)[tree_leaf_nodes(tree, x)].astype(np.int32)


def smallest_dtype(values) -> str:
    v = np.asarray(values, dtype=np.float64).reshape(-1)
    for name, (lo, hi) in (("bool", (0, 1)), ("int4", (-8, 7)), ("int8", (-128, 127)),
                           ("int16", (-32768, 32767)), ("int32", (-(2**31), 2**31 - 1))):
        if v.size == 0 or (np.all(np.isfinite(v)) and np.all(v == np.floor(v))
                           and v.min() >= lo and v.max() <= hi):
            return {"int4": "int8"}.get(name, name)
    return "float32"


def first_max_label(leaf_value: np.ndarray, classes) -> float:
    # Python max with key (value, -i): largest value, ties to the smallest i
    best = max(range(len(leaf_value)), key=lambda i: (float(leaf_value[i]), -i))
    return float(classes[best])


def sigmoid_f32(z32: np.ndarray) -> np.ndarray:
    x = z32.astype(np.float64)
    e = np.exp(-np.abs(x))
    with np.errstate(invalid="ignore"):
        out = np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))
    return out.astype(np.float32)


def predict_tree(m, x, dense_selector=False):
    xs = poison_dense_selector(x) if dense_selector else x
    is_leaf, _, _, _, _, val = node_arrays(m)
    nodes = tree_leaf_nodes(m, xs)
    if m.classes is not None:
        labels = np.array([first_max_label(val[i], m.classes) if is_leaf[i] else 0.0
                           for i in range(len(is_leaf))])
        table = labels[is_leaf]
        return labels[nodes].reshape(-1, 1), smallest_dtype(table)
    return val[nodes].astype(np.float64), "float32"


def forest_parts(m, x, dense_selector=False):
    xs = poison_dense_selector(x) if dense_selector else x
    parts = []
    for t in m.trees:
        _, _, _, _, _, val = node_arrays(t)
        parts.append(val[tree_leaf_nodes(t, xs)].astype(np.float32))
    return parts


def forest_leaf_indices(m, x, dense_selector=False) -> np.ndarray:
    xs = poison_dense_selector(x) if dense_selector else x
    return np.stack([tree_leaf_index(t, xs) for t in m.trees], axis=1).astype(np.int32)


def predict_forest(m, x, dense_selector=False):
    stacked = np.stack(forest_parts(m, x, dense_selector), axis=1)  # (N, T, C)
    if m.aggregation == "mean_probability":
        mean = stacked.astype(np.float64).mean(axis=1).astype(np.float32)
        if m.classes is None:
            return mean.astype(np.float64), "float32"
        idx = np.argmax(mean, axis=1)
        cls = np.asarray(m.classes, np.float64)
        return cls[idx].reshape(-1, 1), smallest_dtype(cls)
    total = stacked.astype(np.float64).sum(axis=1).astype(np.float32)
    raw = np.add(np.multiply(total, np.float32(m.learning_rate)), np.float32(m.base_score))
    if m.classes is None:
        return raw.astype(np.float64), "float32"
    decide = sigmoid_f32(raw) > np.float32(0.5)
    cls = np.asarray(m.classes, np.float64)
    return cls[decide.reshape(-1).astype(np.int64)].reshape(-1, 1), smallest_dtype(cls)


# -- linear ------------------------------------------------------------------


def linear_logits(m, x, sparse_coef=False) -> np.ndarray:
    w = np.asarray(m.coef, np.float64).T  # (F, C)
    x64 = np.asarray(x, np.float32).astype(np.float64)
    acc = np.zeros((x.shape[0], w.shape[1]), np.float64)
    for k in range(w.shape[0]):
        if sparse_coef:
            cols = np.flatnonzero(w[k] != 0)
            if cols.size:
                acc[:, cols] += x64[:, k:k + 1] * w[k, cols]
        else:
            acc += x64[:, k:k + 1] * w[k:k + 1, :]
    return np.add(acc.astype(np.float32), np.asarray(m.intercept, np.float32))


def predict_linear(m, x, sparse_coef=False, softmax=False):
    z = linear_logits(m, x, sparse_coef)
    if m.classes is None:
        return z.astype(np.float64), "float32"
    cls = np.asarray(m.classes, np.float64)
    if len(m.coef) == 1:
        if m.model_type == "logistic_regression":
            decide = sigmoid_f32(z) > np.float32(0.5)
        else:
            decide = z > np.float32(0.0)
        return cls[decide.reshape(-1).astype(np.int64)].reshape(-1, 1), smallest_dtype(cls)
    if softmax and m.model_type == "logistic_regression":
        s = z.astype(np.float64)
        e = np.exp(s - s.max(axis=1, keepdims=True))
        z = (e / e.sum(axis=1, keepdims=True)).astype(np.float32)
    return cls[np.argmax(z, axis=1)].reshape(-1, 1), smallest_dtype(cls)


# -- scalers -----------------------------------------------------------------


def _vec(m, name):
    return np.asarray(m.vector(name), np.float32)


def predict_scaler(m, x):
    x = np.asarray(x, np.float32)
    kind = m.model_type
    if kind == "binarizer":
        out = np.greater(x, np.float32(m.threshold)).astype(np.float32)
    elif kind == "normalizer":
        x64 = x.astype(np.float64)
        if m.norm == "l1":
            n = np.abs(x64).sum(axis=1)
        elif m.norm == "l2":
            n = np.sqrt((x64 * x64).sum(axis=1))
        else:
            n = np.abs(x64).max(axis=1)
        n = np.where(n == 0.0, 1.0, n).reshape(-1, 1).astype(np.float32)
        with np.errstate(divide="ignore", invalid="ignore"):
            out = np.divide(x, n)
    elif kind == "minmax_scaler":
        out = np.add(np.multiply(x, _vec(m, "scale")), _vec(m, "min"))
    elif kind in ("robust_scaler", "standard_scaler"):
        center = _vec(m, "center" if kind == "robust_scaler" else "mean")
        with np.errstate(divide="ignore", invalid="ignore"):
            out = np.divide(np.subtract(x, center), _vec(m, "scale"))
    elif kind == "maxabs_scaler":
        with np.errstate(divide="ignore", invalid="ignore"):
            out = np.divide(x, _vec(m, "scale"))
    else:
        raise ValueError(kind)
    return out.astype(np.float64), "float32"


# -- dispatch ----------------------------------------------------------------

_TREES = ("decision_tree_classifier", "decision_tree_regressor")
_FORESTS = ("random_forest_classifier", "random_forest_regressor", "gbdt_regressor",
            "gbdt_binary_classifier")
_SCALERS = ("binarizer", "normalizer", "minmax_scaler", "robust_scaler", "standard_scaler",
            "maxabs_scaler")


def predict(model, x, *, dense_selector=None, sparse_coef=None, softmax=False):
    """Reference ``execute`` output for ``compile_model(model)`` (default profile
    unless the flags say otherwise)."""
    x = np.asarray(x, np.float32)
    mt = model.model_type
    if dense_selector is None:  # default profile: SOR makes W1 CSR iff 1/F < 0.3
        dense_selector = not (1.0 / model.n_features < 0.3)
    if mt in _TREES:
        if (~node_arrays(model)[0]).sum() == 0:
            dense_selector = False
        return predict_tree(model, x, dense_selector)
    if mt in _FORESTS:
        return predict_forest(model, x, dense_selector)
    if mt in _SCALERS:
        return predict_scaler(model, x)
    if sparse_coef is None:
        w = np.asarray(model.coef, np.float64)
        sparse_coef = np.count_nonzero(w) / w.size < 0.3
    return predict_linear(model, x, sparse_coef, softmax)

