"""Canonical tree form shared by both lowering routes.

The reference numbers a tree's internal nodes in level order and its leaves in
in-order (``pkg/src/mlower/convert.py:110-135``); the leaf index a tree
reports is the in-order position.  :class:`CanonTree` stores a
tree in exactly that numbering, with child links expressed in it:

    left[j], right[j] >= 0   -> internal node (level-order index)
    left[j], right[j] <  0   -> leaf number ``-1 - ref`` (in-order index)

Two builders produce it:

* :func:`canon_from_arrays` walks a model's node arrays (the ``compile_model``
  route, no dense matrices at all);
* :func:`canon_from_encoding` inverts the reference's tensor encoding
  ``(W1, W2, W3, leaf_table)`` found in a ``KernelPlan`` (the ``execute``
  route).  ``W3[j, l] == 0`` iff leaf ``l`` lies in the left subtree of
  internal node ``j`` (``convert.py:150-174``); left subtrees are contiguous
  in-order leaf ranges, so a breadth-first walk over leaf ranges recovers the
  tree, and the full matrix is then re-derived and compared so that a plan that
  is not a tree encoding is rejected instead of mis-lowered.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

import numpy as np

from .errors import UnresolvedKernel
from .models import TreeArrays


@dataclass(frozen=True, eq=False)
class CanonTree:
    feature: np.ndarray     # int32[I]   level order
    threshold: np.ndarray   # float32[I] level order
    left: np.ndarray        # int32[I]   child refs (see module doc)
    right: np.ndarray       # int32[I]
    payload: np.ndarray     # float64[L, C] in-order leaf rows

    @property
    def n_internal(self) -> int:
        return int(self.feature.shape[0])

    @property
    def n_leaves(self) -> int:
        return int(self.payload.shape[0])

    def depth(self) -> int:
        """Edges on the longest root-to-leaf path (0 for a single leaf)."""
        if self.n_internal == 0:
            return 0
        d = np.zeros(self.n_internal, dtype=np.int64)
        best = 1
        for j in range(self.n_internal):  # level order: parents come first
            for c in (self.left[j], self.right[j]):
                if c >= 0:
                    d[c] = d[j] + 1
                else:
                    best = max(best, int(d[j]) + 1)
        return best

    def same_as(self, other: "CanonTree") -> bool:
        return (np.array_equal(self.feature, other.feature)
                and np.array_equal(self.threshold.view(np.uint32), other.threshold.view(np.uint32))
                and np.array_equal(self.left, other.left)
                and np.array_equal(self.right, other.right)
                and np.array_equal(self.payload, other.payload))


def canon_from_arrays(a: TreeArrays, payload_rows: np.ndarray | None = None) -> CanonTree:
    """Renumber a node-array tree; ``payload_rows`` overrides leaf ``value`` rows
    (indexed by original node id), used for the classifier "prediction" payload."""
    internal_ids: list[int] = []
    queue = deque([0])
    while queue:  # breadth-first over internal nodes only
        i = queue.popleft()
        if not a.is_leaf[i]:
            internal_ids.append(i)
            queue.append(int(a.left[i]))
            queue.append(int(a.right[i]))
    leaf_ids: list[int] = []
    stack = [0]
    while stack:  # in-order == pre-order restricted to leaves for full binary trees
        i = stack.pop()
        if a.is_leaf[i]:
            leaf_ids.append(i)
        else:
            stack.append(int(a.right[i]))
            stack.append(int(a.left[i]))
    pos_internal = {nid: j for j, nid in enumerate(internal_ids)}
    pos_leaf = {nid: l for l, nid in enumerate(leaf_ids)}

    def ref(nid: int) -> int:
        return pos_internal[nid] if not a.is_leaf[nid] else -1 - pos_leaf[nid]

    ids = np.asarray(internal_ids, dtype=np.int64)
    left = np.asarray([ref(int(a.left[i])) for i in internal_ids], dtype=np.int32)
    right = np.asarray([ref(int(a.right[i])) for i in internal_ids], dtype=np.int32)
    src = a.value if payload_rows is None else payload_rows
    payload = np.asarray(src, dtype=np.float64)[np.asarray(leaf_ids, dtype=np.int64)]
    return CanonTree(
        feature=a.feature[ids].astype(np.int32) if len(ids) else np.zeros(0, np.int32),
        threshold=a.threshold[ids].astype(np.float32) if len(ids) else np.zeros(0, np.float32),
        left=left.reshape(-1), right=right.reshape(-1),
        payload=payload.reshape(len(leaf_ids), -1),
    )


def left_leaf_ranges(t: CanonTree):
    """Per internal node: (lo, mid, hi) in-order leaf range and its left part."""
    I = t.n_internal
    lo = np.zeros(I, np.int64)
    mid = np.zeros(I, np.int64)
    hi = np.zeros(I, np.int64)
    size = {}

    def leaves_under(ref: int) -> int:
        if ref < 0:
            return 1
        return size[ref]

    for j in range(I - 1, -1, -1):  # children have larger level-order ids
        size[j] = leaves_under(int(t.left[j])) + leaves_under(int(t.right[j]))
    if I:
        lo[0], hi[0] = 0, t.n_leaves
    for j in range(I):
        mid[j] = lo[j] + leaves_under(int(t.left[j]))
        for c, a, b in ((int(t.left[j]), lo[j], mid[j]), (int(t.right[j]), mid[j], hi[j])):
            if c >= 0:
                lo[c], hi[c] = a, b
    return lo, mid, hi


def routes_matrix(t: CanonTree) -> np.ndarray:
    """The reference W3 (I x L, uint8) re-derived from the canonical tree."""
    lo, mid, _ = left_leaf_ranges(t)
    w3 = np.ones((t.n_internal, t.n_leaves), dtype=np.uint8)
    for j in range(t.n_internal):
        w3[j, lo[j]:mid[j]] = 0
    return w3


def canon_from_encoding(w1: np.ndarray, w2: np.ndarray, w3: np.ndarray,
                        table: np.ndarray) -> CanonTree:
    """Invert the reference tree encoding (see module doc); raises
    UnresolvedKernel when the matrices are not a tree encoding."""
    w1 = np.asarray(w1)
    w3 = np.asarray(w3)
    I, L = w3.shape
    if w1.shape[1] != I or np.asarray(w2).reshape(-1).shape[0] != I or table.shape[0] != L or L != I + 1:
        raise UnresolvedKernel(f"tree encoding shapes disagree: W1 {w1.shape}, W3 {w3.shape}, "
                               f"table {table.shape}")
    ones = (w1 != 0)
    if not (ones.sum(axis=0) == 1).all() or not np.all(w1[ones] == 1):
        raise UnresolvedKernel("selector is not one-hot per internal node")
    feature = ones.argmax(axis=0).astype(np.int32)
    left = np.zeros(I, np.int32)
    right = np.zeros(I, np.int32)
    # breadth-first over leaf ranges: the k-th range with >= 2 leaves belongs to
    # the k-th internal node in level order
    ranges = deque([(0, L, None, None)])  # (lo, hi, parent, side)
    nxt = 0
    zero = (w3 == 0)
    while ranges:
        lo, hi, parent, side = ranges.popleft()
        if hi - lo == 1:
            ref = -1 - lo
        else:
            if nxt >= I:
                raise UnresolvedKernel("routes matrix has too few internal nodes")
            j = nxt
            nxt += 1
            row = zero[j]
            mid = lo + int(np.argmin(row[lo:hi])) if not row[lo:hi].all() else hi
            if mid <= lo or mid >= hi:
                raise UnresolvedKernel(f"internal node {j}: left leaf range is not a proper prefix")
            ranges.append((lo, mid, j, 0))
            ranges.append((mid, hi, j, 1))
            ref = j
        if parent is not None:
            (left if side == 0 else right)[parent] = ref
    if nxt != I:
        raise UnresolvedKernel("routes matrix has unused internal nodes")
    t = CanonTree(feature, np.asarray(w2, dtype=np.float32).reshape(-1), left, right,
                  np.asarray(table, dtype=np.float64).reshape(L, -1))
    if not np.array_equal(routes_matrix(t), (w3 != 0).astype(np.uint8)):
        raise UnresolvedKernel("routes matrix is not the encoding of a binary tree")
    return t


def single_leaf(row) -> CanonTree:
    """A tree with no internal node (``broadcast_const``, ``convert.py:194-196``)."""
    return CanonTree(np.zeros(0, np.int32), np.zeros(0, np.float32), np.zeros(0, np.int32),
                     np.zeros(0, np.int32), np.asarray(row, dtype=np.float64).reshape(1, -1))
