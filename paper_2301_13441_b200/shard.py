"""Multi-GPU partitioning of the forest path (one process per GPU).

Row sharding (random forests, the north star; any model): every rank holds a
replica of the program and processes its own rows -- no data-path collective
(``row_range``).

Tree sharding (large gradient-boosted ensembles): each rank walks
a contiguous range of trees for all rows and emits raw float64 partial sums
(``cmlb_forest_partial``); the partials are exchanged with one NCCL
all-gather and combined, then the tail runs on the combined sum
(``cmlb_forest_finish``).

Exactness of the combine.  The reference reduces the (N, T, 1) stack with
numpy's pairwise summation (``kernels.py:185-190`` -> ``pairwise_sum``): the
tree axis is split recursively at n/2 rounded down to a multiple of 8 until
blocks have <= 128 elements.  :func:`pairwise_tree_shards` cuts that very
recursion tree into G nodes, so every shard's partial is exactly numpy's
value for that node and :func:`merge_plan` combines them in the recursion's
own order -- the tree-sharded result is bit-identical to the single-GPU one.
(For C >= 2 ensembles numpy sums sequentially, which cannot be split exactly;
those are row-sharded.)
"""

from __future__ import annotations

import numpy as np


def row_range(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row shard of ``rank`` (weak or strong scaling)."""
    base, extra = divmod(n_rows, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _split(lo: int, n: int):
    n2 = n // 2
    n2 -= n2 % 8
    return (lo, n2), (lo + n2, n - n2)


def pairwise_tree_shards(n_trees: int, world: int):
    """Cut numpy's pairwise recursion over ``n_trees`` into ``world`` nodes.

    Returns ``(ranges, merges)``: ranges[i] = (lo, hi) tree range of shard i
    (left to right), merges = ordered (a, b) pairs meaning p[a] = p[a] + p[b].
    Raises ValueError when the recursion has fewer than ``world`` splittable
    nodes (small ensembles: shard by rows instead).
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    # tree of nodes: node = [lo, n, children]
    root = [0, n_trees, None]
    leaves = [root]
    while len(leaves) < world:
        cand = [nd for nd in leaves if nd[1] > 128]
        if not cand:
            raise ValueError(f"{n_trees} trees cannot be cut into {world} pairwise shards")
        big = max(cand, key=lambda nd: nd[1])
        (l0, ln), (r0, rn) = _split(big[0], big[1])
        left, right = [l0, ln, None], [r0, rn, None]
        big[2] = (left, right)
        i = leaves.index(big)
        leaves[i:i + 1] = [left, right]
    ranges = [(nd[0], nd[0] + nd[1]) for nd in leaves]
    index = {id(nd): i for i, nd in enumerate(leaves)}
    merges: list[tuple[int, int]] = []

    def first_leaf(nd):
        while nd[2] is not None:
            nd = nd[2][0]
        return index[id(nd)]

    def post(nd):
        if nd[2] is None:
            return
        post(nd[2][0])
        post(nd[2][1])
        merges.append((first_leaf(nd[2][0]), first_leaf(nd[2][1])))

    post(root)
    return ranges, merges


def numpy_pairwise(a: np.ndarray) -> float:
    """numpy's own pairwise_sum for a contiguous float64 vector (no +0.0)."""
    n = a.shape[0]
    if n < 8:
        res = 0.0
        for v in a:
            res += float(v)
        return res
    if n <= 128:
        r = [float(v) for v in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    (l0, ln), (r0, rn) = _split(0, n)
    return numpy_pairwise(a[:ln]) + numpy_pairwise(a[ln:])


def combine(partials, merges) -> np.ndarray:
    """Host reference of the device combine (tests): apply merges in order."""
    p = [np.array(x, dtype=np.float64, copy=True) for x in partials]
    for a, b in merges:
        p[a] = p[a] + p[b]
    return p[0]


class TreeShardedForest:
    """One rank's part of a tree-sharded forest program (torch.distributed).

    ``spec`` is the whole-forest ForestSpec.  Every rank builds a program over
    its tree range (for partials) plus the whole-forest program on the root
    (for the tail); ``predict`` gathers partials with NCCL all-gather and the
    root combines in pairwise order and applies the tail on the GPU.
    """

    def __init__(self, spec, group=None, device=None):
        import torch
        import torch.distributed as dist
        from dataclasses import replace

        from .lower import ProgramSpec
        from .runtime import DeviceProgram

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranges, self.merges = pairwise_tree_shards(len(spec.trees), self.world)
        lo, hi = self.ranges[self.rank]
        shard = replace(spec, trees=spec.trees[lo:hi])
        self.device = torch.cuda.current_device() if device is None else device
        self.local = DeviceProgram(ProgramSpec([shard], spec.n_features), self.device)
        self.full = DeviceProgram(ProgramSpec([spec], spec.n_features), self.device) if self.rank == 0 else None
        self.C = spec.n_outputs
        self.out_cols = spec.out_cols
        self.out_dtype = spec.out_dtype

    def predict(self, x):
        """x: this rank's copy of all rows (CUDA). Returns y on rank 0, None elsewhere."""
        import ctypes

        import torch

        from . import _native as N
        from .runtime import TORCH_DTYPE

        n = int(x.shape[0])
        part = torch.empty((n, self.C), dtype=torch.float64, device=x.device)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        if n:
            self.local.forest().partial(x, part, n, int(x.stride(0)), stream)
        gathered = torch.empty((self.world, n, self.C), dtype=torch.float64, device=x.device)
        self.dist.all_gather_into_tensor(gathered, part, group=self.group)
        if self.rank != 0:
            return None
        y = torch.empty((n, self.out_cols), dtype=TORCH_DTYPE[self.out_dtype], device=x.device)
        m = np.asarray(self.merges, dtype=np.int32).reshape(-1)
        mp = m.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        N.check(N.lib().cmlb_forest_finish(self.full.forest().handle, gathered.data_ptr(), self.world, mp,
                                           len(self.merges), n, y.data_ptr(), stream))
        return y
