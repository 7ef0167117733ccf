"""Multi-GPU partitioning of the forest path (one process per GPU).

Row sharding (random forests, the north star; any model): every rank holds a
replica of the program and processes its own rows -- no data-path collective
(``row_range``; single-process multi-device form: ``api.predict(...,
devices=[...])``).

Tree sharding (large gradient-boosted ensembles): each rank walks
a contiguous range of trees for all rows and emits raw float64 partial sums
(``cmlb_forest_partial``); the partials are combined by ONE reduce -- a
pairwise tree reduce over NCCL point-to-point (NVLink), each step
``dst += src`` on the receiving GPU (``cmlb_forest_merge``) -- and the root
applies the ensemble tail (``cmlb_forest_finish``).

Exactness of the reduce.  The reference reduces the (N, T, 1) stack with
numpy's pairwise summation (``kernels.py:185-190`` -> ``pairwise_sum``): the
tree axis is split recursively at n/2 rounded down to a multiple of 8 until
blocks have <= 128 elements.  :func:`pairwise_tree_shards` cuts that very
recursion tree into G nodes, so every shard's partial is exactly numpy's
value for that node, and the reduce follows the recursion's own merge tree:
every step adds two sibling nodes (one float64 IEEE add, commutative, so it
does not matter which GPU performs it).  The tree-sharded result is therefore
bit-identical to the single-GPU one.  A stock ``ncclReduce`` would add the G
partials in the ring's order instead -- for G >= 3 a different rounding
sequence -- which is why the reduce is scheduled here rather than delegated.
For C >= 2 ensembles numpy sums tree after tree, which no cut reproduces:
those are row-sharded (``TreeShardedForest`` raises).

Bytes on the wire: every non-root rank sends its (merged) partial once,
N x 8 bytes (8 MB for config 3's 1M rows); the root receives ceil(log2 G)
of them.  The former all-gather delivered G x N x 8 bytes to every rank.
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


def reduce_steps(merges, rank: int):
    """This rank's part of the pairwise merge tree, in merge order.

    ``("recv", peer)``: receive the peer's partial and add it into ours;
    ``("send", peer)``: send our (complete) partial to the peer, then stop.
    Merges come in post-order, so every partial is complete before it is sent;
    the dependency graph is a tree, so blocking send/recv cannot deadlock."""
    steps = []
    for a, b in merges:
        if a == rank:
            steps.append(("recv", b))
        elif b == rank:
            steps.append(("send", a))
    return steps


def tree_reduce(part, merges, rank: int, send, recv, add):
    """Run the pairwise tree reduce with caller-supplied transport and add.
    Returns True on the rank that ends up holding the total (rank 0)."""
    for kind, peer in reduce_steps(merges, rank):
        if kind == "recv":
            add(part, recv(peer))
        else:
            send(part, peer)
            return False
    return rank == 0


class TreeShardedForest:
    """One rank's part of a tree-sharded forest program (torch.distributed).

    ``spec`` is the whole-forest ForestSpec (scalar ensembles: GBDT, single-
    output forest regressors).  Each rank builds a program over its own tree
    range only (the whole-ensemble tree count rides along for a MEAN tail);
    ``predict`` computes the partial, runs the pairwise tree reduce and the
    root applies the tail.  Transport: NCCL point-to-point on device tensors;
    with a CPU backend (gloo) the partials are staged through host memory.
    """

    def __init__(self, spec, group=None, device=None):
        import torch
        import torch.distributed as dist
        from dataclasses import replace

        from .lower import ProgramSpec
        from .runtime import DeviceProgram

        if spec.n_outputs != 1:
            raise ValueError("tree sharding needs a scalar ensemble: numpy sums a (N, T, C >= 2) stack "
                             "tree after tree, which no shard cut reproduces; shard such models by rows")
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranges, self.merges = pairwise_tree_shards(len(spec.trees), self.world)
        lo, hi = self.ranges[self.rank]
        shard = replace(spec, trees=spec.trees[lo:hi], n_trees_total=len(spec.trees))
        self.device = torch.cuda.current_device() if device is None else device
        self.local = DeviceProgram(ProgramSpec([shard], spec.in_cols), self.device)
        self.out_cols = spec.out_cols
        self.out_dtype = spec.out_dtype
        self.host_staged = dist.get_backend(group) != "nccl"

    def _global(self, peer: int) -> int:
        return peer if self.group is None else self.dist.get_global_rank(self.group, peer)

    def predict(self, x):
        """x: this rank's copy of all rows (CUDA). Returns y on rank 0, None elsewhere."""
        import torch

        from .runtime import TORCH_DTYPE

        n = int(x.shape[0])
        fo = self.local.forest()
        stream = torch.cuda.current_stream(x.device)
        sh = stream.cuda_stream
        part = torch.empty((n, 1), dtype=torch.float64, device=x.device)
        if n:
            self.local.check_input(x)
            fo.partial(x, part, n, int(x.stride(0)), sh)

        def send(t, peer):
            if self.host_staged:
                t = t.cpu()
            self.dist.send(t, self._global(peer), group=self.group)

        def recv(peer):
            buf = torch.empty((n, 1), dtype=torch.float64, device="cpu" if self.host_staged else x.device)
            self.dist.recv(buf, self._global(peer), group=self.group)
            return buf.to(x.device, non_blocking=False) if self.host_staged else buf

        def add(dst, src):
            fo.merge(dst, src, n, sh)

        if not tree_reduce(part, self.merges, self.rank, send, recv, add):
            return None
        y = torch.empty((n, self.out_cols), dtype=TORCH_DTYPE[self.out_dtype], device=x.device)
        fo.finish(part, 1, [], n, y, sh)
        return y
