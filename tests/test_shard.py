"""Multi-GPU partitioning logic on CPU: row shards, pairwise-exact tree shards,
and the partial exchange over a real world_size-2 gloo process group."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_13441_b200 import shard


def test_row_ranges_partition_exactly():
    for n in (0, 1, 7, 10_000_000, 10_000_001):
        for world in (1, 2, 3, 4, 8):
            rs = [shard.row_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("T", [257, 500, 1000, 1023, 4096, 5003])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_tree_shards_reproduce_numpy_pairwise_bitwise(T, world):
    rng = np.random.default_rng(T * 31 + world)
    try:
        ranges, merges = shard.pairwise_tree_shards(T, world)
    except ValueError:
        assert T < 129 * world  # not enough splittable recursion nodes
        return
    assert len(ranges) == world and ranges[0][0] == 0 and ranges[-1][1] == T
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    for _ in range(4):
        e = rng.integers(-40, 40, size=T).astype(float)
        a = (rng.standard_normal(T) * 2.0 ** e).astype(np.float32).astype(np.float64)
        want = a.reshape(1, T, 1).sum(axis=1)[0, 0]  # the reference reduce layout
        partials = [np.array([shard.numpy_pairwise(a[lo:hi])]) for lo, hi in ranges]
        got = 0.0 + shard.combine(partials, merges)[0]
        assert got == want


def test_small_ensembles_refuse_tree_sharding():
    with pytest.raises(ValueError):
        shard.pairwise_tree_shards(100, 2)


def test_reduce_steps_follow_the_merge_tree():
    for T, world in ((1000, 2), (1000, 3), (1000, 8), (5003, 8)):
        _, merges = shard.pairwise_tree_shards(T, world)
        sends = {}
        for r in range(world):
            steps = shard.reduce_steps(merges, r)
            kinds = [k for k, _ in steps]
            # receives first, at most one send, and the send is the rank's last step
            assert "send" not in kinds[:-1]
            if r == 0:
                assert "send" not in kinds
            else:
                assert kinds[-1] == "send"
                sends[r] = steps[-1][1]
        # every non-root rank's partial reaches the root along a chain of sends
        for r in range(1, world):
            seen, cur = set(), r
            while cur != 0:
                assert cur not in seen
                seen.add(cur)
                cur = sends[cur]


def _worker(rank, world, port, T, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    vals = (rng.standard_normal((n, T)) * 2.0 ** rng.integers(-30, 30, size=(n, T))).astype(np.float32)
    vals = vals.astype(np.float64)
    ranges, merges = shard.pairwise_tree_shards(T, world)
    lo, hi = ranges[rank]
    part = torch.tensor([shard.numpy_pairwise(vals[i, lo:hi]) for i in range(n)], dtype=torch.float64)

    def recv(peer):
        buf = torch.empty_like(part)
        dist.recv(buf, peer)
        return buf

    def add(dst, src):
        dst.copy_(torch.from_numpy(dst.numpy() + src.numpy()))

    root = shard.tree_reduce(part, merges, rank, lambda t, peer: dist.send(t, peer), recv, add)
    if rank == 0:
        assert root
        got = 0.0 + part.numpy()
        want = vals.reshape(n, T, 1).sum(axis=1)[:, 0]
        q.put(bool(np.array_equal(got, want)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_tree_shard_reduce_gloo(world):
    """The pairwise tree reduce over real point-to-point sends (world 2 and 4)
    reproduces numpy's (N, T, 1) reduction bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + 7 * world
    procs = [ctx.Process(target=_worker, args=(r, world, port, 1000, 64, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


def test_tree_sharding_refuses_vector_ensembles():
    """C >= 2 forests are summed tree after tree by numpy: no exact tree cut,
    so TreeShardedForest refuses them (they shard by rows)."""
    import bench
    from paper_2301_13441_b200 import lower
    model, _, _ = bench.load_model()
    spec = lower.lower_model(model).stages[0]
    assert spec.n_outputs == 2
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(28500 + os.getpid() % 1000)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        with pytest.raises(ValueError, match="scalar ensemble"):
            shard.TreeShardedForest(spec)
    finally:
        dist.destroy_process_group()
