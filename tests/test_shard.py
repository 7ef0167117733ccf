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
    gathered = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(gathered, part)
    if rank == 0:
        got = 0.0 + shard.combine([g.numpy() for g in gathered], merges)
        want = vals.reshape(n, T, 1).sum(axis=1)[:, 0]
        q.put(bool(np.array_equal(got, want)))
    dist.barrier()
    dist.destroy_process_group()


def test_tree_shard_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 1000, 64, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
