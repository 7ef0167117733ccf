"""Multi-GPU paths on one B200: tree sharding (config 3: GBR 1000 x d10, the
pairwise tree reduce + tail) and row sharding (bit-transparent).

The box has one GPU, so the multi-rank test runs two processes on cuda:0 over
gloo with host-staged partials: the same TreeShardedForest code as the NCCL
path, only the transport of the (N, 1) float64 partials differs.
"""

import os
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import fast

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.gpu


def _gbr(T=1000, depth=10):
    from bench_configs import perfect_gbdt
    return perfect_gbdt(T=T, depth=depth)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_tree_shard_programs_reduce_bit_exact(world):
    """Shard programs (own tree range, whole-ensemble tail) -> partials ->
    pairwise tree reduce with cmlb_forest_merge -> finish on one partial ==
    the single program == the C oracle."""
    from dataclasses import replace

    from paper_2301_13441_b200 import lower, shard
    from paper_2301_13441_b200.lower import ProgramSpec
    from paper_2301_13441_b200.runtime import DeviceProgram
    m = _gbr()
    spec = lower.lower_model(m).stages[0]
    ranges, merges = shard.pairwise_tree_shards(len(spec.trees), world)
    x = torch.randn((50_000, 90), generator=torch.Generator(device="cuda").manual_seed(world), device="cuda")
    n = x.shape[0]
    sh = torch.cuda.current_stream().cuda_stream
    progs, parts = [], []
    for lo, hi in ranges:
        p = DeviceProgram(ProgramSpec([replace(spec, trees=spec.trees[lo:hi], n_trees_total=len(spec.trees))], 90), 0)
        part = torch.empty((n, 1), dtype=torch.float64, device="cuda")
        p.forest().partial(x, part, n, 90, sh)
        progs.append(p)
        parts.append(part)
    for a, b in merges:  # what the ranks do, one merge at a time
        progs[a].forest().merge(parts[a], parts[b], n, sh)
    y = torch.empty((n, 1), dtype=torch.float32, device="cuda")
    progs[0].forest().finish(parts[0], 1, [], n, y, sh)
    single = DeviceProgram(ProgramSpec([spec], 90), 0).run(x)
    assert torch.equal(y, single)
    want, _ = fast.forest_predict(fast.PackedForest(m), x.cpu().numpy())
    assert np.array_equal(y.cpu().numpy().astype(np.float64), want)


def test_tree_shard_mean_tail_uses_whole_ensemble_count():
    """A single-output forest regressor (MEAN over T) sharded by trees divides
    by the whole ensemble's T, not the shard's."""
    from dataclasses import replace

    from paper_2301_13441_b200 import lower, shard
    from paper_2301_13441_b200.lower import ProgramSpec
    from paper_2301_13441_b200.models import ForestModel
    from paper_2301_13441_b200.runtime import DeviceProgram
    g = _gbr(T=600, depth=6)
    m = ForestModel("random_forest_regressor", g.n_features, g.trees, "mean_probability", 1.0, 0.0, None)
    spec = lower.lower_model(m).stages[0]
    ranges, merges = shard.pairwise_tree_shards(len(spec.trees), 4)
    x = torch.randn((20_000, 90), generator=torch.Generator(device="cuda").manual_seed(5), device="cuda")
    n = x.shape[0]
    sh = torch.cuda.current_stream().cuda_stream
    progs, parts = [], []
    for lo, hi in ranges:
        p = DeviceProgram(ProgramSpec([replace(spec, trees=spec.trees[lo:hi], n_trees_total=len(spec.trees))], 90), 0)
        part = torch.empty((n, 1), dtype=torch.float64, device="cuda")
        p.forest().partial(x, part, n, 90, sh)
        progs.append(p)
        parts.append(part)
    for a, b in merges:
        progs[a].forest().merge(parts[a], parts[b], n, sh)
    y = torch.empty((n, 1), dtype=torch.float32, device="cuda")
    progs[0].forest().finish(parts[0], 1, [], n, y, sh)
    want, _ = fast.forest_predict(fast.PackedForest(m), x.cpu().numpy())
    assert np.array_equal(y.cpu().numpy().astype(np.float64), want)


def test_finish_refuses_vector_ensembles():
    from paper_2301_13441_b200 import api
    from paper_2301_13441_b200.errors import UnresolvedKernel
    import bench
    model, _, _ = bench.load_model()
    prog = api.compile_model(model).program(0)  # keep the program alive while its stage is used
    fo = prog.forest()
    part = torch.zeros((4, 2), dtype=torch.float64, device="cuda")
    y = torch.empty((4, 1), dtype=torch.uint8, device="cuda")
    with pytest.raises(UnresolvedKernel):
        fo.finish(part, 1, [], 4, y, torch.cuda.current_stream().cuda_stream)


def _rank(rank, world, port, rows, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2301_13441_b200 import lower
        from paper_2301_13441_b200.shard import TreeShardedForest
        m = _gbr()
        spec = lower.lower_model(m).stages[0]
        tsf = TreeShardedForest(spec, device=0)
        x = torch.randn((rows, 90), generator=torch.Generator(device="cuda").manual_seed(2), device="cuda")
        y = tsf.predict(x)
        torch.cuda.synchronize()
        if rank == 0:
            from paper_2301_13441_b200 import api
            single = api.compile_model(m).program(0).run(x)
            want, _ = fast.forest_predict(fast.PackedForest(m), x.cpu().numpy())
            q.put((bool(torch.equal(y, single)),
                   bool(np.array_equal(y.cpu().numpy().astype(np.float64), want))))
        else:
            assert y is None
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        q.put(("error", rank, repr(e)))
        raise


@pytest.mark.parametrize("world", [2, 3])
def test_tree_sharded_forest_ranks_on_cuda0(world):
    """config 3 (GBR 1000 x d10) tree-sharded over `world` ranks sharing cuda:0:
    TreeShardedForest.predict == single program == C oracle on 100k rows."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 500) + world
    procs = [ctx.Process(target=_rank, args=(r, world, port, 100_000, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    res = q.get(timeout=5)
    assert all(p.exitcode == 0 for p in procs), res
    assert res == (True, True), res


@pytest.mark.parametrize("host", [False, True])
def test_row_sharded_predict_is_bit_transparent(host):
    """api.predict(..., devices=[0, 0, 0]) shards rows (here onto one GPU
    three times) and must equal the unsharded result bit for bit."""
    from paper_2301_13441_b200 import api
    import bench
    model, mu, sigma = bench.load_model()
    compiled = api.compile_model(model)
    rng = np.random.default_rng(4)
    x = (rng.standard_normal((300_001, 28)) * sigma + mu).astype(np.float32)
    if host:
        got = api.predict(compiled, x, devices=[0, 0, 0])
        want = api.predict(compiled, x)
        assert isinstance(got, np.ndarray) and np.array_equal(got, want)
    else:
        xd = torch.from_numpy(x).cuda()
        got = api.predict(compiled, xd, devices=[0, 0, 0])
        assert got.is_cuda and torch.equal(got, api.predict(compiled, xd))


def test_row_sharded_predict_linear_svm_pipeline():
    """Row sharding is model-agnostic (linear / SVC / scalers
    shard rows): LogisticRegression, an SVC and the config-5 pipeline through
    predict(devices=[0, 0]) equal the unsharded result bit for bit."""
    import sys as _sys
    from paper_2301_13441_b200 import api
    from paper_2301_13441_b200.models import LinearModel
    from bench_configs import synthetic_svc
    _sys.path.insert(0, os.path.join(ROOT, "tests"))
    from workloads import config5_pipeline
    rng = np.random.default_rng(9)
    lm = LinearModel("logistic_regression", 96,
                     tuple(tuple(float(v) for v in r) for r in rng.standard_normal((10, 96)).astype(np.float32)),
                     tuple(float(v) for v in rng.standard_normal(10).astype(np.float32)), tuple(float(c) for c in range(10)))
    svc = synthetic_svc(F=64, n_sv=400, C=4, seed=3)
    pipe, xp = config5_pipeline(rows=50_001)
    for model, x in ((lm, rng.standard_normal((70_001, 96)).astype(np.float32)),
                     (svc, rng.standard_normal((20_001, 64)).astype(np.float32)), (pipe, xp)):
        compiled = api.compile_model(model)
        got = api.predict(compiled, x, devices=[0, 0])
        want = api.predict(compiled, x)
        assert np.array_equal(got, want), type(model).__name__


def test_tree_shard_partials_under_skew():
    """Tree-shard partials from SKEW programs (certified order-free sums): a
    single-output regressor built from the RF500 trees' class-1 probabilities
    (certified) -> shard partials -> pairwise merges -> finish == single program
    == the C oracle; the shard programs really run SKEW."""
    from dataclasses import replace

    import bench
    from paper_2301_13441_b200 import lower, shard
    from paper_2301_13441_b200.lower import ProgramSpec
    from paper_2301_13441_b200.models import ForestModel, TreeArrays, TreeModel
    from paper_2301_13441_b200.runtime import DeviceProgram
    rf, mu, sigma = bench.load_model()
    trees = []
    for t in rf.trees:
        a = t.arrays
        v = np.ascontiguousarray(a.value[:, 1:2], np.float32)
        trees.append(TreeModel("decision_tree_regressor", 28, TreeArrays(a.is_leaf, a.feature, a.threshold, a.left,
                                                                          a.right, v), None))
    m = ForestModel("random_forest_regressor", 28, tuple(trees), "mean_probability", 1.0, 0.0, None)
    spec = lower.lower_model(m).stages[0]
    ranges, merges = shard.pairwise_tree_shards(len(spec.trees), 3)
    x = torch.randn((40_000, 28), generator=torch.Generator(device="cuda").manual_seed(8), device="cuda")
    x.mul_(torch.from_numpy(sigma).cuda()).add_(torch.from_numpy(mu).cuda())
    n = x.shape[0]
    sh = torch.cuda.current_stream().cuda_stream
    progs, parts = [], []
    for lo, hi in ranges:
        p = DeviceProgram(ProgramSpec([replace(spec, trees=spec.trees[lo:hi], n_trees_total=len(spec.trees))], 28), 0)
        assert p.forest().info()["variant"] == "skew"
        part = torch.empty((n, 1), dtype=torch.float64, device="cuda")
        p.forest().partial(x, part, n, 28, sh)
        progs.append(p)
        parts.append(part)
    for a_, b_ in merges:
        progs[a_].forest().merge(parts[a_], parts[b_], n, sh)
    y = torch.empty((n, 1), dtype=torch.float32, device="cuda")
    progs[0].forest().finish(parts[0], 1, [], n, y, sh)
    single = DeviceProgram(ProgramSpec([spec], 28), 0)
    assert single.forest().info()["variant"] == "skew"
    assert torch.equal(y, single.run(x))
    want, _ = fast.forest_predict(fast.PackedForest(m), x.cpu().numpy())
    assert np.array_equal(y.cpu().numpy().astype(np.float64), want)
