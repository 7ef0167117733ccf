"""GPU parity: the sm_100a path against the reference's golden vectors and the
oracle.  Classes and leaf indices must be bit-exact; float outputs are held to
bit-exactness too (the kernels replay the reference's float64 order), with the
reference's 1e-5 relative rule (helpers.py:336-339) reported on failure.
"""

import numpy as np
import pytest
import torch

import golden_cases as gc
from oracle import fast, semantics as sem

pytestmark = pytest.mark.gpu

cmlb = pytest.importorskip("paper_2301_13441_b200")
from paper_2301_13441_b200 import api, lower  # noqa: E402
from paper_2301_13441_b200 import _native as N  # noqa: E402
from paper_2301_13441_b200.planio import load_plan_file  # noqa: E402
from paper_2301_13441_b200.runtime import DeviceProgram  # noqa: E402
from paper_2301_13441_b200.errors import UnresolvedKernel  # noqa: E402


def _same(got, want):
    return np.array_equal(got, want) or (
        got.shape == want.shape and np.all((got == want) | (np.isnan(got) & np.isnan(want))))


@pytest.mark.parametrize("name", gc.case_names())
def test_compile_model_matches_reference(name):
    case = gc.get(name)
    compiled = api.compile_model(case.model, profile=case.profile, passes=case.passes)
    out = api.predict(compiled, cmlb.Tensor.from_dense(case.x, cmlb.DType.FLOAT32))
    assert out.dtype.value == case.want_dtype
    got = out.to_numpy().astype(np.float64)
    assert gc.agrees(case, got), f"{name}: tolerance rule violated"
    assert _same(got, case.want), f"{name}: not bit-exact (max |d| {np.nanmax(np.abs(got - case.want))})"


@pytest.mark.parametrize("name", [n for n in gc.case_names() if gc.get(n).plan_path])
def test_execute_reference_plan(name):
    case = gc.get(name)
    plan = load_plan_file(case.plan_path)
    got = api.execute(plan, case.x)  # numpy in -> numpy out
    assert _same(got.astype(np.float64), case.want)


@pytest.mark.parametrize("variant", [N.FOREST_PERFECT, N.FOREST_GENERAL, N.FOREST_RANKED, N.FOREST_MMA,
                                     N.FOREST_SKEW])
@pytest.mark.parametrize("name", [n for n in gc.case_names() if gc.get(n).leaves is not None])
def test_leaf_indices_and_variants(name, variant):
    case = gc.get(name)
    spec = lower.lower_model(case.model, case.profile, case.passes)
    st = spec.stages[0]
    layouts = (N.FOREST_PERFECT, N.FOREST_RANKED, N.FOREST_MMA, N.FOREST_SKEW)
    if variant in layouts and (max(t.depth() for t in st.trees) > 11 or max(t.depth() for t in st.trees) == 0):
        pytest.skip("too deep / no internal node for the perfect layout")
    try:
        prog = DeviceProgram(spec, 0, forest_variant=variant)
    except UnresolvedKernel:
        assert variant in layouts
        pytest.skip("perfect/ranked/mma/skew layout does not fit this forest (or its sums are not order-free)")
    x = torch.from_numpy(case.x).cuda()
    leaves = torch.full((x.shape[0], len(st.trees)), -7, dtype=torch.int32, device="cuda")
    y = prog.run(x, leaf_out=leaves)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(leaves.cpu().numpy(), case.leaves)
    got = y.cpu().numpy().astype(np.float64)
    assert _same(got, case.want)
    prog.close()


def test_device_tensor_path_and_zero_rows():
    case = gc.get("sk_rf24_d8")
    compiled = api.compile_model(case.model)
    x = torch.from_numpy(case.x).cuda()
    y = api.predict(compiled, x)
    assert y.is_cuda and y.dtype == torch.uint8  # BOOL classes {0, 1}
    assert _same(y.cpu().numpy().astype(np.float64), case.want)
    empty = api.predict(compiled, x[:0])
    assert tuple(empty.shape) == (0, 1)
    host_empty = api.predict(compiled, np.zeros((0, case.x.shape[1]), np.float32))
    assert host_empty.shape == (0, 1)


def test_batch_invariance_and_determinism():
    case = gc.get("sk_gbr12_d6")
    compiled = api.compile_model(case.model)
    x = torch.from_numpy(case.x).cuda()
    a = api.predict(compiled, x).cpu().numpy()
    b = api.predict(compiled, x).cpu().numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    for i in (0, 7, 511, x.shape[0] - 1):
        single = api.predict(compiled, x[i:i + 1]).cpu().numpy()
        assert np.array_equal(single.view(np.uint32), a[i:i + 1].view(np.uint32))


def test_input_mismatch():
    from paper_2301_13441_b200.errors import InputMismatch
    case = gc.get("fixture_tree_a")
    compiled = api.compile_model(case.model)
    with pytest.raises(InputMismatch):
        api.predict(compiled, np.zeros((2, 3), np.float32))
    with pytest.raises(InputMismatch):
        api.predict(compiled, np.zeros((2, 2), np.int8))


def _synthetic_forest(rng, T, depth, F, C, gbdt=False):
    """Random near-perfect trees as a model object (ours)."""
    from paper_2301_13441_b200.models import ForestModel, TreeArrays, TreeModel
    trees = []
    for _ in range(T):
        nodes = []

        def grow(d):
            i = len(nodes)
            nodes.append(None)
            if d == depth or (d >= 3 and rng.random() < 0.08):
                v = rng.random(C).astype(np.float32) if not gbdt else \
                    (rng.standard_normal(1) * 2.0 ** rng.integers(-30, 10)).astype(np.float32)
                if not gbdt:
                    v = (v / v.sum()).astype(np.float32)
                nodes[i] = ("leaf", v)
            else:
                f = int(rng.integers(F))
                th = np.float32(rng.standard_normal())
                l = grow(d + 1)
                r = grow(d + 1)
                nodes[i] = ("node", f, th, l, r)
            return i

        grow(0)
        n = len(nodes)
        cw = 1 if gbdt else C
        a = TreeArrays(
            is_leaf=np.array([x[0] == "leaf" for x in nodes]),
            feature=np.array([x[1] if x[0] == "node" else 0 for x in nodes], np.int32),
            threshold=np.array([x[2] if x[0] == "node" else 0 for x in nodes], np.float32),
            left=np.array([x[3] if x[0] == "node" else -1 for x in nodes], np.int32),
            right=np.array([x[4] if x[0] == "node" else -1 for x in nodes], np.int32),
            value=np.array([x[1] if x[0] == "leaf" else np.zeros(cw, np.float32) for x in nodes], np.float32),
        )
        trees.append(TreeModel("decision_tree_regressor", F, a, None))
    if gbdt:
        return ForestModel("gbdt_regressor", F, tuple(trees), "sum", 0.1, 0.25, None)
    return ForestModel("random_forest_classifier", F, tuple(trees), "mean_probability", 1.0, 0.0,
                       tuple(float(c) for c in range(C)))


@pytest.mark.parametrize("T,depth,F,C,gbdt,n", [
    (64, 8, 28, 2, False, 200_000),
    (40, 6, 90, 5, False, 50_000),
    (1000, 10, 90, 1, True, 20_000),
    (300, 14, 20, 3, False, 20_000),   # deeper than the perfect layout -> general
])
def test_large_synthetic_vs_c_oracle(T, depth, F, C, gbdt, n):
    rng = np.random.default_rng(T * 7 + depth)
    m = _synthetic_forest(rng, T, depth, F, C, gbdt)
    x = rng.standard_normal((n, F)).astype(np.float32)
    x[::997, 3] = np.nan
    x[::1013, 5] = np.inf
    want, want_leaves = fast.forest_predict(fast.PackedForest(m), x, want_leaves=True)
    spec = lower.lower_model(m)
    xd = torch.from_numpy(x).cuda()
    ran = 0
    for variant in (N.FOREST_AUTO, N.FOREST_RANKED, N.FOREST_PERFECT, N.FOREST_GENERAL, N.FOREST_MMA):
        try:
            prog = DeviceProgram(spec, 0, forest_variant=variant)
        except UnresolvedKernel:
            continue
        leaves = torch.empty((n, T), dtype=torch.int32, device="cuda")
        y = prog.run(xd, leaf_out=leaves).cpu().numpy().astype(np.float64)
        np.testing.assert_array_equal(leaves.cpu().numpy(), want_leaves)
        assert _same(y, want), f"variant {variant} ({prog.forest().info()})"
        prog.close()
        ran += 1
    assert ran >= 2


def test_pinned_host_streaming_matches_device():
    case = gc.get("sk_dt_d6")
    compiled = api.compile_model(case.model)
    x = torch.from_numpy(np.tile(case.x, (600, 1))).pin_memory()  # ~1M rows, several chunks
    from paper_2301_13441_b200.runtime import run_host
    prog = compiled.program(0)
    y_host = run_host(prog, x, chunk_rows=1 << 17)
    y_dev = prog.run(x.cuda()).cpu()
    assert torch.equal(y_host, y_dev)
    assert _same(y_host[: case.x.shape[0]].numpy().astype(np.float64), case.want)


def test_scaler_then_forest_composition():
    """SURVEY 8d config 5 numeric part: execute(rf, execute(scaler, x))."""
    ss = gc.get("sk_standard_scaler")
    rf = gc.get("sk_rf24_d8")
    x = ss.x
    scaled = api.predict(api.compile_model(ss.model), x)
    np.testing.assert_array_equal(scaled.astype(np.float64), ss.want)
    y = api.predict(api.compile_model(rf.model), scaled.astype(np.float32))
    want, _ = sem.predict(rf.model, scaled.astype(np.float32))
    assert _same(y.astype(np.float64), want)


@pytest.mark.parametrize("cfg", range(7))
def test_ranked_launch_configs(cfg, monkeypatch):
    """Every ranked launch configuration (CMLB_RANKED_CFG) is bit-exact."""
    monkeypatch.setenv("CMLB_RANKED_CFG", str(cfg))
    rng = np.random.default_rng(100 + cfg)
    for m, F in ((_synthetic_forest(rng, 37, 8, 28, 2), 28), (_synthetic_forest(rng, 150, 7, 20, 1, True), 20),
                 (_synthetic_forest(rng, 20, 6, 12, 3), 12)):
        x = rng.standard_normal((30_000, F)).astype(np.float32)
        x[::101, 2] = np.nan
        want, want_leaves = fast.forest_predict(fast.PackedForest(m), x, want_leaves=True)
        try:
            prog = DeviceProgram(lower.lower_model(m), 0, forest_variant=N.FOREST_RANKED)
        except UnresolvedKernel:
            continue  # configuration not instantiated for this shape
        leaves = torch.empty((x.shape[0], len(m.trees)), dtype=torch.int32, device="cuda")
        y = prog.run(torch.from_numpy(x).cuda(), leaf_out=leaves).cpu().numpy().astype(np.float64)
        np.testing.assert_array_equal(leaves.cpu().numpy(), want_leaves)
        assert _same(y, want), (cfg, prog.forest().info())
        prog.close()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_tree_sharded_gbr_is_bit_exact(world):
    """Tree shards (pairwise recursion nodes) -> partials -> ordered combine +
    tail on the GPU == the single-program result == the C oracle (config 3 shape,
    scaled down).  The NCCL path only adds the all-gather transport."""
    import ctypes
    from dataclasses import replace
    from paper_2301_13441_b200 import shard
    from paper_2301_13441_b200.lower import ProgramSpec
    rng = np.random.default_rng(world)
    m = _synthetic_forest(rng, 1000, 10, 90, 1, gbdt=True)
    x = rng.standard_normal((20_000, 90)).astype(np.float32)
    want, _ = fast.forest_predict(fast.PackedForest(m), x)
    spec = lower.lower_model(m).stages[0]
    ranges, merges = shard.pairwise_tree_shards(len(spec.trees), world)
    xd = torch.from_numpy(x).cuda()
    parts = torch.empty((world, x.shape[0], 1), dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for i, (lo, hi) in enumerate(ranges):
        prog = DeviceProgram(ProgramSpec([replace(spec, trees=spec.trees[lo:hi])], 90), 0)
        prog.forest().partial(xd, parts[i], x.shape[0], 90, stream)
    full = DeviceProgram(ProgramSpec([spec], 90), 0)
    y = torch.empty((x.shape[0], 1), dtype=torch.float32, device="cuda")
    mm = np.asarray(merges, np.int32).reshape(-1)
    N.check(N.lib().cmlb_forest_finish(full.forest().handle, parts.data_ptr(), world,
                                       mm.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(merges),
                                       x.shape[0], y.data_ptr(), stream))
    single = full.run(xd)
    assert torch.equal(y, single)
    assert _same(y.cpu().numpy().astype(np.float64), want)


@pytest.mark.parametrize("cfg", range(5))
def test_skew_launch_configs(cfg, monkeypatch):
    """Every SKEW launch configuration (CMLB_SKEW_CFG) is bit-exact, leaves
    included, on certified (order-free) forests of 1, 2 and 3 outputs, with
    ragged last groups (T not a multiple of 32) and NaN rows."""
    monkeypatch.setenv("CMLB_SKEW_CFG", str(cfg))
    from paper_2301_13441_b200.models import ForestModel
    rng = np.random.default_rng(300 + cfg)
    rf2 = _synthetic_forest(rng, 77, 8, 28, 2)
    rf3 = _synthetic_forest(rng, 40, 6, 12, 3)
    g = _synthetic_forest(rng, 70, 7, 20, 1, True)
    reg = ForestModel("random_forest_regressor", 20, g.trees, "mean_probability", 1.0, 0.0, None)
    ran = 0
    for m, F in ((rf2, 28), (rf3, 12), (reg, 20)):
        x = rng.standard_normal((30_000, F)).astype(np.float32)
        x[::101, 2] = np.nan
        x[::103, 1] = np.inf
        want, want_leaves = fast.forest_predict(fast.PackedForest(m), x, want_leaves=True)
        try:
            prog = DeviceProgram(lower.lower_model(m), 0, forest_variant=N.FOREST_SKEW)
        except UnresolvedKernel:
            continue  # not certified order-free, or the configuration does not fit
        ran += 1
        leaves = torch.empty((x.shape[0], len(m.trees)), dtype=torch.int32, device="cuda")
        y = prog.run(torch.from_numpy(x).cuda(), leaf_out=leaves).cpu().numpy().astype(np.float64)
        np.testing.assert_array_equal(leaves.cpu().numpy(), want_leaves)
        assert _same(y, want), (cfg, prog.forest().info())
        y2 = prog.run(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
        assert _same(y2, want)
        prog.close()
    assert ran >= (1 if cfg == 4 else 2)  # cfg 4 (1024 rows per CTA) fits only the narrow forests


def test_auto_picks_skew_for_certified_large_forests():
    import bench
    model, _, _ = bench.load_model()
    prog = api.compile_model(model).program(0)
    assert prog.forest().info()["variant"] == "skew"


def _clustered_forest(rng, T, depth, F, C):
    """A forest whose thresholds crowd into a few tiny intervals (plus far
    outliers): bucket tables get large buckets (many binary-lifting steps)."""
    m = _synthetic_forest(rng, T, depth, F, C)
    from paper_2301_13441_b200.models import ForestModel, TreeArrays, TreeModel
    trees = []
    for t in m.trees:
        a = t.arrays
        thr = a.threshold.copy()
        k = np.flatnonzero(~a.is_leaf)
        pick = rng.random(k.size)
        thr[k] = np.where(pick < 0.8, np.float32(1.0) + rng.integers(0, 4000, k.size).astype(np.float32) * np.float32(1e-7),
                          np.where(pick < 0.9, np.float32(-3e6), np.float32(5e30))).astype(np.float32)
        trees.append(TreeModel(t.model_type, F, TreeArrays(a.is_leaf, a.feature, thr, a.left, a.right, a.value), None))
    return ForestModel(m.model_type, F, tuple(trees), m.aggregation, 1.0, 0.0, m.classes)


@pytest.mark.parametrize("eyt", [0, 1])
@pytest.mark.parametrize("rank_pass", [1, 0])
def test_rank_tables_and_fused_ranking(eyt, rank_pass, monkeypatch):
    """Both rank-table formats (bucket tables, CMLB_RANK_EYT=1 Eytzinger) and
    both ranking placements (the rank pass, CMLB_RANK_PASS=0 per-tile in the
    RANKED walk) are bit-exact, on ordinary and on clustered thresholds."""
    if eyt:
        monkeypatch.setenv("CMLB_RANK_EYT", "1")
    if not rank_pass:
        monkeypatch.setenv("CMLB_RANK_PASS", "0")
    rng = np.random.default_rng(500 + 2 * eyt + rank_pass)
    cases = [(_synthetic_forest(rng, 96, 8, 28, 2), 28), (_synthetic_forest(rng, 130, 7, 20, 1, True), 20),
             (_clustered_forest(rng, 80, 7, 6, 2), 6)]
    for m, F in cases:
        x = rng.standard_normal((40_000, F)).astype(np.float32)
        x[: 20_000] = np.float32(1.0) + rng.integers(-10, 4010, (20_000, F)).astype(np.float32) * np.float32(1e-7)
        x[::101, 2] = np.nan
        x[::103, 1] = np.inf
        x[::107, 0] = -np.inf
        x[::109, 3] = -0.0
        want, want_leaves = fast.forest_predict(fast.PackedForest(m), x, want_leaves=True)
        for variant in (N.FOREST_AUTO, N.FOREST_RANKED):
            prog = DeviceProgram(lower.lower_model(m), 0, forest_variant=variant)
            leaves = torch.empty((x.shape[0], len(m.trees)), dtype=torch.int32, device="cuda")
            y = prog.run(torch.from_numpy(x).cuda(), leaf_out=leaves).cpu().numpy().astype(np.float64)
            np.testing.assert_array_equal(leaves.cpu().numpy(), want_leaves)
            assert _same(y, want), (variant, prog.forest().info())
            prog.close()


def test_cuda_graph_capture_replays_the_program():
    """DeviceProgram.capture records one run as a CUDA graph (the bench's
    timed steps replay it): replays equal eager runs, with the input refilled
    in place between replays, and report the kernels of one run."""
    rng = np.random.default_rng(77)
    m = _synthetic_forest(rng, 96, 8, 28, 2)
    prog = DeviceProgram(lower.lower_model(m), 0)
    x = torch.from_numpy(rng.standard_normal((50_000, 28)).astype(np.float32)).cuda()
    y = torch.empty_like(prog.run(x))
    g, launches = prog.capture(x, y)
    assert launches >= 1
    for seed in (1, 2):
        x.copy_(torch.from_numpy(np.random.default_rng(seed).standard_normal((50_000, 28)).astype(np.float32)))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y, prog.run(x))
    prog.close()
