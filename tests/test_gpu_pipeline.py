"""GPU parity of fused pipelines (column transformer / one-hot / scaler ->
forest, linear, SVM) against the step-by-step oracle (reference semantics for
the reference families, scikit-learn for one-hot and SVM)."""

import numpy as np
import pytest
import torch

import golden_cases as gc
from oracle import ext_semantics as ext
from paper_2301_13441_b200 import _native as N, api
from paper_2301_13441_b200.errors import UnresolvedKernel, ValidationError
from paper_2301_13441_b200.lower import ForestSpec
from paper_2301_13441_b200.runtime import DeviceProgram

pytestmark = pytest.mark.gpu

CASES = [n for n in gc.ext_case_names() if gc.ext_get(n).kind in ("transform", "pipeline")]


@pytest.mark.parametrize("name", CASES)
def test_pipeline_host_api(name):
    case = gc.ext_get(name)
    got = api.predict(api.compile_model(case.model), case.x)
    np.testing.assert_array_equal(np.asarray(got, np.float64).reshape(case.want.shape), case.want)


@pytest.mark.parametrize("name", CASES)
def test_pipeline_device_api(name):
    case = gc.ext_get(name)
    compiled = api.compile_model(case.model)
    y = api.predict(compiled, torch.from_numpy(case.x).cuda())
    np.testing.assert_array_equal(y.cpu().numpy().astype(np.float64).reshape(case.want.shape), case.want)


@pytest.mark.parametrize("variant", [N.FOREST_PERFECT, N.FOREST_GENERAL, N.FOREST_RANKED, N.FOREST_MMA])
def test_pipeline_forest_variants(variant):
    case = gc.ext_get("pipe_ct_rf16")
    spec = api.compile_model(case.model).spec
    assert isinstance(spec.stages[-1], ForestSpec) and spec.stages[-1].prologue is not None
    try:
        prog = DeviceProgram(spec, 0, forest_variant=variant)
    except UnresolvedKernel:
        pytest.skip("variant cannot hold this forest")
    y = prog.run(torch.from_numpy(case.x).cuda())
    np.testing.assert_array_equal(y.cpu().numpy().astype(np.float64), case.want)


def test_unknown_category_raises_host_and_device():
    case = gc.ext_get("pipe_ct_rf16")       # OneHotEncoder(handle_unknown='error')
    compiled = api.compile_model(case.model)
    x = case.x.copy()
    x[37, 12] = 1234.5
    with pytest.raises(ValidationError, match="row 37"):
        api.predict(compiled, x)
    with pytest.raises(ValidationError):
        api.predict(compiled, torch.from_numpy(x).cuda())
    with pytest.raises(ext.UnknownCategory):
        ext.predict(case.model, x)


def test_unknown_category_ignored():
    case = gc.ext_get("onehot_ignore")      # rows 0..19 hold an unseen value
    got = api.predict(api.compile_model(case.model), case.x)
    np.testing.assert_array_equal(np.asarray(got, np.float64), case.want)


def test_pipeline_rf_large_vs_oracle():
    """Config-5 shape at reduced size: StandardScaler(56 numeric) + OneHot(8 x <=16)
    -> the RF500 d8 bench forest re-indexed onto the transformed width."""
    from workloads import config5_pipeline
    m, x = config5_pipeline(rows=20_000)
    got = api.predict(api.compile_model(m), x)
    want, _ = ext.predict(m, x)
    np.testing.assert_array_equal(np.asarray(got, np.float64).reshape(want.shape), want)


@pytest.mark.parametrize("name", CASES)
def test_pipeline_cuda_graph_replay(name):
    """Every fused pipeline program replays as one CUDA graph
    (DeviceProgram.capture, the bench's timed form) with the same outputs;
    programs with membership checks report through the bad-row slot."""
    case = gc.ext_get(name)
    prog = api.compile_model(case.model).program(0)
    x = torch.from_numpy(np.ascontiguousarray(case.x, np.float32)).cuda()
    want = prog.run(x)
    y = torch.empty_like(want)
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda") if prog.has_checks else None
    g, launches = prog.capture(x, y, bad=bad)
    assert launches >= 1
    y.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)
    if bad is not None:
        assert int(bad.item()) == -1
