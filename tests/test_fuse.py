"""Composite lowering (pipelines, column transformers, one-hot): the fused
column maps must reproduce the step-by-step oracle bit-exactly.  CPU-only:
the ops are evaluated here with numpy float32 in the kernel's formulas."""

import numpy as np
import pytest

import golden_cases as gc
from oracle import ext_semantics as ext
from paper_2301_13441_b200 import fuse
from paper_2301_13441_b200.fuse import ColumnsSpec
from paper_2301_13441_b200.lower import ForestSpec, LinearSpec, SVMSpec, lower_model


def apply_ops(ops, x):
    """numpy restatement of common.cuh col_apply (float32, no contraction)."""
    x = np.asarray(x, np.float32)
    out = np.empty((x.shape[0], len(ops)), np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        for f, o in enumerate(ops):
            v = x[:, int(o["src"])]
            a, b = np.float32(o["a"]), np.float32(o["b"])
            op = int(o["op"])
            if op == fuse.COPY:
                r = v
            elif op == fuse.SUB_DIV:
                r = np.divide(np.subtract(v, a), b)
            elif op == fuse.DIV:
                r = np.divide(v, a)
            elif op == fuse.MUL_ADD:
                r = np.add(np.multiply(v, a), b)
            elif op == fuse.GREATER:
                r = (v > a).astype(np.float32)
            else:
                r = (v == a).astype(np.float32)
            out[:, f] = r
    return out


TRANSFORM_CASES = [n for n in gc.ext_case_names() if gc.ext_get(n).kind == "transform"]
PIPE_CASES = [n for n in gc.ext_case_names() if gc.ext_get(n).kind == "pipeline"]


@pytest.mark.parametrize("name", TRANSFORM_CASES)
def test_column_map_matches_sklearn_transform(name):
    case = gc.ext_get(name)
    spec = lower_model(case.model)
    assert len(spec.stages) == 1 and isinstance(spec.stages[0], ColumnsSpec)
    got = apply_ops(spec.stages[0].ops, case.x)
    np.testing.assert_array_equal(got.astype(np.float64), case.want)


@pytest.mark.parametrize("name", PIPE_CASES)
def test_pipeline_prologue_is_fused(name):
    case = gc.ext_get(name)
    spec = lower_model(case.model)
    consumer = spec.stages[-1]
    assert isinstance(consumer, (ForestSpec, LinearSpec, SVMSpec))
    assert consumer.prologue is not None and consumer.n_inputs == case.x.shape[1]
    # the fused ops give the same model inputs as the step-by-step oracle
    steps = case.model.steps
    want_in = case.x
    for s in steps[:-1]:
        want_in = ext.transform(s, want_in)
    np.testing.assert_array_equal(apply_ops(consumer.prologue, case.x), want_in)
    # a check-only stage precedes the consumer iff some encoder raises on unknowns
    checks = [st for st in spec.stages[:-1] if isinstance(st, ColumnsSpec)]
    assert all(not st.emit for st in checks)


def test_compose_scaler_then_onehot_passthrough():
    from paper_2301_13441_b200.extmodels import ColumnTransformerModel, OneHotModel, PipelineModel
    from paper_2301_13441_b200.models import ScalerModel
    ss = ScalerModel("standard_scaler", 3, vectors=(("mean", (1.0, 2.0, 3.0)), ("scale", (2.0, 4.0, 8.0))))
    oh = OneHotModel("one_hot_encoder", 1, (np.array([0.0, 1.0], np.float32),), (None,), "ignore")
    ct = ColumnTransformerModel("column_transformer", 4, (((0, 1, 2), ss), ((3,), oh)), "drop")
    m = PipelineModel("pipeline", 4, (ct,))
    spec = lower_model(m)
    x = np.array([[1, 2, 3, 1], [3, 6, 11, 0], [0, 0, 0, 5]], np.float32)
    np.testing.assert_array_equal(apply_ops(spec.stages[0].ops, x), ext.transform(m, x))


def test_two_arithmetic_ops_on_one_column_are_not_composed():
    from paper_2301_13441_b200.extmodels import PipelineModel
    from paper_2301_13441_b200.models import ScalerModel
    a = ScalerModel("standard_scaler", 2, vectors=(("mean", (1.0, 2.0)), ("scale", (2.0, 4.0))))
    b = ScalerModel("maxabs_scaler", 2, vectors=(("scale", (3.0, 5.0)),))
    spec = lower_model(PipelineModel("pipeline", 2, (a, b)))
    assert len(spec.stages) == 2  # materialise the first map, then apply the second
