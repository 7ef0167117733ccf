"""Lowering: a trained model or a reference ``KernelPlan`` -> fused device program.

The reference runs a plan as an SSA list of per-node numpy kernels
(``pkg/src/mlower/runtime.py:147-212``): for RF500 that is 3,005 invocations
with (N x I) and (N x L) intermediates per tree.  Here the same computation is
recognised as a handful of *operator representations* and each one becomes a
single fused kernel of ``libcmlb.so``:

=====================  =====================================================
stage                  reference pattern (convert.py)
=====================  =====================================================
ForestSpec             per-tree chain ``matmul|sparse(W1) -> greater(W2) ->
                       [cast] -> matmul|sparse(W3) -> argmax ->
                       gather_rows(leaf_table)`` (192-204), or
                       ``broadcast_const`` (194-196); single tree (225-227)
                       or ``stack -> [cast] -> reduce_mean|reduce_sum ->
                       [mul lr -> add base]`` (287-311) with the classifier /
                       binary tails (211-222)
LinearSpec             ``matmul|sparse(coef^T) -> add(b)`` + tails (230-252)
ScalerSpec             Binarizer / Normalizer / MinMax / Robust / Standard /
                       MaxAbs (255-284)
=====================  =====================================================

Two entry routes produce identical specs (tested on CPU):

* :func:`lower_model` -- straight from model arrays, never materialising the
  dense W1/W3 matrices (ingestion at scale);
* :func:`lower_plan` -- from a ``KernelPlan`` (the ``execute(plan, x)``
  drop-in), inverting W1/W2/W3 per tree (``trees.canon_from_encoding``).

Semantics the CPU profile changes are carried as flags: a *dense* selector
matmul poisons rows with non-finite features and a *dense*
linear weight multiplies 0 * inf (``kernels.py:95-100`` vs ``115-123``);
RE removing softmax changes nothing, keeping it (passes without ``re``)
rounds probabilities to float32 before the argmax.  Any other plan shape
raises ``UnresolvedKernel`` -- there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .dtypes import dispatch_name, name_of, smallest_name
from .errors import UnresolvedKernel, ValidationError
from .models import family_of, tree_arrays_of
from .trees import CanonTree, canon_from_arrays, canon_from_encoding, single_leaf

DEFAULT_PASSES = ("re", "dr", "sor")
_PROFILE_THRESHOLD = {"cpu-avx2": 0.3, "plain": 0.0}


# -- program specs -------------------------------------------------------------


@dataclass(eq=False)
class ForestSpec:
    trees: list
    n_features: int
    n_outputs: int
    aggregation: int
    tail: int
    learning_rate: float = 1.0
    base_score: float = 0.0
    classes: tuple = ()
    out_dtype: str = "float32"
    dense_selector: bool = False
    prologue: object = None        # fuse.COL_DTYPE ops over the raw input (fused preprocessing)
    n_inputs: int = 0
    n_trees_total: int = 0         # tree shard of a larger ensemble: its tree count (MEAN tail)

    @property
    def in_cols(self) -> int:
        return self.n_inputs if self.prologue is not None else self.n_features

    @property
    def out_cols(self) -> int:
        return self.n_outputs if self.tail == N.TAIL_VALUES else 1

    def same_as(self, other: "ForestSpec") -> bool:
        head = ("n_features", "n_outputs", "aggregation", "tail", "out_dtype", "dense_selector")
        if any(getattr(self, k) != getattr(other, k) for k in head):
            return False
        if np.float32(self.learning_rate) != np.float32(other.learning_rate):
            return False
        if np.float32(self.base_score) != np.float32(other.base_score):
            return False
        if tuple(map(float, self.classes)) != tuple(map(float, other.classes)):
            return False
        return len(self.trees) == len(other.trees) and all(
            a.same_as(b) for a, b in zip(self.trees, other.trees))


@dataclass(eq=False)
class LinearSpec:
    coef: np.ndarray          # float32 (C, F)
    intercept: np.ndarray     # float32 (C,)
    tail: int
    classes: tuple = ()
    out_dtype: str = "float32"
    sparse_coef: bool = False
    prologue: object = None
    n_inputs: int = 0

    @property
    def n_features(self) -> int:
        return int(self.coef.shape[1])

    @property
    def in_cols(self) -> int:
        return self.n_inputs if self.prologue is not None else self.n_features

    @property
    def out_cols(self) -> int:
        return int(self.coef.shape[0]) if self.tail == N.LIN_VALUES else 1


@dataclass(eq=False)
class ScalerSpec:
    kind: int
    n_features: int
    threshold: float = 0.0
    a: np.ndarray | None = None
    b: np.ndarray | None = None
    out_dtype: str = "float32"

    @property
    def out_cols(self) -> int:
        return self.n_features


@dataclass(eq=False)
class SVMSpec:
    """Kernel SVM (extmodels.SVMModel): libsvm decision + votes (svc) or value (svr)."""

    model: object
    out_dtype: str = "float32"
    prologue: object = None
    n_inputs: int = 0

    @property
    def n_features(self) -> int:
        return self.model.n_features

    @property
    def in_cols(self) -> int:
        return self.n_inputs if self.prologue is not None else self.n_features

    @property
    def out_cols(self) -> int:
        return 1


@dataclass(eq=False)
class ProgramSpec:
    """Stages run back to back; stage i's output feeds stage i+1."""

    stages: list = field(default_factory=list)
    n_features: int = 0

    @property
    def out_dtype(self) -> str:
        return self.stages[-1].out_dtype

    @property
    def out_cols(self) -> int:
        return self.stages[-1].out_cols


# -- profile handling ----------------------------------------------------------


@dataclass(frozen=True)
class Profile:
    """Mirror of the reference ``HardwareProfile`` (``graph.py:128-135``).
    Only ``sparse_threshold`` changes GPU semantics (dense vs CSR selector and
    linear weights, SOR ``passes.py:201-215``)."""

    name: str
    preferred_int_dtype: str
    sparse_threshold: float
    notes: str = ""


BUILTIN_PROFILES = {"cpu-avx2": Profile("cpu-avx2", "int8", 0.3), "plain": Profile("plain", "int32", 0.0)}


def load_profile(name_or_path: str) -> Profile:
    """Builtin name or JSON profile file, validated as ``graph.py:146-168``."""
    import json

    from .errors import ProfileError
    if name_or_path in BUILTIN_PROFILES:
        return BUILTIN_PROFILES[name_or_path]
    try:
        with open(name_or_path, "r", encoding="utf-8") as fh:
            obj = json.load(fh)
    except OSError as e:
        raise ProfileError(f"cannot read profile {name_or_path!r}: {e}") from None
    except json.JSONDecodeError as e:
        raise ProfileError(f"profile {name_or_path!r}: invalid JSON ({e.msg})") from None
    if not isinstance(obj, dict):
        raise ProfileError("profile must be a JSON object")
    try:
        name = obj["name"]
        pref = str(obj["preferred_int_dtype"])
        threshold = float(obj["sparse_threshold"])
    except KeyError as e:
        raise ProfileError(f"profile missing field {e.args[0]!r}") from None
    except (TypeError, ValueError):
        raise ProfileError("sparse_threshold must be a number") from None
    if pref not in ("int8", "int16", "int32"):
        raise ProfileError("preferred_int_dtype must be int8, int16 or int32")
    if not 0.0 <= threshold <= 1.0:
        raise ProfileError("sparse_threshold must lie in [0, 1]")
    return Profile(str(name), pref, threshold, str(obj.get("notes", "")))


def sparse_threshold(profile) -> float:
    if profile is None:
        return _PROFILE_THRESHOLD["cpu-avx2"]
    if isinstance(profile, str):
        return load_profile(profile).sparse_threshold
    return float(profile.sparse_threshold)


def _goes_csr(density: float, profile, passes) -> bool:
    """SOR (passes.py:201-215): matmul weights below the profile threshold."""
    return "sor" in tuple(passes) and density < sparse_threshold(profile)


# -- route 1: model -> spec ----------------------------------------------------


def _class_out(classes) -> str:
    return dispatch_name(smallest_name(np.asarray(classes, np.float64)))


def _first_max_labels(values: np.ndarray, classes) -> np.ndarray:
    """Per leaf: classes[first max of the leaf vector] (convert.py:177-189)."""
    idx = np.argmax(values, axis=1)  # first occurrence == (value, -i) max
    return np.asarray(classes, np.float64)[idx]


def lower_tree_model(m, profile=None, passes=DEFAULT_PASSES) -> ForestSpec:
    a = tree_arrays_of(m)
    dense = not _goes_csr(1.0 / m.n_features, profile, passes)
    if m.classes is not None:
        labels = np.zeros((a.n_nodes, 1), np.float64)
        leaves = np.flatnonzero(a.is_leaf)
        labels[leaves, 0] = _first_max_labels(a.value[leaves].astype(np.float64), m.classes)
        t = canon_from_arrays(a, labels)
        out = dispatch_name(smallest_name(t.payload))
        return ForestSpec([t], m.n_features, 1, N.AGG_NONE, N.TAIL_VALUES, out_dtype=out,
                          dense_selector=dense and t.n_internal > 0)
    t = canon_from_arrays(a)
    return ForestSpec([t], m.n_features, t.payload.shape[1], N.AGG_NONE, N.TAIL_VALUES,
                      out_dtype="float32", dense_selector=dense and t.n_internal > 0)


def lower_forest_model(m, profile=None, passes=DEFAULT_PASSES) -> ForestSpec:
    trees = [canon_from_arrays(tree_arrays_of(t)) for t in m.trees]
    C = trees[0].payload.shape[1]
    dense = not _goes_csr(1.0 / m.n_features, profile, passes) and any(t.n_internal for t in trees)
    if m.aggregation == "mean_probability":
        if m.classes is not None:
            return ForestSpec(trees, m.n_features, C, N.AGG_MEAN, N.TAIL_ARGMAX,
                              classes=tuple(m.classes), out_dtype=_class_out(m.classes),
                              dense_selector=dense)
        return ForestSpec(trees, m.n_features, C, N.AGG_MEAN, N.TAIL_VALUES, dense_selector=dense)
    tail = N.TAIL_SIGMOID if m.classes is not None else N.TAIL_VALUES
    return ForestSpec(trees, m.n_features, 1, N.AGG_SUM, tail, learning_rate=float(m.learning_rate),
                      base_score=float(m.base_score), classes=tuple(m.classes or ()),
                      out_dtype=_class_out(m.classes) if m.classes is not None else "float32",
                      dense_selector=dense)


def lower_linear_model(m, profile=None, passes=DEFAULT_PASSES) -> LinearSpec:
    coef = np.asarray(m.coef, np.float32).reshape(len(m.coef), -1)
    intercept = np.asarray(m.intercept, np.float32)
    sparse = _goes_csr(np.count_nonzero(coef) / coef.size, profile, passes)
    if m.classes is None:
        return LinearSpec(coef, intercept, N.LIN_VALUES, sparse_coef=sparse)
    logistic = m.model_type == "logistic_regression"
    if coef.shape[0] == 1:
        tail = N.LIN_SIGMOID if logistic else N.LIN_SIGN
    else:
        tail = N.LIN_SOFTMAX_ARGMAX if logistic and "re" not in tuple(passes) else N.LIN_ARGMAX
    return LinearSpec(coef, intercept, tail, tuple(m.classes), _class_out(m.classes), sparse)


def lower_scaler_model(m) -> ScalerSpec:
    F = m.n_features
    kind = m.model_type
    vec = lambda name: np.asarray(m.vector(name), np.float32)
    if kind == "binarizer":
        return ScalerSpec(N.SCALER_BINARIZER, F, threshold=float(np.float32(m.threshold)))
    if kind == "normalizer":
        k = {"l1": N.SCALER_NORM_L1, "l2": N.SCALER_NORM_L2, "max": N.SCALER_NORM_MAX}[m.norm]
        return ScalerSpec(k, F)
    if kind == "minmax_scaler":
        return ScalerSpec(N.SCALER_MINMAX, F, a=vec("scale"), b=vec("min"))
    if kind == "robust_scaler":
        return ScalerSpec(N.SCALER_SUB_DIV, F, a=vec("center"), b=vec("scale"))
    if kind == "standard_scaler":
        return ScalerSpec(N.SCALER_SUB_DIV, F, a=vec("mean"), b=vec("scale"))
    if kind == "maxabs_scaler":
        return ScalerSpec(N.SCALER_DIV, F, a=vec("scale"))
    raise UnresolvedKernel(f"unknown scaler kind {kind!r}")


def lower_model(model, profile=None, passes=DEFAULT_PASSES) -> ProgramSpec:
    fam = family_of(model)
    if fam == "tree":
        st = lower_tree_model(model, profile, passes)
    elif fam == "forest":
        st = lower_forest_model(model, profile, passes)
    elif fam == "linear":
        st = lower_linear_model(model, profile, passes)
    elif fam == "svm":
        st = SVMSpec(model, _class_out(model.classes) if model.classes is not None else "float32")
    elif fam in ("columns", "pipeline"):
        from .fuse import lower_composite
        return lower_composite(model, profile, passes)
    else:
        st = lower_scaler_model(model)
    return ProgramSpec([st], model.n_features)


# -- route 2: KernelPlan -> spec -----------------------------------------------


class _PlanView:
    """Producer lookup over a reference (or fixture) KernelPlan."""

    def __init__(self, plan):
        self.plan = plan
        self.prod = {inv.output: inv for inv in plan.invocations}
        self.input_slot = plan.input_slot

    def at(self, slot):
        return self.prod.get(slot)

    def skip_casts(self, slot):
        inv = self.at(slot)
        while inv is not None and inv.kernel in ("cast", "reshape"):
            slot = inv.inputs[0]
            inv = self.at(slot)
        return slot, inv

    @staticmethod
    def weight(inv, name) -> np.ndarray:
        for b in inv.weights:
            if b.name == name:
                return np.asarray(b.tensor.to_numpy(), dtype=np.float64)
        raise UnresolvedKernel(f"{inv.kernel}: missing weight {name!r}")

    def is_input(self, slot) -> bool:
        return slot == self.input_slot

    def dtype(self, slot) -> str:
        return dispatch_name(name_of(self.plan.slot_dtypes[slot]))


def _fail(what: str):
    raise UnresolvedKernel(f"no fused B200 lowering for this plan: {what}")


def _match_tree(v: _PlanView, slot):
    """A tree chain ending at ``slot`` -> (CanonTree, dense selector?)."""
    slot, inv = v.skip_casts(slot)
    if inv is None:
        _fail("tree output is the graph input")
    if inv.kernel == "broadcast_const":
        row = v.weight(inv, "row")
        return single_leaf(row.reshape(-1)), None
    if inv.kernel != "gather_rows":
        _fail(f"expected gather_rows at a tree output, found {inv.kernel}")
    table = v.weight(inv, "table")
    s, am = v.skip_casts(inv.inputs[0])
    if am is None or am.kernel != "argmax":
        _fail("leaf gather not fed by argmax")
    s, routes = v.skip_casts(am.inputs[0])
    if routes is None or routes.kernel not in ("matmul", "sparse_dense_matmul"):
        _fail("argmax not fed by the route matmul")
    w3 = v.weight(routes, "w")
    s, gt = v.skip_casts(routes.inputs[0])
    if gt is None or gt.kernel != "greater":
        _fail("route matmul not fed by greater")
    w2 = v.weight(gt, "rhs").reshape(-1)
    s, sel = v.skip_casts(gt.inputs[0])
    if sel is None or sel.kernel not in ("matmul", "sparse_dense_matmul"):
        _fail("greater not fed by the selector matmul")
    if not v.is_input(v.skip_casts(sel.inputs[0])[0]):
        _fail("selector does not read the graph input")
    w1 = v.weight(sel, "w")
    t = canon_from_encoding(w1, w2, w3, table.reshape(table.shape[0], -1))
    return t, sel.kernel == "matmul"


def _class_table(v: _PlanView, inv) -> tuple:
    tab = v.weight(inv, "table")
    if tab.ndim != 2 or tab.shape[1] != 1:
        _fail("class table is not a column")
    return tuple(float(c) for c in tab[:, 0])


def _forest_body(v: _PlanView, slot, agg_kernel):
    """reduce_* <- [cast] <- stack(trees) -> (trees, dense flag)."""
    slot, red = v.skip_casts(slot)
    if red is None or red.kernel != agg_kernel:
        _fail(f"expected {agg_kernel}")
    _, stack = v.skip_casts(red.inputs[0])
    if stack is None or stack.kernel != "stack":
        _fail("reduction not fed by stack")
    trees, dense = [], set()
    for s in stack.inputs:
        t, d = _match_tree(v, s)
        trees.append(t)
        if d is not None:
            dense.add(d)
    if len(dense) > 1:
        _fail("mixed dense/sparse selectors in one ensemble")
    return trees, bool(dense and dense.pop())


def lower_plan(plan) -> ProgramSpec:
    v = _PlanView(plan)
    F = int(plan.n_features)
    if name_of(plan.input_dtype) != "float32":
        _fail("non-float32 graph input")
    out_slot = plan.output_slot
    out_dtype = v.dtype(out_slot)
    top = v.at(out_slot)
    if top is None:
        _fail("plan output is its input")
    k = top.kernel

    # ---- scalers --------------------------------------------------------
    if k == "cast" and v.at(top.inputs[0]) is not None and v.at(top.inputs[0]).kernel == "greater":
        gt = v.at(top.inputs[0])
        if v.is_input(gt.inputs[0]) and name_of(top.attr("target")) == "float32":
            thr = v.weight(gt, "rhs").reshape(-1)
            return ProgramSpec([ScalerSpec(N.SCALER_BINARIZER, F, threshold=float(np.float32(thr[0])))], F)
    if k == "div" and len(top.inputs) == 2:
        rn = v.at(top.inputs[1])
        if rn is not None and rn.kernel == "row_norm" and v.is_input(top.inputs[0]):
            kind = {"l1": N.SCALER_NORM_L1, "l2": N.SCALER_NORM_L2, "max": N.SCALER_NORM_MAX}[rn.attr("kind")]
            return ProgramSpec([ScalerSpec(kind, F)], F)
    if k in ("add", "div") and len(top.inputs) == 1:
        below = v.at(top.inputs[0])
        vec_top = v.weight(top, "rhs").reshape(-1).astype(np.float32)
        if k == "add" and below is not None and below.kernel == "mul" and v.is_input(below.inputs[0]):
            scale = v.weight(below, "rhs").reshape(-1).astype(np.float32)
            if scale.size == F:
                return ProgramSpec([ScalerSpec(N.SCALER_MINMAX, F, a=scale, b=vec_top)], F)
        if k == "div" and below is not None and below.kernel == "sub" and v.is_input(below.inputs[0]):
            center = v.weight(below, "rhs").reshape(-1).astype(np.float32)
            return ProgramSpec([ScalerSpec(N.SCALER_SUB_DIV, F, a=center, b=vec_top)], F)
        if k == "div" and v.is_input(top.inputs[0]):
            return ProgramSpec([ScalerSpec(N.SCALER_DIV, F, a=vec_top)], F)

    # ---- tails -> score slot -----------------------------------------------
    tail, classes, score = None, (), None
    softmax = False
    if k == "gather_rows":
        s, src = v.skip_casts(top.inputs[0])
        if src is not None and src.kernel == "argmax":
            s2, below = v.skip_casts(src.inputs[0])
            if below is not None and below.kernel in ("softmax", "monotonic_chain"):
                softmax = True
                s2 = below.inputs[0]
                below = v.at(s2)
            if below is not None and below.kernel not in ("matmul", "sparse_dense_matmul"):
                tail, classes, score = "argmax", _class_table(v, top), s2
        elif src is not None and src.kernel == "greater":
            dec = float(v.weight(src, "rhs").reshape(-1)[0])
            s2, below = v.skip_casts(src.inputs[0])
            if below is not None and below.kernel == "sigmoid":
                if dec != 0.5:
                    _fail("sigmoid threshold other than 0.5")
                tail, score = "sigmoid", below.inputs[0]
            else:
                if dec != 0.0:
                    _fail("margin threshold other than 0.0")
                tail, score = "sign", s2
            classes = _class_table(v, top)
    if tail is None:  # no classifier tail: a tree, a regressor forest or a linear regressor
        score = out_slot

    s, inv = v.skip_casts(score)
    if inv is None:
        _fail("score is the graph input")

    # ---- linear -----------------------------------------------------------
    if inv.kernel == "add" and len(inv.inputs) == 1:
        _, mm = v.skip_casts(inv.inputs[0])
        if mm is not None and mm.kernel in ("matmul", "sparse_dense_matmul") and \
                v.is_input(v.skip_casts(mm.inputs[0])[0]):
            coef = v.weight(mm, "w").T.astype(np.float32)           # (C, F)
            intercept = v.weight(inv, "rhs").reshape(-1).astype(np.float32)
            if intercept.size == 1 and coef.shape[0] > 1:
                intercept = np.full(coef.shape[0], intercept[0], np.float32)
            sparse = mm.kernel == "sparse_dense_matmul"
            lin_tail = {None: N.LIN_VALUES, "argmax": N.LIN_SOFTMAX_ARGMAX if softmax else N.LIN_ARGMAX,
                        "sigmoid": N.LIN_SIGMOID, "sign": N.LIN_SIGN}[tail]
            return ProgramSpec([LinearSpec(coef, intercept, lin_tail, classes, out_dtype, sparse)], F)
        # gradient boosting: add(base) <- mul(lr) <- reduce_sum
        if mm is not None and mm.kernel == "mul":
            base = float(v.weight(inv, "rhs").reshape(-1)[0])
            lr = float(v.weight(mm, "rhs").reshape(-1)[0])
            trees, dense = _forest_body(v, mm.inputs[0], "reduce_sum")
            if tail not in (None, "sigmoid"):
                _fail("gradient boosting with an unexpected tail")
            return ProgramSpec([ForestSpec(
                trees, F, 1, N.AGG_SUM, N.TAIL_SIGMOID if tail == "sigmoid" else N.TAIL_VALUES,
                learning_rate=lr, base_score=base, classes=classes, out_dtype=out_dtype,
                dense_selector=dense)], F)

    # ---- random forests ----------------------------------------------------
    if inv.kernel == "reduce_mean":
        trees, dense = _forest_body(v, s, "reduce_mean")
        if tail not in (None, "argmax") or softmax:
            _fail("random forest with an unexpected tail")
        C = trees[0].payload.shape[1]
        return ProgramSpec([ForestSpec(
            trees, F, C, N.AGG_MEAN, N.TAIL_ARGMAX if tail else N.TAIL_VALUES,
            classes=classes, out_dtype=out_dtype, dense_selector=dense)], F)

    # ---- single decision tree ------------------------------------------------
    if tail is None and inv.kernel in ("gather_rows", "broadcast_const"):
        t, dense = _match_tree(v, out_slot)
        return ProgramSpec([ForestSpec([t], F, t.payload.shape[1], N.AGG_NONE, N.TAIL_VALUES,
                                       out_dtype=out_dtype, dense_selector=bool(dense))], F)
    _fail(f"unrecognised pattern ending in {k}")
    raise AssertionError  # pragma: no cover


def specs_equal(a: ProgramSpec, b: ProgramSpec) -> bool:
    if a.n_features != b.n_features or len(a.stages) != len(b.stages):
        return False
    for x, y in zip(a.stages, b.stages):
        if type(x) is not type(y):
            return False
        if isinstance(x, ForestSpec):
            if not x.same_as(y):
                return False
        elif isinstance(x, LinearSpec):
            if not (np.array_equal(x.coef, y.coef) and np.array_equal(x.intercept, y.intercept)
                    and x.tail == y.tail and tuple(x.classes) == tuple(y.classes)
                    and x.out_dtype == y.out_dtype and x.sparse_coef == y.sparse_coef):
                return False
        else:
            for f in ("kind", "n_features", "threshold", "out_dtype"):
                if getattr(x, f) != getattr(y, f):
                    return False
            for f in ("a", "b"):
                p, q = getattr(x, f), getattr(y, f)
                if (p is None) != (q is None) or (p is not None and not np.array_equal(p, q)):
                    return False
    return True


__all__ = ["ForestSpec", "LinearSpec", "ScalerSpec", "ProgramSpec", "lower_model", "lower_plan",
           "specs_equal", "CanonTree"]
