"""Command-line front door on the GPU path: ``compile``, ``run``, ``verify``.

Mirrors the reference CLI (``pkg/src/mlower/cli.py:99-188``): same
subcommands and flags (``--model``, ``--profile``, ``--passes``, ``--input``,
``--output``, ``--random``, ``--seed``), same CSV interchange (shortest
float32 round-trip decimals, ``tensor.py:166-189``, ``dtypes.py:150-157``),
same exit codes (0 ok, 1 verification failure, 2 usage/validation error) and
the same first error line ``error: <code>: <detail>``.  What differs is where
``run`` executes: the fused sm_100a program (``api.predict``).

``verify`` cross-checks the GPU result against the reference's own scalar
oracle (``mlower.oracle.oracle_predict``), so it needs the reference package
importable; ``compile`` prints the fused program instead of the reference's
kernel plan.

    python -m paper_2301_13441_b200 run --model m.json --input x.csv --output y.csv
"""

from __future__ import annotations

import argparse
import io
import sys

import numpy as np

from .errors import FileAccessError, MlowerError, ValidationError

DEFAULT_TOLERANCE = 1e-5
PASS_ORDER = ("re", "dr", "sor")


def format_f32(x) -> str:
    """Shortest decimal that round-trips through float32 (reference dtypes.py:150-157)."""
    v = np.float32(x)
    if np.isnan(v):
        return "nan"
    if np.isinf(v):
        return "inf" if v > 0 else "-inf"
    return np.format_float_positional(v, unique=True, trim="0")


def read_csv(text: str, n_cols: int) -> np.ndarray:
    """CSV -> float32 rows, parsed as Python floats (float64) then rounded once,
    like the reference's ``read_csv_text`` (tensor.py:166-181)."""
    lines = [ln.strip() for ln in text.splitlines()]
    lines = [ln for ln in lines if ln]
    if not lines:
        return np.zeros((0, n_cols), np.float32)
    try:
        arr = np.loadtxt(io.StringIO("\n".join(lines)), delimiter=",", dtype=np.float64, ndmin=2)
    except ValueError as e:
        raise ValidationError(f"CSV: {e}") from None
    return np.ascontiguousarray(arr.astype(np.float32))


def write_csv(values: np.ndarray) -> str:
    arr = np.asarray(values).astype(np.float32).reshape(len(values), -1)
    out = [",".join(format_f32(v) for v in row) for row in arr]
    return "\n".join(out) + ("\n" if out else "")


def _read_text(path: str) -> str:
    try:
        with open(path, "r", encoding="utf-8") as fh:
            return fh.read()
    except OSError as e:
        raise FileAccessError(f"cannot read {path!r}: {e}") from None


def _passes(spec):
    if spec is None:
        return PASS_ORDER
    parts = tuple(p for p in (s.strip() for s in spec.split(",")) if p)
    unknown = set(parts) - set(PASS_ORDER)
    if unknown:
        raise MlowerError(f"unknown pass flags: {','.join(sorted(unknown))}")
    return parts


def _compile(args):
    from .api import compile_model
    from .models import parse_model
    from .lower import load_profile
    profile = load_profile(args.profile)  # builtin name or JSON profile file (graph.py:146-168)
    return compile_model(parse_model(_read_text(args.model)), profile, _passes(args.passes))


def cmd_compile(args) -> int:
    compiled = _compile(args)
    prog = compiled.program()
    for i, st in enumerate(prog.stages):
        spec = st.spec
        line = f"stage {i}: {type(spec).__name__} in={getattr(spec, 'in_cols', spec.n_features)} out={spec.out_cols} " \
               f"dtype={spec.out_dtype}"
        if hasattr(st, "info"):
            line += f" {st.info()}"
        if getattr(spec, "prologue", None) is not None:
            line += f" prologue={len(spec.prologue)} fused column ops"
        sys.stdout.write(line + "\n")
    return 0


def cmd_run(args) -> int:
    from .api import predict
    compiled = _compile(args)
    x = read_csv(_read_text(args.input), compiled.spec.n_features)
    y = predict(compiled, x) if len(x) else np.zeros((0, compiled.spec.out_cols))
    text = write_csv(y)
    if args.output:
        with open(args.output, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


def cmd_verify(args) -> int:
    from .api import predict
    try:
        from mlower.oracle import oracle_predict  # the reference's scalar oracle
        import mlower
    except ImportError:
        raise ValidationError("verify compares against the reference's oracle: install mlower") from None
    compiled = _compile(args)
    model = compiled.model
    F = model.n_features
    if args.input:
        x = read_csv(_read_text(args.input), F)
    else:
        rows = [[0.0] * F]
        for f, t in model.thresholds():  # boundary rows (reference cli.py:61-68)
            r = [0.0] * F
            r[f] = t
            rows.append(r)
        rng = np.random.default_rng(args.seed)
        x = np.asarray(rows + rng.uniform(-10.0, 10.0, size=(args.random, F)).tolist(), np.float32)
    got = np.asarray(predict(compiled, x), np.float64).reshape(len(x), -1)
    ref_model = mlower.parse_model(_read_text(args.model))
    want = np.asarray(oracle_predict(ref_model, [list(map(float, r)) for r in x]), np.float64).reshape(len(x), -1)
    if got.size:
        diff = np.abs(got - want)
        abs_div, rel_div = float(diff.max()), float((diff / np.maximum(np.abs(want), 1.0)).max())
    else:
        abs_div = rel_div = 0.0
    classifier = bool(getattr(model, "is_classifier", False))
    ok = abs_div == 0.0 if classifier else rel_div <= DEFAULT_TOLERANCE
    sys.stdout.write(f"verify: rows={len(x)} outputs={got.shape[1]} mode={'exact' if classifier else 'tolerance'}\n")
    sys.stdout.write(f"max_abs_divergence={format_f32(abs_div)}\n")
    sys.stdout.write(f"max_rel_divergence={format_f32(rel_div)}\n")
    sys.stdout.write(f"result: {'PASS' if ok else 'FAIL'} (tolerance {DEFAULT_TOLERANCE})\n")
    return 0 if ok else 1


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2301_13441_b200",
                                     description="Run trained classical-ML models on the B200 path.")
    sub = parser.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--model", required=True, help="model JSON path")
        p.add_argument("--profile", default="cpu-avx2", help="builtin profile name or JSON profile path")
        p.add_argument("--passes", default=None, help="comma-separated subset of re,dr,sor")

    p = sub.add_parser("compile", help="lower a model, print the fused device program")
    common(p)
    p.set_defaults(fn=cmd_compile)
    p = sub.add_parser("run", help="execute on a CSV batch on the GPU, write predictions")
    common(p)
    p.add_argument("--input", required=True)
    p.add_argument("--output", default=None)
    p.set_defaults(fn=cmd_run)
    p = sub.add_parser("verify", help="compare the GPU path against the reference's scalar oracle")
    common(p)
    p.add_argument("--input", default=None)
    p.add_argument("--random", type=int, default=1000)
    p.add_argument("--seed", type=int, default=0)
    p.set_defaults(fn=cmd_verify)
    return parser


def run_cli(argv) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        return args.fn(args)
    except MlowerError as e:
        sys.stderr.write(f"error: {e.code}: {e}\n")
        return 2


def main() -> None:
    sys.exit(run_cli(sys.argv[1:]))
