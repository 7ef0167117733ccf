"""Error taxonomy of the B200 path, code-for-code compatible with the reference.

Every class keeps the reference's stable ``code`` string (reference:
``pkg/src/mlower/errors.py:10-93``) so callers that print
``error: <code>: <detail>`` or switch on ``.code`` see no difference.  When the
reference package is importable, each class here also derives from the
same-named reference class, so ``except mlower.errors.InputMismatch`` keeps
catching errors raised by this package.

Native status codes returned by ``libcmlb.so`` (``include/cmlb.h``) map onto
these classes in :func:`error_for_status`.
"""

from __future__ import annotations

try:  # optional: reference installed next to us -> share the hierarchy
    import mlower.errors as _ref_errors  # type: ignore
except Exception:  # pragma: no cover - the GPU box has no reference
    _ref_errors = None


def _bases(name: str, *own):
    ref = getattr(_ref_errors, name, None) if _ref_errors is not None else None
    if ref is None:
        return own
    # a base the reference class already derives from (Exception) must not
    # precede it, or the MRO is inconsistent
    return tuple(b for b in own if not issubclass(ref, b)) + (ref,)


class MlowerError(*_bases("MlowerError", Exception)):
    """Root of the taxonomy; ``code`` is the machine-readable identifier."""

    code = "internal"


# (class name, code) in the order the reference declares them.
_TAXONOMY = (
    ("SchemaError", "schema"),
    ("ValidationError", "validation"),
    ("NarrowingCast", "narrowing-cast"),
    ("DTypeMismatch", "dtype-mismatch"),
    ("ShapeMismatch", "shape-mismatch"),
    ("BroadcastError", "broadcast"),
    ("DivisionByZero", "division-by-zero"),
    ("InvalidAxis", "invalid-axis"),
    ("EmptyAxis", "empty-axis"),
    ("IndexOutOfBounds", "index-out-of-bounds"),
    ("AccumulatorOverflowRisk", "accumulator-overflow"),
    ("CyclicGraph", "cyclic-graph"),
    ("DanglingReference", "dangling-reference"),
    ("UnresolvedKernel", "unresolved-kernel"),
    ("ShapeInferenceFailure", "shape-inference"),
    ("InputMismatch", "input-mismatch"),
    ("FeatureMismatch", "feature-mismatch"),
    ("ProfileError", "profile"),
    ("FileAccessError", "io"),
)

for _name, _code in _TAXONOMY:
    globals()[_name] = type(_name, _bases(_name, MlowerError), {"code": _code, "__module__": __name__})


class DeviceError(MlowerError):
    """CUDA / NCCL failure inside the native library (no reference analogue)."""

    code = "device"


# Status codes of include/cmlb.h -> exception class.
_STATUS = {
    1: "ValidationError",
    2: "ShapeMismatch",
    3: "IndexOutOfBounds",
    4: "AccumulatorOverflowRisk",
    5: "UnresolvedKernel",
    6: "InputMismatch",
    7: "DeviceError",
}


def error_for_status(status: int, detail: str) -> MlowerError:
    name = _STATUS.get(int(status), "MlowerError")
    cls = DeviceError if name == "DeviceError" else globals().get(name, MlowerError)
    return cls(detail)


__all__ = ["MlowerError", "DeviceError", "error_for_status"] + [n for n, _ in _TAXONOMY]
