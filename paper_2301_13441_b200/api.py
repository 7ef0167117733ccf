"""Public API: the reference's ``compile_model`` / ``predict`` / ``execute``.

Signatures follow ``pkg/src/mlower/pipeline.py:31-48`` and
``pkg/src/mlower/runtime.py:198-212``:

    compile_model(model, profile=cpu-avx2, passes=("re", "dr", "sor")) -> CompileResult
    predict(compiled, x) -> Tensor
    execute(plan, x) -> Tensor

and so do their contracts: ``x`` must be rank 2 with ``n_features`` columns
and dtype float32 (else ``InputMismatch``, ``runtime.py:200-205``); the output
has the reference's shape and dtype; zero-row batches flow through; results
are deterministic and batch-invariant.

What differs is where the work runs.  ``execute`` accepts a reference
``KernelPlan`` unchanged (``lower.lower_plan`` inverts its tensor encodings),
``compile_model`` lowers the model directly; either way one fused sm_100a
kernel per operator representation runs on the GPU.  Inputs may be

* a reference ``Tensor`` / our :class:`~.tensor.Tensor` / numpy array
  (host): copied in, computed, copied out, returned as the same family;
* a CUDA ``torch.Tensor``: computed in place on its device and stream, the
  result stays on the device (uint8 for BOOL outputs);
* a CPU ``torch.Tensor`` (ideally pinned): streamed through the GPU in
  overlapped chunks, result returned as a CPU tensor.

``predict(..., devices=[0, 1, ...])`` / ``execute(..., devices=...)`` shard the
batch by rows over several GPUs of this process (one program replica per GPU,
no collective); the reference requires this to be bit-transparent
(``SPEC.md:574``), and it is: every row is computed by the same kernel
whatever shard it lands in, and the pieces are concatenated in row order.
"""

from __future__ import annotations

import threading
import warnings
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from .dtypes import name_of
from .errors import InputMismatch, ValidationError
from .lower import DEFAULT_PASSES, ProgramSpec, lower_model, lower_plan
from .models import parse_model
from .runtime import DeviceProgram, run_host
from .tensor import Tensor, wrap_like

DEFAULT_TOLERANCE = 1e-5
DEFAULT_PROFILE = "cpu-avx2"


@dataclass(frozen=True, eq=False)
class CompileResult:
    """Mirror of the reference ``CompileResult`` (``pipeline.py:22-28``).

    ``plan`` is the reference plan when compiled from one (``from_plan``);
    ``spec`` is the lowered fused program description; device programs are
    built lazily per GPU and cached here.
    """

    model: object
    spec: ProgramSpec
    profile: object = DEFAULT_PROFILE
    passes: tuple = DEFAULT_PASSES
    plan: object = None

    def program(self, device: int | None = None) -> DeviceProgram:
        return _program_for(self, device)


_cache_lock = threading.Lock()
_programs: dict = {}   # (id(owner), device) -> DeviceProgram
_plan_specs: dict = {}  # id(plan) -> ProgramSpec


def _evict(key_id: int) -> None:
    # drop the cache entries only: a caller may still hold the DeviceProgram,
    # which frees its device tables itself when it is collected
    with _cache_lock:
        for k in [k for k in _programs if k[0] == key_id]:
            _programs.pop(k)
        _plan_specs.pop(key_id, None)


def _device_of(device) -> int:
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, torch.device):
        return device.index if device.index is not None else torch.cuda.current_device()
    return int(device)


def _program_for(owner, device=None, spec: ProgramSpec | None = None) -> DeviceProgram:
    dev = _device_of(device)
    key = (id(owner), dev)
    with _cache_lock:
        prog = _programs.get(key)
        if prog is not None:
            return prog
    prog = DeviceProgram(spec if spec is not None else owner.spec, dev)
    with _cache_lock:
        if key in _programs:  # lost a race; keep the first
            prog.close()
            return _programs[key]
        _programs[key] = prog
        weakref.finalize(owner, _evict, id(owner))
    return prog


def compile_model(model, profile=DEFAULT_PROFILE, passes=DEFAULT_PASSES) -> CompileResult:
    """Lower ``model`` (ours, the reference's, or model JSON text) to a fused program."""
    if isinstance(model, str):
        model = parse_model(model)
    passes = tuple(passes)
    unknown = set(passes) - set(DEFAULT_PASSES)
    if unknown:
        raise ValidationError(f"unknown pass flags: {sorted(unknown)}")
    return CompileResult(model=model, spec=lower_model(model, profile, passes), profile=profile,
                         passes=passes)


def from_plan(plan, model=None) -> CompileResult:
    """Wrap a reference KernelPlan (e.g. ``mlower.compile_model(m).plan``)."""
    return CompileResult(model=model, spec=_spec_of_plan(plan), plan=plan)


def _spec_of_plan(plan) -> ProgramSpec:
    with _cache_lock:
        spec = _plan_specs.get(id(plan))
    if spec is None:
        spec = lower_plan(plan)
        with _cache_lock:
            _plan_specs[id(plan)] = spec
        weakref.finalize(plan, _evict, id(plan))
    return spec


# -- input handling ---------------------------------------------------------------


def _host_array(x):
    """numpy view of a host input, with the reference's InputMismatch checks."""
    if isinstance(x, np.ndarray):
        arr = x
    elif hasattr(x, "to_numpy") and hasattr(x, "dtype"):
        if name_of(x.dtype) != "float32":
            raise InputMismatch(f"input dtype {name_of(x.dtype)} != float32")
        arr = x.to_numpy()
    else:
        raise InputMismatch(f"unsupported input type {type(x).__name__}")
    if arr.ndim != 2:
        raise InputMismatch(f"input shape {arr.shape} is not rank 2")
    if arr.dtype != np.float32:
        raise InputMismatch(f"input dtype {arr.dtype} != float32")
    return arr


def _run(owner, spec_getter, x, device=None):
    if isinstance(x, torch.Tensor):
        dev = x.device.index if x.is_cuda else device
        prog = _program_for(owner, dev, spec_getter())
        if x.is_cuda:
            return prog.run(x)
        return run_host(prog, x)
    arr = _host_array(x)
    prog = _program_for(owner, device, spec_getter())
    if arr.shape[1] != prog.n_features:
        raise InputMismatch(f"input shape {arr.shape} does not match (batch, {prog.n_features})")
    with warnings.catch_warnings():  # read-only host arrays are only read
        warnings.simplefilter("ignore", UserWarning)
        xt = torch.from_numpy(np.ascontiguousarray(arr))
    out = run_host(prog, xt)
    values = out.numpy()
    if prog.out_dtype == "bool":
        values = values.astype(np.uint8)
    if isinstance(x, np.ndarray):
        return values
    return wrap_like(x, values, prog.out_dtype)


def _run_sharded(owner, spec_getter, x, devices):
    """Row-shard one batch over ``devices`` (threads: one per device, so the
    host copies and kernels of all shards overlap).  Same input/output
    families as :func:`_run`."""
    from concurrent.futures import ThreadPoolExecutor

    from .shard import row_range

    devices = [_device_of(d) for d in devices]
    if not devices:
        raise ValidationError("devices must name at least one GPU")
    if len(devices) == 1:
        return _run(owner, spec_getter, x, devices[0])
    host_wrap = None
    if isinstance(x, torch.Tensor):
        xt = x
    else:
        arr = _host_array(x)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            xt = torch.from_numpy(np.ascontiguousarray(arr))
        host_wrap = x
    progs = [_program_for(owner, d, spec_getter()) for d in devices]
    progs[0].check_input(xt)
    n = int(xt.shape[0])
    ranges = [row_range(n, r, len(devices)) for r in range(len(devices))]

    def piece(i):
        lo, hi = ranges[i]
        prog, dev = progs[i], devices[i]
        if xt.is_cuda:
            with torch.cuda.device(dev):
                xs = xt[lo:hi].to(torch.device("cuda", dev), non_blocking=True)
                y = prog.run(xs)
                torch.cuda.current_stream(dev).synchronize()
                return y
        return run_host(prog, xt[lo:hi])

    with ThreadPoolExecutor(max_workers=len(devices)) as pool:
        outs = list(pool.map(piece, range(len(devices))))
    if xt.is_cuda:
        return torch.cat([o.to(xt.device) for o in outs], dim=0)
    out = torch.cat(outs, dim=0)
    if host_wrap is None:
        return out
    values = out.numpy()
    if progs[0].out_dtype == "bool":
        values = values.astype(np.uint8)
    if isinstance(host_wrap, np.ndarray):
        return values
    return wrap_like(host_wrap, values, progs[0].out_dtype)


def execute(plan, x, device=None, devices=None):
    """Run a reference ``KernelPlan`` on the GPU; drop-in for ``mlower.execute``."""
    if devices is not None:
        return _run_sharded(plan, lambda: _spec_of_plan(plan), x, devices)
    return _run(plan, lambda: _spec_of_plan(plan), x, device)


def predict(compiled, x, device=None, devices=None):
    """Drop-in for ``mlower.predict``; also accepts a reference CompileResult.
    ``devices``: row-shard the batch over these GPUs (bit-transparent)."""
    if isinstance(compiled, CompileResult):
        if devices is not None:
            return _run_sharded(compiled, lambda: compiled.spec, x, devices)
        return _run(compiled, lambda: compiled.spec, x, device)
    plan = getattr(compiled, "plan", None)
    if plan is None:
        raise ValidationError("predict() needs a CompileResult")
    return execute(plan, x, device, devices)


__all__ = ["CompileResult", "compile_model", "from_plan", "predict", "execute", "DEFAULT_TOLERANCE",
           "Tensor"]
