"""CUDA-stream executor: device programs built from lowered specs.

Replaces the reference's interpreter loop (``pkg/src/mlower/runtime.py:198-212``,
one numpy call per plan invocation, 3,005 of them for RF500) with one native
kernel per fused stage, enqueued on the caller's CUDA stream.  PyTorch is used
only for device memory (caching allocator), streams and pinned host buffers;
every byte of compute happens in ``libcmlb.so``.

Programs are immutable after construction and reentrant across streams (the
reference promises a pure, thread-safe ``execute``, ``runtime.py:199``).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _native as N
from .descs import compact_features, forest_desc  # noqa: F401  (re-exported)
from .dtypes import OUT_CODE
from .errors import DeviceError, InputMismatch, ValidationError
from .fuse import ColumnsSpec
from .lower import ForestSpec, LinearSpec, ProgramSpec, ScalerSpec, SVMSpec


def _prologue(spec, desc):
    """Attach a stage's fused-preprocessing ops to its descriptor; returns the
    buffer the caller keeps alive until create() returns."""
    if getattr(spec, "prologue", None) is None:
        desc.prologue, desc.n_inputs = None, 0
        return None
    ops = np.ascontiguousarray(spec.prologue)
    desc.prologue, desc.n_inputs = ops.ctypes.data, int(spec.n_inputs)
    return ops

TORCH_DTYPE = {
    "bool": torch.uint8, "int8": torch.int8, "int16": torch.int16, "int32": torch.int32,
    "float32": torch.float32,
}


class _Forest:
    def __init__(self, spec: ForestSpec, device: int, variant: int = N.FOREST_AUTO):
        self.spec = spec
        d, keep = forest_desc(spec, variant)
        h = N.c_vp()
        N.check(N.lib().cmlb_forest_create(C.byref(d), device, C.byref(h)))
        del keep
        self.handle = h
        self.n_trees = len(spec.trees)

    def info(self) -> dict:
        v, dep, ch, rows = (N.c_i32() for _ in range(4))
        N.check(N.lib().cmlb_forest_info(self.handle, C.byref(v), C.byref(dep), C.byref(ch), C.byref(rows)))
        return {"variant": {1: "perfect", 2: "general", 3: "ranked", 4: "mma", 5: "skew"}[v.value], "depth": dep.value,
                "chunk_trees": ch.value, "rows_per_cta": rows.value}

    def run(self, x, y, n, ldx, stream, leaf_out=None):
        lp = leaf_out.data_ptr() if leaf_out is not None else None
        N.check(N.lib().cmlb_forest_run(self.handle, x.data_ptr(), n, ldx, y.data_ptr(), lp, stream))

    def partial(self, x, out, n, ldx, stream):
        N.check(N.lib().cmlb_forest_partial(self.handle, x.data_ptr(), n, ldx, out.data_ptr(), stream))

    def merge(self, dst, src, n, stream):
        N.check(N.lib().cmlb_forest_merge(self.handle, dst.data_ptr(), src.data_ptr(), n, stream))

    def finish(self, partials, n_shards, merges, n, y, stream):
        m = np.ascontiguousarray(np.asarray(merges, np.int32).reshape(-1))
        N.check(N.lib().cmlb_forest_finish(self.handle, partials.data_ptr(), n_shards,
                                           m.ctypes.data_as(C.POINTER(N.c_i32)), len(merges), n,
                                           y.data_ptr(), stream))

    def close(self):
        if self.handle:
            N.lib().cmlb_forest_destroy(self.handle)
            self.handle = None


class _Linear:
    def __init__(self, spec: LinearSpec, device: int):
        self.spec = spec
        coef = np.ascontiguousarray(spec.coef, np.float32)
        b = np.ascontiguousarray(spec.intercept, np.float32)
        classes = np.ascontiguousarray(np.asarray(spec.classes, np.float64))
        d = N.LinearDesc()
        d.n_features, d.n_outputs = coef.shape[1], coef.shape[0]
        d.coef, d.intercept = N.ptr(coef, N.c_f32), N.ptr(b, N.c_f32)
        d.tail = spec.tail
        d.classes, d.n_classes = N.ptr(classes, N.c_f64), len(spec.classes)
        d.out_dtype = OUT_CODE[spec.out_dtype]
        d.sparse_coef = int(spec.sparse_coef)
        pro = _prologue(spec, d)
        h = N.c_vp()
        N.check(N.lib().cmlb_linear_create(C.byref(d), device, C.byref(h)))
        del pro
        self.handle = h

    def run(self, x, y, n, ldx, stream, leaf_out=None):
        N.check(N.lib().cmlb_linear_run(self.handle, x.data_ptr(), n, ldx, y.data_ptr(), stream))

    def close(self):
        if self.handle:
            N.lib().cmlb_linear_destroy(self.handle)
            self.handle = None


class _Scaler:
    def __init__(self, spec: ScalerSpec, device: int):
        self.spec = spec
        a = np.ascontiguousarray(spec.a if spec.a is not None else np.zeros(1), np.float32)
        b = np.ascontiguousarray(spec.b if spec.b is not None else np.zeros(1), np.float32)
        d = N.ScalerDesc()
        d.kind, d.n_features, d.threshold = spec.kind, spec.n_features, spec.threshold
        d.a, d.b = N.ptr(a, N.c_f32), N.ptr(b, N.c_f32)
        h = N.c_vp()
        N.check(N.lib().cmlb_scaler_create(C.byref(d), device, C.byref(h)))
        self.handle = h

    def run(self, x, y, n, ldx, stream, leaf_out=None):
        N.check(N.lib().cmlb_scaler_run(self.handle, x.data_ptr(), n, ldx, y.data_ptr(), stream))

    def close(self):
        if self.handle:
            N.lib().cmlb_scaler_destroy(self.handle)
            self.handle = None


class _SVM:
    def __init__(self, spec: SVMSpec, device: int):
        self.spec = spec
        m = spec.model
        sv = np.ascontiguousarray(m.support_vectors, np.float32)
        coef = np.ascontiguousarray(m.dual_coef, np.float32)
        ic = np.ascontiguousarray(m.intercept, np.float32)
        svr = m.model_type == "svr"
        ns = np.ascontiguousarray(np.asarray(m.n_support if not svr else (0,), np.int32))
        classes = np.ascontiguousarray(np.asarray(m.classes if not svr else (0.0,), np.float64))
        d = N.SVMDesc()
        d.n_features, d.n_sv, d.kernel, d.degree = m.n_features, sv.shape[0], N.SVM_KERNEL[m.kernel], int(m.degree)
        d.gamma, d.coef0 = float(m.gamma), float(m.coef0)
        d.support_vectors, d.dual_coef, d.intercept = N.ptr(sv, N.c_f32), N.ptr(coef, N.c_f32), N.ptr(ic, N.c_f32)
        d.n_support = N.ptr(ns, N.c_i32) if not svr else None
        d.n_classes = 0 if svr else len(m.classes)
        d.classes = N.ptr(classes, N.c_f64)
        d.out_dtype = OUT_CODE[spec.out_dtype]
        pro = _prologue(spec, d)
        h = N.c_vp()
        N.check(N.lib().cmlb_svm_create(C.byref(d), device, C.byref(h)))
        del pro
        self.handle = h
        self.pairs = 1 if svr else len(m.classes) * (len(m.classes) - 1) // 2

    def run(self, x, y, n, ldx, stream, leaf_out=None, decision=None, exact_rows=None):
        dp = decision.data_ptr() if decision is not None else None
        ep = exact_rows.data_ptr() if exact_rows is not None else None
        N.check(N.lib().cmlb_svm_run(self.handle, x.data_ptr(), n, ldx, y.data_ptr(), dp, ep, stream))

    def close(self):
        if self.handle:
            N.lib().cmlb_svm_destroy(self.handle)
            self.handle = None


class _Columns:
    """One-hot / column-transformer / scaler column map; check-only when its ops
    run fused inside the next stage."""

    def __init__(self, spec: ColumnsSpec, device: int):
        self.spec = spec
        ops = np.ascontiguousarray(spec.ops)
        cols = np.ascontiguousarray([c for c, _ in spec.checks] or [0], np.int32)
        off = np.zeros(len(spec.checks) + 1, np.int64)
        for i, (_, v) in enumerate(spec.checks):
            off[i + 1] = off[i] + len(v)
        vals = np.ascontiguousarray(np.concatenate([v for _, v in spec.checks]) if spec.checks else np.zeros(1),
                                    np.float32)
        d = N.ColumnsDesc()
        d.n_inputs, d.n_outputs, d.ops = spec.n_inputs, int(ops.shape[0]), ops.ctypes.data
        d.n_checks = len(spec.checks)
        d.check_col, d.check_offset, d.check_values = N.ptr(cols, N.c_i32), N.ptr(off, N.c_i64), N.ptr(vals, N.c_f32)
        h = N.c_vp()
        N.check(N.lib().cmlb_columns_create(C.byref(d), device, C.byref(h)))
        self.handle = h

    def run(self, x, y, n, ldx, stream, leaf_out=None, bad=None):
        yp = y.data_ptr() if y is not None else None
        bp = bad.data_ptr() if bad is not None else None
        N.check(N.lib().cmlb_columns_run(self.handle, x.data_ptr(), n, ldx, yp, bp, stream))

    def close(self):
        if self.handle:
            N.lib().cmlb_columns_destroy(self.handle)
            self.handle = None


def raise_unknown_category(bad: torch.Tensor, x_rows_offset: int = 0) -> None:
    """Raise as OneHotEncoder.transform does when a checked row held an unknown value."""
    r = int(bad.item())
    if r >= 0:
        raise ValidationError(f"Found unknown categories in row {r + x_rows_offset} during transform "
                              "(OneHotEncoder handle_unknown='error')")


_BUILDERS = {ForestSpec: _Forest, LinearSpec: _Linear, ScalerSpec: _Scaler, SVMSpec: _SVM, ColumnsSpec: _Columns}


class DeviceProgram:
    """A lowered program resident on one GPU."""

    def __init__(self, spec: ProgramSpec, device: int | None = None, forest_variant: int = N.FOREST_AUTO):
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.spec = spec
        self._lock = threading.Lock()
        with torch.cuda.device(self.device):
            self.stages = []
            for st in spec.stages:
                if isinstance(st, ForestSpec):
                    self.stages.append(_Forest(st, self.device, forest_variant))
                else:
                    self.stages.append(_BUILDERS[type(st)](st, self.device))
        self.n_features = spec.n_features
        self.out_cols = spec.out_cols
        self.out_dtype = spec.out_dtype

    # -- device path ---------------------------------------------------------------
    def check_input(self, x: torch.Tensor) -> None:
        if x.dim() != 2 or x.shape[1] != self.n_features:
            raise InputMismatch(f"input shape {tuple(x.shape)} does not match (batch, {self.n_features})")
        if x.dtype != torch.float32:
            raise InputMismatch(f"input dtype {x.dtype} != float32")

    def run(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None,
            leaf_out: torch.Tensor | None = None, bad: torch.Tensor | None = None) -> torch.Tensor:
        """Run on a CUDA tensor (N, F) float32 with unit column stride.

        One-hot membership checks write the first offending row into ``bad``
        (device int64) when given -- the caller raises after its own sync;
        otherwise this call synchronises and raises ``ValidationError``."""
        self.check_input(x)
        if not x.is_cuda or x.device.index != self.device:
            raise InputMismatch(f"input on {x.device}, program on cuda:{self.device}")
        if x.stride(1) != 1:
            x = x.contiguous()
        n = int(x.shape[0])
        # the program's device first, then its stream: intermediates are
        # allocated on (and so recycled in order with) the stream that uses them
        with torch.cuda.device(self.device):
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            sh = int(stream.cuda_stream)
            with torch.cuda.stream(stream):
                return self._run_stages(x, n, out, stream, sh, leaf_out, bad)

    def _run_stages(self, x, n, out, stream, sh, leaf_out, bad):
        own_bad = None
        if self.has_checks and bad is None:
            bad = own_bad = torch.full((1,), -1, dtype=torch.int64, device=x.device)
        cur, ld = x, int(x.stride(0)) if n > 0 else self.n_features
        for i, st in enumerate(self.stages):
            last = i == len(self.stages) - 1
            spec = st.spec
            if isinstance(spec, ColumnsSpec) and not spec.emit:
                st.run(cur, None, n, max(ld, 1), sh, bad=bad)  # membership check only
                continue
            cols = spec.out_cols
            dt = TORCH_DTYPE[spec.out_dtype]
            y = out if last and out is not None else torch.empty((n, cols), dtype=dt, device=x.device)
            if isinstance(spec, ColumnsSpec):
                st.run(cur, y if n > 0 else None, n, max(ld, 1), sh, bad=bad if spec.checks else None)
            elif n > 0:
                st.run(cur, y, n, max(ld, 1), sh, leaf_out if last else None)
            cur, ld = y, cols
        if own_bad is not None:
            stream.synchronize()
            raise_unknown_category(own_bad)
        return cur

    def capture(self, x: torch.Tensor, out: torch.Tensor, bad: torch.Tensor | None = None):
        """Record one ``run(x -> out)`` as a CUDA graph and return it
        (``torch.cuda.CUDAGraph``; ``.replay()`` launches the whole program with
        one call -- for small batches the per-call host work otherwise exceeds
        the kernels).  The graph keeps reading ``x`` and writing ``out`` (and
        ``bad``, required when the program has membership checks, since a
        capture cannot synchronise); refill ``x`` in place between replays.
        Returns (graph, launches): launches = kernels of one replay."""
        self.check_input(x)
        if self.has_checks and bad is None:
            raise ValidationError("capture of a program with membership checks needs a bad-row slot")
        with torch.cuda.device(self.device):
            side = torch.cuda.Stream(device=torch.device("cuda", self.device))
            side.wait_stream(torch.cuda.current_stream(self.device))
            self.run(x, out=out, stream=side, bad=bad)  # warm: kernel attributes, pools
            side.synchronize()
            g = torch.cuda.CUDAGraph()
            n0 = N.lib().cmlb_launch_count()
            with torch.cuda.graph(g, stream=side):
                self.run(x, out=out, stream=torch.cuda.current_stream(self.device), bad=bad)
            launches = N.lib().cmlb_launch_count() - n0
        return g, int(launches)

    @property
    def has_checks(self) -> bool:
        return any(isinstance(st.spec, ColumnsSpec) and st.spec.checks for st in self.stages)

    def forest(self) -> _Forest:
        if len(self.stages) != 1 or not isinstance(self.stages[0], _Forest):
            raise DeviceError("program is not a single forest")
        return self.stages[0]

    def close(self):
        for st in self.stages:
            st.close()
        self.stages = []

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_HOST_STREAMS: dict = {}  # (device, count) -> streams reused by run_host (creating them cost ~0.1 ms per call)
_HOST_STREAMS_LOCK = threading.Lock()


def _host_streams(device: int, count: int) -> list:
    key = (device, count)
    with _HOST_STREAMS_LOCK:
        st = _HOST_STREAMS.get(key)
        if st is None:
            st = [torch.cuda.Stream(device=torch.device("cuda", device)) for _ in range(count)]
            _HOST_STREAMS[key] = st
    return st


def run_host(program: DeviceProgram, x_host: torch.Tensor, chunk_rows: int = 1 << 18,
             out_host: torch.Tensor | None = None, n_streams: int = 3) -> torch.Tensor:
    """Host (N, F) float32 -> host output, H2D / compute / D2H pipelined in
    row chunks over ``n_streams`` streams so transfers overlap the kernels.
    Defaults measured on B200 for RF500 (tools/e2e_probe.py): 256K-row chunks
    on 3 streams reach 473M rows/s, 96% of the 55 GB/s pinned H2D copy rate."""
    program.check_input(x_host)
    n = int(x_host.shape[0])
    dt = TORCH_DTYPE[program.out_dtype]
    if out_host is None:
        out_host = torch.empty((n, program.out_cols), dtype=dt, pin_memory=x_host.is_pinned())
    if n == 0:
        return out_host
    dev = torch.device("cuda", program.device)
    with torch.cuda.device(program.device):
        streams = _host_streams(program.device, n_streams)
        rows = min(chunk_rows, n)
        xbuf = [torch.empty((rows, program.n_features), dtype=torch.float32, device=dev) for _ in streams]
        ybuf = [torch.empty((rows, program.out_cols), dtype=dt, device=dev) for _ in streams]
        nchunks = (n + rows - 1) // rows
        bads = torch.full((nchunks,), -1, dtype=torch.int64, device=dev) if program.has_checks else None
        cur = torch.cuda.current_stream(dev)
        for s in streams:
            s.wait_stream(cur)
        for i, r0 in enumerate(range(0, n, rows)):
            k = i % n_streams
            s = streams[k]
            r1 = min(n, r0 + rows)
            with torch.cuda.stream(s):
                xb = xbuf[k][: r1 - r0]
                xb.copy_(x_host[r0:r1], non_blocking=True)
                program.run(xb, out=ybuf[k][: r1 - r0], stream=s,
                            bad=bads[i:i + 1] if bads is not None else None)
                out_host[r0:r1].copy_(ybuf[k][: r1 - r0], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        for s in streams:
            s.synchronize()
        if bads is not None:
            b = bads.cpu().numpy()
            hit = np.flatnonzero(b >= 0)
            if hit.size:
                raise_unknown_category(torch.tensor(int(b[hit[0]]) + int(hit[0]) * rows))
    return out_host
