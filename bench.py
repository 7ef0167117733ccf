"""Benchmarks of the BASELINE configs; the default is the north star.

    python bench.py [--config rf500|dt6|gbr1000|lr784|svc10k|pipe5] [--gpus N] [--steps K]
                    [--warmup W] [--impl ours|reference] [--rows R] [--variant ...]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Default (``--config rf500``): RandomForestClassifier 500 x depth-8 on 10M x 28
fp32 rows per GPU (BASELINE.json's metric and config 2).  One step = one pass
of the fused forest kernel (tree operator representation + ensemble tail,
``libcmlb.so``) over this rank's shard, inputs resident in HBM (1.12 GB per
step, larger than the 126 MB L2, so no flush is needed).  Ranks shard rows with
no data-path collective (weak scaling); ``value`` = rows of all ranks /
max-over-ranks device time.  ``--gpus N`` without a launcher starts the N
ranks itself.  ``e2e`` is the same metric through the public API from pinned
host memory, with the H2D copy of X and the D2H copy of the outputs inside the
timed region.  The other configs print the
same line for their own workload.

``roofline`` is the dominant kernel against the resource that bounds it:
  * forest walks (rf500, dt6, gbr1000, pipe5): shared-memory load wavefronts.
    ``achieved`` = ALGORITHMIC wavefronts per row (every node, rank and payload
    load of the walk and the ranking search at one wavefront per warp-wide
    conflict-free access) x the live rows/s; ``peak`` = the
    measured conflict-free wavefront rate (profiles/peaks_smem.json) x SMs x
    the sampled SM clock.  ``traffic`` = ncu-measured wavefronts per launch
    when a committed profile of the same kernel exists (conflict replays show
    up as traffic above the algorithmic count).  HBM and the reference's
    GEMM-equivalent int8 work are reported beside it (``hbm``, ``gemm_equivalent``).
  * lr784: HBM bytes (X read + labels written) against MEASURED_PEAKS.json.
  * svc10k: TF32 tensor flops (2 F n_SV per row) against the measured TF32 peak.

``--impl reference`` times the CPU restatement of the reference path (the
oracle: ``oracle/liboracle.so`` / numpy; the reference itself is pure Python,
25.8 rows/s on RF500) on a bounded row sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ASSET = os.path.join(ROOT, "bench_assets", "rf500_d8.npz")
METRIC = "samples/sec (RandomForest 500x d8, 10M x 28) at 1/2/4/8 B200; % roofline"


def load_model():
    from paper_2301_13441_b200.models import forest_from_node_arrays
    z = np.load(ASSET)
    m = forest_from_node_arrays(z["offsets"], z["is_leaf"], z["feature"], z["threshold"], z["left"],
                                z["right"], z["value"], z["classes"], int(z["n_features"]))
    return m, z["mu"], z["sigma"]


def gemm_equivalent_ops(model) -> int:
    """ops_row = sum_t 2 * I_t * L_t (the GEMM-form int8 work per row)."""
    tot = 0
    for t in model.trees:
        i = int((~t.arrays.is_leaf).sum())
        tot += 2 * i * (i + 1)
    return tot


def _json(path):
    p = os.path.join(ROOT, path)
    if os.path.exists(p):
        with open(p) as fh:
            return json.load(fh)
    return None


def peaks():
    out = {"source": {}}
    mp = _json("MEASURED_PEAKS.json")
    if mp:
        out["hbm_gbs"] = float(mp["hbm_gbs"])
        out["source"]["hbm"] = "MEASURED_PEAKS.json (measured copy)"
    else:
        out["hbm_gbs"] = 6650.0
        out["source"]["hbm"] = "fallback 6.65 TB/s (B200_PROFILING.md)"
    p8 = _json("profiles/peaks_int8.json")
    out["int8_tops"] = float(p8["int8_tops_burst"]) if p8 else 2.0 * float((mp or {}).get("bf16_tflops", 1590.0))
    out["source"]["int8"] = "profiles/peaks_int8.json (measured torch._int_mm 8192^3)" if p8 else "proxy 2x bf16"
    tf = _json("profiles/peaks_tf32.json")
    out["tf32_tflops"] = float(tf["tf32_tflops_burst"]) if tf else 1100.0
    out["source"]["tf32"] = "profiles/peaks_tf32.json (measured cuBLAS TF32)" if tf else "nominal 1.1 PF (guide)"
    sm = _json("profiles/peaks_smem.json")
    out["smem_wf_per_sm_clk"] = float(sm["wavefronts_per_sm_clk"]) if sm else 1.0
    out["source"]["smem"] = ("profiles/peaks_smem.json (measured conflict-free LDS wavefronts per SM per clock)"
                             if sm else "architectural 1 wavefront/clk/SM (not measured)")
    return out


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line).  NVML polled every 2 ms from a thread, so
    even a few-millisecond region (LR, DT6 configs) gets samples; nvidia-smi
    (-lms 50, first sample ~100 ms late) is the fallback."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, dev):
        self.dev = dev
        self.proc = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, reasons)
        self.stop = threading.Event()
        self.t = None

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        import torch
        p = torch.cuda.get_device_properties(self.dev)
        return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(
            f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0")

    def _sample(self):
        nv, h = self.nv
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        try:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), float(self.mx), {n for n, b in zip(self.NAMES, bits) if r & b}))
        except Exception:
            pass

    def _poll(self):
        while not self.stop.is_set():
            self._sample()
            self.stop.wait(0.002)

    def __enter__(self):
        try:
            self.nv = self._nvml_handle()
            self.mx = self.nv[0].nvmlDeviceGetMaxClockInfo(self.nv[1], self.nv[0].NVML_CLOCK_SM)
            # the launch loop holds the GIL; a short switch interval lets the
            # poller run during a few-millisecond region
            self.switch = sys.getswitchinterval()
            sys.setswitchinterval(1e-4)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.t = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.t is not None and self.proc is None:
            self._sample()  # the GPU finished the region microseconds ago
        self.stop.set()
        if self.proc is None and self.t is not None:
            sys.setswitchinterval(self.switch)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        elif self.t is not None:
            self.t.join(timeout=1)

    def summary(self):
        sm, mx, reasons = [], [], set()
        for a, b, r in self.samples:
            sm.append(a)
            mx.append(b)
            reasons |= r
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml 2 ms" if self.samples else "nvidia-smi 50 ms"}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


def _class_width(c: int) -> int:
    for w in (1, 2, 4, 8, 16):
        if c <= w:
            return w
    return 32


def _bucket_steps(u: np.ndarray) -> int:
    """Binary-lifting steps of one feature's bucket table (forest.cu
    build_rank_tables): B = 2n rounded up to a power of two (<= 8192) buckets
    over [u_0, u_n-1]; T = bits of the largest bucket count."""
    n = u.size
    B = 1
    while B < 8192 and B < 2 * n:
        B *= 2
    if n >= 2:
        s = np.float32(B) / (u[-1] - u[0])
        s = s if s < np.float32(1e30) else np.float32(1e30)
        c = np.float32(-u[0] * s)
        t = (u.astype(np.float64) * np.float64(s) + np.float64(c)).astype(np.float32)
        b = np.floor(np.clip(t, 0, B - 1)).astype(np.int64)
    else:
        b = np.zeros(n, np.int64)
    mx = int(np.bincount(b, minlength=B).max()) if n else 0
    return int(mx).bit_length()


def forest_wavefronts_row(spec, info) -> dict:
    """Algorithmic shared-memory wavefronts per row of the ranked/skew walk:
    per tree D node-word loads + D rank loads + the payload load (CT floats,
    CT wavefronts per warp of 32), per feature the bucket-table search (the
    start lookup + T_f binary-lifting steps, T_f from the same bucketing as
    forest.cu build_rank_tables; the ranks go to global memory), all at one
    wavefront per warp-wide conflict-free access, / 32 rows."""
    if info["variant"] not in ("ranked", "skew"):
        return None
    D = int(info["depth"])
    CT = _class_width(spec.n_outputs)
    T = len(spec.trees)
    T_walked = (T + 31) // 32 * 32 if info["variant"] == "skew" else T
    feats = np.concatenate([t.feature for t in spec.trees]) if T else np.zeros(0, np.int64)
    thr = np.concatenate([t.threshold for t in spec.trees]) if T else np.zeros(0, np.float32)
    search = 0
    for f in np.unique(feats):
        nf = np.unique(thr[feats == f]).size
        search += 1 + _bucket_steps(np.unique(thr[feats == f]).astype(np.float32))
    walk = T_walked * (2 * D + CT)
    return {"walk": walk / 32.0, "rank": search / 32.0, "total": (walk + search) / 32.0,
            "trees_walked": T_walked, "depth": D, "payload_floats": CT}


class Workload:
    name = ""
    metric = ""
    features = 0
    default_rows = 0
    out_bytes = 1

    def model(self):
        raise NotImplementedError

    def device_input(self, dev, rank: int, n: int):
        import torch
        g = torch.Generator(device=dev)
        g.manual_seed(self.seed + rank)
        return torch.randn((n, self.features), generator=g, device=dev, dtype=torch.float32)

    def config(self, n: int, world: int, info) -> dict:
        return {"workload": self.describe(n), "rows_per_gpu": n, "features": self.features,
                "parallelism": f"row-shard dp{world}",
                "l2": f"inputs {n * self.features * 4 / 1e9:.2f} GB per step vs 126 MB L2"
                      + (" (no flush needed)" if n * self.features * 4 > 126e6 else
                         " (inputs re-read from L2 between steps)")}

    def describe(self, n):
        return self.name

    def roofline(self, prog, spec, info, rows_per_s: float, kern_ms: float, n: int, pk, clocks, sms) -> dict:
        return None

    def parity(self, prog, x) -> dict:
        return None

    def cpu_baseline(self, x_sample: np.ndarray, threads: int):
        """(callable on a host array, description)."""
        raise NotImplementedError


class ForestWorkload(Workload):
    seed = 1
    variant = "auto"

    def describe(self, n):
        return f"{self.title} on {n} x {self.features} fp32 rows per GPU"

    def roofline(self, prog, spec, info, rows_per_s, kern_ms, n, pk, clocks, sms):
        model = self.model()
        bytes_row = self.features * 4 + self.out_bytes
        hbm = rows_per_s * bytes_row / 1e9
        ops_row = gemm_equivalent_ops(model) if hasattr(model, "trees") else None
        wf = forest_wavefronts_row(spec, info)
        mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
        out = {"kernel_ms": kern_ms}
        if wf is not None:
            peak = pk["smem_wf_per_sm_clk"] * sms * mhz * 1e6 / 1e9
            ach = rows_per_s * wf["total"] / 1e9
            traffic = None
            prof = _json(f"profiles/wavefronts_{self.name}_{info['variant']}.json")
            if prof:
                traffic = float(prof["wavefronts_per_row"]) * n
            out.update({"bound": "smem", "achieved": ach, "peak": peak, "unit": "Gwavefronts/s",
                        "frac": ach / peak, "traffic": traffic,
                        "traffic_unit": "shared-memory load wavefronts per launch (ncu, committed profile)",
                        "basis": f"algorithmic wavefronts per row = {wf['total']:.1f} ({info['variant']} walk "
                                 f"{wf['walk']:.1f} over {wf['trees_walked']} trees x depth {wf['depth']} + ranking "
                                 f"{wf['rank']:.1f}) x live rows/s; peak = measured rate x {sms} SMs x "
                                 f"{mhz:.0f} MHz sampled", "peak_source": pk["source"]["smem"],
                        "wavefronts_row": wf})
        else:
            out.update({"bound": "hbm", "achieved": hbm, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm / pk["hbm_gbs"], "traffic": None})
        out["hbm"] = {"achieved": hbm, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": hbm / pk["hbm_gbs"],
                      "bytes_row": bytes_row, "peak_source": pk["source"]["hbm"]}
        if ops_row:
            tops = rows_per_s * ops_row / 1e12
            out["gemm_equivalent"] = {
                "achieved": tops, "peak": pk["int8_tops"], "unit": "TOPS", "ratio": tops / pk["int8_tops"],
                "ops_row": ops_row, "peak_source": pk["source"]["int8"],
                "note": "informational: the reference's GEMM-form int8 work (sum_t 2 I_t L_t) the walk avoids; "
                        "a ratio above 1 means the walk does less work than the GEMM, not a roofline fraction"}
        return out

    def parity(self, prog, x):
        from oracle import fast  # checker only, outside the timed region
        model = self.model()
        k = min(int(x.shape[0]), 20_000)
        xs = x[:k]
        got = prog.run(xs).cpu().numpy().astype(np.float64)
        want, _ = fast.forest_predict(fast.PackedForest(model), xs.cpu().numpy())
        return {"rows": k, "bit_exact": bool(np.array_equal(got, want)), "oracle": "oracle/liboracle.so"}

    def cpu_baseline(self, x_sample, threads):
        from oracle import fast
        packed = fast.PackedForest(self.model())
        return (lambda xs: fast.forest_predict(packed, xs, threads=threads)), "oracle/liboracle.so (C restatement)"


class RF500(ForestWorkload):
    name = "rf500"
    metric = METRIC
    features = 28
    default_rows = 10_000_000
    title = "RandomForestClassifier 500 trees depth 8"

    def __init__(self):
        self._m = None

    def model(self):
        if self._m is None:
            self._m, self.mu, self.sigma = load_model()
        return self._m

    def device_input(self, dev, rank, n):
        import torch
        self.model()
        x = super().device_input(dev, rank, n)
        return x.mul_(torch.from_numpy(self.sigma).to(dev)).add_(torch.from_numpy(self.mu).to(dev))

    def config(self, n, world, info):
        c = super().config(n, world, info)
        c.update({"forest_source": "sklearn RF500 max_depth=8 fit on make_classification(200k x 28), "
                                   "bench_assets/rf500_d8.npz", "trees": 500})
        return c


class DT6(ForestWorkload):
    name = "dt6"
    metric = "samples/sec (DecisionTreeClassifier depth 6, 100k x 28)"
    features = 28
    default_rows = 100_000
    title = "DecisionTreeClassifier depth 6 (sklearn, make_classification 100k x 28)"
    seed = 11

    def model(self):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import golden_cases as gc
        return gc.get("sk_dt_d6").model

    def device_input(self, dev, rank, n):
        return super().device_input(dev, rank, n).mul_(2.0)

    def parity(self, prog, x):
        from oracle import semantics as sem  # single trees: the numpy restatement
        k = min(int(x.shape[0]), 20_000)
        got = prog.run(x[:k]).cpu().numpy().astype(np.float64)
        want, _ = sem.predict(self.model(), x[:k].cpu().numpy())
        return {"rows": k, "bit_exact": bool(np.array_equal(got, want)), "oracle": "oracle/semantics.py"}

    def cpu_baseline(self, x_sample, threads):
        from oracle import semantics as sem
        m = self.model()
        return (lambda xs: sem.predict(m, xs)), "oracle/semantics.py (numpy restatement of execute, 1 thread)"


class GBR1000(ForestWorkload):
    name = "gbr1000"
    metric = "samples/sec (GradientBoostingRegressor 1000x d10, 1M x 90)"
    features = 90
    default_rows = 1_000_000
    out_bytes = 4
    title = "GradientBoostingRegressor 1000 perfect depth-10 trees (SURVEY 8d throughput model)"
    seed = 2

    def __init__(self):
        self._m = None

    def model(self):
        if self._m is None:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from bench_configs import perfect_gbdt
            self._m = perfect_gbdt()
        return self._m


class Pipe5(ForestWorkload):
    name = "pipe5"
    metric = "samples/sec (StandardScaler + OneHotEncoder + RandomForest 500x d8, 5M x 64)"
    features = 64
    default_rows = 5_000_000
    title = "ColumnTransformer(StandardScaler 56 + OneHotEncoder 8 x 16) -> RF500 d8, fused"

    def __init__(self):
        self._m = None

    def _build(self, n):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from workloads import config5_pipeline
        self._m, self._x = config5_pipeline(rows=n)

    def model(self):
        if self._m is None:
            self._build(16)
        return self._m

    def device_input(self, dev, rank, n):
        import torch
        self._build(n)
        return torch.from_numpy(self._x).to(dev)

    def parity(self, prog, x):
        from oracle import ext_semantics as ext
        k = min(int(x.shape[0]), 5000)
        got = prog.run(x[:k]).cpu().numpy().astype(np.float64)
        want, _ = ext.predict(self.model(), x[:k].cpu().numpy())
        return {"rows": k, "bit_exact": bool(np.array_equal(got, want)),
                "oracle": "reference scaler semantics + scikit-learn one-hot + C forest oracle"}

    def cpu_baseline(self, x_sample, threads):
        from oracle import ext_semantics as ext, fast
        ct, forest = self.model().steps
        packed = fast.PackedForest(forest)
        return (lambda xs: fast.forest_predict(packed, ext.transform(ct, xs), threads=threads)), \
            "numpy column transform + oracle/liboracle.so forest"

    def roofline(self, prog, spec, info, rows_per_s, kern_ms, n, pk, clocks, sms):
        return super().roofline(prog, spec, info, rows_per_s, kern_ms, n, pk, clocks, sms)


class LR784(Workload):
    name = "lr784"
    metric = "samples/sec (LogisticRegression 784->10, 1M x 784)"
    features = 784
    default_rows = 1_000_000
    seed = 3

    def __init__(self):
        self._m = None

    def describe(self, n):
        return f"LogisticRegression 784 -> 10 classes on {n} x 784 fp32 rows per GPU"

    def model(self):
        if self._m is None:
            from paper_2301_13441_b200.models import LinearModel
            rng = np.random.default_rng(3)
            self._m = LinearModel(
                "logistic_regression", 784,
                tuple(tuple(float(v) for v in r) for r in rng.standard_normal((10, 784)).astype(np.float32) * 0.05),
                tuple(float(v) for v in rng.standard_normal(10).astype(np.float32)), tuple(float(c) for c in range(10)))
        return self._m

    def roofline(self, prog, spec, info, rows_per_s, kern_ms, n, pk, clocks, sms):
        bytes_row = 784 * 4 + 1
        gbs = rows_per_s * bytes_row / 1e9
        return {"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
                "traffic": None, "basis": f"algorithmic bytes per row {bytes_row} (X row read + int8 label)",
                "peak_source": pk["source"]["hbm"], "kernel_ms": kern_ms}

    def parity(self, prog, x):
        from oracle import semantics as sem
        k = min(int(x.shape[0]), 4000)
        got = prog.run(x[:k]).cpu().numpy().astype(np.float64)
        want, _ = sem.predict(self.model(), x[:k].cpu().numpy())
        return {"rows": k, "bit_exact": bool(np.array_equal(got, want)), "oracle": "oracle/semantics.py (numpy)"}

    def cpu_baseline(self, x_sample, threads):
        from oracle import semantics as sem
        m = self.model()
        return (lambda xs: sem.predict(m, xs)), "oracle/semantics.py (numpy float64 ascending-k, 1 thread)"


class SVC10k(Workload):
    name = "svc10k"
    metric = "samples/sec (SVC RBF 10k SVs, 1M x 784)"
    features = 784
    default_rows = 1_000_000
    seed = 3

    def __init__(self):
        self._m = None

    def describe(self, n):
        return f"SVC RBF, {self.model().n_sv} support vectors, 10 classes, on {n} x 784 fp32 rows per GPU"

    def model(self):
        if self._m is None:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from bench_configs import svc_model
            self._m = svc_model()
        return self._m

    def device_input(self, dev, rank, n):
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        from bench_configs import svc_inputs
        return svc_inputs(dev, rank, n)

    def roofline(self, prog, spec, info, rows_per_s, kern_ms, n, pk, clocks, sms):
        m = self.model()
        flops_row = 2.0 * m.n_features * m.n_sv
        tf = rows_per_s * flops_row / 1e12
        return {"bound": "tensor", "achieved": tf, "peak": pk["tf32_tflops"], "unit": "TFLOP/s",
                "frac": tf / pk["tf32_tflops"], "traffic": None,
                "basis": f"algorithmic Gram flops per row 2 F n_SV = {flops_row:.3g} (the tcgen05 kernel issues "
                         "3 split-TF32 products per term, 3x this on the tensor pipe)",
                "peak_source": pk["source"]["tf32"], "kernel_ms": kern_ms}

    def parity(self, prog, x):
        from oracle import ext_semantics as ext
        k = min(int(x.shape[0]), 2048)
        got = prog.run(x[:k]).cpu().numpy().astype(np.float64).ravel()
        _, vote = ext.svm_decision(self.model(), x[:k].cpu().numpy())
        want = np.asarray(self.model().classes)[vote]
        return {"rows": k, "bit_exact": bool(np.array_equal(got, want)), "oracle": "oracle/svm_oracle.c (libsvm order)"}

    def cpu_baseline(self, x_sample, threads):
        from oracle import ext_semantics as ext
        m = self.model()
        return (lambda xs: ext.svm_decision(m, xs, threads=threads)), "oracle/svm_oracle.c (libsvm order, C)"


WORKLOADS = {"rf500": RF500, "dt6": DT6, "gbr1000": GBR1000, "lr784": LR784, "svc10k": SVC10k, "pipe5": Pipe5}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm
# ---------------------------------------------------------------------------


def _host_sample(wl, n: int, seed: int) -> np.ndarray:
    """A host copy of the workload's input distribution (same generator family)."""
    import torch
    x = wl.device_input(torch.device("cpu"), seed, n) if not isinstance(wl, Pipe5) else None
    if x is None:
        wl._build(n)
        return wl._x
    return x.numpy()


def time_cpu(wl, target_s: float, threads: int, steps: int = 1, warmup: int = 0):
    """Run the oracle on a bounded host sample sized to ~target_s per step."""
    fn, what = wl.cpu_baseline(None, threads)
    cal = _host_sample(wl, 512, 97)
    t0 = time.perf_counter()
    fn(cal)
    rate = cal.shape[0] / max(time.perf_counter() - t0, 1e-6)
    n = int(min(max(rate * target_s, 256), 5_000_000))
    x = _host_sample(wl, n, 98)
    for _ in range(warmup):
        fn(x[: max(n // 10, 64)])
    t0 = time.perf_counter()
    for _ in range(steps):
        fn(x)
    dt = time.perf_counter() - t0
    return n, dt, what


def cpu_baseline(wl, threads: int, target_s: float = 10.0) -> dict:
    n, dt, what = time_cpu(wl, target_s, threads)
    return {"value": n / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{n} rows x {wl.features} of the workload's input distribution, {dt:.1f} s, {what}"}


def reference_json(model) -> str | None:
    """Our forest / linear model in the reference's model-JSON schema
    (``pkg/exporter/export.py:56-153``), for timing ``mlower`` itself."""
    def tree_nodes(t):
        a = t.arrays
        nodes = []
        for i in range(len(a.is_leaf)):
            if a.is_leaf[i]:
                nodes.append({"leaf": [float(v) for v in np.atleast_1d(a.value[i])]})
            else:
                nodes.append({"feature": int(a.feature[i]), "threshold": float(a.threshold[i]),
                              "left": int(a.left[i]), "right": int(a.right[i])})
        return nodes

    trees = getattr(model, "trees", None)
    if trees is None and hasattr(model, "arrays"):  # single decision tree
        obj = {"model_type": model.model_type, "n_features": int(model.n_features), "nodes": tree_nodes(model)}
        if getattr(model, "classes", None) is not None:
            obj["classes"] = [float(c) for c in model.classes]
        obj["format_version"] = 1
        return json.dumps(obj)
    if trees is not None:
        out = []
        for t in trees:
            a = t.arrays
            nodes = []
            for i in range(len(a.is_leaf)):
                if a.is_leaf[i]:
                    nodes.append({"leaf": [float(v) for v in np.atleast_1d(a.value[i])]})
                else:
                    nodes.append({"feature": int(a.feature[i]), "threshold": float(a.threshold[i]),
                                  "left": int(a.left[i]), "right": int(a.right[i])})
            out.append({"nodes": nodes})
        obj = {"model_type": model.model_type, "n_features": int(model.n_features), "trees": out,
               "aggregation": model.aggregation}
        if model.aggregation == "sum":
            obj.update(learning_rate=float(model.learning_rate), base_score=float(model.base_score))
        if model.classes is not None:
            obj["classes"] = [float(c) for c in model.classes]
    elif hasattr(model, "coef"):
        obj = {"model_type": model.model_type, "n_features": int(model.n_features),
               "coef": [[float(v) for v in r] for r in model.coef], "intercept": [float(v) for v in model.intercept]}
        if getattr(model, "classes", None) is not None:
            obj["classes"] = [float(c) for c in model.classes]
    else:
        return None
    obj["format_version"] = 1
    return json.dumps(obj)


def time_reference_itself(wl, target_s: float = 5.0):
    """The unmodified reference (``mlower``, installed offline in baseline/_ref
    by tools/install_reference.sh) on a bounded sample: compile once, then
    ``execute`` on as many rows as fit ~target_s of this host's time."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "mlower")):
        return {"unavailable": "reference not installed in baseline/_ref (tools/install_reference.sh)"}
    sys.path.insert(0, ref)
    try:
        import mlower
        from mlower.dtypes import DType
        from mlower.tensor import Tensor
        model = wl.model()
        text = reference_json(model) if not isinstance(wl, (Pipe5, SVC10k)) else None
        if text is None:
            return {"unavailable": "no reference model family for this workload (SPEC.md:9)"}
        compiled = mlower.compile_model(mlower.parse_model(text))
        x = _host_sample(wl, 64, 96).astype(np.float32)
        t0 = time.perf_counter()
        mlower.execute(compiled.plan, Tensor.from_dense(x, DType.FLOAT32))
        rate = 64 / max(time.perf_counter() - t0, 1e-6)
        n = int(min(max(rate * target_s, 64), 200_000))
        x = _host_sample(wl, n, 95).astype(np.float32)
        t0 = time.perf_counter()
        mlower.execute(compiled.plan, Tensor.from_dense(x, DType.FLOAT32))
        dt = time.perf_counter() - t0
        return {"value": n / dt, "unit": "samples/s", "cores": 1, "rows": n, "seconds": dt,
                "what": "mlower.execute (the unmodified reference, pure Python + numpy, one process)"}
    except Exception as e:  # report, never fail the arm
        return {"unavailable": f"{type(e).__name__}: {e}"}


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n, dt, what = time_cpu(wl, 5.0, threads, steps=args.steps, warmup=args.warmup)
    value = n * args.steps / dt
    line = {
        "impl": "reference", "metric": wl.metric, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl.describe(wl.default_rows) if not isinstance(wl, SVC10k) else wl.name,
                   "rows_per_step": n, "sample": "bounded host sample of the workload"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
                         "sample": f"{n} rows per step x {args.steps} steps, {what}"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_itself": time_reference_itself(wl),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


def launch_ranks(n: int, argv) -> int:
    """``--gpus N`` without a launcher: start the N ranks (one per GPU) under
    torch.distributed.run ourselves, as the driver would."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} but only {have} CUDA device(s) visible", file=sys.stderr, flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def init_dist(gpus: int):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="rf500", choices=list(WORKLOADS))
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager program runs instead of CUDA graph replays")
    ap.add_argument("--variant", default="auto", choices=["auto", "ranked", "skew", "perfect", "general", "mma"],
                    help="force a forest kernel variant (measurement; default: the measured AUTO choice)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    wl = WORKLOADS[args.config]()
    if args.impl == "reference":
        return run_reference(args, wl)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus, sys.argv[1:] if argv is None else argv)

    import torch
    import torch.distributed as dist

    from paper_2301_13441_b200 import _native as N
    from paper_2301_13441_b200 import api
    from paper_2301_13441_b200.runtime import DeviceProgram, run_host

    rank, world, local = init_dist(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    n = args.rows or wl.default_rows
    model = wl.model()
    compiled = api.compile_model(model)
    if args.variant == "auto":
        prog = compiled.program(dev.index)
    else:
        prog = DeviceProgram(compiled.spec, dev.index, forest_variant={
            "ranked": N.FOREST_RANKED, "skew": N.FOREST_SKEW, "perfect": N.FOREST_PERFECT,
            "general": N.FOREST_GENERAL, "mma": N.FOREST_MMA}[args.variant])
    fstage = next((st for st in prog.stages if hasattr(st, "info")), None)
    info = fstage.info() if fstage is not None else None
    fspec = fstage.spec if fstage is not None else None

    x = wl.device_input(dev, rank, n)
    y = torch.empty((n, prog.out_cols), dtype=prog_dtype(prog), device=dev)
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev) if prog.has_checks else None
    stream = torch.cuda.current_stream(dev)

    def step():
        prog.run(x, out=y, stream=stream, bad=bad)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # the timed steps replay one CUDA graph of the program (DeviceProgram.capture):
    # same kernels, one host call per step instead of the per-stage Python path
    graph_launches = None
    if not args.no_graph:
        try:
            graph, graph_launches = prog.capture(x, y, bad=bad)
            step = graph.replay  # noqa: F811
            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
        except Exception as e:  # capture unsupported for this program: eager steps
            print(f"bench: CUDA graph capture failed ({e}); timing eager runs", file=sys.stderr)
            graph_launches = None

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = N.lib().cmlb_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = N.lib().cmlb_launch_count() - launches0
    if graph_launches is not None:
        launches = graph_launches * args.steps  # replays bypass the library's launch counter
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * n * args.steps / (max_ms / 1e3)

    # ---- end to end through the public API: pinned host X -> outputs on host ----
    xh = x.cpu().pin_memory()
    yh = torch.empty((n, prog.out_cols), dtype=y.dtype).pin_memory()
    run_host(prog, xh[: 1 << 20], out_host=yh[: 1 << 20])  # warm the streams
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.e2e_steps):
        run_host(prog, xh, out_host=yh)
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * n * args.e2e_steps / (float(te.item()) / 1e3)
    same_as_device = bool(torch.equal(yh.to(dev), y))

    if rank == 0:
        pk = peaks()
        clocks = clk.summary()
        kern_ms = statistics.mean(kernel_ms)
        rows_per_s_kernel = n / (kern_ms / 1e3)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        roof = wl.roofline(prog, fspec, info, rows_per_s_kernel, kern_ms, n, pk, clocks, sms)
        cfg = wl.config(n, world, info)
        if info is not None:
            cfg.update({"variant": info["variant"], "chunk": info["chunk_trees"], "rows_per_cta": info["rows_per_cta"]})
        cfg["launch"] = "cuda-graph replay of the program" if graph_launches is not None else "eager program runs"
        line = {
            "metric": wl.metric, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": cfg, "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": n * wl.features * 4,
                    "d2h_bytes_per_step": n * prog.out_cols * y.element_size(), "steps": args.e2e_steps,
                    "same_as_device_path": same_as_device},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if not args.no_parity:
            line["parity"] = wl.parity(prog, x)
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(wl, os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def prog_dtype(prog):
    from paper_2301_13441_b200.runtime import TORCH_DTYPE
    return TORCH_DTYPE[prog.out_dtype]


if __name__ == "__main__":
    sys.exit(main())
