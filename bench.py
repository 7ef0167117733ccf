"""North-star benchmark: RandomForestClassifier 500 x depth-8 on 10M x 28 fp32 rows per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--rows R]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

One step = one pass of the fused forest kernel (tree operator representation
+ ensemble tail, ``libcmlb.so``) over this rank's 10M-row shard, inputs
resident in HBM (1.12 GB per step, larger than the 126 MB L2, so no flush is
needed).  Ranks shard rows with no data-path collective (weak scaling);
``value`` = rows of all ranks / max-over-ranks device time.  ``e2e`` is the
same metric through the public API from pinned host memory, with the H2D copy
of X and the D2H copy of the class labels inside the timed region.

``--impl reference`` times the CPU restatement of the reference path
(``oracle/liboracle.so``, all host threads) on a bounded row sample per step;
the reference itself (``mlower``, pure Python, 25.8 rows/s measured in
SURVEY 6) is not on the GPU box.
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
BYTES_ROW = 28 * 4 + 1      # X row in, uint8 class out


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


def peaks():
    out = {"hbm_gbs": None, "int8_tops": None, "source": {}}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            mp = json.load(fh)
        out["hbm_gbs"] = float(mp["hbm_gbs"])
        out["source"]["hbm"] = "MEASURED_PEAKS.json (measured copy)"
        bf16 = float(mp["bf16_tflops"])
    except Exception:
        out["hbm_gbs"] = 6650.0
        out["source"]["hbm"] = "fallback 6.65 TB/s (B200_PROFILING.md)"
        bf16 = 1590.0
    p8 = os.path.join(ROOT, "profiles", "peaks_int8.json")
    if os.path.exists(p8):
        with open(p8) as fh:
            d = json.load(fh)
        out["int8_tops"] = float(d["int8_tops_burst"])
        out["source"]["int8"] = "profiles/peaks_int8.json (measured torch._int_mm 8192^3)"
    else:
        out["int8_tops"] = 2.0 * bf16
        out["source"]["int8"] = "proxy 2x measured bf16 (int8 not measured)"
    return out


class ClockSampler:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
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
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(model, mu, sigma, target_s: float = 10.0):
    """C oracle on this host's cores over a bounded sample of the workload."""
    from oracle import fast
    packed = fast.PackedForest(model)
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(11)
    cal = (rng.standard_normal((2000, 28)) * sigma + mu).astype(np.float32)
    t0 = time.perf_counter()
    fast.forest_predict(packed, cal, threads=threads)
    rate = 2000 / max(time.perf_counter() - t0, 1e-6)
    n = int(min(max(rate * target_s, 4000), 5_000_000))
    x = (rng.standard_normal((n, 28)) * sigma + mu).astype(np.float32)
    t0 = time.perf_counter()
    fast.forest_predict(packed, x, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{n} rows x 28 (randn*sigma+mu), {dt:.1f} s, oracle/liboracle.so "
                      f"(C restatement of mlower execute semantics)"}


def launch_ranks(n: int, argv) -> int:
    """``--gpus N`` without a launcher: start N ranks (one per GPU) under
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


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import fast
    model, mu, sigma = load_model()
    packed = fast.PackedForest(model)
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(1)
    # size one step to ~5 s of host work
    cal = (rng.standard_normal((2000, 28)) * sigma + mu).astype(np.float32)
    t0 = time.perf_counter()
    fast.forest_predict(packed, cal, threads=threads)
    rate = 2000 / max(time.perf_counter() - t0, 1e-6)
    n = int(min(max(rate * 5.0, 4000), 5_000_000))
    x = (rng.standard_normal((n, 28)) * sigma + mu).astype(np.float32)
    for _ in range(args.warmup):
        fast.forest_predict(packed, x[: max(n // 10, 1000)], threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fast.forest_predict(packed, x, threads=threads)
    dt = time.perf_counter() - t0
    value = n * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "RandomForestClassifier 500 trees depth 8, x28 fp32 rows",
                   "rows_per_step": n, "sample": "bounded host sample of the 10M-row workload"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
                         "sample": f"{n} rows per step x {args.steps} steps, oracle/liboracle.so"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", default="auto", choices=["auto", "ranked", "skew", "perfect", "general", "mma"],
                    help="force a forest kernel variant (measurement; default: the measured AUTO choice)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus, sys.argv[1:] if argv is None else argv)

    import torch
    import torch.distributed as dist

    from paper_2301_13441_b200 import _native as N
    from paper_2301_13441_b200 import api
    from paper_2301_13441_b200.runtime import run_host

    rank, world, local = init_dist(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    model, mu, sigma = load_model()
    compiled = api.compile_model(model)
    if args.variant == "auto":
        prog = compiled.program(dev.index)
    else:
        from paper_2301_13441_b200.runtime import DeviceProgram
        prog = DeviceProgram(compiled.spec, dev.index, forest_variant={
            "ranked": N.FOREST_RANKED, "skew": N.FOREST_SKEW, "perfect": N.FOREST_PERFECT, "general": N.FOREST_GENERAL,
            "mma": N.FOREST_MMA}[args.variant])
    info = prog.forest().info()
    n = args.rows

    g = torch.Generator(device=dev)
    g.manual_seed(1 + rank)
    x = torch.randn((n, 28), generator=g, device=dev, dtype=torch.float32)
    x.mul_(torch.from_numpy(sigma).to(dev)).add_(torch.from_numpy(mu).to(dev))
    y = torch.empty((n, 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        prog.run(x, out=y, stream=stream)
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = N.lib().cmlb_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            prog.run(x, out=y, stream=stream)
            ev[i][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = N.lib().cmlb_launch_count() - launches0
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    kernel_ms = [a.elapsed_time(b) for a, b in ev]
    t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * n * args.steps / (max_ms / 1e3)

    # ---- end to end through the public API: pinned host X -> classes on host ----
    xh = x.cpu().pin_memory()
    yh = torch.empty((n, 1), dtype=torch.uint8).pin_memory()
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
    parity_ok = bool(torch.equal(yh.to(dev), y))

    if rank == 0:
        pk = peaks()
        ops_row = gemm_equivalent_ops(model)
        kern_s = statistics.mean(kernel_ms) / 1e3
        rows_per_s_kernel = n / kern_s
        achieved_tops = rows_per_s_kernel * ops_row / 1e12
        achieved_gbs = rows_per_s_kernel * BYTES_ROW / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic_rf500.json")
        if os.path.exists(tpath):  # ncu dram__bytes_read+write per row, scaled to this launch
            with open(tpath) as fh:
                traffic = json.load(fh)["dram_bytes_per_row"] * n
        clocks = clk.summary()
        smem = None  # the traversal's binding resource: shared-memory load wavefronts
        spath = os.path.join(ROOT, "profiles", "r1_forest_ranked_ncu_summary.json")
        if info["variant"] == "ranked" and os.path.exists(spath):
            with open(spath) as fh:
                js = json.load(fh)
            wf_row = float(str(js["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]).split()[0]) / js["rows"]
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
            ach = rows_per_s_kernel * wf_row / 1e9
            pk_w = sms * mhz * 1e6 / 1e9
            smem = {"achieved": ach, "peak": pk_w, "unit": "Gwavefronts/s", "frac": ach / pk_w,
                    "wavefronts_row": wf_row,
                    "basis": "shared-memory load wavefronts per row (ncu, profiles/r1_forest_ranked_ncu_summary.json) "
                             "x live rows/s; peak = 1 wavefront/clk/SM at the measured SM clock"}
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {
                "workload": f"RandomForestClassifier 500 trees depth 8 on {n} x 28 fp32 rows per GPU",
                "forest_source": "sklearn RF500 max_depth=8 fit on make_classification(200k x 28), "
                                 "bench_assets/rf500_d8.npz",
                "rows_per_gpu": n, "trees": len(model.trees), "features": 28,
                "parallelism": f"row-shard dp{world}", "variant": info['variant'] + ("-path-matrix" if info['variant'] == "mma" else "-traversal"),
                "chunk_trees": info["chunk_trees"], "rows_per_cta": info["rows_per_cta"],
                "l2": "inputs 1.12 GB per step > 126 MB L2 (no flush needed)"},
            "roofline": {
                "bound": "tensor", "achieved": achieved_tops, "peak": pk["int8_tops"], "unit": "TOPS",
                "frac": achieved_tops / pk["int8_tops"], "traffic": traffic,
                "basis": "GEMM-equivalent int8 work of the reference encoding, ops_row = sum_t 2*I_t*L_t "
                         f"= {ops_row} (SURVEY 8d); kernel = {info['variant']} variant",
                "peak_source": pk["source"]["int8"],
                "hbm": {"achieved": achieved_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": achieved_gbs / pk["hbm_gbs"], "bytes_row": BYTES_ROW,
                        "peak_source": pk["source"]["hbm"]},
                "smem": smem,
                "kernel_ms": statistics.mean(kernel_ms)},
            "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": n * 28 * 4,
                    "d2h_bytes_per_step": n * 1, "steps": args.e2e_steps, "parity_vs_device": parity_ok},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(model, mu, sigma)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
