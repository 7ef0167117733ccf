"""Measure the dense TF32 tensor-core peak on this B200 (the SVM Gram GEMM's
roofline; MEASURED_PEAKS.json has HBM and bf16 only).  torch.matmul fp32
8192^3 with TF32 enabled (cuBLAS), best of 10 (burst) and back-to-back for
~4 s (sustained), same method as the driver's bf16 figure.
Writes profiles/peaks_tf32.json."""

import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn((n, n), device="cuda")
    b = torch.randn((n, n), device="cuda")
    for _ in range(5):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    flops = 2.0 * n ** 3
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    t0 = time.time()
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            torch.matmul(a, b)
        iters += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    out = {"tf32_tflops_burst": flops / (best / 1e3) / 1e12,
           "tf32_tflops_sustained": flops * iters / (s.elapsed_time(e) / 1e3) / 1e12,
           "how": "torch.matmul fp32 8192^3 allow_tf32 (cuBLAS), 2*N^3 flops, best of 10 / back-to-back 4 s",
           "gpu": torch.cuda.get_device_name(0)}
    with open(os.path.join(ROOT, "profiles", "peaks_tf32.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
