"""Measure the dense int8 tensor-core peak on this B200 (SURVEY 8d asks for it;
MEASURED_PEAKS.json has HBM and bf16 only).  torch._int_mm 8192^3 (cuBLASLt
int8 -> int32), best of 10 (burst) and back-to-back for ~4 s (sustained),
same method as the driver's bf16 figure.  Writes profiles/peaks_int8.json."""

import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    n = 8192
    a = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(5):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    ops = 2.0 * n ** 3
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    t0 = time.time()
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            torch._int_mm(a, b)
        iters += 20
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    sustained = ops * iters / (s.elapsed_time(e) / 1e3) / 1e12
    out = {"int8_tops_burst": ops / (best / 1e3) / 1e12, "int8_tops_sustained": sustained,
           "how": "torch._int_mm int8 8192^3 (2*N^3 ops), best of 10 / back-to-back 4 s, CUDA events",
           "gpu": torch.cuda.get_device_name(0)}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "peaks_int8.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
