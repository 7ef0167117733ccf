#!/bin/bash
# Linear tile-config sweep (CMLB_LINEAR_IMPL = cfg + 1) on LR 784->10, 1M rows.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for i in 2 5 11 12; do
  CMLB_LINEAR_IMPL=$i timeout 300 python tools/linear_probe.py >> gpurun_out/lin_sweep.txt 2>&1
done
echo done
