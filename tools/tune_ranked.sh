#!/bin/bash
# Bench every ranked launch configuration on the north-star workload.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CFGS:-0 1 2 3 4 5 6}; do
  CMLB_RANKED_CFG=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tune_$c.json 2> gpurun_out/tune_$c.err
done
