#!/bin/bash
# Full ncu capture of the forest kernel at the bench config (fewer rows keep replay short).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-forest} -s 3 -c 1 \
  -o gpurun_out/prof_forest -f python bench.py --rows ${ROWS:-2000000} --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/prof.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof.log
