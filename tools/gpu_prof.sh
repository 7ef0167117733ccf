#!/bin/bash
# Full ncu capture of one kernel.  KERNEL=regex, CMD=command (default: the bench at 2M rows).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CMD=${CMD:-"python bench.py --rows ${ROWS:-2000000} --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1"}
OUT=${OUT:-prof_forest}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-forest} -s ${SKIP:-3} -c 1 \
  -o gpurun_out/$OUT -f $CMD > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$OUT.log
