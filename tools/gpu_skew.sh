#!/bin/bash
# Round-2 session: peaks microbenchmarks, smoke, the new GPU tests, bench (AUTO and
# ranked), the SKEW launch-config sweep, and ncu of the skew kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/peaks_micro.sh > gpurun_out/peaks.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_rf500_ref.py tests/test_gpu_shard.py tests/test_gpu_parity.py -m gpu -q -x \
  -k "${PYK:-not nothing}" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
for v in auto ranked; do
  timeout 600 python bench.py --steps 10 --warmup 3 --variant $v --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
for c in 0 1 2 3 4 5; do
  CMLB_SKEW_CFG=$c timeout 300 python bench.py --steps 10 --warmup 3 --variant skew --no-cpu-baseline --e2e-steps 1 > gpurun_out/skew_cfg$c.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --rows 2000000 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1
KERNEL=forest_skew OUT=prof_skew bash tools/gpu_prof.sh
echo done
