#!/bin/bash
# Round-2 session: smoke, the new GPU tests, bench (AUTO and ranked) and every
# --config, the SKEW launch-config sweep, and ncu of the skew kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest ${PYFILES:-tests/test_gpu_rf500_ref.py tests/test_gpu_shard.py tests/test_gpu_parity.py} -m gpu -q \
  -k "${PYK:-not nothing}" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
for v in auto ranked; do
  timeout 600 python bench.py --steps 10 --warmup 3 --variant $v --no-cpu-baseline > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
for c in ${SKEW_CFGS:-0 1 2 3 4}; do
  CMLB_SKEW_CFG=$c timeout 300 python bench.py --steps 10 --warmup 3 --variant skew --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/skew_cfg$c.json 2>&1
done
for c in ${CONFIGS:-dt6 gbr1000 lr784 svc10k pipe5}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --rows 2000000 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_bench.log 2>&1
CMD="python bench.py --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity" KERNEL=forest_skew OUT=prof_skew bash tools/gpu_prof.sh
echo done
