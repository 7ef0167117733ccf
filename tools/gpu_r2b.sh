#!/bin/bash
# Round-2 session B: peaks, smoke, broad GPU tests, sanitizers, bench default + configs, launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash tools/peaks_micro.sh > gpurun_out/peaks.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest ${PYFILES:-tests} -m gpu -q ${PYARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in ${CONFIGS:-gbr1000 lr784}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_bench.log 2>&1
echo done
