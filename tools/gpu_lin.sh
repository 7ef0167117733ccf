#!/bin/bash
# Linear certified path: tests, queue statistics, bench, launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_linear_cert.py tests/test_gpu_fullsize.py tests/test_gpu_concurrency.py tests/test_gpu_parity.py -m gpu -q -x -k "linear or lin or lr or logreg or concurrency or fullsize" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
CMLB_LINEAR_QSTAT=1 timeout 300 python tools/linear_probe.py > gpurun_out/lin_probe.txt 2>&1
PROBE_C=2 CMLB_LINEAR_QSTAT=1 timeout 300 python tools/linear_probe.py >> gpurun_out/lin_probe.txt 2>&1
timeout 600 python bench.py --config lr784 --steps 20 --warmup 5 > gpurun_out/cfg_lr784.json 2> gpurun_out/cfg_lr784.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_lr.csv \
  python bench.py --config lr784 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_lr.log 2>&1
${EXTRA:-true}
echo done
