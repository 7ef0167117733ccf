#!/bin/bash
# SVM checks: svm tests, sanitizer (svm family), bench svc10k, launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_svm.py tests/test_gpu_concurrency.py tests/test_gpu_pipeline.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -m pytest tests/test_gpu_sanitizer.py -m gpu -q -k svm >> gpurun_out/pytest_gpu.log 2>&1; echo "sanitizer rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config svc10k --steps 3 --warmup 3 > gpurun_out/cfg_svc10k.json 2> gpurun_out/cfg_svc10k.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_svc.csv \
  python bench.py --config svc10k --rows 200000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_svc.log 2>&1
${EXTRA:-true}
echo done
