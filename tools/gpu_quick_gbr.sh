#!/bin/bash
# GBR / RANKED checks: parity files, fullsize, bench gbr1000.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rf500_ref.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config gbr1000 --steps 10 --warmup 3 > gpurun_out/cfg_gbr1000.json 2> gpurun_out/cfg_gbr1000.err
CMLB_RANKED_RUNTIME_DEPTH=1 timeout 900 python bench.py --config gbr1000 --steps 10 --warmup 3 > gpurun_out/cfg_gbr1000_rt.json 2> gpurun_out/cfg_gbr1000_rt.err
${EXTRA:-true}
echo done
