#!/bin/bash
# Bucket rank tables: forest parity files, benches (bucket vs Eytzinger), rank-pass profile.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rf500_ref.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py tests/test_gpu_shard.py tests/test_gpu_sanitizer.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
CMLB_RANK_EYT=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_eyt.json 2> gpurun_out/bench_eyt.err
timeout 900 python bench.py --config gbr1000 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_gbr1000.json 2> gpurun_out/cfg_gbr1000.err
timeout 900 python bench.py --config pipe5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_pipe5.json 2> gpurun_out/cfg_pipe5.err
bash tools/gpu_rankprof.sh
echo done
