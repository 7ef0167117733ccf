#!/bin/bash
# Rank-pass rework: forest parity files, sanitizer, bench (both staging depths), rank profile.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rf500_ref.py tests/test_gpu_fullsize.py tests/test_gpu_sanitizer.py tests/test_gpu_shard.py tests/test_gpu_pipeline.py -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
CMLB_RANK_NB=3 timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_nb3.json 2> gpurun_out/bench_nb3.err
timeout 900 python bench.py --config gbr1000 --steps 10 --warmup 3 > gpurun_out/cfg_gbr1000.json 2> gpurun_out/cfg_gbr1000.err
bash tools/gpu_rankprof.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_bench.log 2>&1
echo done
