timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rf500_ref.py -m gpu -q -x -k "skew or ranked or rf500 or nan or dense" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
bash tools/gpu_rankprof.sh
