#!/bin/bash
# GBR ranked launch-shape sweep (CMLB_RANKED_CFG) + parity of the new shape.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 8 10 7; do
  CMLB_RANKED_CFG=$c timeout 600 python bench.py --config gbr1000 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/gbr_cfg$c.json 2> gpurun_out/gbr_cfg$c.err
done
CMLB_RANKED_CFG=10 timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_rf500_ref.py tests/test_gpu_shard.py -m gpu -q -k "gbr or tree_shard" > gpurun_out/pytest_gbr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gbr.log
echo done
