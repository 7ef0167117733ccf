#!/bin/bash
# ncu of the SVM certifying tier and the forest rank pass + quick benches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config svc10k --steps 5 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > gpurun_out/cfg_svc10k.json 2> gpurun_out/cfg_svc10k.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svm_certify -c 1 -o gpurun_out/prof_certify -f \
  python bench.py --config svc10k --rows 200000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > gpurun_out/prof_certify.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:forest_rank -s 3 -c 1 -o gpurun_out/prof_rank -f \
  python bench.py --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > gpurun_out/prof_rank.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_bench.log 2>&1
echo done
