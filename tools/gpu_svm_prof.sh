#!/bin/bash
# SVC config 4b: launch list (kernel shares) and an instruction-level profile of the certifying tier.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_svc.csv \
  python bench.py --config svc10k --rows 200000 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_svc.log 2>&1
bash tools/gpu_prof_one.sh prof_cert svm_certify 0 python bench.py --config svc10k --rows 200000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
${EXTRA:-true}
echo done
