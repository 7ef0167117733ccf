#!/bin/bash
# LR 784 tile-config sweep + profiles of the SVM certifying tier and the rank pass.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 1 2 3 4 5 6 7 8; do CMLB_LINEAR_IMPL=$c timeout 120 python tools/linear_probe.py >> gpurun_out/linear_sweep.txt 2>&1; done
prof() {  # name kernel-regex skip cmd...
  local name=$1 k=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep --note "$name" > gpurun_out/$name.json 2>> gpurun_out/$name.log
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.src.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/$name.src.csv > gpurun_out/$name.hot.txt 2>&1
}
prof prof_certify svm_certify 0 python bench.py --config svc10k --rows 200000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
prof prof_rank forest_rank 3 python bench.py --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
prof prof_linear linear_tile 3 python tools/linear_probe.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_lr.csv python tools/linear_probe.py > /dev/null 2>&1
echo done
