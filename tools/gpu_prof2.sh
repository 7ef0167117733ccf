#!/bin/bash
# ncu of the SVM certifying tier and the forest rank pass + quick benches.
# Reports are summarised on the box (tools/ncu_summary.py) and deleted: gpurun
# only brings back 64 MiB.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --config svc10k --steps 5 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > gpurun_out/cfg_svc10k.json 2> gpurun_out/cfg_svc10k.err
prof() {  # name kernel-regex skip rows-args...
  local name=$1 k=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep --kernel "" --note "$name" > gpurun_out/$name.json 2>> gpurun_out/$name.log
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.src.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/$name.src.csv > gpurun_out/$name.hot.txt 2>&1
}
prof prof_certify svm_certify 0 python bench.py --config svc10k --rows 200000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
prof prof_rank forest_rank 3 python bench.py --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_bench.log 2>&1
echo done
