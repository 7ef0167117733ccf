#!/bin/bash
# Round-2 session C: targeted tests, benches of every config, summarised profiles.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -n "$PYK" ]; then
  timeout 2400 python -m pytest ${PYFILES:-tests} -m gpu -q -k "$PYK" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
else
  timeout 2400 python -m pytest ${PYFILES:-tests} -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
for c in ${CONFIGS:-gbr1000 svc10k pipe5 dt6 lr784}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
done
prof() {  # name kernel-regex skip cmd...
  local name=$1 k=$2 skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep --note "$name" > gpurun_out/$name.json 2>> gpurun_out/$name.log
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.src.csv 2>/dev/null
  python tools/ncu_hot.py /tmp/$name.src.csv gpurun_out/$name.lines.txt > gpurun_out/$name.hot.txt 2>&1
}
if [ -z "$NOPROF" ]; then
prof prof_certify svm_certify 0 python bench.py --config svc10k --rows 200000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
prof prof_rank forest_rank 3 python bench.py --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
prof prof_lxw linear_exact_whole 3 python tools/linear_probe.py
prof prof_skew forest_skew 3 python bench.py --rows 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
prof prof_ltile linear_tile 3 python tools/linear_probe.py
prof prof_gbr forest_ranked 3 python bench.py --config gbr1000 --rows 500000 --steps 1 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --no-parity > gpurun_out/ncu_bench.log 2>&1
echo done
