#!/bin/bash
# One ncu --set full capture summarised on the box: gpu_prof_one.sh NAME KERNEL_REGEX SKIP CMD...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
name=$1 k=$2 skip=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.log 2>&1
python tools/ncu_summary.py /tmp/$name.ncu-rep --note "$name" > gpurun_out/$name.json 2>> gpurun_out/$name.log
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/$name.src.csv 2>/dev/null
python tools/ncu_hot.py /tmp/$name.src.csv gpurun_out/$name.lines.txt > gpurun_out/$name.hot.txt 2>&1
ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
