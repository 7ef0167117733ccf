#!/bin/bash
# Which role binds the MMA forest variant?  RF500 d8 on 2M rows with parts off
# (CMLB_MMA_PROBE bits: 1 no compares, 2 no blob TMA after the first two, 4 no
# TMEM reads).  Outputs are garbage by design; only the rate matters.
cd "$(dirname "$0")/.."
for p in 0 1 2 4 3 5 6 7; do
  v=$(CMLB_MMA_PROBE=$p timeout 300 python bench.py --variant mma --rows 2000000 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; print(json.loads(sys.stdin.read())['value']/1e6)")
  echo "{\"probe\": $p, \"M_rows_per_s\": $v}"
done
