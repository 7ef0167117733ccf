#!/bin/bash
# RANKED forest with float64 vs float32 payloads in the tree blob (RF500 d8, 10M rows).
cd "$(dirname "$0")/.."
for e in 0 1 0 1; do
  v=$(CMLB_RANKED_DPAY=$e timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e6, d['config']['chunk_trees'])")
  echo "{\"dpay\": $e, \"M_rows_per_s_and_chunk\": \"$v\"}"
done
