#!/bin/bash
# Config 3 (GBR 1000 x d10, 1M x 90) under each ranked launch shape that fits.
cd "$(dirname "$0")/.."
for c in 7 4 5 6; do
  echo "cfg $c: $(CMLB_RANKED_CFG=$c timeout 300 python tools/bench_configs.py --only 3 2>&1 | tail -1 | cut -c1-260)"
done
