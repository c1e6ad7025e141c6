#!/bin/bash
# Kernel ms / roofline fraction of the FP4 classifier per forced MMA N (RSR_FP4_TILE_N).
for cfg in "--config cfg4 --k 1000" "--config cfg4 --k 3000" "--config cfg4 --k 10000" "--config cfg2"; do
  for tn in 160 176 192 208 224 240; do
    RSR_FP4_TILE_N=$tn python bench.py $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', $tn, round(d['roofline']['kernel_ms'],3), round(d['roofline']['frac'],3))"
  done
done
