#!/bin/bash
# FP4 classifier kernel ms / roofline fraction per forced MMA N on mid-size (streamed) cfg4 sets.
for k in 2500 3000 4000; do
  for tn in 160 176 192 208 224 240; do
    RSR_FP4_TILE_N=$tn timeout 200 python bench.py --config cfg4 --k $k --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print($k, $tn, round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"
  done
done
