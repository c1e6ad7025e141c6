#!/bin/bash
# FP4 classifier kernel ms / roofline fraction at the launch's own tile choice, cfg4 path refs.
for k in ${@:-500 1000 1500 2000 2200 2500 3000 5000 10000}; do
  timeout 200 python bench.py --config cfg4 --k $k --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print($k, round(d['roofline']['kernel_ms'],4), round(d['roofline']['frac'],3))"
done
