#!/bin/bash
# Loop wall times (cfg1/cfg3/cfg5) with the async Stage-1 loop vs RSR_SYNC_LOOP=1.
for mode in 0 1; do
  for c in cfg1 cfg3 cfg5; do
    RSR_SYNC_LOOP=$mode python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sync=$mode', '$c', round(d['value'],3), [(s['iterations'], round(s['stage1_s'],3), round(s['stage2_s'],3)) for s in d['stages']])"
  done
done
