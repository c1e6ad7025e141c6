#!/bin/bash
# A/B of the cfg3 and cfg5 loops (total s, per-threshold Stage-1 s) for library builds, interleaved.
for rep in 1 2 3; do
  for lib in "$@"; do
    for c in cfg3 cfg5; do
      RSR_LIB_OVERRIDE=$lib python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', round(d['value'],3), [round(s['stage1_s'],3) for s in d['stages']])"
    done
  done
done
