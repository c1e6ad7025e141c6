#!/bin/bash
# A/B wall time of the cfg3 / cfg5 loops for two library builds, interleaved.
for rep in 1 2; do
  for lib in "$@"; do
    for c in cfg3 cfg5; do
      RSR_LIB_OVERRIDE=$lib python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', round(d['value'],3))"
    done
  done
done
