#!/usr/bin/env bash
# Support compaction on cfg4 (2^22 samples x K s-t path refs, upper side): classifier time,
# MMA-issued fraction and re-pack time per reference count and forced tile width
# (RSR_FP4_TILE_N; "def" = the library's plan), plus compaction off for comparison.
# usage: tools/compact_tile_sweep.sh "K ..." "TN ..."
KS="${1:-10000 100000 500000}"
TNS="${2:-def 240 224 208 192 176 160}"
for k in $KS; do
  st=$((1000000 / k + 4))
  for tn in off $TNS; do
    env=""
    [ "$tn" = off ] && env="RSR_FP4_COMPACT=0"
    [ "$tn" != off ] && [ "$tn" != def ] && env="RSR_FP4_TILE_N=$tn"
    env $env python bench.py --config cfg4 --k $k --steps $st --warmup 3 --no-cpu-baseline \
      --no-e2e --no-secondary --no-loop 2>/dev/null |
      python -c "
import json,sys
d=json.loads(sys.stdin.read().splitlines()[-1]); r=d['roofline']; c=r.get('support_compaction') or {}
print($k, '$tn', 'step_ms', round(d['ms_per_step'],4), 'kernel_ms', round(r['kernel_ms'],4), 'mma_frac', round(r['frac_mma_issued'],4), 'repack_ms', round(c.get('repack_ms') or 0,4), 'rb', c.get('row_bytes'))"
  done
done
