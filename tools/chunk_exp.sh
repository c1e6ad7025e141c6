#!/usr/bin/env bash
# mid-size sets: consecutive resident-sized launches vs hybrid streaming
run() { # k tn chunk
  st=$((2000000 / $1 + 20))
  RSR_FP4_TILE_N=$2 RSR_TC_CHUNK_TILES=$3 python bench.py --config cfg4 --k $1 --steps $st --warmup 5 \
      --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); r=d['roofline']; print($1, $2, '$3', round(r['kernel_ms'], 4), round(r['frac'], 4))"
}
for k in 2500 3000 3500 4000 5000; do
  for tn in 176 208 224 240; do
    nt=$(( (k + tn - 1) / tn ))
    run $k $tn $nt
    run $k $tn $(( (nt + 1) / 2 ))
    run $k $tn $(( (nt + 2) / 3 ))
  done
done
