#!/usr/bin/env bash
# resident-sized launches vs streaming for larger sets (TN 240, 9-tile resident chunks)
run() { st=$((2000000 / $1 + 20)); RSR_FP4_TILE_N=$2 RSR_TC_CHUNK_TILES=$3 python bench.py --config cfg4 --k $1 --steps $st --warmup 5 --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); r=d['roofline']; print($1, $2, '$3', round(r['kernel_ms'], 4), round(r['frac'], 4))"; }
for k in ${KS:-500 7000 8000 10000 15000 20000 40000}; do
  nt=$(( (k + 239) / 240 ))
  run $k 240 $nt
  run $k 240 9
done
