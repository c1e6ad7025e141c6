#!/usr/bin/env bash
# resident-sized consecutive launches vs the streamed default at larger sets (TN = 240)
run() { # k tn chunk
  st=$((2000000 / $1 + 20))
  RSR_FP4_TILE_N=$2 RSR_TC_CHUNK_TILES=$3 python bench.py --config cfg4 --k $1 --steps $st --warmup 5 \
      --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); r=d['roofline']; print($1, $2, '$3', round(r['kernel_ms'], 4), round(r['frac'], 4))"
}
for k in 4500 5000 6000 7000 8000 10000; do
  nt=$(( (k + 239) / 240 ))
  run $k 240 $nt
  for n in 2 3 4 5 6; do
    c=$(( (nt + n - 1) / n ))
    [ $c -le 9 ] && run $k 240 $c
  done
done
