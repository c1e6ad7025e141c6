run() { st=$((2000000 / 1000 + 20)); env "$@" python bench.py --config cfg4 --k 1000 --steps $st --warmup 5 --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); r=d['roofline']; print('$*', round(r['kernel_ms'], 4), round(r['frac'], 4))"; }
for ab in 2 3 4; do for tn in 176 192 208 224; do run RSR_TC_ABUFS=$ab RSR_FP4_TILE_N=$tn; done; done
run RSR_FP4_FLAG_EXCHANGE=1
