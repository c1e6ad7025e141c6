#!/usr/bin/env bash
# FP4 classifier kernel time / roofline fraction on cfg4 (2^22 samples x K s-t path
# refs) per reference count; LIBS: libraries to compare (RSR_LIB_OVERRIDE).
# usage: LIBS="paper_2604_17066_b200/librsr_b200.so tools/librsr_x.so" tools/fp4_k_sweep.sh [K ...]
KS="${@:-1000 2000 3000 5000 10000 100000}"
LIBS="${LIBS:-paper_2604_17066_b200/librsr_b200.so}"
for lib in $LIBS; do
  for k in $KS; do
    st=$((2000000 / k + 20))
    RSR_LIB_OVERRIDE=$lib python bench.py --config cfg4 --k $k --steps $st --warmup 5 \
      --no-cpu-baseline --no-e2e --no-secondary 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); r=d['roofline']; print('$lib', $k, round(r['kernel_ms'], 4), round(r['frac'], 4))"
  done
done
