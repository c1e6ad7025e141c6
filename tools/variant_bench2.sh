#!/bin/bash
# Kernel-time comparison of experiment builds on cfg2 and the cfg4 K=10^3 / 10^4 points.
for lib in "$@"; do
  for args in "--config cfg2" "--config cfg4 --k 1000" "--config cfg4 --k 10000"; do
    RSR_LIB_OVERRIDE=$lib timeout 300 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/vb2.log 2>&1
    python - "$lib" "$args" <<'PY'
import json, sys
l = [x for x in open("gpurun_out/vb2.log") if x.startswith("{")]
if l:
    d = json.loads(l[-1]); print(sys.argv[1], sys.argv[2], round(d["roofline"]["kernel_ms"], 3), round(d["roofline"]["frac"], 3))
else:
    print(sys.argv[1], sys.argv[2], open("gpurun_out/vb2.log").read()[-300:])
PY
  done
done
