#!/bin/bash
# Kernel-time comparison of experiment builds of librsr (tools/librsr_*.so) on the
# cfg2 workload; each line: variant, kernel ms, fraction of the FP4 peak.
for lib in "$@"; do
  RSR_LIB_OVERRIDE=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/vb_$(basename $lib).log 2>&1
  python - "$lib" <<'PY'
import json, sys, os
f = "gpurun_out/vb_" + os.path.basename(sys.argv[1]) + ".log"
l = [x for x in open(f) if x.startswith("{")]
if l:
    d = json.loads(l[-1]); print(sys.argv[1], round(d["roofline"]["kernel_ms"], 3), round(d["roofline"]["frac"], 3))
else:
    print(sys.argv[1], open(f).read()[-300:])
PY
done
