#!/bin/bash
# Functional check of bench.py's multi-rank paths on a single GPU: 2 ranks with gloo
# collectives (host-mediated, no kernel waits on another rank).  Not a performance run.
RSR_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 \
  > gpurun_out/mg.log 2>&1
grep -E "Error|^\{" gpurun_out/mg.log | cut -c1-400 | head -5
RSR_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config cfg4 --k 10000 \
  --ref-shards 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/mg2.log 2>&1
grep -E "Error|^\{" gpurun_out/mg2.log | cut -c1-700 | head -5
for c in cfg1 cfg3 cfg5; do
  RSR_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --config $c --no-cpu-baseline \
    > gpurun_out/mg_$c.log 2>&1
  grep -E "Error|^\{" gpurun_out/mg_$c.log | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$c', d['n_gpus'], round(d['value'],3), [(s['iterations'], s['refs'], s['p_lower']) for s in d['stages']])
    else: print(l.strip()[:300])"
done
