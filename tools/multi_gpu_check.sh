#!/bin/bash
# Multi-GPU checks for a box with >= 2 GPUs (the round-1 pool had one GPU per call,
# so these ran only as gloo tests).  Usage: bash tools/multi_gpu_check.sh [max_gpus]
set -e
MAX=${1:-8}
PORT=29511
for n in 2 4 8; do
  [ "$n" -le "$MAX" ] || break
  echo "== weak scaling, $n GPUs (replicated references, counts all-reduced)"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $PORT bench.py --gpus $n --steps 10 --warmup 3 | tail -1
  echo "== cfg4 K=5e5, $n GPUs, reference-sharded (2-D grid, flags OR-reduced)"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $PORT bench.py --gpus $n --config cfg4 --k 500000 --ref-shards $n \
    --steps 3 --warmup 3 --no-e2e | tail -1
done
for n in 2 4 8; do
  [ "$n" -le "$MAX" ] || break
  echo "== RSR loops on $n GPUs (samples of every batch sharded)"
  for c in cfg3 cfg5; do
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $PORT bench.py --gpus $n --config $c | tail -1
  done
done
