#!/bin/bash
# Bench lines for profiles/: default run (cfg2 + cfg3 loop), reference arm, loops with
# CPU baselines, cfg4 sweep.  Writes gpurun_out/prof_*.json(l).
set -x
python bench.py > gpurun_out/prof_bench.log 2>&1; grep '^{' gpurun_out/prof_bench.log | tail -1 > gpurun_out/prof_bench.json
python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/prof_reference.json
for c in cfg1 cfg3 cfg5; do python bench.py --config $c 2>/dev/null | tail -1 > gpurun_out/prof_loop_$c.json; done
rm -f gpurun_out/prof_cfg4.jsonl
for k in 1000 10000 100000 500000; do python bench.py --config cfg4 --k $k --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/prof_cfg4.jsonl; done
