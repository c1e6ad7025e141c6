#!/bin/bash
# Bench lines for profiles/ (round 2): the default line (cfg4 K=5x10^5 north-star point +
# cfg4 sweep + cfg2 + cfg3 loop in both RNG modes + CPU reference legs), the reference
# arm, the full loops with CPU baselines, the ncu launch list of the default step, an
# ncu --set full capture of the five classifier launches of one default step, the
# classifier K sweep and the samplers.  Writes gpurun_out/prof_*.
set -x
python bench.py > gpurun_out/prof_bench.log 2>&1; grep '^{' gpurun_out/prof_bench.log | tail -1 > gpurun_out/prof_bench.json
python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/prof_reference.json
for c in cfg1 cfg3 cfg5; do
  python bench.py --config $c 2>/dev/null | tail -1 > gpurun_out/prof_loop_$c.json
  python bench.py --config $c --rng device --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/prof_loop_${c}_device.json
done
tools/fp4_k_sweep.sh 500 1000 1500 2000 2500 3000 4000 5000 6000 10000 100000 500000 > gpurun_out/prof_k_sweep.txt 2>&1
python tools/sample_outputs.py > gpurun_out/prof_samplers.txt 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-loop --no-cpu-baseline --no-secondary --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:classify|finalize|sample_rows|encode' -c 200 --csv \
    --log-file gpurun_out/prof_launches.csv $CMD > gpurun_out/prof_ncu_launches.log 2>&1
$CMD > gpurun_out/prof_plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:classify_fp4_pair -s 15 -c 5 \
    -o gpurun_out/prof_fp4_cfg4 $CMD > gpurun_out/prof_ncu_full.log 2>&1
LOOP="python bench.py --config cfg3 --rng device --no-cpu-baseline"
$LOOP > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/prof_loop3_device_launches.csv $LOOP > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/prof_loop3_device_launches.csv > gpurun_out/prof_loop3_device_kernels.txt 2>&1
