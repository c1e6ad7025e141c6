set -x
CMD="python bench.py --steps 2 --warmup 3 --no-loop --no-cpu-baseline --no-secondary --no-e2e"
timeout 600 $CMD > gpurun_out/plain17.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:classify_fp4|finalize|gather_columns|encode|or_rows' -c 200 --csv --log-file gpurun_out/launches17.csv $CMD > gpurun_out/ncu17.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:classify_fp4_pair -s 15 -c 5 -o gpurun_out/fp4_tail_cfg4 $CMD > gpurun_out/ncu17_full.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/reference17.json
