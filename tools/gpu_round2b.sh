set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
timeout 900 python bench.py > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo rc=$? >> gpurun_out/bench8.err
CMD="python bench.py --steps 2 --warmup 3 --no-loop --no-cpu-baseline --no-secondary --no-e2e"
timeout 600 $CMD > gpurun_out/plain8.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:classify|finalize|gather|encode|or_rows' -c 200 --csv --log-file gpurun_out/launches8.csv $CMD > gpurun_out/ncu8.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:classify_fp4_pair -s 15 -c 5 -o gpurun_out/fp4_pair_cfg4 $CMD > gpurun_out/ncu8_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gather_columns -s 3 -c 1 -o gpurun_out/gather_cfg4 $CMD > gpurun_out/ncu8_gather.log 2>&1
