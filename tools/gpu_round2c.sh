set -x
timeout 600 python -m pytest tests/test_gpu_pair.py tests/test_gpu_northstar.py -q -x -k "pair or selfcheck" > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
CMD="python bench.py --steps 2 --warmup 3 --no-loop --no-cpu-baseline --no-secondary --no-e2e"
timeout 600 $CMD > gpurun_out/plain9.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:classify_fp4|finalize|gather_columns|encode|or_rows' -c 200 --csv --log-file gpurun_out/launches9.csv $CMD > gpurun_out/ncu9.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/reference9.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke9.log 2>&1
