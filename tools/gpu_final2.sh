set -x
timeout 900 tools/compact_tile_sweep.sh "100000 500000" "def 208" > gpurun_out/sweep20.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/tfinal2.log 2>&1; echo rc=$? >> gpurun_out/tfinal2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final2.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo rc=$? >> gpurun_out/bench_final2.err
CMD="python bench.py --steps 2 --warmup 3 --no-loop --no-cpu-baseline --no-secondary --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:classify_fp4|finalize|gather_columns|encode|or_rows' -c 200 --csv --log-file gpurun_out/launches20.csv $CMD > gpurun_out/ncu20.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:classify_fp4_pair -s 15 -c 5 -o gpurun_out/fp4_tail224_cfg4 $CMD > gpurun_out/ncu20_full.log 2>&1
