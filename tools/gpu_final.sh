set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/tfinal.log 2>&1; echo rc=$? >> gpurun_out/tfinal.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo rc=$? >> gpurun_out/bench_final.err
