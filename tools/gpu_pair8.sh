set -x
timeout 600 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
timeout 600 python tools/pair_small_n.py > gpurun_out/pair_small_n10.txt 2>&1
for m in 0 1; do RSR_FP4_PAIR=force RSR_FP4_PAIR8=$m timeout 600 tools/compact_tile_sweep.sh "10000 100000 500000" "def" > gpurun_out/sweep10_p8_$m.txt 2>&1; done
