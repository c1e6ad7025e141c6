set -x
timeout 600 python -m pytest tests/test_gpu_pair.py tests/test_gpu_compact.py -q -x > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
for tail in 0 1; do echo "== RSR_FP4_TAIL=$tail"; RSR_FP4_TAIL=$tail timeout 600 tools/compact_tile_sweep.sh "100000 500000" "def"; done > gpurun_out/sweep15.txt 2>&1
