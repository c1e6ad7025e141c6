set -x
timeout 600 python -m pytest tests/test_gpu_pair.py tests/test_gpu_compact.py -q -x > gpurun_out/t14.log 2>&1; echo rc=$? >> gpurun_out/t14.log
for lib in paper_2604_17066_b200/librsr_b200.so tools/librsr_nosplit.so; do
  for tail in 0 1; do
    echo "== $lib RSR_FP4_TAIL=$tail"
    RSR_LIB_OVERRIDE=$lib RSR_FP4_TAIL=$tail timeout 600 tools/compact_tile_sweep.sh "100000 500000" "def"
  done
done > gpurun_out/sweep14.txt 2>&1
