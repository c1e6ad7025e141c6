for c in 1 2 4 1000; do
  echo "cpc=$c"; RSR_SAMPLE_CPC=$c python tools/time_kernels.py 2>&1 | grep "^sample_batch M"
  for cfg in cfg3 cfg5; do RSR_SAMPLE_CPC=$c python bench.py --config $cfg --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value'],3), [round(s['stage1_s'],3) for s in d['stages']])"; done
done
