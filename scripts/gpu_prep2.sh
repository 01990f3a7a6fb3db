timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/prep2_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/prep2_test.log
tail -3 gpurun_out/prep2_test.log
for cfg in c3 c5 c4; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/prep2_$cfg.json
  python -c "
import json; d=json.load(open('gpurun_out/prep2_$cfg.json')); r=d['roofline']
print('$cfg', 'kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), 'value', round(d['value'],2), 'launches', d['gpu_launches'], 'amb', d['screen_ambiguous_rows_last_iter'])"
done
timeout 900 python scripts/shard_probe.py
