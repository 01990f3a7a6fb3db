timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/fuse_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fuse_test.log
tail -3 gpurun_out/fuse_test.log
bash scripts/launches_steady.sh c3 | head -16
for cfg in c3 c5; do
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/fuse_$cfg.json
  python -c "
import json; d=json.load(open('gpurun_out/fuse_$cfg.json')); r=d['roofline']
print('$cfg', 'kernel_ms', round(r['kernel_ms'],4), 'assign_ms', round(r['assign_ms'],4), 'update_ms', round(r['update_ms'],4), 'ms/step', round(d['ms_per_step'],4), 'value', round(d['value'],2))"
done
