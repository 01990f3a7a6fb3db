# round-end style check plus the c1 / c2 lines
bash scripts/gpu_final.sh
for cfg in c2 c1; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/final_$cfg.json
  python -c "
import json; d=json.load(open('gpurun_out/final_$cfg.json')); r=d['roofline']
print('$cfg', 'value', round(d['value'],1), 'kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), r['bound'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'])"
done
