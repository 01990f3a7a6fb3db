# c2 through each assignment variant (kernel and per-iteration time)
for v in rowreg fp8s bf16s tc3xtf32 tc1xtf32s; do
  timeout 300 python bench.py --config c2 --variant $v --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/c2v_$v.json
  python -c "
import json; d=json.load(open('gpurun_out/c2v_$v.json')); r=d['roofline']
print('$v', 'kernel_ms', round(r['kernel_ms'],4), 'assign_ms', round(r['assign_ms'],4), 'ms/step', round(d['ms_per_step'],4), 'launches', d['gpu_launches'])" || tail -2 gpurun_out/c2v_$v.json
done
