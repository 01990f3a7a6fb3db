# gpu_final.sh plus the c5 line
bash scripts/gpu_final.sh
timeout 600 python bench.py --config c5 --steps 5 --no-cpu-baseline > gpurun_out/final_c5.log 2>&1; tail -1 gpurun_out/final_c5.log > gpurun_out/final_c5.json
python -c "
import json; d=json.load(open('gpurun_out/final_c5.json')); r=d['roofline']; print('c5 value', round(d['value'],2), 'kernel', round(r['kernel_ms'],3), 'frac', round(r['frac'],3), 'e2e', d['e2e']['value'] if d.get('e2e') else None)"
