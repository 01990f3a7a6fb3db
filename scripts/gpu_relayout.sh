for ra in 1,3 0,3 0,1,3 0,2; do
  PCB_RELAYOUT_AT=$ra timeout 600 python bench.py --config c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/rl_$ra.json
  python -c "
import json; d=json.load(open('gpurun_out/rl_$ra.json')); e=d['e2e']
print('$ra', 'value', round(d['value'],1), 'e2e', round(e['value'],1), 'phases', {k: round(v,1) for k,v in e['phases_ms'].items()})"
done
