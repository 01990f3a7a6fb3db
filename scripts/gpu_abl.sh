# screen ablations (experiment .so builds; labels wrong, timing only): full / no epilogue ALU / no TMEM loads
for cfg in c5 c3; do
  for lib in paper_2501_05587_b200/lib/libpopcorn_b200.so build_exp/libabl1.so build_exp/libabl2.so; do
    PCB_LIB_PATH=$lib timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 5 2>&1 | tail -1 > gpurun_out/abl.json
    python -c "
import json,sys
try:
    d=json.load(open('gpurun_out/abl.json')); r=d['roofline']; print('$cfg', '$lib'.split('/')[-1], 'kernel_ms', round(r['kernel_ms'],4))
except Exception as e: print('$cfg $lib failed', open('gpurun_out/abl.json').read()[:200])"
  done
done
