# full GPU suite + smoke + c2 / c3 lines (no e2e / CPU legs)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/check_test.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/check_test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in c2 c2 c3; do
  timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/check_$cfg.json
  python -c "
import json; d=json.load(open('gpurun_out/check_$cfg.json')); r=d['roofline']
print('$cfg', 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'assign', round(r['assign_ms'],4), 'update', round(r['update_ms'],4), 'kernel', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
