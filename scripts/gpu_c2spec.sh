# small-d kernel with the delta update's changed-row sums fused (update mode 3): tests, c2 lines, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_update.py tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_capi.py -x -q -p no:cacheprovider > gpurun_out/spec_test.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/spec_test.log
for rep in a b; do
  timeout 300 python bench.py --config c2 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/spec_c2_$rep.json
  python -c "
import json; d=json.load(open('gpurun_out/spec_c2_$rep.json')); r=d['roofline']
print('c2', 'value', round(d['value'],1), 'ms/step', round(d['ms_per_step'],4), 'assign', round(r['assign_ms'],4), 'update', round(r['update_ms'],4), 'kernel', round(r['kernel_ms'],4), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"
done
SKIP=90 COUNT=27 bash scripts/launches_steady.sh c2 steady_c2 | head -14
