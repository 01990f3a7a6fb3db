# small-d constant-bank kernel with cp.async prefetch: tests, c2 lines (vs shared-memory kernel), ncu of c2
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/c2p_test.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/c2p_test.log
for mode in cst cst; do
  if [ $mode = smem ]; then export PCB_ROWCST_OFF=1; fi
  timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/c2p_$mode.json
  python -c "
import json; d=json.load(open('gpurun_out/c2p_$mode.json')); r=d['roofline']
print('$mode', 'kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), r['bound'], 'frac', round(r['frac'],3), d['clocks']['sm_mhz'])"
done
unset PCB_ROWCST_OFF





