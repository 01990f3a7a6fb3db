# small-d FFMA2 kernel: bit-identity + parity tests, then c1/c2 lines (new and scalar)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_update.py -x -q -p no:cacheprovider > gpurun_out/c2_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2_test.log
tail -5 gpurun_out/c2_test.log
for cfg in c2 c1; do
  for mode in pair scalar; do
    if [ $mode = scalar ]; then export PCB_ROWREG_SCALAR=1; else unset PCB_ROWREG_SCALAR; fi
    timeout 300 python bench.py --config $cfg --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/c2_${cfg}_${mode}.json
    python -c "
import json; d=json.load(open('gpurun_out/c2_${cfg}_${mode}.json')); r=d['roofline']
print('$cfg $mode', 'kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), r['bound'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],1))" || tail -3 gpurun_out/c2_${cfg}_${mode}.json
  done
done
