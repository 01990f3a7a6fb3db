# small-d constant-bank kernel: bit-identity tests, c2 / c1 lines (rowcst vs shared-memory rowpair), ncu of c2
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider -k "rowpair or small_d" > gpurun_out/c2c_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2c_test.log
tail -3 gpurun_out/c2c_test.log
for mode in cst smem; do
  if [ $mode = smem ]; then export PCB_ROWCST_OFF=1; else unset PCB_ROWCST_OFF; fi
  for cfg in c2 c1; do
    timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/c2c_${cfg}_${mode}.json
    python -c "
import json; d=json.load(open('gpurun_out/c2c_${cfg}_${mode}.json')); r=d['roofline']
print('$cfg $mode', 'kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), r['bound'], 'frac', round(r['frac'],3), d['clocks'])" || tail -3 gpurun_out/c2c_${cfg}_${mode}.json
  done
done
unset PCB_ROWCST_OFF
bash scripts/profile_kernel.sh "assign_row" c2c c2 auto 4
python scripts/ncu_summary.py gpurun_out/prof_c2c.ncu-rep
ncu -i gpurun_out/prof_c2c.ncu-rep --page details --csv > gpurun_out/prof_c2c_details.csv 2>/dev/null
ncu -i gpurun_out/prof_c2c.ncu-rep --page source --csv > gpurun_out/prof_c2c_source.csv 2>/dev/null


