# small-d constant-bank kernel shapes (PCB_ROWCST_SHAPE 0-3) vs the shared-memory kernel at c2; tests per shape
mkdir -p gpurun_out
for shape in 0 3; do
  export PCB_ROWCST_SHAPE=$shape
  timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider -k "rowpair or small_d" > gpurun_out/c2s_test_$shape.log 2>&1; echo "shape $shape pytest rc=$?"; tail -1 gpurun_out/c2s_test_$shape.log
  for rep in 1 2; do
  timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/c2s_$shape.json
  python -c "
import json; d=json.load(open('gpurun_out/c2s_$shape.json')); r=d['roofline']
print('shape $shape', 'kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), r['bound'], 'frac', round(r['frac'],3), d['clocks']['sm_mhz'])"
  done
done
unset PCB_ROWCST_SHAPE
export PCB_ROWCST_OFF=1
timeout 300 python bench.py --config c2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/c2s_smem.json
python -c "
import json; d=json.load(open('gpurun_out/c2s_smem.json')); r=d['roofline']
print('smem', 'kernel_ms', round(r['kernel_ms'],4), 'ms/step', round(d['ms_per_step'],4), r['bound'], 'frac', round(r['frac'],3), d['clocks']['sm_mhz'])"
