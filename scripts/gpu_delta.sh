# delta-chunked tensor-core ablation: parity tests, then the c4 ablation lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -p no:cacheprovider -k "delta" > gpurun_out/delta_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/delta_test.log
tail -30 gpurun_out/delta_test.log
if grep -q "pytest rc=0" gpurun_out/delta_test.log; then
  for v in deltatc fp8s tc3xtf32; do
    timeout 600 python bench.py --config c4 --variant $v --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/c4_$v.json
    cat gpurun_out/c4_$v.json
  done
  timeout 900 python bench.py --config c4 --variant delta --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/c4_delta.json
  cat gpurun_out/c4_delta.json
fi
