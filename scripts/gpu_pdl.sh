# programmatic dependent launch A/B (PCB_PDL=1 default vs 0): c3, c3 at one 8-rank shard's rows, c2, c5; then the GPU suite
mkdir -p gpurun_out
run() {  # tag, env, args
  tag=$1; shift; pdl=$1; shift
  PCB_PDL=$pdl timeout 400 python bench.py "$@" --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/pdl_$tag.json
  python -c "
import json; d=json.load(open('gpurun_out/pdl_$tag.json')); r=d['roofline']
print('$tag', 'ms/step', round(d['ms_per_step'],4), 'kernel_ms', round(r['kernel_ms'],4), 'value', round(d['value'],1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/pdl_$tag.json
}
for rep in a b; do
  run c3_on_$rep 1 --config c3
  run c3_off_$rep 0 --config c3
  run shard8_on_$rep 1 --config c3 --n-override 1250000
  run shard8_off_$rep 0 --config c3 --n-override 1250000
  run c2_on_$rep 1 --config c2
  run c2_off_$rep 0 --config c2
done
run c5_on 1 --config c5
run c5_off 0 --config c5
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pdl_test.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pdl_test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
