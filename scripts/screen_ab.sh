#!/bin/bash
# A/B the screening kernel implementations at one config under gpurun:
# GPU screen tests, then one bench line per PCB_SCREEN_IMPL value.
cfg=${1:-c3}
out=gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k screen > $out/t_screen.log 2>&1
echo "screen tests rc=$? $(tail -1 $out/t_screen.log)"
for impl in res pair stream; do
  PCB_SCREEN_IMPL=$impl timeout 300 python bench.py --config $cfg --variant tc1xtf32s --steps 10 --warmup 3 \
      --no-e2e --no-cpu-baseline > $out/ab_${cfg}_$impl.json 2> $out/ab_${cfg}_$impl.err
  echo "$impl rc=$? $(python -c "import json,sys;d=json.load(open('$out/ab_${cfg}_$impl.json'));r=d['roofline'];print(round(d['ms_per_step'],3),'assign',round(r['assign_ms'],3),'upd',round(r['update_ms'],3),'frac',round(r['frac'],3),'amb',d['screen_ambiguous_rows_last_iter'])" 2>&1)"
done
