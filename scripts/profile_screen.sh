#!/bin/bash
# ncu captures for the screened variant at a config (default c3), under gpurun.
cfg=${1:-c3}
out=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:assign_screen -s 4 -c 1 \
    -o $out/prof_screen_$cfg -f python bench.py --config $cfg --variant tc1xtf32s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_screen_$cfg.log 2>&1
echo "screen rc=$?"
ncu --set full --clock-control none --import-source on -k regex:segsum -s 4 -c 1 \
    -o $out/prof_segsum_$cfg -f python bench.py --config $cfg --variant tc1xtf32s --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_segsum_$cfg.log 2>&1
echo "segsum rc=$?"
