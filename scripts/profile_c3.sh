#!/bin/bash
# ncu evidence for the dominant kernels at the metric config (run under gpurun).
set -u
cfg=${1:-c3}
out=gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$cfg.csv \
    python bench.py --config $cfg --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:assign_tc -s 1 -c 1 \
    -o $out/prof_assign_$cfg -f python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_assign_$cfg.log 2>&1
echo "assign profile rc=$?"
ncu --set full --clock-control none --import-source on -k regex:segsum -s 1 -c 1 \
    -o $out/prof_update_$cfg -f python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_update_$cfg.log 2>&1
echo "update profile rc=$?"
