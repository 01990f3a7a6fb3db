#!/bin/bash
# One ncu --set full capture of a kernel (regex) in a bench run, under gpurun.
# usage: scripts/profile_kernel.sh <kernel-regex> <tag> [config] [variant] [skip]
re=$1; tag=$2; cfg=${3:-c3}; variant=${4:-auto}; skip=${5:-4}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$re" -s $skip -c 1 \
    -o gpurun_out/prof_$tag -f python bench.py --config $cfg --variant $variant --steps 2 --warmup 3 --no-graph $EXTRA \
    --no-e2e --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
echo "ncu $tag rc=$?"
