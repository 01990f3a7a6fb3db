# A/B of two builds of the library on one box: build_ab/base.so vs the in-tree .so
# (PCB_LIB_PATH), warm-cache ncu durations of one kernel + bench ms/step, alternating
# usage: scripts/gpu_ab_lib.sh <kernel-regex> <config> [extra bench args]
re=$1; cfg=$2; shift 2  # (the ncu duration parse below expects ncu --csv on stdout; bench lines are the A/B)
mkdir -p gpurun_out
for rep in 1 2; do
  for arm in base new; do
    if [ $arm = base ]; then export PCB_LIB_PATH=$PWD/build_ab/base.so; else unset PCB_LIB_PATH; fi
    timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 > gpurun_out/ab_$arm.json
    python -c "
import json; d=json.load(open('gpurun_out/ab_$arm.json')); r=d['roofline']
print('$arm', 'ms/step', round(d['ms_per_step'],4), 'assign', round(r['assign_ms'],4), 'kernel', round(r['kernel_ms'],4), d['clocks']['sm_mhz'])"
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:$re -s 4 -c 4 --csv \
      python bench.py --config $cfg --steps 2 --warmup 6 --no-graph --no-e2e --no-cpu-baseline "$@" 2>/dev/null \
      | python -c "
import csv,sys
rows=[r for r in csv.reader(l for l in sys.stdin if not l.startswith('==')) if len(r)>10]
h=rows[0]; vi=h.index('Metric Value')
print('$arm ncu us', [round(float(r[vi].replace(',',''))/1e3,1) for r in rows[1:]])"
  done
done
