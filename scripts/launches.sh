#!/bin/bash
# Per-kernel launch list (cold, serialised) of a short bench run under ncu.
# usage: scripts/launches.sh [config] [variant] [tag]
cfg=${1:-c3}; variant=${2:-auto}; tag=${3:-${cfg}_${variant}}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 80 -c 80 --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --config $cfg --variant $variant --steps 3 --warmup 3 --no-graph $EXTRA \
  --no-e2e --no-cpu-baseline > gpurun_out/launches_$tag.log 2>&1
echo "ncu rc=$?"
python - "$tag" <<'PY'
import csv, sys, collections
rows = list(csv.reader(l for l in open(f"gpurun_out/launches_{sys.argv[1]}.csv") if not l.startswith("==")))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
t = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) > vi: t[r[ki][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in t.values())
for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v)/len(v)/1e3:9.3f} us x{len(v):3d}  {100*sum(v)/tot:5.1f}%  {k}")
PY
