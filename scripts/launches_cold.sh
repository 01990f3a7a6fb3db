#!/bin/bash
# Launch list (cold, serialised) of the first iterations of a c3 fit: init,
# iteration 0 (3xTF32 on every row) and iterations 1-3.
cfg=${1:-c3}; tag=${2:-cold_$cfg}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 150 --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --config $cfg --steps 1 --warmup 3 --no-graph \
  --no-e2e --no-cpu-baseline > gpurun_out/launches_$tag.log 2>&1
echo "ncu rc=$?"
python - "$tag" <<'PY'
import csv, sys
rows = list(csv.reader(l for l in open(f"gpurun_out/launches_{sys.argv[1]}.csv") if not l.startswith("==")))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
for r in rows[1:]:
    if len(r) > vi: print(f"{float(r[vi].replace(',', ''))/1e3:10.3f}  {r[ki][:80]}")
PY
