# Steady-state launch list with warm caches (ncu --cache-control none): per-kernel durations closer to graph replay
cfg=${1:-c3}; tag=${2:-warm_$cfg}; shift 2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s ${SKIP:-330} -c ${COUNT:-75} --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --config $cfg --steps 4 --warmup 12 --no-graph \
  --no-e2e --no-cpu-baseline "$@" > gpurun_out/launches_$tag.log 2>&1
echo "ncu rc=$?"
python - "$tag" <<'PY'
import csv, sys, collections
rows = list(csv.reader(l for l in open(f"gpurun_out/launches_{sys.argv[1]}.csv") if not l.startswith("==")))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
seq = [(r[ki][:70], float(r[vi].replace(",", ""))) for r in rows[1:] if len(r) > vi]
t = collections.defaultdict(list)
for k, v in seq: t[k].append(v)
tot = sum(v for _, v in seq)
for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v)/len(v)/1e3:9.3f} us x{len(v):3d}  {100*sum(v)/tot:5.1f}%  {k}")
print(f"total {tot/1e3:.1f} us over {len(seq)} launches")
PY
