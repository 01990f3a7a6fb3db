timeout 900 python scripts/shard_probe.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 330 -c 75 --csv \
  --log-file gpurun_out/launches_shard8.csv python bench.py --config c3 --n-override 1250000 --steps 4 --warmup 12 --no-graph \
  --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(l for l in open("gpurun_out/launches_shard8.csv") if not l.startswith("==")))
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
seq = [(r[ki][:60], float(r[vi].replace(",", ""))) for r in rows[1:] if len(r) > vi]
t = collections.defaultdict(list)
for k, v in seq: t[k].append(v)
tot = sum(v for _, v in seq)
for k, v in sorted(t.items(), key=lambda x: -sum(x[1]))[:30]:
    print(f"{sum(v)/len(v)/1e3:9.3f} us x{len(v):3d}  {100*sum(v)/tot:5.1f}%  {k}")
PY
