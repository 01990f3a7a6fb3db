#!/bin/bash
# A/B of library builds in one box session: scripts/ab.sh "<bench args>" lib1.so lib2.so ...
# prints kernel_ms / ms_per_step / value per run (alternating, twice).
args=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    out=$(PCB_LIB_PATH=$lib timeout 300 python bench.py $args --no-e2e --no-cpu-baseline 2>&1 | tail -1)
    python - "$lib" "$out" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2]); r = d["roofline"]
    print(f"{sys.argv[1]:40s} kernel_ms={r['kernel_ms']:.4f} ms/step={d['ms_per_step']:.4f} value={d['value']:.2f} mhz={d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", sys.argv[2][:300])
PY
  done
done
