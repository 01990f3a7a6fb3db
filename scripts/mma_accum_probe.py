"""Record the tensor-core accumulation probe table (tests/mma_probe_cases.py)
as JSON lines: python scripts/mma_accum_probe.py > gpurun_out/mma_probe.jsonl"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import mma_probe_cases as M  # noqa: E402

for name, steps, init, m in M.all_cases():
    print(json.dumps(M.measure(name, steps, init, m)), flush=True)
