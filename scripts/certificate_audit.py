"""Full-size certificate audit of the default screen (tests/audit.py).

    python scripts/certificate_audit.py --config c3 --iters 30 [--variant fp8s] > gpurun_out/audit_c3.jsonl

Same synthetic data as bench.py (make_shard), same fit as run_lloyd
(device init_assignments, initial means, then the Lloyd loop with the
benchmark's relayouts / delta updates); every iteration's pre-repair labels of
ALL rows are compared with the exact argmin.  One JSON line per iteration,
then a summary line.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import torch  # noqa: E402

from bench import CONFIGS, make_shard  # noqa: E402
from audit import audit_fit  # noqa: E402
from paper_2501_05587_b200.engine import LloydEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
ap.add_argument("--iters", type=int, default=30)
ap.add_argument("--variant", default="auto")
ap.add_argument("--n", type=int, default=0)
args = ap.parse_args()
cfg = dict(CONFIGS[args.config])
if args.n:
    cfg["n"] = args.n
n, d, k = cfg["n"], cfg["d"], cfg["k"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
P = make_shard(n, d, k, 0, 0, dev)
eng = LloydEngine(P, k, variant=args.variant, max_iters=args.iters + 1)
eng.init_labels_device(0)
eng.init_centroids_from_labels()
t0 = time.time()
rows = audit_fit(eng, args.iters, log=lambda r: print(json.dumps(r), flush=True))
print(json.dumps({"summary": True, "config": args.config, "n": n, "d": d, "k": k, "variant": eng.variant,
                  "iterations": args.iters, "rows_audited": n * args.iters,
                  "violations": sum(r["violations"] for r in rows),
                  "resolver_mismatches": sum(r["resolver_mismatches"] for r in rows),
                  "max_rel_gap_of_mismatch": max(r["max_rel_gap_of_mismatch"] for r in rows),
                  "wall_s": time.time() - t0}), flush=True)
