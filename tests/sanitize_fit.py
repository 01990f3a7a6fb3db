"""One small Lloyd fit per assignment variant, for compute-sanitizer runs
(tests/test_gpu_sanitizer.py).  Usage: python tests/sanitize_fit.py <variant> [n d k]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2501_05587_b200 as pcb  # noqa: E402

variant = sys.argv[1]
n, d, k = (int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (3000, 96, 40)
P = oracle.make_blobs(n, d, k, seed=3)
res = pcb.run_lloyd(P, pcb.KKMeansConfig(k=k, max_iters=4, variant=variant))
ref = oracle.run_lloyd(P, k, max_iters=4)
ok = abs(res.objective_history[-1] - ref.objective_history[-1]) <= 1e-5 * abs(ref.objective_history[-1])
print(f"sanitize_fit {variant} n={n} d={d} k={k} iterations={res.iterations_run} objective_ok={ok}")
sys.exit(0 if ok else 3)
