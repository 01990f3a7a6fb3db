"""Probe: ambiguous / overflow row counts and candidate-count histogram of the
bf16s screen over the first iterations at a bench config (run under gpurun)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import CONFIGS, make_shard
from paper_2501_05587_b200.engine import LloydEngine

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda"))
eng = LloydEngine(P, k, variant=sys.argv[2] if len(sys.argv) > 2 else "bf16s", max_iters=30)
eng.init_labels_device(0)
eng.init_centroids_from_labels()
for t in range(12):
    eng.iteration(t)
    torch.cuda.synchronize()
    amb = int(eng.amb_count.item())
    line = f"it {t} amb {amb} ({amb / n:.4f})"
    if hasattr(eng, "ovf_count"):
        ovf = int(eng.ovf_count.item())
        if amb <= eng.bypass:
            cn = eng.cand_n[:amb].cpu().numpy()
            h = np.bincount(np.minimum(cn, 40), minlength=41)
            line += f" ovf {ovf} cand_n hist {h.tolist()}"
        else:
            line += f" bypass ovf {ovf}"
    print(line, flush=True)
