"""Cycle accounting of the screen kernel (experiment builds, run with
PCB_LIB_PATH=build_exp/lib<tag>.so): PCB_EXP=14 — cycles the MMA warp spends waiting
for a free accumulator (tempty), the row pair's A tile (afull), a centroid stage
(full), and in total; PCB_EXP=15 — epilogue warps: waiting for an accumulator,
full-path chunks, pair-end bookkeeping, total."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import CONFIGS, make_shard
from paper_2501_05587_b200.engine import LloydEngine
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda"))
eng = LloydEngine(P, k, max_iters=30)
eng.init_labels_device(0); eng.init_centroids_from_labels(); eng.state.zero_()
for t in range(8):
    eng.iteration(t)
torch.cuda.synchronize()
big = torch.zeros(64, dtype=torch.int64, device="cuda")
big[:8] = eng.state
eng.state = big
eng.iteration(8)
torch.cuda.synchronize()
sms = torch.cuda.get_device_properties(0).multi_processor_count
w = big[8:12].cpu().numpy() / sms
if w[3] > 0:  # PCB_EXP=14: MMA warp
    print({"tempty": int(w[0]), "afull": int(w[1]), "full": int(w[2]), "total": int(w[3]),
           "busy(other)": int(w[3] - w[0] - w[1] - w[2])}, "MMA-warp cycles per CTA")
e = big[12:16].cpu().numpy() / (sms * 8)
if e[3] > 0:  # PCB_EXP=15: epilogue warps
    print({"tfull wait": int(e[0]), "full-path chunks": int(e[1]), "pair ends": int(e[2]), "total": int(e[3]),
           "other": int(e[3] - e[0] - e[1] - e[2])}, "cycles per epilogue warp")
