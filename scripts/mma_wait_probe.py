"""MMA-warp wait accounting of the screen kernel (experiment build PCB_EXP=14, run with
PCB_LIB_PATH=build_exp/libe14.so): cycles the MMA warp spends waiting for a free
accumulator (tempty), the row pair's A tile (afull), a centroid stage (full), and in total."""
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
w = big[8:12].cpu().numpy() / torch.cuda.get_device_properties(0).multi_processor_count
print({"tempty": int(w[0]), "afull": int(w[1]), "full": int(w[2]), "total": int(w[3]),
       "busy(other)": int(w[3] - w[0] - w[1] - w[2])}, "cycles per CTA")
