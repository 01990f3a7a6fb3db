"""Where does run_lloyd(host numpy) spend its wall time at a bench config? (diagnostic, under gpurun)"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import CONFIGS, make_shard
import paper_2501_05587_b200 as pcb
from paper_2501_05587_b200 import clustering as cl
from paper_2501_05587_b200.engine import LloydEngine

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
n, d, k = cfg["n"], cfg["d"], cfg["k"]
P = make_shard(n, d, k, 0, 0, torch.device("cuda")).cpu().numpy()
pcb.run_lloyd(P[:100000], pcb.KKMeansConfig(k=k, max_iters=2))
torch.cuda.synchronize()
for rep in range(int(os.environ.get("REPS", "1"))):
    T = {}
    def tic(): torch.cuda.synchronize(); return time.perf_counter()
    t0 = tic()
    c = pcb.KKMeansConfig(k=k, max_iters=30, record_label_history=False)
    Pp, _, _ = cl._prepare_points(P, c); t1 = tic(); T["prepare/validate"] = t1 - t0
    eng = LloydEngine(Pp, k, max_iters=30, check_finite=True, variant=os.environ.get("VARIANT", "auto")); t2 = tic(); T["engine init (H2D + prep)"] = t2 - t1
    eng.init_labels_device(0); t3 = tic(); T["init labels"] = t3 - t2
    eng.init_centroids_from_labels(); t4 = tic(); T["init centroids"] = t4 - t3
    eng.state.zero_()
    ts = []
    for t in range(30):
        a = tic(); eng.iteration(t); ts.append(tic() - a)
        if hasattr(eng, "amb_count") and t < 6 and rep == 0:
            print(t, "amb", int(eng.amb_count.item()), "two", int(eng.two_count.item()) if hasattr(eng, "two_count") else None,
                  "ovf", int(eng.ovf_count.item()) if hasattr(eng, "ovf_count") else None, flush=True)
    t5 = tic(); T["30 iterations"] = t5 - t4
    out = eng.collect(); t6 = tic(); T["collect (D2H)"] = t6 - t5
    del eng
    for k_, v in T.items(): print(f"{k_:28s} {v*1e3:9.2f} ms")
    print("per-iteration ms:", [round(x * 1e3, 2) for x in ts], flush=True)
