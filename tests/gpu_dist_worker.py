"""Worker for the multi-rank GPU engine test: every rank drives its own
LloydEngine on cuda:0, ranks talk through gloo (NCCL cannot put two ranks on
one GPU; the engine code path above the collective is identical)."""
import os
import pickle
import sys


def run(rank, world, port, case, out_dir):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2501_05587_b200 as pcb
    from paper_2501_05587_b200.distributed import Comm, run_lloyd_sharded, shard_range

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    P, k, iters, variant = case
    n = P.shape[0]
    lo, hi = shard_range(n, rank, world)
    cfg = pcb.KKMeansConfig(k=k, max_iters=iters, variant=variant)
    res = run_lloyd_sharded(np.ascontiguousarray(P[lo:hi]), cfg, n, lo, Comm())
    out = {"labels": res.labels, "obj": res.objective_history, "rep": res.repairs, "C": res.centroids,
           "lo": lo, "hi": hi}
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)
    dist.barrier()
    dist.destroy_process_group()
