"""Where does the host-side time of run_lloyd(host numpy) go at c3? (diagnostic)"""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from bench import make_shard
n, d, k = 10_000_000, 128, 1024
P = make_shard(n, d, k, 0, 0, torch.device('cuda')).cpu().numpy()
torch.cuda.synchronize()
def t(label, fn):
    t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize(); print(f"{label:40s} {time.perf_counter()-t0:8.3f} s", flush=True); return r
t("np.isfinite.all", lambda: np.isfinite(P).all())
t("ascontiguousarray", lambda: np.ascontiguousarray(P, dtype=np.float32))
from paper_2501_05587_b200.clustering import init_assignments
t("init_assignments", lambda: init_assignments(n, k, 0))
t("pageable .to(cuda)", lambda: torch.from_numpy(P).to('cuda'))
t("pin_memory copy", lambda: torch.from_numpy(P).pin_memory())
def reg():
    hp = torch.from_numpy(P)
    cudart = torch.cuda.cudart()
    r = cudart.cudaHostRegister(hp.data_ptr(), hp.numel() * 4, 0)
    g = hp.to('cuda', non_blocking=True); torch.cuda.synchronize()
    cudart.cudaHostUnregister(hp.data_ptr())
    return r
t("hostRegister+copy+unregister", reg)
def staged(chunk=1 << 26):
    dst = torch.empty((n, d), dtype=torch.float32, device='cuda')
    flat = torch.from_numpy(P).view(-1); dflat = dst.view(-1)
    bufs = [torch.empty(chunk, dtype=torch.float32).pin_memory() for _ in range(2)]
    evs = [torch.cuda.Event() for _ in range(2)]
    s = torch.cuda.Stream()
    for i, off in enumerate(range(0, flat.numel(), chunk)):
        b = i & 1
        evs[b].synchronize()
        m = min(chunk, flat.numel() - off)
        bufs[b][:m].copy_(flat[off:off + m])
        with torch.cuda.stream(s):
            dflat[off:off + m].copy_(bufs[b][:m], non_blocking=True)
            evs[b].record(s)
    s.synchronize()
    return dst
t("staged 2x256MB pinned", staged)
import paper_2501_05587_b200 as pcb
cfg = pcb.KKMeansConfig(k=k, max_iters=30, record_label_history=False)
t("run_lloyd total", lambda: pcb.run_lloyd(P, cfg))
