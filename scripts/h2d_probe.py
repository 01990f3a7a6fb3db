"""H2D strategies for a 5.12 GB pageable numpy array (diagnostic, run under gpurun)."""
import sys, time, threading
import numpy as np, torch
n, d = 10_000_000, 128
P = np.random.default_rng(0).standard_normal((n, d), dtype=np.float32)
torch.cuda.init()
dst = torch.empty((n, d), dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
def t(label, fn, reps=2):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"{label:44s} {best:7.3f} s  {P.nbytes / best / 1e9:6.1f} GB/s", flush=True)
t("pageable copy_", lambda: dst.copy_(torch.from_numpy(P)))
def staged(chunk_mb, nbuf, nthreads):
    flat = torch.from_numpy(P).view(-1); dflat = dst.view(-1)
    chunk = chunk_mb << 18
    bufs = [torch.empty(chunk, dtype=torch.float32).pin_memory() for _ in range(nbuf)]
    s = torch.cuda.Stream()
    evs = [torch.cuda.Event() for _ in range(nbuf)]
    offs = list(range(0, flat.numel(), chunk))
    torch.set_num_threads(nthreads)
    def run():
        for i, off in enumerate(offs):
            b = i % nbuf
            evs[b].synchronize()
            m = min(chunk, flat.numel() - off)
            bufs[b][:m].copy_(flat[off:off + m])
            with torch.cuda.stream(s):
                dflat[off:off + m].copy_(bufs[b][:m], non_blocking=True)
                evs[b].record(s)
        s.synchronize()
    return run
for cm, nb, nt in [(128, 2, 16), (64, 4, 16), (32, 4, 32), (256, 3, 32), (64, 6, 8)]:
    t(f"staged {cm}MB x{nb} threads={nt}", staged(cm, nb, nt))
def threaded_staged(chunk_mb=64, nw=8):
    flat = torch.from_numpy(P).view(-1); dflat = dst.view(-1)
    chunk = chunk_mb << 18
    offs = list(range(0, flat.numel(), chunk))
    bufs = [torch.empty(chunk, dtype=torch.float32).pin_memory() for _ in range(nw)]
    streams = [torch.cuda.Stream() for _ in range(nw)]
    def work(w):
        torch.set_num_threads(1)
        for i in range(w, len(offs), nw):
            off = offs[i]; m = min(chunk, flat.numel() - off)
            streams[w].synchronize()
            bufs[w][:m].copy_(flat[off:off + m])
            with torch.cuda.stream(streams[w]):
                dflat[off:off + m].copy_(bufs[w][:m], non_blocking=True)
        streams[w].synchronize()
    def run():
        th = [threading.Thread(target=work, args=(w,)) for w in range(nw)]
        [x.start() for x in th]; [x.join() for x in th]
    return run
for cm, nw in [(64, 8), (32, 16), (128, 8)]:
    t(f"threaded staged {cm}MB workers={nw}", threaded_staged(cm, nw))
def register():
    hp = torch.from_numpy(P)
    cudart = torch.cuda.cudart()
    cudart.cudaHostRegister(hp.data_ptr(), hp.numel() * 4, 0)
    dst.copy_(hp, non_blocking=True); torch.cuda.synchronize()
    cudart.cudaHostUnregister(hp.data_ptr())
t("hostRegister whole + copy", register)
import os
print("cpus", os.cpu_count(), "torch threads", torch.get_num_threads())
