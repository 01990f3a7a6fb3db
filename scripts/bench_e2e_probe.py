"""bench.py (default args) with per-phase wall timers on the e2e leg (diagnostic, under gpurun)."""
import sys, os, time, functools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2501_05587_b200 import engine as E

T = {}
def timed(name, f):
    @functools.wraps(f)
    def w(*a, **kw):
        torch.cuda.synchronize(); t = time.perf_counter()
        r = f(*a, **kw)
        torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t
        return r
    return w
for nm in ("__init__", "init_labels_device", "init_centroids_from_labels", "run", "collect"):
    setattr(E.LloydEngine, nm, timed(nm, getattr(E.LloydEngine, nm)))
orig = bench.e2e_run
def e2e(*a, **kw):
    T.clear()
    r = orig(*a, **kw)
    print("e2e phases ms", {k_: round(v * 1e3, 1) for k_, v in T.items()}, r["wall_s"], file=sys.stderr, flush=True)
    return r
bench.e2e_run = e2e
sys.argv = ["bench.py", "--no-cpu-baseline"] + sys.argv[1:]
bench.main()
