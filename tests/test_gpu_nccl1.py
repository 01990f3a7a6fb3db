"""The multi-rank protocol over real NCCL on a one-GPU box.

NCCL refuses two ranks on one device, and gpurun / the round-end tiers give one
GPU, so the multi-rank path (NCCL all-reduce of the fused accumulator, the
device empty-cluster flag read with a lag, the batched host repair rounds, and
the all-reduce captured inside the CUDA graph bench.py times) is run here with
world_size 1 and PCB_FORCE_MULTI=1: every collective is issued through NCCL
on a one-rank communicator.  The fit must equal the single-rank driver's
(labels, objective history, repairs, centroids), and bench.py's multi-rank leg
must capture the NCCL all-reduce in its graph.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys, pickle
sys.path.insert(0, os.environ["PCB_ROOT"])
import numpy as np, torch
import oracle
import paper_2501_05587_b200 as pcb
from paper_2501_05587_b200.distributed import Comm, init_from_env, run_lloyd_sharded
init_from_env("nccl")
comm = Comm()
assert comm.world_size == 1 and comm.multi
out = {}
for name, (n, d, k, iters, variant) in {"blobs": (40000, 64, 48, 12, "auto"), "repair": (3000, 16, 600, 6, "auto"),
                                        "c3shape": (60000, 128, 256, 8, "fp8s")}.items():
    P = oracle.make_blobs(n, d, min(k, 50), seed=n + d)
    cfg = pcb.KKMeansConfig(k=k, max_iters=iters, variant=variant)
    a = run_lloyd_sharded(P, cfg, n, 0, comm)
    b = pcb.run_lloyd(P, pcb.KKMeansConfig(k=k, max_iters=iters, variant=variant))
    out[name] = (a.labels, b.labels, np.asarray(a.objective_history), np.asarray(b.objective_history),
                 a.repairs, b.repairs, a.centroids, b.centroids)
pickle.dump(out, open(os.environ["PCB_OUT"], "wb"))
"""


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _env(**extra):
    env = dict(os.environ, PCB_FORCE_MULTI="1", WORLD_SIZE="1", RANK="0", LOCAL_RANK="0",
               MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), PCB_ROOT=ROOT)
    env.update(extra)
    return env


def test_nccl_one_rank_fit_equals_single_rank(tmp_path):
    import pickle

    import numpy as np
    out = tmp_path / "fits.pkl"
    r = subprocess.run([sys.executable, "-c", WORKER], env=_env(PCB_OUT=str(out)), cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    fits = pickle.load(open(out, "rb"))
    for name, (la, lb, oa, ob, ra, rb, ca, cb) in fits.items():
        np.testing.assert_array_equal(la, lb, err_msg=name)
        np.testing.assert_array_equal(ra, rb, err_msg=name)
        # the one-rank all-reduce is a copy: the histories agree to the f64 sums
        np.testing.assert_allclose(oa, ob, rtol=1e-12, err_msg=name)
        np.testing.assert_allclose(ca, cb, rtol=1e-12, atol=1e-12, err_msg=name)


def test_bench_multi_rank_leg_captures_nccl(tmp_path):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c3", "--n-override", "300000", "--steps", "4",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-iters", "4"]
    r = subprocess.run(cmd, env=_env(NCCL_DEBUG_FILE=str(tmp_path / "nccl.%p.log")), cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "NCCL all-reduce captured" in line["config"]["launch"], line["config"]
    # NCCL's INIT lines reach the debug file when the communicator logs them;
    # with one rank they may be absent, but never a different rank count
    assert line["nccl"]["nranks"] in ([1], []), line["nccl"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
