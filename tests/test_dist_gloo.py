"""Multi-rank Lloyd on CPU with gloo (world sizes 2 and 3).

Runs the shared per-rank iteration sequence (engine.ShardSequence) and the
global repair protocol (distributed.repair_protocol) with the numpy test
double of the kernels, one process per rank, and checks that the row-sharded
run reproduces the single-rank run exactly (labels, objective history,
repairs, centroids) — including empty-cluster repair with global lowest-index
tie breaks across shard boundaries.
"""
import os
import pickle
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from conftest import make_rng


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_single(case):
    """world_size 1 in-process (same shared sequence, LocalComm for repair)."""
    from cpu_shard import NumpyShard
    P, k, iters, seed, cc, tol = case
    n = P.shape[0]
    labels0 = oracle.init_assignments(n, k, seed)
    C0 = oracle.mean_centroids_f64(P, labels0, k)
    res = NumpyShard(P, k, n, 0, None, labels0, C0, iters).fit(iters, cc, tol)
    return res, res["labels"], [res]


def _run(world, case, tmp_path):
    import dist_worker
    if world == 1:
        return _run_single(case)
    out = tmp_path / f"ws{world}"
    out.mkdir()
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=dist_worker.run, args=(r, world, port, case, str(out))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    parts = [pickle.load(open(out / f"rank{r}.pkl", "rb")) for r in range(world)]
    labels = np.concatenate([p["labels"] for p in parts])
    return parts[0], labels, parts


def _cases():
    g = make_rng(21)
    centers = g.uniform(-5, 5, size=(6, 4))
    blobs = centers[g.integers(0, 6, size=501)] + g.normal(0, 0.7, size=(501, 4))
    h = make_rng(22)
    dup = np.vstack([np.zeros((150, 3)), h.normal(0.0, 4.0, size=(61, 3))])
    h.shuffle(dup)
    return {
        "blobs": (blobs, 6, 12, 3, False, 0.0),
        "repair_heavy": (dup, 40, 8, 1, False, 0.0),
        "converging": (blobs, 5, 50, 7, True, 0.0),
    }


@pytest.mark.parametrize("name", ["blobs", "repair_heavy", "converging"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_single_rank(name, world, tmp_path):
    case = _cases()[name]
    ref, ref_labels, _ = _run(1, case, tmp_path)
    got, labels, parts = _run(world, case, tmp_path)
    assert all(p["iters"] == ref["iters"] for p in parts)
    np.testing.assert_array_equal(labels, ref_labels)
    np.testing.assert_allclose(got["objective"], ref["objective"], rtol=1e-12)
    np.testing.assert_array_equal(got["repairs"], ref["repairs"])
    for p in parts:  # replicated centroids are identical on every rank
        np.testing.assert_array_equal(p["centroids"], got["centroids"])
    np.testing.assert_allclose(got["centroids"], ref["centroids"], rtol=1e-12, atol=1e-12)
    assert got["converged"] == ref["converged"]
    if name == "repair_heavy":
        assert ref["repairs"].sum() > 0


def test_single_rank_double_matches_reference_oracle(tmp_path):
    """The CPU double itself follows the reference (f64, clustering.py:291-325)."""
    P, k, iters, seed, cc, tol = _cases()["blobs"]
    ref = oracle.run_lloyd(P, k, max_iters=iters, seed=seed, dtype=np.float64)
    got, labels, _ = _run(1, _cases()["blobs"], tmp_path)
    np.testing.assert_array_equal(labels, ref.labels)
    np.testing.assert_allclose(got["objective"], ref.objective_history, rtol=1e-9)


def test_shard_ranges_cover_rows():
    from paper_2501_05587_b200.distributed import shard_range
    for n in (1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
