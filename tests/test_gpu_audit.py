"""Certificate audit at moderate size: every row of every iteration of real
fits (benchmark regime) against the exact argmin (tests/audit.py).  The
full-size c3 / c5 audit is scripts/certificate_audit.py (profiles/)."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SHAPES = {
    "c3_like": (1_000_000, 128, 1024, 16, "fp8s"),
    "c5_like": (400_000, 64, 4096, 12, "fp8s"),
    "c4_like": (200_000, 784, 256, 12, "fp8s"),
    "bf16_c3_like": (500_000, 128, 1024, 10, "bf16s"),
    "bf16_d48": (300_000, 48, 512, 12, "bf16s"),
}


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_certificate_audit(shape):
    from audit import audit_fit
    from bench import make_shard
    from paper_2501_05587_b200.engine import LloydEngine
    n, d, k, iters, variant = SHAPES[shape]
    P = make_shard(n, d, k, 0, 3, torch.device("cuda", 0))
    eng = LloydEngine(P, k, variant=variant, max_iters=iters + 1)
    eng.init_labels_device(0)
    eng.init_centroids_from_labels()
    rows = audit_fit(eng, iters)
    # every label is the exact argmin: certified rows, the exact candidate
    # stage and the 3xTF32 resolver with its exact near-tie pass alike
    assert sum(r["violations"] + r["resolver_mismatches"] for r in rows) == 0, rows
    assert rows[-1]["ambiguous"] + rows[-1]["two_candidate"] < 0.2 * n, rows
