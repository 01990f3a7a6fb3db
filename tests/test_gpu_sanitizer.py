"""compute-sanitizer over the mbarrier / TMEM pipelines:
racecheck (shared-memory hazards), synccheck (barrier misuse) and memcheck on a
small fit through each tensor-core assignment kernel and the update/repair
kernels it drives.  Each run must report zero errors."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs a B200")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

CASES = [("fp8s", 3000, 96, 40), ("bf16s", 3000, 96, 40), ("tc3xtf32", 2000, 96, 40), ("deltatc", 1000, 40, 20),
         ("rowreg", 3000, 16, 20), ("tc1xtf32s", 2000, 96, 40)]


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_sanitizer_clean(tool, case):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    variant, n, d, k = case
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", sys.executable,
           os.path.join(ROOT, "tests", "sanitize_fit.py"), variant, str(n), str(d), str(k)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    print(out[-3000:])
    if r.returncode == 86 and "closed" in out:
        # the GPU pool's compute-sanitizer wrapper refuses to run (it has left
        # GPUs needing a reset); the tool's verdict is then simply unavailable
        pytest.skip("compute-sanitizer refused by this GPU pool: " + out.strip().splitlines()[0][:120])
    assert r.returncode == 0, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
