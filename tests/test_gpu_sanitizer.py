"""compute-sanitizer memcheck / racecheck / initcheck over every C-ABI entry
point on small ragged inputs (tools/sanitize_run.py)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "initcheck"])
def test_compute_sanitizer(tool):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    cmd = [cs, "--tool", tool, "--error-exitcode", "3"]  # initcheck: unused-memory tracking is off by default
    r = subprocess.run(cmd + [sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-3000:]
    if r.returncode != 0 and "closed on this pool" in tail:
        # the pool's wrapper refuses compute-sanitizer; tests/test_gpu_guard_bands.py covers
        # out-of-bounds writes with canary regions around every output instead
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0 and "sanitize_run ok" in r.stdout, tail
    out = r.stdout + r.stderr
    assert ("ERROR SUMMARY: 0 errors" in out) or ("SUMMARY: 0 hazards displayed (0 errors" in out), tail
