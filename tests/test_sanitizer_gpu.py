"""compute-sanitizer memcheck / racecheck / synccheck over a small workload
of every kernel family (scripts/sanitize_small.py): the hand-rolled mbarrier
rings, TMEM allocation, PDL launches, the fused conv's grid-wide finalize and
the engine's cross-stream slot fences must run clean."""

import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all",
           "python", os.path.join(ROOT, "scripts", "sanitize_small.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed on this pool" in out:
        # the GPU pool's wrapper refuses sanitizer runs (they left GPUs
        # needing a reset); the same workload still runs plain below
        r2 = subprocess.run(["python", os.path.join(ROOT, "scripts", "sanitize_small.py")],
                            cwd=ROOT, capture_output=True, text=True, timeout=600)
        assert r2.returncode == 0 and "sanitize workload ok" in r2.stdout, r2.stderr[-4000:]
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip()[:200])
    log = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(log):
        with open(os.path.join(log, f"sanitizer_{tool}.log"), "w") as f:
            f.write(out)
    assert r.returncode == 0, out[-4000:]
    assert "sanitize workload ok" in out
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
