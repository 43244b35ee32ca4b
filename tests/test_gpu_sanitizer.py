"""compute-sanitizer over the layer kernels (front in both GEMM modes, the
router kernel, the FFN in dense and routed mode, both combines): no shared-
memory hazard (racecheck) and no barrier misuse (synccheck). Round 2 found a
real race of the kind it looks for (DES-Seq coreset flags zeroed and set without a
barrier, tools/c6_stress.py)."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool", ["racecheck", "synccheck"])
def test_layer_kernels_sanitizer_clean(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    cmd = [cs, "--tool", tool]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "racecheck_front.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, out[-4000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]
