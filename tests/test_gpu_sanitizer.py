"""compute-sanitizer memcheck, synccheck and initcheck over a
tiny run of every ABI entry point (scripts/sanitize_tiny.py: attention fwd +
bwd uniform / varlen / trace replay / d = 64, fused and two-pass logprob, DiPO,
LM head fwd + bwd, decode attention + select) must report 0 errors.
(racecheck is run for the record -- profiles/r01_sanitizer.txt -- but it does
not model mbarrier-ordered async-proxy copies, so it is not asserted.)"""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "synccheck", "initcheck"])
def test_sanitizer_clean(cuda_ok, tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([exe, "--tool", tool, "--print-limit", "20", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize_tiny.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    assert "sanitize run ok" in out, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
