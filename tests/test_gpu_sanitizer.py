"""compute-sanitizer racecheck / synccheck / memcheck over small shapes of every
TMA, mbarrier and tcgen05 kernel (sanitizers in CI).  Each run goes
through tools/sanitize_driver.py, which also checks results against the oracle."""

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("family", ["forest", "svm", "linear"])
def test_sanitizer_clean(tool, family):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_driver.py"), family]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}_{family}.log"), "w") as fh:
        fh.write(out)
    assert r.returncode == 0 and f"ok {family}" in out, out[-3000:]
