"""compute-sanitizer memcheck / racecheck / synccheck over small factorizations
(SURVEY.md section 5): the kernels lean on DSMEM, mbarriers, st.async and
cp.async, so every tool must report zero errors on every kernel family
(tools/sanitize_case.py: qr_reg, qr_cluster, the cluster Jacobi at several
cluster widths, the grouped beta products, the rectangular driver, the step API)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"

MODES = {
    "default": {},
    "qr_cluster": {"RUTV_QR_KERNEL": "cluster"},
    "jacobi_cs4": {"RUTV_JACOBI_CS": "4"},
    "serial": {"RUTV_OVERLAP": "0"},
}


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("mode", sorted(MODES))
def test_sanitizer_clean(tool, mode):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not installed")
    if tool == "racecheck" and mode == "serial":
        pytest.skip("covered by the default mode")
    env = dict(os.environ, **MODES[mode])
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1200)
    text = out.stdout + out.stderr
    if "closed on this pool" in text:  # the GPU pool's wrapper refuses compute-sanitizer
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + text.strip().splitlines()[0][:200])
    assert out.returncode == 0, text[-4000:]
    assert "sanitize case ok" in text
    assert "ERROR SUMMARY: 0 errors" in text, text[-4000:]
