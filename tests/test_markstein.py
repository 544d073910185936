"""The exhaustive binary16 quotient check behind k_norm2's binary32 path
(tools/check_markstein.c): Markstein's corrected product equals RN32(w/m)
for every binary16 pair 0 <= w <= m."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_markstein_binary16_exhaustive(tmp_path):
    exe = tmp_path / "mk"
    subprocess.run(["gcc", "-O2", "-mfma", "-fopenmp", "-ffp-contract=off",
                    os.path.join(ROOT, "tools", "check_markstein.c"), "-o", str(exe), "-lm"], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=600).stdout
    assert "mismatches=0" in out, out
