"""The C ABI from plain C (examples/treecode_c.c): no Python or torch in the
process -- treecode potentials against a brute-force sum, FAST vs PARITY."""
import json
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_host_program(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    libdir = os.path.join(ROOT, "paper_2003_01836_b200")
    exe = str(tmp_path / "treecode_c")
    subprocess.run([gcc, "-O2", f"-I{os.path.join(ROOT, 'include')}",
                    os.path.join(ROOT, "examples", "treecode_c.c"), "-o", exe, f"-L{libdir}",
                    "-lbltc", f"-Wl,-rpath,{libdir}", "-lm"], check=True)
    r = subprocess.run([exe, "30000"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["rel_l2_error"] < 1e-4 and out["fast_vs_parity"] < 1e-13
    assert out["strict_max_rel"] <= 1e-10
    assert out["ranks2_rel_l2_error"] < 1e-4
