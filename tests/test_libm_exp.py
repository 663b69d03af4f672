"""The device port of the host exp (csrc/libm_exp.cuh) -- the exp the
reference's Yukawa tiles reach through numba's math.exp (engine.py:190-191,
243) -- compiled for the host and compared with the C library's exp bit for
bit (CPU test); tests/test_gpu_strict.py compares the device build."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_generated_table_is_current():
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen", os.path.join(ROOT, "tools",
                                                                      "gen_exp_table.py"))
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    with open(os.path.join(ROOT, "paper_2003_01836_b200", "csrc", "libm_exp_table.h")) as f:
        text = f.read()
    for v in gen.table():
        assert "0x%016xull" % v in text


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_port_matches_host_libm_bitwise(tmp_path):
    exe = tmp_path / "lec"
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off",
                    "-I", os.path.join(ROOT, "paper_2003_01836_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "libm_exp_check.cpp"), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe), "2000000", "3"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout
