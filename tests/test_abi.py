"""The C-ABI library (CPU-side checks, no device calls): it builds, loads, and
exports every entry point include/bltc.h declares; the Python shim validates
arguments with the reference's exceptions before touching the device."""
import os
import re

import numpy as np
import pytest
from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_2003_01836_b200 import _lib, build_ext
    if not os.path.exists(_lib.LIB_PATH):
        build_ext.build()
    return _lib.load()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "bltc.h")).read()
    return sorted(set(re.findall(r"BLTC_API\s+[\w\s\*]+?\b(bltc_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("bltc_create", "bltc_destroy", "bltc_last_error", "bltc_treecode",
                 "bltc_treecode_device", "bltc_export_tree", "bltc_export_lists",
                 "bltc_export_moments", "bltc_rank_build", "bltc_rank_publish",
                 "bltc_rank_evaluate"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2003_01836_b200 import _lib
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.bltc_version().decode().startswith("libbltc")


def test_library_is_sm100a(lib):
    import subprocess
    from paper_2003_01836_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_null_context_is_a_value_error(lib):
    assert lib.bltc_destroy(None) == 0
    assert lib.bltc_set_timing(None, 1) == -1


def test_param_validation_matches_reference():
    """engine.py:56-62 and kernels.py:49-51 raise ValueError; so does the shim."""
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200.engine import make_params
    for bad in (dict(theta=0.0, degree=4), dict(theta=1.2, degree=4),
                dict(theta=0.5, degree=-1), dict(theta=0.5, degree=4, leaf_size=0),
                dict(theta=0.5, degree=4, batch_size=0)):
        with pytest.raises(ValueError):
            bltc.EvalConfig(**bad)
    with pytest.raises(ValueError):
        bltc.yukawa(-1.0)
    with pytest.raises(ValueError):
        bltc.yukawa(float("nan"))
    cfg = bltc.EvalConfig(theta=1.0, degree=0)
    p = make_params(cfg, "parity")
    assert p.mode == 0 and p.degree == 0 and p.theta == 1.0
    with pytest.raises(ValueError):
        make_params(cfg, "bogus")


def test_cheb_nodes_match_reference_form():
    from oracle.oracle import cheb_nodes as orc_nodes
    from paper_2003_01836_b200.engine import cheb_nodes
    for n in (0, 1, 2, 4, 8, 10, 13):
        np.testing.assert_array_equal(cheb_nodes(n), orc_nodes(n))


def test_plain_c_host_compiles_and_links(tmp_path, lib):
    """examples/treecode_c.c binds the C ABI with no Python / torch: the
    header compiles as C and the program links against libbltc.so."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    libdir = os.path.join(ROOT, "paper_2003_01836_b200")
    subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-O2",
                    f"-I{os.path.join(ROOT, 'include')}",
                    os.path.join(ROOT, "examples", "treecode_c.c"), "-o",
                    str(tmp_path / "treecode_c"), f"-L{libdir}", "-lbltc",
                    f"-Wl,-rpath,{libdir}", "-lm"], check=True)
