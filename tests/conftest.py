"""Shared test setup.

* registers the ``gpu`` marker (tests that need a B200; run with -m gpu)
* puts the repo root on sys.path so ``oracle`` and the package import
* ``golden(name)`` loads a fixture produced by the reference itself
  (tests/golden/make_golden.py)
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as f:
        return {k: f[k] for k in f.files}


def golden_system(g):
    from paper_2003_01836_b200 import cli
    gen = str(g["gen"])
    if gen == "uniform":
        return cli.generate_particles(int(g["n"]), int(g["seed"]))
    return cli.generate_plummer(int(g["n"]), int(g["seed"]))


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as orc
    orc.build()
    return orc
