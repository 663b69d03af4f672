"""bench.py's one-line JSON contract: the reference arm on CPU (the oracle's
C port needs no GPU) and our arm on a B200 (gpu marker), at the smallest
BASELINE config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout   # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "3"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["warmup"] >= 3


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"])
    assert BASE_KEYS <= set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    assert d["config"]["mode"] == "strict"
    assert d["gpu_launches"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 4 * 8 * 20_000 and e["d2h_bytes_per_step"] == 8 * 20_000
    acc = d["accuracy"]
    assert acc["vs_parity_frac_targets_above_1e-10"] == 0.0
