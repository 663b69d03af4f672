#!/usr/bin/env python
"""Small evaluations covering every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize.py

PARITY / FAST / STRICT (forced recompute too), Coulomb / Yukawa, packed and
per-batch kernels, near-field bulk staging, the bitwise upward pass with its
big-cluster split items forced on (BLTC_BW_BIG), simulated
ranks (multi-group forest), the direct-sum oracle and the C host ABI paths."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_01836_b200 as bltc  # noqa: E402
from paper_2003_01836_b200 import cli  # noqa: E402
from paper_2003_01836_b200.decomp import run_distributed  # noqa: E402

os.environ.setdefault("BLTC_BW_BIG", "700")   # big-cluster kernels at this small N
s = cli.generate_plummer(6000, 3)
u = cli.generate_particles(5000, 4)
ctx = bltc.Context(0)
runs = [
    (s, dict(theta=0.8, degree=8, leaf_size=400, batch_size=160)),
    (u, dict(theta=0.7, degree=4, leaf_size=300, batch_size=300)),
    (u, dict(theta=0.7, degree=10, leaf_size=500, batch_size=100,
             kernel=bltc.yukawa(0.5))),
]
for system, kw in runs:
    cfg = bltc.EvalConfig(**kw)
    ref, _ = ctx.treecode(system, cfg, mode="parity")
    for mode in ("fast", "strict"):
        phi, st = ctx.treecode(system, cfg, mode=mode)
        assert np.abs(phi - ref).max() <= 1e-12 * np.abs(ref).max(), mode
    os.environ["BLTC_STRICT_KC"] = "1e300"
    phi, st = ctx.treecode(system, cfg, mode="strict")
    del os.environ["BLTC_STRICT_KC"]
    assert np.array_equal(phi, ref)
    os.environ["BLTC_NEAR_BULK"] = "1"
    ctx.treecode(system, cfg, mode="fast")
    del os.environ["BLTC_NEAR_BULK"]
    os.environ["BLTC_PACK"] = "0"
    ctx.treecode(system, cfg, mode="fast")
    del os.environ["BLTC_PACK"]
    print("ok", kw, flush=True)
cfg = bltc.EvalConfig(theta=0.8, degree=5, leaf_size=300, batch_size=300)
for mode in ("parity", "fast", "strict"):
    run_distributed(s, cfg, ranks=3, mode=mode)
ctx.direct_sum(s, bltc.coulomb(), np.arange(0, 6000, 37), mode="parity")
ctx.direct_sum(s, bltc.coulomb(), np.arange(0, 6000, 37), mode="fast")
cfg = bltc.EvalConfig(theta=0.8, degree=3, leaf_size=200, batch_size=200,
                      kernel=bltc.test_constant())
ctx.treecode(u, cfg, mode="strict")
# Yukawa: shifted-exponential (YS) far / near kernels and their fallbacks
for kappa in (0.5, 40.0):
    ycfg = bltc.EvalConfig(theta=0.7, degree=8, leaf_size=500, batch_size=160,
                           kernel=bltc.yukawa(kappa))
    for mode in ("fast", "strict"):
        ctx.treecode(u, ycfg, mode=mode)
print("sanitize workload done", flush=True)
