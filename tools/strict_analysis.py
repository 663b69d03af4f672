"""Where FAST breaks the strict per-target 1e-10 bar: |phi| of the violators
relative to max|phi| and rms, and how many targets a |phi| < tau max|phi|
filter would flag (C4)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2003_01836_b200 as bltc  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
system = bench.make_system(cfg, device=0)
econf = bench.eval_config(cfg, None, None)
ctx = bltc.Context(0)
phi_f, _ = ctx.treecode(system, econf, mode="fast")
phi_p, _ = ctx.treecode(system, econf, mode="parity")
d = np.abs(phi_f - phi_p)
rel = d / np.abs(phi_p)
bad = rel > 1e-10
mx, rms = np.abs(phi_p).max(), np.sqrt(np.mean(phi_p ** 2))
out = {"n": int(len(phi_p)), "violators": int(bad.sum()),
       "violator_abs_over_max_max": float((np.abs(phi_p[bad]) / mx).max()) if bad.any() else None,
       "violator_abs_over_rms_max": float((np.abs(phi_p[bad]) / rms).max()) if bad.any() else None,
       "abs_err_over_max": float(d.max() / mx), "max_over_rms": float(mx / rms),
       "flagged": {str(t): int((np.abs(phi_f) < t * mx).sum()) for t in (1e-6, 1e-5, 1e-4, 1e-3)}}
print(json.dumps(out))
