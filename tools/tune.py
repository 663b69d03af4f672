"""Time the tuned FAST-kernel variants (BLTC_FAR / BLTC_NEAR = "tpt,minb")."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2003_01836_b200 as bltc  # noqa: E402

VARIANTS = [("2,2", "2,2", "0"), ("2,2", "2,2", "1"), ("2,3", "2,3", "0"), ("1,4", "1,4", "0"),
            ("3,2", "2,4", "0")]
configs = sys.argv[1:] or ["c4"]
ctx = bltc.Context(0)
for name in configs:
    cfg = bench.CONFIGS[name]
    system = bench.make_system(cfg)
    econf = bench.eval_config(cfg, None, None)
    os.environ["BLTC_FAR"] = "2,2"
    os.environ["BLTC_NEAR"] = "2,2"
    os.environ["BLTC_FORM"] = "0"
    ref, _ = ctx.treecode(system, econf, mode="fast")
    scale = np.abs(ref).max()
    for far, near, form in VARIANTS:
        os.environ["BLTC_FAR"] = far
        os.environ["BLTC_NEAR"] = near
        os.environ["BLTC_FORM"] = form
        best = None
        for _ in range(2):
            phi, st = ctx.treecode(system, econf, mode="fast")
            if best is None or st.far_s + st.near_s < best.far_s + best.near_s:
                best = st
        dev = float(np.abs(phi - ref).max() / scale)
        print(json.dumps({"config": name, "far": far, "near": near, "form": form,
                          "far_ms": best.far_s * 1e3, "near_ms": best.near_s * 1e3,
                          "far_frac": 2 * 7 * best.approx_pairs / best.far_s / 34.2e12,
                          "near_frac": 2 * 12 * best.direct_pairs / best.near_s / 34.2e12,
                          "dev": dev}), flush=True)
