#!/usr/bin/env python
"""Bitwise upward pass (STRICT / PARITY moments) variants on one workload:
the big-cluster threshold (BLTC_BW_BIG).  (Earlier sweeps in
profiles/r2_moments_sweep*.jsonl also covered a thread-block-cluster /
DSMEM variant, its ring depth and the mbarrier suspend hint.)
Prints the precompute (moments) phase per variant, STRICT mode.

    python tools/moments_sweep.py --config c4
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import paper_2003_01836_b200 as bltc
    cfg = bench.CONFIGS[args.config]
    econf = bench.eval_config(cfg, None, None)
    system = bench.make_system(cfg, device=0)
    ctx = bltc.Context(0)
    ref = None
    variants = [{}]
    for big in ("65536", "262144", "524288"):
        variants.append({"BLTC_BW_BIG": big})
    # (profiles/r2_moments_sweep6_split_*.jsonl also compared split-kernel
    # launch configurations through a since-removed switch, "BLTC_BW_SPLIT"
    # 1 / 2 / 3 = producers, ring slots, CTAs per SM 4 / 8 / 2 (now the
    # default), 4 / 16 / 1, 2 / 8 / 2, against 8 / 16 / 1 ({})
    for v in variants:
        os.environ.update(v)
        ts = []
        for _ in range(args.reps):
            phi, st = ctx.treecode(system, econf, mode="strict")
            ts.append(st.precompute_s)
        for k in v:
            del os.environ[k]
        if ref is None:
            ref = phi
        print(json.dumps({"config": args.config, "env": v, "precompute_s": float(np.median(ts)),
                          "same_result": bool(np.array_equal(phi, ref))}), flush=True)


if __name__ == "__main__":
    main()
