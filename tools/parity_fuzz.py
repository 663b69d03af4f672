#!/usr/bin/env python
"""PARITY / STRICT / FAST against the CPU oracle over random small
workloads, edge cases included: N from 1 to 30000, separate or coincident
targets, duplicated points, degree 0-20, theta in (0, 1], leaf / batch sizes
from 1, Coulomb / Yukawa / constant kernels.  PARITY must equal the oracle
bit for bit, STRICT within 1e-10 per target (relative, condition-aware for
|phi| = 0), FAST within 1e-10 of max |phi|.  Prints one JSON line per run
and a summary.

    python tools/parity_fuzz.py --runs 300 > profiles/r2_parity_fuzz.jsonl
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=300)
    ap.add_argument("--seed", type=int, default=31)
    args = ap.parse_args()
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200.particles import ParticleSystem, Points
    from oracle import oracle
    rng = np.random.default_rng(args.seed)
    ctx = bltc.Context(0)
    bad = {"parity": 0, "strict": 0, "fast": 0}
    for run in range(args.runs):
        n = int(rng.choice([1, 2, 3, 5, 17, 64, 300, 1000, 4000, 12000, 30000]))
        pts = rng.uniform(-1, 1, (n, 3))
        if n > 4 and rng.random() < 0.3:   # duplicated points
            k = int(rng.integers(1, n // 2 + 1))
            pts[-k:] = pts[:k]
        if n > 4 and rng.random() < 0.15:   # a flat slab (zero extent in z)
            pts[:, 2] = 0.25
        q = rng.uniform(-1, 1, n)
        coincident = rng.random() < 0.7
        if coincident:
            tp = pts
        else:
            nt = int(rng.choice([1, 7, 200, 1500]))
            tp = rng.uniform(-1.2, 1.2, (nt, 3))
        deg = int(rng.choice([0, 1, 2, 4, 8, 10, 12, 13, 16, 20]))
        theta = float(rng.choice([0.05, 0.3, 0.5, 0.7, 0.9, 1.0]))
        leaf = int(rng.choice([1, 2, 10, 100, 600]))
        batch = leaf if (coincident and rng.random() < 0.5) else int(rng.choice([1, 3, 50, 400]))
        kind = int(rng.choice([0, 0, 1, 2]))
        kappa = float(rng.choice([0.0, 0.5, 3.0])) if kind == 1 else 0.0
        kern = [bltc.coulomb(), bltc.yukawa(kappa), bltc.test_constant()][kind]
        src = Points.from_array(pts)
        tgt = src if coincident else Points.from_array(tp)
        system = ParticleSystem(targets=tgt, sources=src, charges=q)
        cfg = bltc.EvalConfig(theta=theta, degree=deg, leaf_size=leaf, batch_size=batch,
                              kernel=kern)
        ref, _ = oracle.treecode_potentials(tgt.x, tgt.y, tgt.z, src.x, src.y, src.z, q,
                                            coincident, theta, deg, leaf, batch, kind,
                                            kappa)
        rec = {"run": run, "n": n, "nt": len(tgt.x), "coincident": coincident, "degree": deg,
               "theta": theta, "leaf": leaf, "batch": batch, "kind": kind, "kappa": kappa}
        phi_p, _ = ctx.treecode(system, cfg, mode="parity")
        rec["parity_bitwise"] = bool(np.array_equal(phi_p, ref))
        phi_s, _ = ctx.treecode(system, cfg, mode="strict")
        scale = np.abs(ref).max() if len(ref) else 0.0
        d = np.abs(phi_s - ref)
        ok_s = bool(np.all((d <= 1e-10 * np.abs(ref)) | (d <= 1e-15 * scale)))
        rec["strict_ok"] = ok_s
        phi_f, _ = ctx.treecode(system, cfg, mode="fast")
        rec["fast_dev"] = float(np.abs(phi_f - ref).max() / scale) if scale > 0 else 0.0
        bad["parity"] += not rec["parity_bitwise"]
        bad["strict"] += not ok_s
        bad["fast"] += rec["fast_dev"] > 1e-10
        print(json.dumps(rec), flush=True)
    print(json.dumps({"summary": True, "runs": args.runs, "failures": bad}), flush=True)


if __name__ == "__main__":
    main()
