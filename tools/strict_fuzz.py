#!/usr/bin/env python
"""STRICT across parameter space: random workloads (uniform cube / Plummer
sphere, 20k-300k particles, Coulomb / Yukawa with kappa in [0.05, 20],
degree 1-12, theta 0.35-0.95, several leaf / batch sizes), each evaluated in
PARITY (= the reference, bitwise) and in STRICT.  Per workload: the
certificate's measured error constant max |phi_fast - phi_ref| / (eps S_i)
(STRICT with Kc = 0: nothing recomputed), the recomputed count with the
shipped Kc, and STRICT's max per-target relative deviation from PARITY over
ALL targets (must be <= 1e-10).

    python tools/strict_fuzz.py --runs 120 > profiles/r2_strict_fuzz.jsonl
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EPS = 2.0 ** -53


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=100)
    ap.add_argument("--seed", type=int, default=2026)
    ap.add_argument("--max-n", type=int, default=300_000)
    ap.add_argument("--large", action="store_true",
                    help="instead: the fuzz's worst corner (degree 1-2, many terms per "
                         "target) at 8M and 32M particles")
    args = ap.parse_args()
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200 import cli
    rng = np.random.default_rng(args.seed)
    ctx = bltc.Context(0)
    ctx.keep_strict_bounds(True)
    worst_ratio, worst_rel, bad = 0.0, 0.0, 0
    large = [(n, deg, kap, th, lf, bt) for n in (8_000_000, 32_000_000)
             for deg, kap, th, lf, bt in ((1, 0.0, 0.7, 500, 500), (2, 18.6, 0.42, 200, 64),
                                          (1, 0.0, 0.42, 200, 64), (2, 0.0, 0.59, 2000, 160))]
    if args.large:
        args.runs = len(large)
    for run in range(args.runs):
        if args.large:
            n, deg, kappa, theta, leaf, batch = large[run]
            gen, yuk = "uniform", kappa > 0
            system = cli.generate_particles(n, run + 1)
        else:
            n = int(rng.integers(20_000, args.max_n))
            gen = "plummer" if rng.random() < 0.4 else "uniform"
            system = (cli.generate_plummer if gen == "plummer" else cli.generate_particles)(
                n, int(rng.integers(1, 10_000)))
            yuk = rng.random() < 0.35
            kappa = float(np.exp(rng.uniform(np.log(0.05), np.log(20.0)))) if yuk else 0.0
            deg = int(rng.integers(1, 13))
            theta = float(rng.uniform(0.35, 0.95))
            leaf = int(rng.choice([200, 500, 1000, 2000]))
            batch = int(rng.choice([64, 160, 300, 500, leaf]))
        cfg = bltc.EvalConfig(theta=theta, degree=deg, leaf_size=leaf, batch_size=batch,
                              kernel=bltc.yukawa(kappa) if yuk else bltc.coulomb())
        ref, _ = ctx.treecode(system, cfg, mode="parity")
        os.environ["BLTC_STRICT_KC"] = "0"
        phi0, _ = ctx.treecode(system, cfg, mode="strict")
        S, _ = ctx.export_strict_bounds()
        del os.environ["BLTC_STRICT_KC"]
        phi, st = ctx.treecode(system, cfg, mode="strict")
        nz = ref != 0
        ratio = float((np.abs(phi0 - ref) / (EPS * S)).max())
        rel = float((np.abs(phi[nz] - ref[nz]) / np.abs(ref[nz])).max())
        above = int((np.abs(phi - ref) > 1e-10 * np.abs(ref)).sum())
        worst_ratio, worst_rel, bad = max(worst_ratio, ratio), max(worst_rel, rel), bad + above
        print(json.dumps({"run": run, "gen": gen, "n": n, "kernel": "yukawa" if yuk else "coulomb",
                          "kappa": kappa, "degree": deg, "theta": theta, "leaf": leaf,
                          "batch": batch, "ratio_max": ratio, "recomputed": int(st.n_recomputed),
                          "strict_max_rel": rel, "targets_above_1e-10": above}), flush=True)
    print(json.dumps({"summary": True, "runs": args.runs, "worst_ratio": worst_ratio,
                      "worst_strict_rel": worst_rel, "targets_above_1e-10": bad}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
