#!/usr/bin/env python
"""Calibrate and check STRICT mode (csrc/strict.cu) on bench workloads.

For each config: PARITY (= the reference, bitwise) is the yardstick.
1. STRICT with Kc = 0 (nothing recomputed: the FAST kernels on the
   reference's moments) and the per-target certificate mass S_i kept:
   ratio_i = |phi_i - phi_ref,i| / (eps S_i) -- its maximum over all targets
   is the measured error constant the default Kc must exceed;
   also the share of targets Kc eps S_i > tau |phi_i| would flag for several Kc.
2. STRICT with the default Kc: recomputed count, strict per-target max
   relative difference vs PARITY over ALL targets (must be <= 1e-10), the
   share above 1e-10 (must be 0), bitwise share, and the times of FAST /
   STRICT / PARITY steps.

    python tools/strict_calibrate.py --configs c2,c3,c4 > gpurun_out/strict.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

EPS = 2.0 ** -53
TAU = 0.5e-10


def timed(fn, reps=2):
    import torch
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2")
    ap.add_argument("--batch-size", type=int, default=None)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import paper_2003_01836_b200 as bltc
    for name in args.configs.split(","):
        cfg = bench.CONFIGS[name]
        econf = bench.eval_config(cfg, args.batch_size, None)
        system = bench.make_system(cfg, device=0)
        ctx = bltc.Context(0)
        ctx.keep_strict_bounds(True)
        (phi_p, st_p), t_p = timed(lambda: ctx.treecode(system, econf, mode="parity"), 1)
        os.environ["BLTC_STRICT_KC"] = "0"
        phi_0, st_0 = ctx.treecode(system, econf, mode="strict")
        S, _ = ctx.export_strict_bounds()
        del os.environ["BLTC_STRICT_KC"]
        d0 = np.abs(phi_0 - phi_p)
        ratio = d0 / (EPS * S)
        a = np.abs(phi_0)
        rec = {"config": name, "n": int(cfg["n"]), "batch_size": econf.batch_size,
               "ratio_max": float(ratio.max()),
               "ratio_q": {q: float(np.quantile(ratio, q)) for q in (0.5, 0.99, 0.9999)},
               "kc0_strict_max_rel": float((d0 / np.abs(phi_p)).max()),
               "kc0_frac_above_1e-10": float((d0 > 1e-10 * np.abs(phi_p)).mean()),
               "flag_frac": {str(kc): float((kc * EPS * S > TAU * a).mean())
                             for kc in (0.25, 0.5, 1, 2, 4, 8, 16, 64)},
               "cond_median": float(np.median(S / np.maximum(a, 1e-300)))}
        (phi_s, st_s), t_s = timed(lambda: ctx.treecode(system, econf, mode="strict"), args.reps)
        _, kc = ctx.export_strict_bounds()
        _, t_f = timed(lambda: ctx.treecode(system, econf, mode="fast"), args.reps)
        ds = np.abs(phi_s - phi_p)
        nz = phi_p != 0
        rec.update({
            "kc": kc,
            "n_recomputed": int(st_s.n_recomputed),
            "strict_max_rel": float((ds[nz] / np.abs(phi_p[nz])).max()),
            "strict_frac_above_1e-10": float((ds[nz] > 1e-10 * np.abs(phi_p[nz])).mean()),
            "strict_bitwise_frac": float((phi_s == phi_p).mean()),
            "strict_condition_aware": float(ds.max() / np.abs(phi_p).max()),
            "time_s": {"fast": t_f, "strict": t_s, "parity": t_p},
            "device_s": {"strict_precompute": st_s.precompute_s,
                         "strict_fixup": st_s.strict_s, "strict_far": st_s.far_s,
                         "strict_near": st_s.near_s, "parity_precompute": st_p.precompute_s},
        })
        print(json.dumps(rec), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
