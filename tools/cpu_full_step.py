#!/usr/bin/env python
"""Unsampled CPU step of the reference algorithm (oracle/ C port, all host
threads) next to bench.py's sampled + extrapolated estimate, on the same
workload: the anchor for the reference arm's extrapolation.

    python tools/cpu_full_step.py --config c4 > profiles/r2_cpu_full_step_c4.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--ref-budget", type=float, default=1.5e10)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    econf = bench.eval_config(cfg, None, None)
    system = bench.make_system(cfg)
    ref = bench.CpuReference(system, econf, budget_pairs=args.ref_budget)
    sampled = ref.step()
    sel_sampled = ref.sel
    ref.sel = np.arange(ref.batches.nb)
    ref.frac = 1.0
    t0 = time.perf_counter()
    full = ref.step()
    wall = time.perf_counter() - t0
    out = {"config": args.config, "workload": cfg["workload"], "batch_size": econf.batch_size,
           "threads": ref.threads, "cpu_model": bench.cpu_model(),
           "setup_s": ref.setup_s, "moments_s": ref.moments_s,
           "full_eval_s": wall, "full_step_s": full["est_step_s"],
           "sampled_batches": int(len(sel_sampled)), "sampled_estimate_step_s":
           sampled["est_step_s"],
           "extrapolation_error": sampled["est_step_s"] / full["est_step_s"] - 1.0,
           "full_particles_per_s": full["value"]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
