#!/usr/bin/env python
"""Time the UNMODIFIED reference package (Python + numba, installed by
tools/ref_suite/prepare.sh into baseline/_ref) on the host cores: its own
treecode_potentials (engine.py:350-372) with threads = all cores, on a bench
workload -- the anchor for the C port that bench.py's cpu_baseline and
--impl reference run (profiles/r2_reference_numba_*.json).

    PYTHONPATH=baseline/_ref python tools/reference_numba_step.py --config c2
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import numpy as np
    from bltc.engine import EvalConfig, treecode_potentials
    from bltc.kernels import coulomb, yukawa
    from bltc.particles import ParticleSystem, Points
    cfg = bench.CONFIGS[args.config]
    mine = bench.make_system(cfg)
    s = mine.sources
    system = ParticleSystem.from_single_set(Points(np.asarray(s.x), np.asarray(s.y),
                                                   np.asarray(s.z)), np.asarray(mine.charges))
    kernel = yukawa(cfg["kappa"]) if cfg["kind"] == 1 else coulomb()
    econf = EvalConfig(theta=cfg["theta"], degree=cfg["degree"], leaf_size=cfg["leaf"],
                       batch_size=cfg["batch"], kernel=kernel)
    threads = os.cpu_count() or 1
    # numba compiles on first use: warm on a small system, untimed
    small = ParticleSystem.from_single_set(Points(np.asarray(s.x[:5000]), np.asarray(s.y[:5000]),
                                                  np.asarray(s.z[:5000])),
                                           np.asarray(mine.charges[:5000]))
    treecode_potentials(small, econf, threads=threads)
    times = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        phi, st = treecode_potentials(system, econf, threads=threads)
        times.append(time.perf_counter() - t0)
    out = {"config": args.config, "workload": cfg["workload"], "impl": "reference (numba)",
           "threads": threads, "cpu_model": bench.cpu_model(),
           "step_s": min(times), "particles_per_s": cfg["n"] / min(times),
           "phases_s": {"setup": st.setup_s, "precompute": st.precompute_s,
                        "compute": st.compute_s},
           "pairs": {"direct": st.direct_pairs, "approx": st.approx_pairs}}
    # the same workload through this package (PARITY): bitwise the reference
    try:
        import paper_2003_01836_b200 as ours
        oconf = ours.EvalConfig(theta=cfg["theta"], degree=cfg["degree"], leaf_size=cfg["leaf"],
                                batch_size=cfg["batch"],
                                kernel=ours.yukawa(cfg["kappa"]) if cfg["kind"] == 1
                                else ours.coulomb())
        phi_p, _ = ours.treecode_potentials(mine, oconf, mode="parity")
        out["gpu_parity_bitwise_equal"] = bool(np.array_equal(phi_p, phi))
        phi_s, _ = ours.treecode_potentials(mine, oconf, mode="strict")
        d = np.abs(phi_s - phi)
        nz = phi != 0
        out["gpu_strict_max_rel"] = float((d[nz] / np.abs(phi[nz])).max())
        out["gpu_strict_targets_above_1e-10"] = int((d[nz] > 1e-10 * np.abs(phi[nz])).sum())
    except Exception as exc:   # reported, not required
        out["gpu_parity_bitwise_equal"] = repr(exc)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
