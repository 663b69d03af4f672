#!/usr/bin/env python
"""Accuracy cost of the batch size N_B (the performance knob): time, pair
counts and relative L2 error against a direct sum on the reference harness's
4000-target verification sample (cli.py:287-290), per N_B, STRICT mode, one
B200.  The reference default is N_L = N_B = 2000 (engine.py:52-53).

    python tools/nb_table.py --config c4 --batch-sizes 160,250,500,1000,2000
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
    ap.add_argument("--config", default="c4")
    ap.add_argument("--batch-sizes", default="160,250,500,1000,2000")
    ap.add_argument("--mode", default="strict")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200 import cli, engine
    cfg = bench.CONFIGS[args.config]
    system = bench.make_system(cfg, device=0)
    n = cfg["n"]
    sample = cli.sample_indices(n, 4000, seed=1)
    ctx = bltc.Context(0, torch.cuda.current_stream().cuda_stream)
    econf0 = bench.eval_config(cfg, None, None)
    ds = ctx.direct_sum(system, econf0.kernel, sample, mode="parity")
    s = system.sources
    dev = [torch.from_numpy(a).cuda() for a in (s.x, s.y, s.z, system.charges)]
    phi = torch.empty(n, dtype=torch.float64, device="cuda")
    ptrs = [t.data_ptr() for t in dev]
    for nb in [int(v) for v in args.batch_sizes.split(",")]:
        econf = bench.eval_config(cfg, nb, None)
        params = engine.make_params(econf, args.mode)

        def step():
            return ctx.treecode_device(params, n, ptrs[0], ptrs[1], ptrs[2], n, ptrs[0],
                                       ptrs[1], ptrs[2], ptrs[3], True, phi.data_ptr())
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            st = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        err = cli.relative_error(ds, phi.cpu().numpy()[sample])
        print(json.dumps({"config": args.config, "mode": args.mode, "leaf_size": econf.leaf_size,
                          "batch_size": nb, "ms": ms, "error": err,
                          "direct_pairs": st.direct_pairs, "approx_pairs": st.approx_pairs,
                          "batches": st.n_batches, "recomputed": st.n_recomputed,
                          "far_s": st.far_s, "near_s": st.near_s}), flush=True)


if __name__ == "__main__":
    main()
