"""Sweep leaf/batch sizes (and FAST tuning env) on one generated workload.

    python tools/sweep_c4.py --config c4 --leaf 1000,2000 --batch 250,500,1000
Prints one JSON line per setting: step ms (CUDA events around the device
pipeline), far/near ms and pair counts."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2003_01836_b200 as bltc  # noqa: E402
from paper_2003_01836_b200 import engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--leaf", default="2000")
ap.add_argument("--batch", default="500")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--mode", default="fast", choices=["fast", "parity"])
ap.add_argument("--env", default="", help="semicolon-separated KEY=VAL sets to try, '|'-joined")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
system = bench.make_system(cfg)
n = cfg["n"]
s = system.sources
dev = [torch.from_numpy(a).cuda() for a in (s.x, s.y, s.z, system.charges)]
phi = torch.empty(n, dtype=torch.float64, device="cuda")
p = [t.data_ptr() for t in dev]
stream = torch.cuda.current_stream()
ctx = bltc.Context(0, stream.cuda_stream)
envsets = [e for e in args.env.split("|")] if args.env else [""]
for env in envsets:
    for kv in filter(None, env.split(";")):
        k, v = kv.split("=", 1)
        os.environ[k] = v
    for leaf in map(int, args.leaf.split(",")):
        for batch in map(int, args.batch.split(",")):
            econf = bench.eval_config(cfg, batch, leaf)
            params = engine.make_params(econf, args.mode)
            def step():
                return ctx.treecode_device(params, n, p[0], p[1], p[2], n, p[0], p[1], p[2],
                                           p[3], True, phi.data_ptr())
            step()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sts = [step() for _ in range(args.steps)]
            e1.record(stream)
            torch.cuda.synchronize()
            st = sts[-1]
            print(json.dumps({"env": env, "leaf": leaf, "batch": batch,
                              "ms": e0.elapsed_time(e1) / args.steps,
                              "far_ms": 1e3 * st.far_s, "near_ms": 1e3 * st.near_s,
                              "setup_ms": 1e3 * st.setup_s, "pre_ms": 1e3 * st.precompute_s,
                              "approx": st.approx_pairs, "direct": st.direct_pairs,
                              "clusters": st.n_clusters, "batches": st.n_batches,
                              "packed": st.packed}), flush=True)
    for kv in filter(None, env.split(";")):
        os.environ.pop(kv.split("=")[0], None)
