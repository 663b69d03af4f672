"""Run a few BLTC steps of a bench config (for ncu launch lists / profiles)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2003_01836_b200 as bltc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--batch-size", type=int, default=None)
ap.add_argument("--mode", default="fast")
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
system = bench.make_system(cfg)
econf = bench.eval_config(cfg, args.batch_size, None)
ctx = bltc.Context(0)
for i in range(args.steps):
    phi, st = ctx.treecode(system, econf, mode=args.mode)
    print(i, st, file=sys.stderr)
