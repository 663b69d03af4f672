"""Bitwise upward pass on ONE big cluster (a single leaf of n uniform
sources, degree 8, STRICT): the split items' per-source cost in isolation
(M = 9 CTAs, one per k1, each streaming all n sources).

    python tools/moments_big_probe.py [n1,n2,...]
"""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2003_01836_b200 import engine, cli
from paper_2003_01836_b200.engine import EvalConfig
from paper_2003_01836_b200.decomp import DeviceRankEngine
ns = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [131073, 1 << 20, 1 << 21]
for n in ns:
    s = cli.generate_particles(n, 1)
    econf = EvalConfig(theta=0.8, degree=8, leaf_size=n, batch_size=n)
    e = DeviceRankEngine(econf, "strict", context=engine.Context(0))
    inp = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (s.sources.x, s.sources.y, s.sources.z, s.charges)]
    e.build(*inp); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); t = time.perf_counter(); e.build(*inp); torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    sz = e.ctx.rank_publish_sizes()
    print(json.dumps({"n": n, "build_ms": best * 1e3, "rows": sz["n_moment_rows"], "cycles_per_source_at_1.9GHz": best * 1.9e9 / n}), flush=True)
