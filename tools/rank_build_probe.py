"""Rank build time (local tree, batches, moment rows) of rank 0 at the C4
workload for R = 1, 2, 4, 8 RCB ranks, with the domain as occupied-cell boxes
(decomp.domain_boxes) vs one bounding box: how many moment rows each rank
computes and what the bitwise upward pass costs there.

    python tools/rank_build_probe.py
"""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2003_01836_b200 import engine
from paper_2003_01836_b200.decomp import DeviceRankEngine, rcb_partition, domain_boxes
cfg = bench.CONFIGS["c4"]; system = bench.make_system(cfg); econf = bench.eval_config(cfg, None, None)
src = system.sources
lo = [float(np.min(a)) for a in (src.x, src.y, src.z)]; hi = [float(np.max(a)) for a in (src.x, src.y, src.z)]
for R in (1, 2, 4, 8):
    part = rcb_partition(src, R)
    for mode in ("strict",):
        for dom in ("cells", "box"):
            r = 0
            idx = part.rank_indices(r)
            inp = [torch.from_numpy(np.ascontiguousarray(np.asarray(a)[idx])).cuda() for a in (src.x, src.y, src.z, system.charges)]
            e = DeviceRankEngine(econf, mode, context=engine.Context(0))
            e.set_domain_boxes(domain_boxes(src.x, src.y, src.z)) if dom == 'cells' else e.set_domain(lo, hi)
            best = 1e9
            for rep in range(3):
                torch.cuda.synchronize(); t = time.perf_counter(); e.build(*inp); torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t)
            sz = e.ctx.rank_publish_sizes()
            print(json.dumps({"R": R, "mode": mode, "domain": dom, "build_ms": best * 1e3, "rows": sz["n_moment_rows"], "clusters": sz["n_clusters"]}), flush=True)
