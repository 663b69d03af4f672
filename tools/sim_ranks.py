"""Projected multi-GPU step from simulated ranks on ONE GPU.

Runs the distributed pipeline of decomp.run_distributed rank by rank on one
device (one libbltc context per rank), timing each rank's phases with CUDA
events: build (tree, batches, moments), publish, LET step one (needs),
serve + assemble of the fetched rows / slices, evaluate.  With
``--exchange replicate`` (bench.py's N > 1 default: one packed all-gather of
every rank's forest) the LET steps are skipped and every rank evaluates
against the whole forest.  The projected R-GPU step is the max over ranks
of the rank's device time plus the exchange volume over NVLink at an
assumed 400 GB/s per GPU with 4 (LET) / 2 (replicate) collectives of 30 us
latency.  This is a projection, not a measurement.

    python tools/sim_ranks.py --config c4 --ranks 2,4,8 [--mode strict] [--exchange replicate]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2003_01836_b200 import engine  # noqa: E402
from paper_2003_01836_b200.decomp import (DeviceRankEngine, domain_boxes, let_assemble,  # noqa: E402
                                          let_plan, let_serve, rcb_partition)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--ranks", default="2,4,8")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", default="strict", choices=["strict", "fast", "parity"])
ap.add_argument("--exchange", default="replicate", choices=["let", "replicate"])
args = ap.parse_args()
cfg = bench.CONFIGS[args.config]
system = bench.make_system(cfg)
econf = bench.eval_config(cfg, None, None)
src = system.sources


def timed(fn):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1), 1e3 * (time.perf_counter() - t0)


for R in map(int, args.ranks.split(",")):
    part = rcb_partition(src, R)
    ctxs = [engine.Context(0) for _ in range(R)]
    engs = [DeviceRankEngine(econf, args.mode, context=ctxs[r]) for r in range(R)]
    boxes = domain_boxes(src.x, src.y, src.z)
    for e in engs:
        e.set_domain_boxes(boxes)
    inputs = []
    for r in range(R):
        idx = part.rank_indices(r)
        inputs.append([torch.from_numpy(np.ascontiguousarray(np.asarray(a)[idx])).cuda()
                       for a in (src.x, src.y, src.z, system.charges)])
    best = None
    mins = {}
    for rep in range(args.reps):
        ph = {r: {} for r in range(R)}
        pubs = {}
        for r in range(R):
            _, ph[r]["build_ms"], _ = timed(lambda: engs[r].build(*inputs[r]))
            pubs[r], ph[r]["publish_ms"], _ = timed(lambda: engs[r].publish())
        recs = [pubs[r].records for r in range(R)]
        ncols = int(pubs[0].moments.shape[1])
        fetched_bytes = {r: 0 for r in range(R)}
        forests = {}
        if args.exchange == "replicate":
            block = {o: sum(int(t.numel()) * 8 for t in (pubs[o].records, pubs[o].particles,
                                                        pubs[o].moments)) for o in range(R)}
            for r in range(R):
                ph[r]["needs_ms"] = ph[r]["let_host_ms"] = 0.0
                forests[r] = [pubs[o] for o in range(R)]
                fetched_bytes[r] = sum(block[o] for o in range(R) if o != r)
        for r in range(R) if args.exchange == "let" else ():
            flags, ph[r]["needs_ms"], _ = timed(lambda: engs[r].needs(R, r, recs))
            t0 = time.perf_counter()
            forest = []
            plan = let_plan(flags, recs, r)
            for o in range(R):
                if o == r:
                    forest.append(pubs[r])
                    continue
                payload = let_serve(pubs[o], plan.a[o], plan.d[o], plan.npart[o])
                fetched_bytes[r] += payload.numel() * 8
                p_o, _ = let_assemble(recs[o], plan.a[o], plan.d[o], payload, ncols,
                                      plan.npart[o], plan.nboth[o])
                forest.append(p_o)
            torch.cuda.synchronize()
            ph[r]["let_host_ms"] = 1e3 * (time.perf_counter() - t0)
            forests[r] = forest
        for r in range(R):
            _, ph[r]["evaluate_ms"], _ = timed(lambda: engs[r].evaluate(R, r, forests[r]))
            st = engs[r].stats
            ph[r]["far_ms"], ph[r]["near_ms"] = 1e3 * st.far_s, 1e3 * st.near_s
            ph[r]["pairs"] = int(st.direct_pairs + st.approx_pairs)
        # per rank and phase, the minimum over repetitions (first-touch
        # allocations of the simulated ranks' buffers are not steady state)
        for r in range(R):
            dm = mins.setdefault(r, {})
            for k, v in ph[r].items():
                dm[k] = min(dm.get(k, v), v) if k != "pairs" else v
        ph = {r: dict(mins[r]) for r in range(R)}
        dev = {r: sum(ph[r][k] for k in ("build_ms", "publish_ms", "needs_ms", "let_host_ms",
                                           "evaluate_ms")) for r in range(R)}
        rec_bytes = sum(int(x.numel()) * 8 for x in recs)
        if args.exchange == "replicate":
            xfer_ms = max(fetched_bytes[r] / 400e9 * 1e3 for r in range(R)) + 2 * 0.03
        else:
            xfer_ms = max((fetched_bytes[r] + rec_bytes) / 400e9 * 1e3 for r in range(R)) + 4 * 0.03
        proj = max(dev.values()) + xfer_ms
        if best is None or proj < best["projected_step_ms"]:
            best = {"ranks": R, "projected_step_ms": proj, "max_rank_device_ms": max(dev.values()),
                    "mean_rank_device_ms": float(np.mean(list(dev.values()))),
                    "exchange_ms_assumed": xfer_ms,
                    "fetched_MB_max": max(fetched_bytes.values()) / 1e6,
                    "records_MB": rec_bytes / 1e6, "per_rank": ph}
    print(json.dumps({"config": args.config, "n": cfg["n"], "batch_size": econf.batch_size,
                      "mode": args.mode, "exchange": args.exchange,
                      **best}), flush=True)
    for c in ctxs:
        c.close()
