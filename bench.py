#!/usr/bin/env python
"""BLTC evaluation benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
                    [--impl ours|reference] [--mode strict|fast|parity]

One step = one full BLTC evaluation of the workload (source tree, target
batches, interaction lists, moments, far + near field, un-permute) through
libbltc's CUDA kernels, inputs resident in HBM, in the shipped default mode
STRICT (every target within 1e-10 of the reference: FAST kernels on the
reference's moments, near-cancelling targets recomputed in the reference's
arithmetic).  ``value`` is particles/s over all ranks; ``e2e`` is the same
metric through the public API with host buffers, H2D/D2H inside the timed
region.  ``roofline`` is the dominant kernel's (far field) FP64 throughput
against the nominal FP64 peak at the SM clock sampled during the timed
region (148 SMs x 64 FP64 lanes x 2 flop x f_SM).  ``cpu_baseline`` is the
CPU restatement of the reference algorithm (oracle/, "port") on the host
cores on a bounded sample, extrapolated by pair count.

N > 1 (torchrun, one rank per GPU): targets are partitioned by recursive
coordinate bisection (decomp.py:76-130), each rank builds its tree and
moments, one all-gather over NCCL replicates the forest, each rank
evaluates its batches; timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BLTC eval time & particles/s (N=8M Coulomb n=8 θ=0.8), %FP64 peak, 1/2/4/8 GPU"

CONFIGS = {
    # BASELINE.json configs; c4 is the metric's workload (8M Coulomb n=8 theta=0.8)
    "c1": dict(workload="C1: N=20k uniform cube, Coulomb, n=4, theta=0.7", gen="uniform",
               n=20_000, kind=0, kappa=0.0, degree=4, theta=0.7, leaf=2000, batch=2000),
    # C2/C3: N_B=160 (= any of 64..200 for this uniform cube: octree level-5
    # batches of ~30 targets) measured fastest on B200 with packed, longest-
    # first items: C2 42 ms vs 50 ms at N_B=1000 and 47 ms at 250, C3 101 ms
    # vs 121 / 115 ms (tools/sweep_c4.py)
    "c2": dict(workload="C2: N=1M uniform cube, Coulomb, n=8, theta=0.8", gen="uniform",
               n=1_000_000, kind=0, kappa=0.0, degree=8, theta=0.8, leaf=2000, batch=160),
    "c3": dict(workload="C3: N=1M uniform cube, Yukawa kappa=0.5, n=8, theta=0.8",
               gen="uniform", n=1_000_000, kind=1, kappa=0.5, degree=8, theta=0.8, leaf=2000,
               batch=160),
    # N_B (batch size) is the performance knob; the CPU
    # baseline / reference arm run with the same value.  160 is the fastest
    # measured for C4 on B200 with packed work items (N_B=125: 0.929 s,
    # 160: 0.908 s, 250: 0.927 s, 400: 0.960 s; N_L 1000-3000 within 0.5%;
    # tools/sweep_c4.py, gpurun_out/sweep27/28).
    "c4": dict(workload="C4: N=8M Plummer (a=1, r<=10a), Coulomb, n=8, theta=0.8",
               gen="plummer", n=8_000_000, kind=0, kappa=0.0, degree=8, theta=0.8, leaf=2000,
               batch=160),
    "c4u": dict(workload="N=8M uniform cube, Coulomb, n=8, theta=0.8", gen="uniform",
                n=8_000_000, kind=0, kappa=0.0, degree=8, theta=0.8, leaf=2000, batch=2000),
    # accuracy context for the north star's "~1e-7 relative error" at 8M: the
    # same cube / Plummer sphere at C5's n = 10, theta = 0.7
    "c4u_n10": dict(workload="N=8M uniform cube, Coulomb, n=10, theta=0.7", gen="uniform",
                    n=8_000_000, kind=0, kappa=0.0, degree=10, theta=0.7, leaf=2000,
                    batch=160),
    "c4_n10": dict(workload="N=8M Plummer (a=1, r<=10a), Coulomb, n=10, theta=0.7",
                   gen="plummer", n=8_000_000, kind=0, kappa=0.0, degree=10, theta=0.7,
                   leaf=2000, batch=160),
    # C5: N_B=160 (level-7 batches): 10.1 s vs 11.2 s at 250 and 11.7 s at 1000
    "c5": dict(workload="C5: N=64M uniform cube, Coulomb, n=10, theta=0.7", gen="uniform",
               n=64_000_000, kind=0, kappa=0.0, degree=10, theta=0.7, leaf=2000, batch=160),
    # the paper's strong-scaling case (16.2 s on 32 P100)
    "paper64m": dict(workload="64M uniform cube, Coulomb, n=8, theta=0.8, N_L=N_B=4000 "
                              "(paper strong-scaling case)", gen="uniform", n=64_000_000,
                     kind=0, kappa=0.0, degree=8, theta=0.8, leaf=4000, batch=4000),
    "paper64m_y": dict(workload="64M uniform cube, Yukawa kappa=0.5, n=8, theta=0.8, "
                                "N_L=N_B=4000 (paper strong-scaling case)", gen="uniform",
                       n=64_000_000, kind=1, kappa=0.5, degree=8, theta=0.8, leaf=4000,
                       batch=4000),
}

# Minimal FP64-pipe slots per pair: far / near field.
# Yukawa: SURVEY.md counts libdevice exp as 15 slots (25 / 30); the kernels
# fold kappa into a table-driven exp of 8 slots (eval_common.cuh exp_neg_kr),
# so the algorithmic count here is the lower 17 / 22 (the roofline is not
# inflated).
SLOTS = {0: (7, 12), 1: (16, 21), 2: (1, 1)}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "power.draw")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self) -> dict:
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7],
                             float(parts[7]) if parts[7] not in ("", "[N/A]") else 0.0))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k, v in enumerate(r[2]) if v == "Active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "power_w_max": max(r[3] for r in rows), "samples": len(rows)}


# ---------------------------------------------------------------------------


def make_system(cfg: dict, seed: int = 1, device: int | None = None):
    """The workload's particles.  Uniform cubes are generated on the GPU when
    ``device`` is given (bltc_philox_uniform: numpy's Philox stream bit for
    bit, tests/test_gpu_generate.py), then copied to the host; Plummer and the
    CPU reference arm use numpy."""
    from paper_2003_01836_b200 import cli
    if cfg["gen"] == "uniform" and device is not None:
        from paper_2003_01836_b200.particles import ParticleSystem, Points
        x, y, z, q = (t.cpu().numpy() for t in cli.generate_particles_device(cfg["n"], seed,
                                                                            device))
        return ParticleSystem.from_single_set(Points(x, y, z), q)
    gen = cli.generate_particles if cfg["gen"] == "uniform" else cli.generate_plummer
    return gen(cfg["n"], seed)


def eval_config(cfg: dict, batch: int | None, leaf: int | None):
    from paper_2003_01836_b200 import EvalConfig, coulomb, test_constant, yukawa
    kernel = [coulomb(), yukawa(cfg["kappa"]), test_constant()][cfg["kind"]]
    return EvalConfig(theta=cfg["theta"], degree=cfg["degree"],
                      leaf_size=leaf or cfg["leaf"], batch_size=batch or cfg["batch"],
                      kernel=kernel)


def launch_count() -> int:
    """libbltc's process-wide kernel launch counter (bltc_launch_count)."""
    import ctypes
    from paper_2003_01836_b200 import _lib
    v = ctypes.c_int64()
    _lib.check(_lib.load().bltc_launch_count(ctypes.byref(v)))
    return int(v.value)


def probe_fp64(device: int) -> float:
    import ctypes
    from paper_2003_01836_b200 import _lib
    lib = _lib.load()
    v = ctypes.c_double()
    _lib.check(lib.bltc_probe_fp64(device, 0.3, ctypes.byref(v)))
    return v.value


class CpuReference:
    """The reference's CPU algorithm (oracle/: C restatement of the reference
    path, "port") on this host's cores, on a bounded sample of the workload:
    full tree / batches / lists / moments (timed once), then evaluation of a
    random sample of target batches (timed per step), extrapolated to the
    whole workload by pair count."""

    def __init__(self, system, econf, budget_pairs: float = 1.5e10, threads: int | None = None):
        from oracle import oracle as orc
        self.orc = orc
        self.threads = threads or os.cpu_count() or 1
        self.system, self.econf = system, econf
        s = system.sources
        t0 = time.perf_counter()
        tree = orc.build_source_tree(s.x, s.y, s.z, system.charges, econf.leaf_size)
        if econf.batch_size == econf.leaf_size:
            lf = tree.leaf_dfs
            batches = orc.Batches(tree=tree, start=tree.start[lf], stop=tree.stop[lf],
                                  center=tree.center[lf], radius=tree.radius[lf])
        else:
            batches = orc.build_target_batches(s.x, s.y, s.z, econf.batch_size)
        lists = orc.build_lists(batches, tree, econf.theta, econf.degree)
        t1 = time.perf_counter()
        rows, mrow = orc.compute_moments(tree, econf.degree, np.unique(lists.a_idx),
                                         self.threads)
        t2 = time.perf_counter()
        self.setup_s, self.moments_s = t1 - t0, t2 - t1
        self.tree, self.batches, self.lists, self.rows, self.mrow = tree, batches, lists, rows, mrow
        nt = batches.stop - batches.start
        m3 = (econf.degree + 1) ** 3
        csum = np.concatenate([[0], np.cumsum(tree.count[lists.d_idx])])
        cost = nt * (csum[lists.d_ptr[1:]] - csum[lists.d_ptr[:-1]]) + nt * m3 * np.diff(lists.a_ptr)
        order = np.random.default_rng(0).permutation(batches.nb)
        take = int(np.searchsorted(np.cumsum(cost[order]), budget_pairs)) + 1
        self.sel = np.sort(order[:min(take, batches.nb)])
        self.frac = float(cost[self.sel].sum() / cost.sum())

    def step(self) -> dict:
        t0 = time.perf_counter()
        self.last = self.orc.evaluate(self.batches,
                                      [self.orc.SourceGroup(self.tree, self.rows, self.mrow,
                                                            self.lists)],
                                      self.econf.degree, self.econf.kernel.code,
                                      self.econf.kernel.kappa, self.threads, sel=self.sel)
        t = time.perf_counter() - t0
        est = self.setup_s + self.moments_s + t / self.frac
        return {"value": self.system.n_targets / est, "unit": "particles/s",
                "cores": self.threads, "kind": "port", "extrapolated": True,
                "cpu_model": cpu_model(), "sampled_pair_fraction": self.frac,
                "sample": (f"oracle/ C port of the reference path on {self.threads} host threads: "
                           f"tree+batches+lists {self.setup_s:.1f}s (serial, as in the "
                           f"reference) and moments {self.moments_s:.1f}s measured in full; "
                           f"evaluation of {len(self.sel)}/{self.batches.nb} random target "
                           f"batches = {self.frac:.4f} of the pairs took {t:.1f}s; "
                           f"extrapolated full step {est:.1f}s"),
                "est_step_s": est}


    def sampled_parity(self, phi_parity, phi_mode) -> dict:
        """Full-size parity on the sampled batches: the CPU restatement's
        potentials of every target in the evaluated sample against the GPU's
        PARITY (bitwise expected) and measured-mode (STRICT / FAST) results."""
        b = self.batches
        pos = np.concatenate([np.arange(b.start[i], b.stop[i]) for i in self.sel])
        out, carry = self.last
        ref = (out + carry)[pos]
        orig = b.tree.order[pos]
        dp = np.abs(phi_parity[orig] - ref)
        df = np.abs(phi_mode[orig] - ref)
        nz = ref != 0
        return {"targets": int(pos.shape[0]), "batches": int(len(self.sel)),
                "parity_bitwise_equal": bool(np.array_equal(phi_parity[orig], ref)),
                "parity_max_abs_diff": float(dp.max()),
                "mode_condition_aware": float(df.max() / np.abs(ref).max()),
                "mode_strict_max_rel": float((df[nz] / np.abs(ref[nz])).max()),
                "mode_frac_targets_above_1e-10": float((df[nz] / np.abs(ref[nz]) > 1e-10).mean())}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(system, cfg, econf, budget_pairs: float = 1.5e10):
    return CpuReference(system, econf, budget_pairs).step()


# ---------------------------------------------------------------------------


def accuracy_block(ctx, system, econf, mode, phi, args, cpu_ref=None) -> dict:
    """Accuracy of the timed result at the full workload size.

    * relative L2 error against a direct sum on the reference harness's
      verification sample (cli.py:287-290: child-2 stream, M targets), for
      the measured mode and for PARITY mode (which is the reference's own
      result bit for bit -- tests/test_gpu_parity.py), so the two errors can
      be compared (BASELINE.json: within 1%);
    * per-target deviation of the measured mode from PARITY over ALL targets:
      strict max |d_i| / |phi_i| and condition-aware max |d_i| / max |phi|;
    * the GPU direct sum is cross-checked bitwise against the CPU oracle on a
      few of the sample targets."""
    from oracle import oracle as orc
    from paper_2003_01836_b200 import cli
    n = system.n_targets
    sample = cli.sample_indices(n, args.accuracy_sample, seed=1)
    t0 = time.perf_counter()
    ds = ctx.direct_sum(system, econf.kernel, sample, mode="parity")
    t_ds = time.perf_counter() - t0
    s = system.sources
    k = min(32, sample.shape[0])
    cpu = orc.direct_sum(s.x, s.y, s.z, s.x, s.y, s.z, system.charges, econf.kernel.code,
                         econf.kernel.kappa, sample[:k], threads=os.cpu_count() or 1)
    phi_p, _ = ctx.treecode(system, econf, mode="parity")
    err = cli.relative_error(ds, phi[sample])
    err_p = cli.relative_error(ds, phi_p[sample])
    d = np.abs(phi - phi_p)
    nz = phi_p != 0
    strict = float((d[nz] / np.abs(phi_p[nz])).max()) if nz.any() else 0.0
    sampled = None
    if cpu_ref is not None and getattr(cpu_ref, "last", None) is not None:
        sampled = cpu_ref.sampled_parity(phi_p, phi)
    # the accuracy cost of the batch size: the same mode at the reference's
    # default N_L = N_B = 2000 (engine.py:52-53), same verification sample
    at_default = None
    if econf.batch_size != 2000 or econf.leaf_size != 2000:
        from paper_2003_01836_b200 import EvalConfig
        dconf = EvalConfig(theta=econf.theta, degree=econf.degree, leaf_size=2000,
                           batch_size=2000, kernel=econf.kernel)
        t0 = time.perf_counter()
        phi_d, _ = ctx.treecode(system, dconf, mode=mode)
        at_default = {"leaf_size": 2000, "batch_size": 2000,
                      "error": cli.relative_error(ds, phi_d[sample]),
                      "wall_s_untimed_single_call": time.perf_counter() - t0,
                      "note": "the timed workload's N_B trades accuracy for speed; "
                              "profiles/r2_nb_table.jsonl has time and error per N_B"}
    return {"sample": int(sample.shape[0]), "error": err, "error_parity_mode": err_p,
            "error_at_reference_default_batch": at_default,
            "full_size_parity_vs_cpu_reference": sampled,
            "error_ratio": err / err_p if err_p else None,
            "vs_parity_strict_max_rel": strict,
            "vs_parity_condition_aware": float(d.max() / np.abs(phi_p).max()),
            "vs_parity_frac_targets_above_1e-10": float((d[nz] / np.abs(phi_p[nz]) > 1e-10).mean()),
            "direct_sum": f"GPU bltc_direct_sum PARITY ({t_ds:.1f}s); bitwise equal to the CPU "
                          f"oracle on {k} targets: {bool(np.array_equal(cpu, ds[:k]))}",
            "parity_mode_is_reference": "PARITY == reference bitwise (tests/test_gpu_parity.py)"}


def run_reference(args, cfg):
    """--impl reference: the reference's CPU algorithm (oracle/'s C port: the
    reference is Python/numba, not a compiled library -- its own timing on
    the same host is anchored separately, tools/reference_numba_step.py) on
    this host's cores, each step a bounded sample of the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    econf = eval_config(cfg, args.batch_size, args.leaf_size)
    system = make_system(cfg)
    ref = CpuReference(system, econf, budget_pairs=args.ref_budget)
    vals = []
    res = None
    for i in range(args.warmup + args.steps):
        res = ref.step()
        if i >= args.warmup:
            vals.append(res["value"])
        log(f"reference step {i}: {res['sample']}")
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "extrapolated": True, "metric": METRIC, "value": value,
        "unit": "particles/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg["n"] / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": cfg["n"], "theta": cfg["theta"],
                   "degree": cfg["degree"], "leaf_size": econf.leaf_size,
                   "batch_size": econf.batch_size, "kernel": ["coulomb", "yukawa", "const"][cfg["kind"]]},
        "cpu_baseline": {"value": value, "unit": "particles/s", "cores": res["cores"],
                         "kind": res["kind"], "sample": res["sample"], "extrapolated": True,
                         "cpu_model": res["cpu_model"],
                         "sampled_pair_fraction": res["sampled_pair_fraction"],
                         "anchor": "profiles/r2_cpu_full_step_*.json: unsampled full steps of "
                                   "the same C port, checking the extrapolation; "
                                   "profiles/r2_reference_numba_*.json: the unmodified numba "
                                   "reference on the same host (C4: 410.4 s per step on 16 "
                                   "threads, 1.5x slower than this port)"},
        "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, cfg):
    import torch

    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200 import engine

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: BLTC_BENCH_SHARE_GPU=1 maps every rank to cuda:0 and uses
    # gloo (NCCL refuses two ranks on one device) -- exercises the N>1 flow
    # on a one-GPU box; never used for a reported number
    share = os.environ.get("BLTC_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.rank_path:
        # keep stdout to the one JSON line (NCCL prints its version at INFO)
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    econf = eval_config(cfg, args.batch_size, args.leaf_size)
    system = make_system(cfg, device=local)
    n = cfg["n"]
    stream = torch.cuda.current_stream()
    ctx = bltc.Context(local, stream.cuda_stream)
    mode = args.mode
    params = engine.make_params(econf, mode)
    probe_tflops = 2.0 * probe_fp64(local) / 1e12

    if dist is not None:
        from paper_2003_01836_b200 import decomp
        runner = decomp.DeviceRankRunner(ctx, system, econf, mode=mode, group=dist.group.WORLD)
        step = runner.step
        n_local = runner.n_local
    else:
        s = system.sources
        dev = [torch.from_numpy(a).cuda() for a in (s.x, s.y, s.z, system.charges)]
        phi = torch.empty(n, dtype=torch.float64, device="cuda")
        ptrs = [t.data_ptr() for t in dev]

        def step():
            return ctx.treecode_device(params, n, ptrs[0], ptrs[1], ptrs[2], n, ptrs[0],
                                       ptrs[1], ptrs[2], ptrs[3], True, phi.data_ptr())
        n_local = n

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    stats = []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        l0 = launch_count()
        e0.record(stream)
        for _ in range(args.steps):
            stats.append(step())
        e1.record(stream)
        barrier()
        l1 = launch_count()
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = n / (ms * 1e-3)

    st = stats[-1]
    far_s = float(np.mean([x.far_s for x in stats]))
    near_s = float(np.mean([x.near_s for x in stats]))
    s_far, s_near = SLOTS[cfg["kind"]]
    far_tflops = 2.0 * s_far * st.approx_pairs / far_s / 1e12 if far_s > 0 else 0.0
    near_tflops = 2.0 * s_near * st.direct_pairs / near_s / 1e12 if near_s > 0 else 0.0
    launches = l1 - l0   # every libbltc kernel launched in the timed region
    # nominal FP64 peak: SMs x 64 FP64 lanes x 2 flop x the sampled SM clock
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count

    # ---- e2e through the public API with host buffers (H2D/D2H inside)
    e2e = None
    if dist is None:
        s = system.sources
        pinned = [torch.from_numpy(a).pin_memory() for a in (s.x, s.y, s.z, system.charges)]
        hx, hy, hz, hq = [t.numpy() for t in pinned]
        pts = bltc.Points(hx, hy, hz)
        psys = bltc.ParticleSystem.from_single_set(pts, hq)
        out = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
        for _ in range(2):
            bltc.treecode_potentials(psys, econf, mode=mode, context=ctx)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            ctx.treecode(psys, econf, mode=mode, out=out)
        t1 = time.perf_counter()
        e2e_s = (t1 - t0) / args.steps
        # the same call with the caller's ordinary (pageable) numpy arrays, as
        # a reference-side caller passes them (the driver's e2e is pinned)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            bltc.treecode_potentials(system, econf, mode=mode, context=ctx)
        e2e_pageable_s = (time.perf_counter() - t0) / args.steps
        e2e = {"value": n / e2e_s, "unit": "particles/s", "h2d_bytes_per_step": 4 * 8 * n,
               "d2h_bytes_per_step": 8 * n, "ms_per_step": 1e3 * e2e_s,
               "api": "paper_2003_01836_b200.treecode_potentials -> bltc_treecode (C ABI)",
               "host_buffers": "pinned",
               "pageable_ms_per_step": 1e3 * e2e_pageable_s}
    else:
        # run_distributed: host arrays in, RCB on the host, H2D of the rank's
        # slice, device pipeline + NCCL forest all-gather, D2H + gather of phi
        from paper_2003_01836_b200 import decomp
        eng = lambda: decomp.DeviceRankEngine(econf, mode, context=ctx)  # noqa: E731
        # FAST: the RCB cuts on the device (DeviceRcb), PARITY: the reference's
        # numpy RCB (its within-rank order is part of the bitwise result)
        part = "device" if mode == "fast" else "host"
        decomp.run_distributed(system, econf, ranks=world, mode=mode, engine_factory=eng,
                               partition=part)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            decomp.run_distributed(system, econf, ranks=world, mode=mode, engine_factory=eng,
                                   partition=part)
        torch.cuda.synchronize()
        t = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64,
                         device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
        e2e = {"value": n / e2e_s, "unit": "particles/s", "h2d_bytes_per_step": 4 * 8 * n,
               "d2h_bytes_per_step": 8 * n, "ms_per_step": 1e3 * e2e_s,
               "api": "paper_2003_01836_b200.decomp.run_distributed (RCB on the device for "
                      "FAST, LET exchange over NCCL)"}

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    traffic = None
    tp = os.path.join(ROOT, "profiles", "far_traffic.json")
    if world == 1 and os.path.exists(tp):   # a single-device capture
        try:
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("config") == args.config and tj.get("batch_size") == econf.batch_size:
                traffic = tj.get("bytes_per_launch")
        except (OSError, ValueError):
            traffic = None

    line = {
        "metric": METRIC, "value": value, "unit": "particles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "n": n, "theta": cfg["theta"],
                   "degree": cfg["degree"], "leaf_size": econf.leaf_size,
                   "batch_size": econf.batch_size,
                   "kernel": ["coulomb", "yukawa", "const"][cfg["kind"]], "mode": mode,
                   "parallelism": f"rcb{world}" if world > 1 else "single",
                   "l2": "inputs (32 B/particle = 256 MB at 8M) larger than the 126 MB L2"},
        "phases_s": {"setup": st.setup_s, "precompute": st.precompute_s,
                     "compute": st.compute_s, "far": far_s, "near": near_s,
                     "strict_certify_recompute": float(np.mean([x.strict_s for x in stats]))},
        "strict": {"recomputed_targets": int(st.n_recomputed),
                   "note": "STRICT: targets whose FAST value is not certified within 0.5e-10 "
                           "of the reference are recomputed in the reference's arithmetic "
                           "(-1: evaluated as PARITY)"},
        "pairs": {"approx": st.approx_pairs, "direct": st.direct_pairs,
                  "clusters": st.n_clusters, "batches": st.n_batches,
                  "moments": st.n_moments},
        "roofline": {"bound": "fp64",
                     "kernel": ("k_far_packed" if getattr(st, "packed", 0) else "k_far_fast") + " (far field)",
                     "achieved": far_tflops, "peak": None, "unit": "TFLOP/s", "frac": None,
                     "traffic": traffic,
                     "work": f"{s_far} FP64 slots/pair x approx pairs (2 flop/slot)",
                     "peak_source": "nominal FP64: SMs x 64 FP64 lanes x 2 flop x the median SM "
                                    "clock sampled during the timed region (MEASURED_PEAKS.json "
                                    "has no FP64 entry)",
                     "peak_probe": probe_tflops,
                     "peak_probe_source": "bltc_probe_fp64: sustained DFMA loop in this process "
                                          "(~0.3 s), for reference"},
        "near_roofline": {"kernel": ("k_near_packed" if getattr(st, "packed", 0) else "k_near_fast")
                                     + " (near field)", "achieved": near_tflops, "frac": None,
                          "work": f"{s_near} FP64 slots/pair x direct pairs"},
        "interaction_tflops": (2.0 * (s_far * st.approx_pairs + s_near * st.direct_pairs)
                               / (far_s + near_s) / 1e12) if far_s + near_s > 0 else None,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    csum = line["clocks"]
    f_mhz = csum.get("sm_mhz") or csum.get("sm_max_mhz")
    if f_mhz:
        nominal_tflops = sm_count * 64 * 2 * f_mhz * 1e6 / 1e12
        line["roofline"]["peak"] = nominal_tflops
        line["roofline"]["frac"] = far_tflops / nominal_tflops
        line["near_roofline"]["frac"] = near_tflops / nominal_tflops
        if line["interaction_tflops"]:
            line["interaction_frac"] = line["interaction_tflops"] / nominal_tflops
    if e2e is not None:
        line["e2e"] = e2e
    cpu_ref = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu_ref = CpuReference(system, econf, budget_pairs=args.ref_budget)
            cb = cpu_ref.step()
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind",
                                                      "sample", "extrapolated", "cpu_model",
                                                      "sampled_pair_fraction")}
        except Exception as exc:   # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if dist is None and not args.no_accuracy:
        try:
            line["accuracy"] = accuracy_block(ctx, system, econf, mode, out, args, cpu_ref)
        except Exception as exc:   # reported, never required for the timing line
            line["accuracy"] = {"error": repr(exc)}
    print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c4")
    ap.add_argument("--mode", choices=["strict", "fast", "parity"], default="strict")
    ap.add_argument("--batch-size", type=int, default=None)
    ap.add_argument("--leaf-size", type=int, default=None)
    ap.add_argument("--ref-budget", type=float, default=1.5e10,
                    help="pairs evaluated by the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true")
    ap.add_argument("--accuracy-sample", type=int, default=4000)
    ap.add_argument("--rank-path", action="store_true",
                    help="use the distributed (RCB + NCCL all-gather) path even at N=1")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: --warmup raised to 3 (timing rules)")
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
