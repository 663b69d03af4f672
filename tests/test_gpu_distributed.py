"""GPU distributed path (bltc_rank_build / _publish / _evaluate through the
DeviceRankEngine) with the ranks simulated back to back on one device: the
semantics a one-process-per-GPU NCCL run computes, checked against the
reference's run_distributed (golden vectors) and the oracle."""
import os

import numpy as np
import pytest
from conftest import golden, golden_system

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bltc():
    import paper_2003_01836_b200 as pkg
    pkg._lib.load()
    return pkg


def _cfg(bltc, g):
    kernel = [bltc.coulomb(), bltc.yukawa(float(g["kappa"]))][int(g["kind"])]
    return bltc.EvalConfig(theta=float(g["theta"]), degree=int(g["degree"]),
                           leaf_size=int(g["leaf"]), batch_size=int(g["batch"]), kernel=kernel)


def _check(phi, ref, exact_bits, scale_tol=1e-13):
    if exact_bits:
        np.testing.assert_array_equal(phi, ref)
    else:
        assert np.abs(phi - ref).max() <= scale_tol * np.abs(ref).max()


@pytest.mark.parametrize("case", ["dist_r3", "dist_r4_yukawa"])
@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_simulated_ranks_match_reference(bltc, case, mode):
    from paper_2003_01836_b200.decomp import run_distributed
    g = golden(case)
    s = golden_system(g)
    phi, st = run_distributed(s, _cfg(bltc, g), ranks=int(g["ranks"]), mode=mode)
    _check(phi, g["phi"], mode == "parity", 1e-13)
    assert st.direct_pairs == int(g["direct_pairs"])
    assert st.approx_pairs == int(g["approx_pairs"])


def test_single_rank_is_serial_engine_bitwise(bltc):
    """R=1 reproduces treecode_potentials bitwise (test_decomp.py:214-221)."""
    from paper_2003_01836_b200 import cli
    from paper_2003_01836_b200.decomp import run_distributed
    s = cli.generate_particles(5000, 91)
    cfg = bltc.EvalConfig(theta=0.7, degree=5, leaf_size=250, batch_size=250)
    serial, _ = bltc.treecode_potentials(s, cfg, mode="parity")
    phi, st = run_distributed(s, cfg, ranks=1, mode="parity")
    np.testing.assert_array_equal(phi, serial)
    assert st.n_ranks == 1 and st.fetch_stats == {}


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_plummer_ranks_vs_oracle(bltc, oracle, ranks):
    from paper_2003_01836_b200 import cli
    from paper_2003_01836_b200.decomp import run_distributed
    s = cli.generate_plummer(120_000, 5)
    src = s.sources
    cfg = bltc.EvalConfig(theta=0.8, degree=8, leaf_size=1000, batch_size=500)
    ref, info = oracle.run_distributed(src.x, src.y, src.z, s.charges, ranks, 0.8, 8, 1000, 500,
                                       0, 0.0, threads=os.cpu_count() or 1)
    phi, st = run_distributed(s, cfg, ranks=ranks, mode="parity")
    np.testing.assert_array_equal(phi, ref)
    assert (st.direct_pairs, st.approx_pairs) == (info["direct_pairs"], info["approx_pairs"])
    phi_f, _ = run_distributed(s, cfg, ranks=ranks, mode="fast")
    _check(phi_f, ref, False)


@pytest.mark.parametrize("case", ["dist_r3", "dist_r4_yukawa"])
def test_let_exchange_matches_reference_fetch(bltc, case):
    """The two-step LET exchange on the device (bltc_rank_needs + the fetched,
    remapped forest): potentials bitwise those of the replicated forest, fetch
    volume per (origin, owner) equal to the reference's build_let."""
    from paper_2003_01836_b200.decomp import run_distributed
    g = golden(case)
    s = golden_system(g)
    R = int(g["ranks"])
    phi_l, st_l = run_distributed(s, _cfg(bltc, g), ranks=R, mode="parity", exchange="let")
    phi_r, st_r = run_distributed(s, _cfg(bltc, g), ranks=R, mode="parity",
                                  exchange="replicate")
    np.testing.assert_array_equal(phi_l, phi_r)
    fetch = np.array([[o, w, f.tree_records, f.clusters, f.moments, f.particles]
                      for (o, w), f in sorted(st_l.fetch_stats.items())], dtype=np.int64)
    np.testing.assert_array_equal(fetch, g["fetch"])
    assert (st_l.direct_pairs, st_l.approx_pairs) == (st_r.direct_pairs, st_r.approx_pairs)


@pytest.mark.parametrize("ranks", [2, 3, 8])
def test_device_rcb_same_rank_sets(bltc, ranks):
    """RCB on the device: the reference's cuts -- every rank receives the same
    particle set (and count) as numpy's rcb_partition, only the order within
    a rank differs."""
    import torch
    from paper_2003_01836_b200 import cli
    from paper_2003_01836_b200.decomp import DeviceRcb, rcb_partition
    s = cli.generate_plummer(50_000, 21)
    src = s.sources
    host = rcb_partition(src, ranks)
    dev = torch.device("cuda", 0)
    d = DeviceRcb(*(torch.from_numpy(np.asarray(v)).to(dev) for v in (src.x, src.y, src.z)),
                  ranks)
    np.testing.assert_array_equal(d.counts, host.counts)
    for r in range(ranks):
        np.testing.assert_array_equal(np.sort(d.rank_indices(r).cpu().numpy()),
                                      np.sort(host.rank_indices(r)))


def test_fast_device_partition_matches_reference(bltc):
    from paper_2003_01836_b200.decomp import run_distributed
    g = golden("dist_r4_yukawa")
    s = golden_system(g)
    phi, st = run_distributed(s, _cfg(bltc, g), ranks=int(g["ranks"]), mode="fast",
                              partition="device")
    _check(phi, g["phi"], False, 1e-13)
    assert (st.direct_pairs, st.approx_pairs) == (int(g["direct_pairs"]),
                                                  int(g["approx_pairs"]))


@pytest.mark.parametrize("case", ["dist_r3", "dist_r4_yukawa"])
@pytest.mark.parametrize("mode", ["parity", "fast", "strict"])
def test_c_run_distributed_matches_reference(bltc, case, mode):
    """bltc_run_distributed (one C call, one host thread per rank) reproduces
    the reference's run_distributed: PARITY bitwise, STRICT within 1e-10 on
    every target."""
    from paper_2003_01836_b200.decomp import run_distributed_native
    g = golden(case)
    s = golden_system(g)
    phi, st = run_distributed_native(s, _cfg(bltc, g), ranks=int(g["ranks"]), devices=[0],
                                     mode=mode)
    if mode == "strict":
        ref = g["phi"]
        assert np.all(np.abs(phi - ref) <= 1e-10 * np.abs(ref))
    else:
        _check(phi, g["phi"], mode == "parity", 1e-13)
    assert st.direct_pairs == int(g["direct_pairs"])
    assert st.approx_pairs == int(g["approx_pairs"])
    np.testing.assert_array_equal(st.rank_counts, np.diff(g["rank_start"]))


def test_c_run_distributed_plummer_vs_python_path(bltc):
    from paper_2003_01836_b200 import cli
    from paper_2003_01836_b200.decomp import run_distributed, run_distributed_native
    s = cli.generate_plummer(60_000, 9)
    cfg = bltc.EvalConfig(theta=0.8, degree=6, leaf_size=500, batch_size=500)
    a, sa = run_distributed(s, cfg, ranks=4, mode="parity")
    b, sb = run_distributed_native(s, cfg, ranks=4, devices=[0], mode="parity")
    np.testing.assert_array_equal(a, b)
    assert (sa.direct_pairs, sa.approx_pairs) == (sb.direct_pairs, sb.approx_pairs)


def test_c_run_distributed_rejects_bad_partition(bltc):
    import ctypes
    from paper_2003_01836_b200 import _lib, cli
    from paper_2003_01836_b200.engine import cheb_nodes, make_params
    s = cli.generate_particles(100, 1)
    cfg = bltc.EvalConfig(theta=0.8, degree=2, leaf_size=10, batch_size=10)
    p = make_params(cfg)
    x = np.ascontiguousarray(s.sources.x)
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    ip = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    order = np.arange(100, dtype=np.int64)
    start = np.array([0, 60, 90], dtype=np.int64)        # does not end at n
    dev = np.zeros(1, np.int32)
    phi = np.empty(100)
    rc = _lib.load().bltc_run_distributed(
        2, dev.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 1, ctypes.byref(p),
        dp(cheb_nodes(2)), 100, dp(x), dp(x), dp(x), dp(x), ip(order), ip(start), dp(phi), None)
    assert rc == -1


def test_rank_domain_filter_keeps_results(bltc):
    """bltc_rank_set_domain: a rank publishes only the moment rows some batch
    of the global domain could accept -- fewer rows (at R = 1 the root and
    the other clusters no batch can reach drop out), bitwise the same PARITY
    potentials as publishing every size-eligible row."""
    import torch

    from paper_2003_01836_b200 import cli
    from paper_2003_01836_b200.decomp import DeviceRankEngine
    s = cli.generate_plummer(60_000, 8)
    src = s.sources
    cfg = bltc.EvalConfig(theta=0.8, degree=6, leaf_size=500, batch_size=160)
    lo = [float(np.min(a)) for a in (src.x, src.y, src.z)]
    hi = [float(np.max(a)) for a in (src.x, src.y, src.z)]
    out, rows = {}, {}
    for filt in (False, True):
        eng = DeviceRankEngine(cfg, "parity")
        if filt:
            eng.set_domain(lo, hi)
        eng.build(*(np.asarray(a) for a in (src.x, src.y, src.z, s.charges)))
        pub = eng.publish()
        rows[filt] = pub.sizes[2]
        out[filt] = eng.evaluate(1, 0, [pub]).cpu().numpy()
        eng.ctx.close()
    assert rows[True] < rows[False]
    np.testing.assert_array_equal(out[True], out[False])
    ref, _ = bltc.treecode_potentials(s, cfg, mode="parity")
    np.testing.assert_array_equal(out[True], ref)


@pytest.mark.gpu
def test_rank_domain_cell_boxes(bltc):
    """bltc_rank_set_domain_boxes with decomp.domain_boxes' occupied-cell
    boxes: at most the one-box domain's rows; invalid boxes rejected."""
    from paper_2003_01836_b200 import cli
    from paper_2003_01836_b200.decomp import DeviceRankEngine, domain_boxes, rcb_partition
    s = cli.generate_plummer(60_000, 9)
    src = s.sources
    cfg = bltc.EvalConfig(theta=0.8, degree=6, leaf_size=500, batch_size=160)
    boxes = domain_boxes(src.x, src.y, src.z)
    part = rcb_partition(src, 2)
    idx = part.rank_indices(0)
    rows = {}
    for mode in ("box", "cells"):
        eng = DeviceRankEngine(cfg, "parity")
        if mode == "box":
            eng.set_domain(boxes[:, :3].min(axis=0), boxes[:, 3:].max(axis=0))
        else:
            eng.set_domain_boxes(boxes)
        eng.build(*(np.ascontiguousarray(np.asarray(a)[idx])
                    for a in (src.x, src.y, src.z, s.charges)))
        rows[mode] = eng.publish_sizes()[2]
        eng.ctx.close()
    assert rows["cells"] <= rows["box"]
    # (run_distributed passes the cell boxes to every rank: the oracle
    # comparisons of the distributed tests above run through them)
    ctx = bltc.Context(0)
    with pytest.raises(ValueError):
        ctx.rank_set_domain_boxes(np.array([[0.0, 0.0, 0.0, -1.0, 1.0, 1.0]]))
    with pytest.raises(ValueError):
        ctx.rank_set_domain_boxes(np.array([[np.nan, 0.0, 0.0, 1.0, 1.0, 1.0]]))
    ctx.rank_set_domain_boxes(np.empty((0, 6)))
    ctx.close()
