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
    exact = mode == "parity" and int(g["kind"]) == 0
    _check(phi, g["phi"], exact, 1e-14 if mode == "parity" else 1e-13)
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
