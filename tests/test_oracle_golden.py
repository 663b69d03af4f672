"""Pin the CPU oracle against golden vectors the reference itself produced.

The oracle (oracle/bltc_oracle.c + oracle/oracle.py) is the checker for the
CUDA path, so before it is trusted it must reproduce the reference: tree,
batches and interaction lists element for element, moments and potentials
bit for bit (Yukawa included: both sides call the host libm exp).
"""
import numpy as np
import pytest
from conftest import golden, golden_system

CASES = ["c1_coulomb", "small_yukawa", "small_const", "plummer", "deg8"]


def _state(orc, g):
    s = golden_system(g)
    src = s.sources
    return orc.treecode_potentials(src.x, src.y, src.z, src.x, src.y, src.z, s.charges,
                                   True, float(g["theta"]), int(g["degree"]), int(g["leaf"]),
                                   int(g["batch"]), int(g["kind"]), float(g["kappa"]),
                                   threads=4, all_moments=True, return_state=True)


def test_generator_matches_reference():
    from paper_2003_01836_b200 import cli
    g = golden("generators")
    s = cli.generate_particles(1000, 1)
    np.testing.assert_array_equal(s.sources.x, g["x"])
    np.testing.assert_array_equal(s.sources.y, g["y"])
    np.testing.assert_array_equal(s.sources.z, g["z"])
    np.testing.assert_array_equal(s.charges, g["q"])
    np.testing.assert_array_equal(cli.sample_indices(1000, 50, 1), g["sample"])


@pytest.mark.parametrize("case", CASES)
def test_oracle_structures_bit_exact(oracle, case):
    g = golden(case)
    phi, stats, st = _state(oracle, g)
    t, b, lists = st["tree"], st["batches"], st["lists"]
    np.testing.assert_array_equal(t.perm, g["tree_perm"])
    np.testing.assert_array_equal(t.start, g["tree_start"])
    np.testing.assert_array_equal(t.stop, g["tree_stop"])
    np.testing.assert_array_equal(t.lo, g["tree_lo"])
    np.testing.assert_array_equal(t.hi, g["tree_hi"])
    np.testing.assert_array_equal(t.center, g["tree_center"])
    np.testing.assert_array_equal(t.radius, g["tree_radius"])
    np.testing.assert_array_equal(t.eligible.astype(np.uint8), g["tree_eligible"])
    np.testing.assert_array_equal(t.child_count, g["tree_child_count"])
    has = t.child_count > 0
    np.testing.assert_array_equal(t.child_start[has], g["tree_child_start"][has])
    np.testing.assert_array_equal(b.tree.perm, g["batch_perm"])
    np.testing.assert_array_equal(b.start, g["batch_start"])
    np.testing.assert_array_equal(b.stop, g["batch_stop"])
    np.testing.assert_array_equal(b.center, g["batch_center"])
    np.testing.assert_array_equal(b.radius, g["batch_radius"])
    np.testing.assert_array_equal(lists.a_ptr, g["lists_approx_ptr"])
    np.testing.assert_array_equal(lists.a_idx, g["lists_approx_idx"])
    np.testing.assert_array_equal(lists.d_ptr, g["lists_direct_ptr"])
    np.testing.assert_array_equal(lists.d_idx, g["lists_direct_idx"])
    assert stats.direct_pairs == int(g["direct_pairs"])
    assert stats.approx_pairs == int(g["approx_pairs"])
    assert stats.n_clusters == int(g["n_clusters"])
    assert stats.n_batches == int(g["n_batches"])
    # Chebyshev grid, axis 0, of every cluster (interp.py:35-56)
    for c in range(0, t.n_nodes, max(1, t.n_nodes // 25)):
        np.testing.assert_array_equal(
            oracle.cheb_points(int(g["degree"]), t.lo[c, 0], t.hi[c, 0]), g["tree_grid0"][c])


@pytest.mark.parametrize("case", CASES)
def test_oracle_moments_and_phi(oracle, case):
    g = golden(case)
    phi, stats, st = _state(oracle, g)
    rows, mrow = st["rows"], st["mrow"]
    has = g["moments_has"].astype(bool)
    np.testing.assert_array_equal(mrow >= 0, has)
    np.testing.assert_array_equal(rows[mrow[has]], g["moments"][has])
    # Yukawa included: numba's math.exp lowers to the host libm exp, as here.
    np.testing.assert_array_equal(phi, g["phi"])


def test_oracle_intermediate(oracle):
    g = golden("c1_coulomb")
    _, _, st = _state(oracle, g)
    qt, fl = oracle.compute_intermediate(st["tree"], int(g["qtilde_cluster"]), int(g["degree"]))
    np.testing.assert_array_equal(qt, g["qtilde"])
    np.testing.assert_array_equal(fl, g["qtilde_flags"])


def test_oracle_all_direct_criterion3(oracle):
    g = golden("alldirect")
    s = golden_system(g)
    src = s.sources
    phi, stats = oracle.treecode_potentials(src.x, src.y, src.z, src.x, src.y, src.z,
                                            s.charges, True, 1e-9, 8, 2000, 2000, 0, 0.0,
                                            threads=4)
    assert stats.approx_pairs == 0
    np.testing.assert_array_equal(phi, g["phi"])


@pytest.mark.parametrize("case", ["c1_coulomb", "small_yukawa", "plummer"])
def test_oracle_direct_sum_and_error(oracle, case):
    g = golden(case)
    s = golden_system(g)
    src = s.sources
    ds = oracle.direct_sum(src.x, src.y, src.z, src.x, src.y, src.z, s.charges,
                           int(g["kind"]), float(g["kappa"]), g["sample"], threads=4)
    np.testing.assert_array_equal(ds, g["sample_direct"])
    from paper_2003_01836_b200.cli import relative_error
    err = relative_error(ds, g["phi"][g["sample"]])
    assert abs(err - float(g["sample_error"])) <= 1e-6 * float(g["sample_error"])


def test_oracle_edge_cases(oracle):
    g = golden("edge_cases")
    corners = np.array([[sx, sy, sz] for sx in (-0.5, 0.5) for sy in (-0.5, 0.5)
                        for sz in (-0.5, 0.5)])
    t = oracle.partition(corners[:, 0], corners[:, 1], corners[:, 2], 1)
    np.testing.assert_array_equal(t.start, g["corners_t_start"])
    np.testing.assert_array_equal(t.lo, g["corners_t_lo"])
    np.testing.assert_array_equal(t.perm, g["corners_t_perm"])
    same = np.tile([[0.3, -0.2, 0.9]], (3000, 1))
    t = oracle.partition(same[:, 0], same[:, 1], same[:, 2], 2000)
    assert t.n_nodes == 1 and not t.eligible[0]
    np.testing.assert_array_equal(t.eligible.astype(np.uint8), g["identical_t_eligible"])
    phi, stats = oracle.treecode_potentials(g["sep_tx"], g["sep_ty"], g["sep_tz"], g["sep_sx"],
                                            g["sep_sy"], g["sep_sz"], g["sep_q"], False, 0.7, 5,
                                            300, 200, 0, 0.0)
    np.testing.assert_array_equal(phi, g["sep_phi"])
    assert stats.direct_pairs == int(g["sep_direct"])
    assert stats.approx_pairs == int(g["sep_approx"])


@pytest.mark.parametrize("case", ["dist_r3", "dist_r4_yukawa"])
def test_oracle_distributed(oracle, case):
    g = golden(case)
    s = golden_system(g)
    src = s.sources
    phi, info = oracle.run_distributed(src.x, src.y, src.z, s.charges, int(g["ranks"]),
                                       float(g["theta"]), int(g["degree"]), int(g["leaf"]),
                                       int(g["batch"]), int(g["kind"]), float(g["kappa"]),
                                       threads=4)
    np.testing.assert_array_equal(info["order"], g["order"])
    np.testing.assert_array_equal(info["rank_start"], g["rank_start"])
    assert info["direct_pairs"] == int(g["direct_pairs"])
    assert info["approx_pairs"] == int(g["approx_pairs"])
    np.testing.assert_array_equal(phi, g["phi"])
