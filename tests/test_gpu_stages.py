"""Stage-level drop-ins on the reference's own structures (golden vectors
produced by the reference: tree, batches, lists, moments): each stage alone,
bit for bit in PARITY mode (stages.py, bltc_stage_*)."""
import numpy as np
import pytest
from conftest import golden, golden_system

pytestmark = pytest.mark.gpu

CASES = ["c1_coulomb", "plummer", "small_yukawa", "deg8"]


@pytest.fixture(scope="module")
def bltc():
    import paper_2003_01836_b200 as pkg
    pkg._lib.load()
    return pkg


def _cfg(bltc, g):
    kind = int(g["kind"])
    kernel = [bltc.coulomb(), bltc.yukawa(float(g["kappa"])), bltc.test_constant()][kind]
    return bltc.EvalConfig(theta=float(g["theta"]), degree=int(g["degree"]),
                           leaf_size=int(g["leaf"]), batch_size=int(g["batch"]), kernel=kernel)


def _structures(g):
    from paper_2003_01836_b200.stages import FlatBatches, FlatLists, FlatTree
    s = golden_system(g)
    src = s.sources
    tp = g["tree_perm"]                       # original -> reordered
    order = np.empty_like(tp)
    order[tp] = np.arange(tp.shape[0])
    tree = FlatTree(start=g["tree_start"], stop=g["tree_stop"], lo=g["tree_lo"],
                    hi=g["tree_hi"], child_start=g["tree_child_start"],
                    child_count=g["tree_child_count"], x=src.x[order], y=src.y[order],
                    z=src.z[order], q=s.charges[order])
    bp = g["batch_perm"]
    border = np.empty_like(bp)
    border[bp] = np.arange(bp.shape[0])
    t = s.targets
    batches = FlatBatches(start=g["batch_start"], stop=g["batch_stop"], center=g["batch_center"],
                          radius=g["batch_radius"], x=t.x[border], y=t.y[border],
                          z=t.z[border], perm=bp)
    lists = FlatLists(g["lists_approx_ptr"], g["lists_approx_idx"], g["lists_direct_ptr"],
                      g["lists_direct_idx"])
    return tree, batches, lists


@pytest.mark.parametrize("case", CASES)
def test_stage_lists_bit_exact(bltc, case):
    from paper_2003_01836_b200 import stages
    g = golden(case)
    tree, batches, _ = _structures(g)
    L = stages.build_interaction_lists(batches, tree, _cfg(bltc, g))
    np.testing.assert_array_equal(L.a_ptr, g["lists_approx_ptr"])
    np.testing.assert_array_equal(L.a_idx, g["lists_approx_idx"])
    np.testing.assert_array_equal(L.d_ptr, g["lists_direct_ptr"])
    np.testing.assert_array_equal(L.d_idx, g["lists_direct_idx"])


@pytest.mark.parametrize("case", CASES)
def test_stage_moments(bltc, case):
    from paper_2003_01836_b200 import stages
    g = golden(case)
    tree, _, _ = _structures(g)
    ids = np.nonzero(g["moments_has"])[0]
    rows = stages.compute_moments(tree, _cfg(bltc, g), ids, mode="parity")
    np.testing.assert_array_equal(rows, g["moments"][ids])
    rows_all = stages.compute_moments(tree, _cfg(bltc, g), None, mode="parity")
    np.testing.assert_array_equal(rows_all, g["moments"][ids])   # default: every eligible
    fast = stages.compute_moments(tree, _cfg(bltc, g), ids, mode="fast")
    ref = g["moments"][ids]
    assert (np.abs(fast - ref) / (np.abs(ref).max(axis=1, keepdims=True) + 1e-300)).max() <= 1e-13


@pytest.mark.parametrize("case", CASES)
def test_stage_potentials(bltc, case):
    from paper_2003_01836_b200 import stages
    g = golden(case)
    tree, batches, lists = _structures(g)
    has = g["moments_has"].astype(bool)
    mrow = np.where(has, np.cumsum(has) - 1, -1)
    rows = g["moments"][has]
    cfg = _cfg(bltc, g)
    phi, st = stages.compute_potentials(batches, tree, rows, lists, cfg, mode="parity",
                                        moment_row=mrow, return_stats=True)
    ref = g["phi"]
    np.testing.assert_array_equal(phi, ref)
    assert (st.direct_pairs, st.approx_pairs) == (int(g["direct_pairs"]), int(g["approx_pairs"]))
    phi_f = stages.compute_potentials(batches, tree, rows, lists, cfg, mode="fast",
                                         moment_row=mrow)
    assert np.abs(phi_f - ref).max() <= 1e-13 * np.abs(ref).max()


def test_stage_potentials_validates(bltc):
    from paper_2003_01836_b200 import stages
    g = golden("c1_coulomb")
    tree, batches, lists = _structures(g)
    mrow = np.full(len(tree.start), -1)   # approximated clusters without a row
    with pytest.raises(ValueError):
        stages.compute_potentials(batches, tree, np.zeros((0, 125)), lists, _cfg(bltc, g),
                                  moment_row=mrow)


def test_stage_potentials_validates_batches_and_perm(bltc):
    """Bad caller structures are rejected on the host (ValueError), before
    any device read: batch ranges beyond the targets, non-monotone CSR
    offsets, perm entries out of range."""
    import copy
    from paper_2003_01836_b200 import stages
    g = golden("c1_coulomb")
    tree, batches, lists = _structures(g)
    has = g["moments_has"].astype(bool)
    mrow = np.where(has, np.cumsum(has) - 1, -1)
    rows = g["moments"][has]
    cfg = _cfg(bltc, g)
    bad = copy.copy(batches)
    bad.stop = batches.stop.copy()
    bad.stop[-1] = len(batches.x) + 5
    with pytest.raises(ValueError, match="batch target range"):
        stages.compute_potentials(bad, tree, rows, lists, cfg, mode="parity", moment_row=mrow)
    bad = copy.copy(batches)
    bad.perm = batches.perm.copy()
    bad.perm[0] = len(batches.x)
    with pytest.raises(ValueError, match="perm"):
        stages.compute_potentials(bad, tree, rows, lists, cfg, mode="parity", moment_row=mrow)
    badl = copy.copy(lists)
    badl.a_ptr = lists.a_ptr.copy()
    badl.a_ptr[1] = badl.a_ptr[2] + 1
    with pytest.raises(ValueError):
        stages.compute_potentials(batches, tree, rows, badl, cfg, mode="parity", moment_row=mrow)


def test_compute_all_moments_reference_shape(bltc):
    """compute_all_moments (moments.py:147-150): list indexed by cluster,
    ClusterMoments for eligible clusters, None otherwise -- bitwise rows."""
    from paper_2003_01836_b200 import stages
    g = golden("plummer")
    tree, _, _ = _structures(g)
    mm = stages.compute_all_moments(tree, _cfg(bltc, g), mode="parity")
    has = g["moments_has"].astype(bool)
    assert len(mm) == len(has)
    for ci, m in enumerate(mm):
        assert (m is not None) == bool(has[ci])
        if m is not None:
            assert m.cluster_index == ci
            np.testing.assert_array_equal(m.q_hat, g["moments"][ci])
