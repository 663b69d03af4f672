"""GPU parity: the CUDA path against the reference's golden vectors and the
pinned CPU oracle, through the C ABI (libbltc.so via ctypes).

Bars:
* tree, batches, interaction lists: bit-exact
* moments: bit-exact
* PARITY potentials: bit-exact (Coulomb, Yukawa -- the device port of the
  host libm exp, csrc/libm_exp.cuh -- and constant)
* FAST potentials: condition-aware max|d| / max|phi| <= 1e-13 and strict
  per-target relative <= 1e-10 away from near-cancelling targets
"""
import numpy as np
import pytest
from conftest import golden, golden_system

pytestmark = pytest.mark.gpu

CASES = ["c1_coulomb", "small_yukawa", "small_const", "plummer", "deg8"]


@pytest.fixture(scope="module")
def bltc():
    import paper_2003_01836_b200 as pkg
    pkg._lib.load()
    return pkg


@pytest.fixture(scope="module")
def ctx(bltc):
    c = bltc.Context(0)
    yield c
    c.close()


def _config(bltc, g):
    kind = int(g["kind"])
    kernel = [bltc.coulomb(), bltc.yukawa(float(g["kappa"])), bltc.test_constant()][kind]
    return bltc.EvalConfig(theta=float(g["theta"]), degree=int(g["degree"]),
                           leaf_size=int(g["leaf"]), batch_size=int(g["batch"]), kernel=kernel)


def _phi_check(phi, ref, kind, exact):
    if exact:
        np.testing.assert_array_equal(phi, ref)
    else:
        # FAST is the uncertified mode: its contract is the condition-aware
        # bar (|d_i| <= 1e-13 max |phi|), NOT the per-target one -- a near-
        # cancelling target can exceed 1e-10 relative.  The per-target bar on
        # EVERY target (no masking) is STRICT's: tests/test_gpu_strict.py.
        scale = np.abs(ref).max()
        assert np.abs(phi - ref).max() <= 1e-13 * scale


@pytest.mark.parametrize("case", CASES)
def test_structures_and_moments_bit_exact(bltc, ctx, case):
    g = golden(case)
    system = golden_system(g)
    cfg = _config(bltc, g)
    phi, stats = ctx.treecode(system, cfg, mode="parity", all_moments=True)
    t = ctx.export_tree(0)
    np.testing.assert_array_equal(t["perm"], g["tree_perm"])
    np.testing.assert_array_equal(t["start"], g["tree_start"])
    np.testing.assert_array_equal(t["stop"], g["tree_stop"])
    np.testing.assert_array_equal(t["lo"], g["tree_lo"])
    np.testing.assert_array_equal(t["hi"], g["tree_hi"])
    np.testing.assert_array_equal(t["child_count"], g["tree_child_count"])
    has = t["child_count"] > 0
    np.testing.assert_array_equal(t["child_start"][has], g["tree_child_start"][has])
    b = ctx.export_batches()
    np.testing.assert_array_equal(b["start"], g["batch_start"])
    np.testing.assert_array_equal(b["stop"], g["batch_stop"])
    np.testing.assert_array_equal(b["center"], g["batch_center"])
    np.testing.assert_array_equal(b["radius"], g["batch_radius"])
    np.testing.assert_array_equal(ctx.export_tree(1)["perm"], g["batch_perm"])
    L = ctx.export_lists()
    np.testing.assert_array_equal(L["a_ptr"], g["lists_approx_ptr"])
    np.testing.assert_array_equal(L["a_idx"], g["lists_approx_idx"])
    np.testing.assert_array_equal(L["d_ptr"], g["lists_direct_ptr"])
    np.testing.assert_array_equal(L["d_idx"], g["lists_direct_idx"])
    ids, rows = ctx.export_moments()
    elig = np.nonzero(g["moments_has"])[0]
    np.testing.assert_array_equal(ids, elig)
    np.testing.assert_array_equal(rows, g["moments"][elig])
    assert stats.direct_pairs == int(g["direct_pairs"])
    assert stats.approx_pairs == int(g["approx_pairs"])
    assert stats.n_clusters == int(g["n_clusters"])
    assert stats.n_batches == int(g["n_batches"])
    _phi_check(phi, g["phi"], int(g["kind"]), exact=True)


@pytest.mark.parametrize("case", ["c1_coulomb", "plummer", "deg8"])
@pytest.mark.parametrize("big", ["1", "700"])
def test_split_moments_bit_exact(bltc, case, big, monkeypatch):
    """The bitwise upward pass's split items (one CTA per k1, the t2 slot
    holding a[k1] t2 -- the path of clusters above 2^17 sources), forced onto
    every cluster above ``big`` sources: moments still bitwise the reference."""
    monkeypatch.setenv("BLTC_BW_BIG", big)
    g = golden(case)
    c = bltc.Context(0)
    c.build(golden_system(g), _config(bltc, g), mode="parity", all_moments=True)
    ids, rows = c.export_moments()
    elig = np.nonzero(g["moments_has"])[0]
    np.testing.assert_array_equal(ids, elig)
    np.testing.assert_array_equal(rows, g["moments"][elig])
    c.close()


@pytest.mark.parametrize("case", ["c1_coulomb", "plummer", "deg8"])
def test_build_only_structures_bit_exact(bltc, case):
    """bltc_build: setup + moments without an evaluation, same structures."""
    g = golden(case)
    c = bltc.Context(0)
    st = c.build(golden_system(g), _config(bltc, g), mode="parity", all_moments=True)
    t = c.export_tree(0)
    np.testing.assert_array_equal(t["perm"], g["tree_perm"])
    np.testing.assert_array_equal(t["start"], g["tree_start"])
    np.testing.assert_array_equal(t["lo"], g["tree_lo"])
    b = c.export_batches()
    np.testing.assert_array_equal(b["start"], g["batch_start"])
    np.testing.assert_array_equal(b["radius"], g["batch_radius"])
    L = c.export_lists()
    np.testing.assert_array_equal(L["a_idx"], g["lists_approx_idx"])
    np.testing.assert_array_equal(L["d_idx"], g["lists_direct_idx"])
    ids, rows = c.export_moments()
    elig = np.nonzero(g["moments_has"])[0]
    np.testing.assert_array_equal(ids, elig)
    np.testing.assert_array_equal(rows, g["moments"][elig])
    assert (st.direct_pairs, st.approx_pairs) == (int(g["direct_pairs"]), int(g["approx_pairs"]))
    assert st.compute_s == 0.0 or st.compute_s < 1e-3
    c.close()


@pytest.mark.parametrize("case", CASES)
def test_parity_mode_potentials(bltc, case):
    g = golden(case)
    phi, _ = bltc.treecode_potentials(golden_system(g), _config(bltc, g), mode="parity")
    _phi_check(phi, g["phi"], int(g["kind"]), exact=True)


@pytest.mark.parametrize("case", CASES)
def test_fast_mode_potentials(bltc, case):
    g = golden(case)
    phi, stats = bltc.treecode_potentials(golden_system(g), _config(bltc, g), mode="fast")
    _phi_check(phi, g["phi"], int(g["kind"]), exact=False)
    assert stats.direct_pairs == int(g["direct_pairs"])
    assert stats.approx_pairs == int(g["approx_pairs"])


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_all_direct_criterion3(bltc, mode):
    """theta=1e-9: no approximation at all (test_acceptance.py:86-97)."""
    g = golden("alldirect")
    cfg = bltc.EvalConfig(theta=1e-9, degree=8, leaf_size=2000, batch_size=2000)
    phi, stats = bltc.treecode_potentials(golden_system(g), cfg, mode=mode)
    assert stats.approx_pairs == 0
    _phi_check(phi, g["phi"], 0, exact=(mode == "parity"))


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_separate_targets_and_sources(bltc, mode):
    g = golden("edge_cases")
    tg = bltc.Points(g["sep_tx"], g["sep_ty"], g["sep_tz"])
    sr = bltc.Points(g["sep_sx"], g["sep_sy"], g["sep_sz"])
    system = bltc.ParticleSystem(targets=tg, sources=sr, charges=g["sep_q"])
    cfg = bltc.EvalConfig(theta=0.7, degree=5, leaf_size=300, batch_size=200)
    phi, stats = bltc.treecode_potentials(system, cfg, mode=mode)
    assert stats.direct_pairs == int(g["sep_direct"])
    assert stats.approx_pairs == int(g["sep_approx"])
    _phi_check(phi, g["sep_phi"], 0, exact=(mode == "parity"))


def test_degenerate_geometries(bltc, ctx):
    g = golden("edge_cases")
    corners = np.array([[sx, sy, sz] for sx in (-0.5, 0.5) for sy in (-0.5, 0.5)
                        for sz in (-0.5, 0.5)])
    system = bltc.ParticleSystem.from_single_set(bltc.Points.from_array(corners), np.ones(8))
    cfg = bltc.EvalConfig(theta=0.8, degree=2, leaf_size=1, batch_size=1)
    ctx.treecode(system, cfg, mode="parity")
    t = ctx.export_tree(0)
    np.testing.assert_array_equal(t["start"], g["corners_t_start"])
    np.testing.assert_array_equal(t["lo"], g["corners_t_lo"])
    np.testing.assert_array_equal(t["perm"], g["corners_t_perm"])
    same = np.tile([[0.3, -0.2, 0.9]], (3000, 1))
    system = bltc.ParticleSystem.from_single_set(bltc.Points.from_array(same), np.ones(3000))
    phi, stats = ctx.treecode(system, bltc.EvalConfig(theta=0.8, degree=4), mode="parity")
    assert stats.n_clusters == 1
    # every pair is singular: all potentials are exactly zero
    np.testing.assert_array_equal(phi, np.zeros(3000))


def test_single_leaf_and_single_target(bltc):
    pts = bltc.Points.from_array(np.array([[0.1, 0.2, 0.3]]))
    system = bltc.ParticleSystem.from_single_set(pts, np.array([2.0]))
    phi, stats = bltc.treecode_potentials(system, bltc.EvalConfig(theta=0.8, degree=8))
    assert phi.shape == (1,) and phi[0] == 0.0
    assert stats.n_clusters == 1 and stats.n_batches == 1


def test_constant_kernel_exact(bltc):
    """G == 1 is reproduced exactly by interpolation (test_engine.py:187-198)."""
    from paper_2003_01836_b200 import cli
    s = cli.generate_particles(3000, 29)
    cfg = bltc.EvalConfig(theta=0.9, degree=3, leaf_size=150, batch_size=150,
                          kernel=bltc.test_constant())
    for mode in ("parity", "fast"):
        phi, stats = bltc.treecode_potentials(s, cfg, mode=mode)
        assert stats.approx_pairs > 0
        np.testing.assert_allclose(phi, s.charges.sum() - s.charges, rtol=0, atol=1e-12)


def test_yukawa_zero_kappa_is_coulomb(bltc):
    """kappa=0 Yukawa == Coulomb bitwise in PARITY (test_engine.py:251-256)."""
    from paper_2003_01836_b200 import cli
    s = cli.generate_particles(4000, 47)
    base = dict(theta=0.7, degree=5, leaf_size=200, batch_size=200)
    pc, _ = bltc.treecode_potentials(s, bltc.EvalConfig(kernel=bltc.coulomb(), **base),
                                     mode="parity")
    py, _ = bltc.treecode_potentials(s, bltc.EvalConfig(kernel=bltc.yukawa(0.0), **base),
                                     mode="parity")
    np.testing.assert_array_equal(pc, py)


def test_deterministic_repeats(bltc):
    from paper_2003_01836_b200 import cli
    s = cli.generate_plummer(50_000, 11)
    cfg = bltc.EvalConfig(theta=0.8, degree=8, leaf_size=500, batch_size=250)
    for mode in ("parity", "fast"):
        a, _ = bltc.treecode_potentials(s, cfg, mode=mode)
        b, _ = bltc.treecode_potentials(s, cfg, mode=mode)
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("gen,n,leaf,batch,deg,theta", [
    ("uniform", 200_000, 2000, 2000, 8, 0.8),
    ("plummer", 200_000, 2000, 1000, 8, 0.8),
    ("uniform", 150_000, 1000, 500, 10, 0.7),
    ("uniform", 150_000, 2000, 160, 8, 0.8),    # the C2/C3 bench batch size
])
def test_oracle_parity_mid_size(bltc, ctx, oracle, gen, n, leaf, batch, deg, theta):
    """Mid-size runs against the oracle: structures bit-exact, PARITY phi
    bit-exact, FAST within tolerance."""
    import os
    from paper_2003_01836_b200 import cli
    s = (cli.generate_particles if gen == "uniform" else cli.generate_plummer)(n, 2)
    src = s.sources
    ref, ost, st = oracle.treecode_potentials(src.x, src.y, src.z, src.x, src.y, src.z,
                                              s.charges, True, theta, deg, leaf, batch, 0, 0.0,
                                              threads=os.cpu_count() or 1, return_state=True)
    cfg = bltc.EvalConfig(theta=theta, degree=deg, leaf_size=leaf, batch_size=batch)
    phi, stats = ctx.treecode(s, cfg, mode="parity")
    t = ctx.export_tree(0)
    np.testing.assert_array_equal(t["perm"], st["tree"].perm)
    np.testing.assert_array_equal(t["lo"], st["tree"].lo)
    np.testing.assert_array_equal(t["hi"], st["tree"].hi)
    L = ctx.export_lists()
    np.testing.assert_array_equal(L["a_idx"], st["lists"].a_idx)
    np.testing.assert_array_equal(L["d_idx"], st["lists"].d_idx)
    ids, rows = ctx.export_moments()
    np.testing.assert_array_equal(ids, np.unique(st["lists"].a_idx))
    np.testing.assert_array_equal(rows, st["rows"])
    assert (stats.direct_pairs, stats.approx_pairs) == (ost.direct_pairs, ost.approx_pairs)
    np.testing.assert_array_equal(phi, ref)
    phi_f, _ = ctx.treecode(s, cfg, mode="fast")
    _phi_check(phi_f, ref, 0, exact=False)


def test_context_reuse_across_sizes(bltc, oracle):
    """One context serving runs whose node counts grow and shrink (the
    partition scratch is shared between the source tree and the target
    batches, and grown level by level): structures stay bit-exact."""
    from paper_2003_01836_b200 import cli
    s = cli.generate_plummer(120_000, 5)
    src = s.sources
    c = bltc.Context(0)
    try:
        for leaf, batch in [(2000, 2000), (400, 60), (2000, 25), (60, 400), (1000, 250)]:
            cfg = bltc.EvalConfig(theta=0.8, degree=4, leaf_size=leaf, batch_size=batch)
            c.treecode(s, cfg, mode="fast")
            tree = oracle.build_source_tree(src.x, src.y, src.z, s.charges, leaf)
            t = c.export_tree(0)
            np.testing.assert_array_equal(t["perm"], tree.perm)
            np.testing.assert_array_equal(t["start"], tree.start)
            np.testing.assert_array_equal(t["lo"], tree.lo)
            np.testing.assert_array_equal(t["hi"], tree.hi)
            bt = oracle.build_target_batches(src.x, src.y, src.z, batch)
            b = c.export_batches()
            np.testing.assert_array_equal(b["start"], bt.start)
            np.testing.assert_array_equal(b["stop"], bt.stop)
            np.testing.assert_array_equal(b["radius"], bt.radius)
    finally:
        c.close()


@pytest.mark.parametrize("case", ["c1_coulomb", "plummer", "deg8"])
def test_fast_moments_close(bltc, ctx, case):
    """FAST upward pass (warp-cooperative, reciprocal-based factors, fused
    accumulation, piece-ordered reduction): rows within 1e-13 of the row's
    magnitude scale of the reference's moments."""
    g = golden(case)
    ctx.treecode(golden_system(g), _config(bltc, g), mode="fast", all_moments=True)
    ids, rows = ctx.export_moments()
    elig = np.nonzero(g["moments_has"])[0]
    np.testing.assert_array_equal(ids, elig)
    ref = g["moments"][elig]
    scale = np.abs(ref).max(axis=1, keepdims=True) + 1e-300
    assert (np.abs(rows - ref) / scale).max() <= 1e-13


@pytest.mark.parametrize("batch,leaf,deg", [(1, 8, 4), (2, 16, 5), (3, 40, 7), (7, 7, 8),
                                            (33, 64, 10), (65, 100, 8)])
def test_packed_items_ragged_batches(bltc, batch, leaf, deg):
    """Packed FAST items over windows spanning many tiny batches (odd sizes,
    one-target batches, windows split by the segment limit): FAST agrees with
    PARITY (the reference's arithmetic), also forced onto the packed path."""
    import os
    from paper_2003_01836_b200 import cli
    s = cli.generate_plummer(6000, 17)
    cfg = bltc.EvalConfig(theta=0.7, degree=deg, leaf_size=leaf, batch_size=batch)
    ref, _ = bltc.treecode_potentials(s, cfg, mode="parity")
    for force in ("", "1"):
        if force:
            os.environ["BLTC_PACK"] = force
        try:
            phi, st = bltc.treecode_potentials(s, cfg, mode="fast")
        finally:
            os.environ.pop("BLTC_PACK", None)
        _phi_check(phi, ref, 0, exact=False)
        if force:
            assert st.packed == 1


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_schedule_variants_bitwise_equal(bltc, mode, monkeypatch):
    """Work-item order (longest-first vs stream order) and the near-field
    staging engine (cp.async vs cp.async.bulk) change no bit of the result."""
    from paper_2003_01836_b200 import cli
    s = cli.generate_plummer(60_000, 13)
    cfg = bltc.EvalConfig(theta=0.8, degree=8, leaf_size=1000, batch_size=160)
    base, _ = bltc.treecode_potentials(s, cfg, mode=mode)
    for env in ({"BLTC_ITEM_SORT": "0"}, {"BLTC_NEAR_BULK": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        phi, _ = bltc.treecode_potentials(s, cfg, mode=mode)
        for k in env:
            monkeypatch.delenv(k)
        np.testing.assert_array_equal(phi, base)


@pytest.mark.parametrize("kappa", [1e-3, 5.0, 400.0, 5000.0])
def test_fast_yukawa_kappa_range(bltc, kappa):
    """FAST's folded-kappa exp (clamped at kappa r = 700) against PARITY over
    screening lengths from nearly Coulomb to underflowing far fields."""
    from paper_2003_01836_b200 import cli
    s = cli.generate_particles(40_000, 5)
    cfg = bltc.EvalConfig(theta=0.7, degree=8, leaf_size=500, batch_size=160,
                          kernel=bltc.yukawa(kappa))
    ref, _ = bltc.treecode_potentials(s, cfg, mode="parity")
    phi, _ = bltc.treecode_potentials(s, cfg, mode="fast")
    assert np.all(np.isfinite(phi))
    assert np.abs(phi - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("deg", list(range(1, 13)))
def test_every_packed_degree(bltc, oracle, deg, monkeypatch):
    """Degrees 1..12 run on the packed kernels: PARITY bitwise the oracle and
    the generic k_eval_parity path, FAST within tolerance of PARITY."""
    import os
    from paper_2003_01836_b200 import cli
    s = cli.generate_particles(8000, 29)
    src = s.sources
    cfg = bltc.EvalConfig(theta=0.75, degree=deg, leaf_size=400, batch_size=100)
    ref, _ = oracle.treecode_potentials(src.x, src.y, src.z, src.x, src.y, src.z, s.charges,
                                        True, 0.75, deg, 400, 100, 0, 0.0,
                                        threads=os.cpu_count() or 1)
    phi_p, st = bltc.treecode_potentials(s, cfg, mode="parity")
    np.testing.assert_array_equal(phi_p, ref)
    assert st.packed == 1
    monkeypatch.setenv("BLTC_PARITY_PACKED", "0")
    phi_g, _ = bltc.treecode_potentials(s, cfg, mode="parity")
    monkeypatch.delenv("BLTC_PARITY_PACKED")
    np.testing.assert_array_equal(phi_g, ref)
    phi_f, stf = bltc.treecode_potentials(s, cfg, mode="fast")
    assert stf.packed == 1
    _phi_check(phi_f, ref, 0, exact=False)
