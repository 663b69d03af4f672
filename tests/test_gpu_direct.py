"""GPU verification oracle (bltc_direct_sum): PARITY bitwise against the
reference's direct_sum_oracle golden samples; FAST within 1e-13."""
import numpy as np
import pytest
from conftest import golden, golden_system

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2003_01836_b200 as pkg
    c = pkg.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("case", ["c1_coulomb", "small_yukawa", "plummer"])
def test_direct_sum_matches_reference_oracle(ctx, case):
    import paper_2003_01836_b200 as bltc
    g = golden(case)
    s = golden_system(g)
    kernel = [bltc.coulomb(), bltc.yukawa(float(g["kappa"]))][int(g["kind"])]
    ref = g["sample_direct"]
    par = ctx.direct_sum(s, kernel, g["sample"], mode="parity")
    np.testing.assert_array_equal(par, ref)   # Yukawa too: libm exp ported bitwise
    fast = ctx.direct_sum(s, kernel, g["sample"], mode="fast")
    assert np.abs(fast - ref).max() <= 1e-13 * np.abs(ref).max()


def test_direct_sum_full_and_error_metric(ctx):
    """Full direct sum at N=20k; the BLTC error on it equals the reference's
    C1 error (1.44e-5) within 1%."""
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200.cli import relative_error
    g = golden("c1_coulomb")
    s = golden_system(g)
    ds = ctx.direct_sum(s, bltc.coulomb(), None, mode="fast")
    cfg = bltc.EvalConfig(theta=0.7, degree=4)
    phi, _ = bltc.treecode_potentials(s, cfg, mode="fast")
    err = relative_error(ds, phi)
    ref_err = relative_error(ds, g["phi"])
    assert abs(err - ref_err) <= 0.01 * ref_err
    assert abs(ref_err - 1.44e-5) <= 0.01e-5
