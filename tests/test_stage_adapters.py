"""The stage adapters flatten the reference's own objects exactly like the
oracle's flat arrays (host logic; needs the reference package, which exists
only in the build container -- skipped elsewhere)."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    pytest.importorskip("numba")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    import bltc
    from bltc import engine, tree
    return bltc, engine, tree


def test_flatten_reference_objects(ref, oracle):
    from paper_2003_01836_b200 import cli, stages
    bltc, engine, tree = ref
    s = cli.generate_particles(3000, 3)
    src = s.sources
    rt = tree.build_source_tree(bltc.particles.Points(src.x, src.y, src.z), s.charges, 200, 4)
    rb = tree.build_target_batches(bltc.particles.Points(src.x, src.y, src.z), 150)
    cfg = engine.EvalConfig(theta=0.7, degree=4, leaf_size=200, batch_size=150)
    rl = engine.build_interaction_lists(rb, rt, cfg)
    ft, fb, fl = stages.flat_tree(rt), stages.flat_batches(rb), stages.flat_lists(rl)
    ot = oracle.build_source_tree(src.x, src.y, src.z, s.charges, 200)
    ob = oracle.build_target_batches(src.x, src.y, src.z, 150)
    ol = oracle.build_lists(ob, ot, 0.7, 4)
    np.testing.assert_array_equal(ft.start, ot.start)
    np.testing.assert_array_equal(ft.lo, ot.lo)
    has = ot.child_count > 0
    np.testing.assert_array_equal(ft.child_start[has], ot.child_start[has])
    np.testing.assert_array_equal(ft.x, ot.x)
    np.testing.assert_array_equal(ft.q, ot.q)
    np.testing.assert_array_equal(fb.start, ob.start)
    np.testing.assert_array_equal(fb.radius, ob.radius)
    np.testing.assert_array_equal(fb.perm, ob.tree.perm)
    np.testing.assert_array_equal(fl.a_ptr, ol.a_ptr)
    np.testing.assert_array_equal(fl.a_idx, ol.a_idx)
    np.testing.assert_array_equal(fl.d_idx, ol.d_idx)
    assert fl.approx == rl.approx and fl.direct == rl.direct
