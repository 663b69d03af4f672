"""The reference-suite substitution plugin (tools/ref_suite/) on CPU: with
the unmodified reference installed in baseline/_ref (tools/ref_suite/
prepare.sh), pytest collects the reference's own tests and the plugin
rebinds every hot-path entry point in the loaded bltc modules to this
package.  (Running them needs a B200: tools/ref_suite/run.sh.)"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "_tests")),
                    reason="reference not staged (tools/ref_suite/prepare.sh)")
def test_plugin_collects_and_substitutes():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tools", "ref_suite"), ROOT])
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "bltc_b200_substitute",
                        "-p", "no:cacheprovider", "--collect-only", "-q"],
                       cwd=os.path.join(REF, "_tests"), env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "123 tests collected" in r.stdout
    # the header names every substituted entry point and where it was rebound
    r2 = subprocess.run([sys.executable, "-m", "pytest", "-p", "bltc_b200_substitute",
                         "-p", "no:cacheprovider", "--collect-only"],
                        cwd=os.path.join(REF, "_tests"), env=env, capture_output=True,
                        text=True, timeout=600)
    for name in ("bltc.engine.treecode_potentials", "bltc.engine.compute_potentials",
                 "bltc.engine.build_interaction_lists", "bltc.moments.compute_all_moments",
                 "bltc.moments.compute_modified_charges", "bltc.decomp.run_distributed"):
        assert f"{name} -> paper_2003_01836_b200" in r2.stdout, name
    assert "bltc.cli.treecode_potentials" in r2.stdout   # the reference's own callers too
