"""pytest plugin: run the REFERENCE's own test suite with its hot-path entry
points bound to this package.

    python -m pytest -p bltc_b200_substitute baseline/_ref/_tests/test_engine.py ...

(`tools/ref_suite/run.sh` sets PYTHONPATH: the reference package installed in
baseline/_ref by `tools/ref_suite/prepare.sh`, this directory, the repo.)

Before the test modules are imported, every binding of the reference's
entry points inside the ``bltc`` package is replaced by this package's
device implementation, so the reference tests -- and the reference's own
callers of these functions (cli.run_benchmark, decomp internals) -- run on
the B200 path:

  bltc.engine.treecode_potentials        engine.py:350   -> treecode_potentials
  bltc.engine.build_interaction_lists    engine.py:128   -> stages.build_interaction_lists
  bltc.engine.compute_potentials         engine.py:315   -> stages.compute_potentials
  bltc.moments.compute_modified_charges  moments.py:132  -> stages.compute_moments (1 cluster)
  bltc.moments.compute_all_moments       moments.py:147  -> stages.compute_all_moments
  bltc.decomp.run_distributed            decomp.py:483   -> decomp.run_distributed

The oracles the reference tests check against stay the reference's own
(conftest.direct_oracle, moments_reference, cli.direct_sum_oracle), so a
pass is a comparison of the B200 path with the reference's CPU code.  The
evaluation mode is this package's default (STRICT) unless BLTC_MODE is set.
"""
from __future__ import annotations

import os
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SUBSTITUTED: dict = {}


def _degree_of(tree) -> int:
    for c in tree.clusters:
        if getattr(c, "eligible", False):
            return int(c.grids[0].degree)
    return int(tree.clusters[0].grids[0].degree)


def _make_substitutes():
    import bltc.engine as ref_engine
    import bltc.moments as ref_moments

    import paper_2003_01836_b200 as ours
    from paper_2003_01836_b200 import decomp as our_decomp
    from paper_2003_01836_b200 import stages

    def _cfg(degree):
        # moment stages only read the degree (the leaf/batch sizes and the
        # kernel play no part in the upward pass)
        return ours.EvalConfig(theta=0.5, degree=degree, leaf_size=2000, batch_size=2000)

    def treecode_potentials(system, config, threads=1):
        return ours.treecode_potentials(system, config, threads)

    def build_interaction_lists(batch_set, tree, config):
        return stages.build_interaction_lists(batch_set, tree, config)

    def compute_potentials(batch_set, tree, moments, lists, config, threads=1):
        return stages.compute_potentials(batch_set, tree, moments, lists, config, threads)

    def compute_modified_charges(cluster, tree):
        if not cluster.eligible:
            raise ref_moments.IneligibleCluster(
                f"cluster {cluster.index} has a degenerate box extent; "
                "it is evaluated directly, never approximated")
        # the one cluster as a one-node flat tree: a hand-built cluster over
        # a SimpleNamespace(points, charges) needs no SourceTree around it
        f64 = lambda v: np.ascontiguousarray(v, dtype=np.float64)  # noqa: E731
        i64 = lambda v: np.ascontiguousarray(v, dtype=np.int64)    # noqa: E731
        one = stages.FlatTree(start=i64([cluster.start]), stop=i64([cluster.stop]),
                              lo=f64(cluster.box.lo).reshape(1, 3),
                              hi=f64(cluster.box.hi).reshape(1, 3),
                              child_start=i64([0]), child_count=i64([0]),
                              x=f64(tree.points.x), y=f64(tree.points.y), z=f64(tree.points.z),
                              q=f64(tree.charges))
        rows = stages.compute_moments(one, _cfg(int(cluster.grids[0].degree)), [0])
        return ref_moments.ClusterMoments(cluster.index, rows[0].copy())

    def compute_all_moments(tree):
        out = stages.compute_all_moments(tree, _cfg(_degree_of(tree)))
        return [None if m is None else ref_moments.ClusterMoments(m.cluster_index, m.q_hat)
                for m in out]

    def run_distributed(system, config, ranks, threads=1):
        return our_decomp.run_distributed(system, config, ranks, threads)

    return {
        (ref_engine, "treecode_potentials"): treecode_potentials,
        (ref_engine, "build_interaction_lists"): build_interaction_lists,
        (ref_engine, "compute_potentials"): compute_potentials,
        (ref_moments, "compute_modified_charges"): compute_modified_charges,
        (ref_moments, "compute_all_moments"): compute_all_moments,
        ("bltc.decomp", "run_distributed"): run_distributed,
    }


def _patch_everywhere(original, replacement) -> list[str]:
    """Rebind ``original`` to ``replacement`` in every loaded bltc module
    (the reference modules import each other's functions by name)."""
    hits = []
    for name, mod in list(sys.modules.items()):
        if not (name == "bltc" or name.startswith("bltc.")) or not isinstance(mod, types.ModuleType):
            continue
        for attr, val in list(vars(mod).items()):
            if val is original:
                setattr(mod, attr, replacement)
                hits.append(f"{name}.{attr}")
    return hits


def pytest_configure(config):
    import importlib
    for m in ("bltc", "bltc.engine", "bltc.moments", "bltc.decomp", "bltc.cli"):
        importlib.import_module(m)
    for (mod, attr), repl in _make_substitutes().items():
        if isinstance(mod, str):
            mod = sys.modules[mod]
        original = getattr(mod, attr)
        SUBSTITUTED[f"{mod.__name__}.{attr}"] = _patch_everywhere(original, repl)
    config.addinivalue_line("markers", "slow: reference marker")


def pytest_report_header(config):
    from paper_2003_01836_b200 import _lib
    from paper_2003_01836_b200.engine import DEFAULT_MODE
    lines = [f"B200 substitution (mode {DEFAULT_MODE}, libbltc {_lib.LIB_PATH}):"]
    for k, v in SUBSTITUTED.items():
        lines.append(f"  {k} -> paper_2003_01836_b200 ({', '.join(v)})")
    return lines
