"""Harness on the GPU path (test_cli.py of the reference): the device oracle,
run_benchmark (single, sweep sharing one oracle, distributed) and the CLI."""
import csv
import io

import numpy as np
import pytest

from paper_2003_01836_b200 import EvalConfig, cli, coulomb, yukawa
from paper_2003_01836_b200.particles import ParticleSystem, Points, write_particles_csv

pytestmark = pytest.mark.gpu


def _random_system(n, seed):
    rng = np.random.default_rng(seed)
    return ParticleSystem.from_single_set(Points.from_array(rng.uniform(-1, 1, (n, 3))),
                                          rng.uniform(-1, 1, n))


def test_oracle_two_particles_by_hand():
    pts = Points.from_array(np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 0.0]]))
    s = ParticleSystem.from_single_set(pts, np.array([3.0, 5.0]))
    np.testing.assert_array_equal(cli.direct_sum_oracle(s, coulomb()), [2.5, 1.5])
    f = np.exp(-1.0) / 2.0
    np.testing.assert_allclose(cli.direct_sum_oracle(s, yukawa(0.5)), [5.0 * f, 3.0 * f],
                               rtol=1e-15)


def test_oracle_sampling_is_a_restriction():
    s = _random_system(400, 13)
    full = cli.direct_sum_oracle(s, coulomb())
    sample = np.array([0, 17, 211, 399], dtype=np.int64)
    np.testing.assert_array_equal(cli.direct_sum_oracle(s, coulomb(), sample), full[sample])


def test_oracle_all_coincident_sample():
    n = 5000
    pts = Points(np.zeros(n), np.zeros(n), np.zeros(n))
    s = ParticleSystem.from_single_set(pts, np.ones(n))
    phi = cli.direct_sum_oracle(s, coulomb(), sample_indices=np.arange(3, dtype=np.int64))
    np.testing.assert_array_equal(phi, np.zeros(3))


def test_run_benchmark_single_run_with_verification():
    s = cli.generate_particles(3000, seed=5)
    cfg = EvalConfig(theta=0.7, degree=7, leaf_size=100, batch_size=100)
    recs = cli.run_benchmark(s, cfg, seed=5, verify=500)
    assert len(recs) == 1
    r = recs[0]
    assert r.error["sample_size"] == 500 and r.error["value"] <= 1e-5
    assert r.fetch_stats is None
    assert r.interaction_counts["direct_pairs"] > 0 and r.times["total_s"] > 0


def test_run_benchmark_sweep_shares_one_oracle():
    s = cli.generate_particles(3000, seed=6)
    cfg = EvalConfig(theta=0.5, degree=1, leaf_size=100, batch_size=100)
    thetas, degrees = [0.5, 0.7, 0.9], [1, 3, 5, 7, 9, 11, 13]
    recs = cli.run_benchmark(s, cfg, seed=6, verify=400, sweep=(thetas, degrees))
    assert [(r.theta, r.degree) for r in recs] == [(t, d) for t in thetas for d in degrees]
    for th in thetas:
        errs = [r.error["value"] for r in recs if r.theta == th]
        for lo, hi in zip(errs[1:], errs[:-1]):
            assert lo <= 2.0 * hi
        assert errs[-1] <= 1e-9


def test_run_benchmark_distributed_records_fetch_stats():
    s = cli.generate_particles(2000, seed=7)
    cfg = EvalConfig(theta=0.7, degree=4, leaf_size=100, batch_size=100)
    r = cli.run_benchmark(s, cfg, seed=7, ranks=2, verify=200)[0]
    assert set(r.fetch_stats) == {"0->1", "1->0"}
    for fs in r.fetch_stats.values():
        assert set(fs) == {"tree_records", "clusters", "moments", "particles"}
    assert r.error["value"] <= 1e-4


def test_main_run_verify_and_sweep(tmp_path, capsys):
    out = tmp_path / "run.json"
    assert cli.main(["run", "--n-particles", "2000", "--seed", "3", "--theta", "0.7",
                     "--degree", "5", "--leaf-size", "100", "--batch-size", "100",
                     "--verify", "300", "--output", str(out)]) == 0
    recs = cli.records_from_json(out.read_text())
    assert recs[0].n_particles == 2000 and recs[0].error["sample_size"] == 300
    out = tmp_path / "verify.json"
    assert cli.main(["verify", "--n-particles", "1500", "--seed", "4", "--theta", "0.7",
                     "--degree", "6", "--leaf-size", "100", "--batch-size", "100",
                     "--output", str(out)]) == 0
    r = cli.records_from_json(out.read_text())[0]
    assert r.error["sample_size"] == 1500 and r.error["value"] <= 1e-4
    assert cli.main(["run", "--n-particles", "800", "--seed", "5", "--theta", "0.8",
                     "--degree", "3", "--leaf-size", "100", "--batch-size", "100",
                     "--format", "csv"]) == 0
    rows = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    assert rows[0]["n_particles"] == "800" and rows[0]["error.value"] == ""
    out = tmp_path / "sweep.csv"
    assert cli.main(["sweep", "--n-particles", "1200", "--seed", "9", "--thetas", "0.6,0.9",
                     "--degrees", "2,4", "--leaf-size", "100", "--batch-size", "100",
                     "--format", "csv", "--output", str(out)]) == 0
    with open(out, newline="") as f:
        rows = list(csv.DictReader(f))
    assert [(r["theta"], r["degree"]) for r in rows] == \
        [("0.6", "2"), ("0.6", "4"), ("0.9", "2"), ("0.9", "4")]


def test_main_particle_file_and_distributed(tmp_path):
    s = _random_system(600, 23)
    path = tmp_path / "parts.csv"
    write_particles_csv(str(path), s)
    out = tmp_path / "run.json"
    assert cli.main(["run", "--particles", str(path), "--theta", "0.7", "--degree", "4",
                     "--leaf-size", "100", "--batch-size", "100", "--verify", "600",
                     "--output", str(out)]) == 0
    r = cli.records_from_json(out.read_text())[0]
    assert r.n_particles == 600 and r.error["value"] <= 1e-4
    out = tmp_path / "dist.json"
    assert cli.main(["run", "--n-particles", "2000", "--seed", "8", "--ranks", "2",
                     "--theta", "0.7", "--degree", "4", "--leaf-size", "100",
                     "--batch-size", "100", "--output", str(out)]) == 0
    r = cli.records_from_json(out.read_text())[0]
    assert r.ranks == 2 and set(r.fetch_stats) == {"0->1", "1->0"}
