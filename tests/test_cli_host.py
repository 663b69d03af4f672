"""Harness host logic on CPU (test_cli.py of the reference): generation,
error metric, run records in JSON / CSV, particle files, argument parsing."""
import csv
import json

import numpy as np
import pytest

from paper_2003_01836_b200 import cli
from paper_2003_01836_b200.particles import (ParticleSystem, Points, read_particles_csv,
                                             write_particles_csv)


def _random_system(n, seed):
    rng = np.random.default_rng(seed)
    return ParticleSystem.from_single_set(Points.from_array(rng.uniform(-1, 1, (n, 3))),
                                          rng.uniform(-1, 1, n))


def test_generate_particles_deterministic_and_bounded():
    a = cli.generate_particles(500, seed=42)
    b = cli.generate_particles(500, seed=42)
    np.testing.assert_array_equal(a.sources.x, b.sources.x)
    np.testing.assert_array_equal(a.charges, b.charges)
    c = cli.generate_particles(500, seed=43)
    assert not np.array_equal(a.sources.x, c.sources.x)
    for arr in (a.sources.x, a.sources.y, a.sources.z, a.charges):
        assert arr.shape == (500,) and arr.min() >= -1.0 and arr.max() <= 1.0
    assert a.coincident
    assert len(cli.generate_particles(0, seed=1).targets) == 0
    with pytest.raises(ValueError):
        cli.generate_particles(-1, seed=1)


def test_plummer_truncated():
    s = cli.generate_plummer(20_000, 3)
    r = np.sqrt(s.sources.x ** 2 + s.sources.y ** 2 + s.sources.z ** 2)
    assert r.max() <= 10.0 + 1e-12
    # half-mass radius of the truncated Plummer sphere (a = 1) ~ 1.3
    assert 1.1 < np.median(r) < 1.5


def test_relative_error_frozen_cases():
    ds = np.array([3.0, 4.0])
    assert cli.relative_error(ds, ds.copy()) == 0.0
    assert cli.relative_error(ds, 1.1 * ds) == pytest.approx(0.1, rel=1e-12)
    assert cli.relative_error(ds, np.array([3.0, 3.0])) == 0.2
    with pytest.raises(cli.ZeroReference):
        cli.relative_error(np.zeros(4), np.ones(4))
    with pytest.raises(ValueError):
        cli.relative_error(np.ones(4), np.ones(5))


def test_sample_indices_child_stream():
    a = cli.sample_indices(1000, 50, seed=7)
    assert a.shape == (50,) and np.all(np.diff(a) > 0)
    np.testing.assert_array_equal(a, cli.sample_indices(1000, 50, seed=7))
    assert cli.sample_indices(10, 50, seed=7).shape == (10,)


def _record(extras=True):
    return cli.RunRecord(
        n_particles=1000, kernel="yukawa", kappa=0.5, theta=0.7, degree=6, leaf_size=200,
        batch_size=200, ranks=2, seed=9,
        times={"setup_s": 0.125, "precompute_s": 0.25, "compute_s": 0.5, "total_s": 0.875},
        error={"value": 1.5e-7, "sample_size": 100} if extras else None,
        interaction_counts={"direct_pairs": 123, "approx_pairs": 456},
        fetch_stats={"0->1": {"tree_records": 9, "clusters": 4, "moments": 2,
                              "particles": 50}} if extras else None)


def test_records_json_round_trip():
    recs = [_record(), _record(False)]
    back = cli.records_from_json(cli.records_to_json(recs))
    assert [r.to_dict() for r in back] == [r.to_dict() for r in recs]


def test_records_csv_columns(tmp_path):
    path = tmp_path / "out.csv"
    cli.write_records([_record()], str(path), "csv")
    with open(path, newline="") as f:
        rows = list(csv.DictReader(f))
    assert len(rows) == 1
    row = rows[0]
    assert row["theta"] == "0.7"
    assert row["times.total_s"] == "0.875"
    assert float(row["error.value"]) == 1.5e-7
    assert row["interaction_counts.direct_pairs"] == "123"
    assert json.loads(row["fetch_stats"])["0->1"]["particles"] == 50
    with pytest.raises(ValueError):
        cli.write_records([_record()], str(tmp_path / "x"), "yaml")


def test_particles_csv_round_trip(tmp_path):
    s = _random_system(200, 17)
    path = tmp_path / "parts.csv"
    write_particles_csv(str(path), s)
    back = read_particles_csv(str(path))
    for a, b in ((back.sources.x, s.sources.x), (back.sources.y, s.sources.y),
                 (back.sources.z, s.sources.z), (back.charges, s.charges)):
        np.testing.assert_array_equal(a, b)
    assert back.coincident


def test_parser_subcommands():
    p = cli.build_parser()
    a = p.parse_args(["sweep", "--thetas", "0.6,0.9", "--degrees", "2,4"])
    assert a.command == "sweep" and cli._parse_list(a.thetas, float) == [0.6, 0.9]
    a = p.parse_args(["verify", "--n-particles", "10"])
    assert a.verify is None and a.format == "json"
    with pytest.raises(SystemExit):
        p.parse_args([])


def test_full_oracle_refusal_before_device():
    n = cli.FULL_ORACLE_LIMIT + 1
    pts = Points(np.zeros(n), np.zeros(n), np.zeros(n))
    with pytest.raises(cli.OracleTooLarge):
        cli.direct_sum_oracle(ParticleSystem.from_single_set(pts, np.ones(n)),
                              __import__("paper_2003_01836_b200").coulomb())


def test_philox_model_matches_numpy():
    """The Philox4x64-10 model the device generator implements (counter
    incremented before each 4-word block, u >> 11 scaled by 2^-53)
    reproduces numpy's uniform stream from the exported key / counter."""
    from numpy.random import Generator, Philox, SeedSequence
    M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
    W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
    MASK = (1 << 64) - 1

    def block(c, k):
        c, k = list(c), list(k)
        for r in range(10):
            if r:
                k = [(k[0] + W0) & MASK, (k[1] + W1) & MASK]
            p0, p1 = M0 * c[0], M1 * c[2]
            c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & MASK, (p0 >> 64) ^ c[3] ^ k[1], p0 & MASK]
        return c

    child = SeedSequence(12345).spawn(2)[0]
    key, ctr = cli.philox_state(child)
    c = [int(v) for v in ctr]
    words = []
    for _ in range(4):
        c[0] = (c[0] + 1) & MASK
        words += block(c, [int(v) for v in key])
    mine = np.array([-1.0 + 2.0 * ((u >> 11) * (1.0 / 9007199254740992.0)) for u in words[:15]])
    ref = Generator(Philox(child)).uniform(-1.0, 1.0, (5, 3)).ravel()
    np.testing.assert_array_equal(mine, ref)
