"""Distributed host logic on CPU: RCB against the reference, and the full
run_distributed orchestration (exchange, owner order, assembly) with
world-size-2 gloo process groups and an oracle-backed rank engine."""
import os
import socket

import numpy as np
import pytest
from conftest import golden, golden_system

from paper_2003_01836_b200 import cli
from paper_2003_01836_b200.decomp import rcb_partition
from paper_2003_01836_b200.particles import Points


@pytest.mark.parametrize("case", ["dist_r3", "dist_r4_yukawa"])
def test_rcb_matches_reference_order(case):
    g = golden(case)
    s = golden_system(g)
    part = rcb_partition(s.sources, int(g["ranks"]))
    np.testing.assert_array_equal(part.order, g["order"])
    np.testing.assert_array_equal(part.rank_start, g["rank_start"])


def test_rcb_reference_cases():
    # test_decomp.py:27-103 of the reference
    corners = np.array([[sx, sy, sz] for sx in (-0.5, 0.5) for sy in (-0.5, 0.5)
                        for sz in (-0.5, 0.5)])
    part = rcb_partition(Points.from_array(corners), 2)
    np.testing.assert_array_equal(part.counts, [4, 4])
    for r in (0, 1):
        assert len(set(corners[part.rank_indices(r), 0])) == 1
    rng = np.random.default_rng(57)
    part = rcb_partition(Points.from_array(rng.uniform(-1, 1, (100_000, 3))), 6)
    assert set(part.counts.tolist()) == {16666, 16667}
    rng = np.random.default_rng(59)
    for n, ranks in ((1003, 7), (97, 13), (64, 64), (100, 3)):
        part = rcb_partition(Points.from_array(rng.uniform(-1, 1, (n, 3))), ranks)
        assert part.counts.sum() == n and part.counts.max() - part.counts.min() <= 1
        assert np.array_equal(np.sort(part.order), np.arange(n))
    with pytest.raises(ValueError):
        rcb_partition(Points.from_array(rng.uniform(-1, 1, (3, 3))), 4)
    with pytest.raises(ValueError):
        rcb_partition(Points.from_array(rng.uniform(-1, 1, (3, 3))), 0)


def test_run_distributed_requires_coincident():
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200.decomp import run_distributed
    rng = np.random.default_rng(97)
    t = Points.from_array(rng.uniform(-1, 1, (100, 3)))
    s = Points.from_array(rng.uniform(-1, 1, (100, 3)))
    system = bltc.ParticleSystem(targets=t, sources=s, charges=rng.uniform(-1, 1, 100))
    with pytest.raises(ValueError):
        run_distributed(system, bltc.EvalConfig(theta=0.7, degree=3), ranks=2)


def test_run_distributed_native_validates_before_the_device():
    """The one-call C path raises the reference's ValueErrors (decomp.py:
    85-88, 493-495) before touching a GPU."""
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200.decomp import run_distributed_native
    rng = np.random.default_rng(98)
    t = Points.from_array(rng.uniform(-1, 1, (50, 3)))
    s = Points.from_array(rng.uniform(-1, 1, (50, 3)))
    cfg = bltc.EvalConfig(theta=0.7, degree=3)
    with pytest.raises(ValueError):
        run_distributed_native(bltc.ParticleSystem(targets=t, sources=s,
                                                   charges=rng.uniform(-1, 1, 50)), cfg, 2,
                               devices=[0])
    same = bltc.ParticleSystem.from_single_set(s, rng.uniform(-1, 1, 50))
    with pytest.raises(ValueError):
        run_distributed_native(same, cfg, 0, devices=[0])
    with pytest.raises(ValueError):
        run_distributed_native(same, cfg, 51, devices=[0])   # fewer particles than ranks


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir, exchange="replicate"):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import paper_2003_01836_b200 as bltc
    from conftest import golden, golden_system
    from paper_2003_01836_b200.decomp import run_distributed
    from rank_engine_oracle import OracleRankEngine
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden(case)
    s = golden_system(g)
    kernel = [bltc.coulomb(), bltc.yukawa(float(g["kappa"]))][int(g["kind"])]
    cfg = bltc.EvalConfig(theta=float(g["theta"]), degree=int(g["degree"]),
                          leaf_size=int(g["leaf"]), batch_size=int(g["batch"]), kernel=kernel)
    phi, st = run_distributed(s, cfg, ranks=world, engine_factory=lambda: OracleRankEngine(cfg),
                              exchange=exchange)
    np.save(os.path.join(out_dir, f"phi{rank}.npy"), phi)
    fetch = [[o, w, f.tree_records, f.clusters, f.moments, f.particles]
             for (o, w), f in sorted(st.fetch_stats.items())]
    np.save(os.path.join(out_dir, f"fetch{rank}.npy"), np.array(fetch, dtype=np.int64))
    np.save(os.path.join(out_dir, f"pairs{rank}.npy"), np.array([st.direct_pairs,
                                                                 st.approx_pairs]))
    dist.destroy_process_group()


def test_gloo_world2_orchestration_matches_oracle(tmp_path, oracle):
    """Two processes, gloo all-gather of the published buffers: the assembled
    potentials equal the reference's run_distributed bitwise."""
    import torch.multiprocessing as mp
    case = "dist_r3"
    g = golden(case)
    s = golden_system(g)
    src = s.sources
    ref, info = oracle.run_distributed(src.x, src.y, src.z, s.charges, 2, float(g["theta"]),
                                       int(g["degree"]), int(g["leaf"]), int(g["batch"]),
                                       int(g["kind"]), float(g["kappa"]))
    mp.start_processes(_worker, args=(2, _free_port(), case, str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    for r in range(2):
        np.testing.assert_array_equal(np.load(tmp_path / f"phi{r}.npy"), ref)
        pairs = np.load(tmp_path / f"pairs{r}.npy")
        assert (int(pairs[0]), int(pairs[1])) == (info["direct_pairs"], info["approx_pairs"])


def test_single_process_orchestration_matches_oracle(oracle):
    """ranks=4 simulated in one process (the no-process-group path)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200.decomp import run_distributed
    from rank_engine_oracle import OracleRankEngine
    g = golden("dist_r4_yukawa")
    s = golden_system(g)
    cfg = bltc.EvalConfig(theta=0.7, degree=6, leaf_size=300, batch_size=300,
                          kernel=bltc.yukawa(0.5))
    phi, st = run_distributed(s, cfg, ranks=4, engine_factory=lambda: OracleRankEngine(cfg))
    np.testing.assert_array_equal(phi, g["phi"])
    assert st.direct_pairs == int(g["direct_pairs"])
    assert st.approx_pairs == int(g["approx_pairs"])
    assert sorted(st.rank_counts.tolist()) == [2000] * 4
    assert set(st.fetch_stats) == {(o, w) for o in range(4) for w in range(4) if o != w}


def test_gloo_world3_let_exchange_matches_reference(tmp_path):
    """Three processes, the two-step LET exchange (records all-gather, need
    flags, all-to-all of ids and of exactly the referenced moment rows and
    particle slices): potentials bitwise the reference's run_distributed and
    the fetch volume per (origin, owner) equal to the reference's LET."""
    import torch.multiprocessing as mp
    case = "dist_r3"
    g = golden(case)
    mp.start_processes(_worker, args=(3, _free_port(), case, str(tmp_path), "let"), nprocs=3,
                       join=True, start_method="spawn")
    for r in range(3):
        np.testing.assert_array_equal(np.load(tmp_path / f"phi{r}.npy"), g["phi"])
        mine = np.load(tmp_path / f"fetch{r}.npy")
        np.testing.assert_array_equal(mine, g["fetch"][g["fetch"][:, 0] == r])


def test_single_process_let_matches_reference_fetch():
    """ranks=4 in one process with the LET exchange: potentials bitwise, fetch
    statistics equal to the reference's, no sufficiency/minimality violation."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200.decomp import let_local, let_violations, run_distributed
    from rank_engine_oracle import OracleRankEngine
    g = golden("dist_r4_yukawa")
    s = golden_system(g)
    cfg = bltc.EvalConfig(theta=0.7, degree=6, leaf_size=300, batch_size=300,
                          kernel=bltc.yukawa(0.5))
    phi, st = run_distributed(s, cfg, ranks=4, engine_factory=lambda: OracleRankEngine(cfg),
                              exchange="let")
    np.testing.assert_array_equal(phi, g["phi"])
    fetch = np.array([[o, w, f.tree_records, f.clusters, f.moments, f.particles]
                      for (o, w), f in sorted(st.fetch_stats.items())], dtype=np.int64)
    np.testing.assert_array_equal(fetch, g["fetch"])
    # violations of one origin's fetched forest
    part = rcb_partition(s.sources, 4)
    engines = {}
    for r in range(4):
        idx = part.rank_indices(r)
        engines[r] = OracleRankEngine(cfg)
        src = s.sources
        engines[r].build(src.x[idx], src.y[idx], src.z[idx], s.charges[idx])
    pubs = {r: engines[r].publish() for r in range(4)}
    needs = {r: (lambda recs, r=r: engines[r].needs(4, r, recs)) for r in range(4)}
    forests, _ = let_local(pubs, needs, 4)
    recs = [pubs[r].records for r in range(4)]
    for me in range(4):
        v = let_violations(forests[me], engines[me].needs(4, me, recs), me)
        assert v == {"sufficiency": 0, "minimality": 0}


def test_device_rcb_flags_ties_at_a_cut():
    """DeviceRcb (torch, here on CPU tensors) takes the reference's cuts with
    order-statistic selection; when particles share the coordinate at a cut's order
    statistic it flags ``tied`` (run_distributed then uses the reference's
    own rcb_partition), and on continuous data it reproduces the reference's
    rank SETS exactly."""
    import torch
    from paper_2003_01836_b200.decomp import DeviceRcb
    g = np.arange(9, dtype=np.float64)   # 729 points: the first cut (364) falls in a tie
    lattice = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    d = DeviceRcb(*(torch.from_numpy(np.ascontiguousarray(lattice[:, k])) for k in range(3)), 4)
    assert d.tied
    s = cli.generate_particles(5000, 3).sources
    d = DeviceRcb(*(torch.from_numpy(np.asarray(v)) for v in (s.x, s.y, s.z)), 4)
    assert not d.tied
    ref = rcb_partition(s, 4)
    for r in range(4):
        mine = np.sort(d.rank_indices(r).numpy())
        np.testing.assert_array_equal(mine, np.sort(np.asarray(ref.rank_indices(r))))


def _packed_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2003_01836_b200.decomp import (RECORD_DOUBLES, Published, all_gather_published,
                                              all_gather_sizes, packed_doubles,
                                              unpack_published)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ncols = 10

    def make(r):   # ragged sizes, rank 1 without moment rows
        nc, n, nrow = 3 + 2 * r, 5 + 7 * r, (0 if r == 1 else 2 + r)
        g = torch.Generator().manual_seed(r)
        return Published(torch.rand(nc, RECORD_DOUBLES, generator=g, dtype=torch.float64),
                         torch.rand(4, n, generator=g, dtype=torch.float64),
                         torch.rand(nrow, ncols, generator=g, dtype=torch.float64))

    mine = make(rank)
    # the staged path (pub given as three tensors) ...
    forest = all_gather_published(mine, world)
    # ... and the zero-copy path (pub already a view of a packed block)
    sizes = all_gather_sizes(mine.sizes, world)
    cap = max(packed_doubles(s, ncols) for s in sizes)
    block = torch.zeros(cap, dtype=torch.float64)
    view = unpack_published(block, mine.sizes, ncols)
    view.records.copy_(mine.records)
    view.particles.copy_(mine.particles)
    view.moments.copy_(mine.moments)
    view.block = block
    forest2 = all_gather_published(view, world, all_sizes=sizes)
    ok = True
    for r in range(world):
        want = make(r)
        for f in (forest[r], forest2[r]):
            ok &= f.sizes == want.sizes
            ok &= bool(torch.equal(f.records, want.records) and
                       torch.equal(f.particles, want.particles) and
                       torch.equal(f.moments, want.moments))
    np.save(os.path.join(out_dir, f"ok{rank}.npy"), np.array([ok]))
    dist.destroy_process_group()


def test_gloo_world3_packed_all_gather(tmp_path):
    """The single packed all-gather of {records, particles, moment rows}
    (north_star's one exchange): ragged per-rank sizes, a rank without
    moment rows, staged and zero-copy publication -- every rank receives
    every block exactly."""
    import torch.multiprocessing as mp
    mp.start_processes(_packed_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3,
                       join=True, start_method="spawn")
    for r in range(3):
        assert bool(np.load(tmp_path / f"ok{r}.npy")[0])


def test_domain_boxes_cover_the_points():
    """bltc_domain_cells (host): minimal boxes of the occupied cells of a
    grid over the points' bounding box -- every point lies in one of them,
    each is inside the bounding box, at most grid^3 of them; a Plummer
    sphere leaves the bounding box's corners uncovered (what lets a rank skip
    its top clusters' moment rows)."""
    from paper_2003_01836_b200 import cli, decomp
    s = cli.generate_plummer(20000, 3)
    x, y, z = (np.asarray(a) for a in (s.sources.x, s.sources.y, s.sources.z))
    for grid in (1, 4, 16):
        b = decomp.domain_boxes(x, y, z, grid)
        assert 1 <= len(b) <= grid ** 3
        assert (b[:, :3] <= b[:, 3:]).all()
        P = np.stack([x, y, z], 1)
        lo, hi = P.min(0), P.max(0)
        assert (b[:, :3] >= lo).all() and (b[:, 3:] <= hi).all()
        inside = np.zeros(len(x), dtype=bool)
        for bb in b:
            inside |= ((P >= bb[:3]) & (P <= bb[3:])).all(1)
        assert inside.all()
        if grid == 1:
            np.testing.assert_array_equal(b[0], np.concatenate([lo, hi]))
    corner = hi
    b = decomp.domain_boxes(x, y, z, 16)
    assert not ((corner >= b[:, :3]) & (corner <= b[:, 3:])).all(1).any()
    # the degenerate case: identical points, one box of zero extent
    b = decomp.domain_boxes(np.ones(5), np.ones(5), np.ones(5), 8)
    np.testing.assert_array_equal(b, [[1, 1, 1, 1, 1, 1]])
    with pytest.raises(ValueError, match="finite"):
        decomp.domain_boxes(np.array([np.nan]), np.zeros(1), np.zeros(1))
