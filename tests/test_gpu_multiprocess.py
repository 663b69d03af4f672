"""The one-process-per-rank device path with real process groups: ranks are
separate processes (torch.distributed, gloo -- several ranks share the one
GPU available here, NCCL refuses duplicate devices), each running libbltc's
rank pipeline, the two-step LET exchange and the result gather.  Potentials
and fetch volumes equal the reference's run_distributed (golden vectors)."""
import os
import socket

import numpy as np
import pytest
from conftest import golden, golden_system

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_dir, backend="gloo"):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    import torch
    import torch.distributed as dist

    import paper_2003_01836_b200 as bltc
    from conftest import golden, golden_system
    from paper_2003_01836_b200.decomp import DeviceRankRunner, run_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank % torch.cuda.device_count() if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden(case)
    s = golden_system(g)
    kernel = [bltc.coulomb(), bltc.yukawa(float(g["kappa"]))][int(g["kind"])]
    cfg = bltc.EvalConfig(theta=float(g["theta"]), degree=int(g["degree"]),
                          leaf_size=int(g["leaf"]), batch_size=int(g["batch"]), kernel=kernel)
    for exchange in ("let", "replicate"):
        phi, st = run_distributed(s, cfg, ranks=world, mode="parity", exchange=exchange)
        np.save(os.path.join(out_dir, f"phi_{exchange}{rank}.npy"), phi)
        fetch = [[o, w, f.tree_records, f.clusters, f.moments, f.particles]
                 for (o, w), f in sorted(st.fetch_stats.items())]
        np.save(os.path.join(out_dir, f"fetch_{exchange}{rank}.npy"),
                np.array(fetch, dtype=np.int64))
        np.save(os.path.join(out_dir, f"pairs_{exchange}{rank}.npy"),
                np.array([st.direct_pairs, st.approx_pairs]))
    # the benchmark's per-rank runner (device-resident inputs), PARITY
    ctx = bltc.Context(dev, torch.cuda.current_stream(dev).cuda_stream)
    for exchange in ("replicate", "let"):
        runner = DeviceRankRunner(ctx, s, cfg, mode="parity", exchange=exchange)
        runner.step()
        runner.step()   # reused buffers / context
        np.save(os.path.join(out_dir, f"runner_{exchange}{rank}.npy"), runner.phi.cpu().numpy())
    ctx.close()
    dist.destroy_process_group()


def _n_gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("backend", ["gloo", "nccl"])
@pytest.mark.parametrize("case", ["dist_r3", "dist_r4_yukawa"])
def test_process_group_ranks_match_reference(tmp_path, case, backend):
    """gloo: every rank on the one GPU; nccl: one rank per GPU over NVLink
    (the bench's N > 1 path: the single packed all-gather, and the LET) --
    needs as many GPUs as ranks."""
    import torch.multiprocessing as mp
    from paper_2003_01836_b200.decomp import rcb_partition
    g = golden(case)
    R = int(g["ranks"])
    if backend == "nccl" and _n_gpus() < R:
        pytest.skip(f"NCCL ranks need {R} GPUs, {_n_gpus()} visible")
    mp.start_processes(_worker, args=(R, _free_port(), case, str(tmp_path), backend), nprocs=R,
                       join=True, start_method="spawn")
    part = rcb_partition(golden_system(g).sources, R)
    for r in range(R):
        for ex in ("let", "replicate"):
            phi = np.load(tmp_path / f"phi_{ex}{r}.npy")
            np.testing.assert_array_equal(phi, g["phi"])
            pairs = np.load(tmp_path / f"pairs_{ex}{r}.npy")
            assert (int(pairs[0]), int(pairs[1])) == (int(g["direct_pairs"]),
                                                      int(g["approx_pairs"]))
        mine = np.load(tmp_path / f"fetch_let{r}.npy")
        np.testing.assert_array_equal(mine, g["fetch"][g["fetch"][:, 0] == r])
        # the runner's rank slice equals the assembled result on its targets
        for ex in ("replicate", "let"):
            run = np.load(tmp_path / f"runner_{ex}{r}.npy")
            np.testing.assert_array_equal(run, np.load(tmp_path / f"phi_let{r}.npy")[
                part.rank_indices(r)])
