import os, sys, socket
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))

def _worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch, torch.distributed as dist
    import paper_2003_01836_b200 as bltc
    from conftest import golden, golden_system
    from paper_2003_01836_b200.decomp import run_distributed, rcb_partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden("dist_r3"); s = golden_system(g)
    cfg = bltc.EvalConfig(theta=float(g["theta"]), degree=int(g["degree"]), leaf_size=int(g["leaf"]), batch_size=int(g["batch"]))
    for ex in ("replicate", "let"):
        phi, st = run_distributed(s, cfg, ranks=world, mode="parity", exchange=ex)
        part = rcb_partition(s.sources, world)
        for o in range(world):
            idx = part.rank_indices(o)
            bad = int((phi[idx] != g["phi"][idx]).sum())
            print(f"proc {rank} exchange {ex}: owner slice {o}: {bad} mismatches", flush=True)
    dist.destroy_process_group()

if __name__ == "__main__":
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0)); port = so.getsockname()[1]
    mp.start_processes(_worker, args=(3, port, "/tmp"), nprocs=3, join=True, start_method="spawn")
