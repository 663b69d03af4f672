import os, sys, socket
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
OUT = os.path.join(ROOT, "gpurun_out", "dbg")

def _worker(rank, world, port):
    sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch, torch.distributed as dist
    import paper_2003_01836_b200 as bltc
    from paper_2003_01836_b200 import decomp
    from conftest import golden, golden_system
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden("dist_r3"); s = golden_system(g)
    cfg = bltc.EvalConfig(theta=float(g["theta"]), degree=int(g["degree"]), leaf_size=int(g["leaf"]), batch_size=int(g["batch"]))
    part = decomp.rcb_partition(s.sources, world)
    eng = decomp.DeviceRankEngine(cfg, "parity")
    idx = part.rank_indices(rank)
    src = s.sources
    eng.build(src.x[idx], src.y[idx], src.z[idx], s.charges[idx])
    pub = eng.publish()
    np.save(f"{OUT}/rec{rank}.npy", pub.records.cpu().numpy()); np.save(f"{OUT}/par{rank}.npy", pub.particles.cpu().numpy()); np.save(f"{OUT}/mom{rank}.npy", pub.moments.cpu().numpy())
    records = decomp.all_gather_records(pub, world)
    flags = eng.needs(world, rank, records)
    for o in range(world):
        np.save(f"{OUT}/flags{rank}_{o}.npy", flags[o].cpu().numpy())
        np.save(f"{OUT}/grec{rank}_{o}.npy", records[o].cpu().numpy())
    forest, fetch = decomp.let_exchange(pub, lambda recs: eng.needs(world, rank, recs), world, rank)
    for o in range(world):
        if o == rank: continue
        np.save(f"{OUT}/frec{rank}_{o}.npy", forest[o].records.cpu().numpy())
        np.save(f"{OUT}/fpar{rank}_{o}.npy", forest[o].particles.cpu().numpy())
        np.save(f"{OUT}/fmom{rank}_{o}.npy", forest[o].moments.cpu().numpy())
    dist.destroy_process_group()

if __name__ == "__main__":
    import torch.multiprocessing as mp
    os.makedirs(OUT, exist_ok=True)
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0)); port = so.getsockname()[1]
    mp.start_processes(_worker, args=(3, port), nprocs=3, join=True, start_method="spawn")
    # check against the local assembly
    import torch
    from paper_2003_01836_b200 import decomp
    pubs = {r: decomp.Published(torch.from_numpy(np.load(f"{OUT}/rec{r}.npy")), torch.from_numpy(np.load(f"{OUT}/par{r}.npy")), torch.from_numpy(np.load(f"{OUT}/mom{r}.npy"))) for r in range(3)}
    for me in range(3):
        for o in range(3):
            gr = np.load(f"{OUT}/grec{me}_{o}.npy")
            print(me, o, "gathered records equal:", np.array_equal(gr, pubs[o].records.numpy()))
        flags = [torch.from_numpy(np.load(f"{OUT}/flags{me}_{o}.npy")) for o in range(3)]
        plan = decomp.let_plan(flags, [pubs[o].records for o in range(3)], me)
        for o in range(3):
            if o == me: continue
            payload = decomp.let_serve(pubs[o], plan.a[o], plan.d[o], plan.npart[o])
            p, _ = decomp.let_assemble(pubs[o].records, plan.a[o], plan.d[o], payload, pubs[o].moments.shape[1], plan.npart[o], plan.nboth[o])
            for k, nm in (("records", "frec"), ("particles", "fpar"), ("moments", "fmom")):
                got = np.load(f"{OUT}/{nm}{me}_{o}.npy")
                exp = getattr(p, k).numpy()
                print(me, o, k, got.shape, exp.shape, "equal:", got.shape == exp.shape and np.array_equal(got, exp))
