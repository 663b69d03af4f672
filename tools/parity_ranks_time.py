"""Time PARITY run_distributed (ranks simulated on one GPU) and the serial
PARITY engine on a Plummer workload -- packed PARITY kernels against
k_eval_parity (BLTC_PARITY_PACKED=0)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_01836_b200 as b  # noqa: E402
from paper_2003_01836_b200 import cli  # noqa: E402
from paper_2003_01836_b200.decomp import run_distributed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 250
s = cli.generate_plummer(n, 3)
cfg = b.EvalConfig(theta=0.8, degree=8, leaf_size=2000, batch_size=nb)
tag = "packed" if os.environ.get("BLTC_PARITY_PACKED", "1") != "0" else "k_eval_parity"
for ranks in (1, 4):
    for _ in range(2):
        t = time.perf_counter()
        if ranks == 1:
            phi, st = b.treecode_potentials(s, cfg, mode="parity")
        else:
            phi, st = run_distributed(s, cfg, ranks=ranks, mode="parity")
        dt = time.perf_counter() - t
    extra = ""
    if ranks == 1:
        extra = f" far {st.far_s:.3f} near {st.near_s:.3f} compute {st.compute_s:.3f}"
    else:
        extra = " per-rank eval " + " ".join(f"{r.eval_s:.3f}" for r in st.rank_timings)
    print(f"{tag} n={n} N_B={nb} ranks={ranks}: {dt:.3f} s{extra} "
          f"sum|phi|={float(np.abs(phi).sum()).hex()}")
