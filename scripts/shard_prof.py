"""One term shard of config 5 (rank r of P, dist.term_partition) evaluated twice: for an ncu launch
list of the per-rank kernels (seed, k_tc, fix-up).   python scripts/shard_prof.py [--P 8] [--r 3]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_11571_b200 as pe, synth
from paper_2004_11571_b200.dist import term_partition
P = int(sys.argv[sys.argv.index("--P") + 1]) if "--P" in sys.argv else 8
r = int(sys.argv[sys.argv.index("--r") + 1]) if "--r" in sys.argv else 3
w = synth.gen_config(5)
order, bounds = term_partition(w.exps, P)
mine = np.sort(order[bounds[r]:bounds[r + 1]])
with pe.Context(w.p, w.coeffs[mine], w.exps[mine], w.alpha, n=w.n) as ctx:
    d = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
    for _ in range(3):
        ctx.eval_device(w.j0, w.T, d.data_ptr())
    torch.cuda.synchronize()
    print("ok", ctx.G, ctx.info()["tc_pieces"])
