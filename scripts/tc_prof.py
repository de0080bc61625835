"""Profiling driver: config 5 (or --t N terms of its shape) through PE_PATH_TC, 2 evaluations
(the second is the one to capture: ncu -k regex:k_tc -s 1 -c 1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2004_11571_b200 as pe  # noqa: E402
import synth  # noqa: E402

t = int(sys.argv[sys.argv.index("--t") + 1]) if "--t" in sys.argv else None
cfg = int(sys.argv[sys.argv.index("--cfg") + 1]) if "--cfg" in sys.argv else 5
T = int(sys.argv[sys.argv.index("--T") + 1]) if "--T" in sys.argv else None
path = pe.PATH_INT if "--int" in sys.argv else pe.PATH_FAST if "--fast" in sys.argv else pe.PATH_TC
w = synth.gen_config(cfg, t=t, T=T)
with pe.Context.from_workload(w, path=path) as ctx:
    d = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
    for _ in range(2):
        ctx.eval_device(w.j0, w.T, d.data_ptr())
    torch.cuda.synchronize()
print("ok", ctx.G if False else "", flush=True)
