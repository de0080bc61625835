"""Config-5 shape (t = 10^7, T = 16384) with p = 2^31 - 1: k_tc (4-digit mode) vs k_step's 32-bit
Shoup path, device ms per evaluation (CUDA events around pe_eval_device), and equality."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2004_11571_b200 as pe, synth

w = synth.gen_config(5)
p = (1 << 31) - 1
w.p = p
w.alpha = np.where(w.alpha % p == 0, np.uint64(2), w.alpha).astype(np.uint64)
res = {}
outs = {}
for name, path in (("tc", pe.PATH_AUTO), ("int32", pe.PATH_INT)):
    with pe.Context.from_workload(w, path=path) as ctx:
        d = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
        ctx.eval_device(w.j0, w.T, d.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            ctx.eval_device(w.j0, w.T, d.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        res[name] = {"ms": e0.elapsed_time(e1) / 3, "uses_tc": ctx.uses_tc(w.T), "info": ctx.info()["path"]}
        outs[name] = d.cpu().numpy()
res["equal"] = bool(np.array_equal(outs["tc"], outs["int32"]))
res["tc_term_points_per_s"] = w.t * w.T / (res["tc"]["ms"] * 1e-3)
print(json.dumps(res))
