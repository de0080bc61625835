"""Automatic-threshold check for p < 2^31 (k_tc 4-digit mode vs k_step 32-bit Shoup): device ms per
evaluation on config-2 / config-3 shapes at p = 2^31 - 1 over T."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2004_11571_b200 as pe, synth


def dev_ms(w, path, T, reps=5):
    with pe.Context.from_workload(w, path=path) as ctx:
        d = torch.empty((ctx.G, T), dtype=torch.int64, device="cuda")
        ctx.eval_device(w.j0, T, d.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ctx.eval_device(w.j0, T, d.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, ctx.info()["t_padded"]


p = (1 << 31) - 1
for cfg in (2, 3):
    w = synth.gen_config(cfg)
    w.p = p
    w.alpha = np.where(w.alpha % p == 0, np.uint64(2), w.alpha).astype(np.uint64)
    for T in (512, 1024, 2048, 4096, 8192):
        a, tp = dev_ms(w, pe.PATH_INT, T)
        b, _ = dev_ms(w, pe.PATH_TC, T)
        print(json.dumps({"config": cfg, "t_padded": tp, "T": T, "int32_ms": round(a, 3), "tc_ms": round(b, 3)}), flush=True)
