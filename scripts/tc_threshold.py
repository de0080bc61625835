"""k_tc (forced) vs k_step on configs 2-4 and T sweeps: device ms per evaluation (CUDA events
around pe_eval_device), to set the automatic tensor-core threshold."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2004_11571_b200 as pe
import synth


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
        return e0.elapsed_time(e1) / reps


for cfg, Ts in ((2, (256, 512, 1000, 2048, 4096)), (3, (256, 512, 1024, 2048, 4096)), (4, (1024, 2048, 4096))):
    w = synth.gen_config(cfg)
    base = pe.PATH_AUTO if cfg == 4 else pe.PATH_INT
    for T in Ts:
        a = dev_ms(w, base, T)
        b = dev_ms(w, pe.PATH_TC, T)
        print(json.dumps({"config": cfg, "t": w.t, "T": T, "scalar_ms": round(a, 3), "tc_ms": round(b, 3),
                          "scalar_path": "fp64" if cfg == 4 else "int"}), flush=True)
