"""Development check of the tensor-core path on the GPU: forced PE_PATH_TC against the oracle on
small inputs, then config 5 timing of k_tc vs k_step (CUDA events via pe_kernel_stats).

    python scripts/tc_dev.py [--big]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2004_11571_b200 as pe  # noqa: E402
import synth  # noqa: E402


def run(w, path, j0=None, T=None):
    with pe.Context.from_workload(w, path=path) as ctx:
        return ctx.eval(w.j0 if j0 is None else j0, w.T if T is None else T)


def small():
    cases = [synth.random_small(1, synth.P62, 5, 40, 4, 17),
             synth.random_small(2, synth.P62, 6, 3000, 6, 100),
             synth.random_small(3, 1000003, 4, 500, 5, 33)]
    for i, w in enumerate(cases):
        ref = oracle.eval_workload(w)
        got = run(w, pe.PATH_TC)
        bad = int((got != ref).sum())
        print(json.dumps({"case": i, "t": w.t, "T": w.T, "G": int(ref.shape[0]), "mismatch": bad}), flush=True)
        if bad:
            idx = np.argwhere(got != ref)[:4]
            print("first", idx.tolist(), [int(got[tuple(x)]) for x in idx], [int(ref[tuple(x)]) for x in idx])
    w = synth.gen_config(1)
    ref = oracle.eval_workload(w)
    got = run(w, pe.PATH_TC)
    print(json.dumps({"case": "config1", "mismatch": int((got != ref).sum())}), flush=True)
    w = synth.gen_config(2, T=20000)
    a = run(w, pe.PATH_TC)
    b = run(w, pe.PATH_INT)
    print(json.dumps({"case": "config2 T=20000 tc vs int", "mismatch": int((a != b).sum())}), flush=True)


def big():
    import torch
    w = synth.gen_config(5)
    for path in (pe.PATH_TC, pe.PATH_INT):
        with pe.Context.from_workload(w, path=path) as ctx:
            d = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
            ctx.eval_device(w.j0, w.T, d.data_ptr())
            torch.cuda.synchronize()
            ctx.set_timing(True)
            t0 = time.time()
            for _ in range(3):
                ctx.eval_device(w.j0, w.T, d.data_ptr())
            torch.cuda.synchronize()
            st = ctx.kernel_stats()
            out = d.cpu().numpy().view(np.uint64)
            print(json.dumps({"path": path, "info": ctx.info(), "wall_ms": (time.time() - t0) / 3 * 1e3,
                              "step_ms": st["step_ms"] / 3, "fixup_ms": st["fixup_ms"] / 3,
                              "tp_per_s": w.t * w.T / (st["step_ms"] / 3 * 1e-3)}), flush=True)
            if path == pe.PATH_TC:
                tc_out = out.copy()
            else:
                print(json.dumps({"config5 tc vs int mismatches": int((tc_out != out).sum())}), flush=True)


if __name__ == "__main__":
    small()
    if "--big" in sys.argv:
        big()
