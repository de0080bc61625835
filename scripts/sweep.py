"""Sweep k_step tuning knobs (R, warps, chunk, core) on one workload; prints one JSON line per point.

    python scripts/sweep.py --config 5 --R 2,4,8,16 --warps 4,8,16 [--core shoup|hyb] [--steps 3]
"""
import argparse
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_11571_b200 as pe  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--R", default="4,8")
ap.add_argument("--warps", default="8")
ap.add_argument("--chunk", default="0")
ap.add_argument("--core", default="shoup")
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--T", type=int, default=0)
ap.add_argument("--p", type=int, default=0, help="override the prime (alpha redrawn in [1, p))")
args = ap.parse_args()
if args.core != "auto":
    os.environ["PE_CORE"] = args.core
w = synth.gen_config(args.config)
if args.p:
    import numpy as np
    w.p = args.p
    w.alpha = synth.uniform_mod(np.random.default_rng(args.p), 1, args.p, w.n - 2)
T = args.T or w.T
out = torch.empty((1024 * 1024 * 64,), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream()
for R, W, ch in itertools.product([int(x) for x in args.R.split(",")], [int(x) for x in args.warps.split(",")],
                                  [int(x) for x in args.chunk.split(",")]):
    try:
        ctx = pe.Context.from_workload(w, R=R, warps=W, chunk=ch, path=args.path)
    except pe.PEError as e:
        print(json.dumps({"R": R, "warps": W, "chunk": ch, "error": str(e)}), flush=True)
        continue
    G = ctx.G
    ctx.eval_device(w.j0, T, out.data_ptr(), T, s.cuda_stream)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    for _ in range(args.steps):
        ctx.eval_device(w.j0, T, out.data_ptr(), T, s.cuda_stream)
    torch.cuda.synchronize()
    st = ctx.kernel_stats()
    info = ctx.info()
    ms = st["step_ms"] / args.steps          # per step (a step may be several passes)
    print(json.dumps({"config": args.config, "core": args.core, "R": R, "warps": W, "chunk": ch,
                      "path": info["path"], "t_padded": info["t_padded"], "n_slots": info["n_slots"],
                      "k_step_ms_per_step": round(ms, 3), "passes": st["step_launches"] // args.steps, "fixup_ms": round(st["fixup_ms"] / args.steps, 3),
                      "Tterm_pt_s": round(w.t * T / (ms * 1e-3) / 1e12, 4)}), flush=True)
    ctx.close()
