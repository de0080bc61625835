"""k_tc (forced; the V = 32 geometry of p >= 2^54, automatic swapped form) vs the scalar k_step
(PE_PATH_INT) over T, for config-2/3 shapes at three term counts: device ms per evaluation (CUDA
events around pe_eval_device, mean of 5 after a warm-up) -- sets tc_min_T for p >= 2^54.

    python scripts/tc_threshold_v32.py > profiles/r02_tc_threshold_v32.jsonl
    python scripts/tc_threshold_v32.py --p50 > profiles/r02_tc_threshold_v32_p50.jsonl   (7 digits vs FP64 Alg. 2)
    python scripts/tc_threshold_v32.py --p31 > profiles/r02_tc_threshold_p31_shoup32.jsonl (4 digits vs 32-bit k_step)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_11571_b200 as pe  # noqa: E402
import synth  # noqa: E402


def dev_ms(ctx, w, T, reps=5):
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


P50 = (1 << 50) - 27
seven = "--p50" in sys.argv     # the 7-digit mode (2^31 <= p < 2^54) against the FP64 Alg. 2 k_step
four = "--p31" in sys.argv      # the 4-digit mode (p = 2^31 - 1) against the 32-bit Shoup k_step
P31 = (1 << 31) - 1
for cfg, t in ((2, 10_000), (2, 100_000), (3, 300_000), (3, 1_000_000)):
    w = synth.gen_config(cfg, t=t)
    if seven:
        w.p = P50
        w.coeffs %= np.uint64(P50)
        w.alpha = (w.alpha % np.uint64(P50 - 1)) + np.uint64(1)
    if four:
        w.p = P31
        w.alpha = (w.alpha % np.uint64(P31 - 1)) + np.uint64(1)
    scalar = pe.PATH_FP64 if seven else pe.PATH_INT
    with pe.Context.from_workload(w, path=scalar) as ci, pe.Context.from_workload(w, path=pe.PATH_TC) as ct:
        for T in ((128, 256, 384, 512, 768, 1024, 1536, 2048) if four else (32, 64, 128, 192, 256, 384, 512, 768, 1024)):
            a, b = dev_ms(ci, w, T), dev_ms(ct, w, T)
            print(json.dumps({"cfg": cfg, "t": t, "t_pad": ct.info()["t_padded"], "min_T_now": ct.info()["tc_min_T"],
                              "T": T, "k_step_ms": a, "k_tc_ms": b, "tc_faster": b < a}), flush=True)
