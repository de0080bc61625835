"""Per-config numbers for BASELINE.md's "B200 measurements" table: every BASELINE config through the
automatic path and through the scalar k_step (PE_PATH_INT / FP64), device ms per evaluation (CUDA
events, median of --reps after 2 warm-ups), term-points/s, the hot kernel, R and the fraction of the
integer-pipe mulmod roofline (148 SMs x 1965 MHz x 64 IMAD lanes / 14 slots = 1.329e12 products/s);
plus a bitwise comparison of the two paths and of 16 sampled columns against the direct oracle.

    python scripts/config_table.py [--reps 5] > profiles/r02_config_table.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2004_11571_b200 as pe  # noqa: E402
import synth  # noqa: E402

R_INT = 148 * 1965e6 * 64 / 14


def timed(ctx, w, out, reps):
    s = torch.cuda.current_stream()
    for _ in range(2):
        ctx.eval_device(w.j0, w.T, out.data_ptr(), w.T, s.cuda_stream)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.eval_device(w.j0, w.T, out.data_ptr(), w.T, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    for cfg in (1, 2, 3, 4, 5):
        w = synth.gen_config(cfg)
        res = {"config": cfg, "t": w.t, "n": w.n, "T": w.T, "p": w.p}
        outs = {}
        for name, path in (("auto", pe.PATH_AUTO), ("scalar", pe.PATH_FP64 if w.p < (1 << 50) else pe.PATH_INT)):
            with pe.Context.from_workload(w, path=path) as ctx:
                out = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
                ms = timed(ctx, w, out, reps)
                info = ctx.info()
                res[name] = {"ms": ms, "term_points_per_s": w.t * w.T / (ms * 1e-3), "kernel": ctx.eval_kernel(w.T),
                             "scalar_core": info["path"], "R": info["R"], "t_padded": info["t_padded"]}
                if name == "scalar":
                    res[name]["frac_of_R_int"] = w.t * w.T / (ms * 1e-3) / R_INT
                outs[name] = out.cpu().numpy().view(np.uint64)
                res["G"] = ctx.G
        ks = np.unique(np.linspace(0, w.T - 1, 16).astype(np.uint64))
        ref = oracle.eval_workload(w, ks=ks)
        res["bit_exact"] = bool(np.array_equal(outs["auto"], outs["scalar"]) and
                                np.array_equal(outs["auto"][:, ks.astype(np.int64)], ref))
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
