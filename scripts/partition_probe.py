"""Which multi-GPU decomposition for config 5?  Measured on ONE B200: the per-rank
device time of each decomposition's work at P = 1, 2, 4, 8 (every rank's share run on this GPU in
turn, CUDA events, median of `--reps`), plus a modelled gather, give the predicted strong-scaling
curve (the round-end driver has no 8-GPU node).

  term ranges  (dist.TermShardedEval): rank r = ~t/P consecutive terms (bucket order), all T points
  point ranges (dist.ShardedEval):     rank r = all terms, columns [r T/P, (r+1) T/P)

    python scripts/partition_probe.py [--reps 5] > profiles/r02_partition_probe.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_11571_b200 as pe  # noqa: E402
import synth  # noqa: E402
from paper_2004_11571_b200.dist import shard_range, term_partition  # noqa: E402

NVLINK_GBS = 900.0      # NVLink 5 per direction per GPU (guide nominal); the root's ingress bound


def timed(ctx, j0, T, out, reps):
    s = torch.cuda.current_stream()
    for _ in range(2):
        ctx.eval_device(j0, T, out.data_ptr(), out.shape[1], s.cuda_stream)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.eval_device(j0, T, out.data_ptr(), out.shape[1], s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
    w = synth.gen_config(5)
    G, T = 961, w.T
    out_bytes = G * T * 8
    base = None
    with pe.Context.from_workload(w) as full:
        G = full.G
        out = torch.empty((G, T), dtype=torch.int64, device="cuda")
        base = timed(full, w.j0, T, out, reps)
        print(json.dumps({"P": 1, "decomposition": "single", "max_rank_ms": base, "kernel": full.eval_kernel(T)}),
              flush=True)
        for P in (2, 4, 8):
            per = []
            for r in range(P):
                off, cnt = shard_range(T, P, r)
                o = torch.empty((G, cnt), dtype=torch.int64, device="cuda")
                per.append((timed(full, w.j0 + off, cnt, o, reps), full.eval_kernel(cnt)))
            gather = out_bytes * (P - 1) / P / (NVLINK_GBS * 1e9) * 1e3
            mx = max(x for x, _ in per)
            print(json.dumps({"P": P, "decomposition": "point ranges", "rank_ms": [x for x, _ in per],
                              "kernels": [k for _, k in per], "max_rank_ms": mx, "gather_ms_model": gather,
                              "predicted_ms": mx + gather, "predicted_speedup": base / (mx + gather)}), flush=True)
    for P in (2, 4, 8):
        order, bounds = term_partition(w.exps, P)
        per, rows = [], 0
        for r in range(P):
            mine = np.sort(order[bounds[r]:bounds[r + 1]])
            with pe.Context(w.p, w.coeffs[mine], w.exps[mine], w.alpha, n=w.n) as ctx:
                o = torch.empty((ctx.G, T), dtype=torch.int64, device="cuda")
                per.append((timed(ctx, w.j0, T, o, reps), ctx.eval_kernel(T), ctx.G))
                del o
            torch.cuda.empty_cache()
        ingress = sum(g for _, _, g in per[1:]) * T * 8
        gather = ingress / (NVLINK_GBS * 1e9) * 1e3
        mx = max(x for x, _, _ in per)
        print(json.dumps({"P": P, "decomposition": "term ranges", "rank_ms": [x for x, _, _ in per],
                          "kernels": [k for _, k, _ in per], "rows": [g for _, _, g in per], "max_rank_ms": mx,
                          "gather_ms_model": gather, "predicted_ms": mx + gather,
                          "predicted_speedup": base / (mx + gather)}), flush=True)
        # overlapped form (TermShardedEval.run_blocks): each rank evaluates rows [0, s_r) then
        # [s_r, G_r) (pe_row_split); block 0's rows cross NVLink while block 1 is evaluated
        blk = []
        for r in range(P):
            mine = np.sort(order[bounds[r]:bounds[r + 1]])
            with pe.Context(w.p, w.coeffs[mine], w.exps[mine], w.alpha, n=w.n) as ctx:
                sp = ctx.row_split()
                o = torch.empty((ctx.G, T), dtype=torch.int64, device="cuda")
                s_ = torch.cuda.current_stream()
                for _ in range(2):
                    ctx.eval_device_rows(w.j0, T, 0, sp or ctx.G, o.data_ptr(), T, s_.cuda_stream)
                    if sp:
                        ctx.eval_device_rows(w.j0, T, sp, ctx.G, o.data_ptr(), T, s_.cuda_stream)
                t0s, t1s = [], []
                for _ in range(reps):
                    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                    e[0].record(s_)
                    ctx.eval_device_rows(w.j0, T, 0, sp or ctx.G, o.data_ptr(), T, s_.cuda_stream)
                    e[1].record(s_)
                    if sp:
                        ctx.eval_device_rows(w.j0, T, sp, ctx.G, o.data_ptr(), T, s_.cuda_stream)
                    e[2].record(s_)
                    torch.cuda.synchronize()
                    t0s.append(e[0].elapsed_time(e[1]))
                    t1s.append(e[1].elapsed_time(e[2]))
                blk.append((statistics.median(t0s), statistics.median(t1s), sp or ctx.G, ctx.G))
                del o
            torch.cuda.empty_cache()
        in0 = sum(b[2] for b in blk[1:]) * T * 8 / (NVLINK_GBS * 1e9) * 1e3
        in1 = sum(b[3] - b[2] for b in blk[1:]) * T * 8 / (NVLINK_GBS * 1e9) * 1e3
        emax = max(b[0] + b[1] for b in blk)
        e1min = min(b[1] for b in blk)
        pred = emax + max(0.0, in0 - e1min) + in1
        print(json.dumps({"P": P, "decomposition": "term ranges, 2 row blocks (overlapped gather)",
                          "rank_block_ms": [[b[0], b[1]] for b in blk], "splits": [b[2] for b in blk],
                          "max_rank_ms": emax, "gather_block0_ms_model": in0, "gather_block1_ms_model": in1,
                          "predicted_ms": pred, "predicted_speedup": base / pred}), flush=True)


if __name__ == "__main__":
    main()
