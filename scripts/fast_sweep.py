"""Crossover of the fast product-tree method (PE_PATH_FAST, csrc/fast.cu) against the tensor-core
matrix method (PE_PATH_TC, csrc/tc.cuh) over T: device ms per evaluation
(CUDA events, median of --reps) on config-3 terms (10^6 terms, 256 buckets) and config-5 terms
(10^7 terms, 961 Zipf buckets), plus a bitwise equality check of the two outputs at each point.

    python scripts/fast_sweep.py [--reps 3] [--cfg 3,5] > profiles/r02_fast_sweep.jsonl
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2004_11571_b200 as pe  # noqa: E402
import synth  # noqa: E402


def timed(ctx, j0, T, out, reps):
    s = torch.cuda.current_stream()
    ctx.eval_device(j0, T, out.data_ptr(), T, s.cuda_stream)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.eval_device(j0, T, out.data_ptr(), T, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
    only_tc = "--only-tc" in sys.argv
    with_step = "--with-step" in sys.argv      # also the scalar matrix method (k_step, PE_PATH_INT)
    step_max = int(sys.argv[sys.argv.index("--step-max") + 1]) if "--step-max" in sys.argv else 65536
    Tsel = [int(x) for x in sys.argv[sys.argv.index("--T") + 1].split(",")] if "--T" in sys.argv else None
    cfgs = [int(x) for x in (sys.argv[sys.argv.index("--cfg") + 1] if "--cfg" in sys.argv else "3,5").split(",")]
    Ts = {3: [512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072, 262144],
          5: [4096, 16384, 32768, 65536]}
    for cfg in cfgs:
        w = synth.gen_config(cfg)
        st = pe.Context.from_workload(w, path=pe.PATH_INT) if with_step else None
        with pe.Context.from_workload(w, path=pe.PATH_TC) as tc, pe.Context.from_workload(w, path=pe.PATH_FAST) as fa:
            G = tc.G
            for T in (Tsel or Ts[cfg]):
                a = torch.empty((G, T), dtype=torch.int64, device="cuda")
                b = torch.empty_like(a)
                t_tc = timed(tc, w.j0, T, a, reps)
                t_fa = float("nan") if only_tc else timed(fa, w.j0, T, b, reps)
                same = None if only_tc else bool(torch.equal(a, b))
                t_st = None
                if st is not None and T <= step_max:
                    t_st = timed(st, w.j0, T, b, max(1, reps // 2))
                    same = same and bool(torch.equal(a, b))
                print(json.dumps({"workload": w.name, "t": w.t, "G": G, "T": T, "k_tc_ms": t_tc, "fast_ms": t_fa,
                                  "fast_over_tc": t_fa / t_tc, "bitwise_equal": same, "k_step_ms": t_st,
                                  "fast_over_step": (t_fa / t_st) if t_st else None,
                                  "k_tc_term_points_per_s": w.t * T / (t_tc * 1e-3),
                                  "fast_term_points_per_s": w.t * T / (t_fa * 1e-3)}), flush=True)
                del a, b
                torch.cuda.empty_cache()
        if st is not None:
            st.close()


if __name__ == "__main__":
    main()
