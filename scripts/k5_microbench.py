"""K5 microbenchmarks: register-resident pipe rates and the mulmod+add step rate (no memory).
Prints ops / clock / SM (from clock64 cycles) and ops/s (from CUDA events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_11571_b200 as pe

P62 = (1 << 62) - 57
P50 = (1 << 50) - 27
names = {20: "hyb_noacc", 21: "shoup4_noacc", pe.CORE_HYB: "hyb_step", pe.CORE_SHOUP4: "shoup4_step", pe.CORE_SHOUP2: "shoup2_step", pe.CORE_FP64: "fp64_alg2_step",
         10: "IMAD.WIDE.U32", 11: "IMAD", 12: "DFMA", 13: "IMAD.HI.U32", 14: "IADD3"}
res = []
for v in [int(x) for x in sys.argv[1:]] or (10, 11, 13, 14, 12, pe.CORE_HYB, pe.CORE_SHOUP4, pe.CORE_SHOUP2, pe.CORE_FP64):
    for R in (4, 8, 16):
        for threads, blocks in ((256, 148 * 4), (512, 148 * 2)):
            p = P50 if v == pe.CORE_FP64 else P62
            iters = 4096 if v >= 10 else 512
            try:
                ms, steps, cyc = pe.bench_core(v, p, R, blocks, threads, iters)
            except pe.PEError as e:
                print(json.dumps(dict(variant=names[v], R=R, threads=threads, error=str(e))), flush=True)
                continue
            # per-SM rate: each SM runs blocks/148 blocks; cycles measured per block (concurrent)
            per_clk_sm = steps / 148 / cyc if cyc else 0.0
            r = dict(variant=names[v], R=R, threads=threads, blocks=blocks, ms=round(ms, 4),
                     per_s=steps / (ms * 1e-3), per_clk_sm_est=round(per_clk_sm, 3),
                     clk_mhz_est=round(cyc / (ms * 1e3), 1))
            res.append(r)
            print(json.dumps(r), flush=True)
