"""Run one K5 microbenchmark variant (for ncu): python scripts/k5_one.py VARIANT R THREADS BLOCKS ITERS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_11571_b200 as pe
v, R, th, bl, it = (int(x) for x in sys.argv[1:6])
p = (1 << 50) - 27 if v == pe.CORE_FP64 else (1 << 62) - 57
ms, steps, cyc = pe.bench_core(v, p, R, bl, th, it)
print(f"variant={v} R={R} {steps / (ms * 1e-3) / 1e12:.3f} T/s  {steps / (ms * 1e-3) / (148 * 1965e6):.2f}/clk/SM")
