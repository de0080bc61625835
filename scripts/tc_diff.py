"""Debug: where do the tensor-core path and k_step disagree (rows, chunk, u, v)."""
import os, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2004_11571_b200 as pe
import synth

cfg = int(sys.argv[1]); T = int(sys.argv[2]); t = int(sys.argv[3]) if len(sys.argv) > 3 else None
w = synth.gen_config(cfg, t=t, T=T)
with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
    b = ctx.eval(w.j0, w.T)
with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
    for rep in range(3):
        a = ctx.eval(w.j0, w.T)
        bad = np.argwhere(a != b)
        print("rep", rep, "mismatches", len(bad), "of", a.size, flush=True)
        if len(bad):
            cols = bad[:, 1]
            key = collections.Counter(zip(bad[:, 0].tolist(), (cols // 128).tolist()))
            full = sum(1 for k, c in key.items() if c == 128)
            print("  (row,u) groups", len(key), "entirely wrong", full)
            print("  u", sorted(collections.Counter(((cols % 16384) // 128).tolist()).items())[:12])
            print("  u%32", sorted(collections.Counter(((cols % 16384) // 128 % 32).tolist()).items()))
            print("  rows", collections.Counter(bad[:, 0].tolist()).most_common(6))
