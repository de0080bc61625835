"""Small end-to-end runs for compute-sanitizer (configs 1 and 2-small, every core), checked vs oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, synth
import paper_2004_11571_b200 as pe
cases = [(synth.gen_config(1), {}), (synth.gen_config(2, t=5000, T=70), {"R": 2, "warps": 4, "chunk": 32}),
         (synth.gen_config(4, t=3000, T=40), {}), (synth.gen_config(4, t=3000, T=40), {"path": pe.PATH_INT}),
         (synth.random_small(5, (1 << 63) - 25, 5, 200, 3, 20, 1), {"R": 1})]
for w, kw in cases:
    with pe.Context.from_workload(w, **kw) as ctx:
        out = ctx.eval(w.j0, w.T)
    assert np.array_equal(out, oracle.eval_workload(w)), (w.name, kw)
print("sanitize_run ok", len(cases))
