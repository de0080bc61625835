"""A/B of k_tc runtime knobs on config 5 (interleaved rounds so power-cap drift hits every variant
alike): median device ms per evaluation (CUDA events) for each env setting.

    python scripts/ktc_ab.py [--rounds 5] [--n 10] VAR=VAL[;VAR=VAL] ...
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


def main():
    args = [a for a in sys.argv[1:] if "=" in a]
    rounds = int(sys.argv[sys.argv.index("--rounds") + 1]) if "--rounds" in sys.argv else 5
    n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 10
    variants = [dict(kv.split("=", 1) for kv in a.split(";")) for a in args] or [{}]
    w = synth.gen_config(5)
    s = torch.cuda.current_stream()
    res = {i: [] for i in range(len(variants))}
    with pe.Context.from_workload(w) as ctx:
        out = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
        for _ in range(3):
            ctx.eval_device(w.j0, w.T, out.data_ptr(), w.T, s.cuda_stream)
        for r in range(rounds):
            for i, v in enumerate(variants):
                old = {k: os.environ.get(k) for k in v}
                os.environ.update(v)
                ctx.eval_device(w.j0, w.T, out.data_ptr(), w.T, s.cuda_stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(n):
                    ctx.eval_device(w.j0, w.T, out.data_ptr(), w.T, s.cuda_stream)
                e1.record(s)
                torch.cuda.synchronize()
                res[i].append(e0.elapsed_time(e1) / n)
                for k, x in old.items():
                    if x is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = x
    for i, v in enumerate(variants):
        print(json.dumps({"env": v, "ms_median": statistics.median(res[i]), "ms": res[i]}), flush=True)


if __name__ == "__main__":
    main()
