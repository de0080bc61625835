"""Timeline of the pipelined e2e loop (bench.py e2e): polynomial i+1's pe_create on a host thread
while polynomial i is evaluated.  Prints per-step host timestamps (ms from the loop start) of the
create (worker) and eval / destroy (main) calls, for the uint32 and the compact entry points."""
import argparse, ctypes, os, sys, time
from concurrent.futures import ThreadPoolExecutor
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_11571_b200 as pe, synth

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--pre-ctx", action="store_true", help="keep a device handle alive and evaluate it first (as bench.py)")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--mma", action="store_true", help="run pe.bench_mma first (as bench.py)")
ap.add_argument("--prelude", default="", help="comma list of bench.py steps to replay first: dev,tiny,ctx,sh")
ap.add_argument("--modes", default="u32,compact")
args = ap.parse_args()
w = synth.gen_config(args.cfg)
pre = set(filter(None, args.prelude.split(",")))
keep = []
if "dist" in pre:
    import torch.distributed as dist  # noqa: F401
    from paper_2004_11571_b200.dist import ShardedEval as _SE  # noqa: F401
if "fork" in pre:
    import subprocess
    subprocess.run(["nvidia-smi", "-L"], stdout=subprocess.DEVNULL)
if "dev" in pre:
    torch.cuda.set_device(0)
    _st = torch.cuda.current_stream(torch.device("cuda", 0))
if "tiny" in pre:
    t1 = pe.Context(w.p, w.coeffs[:1], w.exps[:1], w.alpha, n=w.n)
    t1.uses_tc(w.T)
    t1.close()
if "ctx" in pre:
    c = pe.Context(w.p, w.coeffs, w.exps, w.alpha, n=w.n)
    c.info()
    keep.append(c)
    if "sh" in pre:
        from paper_2004_11571_b200.dist import ShardedEval
        keep.append(ShardedEval(c.G, w.T, torch.device("cuda", 0)))
if "fork2" in pre:
    import subprocess
    subprocess.run(["nvidia-smi", "-L"], stdout=subprocess.DEVNULL)
L = pe.lib()
pin = lambda a: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).pin_memory()
if "order" in pre:     # bench.py's allocation order: coeffs, exps, alpha, result, uint8 exps
    hc, he, ha = pin(w.coeffs), pin(np.ascontiguousarray(w.exps).view(np.int32)), pin(w.alpha)
    out0 = torch.empty((w.G if hasattr(w, "G") else 961, w.T), dtype=torch.int64).pin_memory()
else:
    hc, ha = pin(w.coeffs), pin(w.alpha)
    he = pin(np.ascontiguousarray(w.exps).view(np.int32))
    out0 = None
he8 = torch.from_numpy(np.ascontiguousarray(w.exps.astype(np.uint8))).pin_memory()
T0 = [0.0]
now = lambda: 1e3 * (time.perf_counter() - T0[0])


def create(compact):
    a = now()
    if compact:
        h = L.pe_create_compact(w.p, w.t, w.n, ctypes.c_void_p(hc.data_ptr()), ctypes.c_void_p(he8.data_ptr()),
                                ctypes.c_void_p(ha.data_ptr()), None)
    else:
        h = L.pe_create(w.p, w.t, w.n, ctypes.c_void_p(hc.data_ptr()), ctypes.c_void_p(he.data_ptr()),
                        ctypes.c_void_p(ha.data_ptr()))
    assert h
    return h, a, now()


h0, _, _ = create(False)
G = L.pe_num_buckets(h0)
L.pe_destroy(h0)
out = out0 if out0 is not None and out0.shape[0] == G else torch.empty((G, w.T), dtype=torch.int64).pin_memory()
if args.pre_ctx:
    ctx = pe.Context(w.p, w.coeffs, w.exps, w.alpha, n=w.n)
    dout = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    for _ in range(23):
        ctx.eval_device(w.j0, w.T, dout.data_ptr(), w.T, st.cuda_stream)
    torch.cuda.synchronize()
if args.mma:
    print("mma", pe.bench_mma(64), pe.bench_mma(128))
for compact in [m == "compact" for m in args.modes.split(",")]:
    for mode in ["serial"] + ["pipelined"] * args.reps:
        with ThreadPoolExecutor(1) as ex:
            for _ in range(2):                       # warm the worker and the memory pool (2 in flight)
                ha_, _, _ = ex.submit(create, compact).result()
                hb_, _, _ = ex.submit(create, compact).result()
                L.pe_destroy(ha_)
                L.pe_destroy(hb_)
            torch.cuda.synchronize()
            T0[0] = time.perf_counter()
            fut = ex.submit(create, compact)
            rows = []
            for i in range(args.k):
                h, ca, cb = fut.result()
                if mode == "pipelined" and i + 1 < args.k:
                    fut = ex.submit(create, compact)
                ea = now()
                assert L.pe_eval(h, w.j0, w.T, ctypes.c_void_p(out.data_ptr())) == 0
                eb = now()
                L.pe_destroy(h)
                db = now()
                if mode == "serial" and i + 1 < args.k:
                    fut = ex.submit(create, compact)
                rows.append((ca, cb, ea, eb, db))
            tot = now()
        print(f"{'compact' if compact else 'u32'} {mode}: {tot / args.k:.2f} ms/step")
        for r in rows:
            print("   create %7.2f..%7.2f  eval %7.2f..%7.2f  destroy ..%7.2f" % r)
        sys.stdout.flush()
