"""pe_eval (host result) wall time on one handle, first call vs repeated calls (plans cached), and
pe_eval_device alone: config 5, pinned output."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_11571_b200 as pe, synth
w = synth.gen_config(5)
L = pe.lib()
with pe.Context.from_workload(w) as ctx:
    out = torch.empty((ctx.G, w.T), dtype=torch.int64).pin_memory()
    for i in range(4):
        t0 = time.perf_counter()
        rc = L.pe_eval(ctx._h, w.j0, w.T, ctypes.c_void_p(out.data_ptr()))
        print(f"pe_eval call {i}: {1e3*(time.perf_counter()-t0):.2f} ms rc={rc}", flush=True)
    d = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx.eval_device(w.j0, w.T, d.data_ptr()); torch.cuda.synchronize()
        print(f"pe_eval_device call {i}: {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
# host cost of building k_tc plans: pe_tc_info builds the one-chunk plan of a fresh handle
with pe.Context.from_workload(w) as ctx2:
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ctx2.info(); t1 = time.perf_counter()
    print(f"first pe_tc_info (host plan build): {1e3*(t1-t0):.2f} ms", flush=True)
    t0 = time.perf_counter(); ctx2.info(); t1 = time.perf_counter()
    print(f"second pe_tc_info: {1e3*(t1-t0):.2f} ms", flush=True)
    d = torch.empty((ctx2.G, w.T), dtype=torch.int64, device="cuda")
    for i in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ctx2.eval_device(w.j0, w.T, d.data_ptr()); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(f"fresh handle pe_eval_device call {i}: enqueue {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms", flush=True)
