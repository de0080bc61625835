"""Wall-clock breakdown of one e2e cycle (pe_create -> pe_eval -> pe_destroy) on config 5, pinned inputs."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2004_11571_b200 as pe, synth
w = synth.gen_config(5)
L = pe.lib()
pin = lambda a: torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a.view(np.int32)).pin_memory()
hc, he, ha = pin(w.coeffs), pin(np.ascontiguousarray(w.exps)), pin(w.alpha)
for it in range(4):
    t0 = time.perf_counter()
    h = L.pe_create(w.p, w.t, w.n, ctypes.c_void_p(hc.data_ptr()), ctypes.c_void_p(he.data_ptr()), ctypes.c_void_p(ha.data_ptr()))
    t1 = time.perf_counter()
    G = L.pe_num_buckets(h)
    if it == 0:
        out = torch.empty((G, w.T), dtype=torch.int64).pin_memory()
    rc = L.pe_eval(h, w.j0, w.T, ctypes.c_void_p(out.data_ptr()))
    t2 = time.perf_counter()
    L.pe_destroy(h)
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.1f} ms  eval(+D2H) {1e3*(t2-t1):7.1f} ms  destroy {1e3*(t3-t2):6.1f} ms  total {1e3*(t3-t0):7.1f} ms", flush=True)
