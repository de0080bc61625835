"""Handles used from several streams and threads at once (include/pe.h: pe_destroy waits for the
handle's own streams and for the latest evaluation on each caller stream, not for the whole
device; k_tc claims whole SMs so another stream's kernels cannot share an SM with it).

Every result is compared bit for bit with a serial evaluation of the same workload, which the
parity tests tie to the CPU oracle; the first one is also checked against the oracle here."""
import threading

import numpy as np
import pytest
import torch

import oracle
import paper_2004_11571_b200 as pe
import synth

pytestmark = pytest.mark.gpu


def _serial(w):
    with pe.Context.from_workload(w) as ctx:
        return ctx.eval(w.j0, w.T)


def test_destroy_waits_for_work_on_a_caller_stream():
    """Five evaluations queued on a side stream, the handle destroyed at once, a new handle created
    (it reuses the freed pool memory) -- the queued evaluations still read the first handle's
    buffers and must finish with the right result."""
    w = synth.gen_config(3)
    ref = _serial(w)
    ks = np.array([0, 1, 2047, w.T - 1], np.uint64)
    assert np.array_equal(ref[:, ks.astype(np.int64)], oracle.eval_workload(w, ks=ks))
    side = torch.cuda.Stream()
    ctx = pe.Context.from_workload(w)
    G = ctx.G
    outs = [torch.full((G, w.T), -1, dtype=torch.int64, device="cuda") for _ in range(5)]
    torch.cuda.synchronize()
    for o in outs:
        ctx.eval_device(w.j0, w.T, o.data_ptr(), w.T, side.cuda_stream)
    ctx.close()                                  # pe_destroy: waits for the side stream's last eval
    other = pe.Context.from_workload(synth.gen_config(3, seed=7))   # allocations reuse the pool
    other.close()
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint64), ref)


def test_create_on_a_thread_while_another_handle_evaluates():
    """The pipelined pattern of bench.py's e2e figure: polynomial i+1's pe_create on a worker thread
    while polynomial i is evaluated on the main thread; three rounds, two workloads alternating."""
    ws = [synth.gen_config(3), synth.gen_config(3, seed=11)]
    refs = [_serial(w) for w in ws]
    results = {}

    def make(i):
        results[i] = pe.Context.from_workload(ws[i % 2])

    make(0)
    for i in range(6):
        th = threading.Thread(target=make, args=(i + 1,))
        th.start()
        ctx = results.pop(i)
        out = ctx.eval(ws[i % 2].j0, ws[i % 2].T)
        ctx.close()
        th.join()
        assert np.array_equal(out, refs[i % 2]), f"polynomial {i}"
    results.pop(6).close()


def test_tc_exclusive_off_gives_the_same_bits(monkeypatch):
    """k_tc's static schedule needs every CTA on its own SM, so by default it asks for the whole
    per-block shared-memory opt-in (no other kernel's CTA fits beside it); PE_TC_EXCLUSIVE=0 asks
    only for what it uses.  Both give the same bits."""
    w = synth.gen_config(3)
    ref = _serial(w)
    monkeypatch.setenv("PE_TC_EXCLUSIVE", "0")
    assert np.array_equal(_serial(w), ref)
