"""Multi-rank point sharding + gather (paper_2004_11571_b200/dist.py) on CPU with gloo.

The per-rank evaluation is injected: here each rank evaluates its column block with the CPU
oracle (test infrastructure), so this checks the host logic -- shard ranges, uneven tails,
empty ranks, the gather and the [P][G][T_r] -> [G][T] permutation -- against one
single-process oracle call.  On GPUs the same object drives pe_eval_device over NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2004_11571_b200.dist import ShardedEval, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, T, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        w = synth.random_small(42, synth.P62, 6, 300, 3, T, 5)
        G = oracle.buckets(w.exps, w.n).shape[0]
        sh = ShardedEval(G, T, torch.device("cpu"))

        def eval_local(j_first, cnt, out):
            r = oracle.eval_direct(w.p, w.n, w.coeffs, w.exps, w.alpha, j_first, cnt)
            out[:, :cnt] = torch.from_numpy(r.view(np.int64))

        res = sh.run(eval_local, w.j0)
        if rank == 0:
            q.put(res.numpy().view(np.uint64).copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 37), (3, 37), (2, 1), (4, 6)])
def test_sharded_gather_matches_single(world, T):
    import oracle
    import synth
    w = synth.random_small(42, synth.P62, 6, 300, 3, T, 5)
    ref = oracle.eval_direct(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, T)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, ref)


def test_shard_range_cover():
    for T in (0, 1, 5, 16384, 16385):
        for world in (1, 2, 3, 8):
            cols = []
            for r in range(world):
                off, cnt = shard_range(T, world, r)
                cols += list(range(off, off + cnt))
            assert cols == list(range(T))
