"""Multi-rank point sharding + gather (paper_2004_11571_b200/dist.py) on CPU with gloo.

The per-rank evaluation is injected: here each rank evaluates its column block with the CPU
oracle (test infrastructure), so this checks the host logic -- shard ranges, uneven tails,
empty ranks, the gather and the root's placement -- against one single-process oracle call.
libpe's device calls (pe_unshard_columns, pe_rows_addmod) need a GPU, so the CPU runs inject host
stand-ins for them (``_unshard_host`` / ``_addmod_host``, Python integers); on GPUs the same
objects drive pe_eval_device and the libpe calls over NCCL (tests/test_gpu_dist.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2004_11571_b200.dist import ShardedEval, shard_range


def _unshard_host(out, blocks, T):
    P, G, Tr = blocks.shape
    for r in range(P):
        cnt = max(0, min(Tr, T - r * Tr))
        if cnt:
            out[:, r * Tr:r * Tr + cnt] = blocks[r, :, :cnt]


def _addmod_host(p):
    def f(dst, src):
        a = dst.numpy().view(np.uint64).astype(object)
        b = src.numpy().view(np.uint64).astype(object)
        dst.copy_(torch.from_numpy(((a + b) % p).astype(np.uint64).view(np.int64)))
    return f


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
        sh = ShardedEval(G, T, torch.device("cpu"), unshard=_unshard_host)

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


# ---------------------------------------------------------------- term-range sharding
def _term_worker(rank, world, port, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2004_11571_b200.dist import TermShardedEval, bucket_keys, term_partition
        seed, t, T, big, p = args
        w = synth.random_small(seed, p, 6, t, 3, T, 5)
        if big:   # one bucket holding most terms: it spans several ranks (middle ranks: 1 row)
            w.exps[: int(0.8 * t), :2] = (2, 2)
        order, bounds = term_partition(w.exps, world)
        sh = TermShardedEval(bucket_keys(w.exps)[order], bounds, T, w.p, torch.device("cpu"),
                             addmod=_addmod_host(w.p))
        mine = order[bounds[rank]:bounds[rank + 1]]

        def eval_local(out):      # rank's own handle: here the CPU oracle on its terms
            r = oracle.eval_direct(w.p, w.n, w.coeffs[mine], w.exps[mine], w.alpha, w.j0, T)
            assert r.shape == tuple(out.shape)
            out.copy_(torch.from_numpy(r.view(np.int64)))

        res = sh.run(eval_local)
        if rank == 0:
            q.put(res.numpy().view(np.uint64).copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,t,T,big,p", [(2, 300, 9, False, (1 << 62) - 57), (3, 301, 7, False, (1 << 62) - 57),
                                             (4, 250, 5, True, (1 << 62) - 57), (3, 2, 4, False, (1 << 62) - 57),
                                             (2, 1, 3, False, (1 << 62) - 57), (4, 250, 5, True, (1 << 63) - 25)])
def test_term_sharded_matches_single(world, t, T, big, p):
    """Bucket-contiguous term ranges + P2P row gather + boundary rows summed mod p reproduce the
    single-process oracle, including a bucket spanning several ranks, empty ranks (t < world) and
    a prime above 2^62 (boundary sums up to 2p - 2 >= 2^63)."""
    import oracle
    import synth
    seed = 77
    w = synth.random_small(seed, p, 6, t, 3, T, 5)
    if big:
        w.exps[: int(0.8 * t), :2] = (2, 2)
    ref = oracle.eval_direct(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, T)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_term_worker, args=(r, world, port, (seed, t, T, big, p), q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got, ref)


def test_term_partition_bookkeeping():
    """Row offsets / overlaps: ranks cover the global rows in order, sharing only boundary buckets."""
    import synth
    from paper_2004_11571_b200.dist import bucket_keys, term_partition
    w = synth.gen_config(2, t=5000, T=1)
    for world in (1, 2, 3, 8):
        order, bounds = term_partition(w.exps, world)
        ks = bucket_keys(w.exps)[order]
        assert np.all(ks[1:] <= ks[:-1])                       # descending bucket order
        # the bookkeeping TermShardedEval derives (no process group needed here)
        new_row = np.r_[True, ks[1:] != ks[:-1]]
        row_of = np.cumsum(new_row) - 1
        covered = []
        for r in range(world):
            a, b = bounds[r], bounds[r + 1]
            rows = sorted(set(row_of[a:b].tolist()))
            assert rows == list(range(rows[0], rows[-1] + 1))
            covered += rows if not (a > 0 and not new_row[a]) else rows[1:]
        assert covered == list(range(int(row_of[-1]) + 1))


# ---------------------------------------------------------------- overlapped row blocks
def _blocks_worker(rank, world, port, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2004_11571_b200.dist import TermShardedEval, bucket_keys, term_partition
        seed, t, T, p = args
        w = synth.random_small(seed, p, 6, t, 3, T, 5)
        w.exps[: int(0.5 * t), :2] = (2, 2)                     # one bucket across ranks
        order, bounds = term_partition(w.exps, world)
        sh = TermShardedEval(bucket_keys(w.exps)[order], bounds, T, w.p, torch.device("cpu"),
                             addmod=_addmod_host(w.p))
        mine = order[bounds[rank]:bounds[rank + 1]]
        full = oracle.eval_direct(w.p, w.n, w.coeffs[mine], w.exps[mine], w.alpha, w.j0, T) if mine.size else None
        splits = [None] * world
        my_split = (rank * 7 + 1) % max(1, sh.G_r[rank]) if sh.G_r[rank] else 0   # arbitrary splits, some 0
        dist.all_gather_object(splits, my_split)
        sh.set_splits(splits)
        calls = []

        def eval_rows(a, b, local):            # rows [a, b) of this rank's output
            calls.append((a, b))
            local[a:b].copy_(torch.from_numpy(full[a:b].view(np.int64)))

        res = sh.run_blocks(eval_rows)
        assert sorted(calls) == sorted(sh._blocks(rank))
        if rank == 0:
            q.put(res.numpy().view(np.uint64).copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,t,T,p", [(2, 300, 7, (1 << 62) - 57), (3, 400, 5, (1 << 63) - 25),
                                         (4, 500, 3, (1 << 62) - 57)])
def test_term_sharded_row_blocks_match_single(world, t, T, p):
    """The overlapped gather (each rank's rows in two blocks, block 0 sent while block 1 is being
    evaluated; TermShardedEval.run_blocks) reproduces the single-process oracle, whatever the
    ranks' splits -- including none, and splits that cut a shared boundary row's rank."""
    import oracle
    import synth
    seed = 91
    w = synth.random_small(seed, p, 6, t, 3, T, 5)
    w.exps[: int(0.5 * t), :2] = (2, 2)
    ref = oracle.eval_direct(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, T)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blocks_worker, args=(r, world, port, (seed, t, T, p), q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert np.array_equal(got, ref)
