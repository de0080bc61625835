"""The multi-GPU assembly on one GPU: per-rank handles evaluated on cuda:0 and put
together by the same dist.py bookkeeping the NCCL path uses (TermShardedEval / ShardedEval
``assemble``, no process group), with libpe's pe_rows_addmod / pe_unshard_columns doing the
placement and the boundary-bucket sums.  Compared with the CPU oracle (HM16's
point ranges, MT18-style term ranges)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2004_11571_b200 as pe
import synth
from paper_2004_11571_b200.dist import ShardedEval, TermShardedEval, bucket_keys, term_partition

pytestmark = pytest.mark.gpu

P62, P63 = synth.P62, (1 << 63) - 25


def _zipf_workload(p, seed, t=120_000, T=8192 + 300):
    """Config-3-like terms with one bucket holding 60% of them (it spans >= 3 ranges for P >= 3)
    and a tail of small buckets; T = one chunk + a ragged 300 (two tensor-core chunks)."""
    w = synth.gen_config(3, t=t, T=T, seed=seed)
    w.p = p
    rng = np.random.default_rng(seed)
    w.coeffs = synth.uniform_mod(rng, 0, p, w.t)
    w.alpha = synth.uniform_mod(rng, 1, p, w.n - 2)
    w.exps[: int(0.6 * w.t), :2] = (7, 3)
    return w


@pytest.mark.parametrize("p", [P62, P63])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_term_sharded_assembly(p, P):
    w = _zipf_workload(p, 700 + P)
    ref = oracle.eval_incremental_blocked(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    order, bounds = term_partition(w.exps, P)
    sh = TermShardedEval(bucket_keys(w.exps)[order], bounds, w.T, w.p, torch.device("cuda"), world=P, rank=0)
    assert sum(sh.overlap) >= min(2, P - 1)               # the big bucket is cut by every boundary in it
    s = torch.cuda.current_stream().cuda_stream
    locals_ = []
    for r in range(P):
        mine = np.sort(order[bounds[r]:bounds[r + 1]])
        with pe.Context(w.p, w.coeffs[mine], w.exps[mine], w.alpha, n=w.n) as ctx:
            assert ctx.G == sh.G_r[r] and ctx.uses_tc(w.T)
            loc = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
            ctx.eval_device(w.j0, w.T, loc.data_ptr(), w.T, s)
            torch.cuda.synchronize()
        locals_.append(loc)
    out = sh.assemble(locals_).cpu().numpy().view(np.uint64)
    assert out.shape == ref.shape
    bad = np.argwhere(out != ref)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"


@pytest.mark.parametrize("P", [2, 3, 8])
def test_point_sharded_assembly(P):
    """Point ranges: every rank's handle is the full term set, seeded at its own first point;
    T = 1000 is split unevenly over P (ragged last shard)."""
    w = synth.gen_config(2, t=30_000, T=1000)
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    s = torch.cuda.current_stream().cuda_stream
    with pe.Context.from_workload(w) as ctx:
        sh = ShardedEval(ctx.G, w.T, torch.device("cuda"), world=P, rank=0)

        def eval_rank(r, j_first, cnt, out_view):
            ctx.eval_device(j_first, cnt, out_view.data_ptr(), out_view.shape[1], s)

        out = sh.assemble(eval_rank, w.j0).cpu().numpy().view(np.uint64)
    assert np.array_equal(out, ref)


def test_rows_addmod_no_wrap_above_2_62():
    """pe_rows_addmod at p = 2^63 - 25: (p-1) + (p-1) = 2p - 2 >= 2^63 must give p - 2 (the int64
    overflow of round 1's Python boundary sum), and a strided sub-block leaves the rest alone."""
    p = P63
    a = np.array([[p - 1, p - 1, 0, 5], [1, p - 2, 7, 7]], np.uint64)
    b = np.array([[p - 1, 1, 0, p - 5], [p - 1, 1, 9, 9]], np.uint64)
    want = [[(int(x) + int(y)) % p for x, y in zip(ra, rb)] for ra, rb in zip(a, b)]
    da = torch.from_numpy(a.view(np.int64)).cuda()
    db = torch.from_numpy(b.view(np.int64)).cuda()
    pe.rows_addmod(p, da.data_ptr(), 4, db.data_ptr(), 4, 2, 4)
    assert da.cpu().numpy().view(np.uint64).tolist() == want
    dc = torch.from_numpy(a.view(np.int64)).cuda()
    pe.rows_addmod(p, dc.data_ptr(), 4, db.data_ptr(), 4, 2, 2)           # columns 0..1 only
    got = dc.cpu().numpy().view(np.uint64)
    assert got[:, :2].tolist() == [r[:2] for r in want] and np.array_equal(got[:, 2:], a[:, 2:])
    with pytest.raises(pe.PEError):
        pe.rows_addmod(1 << 63, da.data_ptr(), 4, db.data_ptr(), 4, 2, 4)


def test_unshard_columns_ragged():
    P, G, Tr, T = 3, 5, 4, 10
    blocks = torch.arange(P * G * Tr, dtype=torch.int64, device="cuda").reshape(P, G, Tr)
    out = torch.full((G, T + 2), -1, dtype=torch.int64, device="cuda")
    pe.unshard_columns(out.data_ptr(), T + 2, blocks.data_ptr(), P, G, Tr, T)
    want = torch.cat([blocks[r] for r in range(P)], dim=1)[:, :T]
    assert torch.equal(out[:, :T], want) and bool((out[:, T:] == -1).all())


def test_eval_device_rows_blocks_equal_full():
    """pe_eval_device_rows: rows [0, s) then [s, G) (the handle's own split, and an arbitrary one)
    fill exactly what one pe_eval_device does -- the building block of the overlapped gather
    (TermShardedEval.run_blocks); a strict row range off the tensor-core path is PE_ENOTSUP."""
    w = synth.gen_config(3, t=200_000, T=9000)
    s_ = torch.cuda.current_stream().cuda_stream
    with pe.Context.from_workload(w) as ctx:
        G = ctx.G
        full = torch.empty((G, w.T), dtype=torch.int64, device="cuda")
        ctx.eval_device(w.j0, w.T, full.data_ptr(), w.T, s_)
        for split in (ctx.row_split(), G // 3, 1, G - 1):
            assert 0 < split < G
            part = torch.full_like(full, -1)
            ctx.eval_device_rows(w.j0, w.T, 0, split, part.data_ptr(), w.T, s_)
            assert bool((part[split:] == -1).all())                     # other rows untouched
            ctx.eval_device_rows(w.j0, w.T, split, G, part.data_ptr(), w.T, s_)
            torch.cuda.synchronize()
            assert torch.equal(part, full), split
    with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
        assert ctx.row_split() == 0
        buf = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
        with pytest.raises(pe.PEError) as ei:
            ctx.eval_device_rows(w.j0, w.T, 0, 5, buf.data_ptr(), w.T, s_)
        assert ei.value.code == pe.PE_ENOTSUP
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(full.cpu().numpy().view(np.uint64), ref)
