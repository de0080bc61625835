"""NEXT-2: Berlekamp-Massey per bucket on the GPU (csrc/bm.cu) -- parity with the pinned Python
oracle (oracle/bm.py), and BM as an oracle-free validator of the evaluation output (pin P9 at
full size: the bucket sequence of r distinct monomial values has connection polynomial
prod (1 - m_i z), Ben-Or/Tiwari)."""
import numpy as np
import pytest

import oracle
import paper_2004_11571_b200 as pe
import synth
from oracle.bm import berlekamp_massey

pytestmark = pytest.mark.gpu
P62 = synth.P62


@pytest.mark.parametrize("p,T", [(P62, 40), (1_000_003, 33), (13, 20), ((1 << 63) - 25, 17)])
def test_bm_random_sequences_match_oracle(p, T):
    rng = np.random.default_rng(p % 1000 + T)
    seqs = [rng.integers(0, p, T, dtype=np.uint64) for _ in range(20)]
    # low-complexity sequences: sums of r geometric progressions, zeros, impulses
    for r in (1, 2, 3, T // 2):
        ms = rng.integers(1, p, r, dtype=np.uint64)
        cs = rng.integers(1, p, r, dtype=np.uint64)
        seqs.append(np.array([sum(int(c) * pow(int(m), k, p) for c, m in zip(cs, ms)) % p for k in range(T)],
                             np.uint64))
    seqs.append(np.zeros(T, np.uint64))
    imp = np.zeros(T, np.uint64)
    imp[-1] = 1
    seqs.append(imp)
    S = np.stack(seqs)
    ln, lam = pe.berlekamp_massey(p, S)
    for g in range(S.shape[0]):
        L, C = berlekamp_massey(S[g].tolist(), p)
        assert int(ln[g]) == L, g
        assert lam[g, :L + 1].tolist() == C and not lam[g, L + 1:].any(), g


def _poly_at(c, x, p):
    v = 0
    for ci in reversed(c):
        v = (v * x + int(ci)) % p
    return v


def test_bm_validates_config2_output():
    """config 2 (many small buckets): evaluate at j = 0..T-1 with T >= 2 * max bucket, BM every row,
    compare with prod (1 - m_i z) over each bucket's distinct nonzero-coefficient m_i."""
    w = synth.gen_config(2, t=20_000, T=1)
    import collections
    keys = [(int(e[0]), int(e[1])) for e in w.exps]
    sizes = collections.Counter(keys)
    T = 2 * max(sizes.values()) + 4
    with pe.Context.from_workload(w) as ctx:
        out = ctx.eval(0, T)
        rows = ctx.buckets().tolist()
        m = ctx.monomials()
    ln, lam = pe.berlekamp_massey(w.p, out)
    members = collections.defaultdict(dict)
    for i, k in enumerate(keys):
        d = members[k]
        d[int(m[i])] = (d.get(int(m[i]), 0) + int(w.coeffs[i])) % w.p
    for g, r in enumerate(rows):
        ms = [mi for mi, c in members[tuple(r)].items() if c]
        assert int(ln[g]) == len(ms), g
        for mi in ms[:5]:
            assert _poly_at(lam[g, :len(ms) + 1], pow(mi, w.p - 2, w.p), w.p) == 0


def test_bm_validates_config5_full_size():
    """Full config 5 (t = 10^7, T = 16384) on the device: BM on every bucket with fewer than T/2
    terms must give L = #distinct m_i and C(1/m_i) = 0 -- an oracle-free check of every column."""
    import torch
    w = synth.gen_config(5)
    with pe.Context.from_workload(w) as ctx:
        G, T = ctx.G, w.T
        rows = ctx.buckets().tolist()
        m = ctx.monomials()
        d_out = torch.empty((G, T), dtype=torch.int64, device="cuda")
        ctx.eval_device(w.j0, T, d_out.data_ptr(), T, 0)
        torch.cuda.synchronize()
    lam = torch.empty((G, T + 1), dtype=torch.int64, device="cuda")
    ln = torch.empty(G, dtype=torch.int32, device="cuda")
    rc = pe.lib().pe_bm_device(w.p, G, T, d_out.data_ptr(), T, lam.data_ptr(), T + 1, ln.data_ptr(), None)
    assert rc == 0
    torch.cuda.synchronize()
    ln = ln.cpu().numpy()
    key = (w.exps[:, 0].astype(np.int64) << 32) | w.exps[:, 1].astype(np.int64)
    order = np.argsort(key, kind="stable")
    ks, starts = np.unique(key[order], return_index=True)
    ends = np.append(starts[1:], len(order))
    row_of = {(int(r[0]) << 32) | int(r[1]): g for g, r in enumerate(rows)}
    checked = 0
    rng = np.random.default_rng(5)
    for kv, a, b in zip(ks, starts, ends):
        if b - a >= T // 2:
            continue
        g = row_of[int(kv)]
        idx = order[a:b]
        ms, inv = np.unique(m[idx], return_inverse=True)
        csum = np.zeros(len(ms), dtype=object)
        for j, ii in zip(inv, idx):
            csum[j] = (csum[j] + int(w.coeffs[ii])) % w.p
        r_g = int(sum(1 for c in csum if c))
        assert int(ln[g]) == r_g, (g, int(ln[g]), r_g)
        if checked < 6:                                        # evaluate C_g at a few 1/m_i
            c = lam[g, : r_g + 1].cpu().numpy().view(np.uint64)
            for mi in rng.choice(ms, 2):
                assert _poly_at(c, pow(int(mi), w.p - 2, w.p), w.p) == 0
        checked += 1
    assert checked >= 790                                      # 798 of the 961 buckets have < T/2 terms
