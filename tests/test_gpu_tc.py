"""GPU parity of the tensor-core path (PE_PATH_TC, csrc/tc.cuh) against the CPU oracle through
the C ABI.  The path factors each bucket's 128 x 64-point chunk into giant-step x baby-step
values (the Vandermonde structure m_i^{j} = m_i^{j_s + 64u} m_i^{v}, u < 128, v < 64,
PAPER.md:420-427) and sums their 64 byte-pair products on int8 tensor cores; results must be bit-identical to the oracle
(canonical residues are unique, R14)."""
import math

import numpy as np
import pytest

import oracle
import paper_2004_11571_b200 as pe
import synth

pytestmark = pytest.mark.gpu

P62 = synth.P62


def tc_eval(w, j0=None, T=None, path=pe.PATH_TC):
    with pe.Context.from_workload(w, path=path) as ctx:
        T = w.T if T is None else T
        assert ctx.uses_tc(T), ctx.info()
        out = ctx.eval(w.j0 if j0 is None else j0, T)
        rows = ctx.buckets()
    return rows, out


def check_tc(w, **kw):
    rows, out = tc_eval(w, **kw)
    assert rows.tolist() == oracle.buckets(w.exps, w.n).tolist()
    ref = oracle.eval_workload(w)
    bad = np.argwhere(out != ref)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"


@pytest.mark.parametrize("p,n,t,maxdeg,j0,T", [
    (P62, 6, 300, 4, 1, 1),               # T = 1 (one column of an 8192-point chunk)
    (P62, 6, 300, 4, 1, 129),             # ragged inside the first chunk (u = 1, v = 0)
    (P62, 5, 500, 3, 0, 70),              # j0 = 0
    (P62, 5, 200, 3, 2**64 - 40, 40),     # largest j range (seed exponents near 2^64)
    (13, 4, 60, 3, 0, 50),                # tiny prime
    (3, 5, 40, 2, 5, 20),                 # smallest prime
    ((1 << 62) - 57, 2, 30, 6, 1, 10),    # n = 2 (m = 1: every column = coefficient sums)
    (2**31 - 1, 3, 100, 9, 1, 64),        # n = 3, 31-bit p through the 64-bit tensor path
    ((1 << 50) - 27, 7, 600, 4, 3, 77),   # 50-bit p (auto would take FP64 Alg. 2)
    ((1 << 63) - 25, 6, 700, 4, 5, 300),  # largest supported p: exact-quotient giant-step chains
    ((1 << 54) - 33, 6, 700, 4, 2, 300),  # largest 7-digit-mode p (lazy values < 4p < 2^56)
    ((1 << 31) + 11, 6, 700, 4, 2, 300),  # smallest 7-digit-mode p
    ((1 << 62) + 135, 5, 400, 3, 1, 129), # just above 2^62
])
def test_tc_edge_shapes(p, n, t, maxdeg, j0, T):
    w = synth.random_small(500 + t + n, p, n, t, maxdeg, T, j0, coeff_hi=2**64 - 1)
    check_tc(w)


def test_tc_two_chunks_and_tail():
    """T = 2 x 16384 + 1000: three chunks (seeds at j0, j0 + 16384, j0 + 32768), ragged tail."""
    w = synth.random_small(520, P62, 6, 2000, 4, 2 * 16384 + 1000, 7)
    _, out = tc_eval(w)
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, ref)


def test_tc_config1_and_config2_full():
    check_tc(synth.gen_config(1))
    check_tc(synth.gen_config(2))


def test_tc_pieces_of_one_large_bucket():
    """One (x,y) bucket of 20 000 terms split into several accumulation pieces (<= 8192 terms each,
    the u32 exactness bound of DESIGN.md §7, and <= twice the per-SM load: 1024 here) summed by the
    fix-up; plus a 1-term and a 33-term bucket."""
    w = synth.random_small(521, P62, 8, 20_034, 5, 300, 1)
    w.exps[:, :2] = 4
    w.exps[0, :2] = (9, 9)
    w.exps[1:34, :2] = (0, 1)
    with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
        assert ctx.info()["tc_pieces"] >= 5
    _, out = tc_eval(w)
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, ref)
    ks = np.array([0, 1, 127, 128, 299], np.uint64)
    assert np.array_equal(out[:, ks.astype(np.int64)], oracle.eval_workload(w, ks=ks))


def test_tc_config3_full_incremental():
    w = synth.gen_config(3)
    _, out = tc_eval(w)
    inc = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, inc)


def test_tc_multi_pass_partial_cap(monkeypatch):
    """PE_PARTIAL_MB=1: the partial buffer holds one chunk, so T = 40000 runs as 3 passes."""
    monkeypatch.setenv("PE_PARTIAL_MB", "1")
    w = synth.random_small(522, P62, 5, 900, 4, 40_000, 2)
    _, out = tc_eval(w)
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, ref)


def test_tc_duplicates_zero_coeffs_alpha_ge_p():
    w = synth.random_small(523, P62, 5, 400, 2, 50, 1, dup=True)
    w.coeffs[::7] = 0
    w.coeffs[1::11] = np.uint64(P62 + 5)
    w.alpha = (w.alpha + np.uint64(P62)).astype(np.uint64)
    check_tc(w)


def test_tc_equals_scalar_step_and_fermat():
    """The tensor path equals k_step on the same inputs (P13), and is Fermat-periodic (P5)."""
    w = synth.gen_config(2, t=30_000, T=20_000)
    _, a = tc_eval(w)
    with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
        assert not ctx.uses_tc(w.T)
        b = ctx.eval(w.j0, w.T)
    assert np.array_equal(a, b)
    _, c = tc_eval(w, j0=w.j0 + (w.p - 1))
    assert np.array_equal(a, c)


def v32_min_T(tp):
    """pe.cu tc_min_T_v32: the automatic threshold of the V = 32 geometry (p >= 2^54), fitted to the
    measured crossovers (profiles/r02_tc_threshold_v32.jsonl)."""
    return min(8192, max(192, math.ceil(max(3400.0 * tp ** -0.19, 7.3e6 / tp))))


def test_tc_auto_selection():
    """PE_PATH_AUTO: tensor path for any p < 2^63 and T >= the handle's threshold (p >= 2^54:
    max(3400 t_pad^-0.19, 7.3e6 / t_pad) in [192, 8192]; 2^31 <= p < 2^54: max(2200 t_pad^-0.144,
    7.3e6 / t_pad) in [192, 8192]; p < 2^31: max(1350 t_pad^-0.045, 1.1e7 / t_pad) in [512, 8192]);
    never for PE_PATH_INT or PE_PATH_FP64."""
    w = synth.random_small(524, P62, 5, 100, 3, 10, 1)
    with pe.Context.from_workload(w) as ctx:
        tp = ctx.info()["t_padded"]
        m = ctx.info()["tc_min_T"]
        assert abs(m - v32_min_T(tp)) <= 1 and m > 4000                  # tiny handle: k_step almost always
        assert ctx.uses_tc(m) and not ctx.uses_tc(m - 1)
    w2 = synth.gen_config(2, T=10)
    with pe.Context.from_workload(w2) as ctx:
        tp = ctx.info()["t_padded"]
        assert abs(ctx.info()["tc_min_T"] - v32_min_T(tp)) <= 1 and ctx.uses_tc(1000)   # config 2
    w3 = synth.gen_config(3, t=600_000, T=10)
    with pe.Context.from_workload(w3) as ctx:
        m = ctx.info()["tc_min_T"]
        assert 192 <= m <= 300 and ctx.uses_tc(m) and not ctx.uses_tc(m - 1)
    w7 = synth.gen_config(3, t=600_000, T=10)                          # 7-digit mode: its own fit
    w7.p = (1 << 50) - 27
    w7.coeffs %= np.uint64(w7.p)
    w7.alpha = (w7.alpha % np.uint64(w7.p - 1)) + np.uint64(1)
    with pe.Context.from_workload(w7) as ctx:
        tp = ctx.info()["t_padded"]
        m = ctx.info()["tc_min_T"]
        assert abs(m - min(8192, max(192, math.ceil(max(2200.0 * tp ** -0.144, 7.3e6 / tp))))) <= 1
        assert ctx.uses_tc(m) and not ctx.uses_tc(m - 1)
    w31 = synth.random_small(527, (1 << 31) - 1, 6, 600_000 // 8, 9, 10, 1)   # p < 2^31: vs 32-bit k_step
    with pe.Context.from_workload(w31) as ctx:
        tp = ctx.info()["t_padded"]
        assert abs(ctx.info()["tc_min_T"] - min(8192, max(512, math.ceil(max(1350.0 * tp ** -0.045, 1.1e7 / tp))))) <= 1
    with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
        assert not ctx.uses_tc(10**6)
    w50 = synth.random_small(525, (1 << 50) - 27, 5, 100, 3, 10, 1)
    with pe.Context.from_workload(w50) as ctx:       # FP64 Alg. 2 for short ranges, tensor form for long
        assert ctx.info()["path"] == "fp64" and ctx.uses_tc(10**6) and not ctx.uses_tc(100)
    with pe.Context.from_workload(w50, path=pe.PATH_FP64) as ctx:
        assert not ctx.uses_tc(10**6)
    w63 = synth.random_small(526, (1 << 63) - 25, 5, 100, 3, 10, 1)
    with pe.Context.from_workload(w63) as ctx:           # 2^62 <= p < 2^63: exact-quotient chains
        assert ctx.uses_tc(10**6) and not ctx.uses_tc(100)
    with pe.Context.from_workload(w63, path=pe.PATH_INT) as ctx:
        assert not ctx.uses_tc(10**6)


def test_tc_batch_polys():
    """pe_create_batch through the tensor path: f and h of config-2 shape at the same points."""
    f = synth.gen_config(2, t=20_000, T=300)
    h = synth.gen_config(2, t=20_000, T=300, seed=77)
    with pe.Context.batch(f.p, [(f.coeffs, f.exps), (h.coeffs, h.exps)], f.alpha, f.n,
                          path=pe.PATH_TC) as ctx:
        assert ctx.uses_tc(f.T)
        ro = ctx.poly_rows().astype(np.int64)
        out = ctx.eval(f.j0, f.T)
    assert np.array_equal(out[ro[0]:ro[1]], oracle.eval_incremental(f.p, f.n, f.coeffs, f.exps, f.alpha, f.j0, f.T))
    assert np.array_equal(out[ro[1]:ro[2]], oracle.eval_incremental(f.p, f.n, h.coeffs, h.exps, f.alpha, f.j0, f.T))


@pytest.mark.parametrize("R", [1, 2])
def test_tc_small_tiles_odd_kblocks(R):
    """R = 1 / 2 pads buckets to 32 / 64 terms only, so the padded term count can be an odd number
    of K-blocks (the baby-step plane builder works in pairs of K-blocks)."""
    w = synth.random_small(530 + R, P62, 4, 33, 2, 200, 3)
    with pe.Context.from_workload(w, path=pe.PATH_TC, R=R) as ctx:
        assert ctx.info()["R"] == R and ctx.uses_tc(w.T)
        assert (ctx.info()["t_padded"] // 32) % 2 == 1 or R == 2
        out = ctx.eval(w.j0, w.T)
    assert np.array_equal(out, oracle.eval_workload(w))


def test_mma_probe_rate():
    """pe_bench_mma runs and reports a plausible int8 rate (> 100 TOPS at N = 128)."""
    assert pe.bench_mma(128, 4000) > 1e14


@pytest.mark.parametrize("T", [16385, 2 * 8192, 3 * 8192 + 5])
def test_tc_host_eval_column_blocks(T):
    """pe_eval on the tensor path evaluates two row blocks (launches over a subset of the buckets)
    and overlaps the first block's device->host copy with the second's evaluation: the result
    equals pe_eval_device's (one launch over all rows) and the oracle's incremental evaluation."""
    import torch
    w = synth.random_small(540 + T % 97, P62, 6, 900, 4, T, 11)
    with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
        host = ctx.eval(w.j0, w.T)
        d = torch.empty((ctx.G, w.T), dtype=torch.int64, device="cuda")
        ctx.eval_device(w.j0, w.T, d.data_ptr())
        torch.cuda.synchronize()
        dev = d.cpu().numpy().view(np.uint64)
    assert np.array_equal(host, dev)
    assert np.array_equal(host, oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T))


@pytest.mark.parametrize("nbig", [8192, 8193, 16384 + 33])
def test_tc_piece_boundaries_and_max_tile(nbig):
    """A bucket of exactly one / just over one / two pieces (8192 terms each: the u32 exactness
    bound) with the largest tile (R = 16, buckets padded to 512 terms), many units per CTA."""
    t = nbig + 300
    w = synth.random_small(550 + nbig % 101, P62, 8, t, 5, 200, 2)
    w.exps[:, :2] = 3
    w.exps[:nbig, :2] = (7, 7)
    with pe.Context.from_workload(w, path=pe.PATH_TC, R=16) as ctx:
        assert ctx.info()["R"] == 16
        out = ctx.eval(w.j0, w.T)
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, ref)


def test_tc_63bit_prime_equals_scalar_step():
    """2^62 <= p < 2^63 (exact-quotient giant-step chains, values < 2p < 2^64): the tensor path
    equals k_step's lazy-2 Shoup path on a config-2-shaped instance spanning several chunks."""
    w = synth.random_small(560, (1 << 63) - 25, 8, 20_000, 6, 17_000, 3)
    with pe.Context.from_workload(w) as ctx:
        assert ctx.uses_tc(w.T)
        a = ctx.eval(w.j0, w.T)
    with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
        assert not ctx.uses_tc(w.T)
        b = ctx.eval(w.j0, w.T)
    assert np.array_equal(a, b)
    ks = np.array([0, 1, 8191, 8192, 16999], np.uint64)
    assert np.array_equal(a[:, ks.astype(np.int64)], oracle.eval_workload(w, ks=ks))


def test_tc_31bit_prime_equals_scalar_step():
    """p < 2^31: exact-quotient chains keep every value below 2^32, so the tensor path uses 4 byte
    digits (16 pairs, diagonals 0..6, one round of 5 MMAs); equals k_step's 32-bit Shoup path."""
    w = synth.random_small(570, (1 << 31) - 1, 8, 20_000, 6, 17_000, 3)
    with pe.Context.from_workload(w) as ctx:
        assert ctx.uses_tc(w.T)
        a = ctx.eval(w.j0, w.T)
    with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
        assert not ctx.uses_tc(w.T)
        b = ctx.eval(w.j0, w.T)
    assert np.array_equal(a, b)
    ks = np.array([0, 1, 8191, 8192, 16999], np.uint64)
    assert np.array_equal(a[:, ks.astype(np.int64)], oracle.eval_workload(w, ks=ks))


def test_tc_7digit_mode_equals_scalar_step():
    """2^31 <= p < 2^54 (here config 4's 2^50 - 27): 7 byte digits, 49 pairs in rounds of 12 + 6
    MMAs; equals k_step's FP64 Alg. 2 path on a config-4-shaped instance."""
    w = synth.gen_config(4, t=60_000, T=9000)
    with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
        a = ctx.eval(w.j0, w.T)
    with pe.Context.from_workload(w, path=pe.PATH_FP64) as ctx:
        assert not ctx.uses_tc(w.T)
        b = ctx.eval(w.j0, w.T)
    assert np.array_equal(a, b)
    ks = np.array([0, 1, 8191, 8192, 8999], np.uint64)
    assert np.array_equal(a[:, ks.astype(np.int64)], oracle.eval_workload(w, ks=ks))


@pytest.mark.parametrize("p", [P62, (1 << 54) + 159, (1 << 62) + 135, (1 << 63) - 25])
@pytest.mark.parametrize("form", [pe.TC_FORM_PLAIN, pe.TC_FORM_SWAPPED])
def test_tc_plain_and_swapped_forms(p, form):
    """For 8-digit primes (p >= 2^54) pe_config.tc_form picks the plain form (default: baby-step
    planes built per handle, giant steps generated per unit, tc.cuh MODE 0 / 1) or the swapped one
    (giant-step planes per handle, baby steps c m^{j_s + v} generated, MODE 4 / 5).  Both equal the
    incremental checker in full and the direct oracle on sampled columns, across a ragged third
    chunk, with lazy (p < 2^62) and exact (p >= 2^62) chains."""
    w = synth.random_small(590 + p % 97, p, 7, 3000, 5, 2 * 8192 + 777, 11)
    with pe.Context.from_workload(w, path=pe.PATH_TC, tc_form=form) as ctx:
        assert ctx.tc_form() == form
        out = ctx.eval(w.j0, w.T)
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, ref)
    ks = np.array([0, 8191, 8192, w.T - 1], np.uint64)
    assert np.array_equal(out[:, ks.astype(np.int64)], oracle.eval_workload(w, ks=ks))


def test_tc_form_defaults_and_limits(monkeypatch):
    """Automatic = swapped for 8-digit primes, plain for 7-digit ones (PE_TC_SWAP=0/1 overrides);
    7-digit primes may request the swapped form; the 4-digit mode (p < 2^31) has only the plain
    form (a request for the swapped one builds it); out-of-range tc_form values are PE_EINVAL."""
    monkeypatch.delenv("PE_TC_SWAP", raising=False)
    w = synth.random_small(599, P62, 5, 300, 3, 100, 1)
    with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
        assert ctx.tc_form() == pe.TC_FORM_SWAPPED
    monkeypatch.setenv("PE_TC_SWAP", "0")
    with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
        assert ctx.tc_form() == pe.TC_FORM_PLAIN
    with pe.Context.from_workload(w, path=pe.PATH_TC, tc_form=pe.TC_FORM_SWAPPED) as ctx:
        assert ctx.tc_form() == pe.TC_FORM_SWAPPED   # an explicit request beats the env override
    monkeypatch.delenv("PE_TC_SWAP", raising=False)
    w2 = synth.random_small(598, (1 << 50) - 27, 5, 300, 3, 100, 1)     # 7 digits: both forms exist
    for form in (pe.TC_FORM_AUTO, pe.TC_FORM_SWAPPED):
        with pe.Context.from_workload(w2, path=pe.PATH_TC, tc_form=form) as ctx:
            assert ctx.tc_form() == (pe.TC_FORM_SWAPPED if form == pe.TC_FORM_SWAPPED else pe.TC_FORM_PLAIN)
            assert np.array_equal(ctx.eval(w2.j0, w2.T), oracle.eval_workload(w2))
    w3 = synth.random_small(597, (1 << 31) - 1, 5, 300, 3, 100, 1)      # 4 digits: plain only
    with pe.Context.from_workload(w3, path=pe.PATH_TC, tc_form=pe.TC_FORM_SWAPPED) as ctx:
        assert ctx.tc_form() == pe.TC_FORM_PLAIN
        assert np.array_equal(ctx.eval(w3.j0, w3.T), oracle.eval_workload(w3))
    with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
        assert ctx.tc_form() == 0
    with pytest.raises(pe.PEError) as e:
        pe.Context.from_workload(w, tc_form=3)
    assert e.value.code == -1


def test_auto_form_falls_back_to_plain_when_memory_is_short(monkeypatch):
    """An automatic handle whose swapped-form planes (1 KB per term) exceed PE_TC_MEM_MB but whose
    plain-form planes (256 B per term) fit gets the plain form -- same bits, checked against the
    oracle; a cap below both leaves it on k_step."""
    monkeypatch.delenv("PE_TC_SWAP", raising=False)
    w = synth.gen_config(3)   # 10^6 terms: swapped ~1.1 GB, plain ~0.36 GB of tensor-path memory
    ks = np.array([0, 1, 777, w.T - 1], np.uint64)
    ref = oracle.eval_workload(w, ks=ks)
    monkeypatch.setenv("PE_TC_MEM_MB", "600")
    with pe.Context.from_workload(w) as ctx:
        assert ctx.tc_form() == pe.TC_FORM_PLAIN and ctx.uses_tc(w.T)
        out = ctx.eval(w.j0, w.T)
    assert np.array_equal(out[:, ks.astype(np.int64)], ref)
    monkeypatch.setenv("PE_TC_MEM_MB", "100")
    with pe.Context.from_workload(w) as ctx:
        assert ctx.tc_form() == 0 and not ctx.uses_tc(w.T)
        out = ctx.eval(w.j0, w.T)
    assert np.array_equal(out[:, ks.astype(np.int64)], ref)


@pytest.mark.parametrize("pad,direct,cap_mb", [(13, "1", 0), (14, "1", 0), (0, "0", 0), (6, "1", 8)])
def test_tc_direct_rows_ld_and_padding(monkeypatch, pad, direct, cap_mb):
    """k_tc writes a bucket's sole piece straight into its output row when the rows keep 16-B
    alignment (even ld, aligned base) -- an odd ld (pad 13) or PE_TC_DIRECT=0 sends every row
    through the fix-up instead.  Either way the result equals the oracle, padding columns stay
    untouched, and a ragged multi-pass range (partial-buffer cap) splits passes at chunk
    boundaries of the output row."""
    import torch
    monkeypatch.setenv("PE_TC_DIRECT", direct)
    if cap_mb:
        monkeypatch.setenv("PE_PARTIAL_MB", str(cap_mb))   # one 4096-point chunk per pass: 2 passes
    w = synth.gen_config(2, t=60_000, T=5000)      # buckets of one piece and of several
    ks = np.array([0, 1, 2047, 4095, 4096, 4999], np.uint64)
    ref = oracle.eval_workload(w, ks=ks)
    with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
        G, T = ctx.G, w.T
        assert ctx.info()["tc_pieces"] >= G
        buf = torch.full((G, T + pad), -1, dtype=torch.int64, device="cuda")
        ctx.eval_device(w.j0, T, buf.data_ptr(), T + pad)
        torch.cuda.synchronize()
    got = buf.cpu().numpy().view(np.uint64)
    assert np.array_equal(got[:, ks.astype(np.int64)], ref)
    if pad:
        assert np.all(got[:, T:] == np.uint64(2**64 - 1))
