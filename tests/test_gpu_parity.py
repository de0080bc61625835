"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
on the same seeded inputs.  Bit-exact: results are canonical
residues, unique (reading R14)."""
import os

import numpy as np
import pytest

import oracle
import paper_2004_11571_b200 as pe
import synth

pytestmark = pytest.mark.gpu

P62, P50 = synth.P62, synth.P50


def gpu_eval(w, j0=None, T=None, **kw):
    with pe.Context.from_workload(w, **kw) as ctx:
        out = ctx.eval(w.j0 if j0 is None else j0, w.T if T is None else T)
        rows = ctx.buckets()
    return rows, out


def check_full(w, **kw):
    rows, out = gpu_eval(w, **kw)
    assert rows.tolist() == oracle.buckets(w.exps, w.n).tolist()
    ref = oracle.eval_workload(w)
    assert out.shape == ref.shape
    bad = np.argwhere(out != ref)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"
    return out


# ---------------------------------------------------------------- BASELINE configs
def test_config1_full():
    check_full(synth.gen_config(1))


def test_config2_full():
    check_full(synth.gen_config(2))


@pytest.mark.parametrize("cfg,path", [(3, pe.PATH_AUTO), (3, pe.PATH_INT), (4, pe.PATH_AUTO), (4, pe.PATH_FP64)])
def test_config3_4_full_incremental_and_sampled_direct(cfg, path):
    """Configs 3 and 4 in full: PATH_AUTO takes the tensor-core form (T = 4096 >= the threshold),
    PATH_INT / PATH_FP64 the scalar Shoup / FP64 Alg. 2 k_step."""
    w = synth.gen_config(cfg)
    with pe.Context.from_workload(w, path=path) as ctx:
        assert ctx.uses_tc(w.T) == (path == pe.PATH_AUTO)
    rows, out = gpu_eval(w, path=path)
    assert rows.tolist() == oracle.buckets(w.exps, w.n).tolist()
    inc = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, inc)
    ks = np.array([0, 1, 31, 32, 1023, 1024, 2047, 4095], np.uint64)
    ref = oracle.eval_workload(w, ks=ks)
    assert np.array_equal(out[:, ks.astype(np.int64)], ref)


def test_config4_fp64_equals_int():
    w = synth.gen_config(4, t=200_000, T=512)
    _, a = gpu_eval(w, path=pe.PATH_FP64)
    _, b = gpu_eval(w, path=pe.PATH_INT)
    assert np.array_equal(a, b)
    ref = oracle.eval_workload(w, ks=np.arange(0, 512, 37, dtype=np.uint64))
    assert np.array_equal(a[:, 0:512:37], ref)


@pytest.fixture(scope="module")
def config5_ref():
    """BASELINE config 5 (t = 10^7, T = 16384) and its FULL G x T output from the Alg. 1 checker
    (PAPER.md:505-534), blocked over (row, 512-point block) tasks so the Zipf-skewed rows spread
    over the host cores; about 1.6e11 checker products."""
    w = synth.gen_config(5)
    full = oracle.eval_incremental_blocked(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T, block=512)
    return w, full


@pytest.mark.parametrize("path,compact,form", [(pe.PATH_AUTO, False, pe.TC_FORM_AUTO), (pe.PATH_INT, False, pe.TC_FORM_AUTO),
                                              (pe.PATH_AUTO, True, pe.TC_FORM_AUTO), (pe.PATH_TC, False, pe.TC_FORM_PLAIN)])
def test_config5_full(path, compact, form, config5_ref):
    """Full size in the bench launch configuration (PATH_AUTO = the tensor-core k_tc in its default
    swapped form; PATH_TC + TC_FORM_PLAIN = its plain form; PATH_INT = the scalar k_step; compact =
    the uint8-exponent entry pe_create_compact), compared over the WHOLE G x T output with the
    incremental checker, plus columns against the direct definition -- chosen to hit every TMEM lane
    quarter (u = 0..127 in groups of 32) of the four 4096-point chunks (128 x 32 points, the V = 32
    geometry of p >= 2^54), the chunk edges and v = 0 / 31."""
    w, full = config5_ref
    with pe.Context.from_workload(w, path=path, compact=compact, tc_form=form) as ctx:
        assert ctx.uses_tc(w.T) == (path != pe.PATH_INT)
        if path != pe.PATH_INT:
            assert ctx.tc_form() == (pe.TC_FORM_PLAIN if form == pe.TC_FORM_PLAIN else pe.TC_FORM_SWAPPED)
        out = ctx.eval(w.j0, w.T)
        rows = ctx.buckets()
    assert rows.tolist() == oracle.buckets(w.exps, w.n).tolist()
    bad = np.argwhere(out != full)
    assert bad.size == 0, f"{len(bad)} mismatches vs the incremental checker, first {bad[:5].tolist()}"
    ks = np.array(sorted({0, 1, 31, 32, 777, 4095, 4096, 8191, 8192, 12345, 16382, 16383}
                         | {c * 4096 + u * 32 + v for c in range(4) for u in (5, 40, 77, 120) for v in (0, 17) if (u + v + c) % 2}
                         | {c * 4096 + u * 32 + 31 for c in (0, 3) for u in (31, 32, 95, 96)}), np.uint64)
    ref = oracle.eval_workload(w, ks=ks)
    assert np.array_equal(out[:, ks.astype(np.int64)], ref)


# ---------------------------------------------------------------- tuning invariance (P13)
@pytest.mark.parametrize("R,warps,chunk", [(1, 8, 0), (2, 4, 32), (4, 16, 64), (8, 1, 96), (16, 8, 0),
                                           (8, 8, 0), (16, 2, 32)])
def test_tuning_invariance(R, warps, chunk):
    w = synth.gen_config(2, t=20_000, T=161)
    ref = oracle.eval_workload(w)
    _, out = gpu_eval(w, R=R, warps=warps, chunk=chunk)
    assert np.array_equal(out, ref)


def test_multi_pass_partial_buffer(monkeypatch):
    monkeypatch.setenv("PE_PARTIAL_MB", "1")            # forces several point passes
    w = synth.gen_config(3, t=50_000, T=700)
    rows, out = gpu_eval(w, R=1)
    ref = oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    assert np.array_equal(out, ref)


def test_eval_device_ld_and_stream():
    import torch
    w = synth.gen_config(1)
    ref = oracle.eval_workload(w)
    G, T = ref.shape
    s = torch.cuda.Stream()
    buf = torch.full((G, T + 13), -1, dtype=torch.int64, device="cuda")
    with pe.Context.from_workload(w) as ctx:
        ctx.eval_device(w.j0, T, buf.data_ptr(), T + 13, s.cuda_stream)
        s.synchronize()
    got = buf.cpu().numpy().view(np.uint64)
    assert np.array_equal(got[:, :T], ref)
    assert np.all(got[:, T:] == np.uint64(2**64 - 1))     # padding columns untouched


# ---------------------------------------------------------------- edge cases
@pytest.mark.parametrize("p,n,t,maxdeg,j0,T", [
    (P62, 6, 300, 4, 1, 1),              # T = 1
    (P62, 6, 300, 4, 1, 33),             # ragged vs the 32-point super-group
    (P62, 5, 500, 3, 0, 70),             # j0 = 0 (beta^0)
    (P62, 5, 200, 3, 2**64 - 40, 40),    # largest j range
    (13, 4, 60, 3, 0, 50),               # tiny prime (unlucky-point size)
    (3, 5, 40, 2, 5, 20),                # smallest prime
    ((1 << 63) - 25, 6, 400, 3, 7, 45),  # INT lazy-2 path (p >= 2^62)
    (P50, 7, 600, 4, 3, 77),             # FP64 path
    (2**31 - 1, 3, 100, 9, 1, 64),       # n = 3
    (1009, 2, 50, 6, 1, 10),             # n = 2 (nothing evaluated)
])
def test_edge_shapes(p, n, t, maxdeg, j0, T):
    w = synth.random_small(100 + t + n, p, n, t, maxdeg, T, j0, coeff_hi=2**64 - 1)
    check_full(w)


def test_single_term_and_single_bucket():
    w = synth.random_small(201, P62, 5, 1, 3, 40, 1)
    check_full(w)
    w = synth.random_small(202, P62, 6, 700, 4, 40, 1)
    w.exps[:, :2] = 3                                         # G = 1
    check_full(w)


def test_duplicates_zero_coeffs_alpha_ge_p():
    w = synth.random_small(203, P62, 5, 400, 2, 50, 1, dup=True)
    w.coeffs[::7] = 0
    w.coeffs[1::11] = np.uint64(P62 + 5)
    w.alpha = (w.alpha + np.uint64(P62)).astype(np.uint64)    # alpha >= p, reduced by the callee
    check_full(w)


def test_fermat_periodicity_gpu():
    w = synth.random_small(204, P62, 6, 500, 3, 64, 1)
    _, a = gpu_eval(w, j0=1)
    _, b = gpu_eval(w, j0=1 + (P62 - 1))
    assert np.array_equal(a, b)


def test_empty_polynomial_and_T0():
    with pe.Context(P62, np.zeros(0, np.uint64), np.zeros((0, 4), np.uint32), [2, 3], n=4) as ctx:
        assert ctx.G == 0
        assert ctx.eval(1, 5).shape == (0, 5)
    w = synth.gen_config(1)
    with pe.Context.from_workload(w) as ctx:
        assert ctx.eval(1, 0).shape == (ctx.G, 0)


def test_monomials_match_python():
    w = synth.random_small(205, P62, 7, 3000, 5, 1, 1, dup=True)
    with pe.Context.from_workload(w) as ctx:
        m = ctx.monomials()
    for i in range(0, 3000, 17):
        v = 1
        for a, e in zip(w.alpha, w.exps[i, 2:]):
            v = v * pow(int(a), int(e), P62) % P62
        assert int(m[i]) == v


def test_large_exponents_no_power_table():
    """Exponents beyond the power-table limit take the direct-power branch of k_setup."""
    w = synth.random_small(206, P62, 4, 200, 3, 20, 1)
    w.exps[::3, 2] = np.uint32(3_000_000)
    w.exps[1::5, 3] = np.uint32(4_000_000_000)
    check_full(w)


def test_error_codes_gpu():
    with pytest.raises(pe.PEError) as ei:
        pe.Context(15, [1], [[0, 0, 1]], [2])
    assert ei.value.code == pe.PE_ENOTPRIME
    w = synth.gen_config(1)
    with pe.Context.from_workload(w) as ctx:
        with pytest.raises(pe.PEError) as ei:
            ctx.eval(2**64 - 10, 20)
        assert ei.value.code == pe.PE_ERANGE


def test_shoup_core_parity_50bit(monkeypatch):
    """PE_CORE=shoup on a 50-bit prime (config 4 shape) equals the FP64 Alg. 2 default."""
    monkeypatch.setenv("PE_CORE", "shoup")
    check_full(synth.gen_config(4, t=20_000, T=70))


# ---------------------------------------------------------------- NEXT-1: batched polynomials
def test_batch_polys_same_points():
    """pe_create_batch: f_0..f_3 at the same beta^j (PAPER.md:367-392 gcd images); rows per
    polynomial equal separate single-polynomial oracle evaluations."""
    p, n, T, j0 = P62, 6, 45, 1
    rng = np.random.default_rng(301)
    alpha = rng.integers(1, p, n - 2, dtype=np.uint64)
    polys = []
    for seed, t in ((302, 400), (303, 0), (304, 1), (305, 250)):
        w = synth.random_small(seed, p, n, t, 3, T, j0) if t else None
        polys.append((w.coeffs, w.exps) if w else (np.zeros(0, np.uint64), np.zeros((0, n), np.uint32)))
    # neighbouring polynomials sharing a key at the boundary: last key of f_2 == first key of f_3
    polys[2] = (polys[2][0], polys[2][1].copy())
    polys[2][1][0, :2] = polys[3][1][:, :2].max(axis=0)
    with pe.Context.batch(p, polys, alpha, n) as ctx:
        rows_off = ctx.poly_rows().astype(np.int64)
        out = ctx.eval(j0, T)
        rows = ctx.buckets()
    assert rows_off[0] == 0 and rows_off[-1] == out.shape[0] and len(rows_off) == len(polys) + 1
    for k, (c, e) in enumerate(polys):
        a, b = rows_off[k], rows_off[k + 1]
        if c.size == 0:
            assert a == b
            continue
        ref = oracle.eval_direct(p, n, c, e, alpha, j0, T)
        assert rows[a:b].tolist() == oracle.buckets(e, n).tolist(), k
        assert np.array_equal(out[a:b], ref), k


def test_batch_config3_pair():
    """f and h of config-3 shape (10^5 terms each) in one launch."""
    f = synth.gen_config(3, t=100_000, T=200)
    h = synth.gen_config(3, t=100_000, T=200, seed=99)
    with pe.Context.batch(f.p, [(f.coeffs, f.exps), (h.coeffs, h.exps)], f.alpha, f.n) as ctx:
        ro = ctx.poly_rows().astype(np.int64)
        out = ctx.eval(f.j0, f.T)
    inc_f = oracle.eval_incremental(f.p, f.n, f.coeffs, f.exps, f.alpha, f.j0, f.T)
    inc_h = oracle.eval_incremental(f.p, f.n, h.coeffs, h.exps, f.alpha, f.j0, f.T)
    assert np.array_equal(out[ro[0]:ro[1]], inc_f) and np.array_equal(out[ro[1]:ro[2]], inc_h)


# ---------------------------------------------------------------- NEXT-3: 32-bit primes
@pytest.mark.parametrize("p,R", [((1 << 31) - 1, 16), ((1 << 31) - 1, 8), (2_147_483_629, 4), (65_521, 2),
                                 (3, 1), (1_000_003, 16)])
def test_int32_path_parity(p, R):
    """p < 2^31 -> 32-bit Shoup products (pe_info path 'int32'), bit-exact vs the oracle."""
    w = synth.gen_config(3, t=40_000, T=77)
    w.p = p
    w.alpha = synth.uniform_mod(np.random.default_rng(p), 1, p, w.n - 2)
    with pe.Context.from_workload(w, R=R) as ctx:
        assert ctx.info()["path"] == "int32"
    check_full(w, R=R)


def test_int32_equals_int64_core():
    """Same 31-bit instance through the 32-bit path and (PE_CORE=shoup) the 64-bit Shoup path."""
    w = synth.random_small(310, (1 << 31) - 1, 7, 2000, 4, 66, 5, coeff_hi=2**64 - 1)
    _, a = gpu_eval(w)
    os.environ["PE_CORE"] = "shoup"
    try:
        _, b = gpu_eval(w)
    finally:
        del os.environ["PE_CORE"]
    assert np.array_equal(a, b)
