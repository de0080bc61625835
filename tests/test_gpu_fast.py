"""The asymptotically fast method (PE_PATH_FAST, csrc/fast.cu, PAPER.md:
578-591): per bucket the T outputs are the first T coefficients of sum_i a_i / (1 - m_i z), built by
a product tree + Newton inversion with NTT/CRT products.  Same canonical residues as the matrix
method, so it is compared element by element with the CPU oracle (direct definition or the Alg. 1
checker) on the shapes that exercise each of its regimes."""
import numpy as np
import pytest

import oracle
import paper_2004_11571_b200 as pe
import synth

pytestmark = pytest.mark.gpu

P62 = synth.P62


def fast_eval(w, j0=None, T=None):
    with pe.Context.from_workload(w, path=pe.PATH_FAST) as ctx:
        T = w.T if T is None else T
        assert ctx.eval_kernel(T) == "fast"
        out = ctx.eval(w.j0 if j0 is None else j0, T)
        rows = ctx.buckets()
    return rows, out


def check_direct(w):
    rows, out = fast_eval(w)
    assert rows.tolist() == oracle.buckets(w.exps, w.n).tolist()
    ref = oracle.eval_workload(w)
    bad = np.argwhere(out != ref)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"


def check_incremental(w):
    _, out = fast_eval(w)
    ref = oracle.eval_incremental_blocked(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T)
    bad = np.argwhere(out != ref)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"


@pytest.mark.parametrize("p,n,t,maxdeg,j0,T", [
    (P62, 6, 300, 4, 1, 1),                # T = 1: N(0) = sum of the seeds
    (P62, 6, 300, 4, 1, 2),
    (P62, 6, 300, 4, 1, 33),               # ragged: T2 = 64
    (P62, 5, 500, 3, 0, 70),               # j0 = 0
    (P62, 5, 200, 3, 2**64 - 40, 40),      # seeds with 64-bit exponents
    (13, 4, 60, 3, 0, 50),                 # tiny prime (smaller than every NTT prime)
    (3, 5, 40, 2, 5, 20),                  # smallest prime
    (P62, 2, 30, 6, 1, 10),                # n = 2: m = 1, D = (1 - z)^s
    (2**31 - 1, 3, 100, 9, 1, 64),
    ((1 << 50) - 27, 7, 600, 4, 3, 77),
    ((1 << 62) - 87, 6, 700, 4, 5, 300),
    ((1 << 62) + 135, 5, 400, 3, 1, 129),   # just above 2^62
    ((1 << 63) - 25, 6, 700, 4, 5, 300),    # largest supported p: 2 L p^2 < 2^147 < prod q_j
    (P62, 6, 300, 4, 1, 4097),             # T2 = 8192: the first block-convolved length
    (P62, 6, 5000, 4, 1, 2048),            # buckets longer than T2 (truncated upper levels)
])
def test_fast_edge_shapes(p, n, t, maxdeg, j0, T):
    check_direct(synth.random_small(800 + t + n, p, n, t, maxdeg, T, j0, coeff_hi=2**64 - 1))


def test_fast_configs_1_2():
    check_direct(synth.gen_config(1))
    check_direct(synth.gen_config(2))


def test_fast_config3_full():
    """T = 4096: the largest single-block product (8192-point transforms)."""
    check_incremental(synth.gen_config(3))


def test_fast_block_convolution():
    """T = 3 x 4096 + 5 (T2 = 16384): operands longer than one 4096-coefficient block, so products
    are block-pairwise transform-domain convolutions with overlap-add; 10^5 terms in ~200 buckets."""
    check_incremental(synth.gen_config(2, t=100_000, T=3 * 4096 + 5))


def test_fast_deep_tree_truncated():
    """One bucket of 50 000 terms with T = 1000: the tree runs 11 levels past T2 = 1024, so every
    upper product is truncated mod z^T2; plus singleton and 33-term buckets."""
    w = synth.random_small(821, P62, 8, 50_034, 5, 1000, 1)
    w.exps[:, :2] = 4
    w.exps[0, :2] = (9, 9)
    w.exps[1:34, :2] = (0, 1)
    check_incremental(w)


def test_fast_duplicates_zero_coeffs_alpha_ge_p():
    w = synth.random_small(822, P62, 5, 400, 2, 50, 1, dup=True)
    w.coeffs[::7] = 0
    w.coeffs[1::11] = np.uint64(P62 + 5)
    w.alpha = (w.alpha + np.uint64(P62)).astype(np.uint64)
    check_direct(w)


def test_fast_equals_tc_and_step():
    """The three hot kernels agree bit for bit on one instance (T = 9000: two k_tc chunks)."""
    w = synth.gen_config(2, t=20_000, T=9000)
    _, f = fast_eval(w)
    with pe.Context.from_workload(w, path=pe.PATH_TC) as ctx:
        t = ctx.eval(w.j0, w.T)
    with pe.Context.from_workload(w, path=pe.PATH_INT) as ctx:
        s = ctx.eval(w.j0, w.T)
    assert np.array_equal(f, t) and np.array_equal(f, s)


def test_fast_limits():
    w = synth.random_small(824, P62, 5, 50, 3, 10, 1)
    with pe.Context.from_workload(w, path=pe.PATH_FAST) as ctx:
        with pytest.raises(pe.PEError) as ei:
            ctx.eval(1, (1 << 20) + 1)
        assert ei.value.code == pe.PE_ERANGE


def test_fast_automatic_choice_without_tensor_path(monkeypatch):
    """With the tensor-core form off (PE_TC=0), an automatic handle takes the fast method for
    T >= 8192 when buckets hold >= 2048 terms on average (its measured crossover with k_step,
    profiles/r02_fast_sweep_config3.jsonl), and k_step otherwise; bit-exact either way."""
    monkeypatch.setenv("PE_TC", "0")
    w = synth.gen_config(3, t=300_000, T=8192)             # 256 buckets of ~1170 terms: k_step
    with pe.Context.from_workload(w) as ctx:
        assert ctx.eval_kernel(w.T) == "k_step"
    w = synth.gen_config(3, t=600_000, T=8192)             # ~2340 terms per bucket: fast from T = 8192
    w.exps[:, :2] %= np.uint32(14)                         # 196 buckets
    with pe.Context.from_workload(w) as ctx:
        assert ctx.eval_kernel(8191) == "k_step" and ctx.eval_kernel(w.T) == "fast"
        out = ctx.eval(w.j0, w.T)
    ks = np.array([0, 1, 4097, 8191], np.uint64)
    assert np.array_equal(out[:, ks.astype(np.int64)], oracle.eval_workload(w, ks=ks))


def test_fast_batched_polynomials():
    """pe_create_batch with the fast method: f and h of config-3 shape at the same points (the gcd
    workload), rows per polynomial equal to the incremental checker."""
    f = synth.gen_config(3, t=60_000, T=3000)
    h = synth.gen_config(3, t=40_000, T=3000, seed=77)
    with pe.Context.batch(f.p, [(f.coeffs, f.exps), (h.coeffs, h.exps)], f.alpha, f.n, path=pe.PATH_FAST) as ctx:
        assert ctx.eval_kernel(f.T) == "fast"
        ro = ctx.poly_rows().astype(np.int64)
        out = ctx.eval(f.j0, f.T)
    inc_f = oracle.eval_incremental(f.p, f.n, f.coeffs, f.exps, f.alpha, f.j0, f.T)
    inc_h = oracle.eval_incremental(f.p, f.n, h.coeffs, h.exps, f.alpha, f.j0, f.T)
    assert np.array_equal(out[ro[0]:ro[1]], inc_f) and np.array_equal(out[ro[1]:ro[2]], inc_h)
