"""Pins for the CPU oracle (DESIGN.md "Oracle pins" P1-P12) -- CPU only.

The oracle (oracle/oracle.c) is checked against things other than itself: values printed in
the paper/SPEC (tests/golden/, cited per case), closed forms, invariants that the
mathematics fixes, and a Python big-integer brute force (oracle/brute.py) written without
any modular shortcut.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle.brute import brute_eval
import synth
from conftest import GOLDEN

P62, P50 = synth.P62, synth.P50


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _rows_ref(exps):
    """Row order fixed by DESIGN.md reading R2: distinct (dx,dy), descending lex."""
    return sorted({(int(r[0]), int(r[1])) for r in exps}, reverse=True)


# ---------------------------------------------------------------- P1, P2: SPEC worked examples
def test_spec_worked_examples():
    g = _golden("spec_worked_examples.json")
    for case in g["cases"]:
        rows = oracle.buckets(np.array(case["exps"]), case["n"])
        assert rows.tolist() == case["rows"], case["pin"]
        for j, want in case["points"].items():
            out = oracle.eval_direct(case["p"], case["n"], case["coeffs"], case["exps"], case["alpha"],
                                     int(j), 1)
            assert out[:, 0].tolist() == want, (case["pin"], j)
            _, bout = brute_eval(case["p"], case["n"], case["coeffs"], case["exps"], case["alpha"], int(j), 1)
            assert [r[0] for r in bout] == want, (case["pin"], "brute", j)
    for s in g["scalar"]:
        fn = {"powmod": oracle.powmod, "mulmod": oracle.mulmod}[s["op"]]
        assert fn(*s["args"]) == s["value"], s["pin"]


# ---------------------------------------------------------------- P3: closed forms at config primes
def test_closed_forms_config_primes():
    g = _golden("closed_forms_config_primes.json")
    for c in g["cases"]:
        out = oracle.eval_direct(c["p"], 3, [1], [[0, 0, 1]], [2], c["j"], 1)
        assert int(out[0, 0]) == c["value"], c
        assert oracle.powmod(2, c["j"], c["p"]) == c["value"]
        # sampled mode gives the same column
        out2 = oracle.eval_direct(c["p"], 3, [1], [[0, 0, 1]], [2], c["j"] - 5, ks=[5])
        assert int(out2[0, 0]) == c["value"]


# ---------------------------------------------------------------- P10, P11: paper / hand examples
def test_unlucky_point():
    g = _golden("paper_unlucky_point.json")
    out = oracle.eval_direct(g["p"], g["n"], g["coeffs"], g["exps"], g["alpha"], g["j0"], g["T"])
    assert out.tolist() == g["out"]
    assert out[0, 0] == 0                                     # vanishes at beta^0


def test_hand_example_p13():
    g = _golden("hand_example_p13.json")
    assert oracle.buckets(np.array(g["exps"]), g["n"]).tolist() == g["rows"]
    out = oracle.eval_direct(g["p"], g["n"], g["coeffs"], g["exps"], g["alpha"], g["j0"], g["T"])
    assert out.T.tolist() == g["out_by_point"]
    inc = oracle.eval_incremental(g["p"], g["n"], g["coeffs"], g["exps"], g["alpha"], g["j0"], g["T"])
    assert inc.T.tolist() == g["out_by_point"]


# ---------------------------------------------------------------- brute force on random tiny inputs
@pytest.mark.parametrize("p,n,t,maxdeg,j0,T", [
    (13, 4, 12, 3, 0, 6), (101, 5, 30, 3, 1, 5), (2**31 - 1, 4, 20, 4, 3, 4),
    (P62, 5, 15, 3, 1, 3), (P50, 3, 10, 5, 7, 3), (7, 2, 9, 4, 0, 3), (3, 6, 25, 2, 1, 4),
])
def test_oracle_vs_bruteforce(p, n, t, maxdeg, j0, T):
    w = synth.random_small(1000 + p % 997 + n, p, n, t, maxdeg, T, j0, dup=True, coeff_hi=2 * p)
    rows, bout = brute_eval(p, n, w.coeffs, w.exps, w.alpha, j0, T)
    assert oracle.buckets(w.exps, n).tolist() == [list(r) for r in rows]
    out = oracle.eval_direct(p, n, w.coeffs, w.exps, w.alpha, j0, T)
    assert out.tolist() == bout


# ---------------------------------------------------------------- P4: j = 0 -> coefficient sums
@pytest.mark.parametrize("seed,p,n", [(1, P62, 6), (2, P50, 9), (3, 1009, 4)])
def test_j0_gives_coefficient_sums(seed, p, n):
    w = synth.random_small(seed, p, n, 300, 4, 1, 0, coeff_hi=(1 << 64) - 1)   # coefficients >= p too
    rows = _rows_ref(w.exps)
    want = {r: 0 for r in rows}
    for c, e in zip(w.coeffs, w.exps):
        want[(int(e[0]), int(e[1]))] += int(c)
    out = oracle.eval_direct(p, n, w.coeffs, w.exps, w.alpha, 0, 1)
    assert out[:, 0].tolist() == [want[r] % p for r in rows]


# ---------------------------------------------------------------- P5: Fermat periodicity
def test_fermat_periodicity_large_exponents():
    w = synth.random_small(5, P62, 5, 40, 3, 3, 1)
    a = oracle.eval_direct(P62, 5, w.coeffs, w.exps, w.alpha, 1, 3)
    b = oracle.eval_direct(P62, 5, w.coeffs, w.exps, w.alpha, 1 + (P62 - 1), 3)
    c = oracle.eval_direct(P62, 5, w.coeffs, w.exps, w.alpha, 1 + 3 * (P62 - 1), 3)   # j ~ 2^63.6
    assert np.array_equal(a, b) and np.array_equal(a, c)


# ---------------------------------------------------------------- P6: linearity
def test_linearity():
    f = synth.random_small(6, P62, 6, 200, 3, 5, 1)
    g = synth.random_small(7, P62, 6, 150, 3, 5, 1)
    g.alpha = f.alpha
    fg_c = np.concatenate([f.coeffs, g.coeffs])
    fg_e = np.concatenate([f.exps, g.exps])               # duplicates allowed (reading R7)
    of = oracle.eval_direct(P62, 6, f.coeffs, f.exps, f.alpha, 1, 5)
    og = oracle.eval_direct(P62, 6, g.coeffs, g.exps, f.alpha, 1, 5)
    ofg = oracle.eval_direct(P62, 6, fg_c, fg_e, f.alpha, 1, 5)
    rf = {tuple(r): i for i, r in enumerate(oracle.buckets(f.exps, 6).tolist())}
    rg = {tuple(r): i for i, r in enumerate(oracle.buckets(g.exps, 6).tolist())}
    for i, r in enumerate(oracle.buckets(fg_e, 6).tolist()):
        r = tuple(r)
        s = [0] * 5
        if r in rf:
            s = [x + int(y) for x, y in zip(s, of[rf[r]])]
        if r in rg:
            s = [x + int(y) for x, y in zip(s, og[rg[r]])]
        assert [x % P62 for x in s] == ofg[i].tolist()


# ---------------------------------------------------------------- P7: incremental == direct
@pytest.mark.parametrize("seed,p,n,j0,T", [(8, P62, 6, 1, 20), (9, P50, 9, 0, 17), (10, 13, 4, 5, 9),
                                           (11, (1 << 63) - 25, 5, 2**40, 6)])
def test_incremental_equals_direct(seed, p, n, j0, T):
    w = synth.random_small(seed, p, n, 400, 5, T, j0)
    d = oracle.eval_direct(p, n, w.coeffs, w.exps, w.alpha, j0, T)
    i = oracle.eval_incremental(p, n, w.coeffs, w.exps, w.alpha, j0, T)
    assert np.array_equal(d, i)
    for block in (1, 4, T, T + 3):       # the blocked checker (re-seeded per block) is the same
        assert np.array_equal(d, oracle.eval_incremental_blocked(p, n, w.coeffs, w.exps, w.alpha, j0, T, block))


def _m_python(alpha, e, p):
    v = 1
    for a, k in zip(alpha, e):
        v = v * pow(int(a), int(k), p) % p
    return v


# ---------------------------------------------------------------- P8: single-term bucket progression
def test_single_term_geometric_progression():
    w = synth.random_small(12, P62, 7, 60, 6, 12, 3)
    out = oracle.eval_direct(P62, 7, w.coeffs, w.exps, w.alpha, 3, 12)
    rows = oracle.buckets(w.exps, 7).tolist()
    keys = [(int(e[0]), int(e[1])) for e in w.exps]
    checked = 0
    for g, r in enumerate(rows):
        members = [i for i, k in enumerate(keys) if k == tuple(r)]
        if len(members) != 1:
            continue
        m = _m_python(w.alpha, w.exps[members[0], 2:], P62)
        for k in range(11):
            assert int(out[g, k + 1]) == int(out[g, k]) * m % P62
        checked += 1
    assert checked > 5


# ---------------------------------------------------------------- P9: linear recurrence per bucket
def _poly_from_roots(roots, p):
    c = [1]
    for r in roots:                      # multiply by (z - r)
        nc = [0] * (len(c) + 1)
        for i, a in enumerate(c):
            nc[i + 1] = (nc[i + 1] + a) % p
            nc[i] = (nc[i] - a * r) % p
        c = nc
    return c                             # c[k] = coefficient of z^k


def test_linear_recurrence_annihilator():
    p, n, T = 1_000_003, 5, 14
    w = synth.random_small(13, p, n, 40, 3, T, 1)
    w.exps[:, 0] = np.arange(40) % 6                    # 6 buckets of <= 7 terms
    w.exps[:, 1] = 0
    out = oracle.eval_direct(p, n, w.coeffs, w.exps, w.alpha, 1, T)
    rows = oracle.buckets(w.exps, n).tolist()
    for g, r in enumerate(rows):
        ms = sorted({_m_python(w.alpha, w.exps[i, 2:], p) for i in range(40) if int(w.exps[i, 0]) == r[0]})
        lam = _poly_from_roots(ms, p)
        for s in range(T - len(ms)):
            assert sum(lam[k] * int(out[g, s + k]) for k in range(len(lam))) % p == 0


# ---------------------------------------------------------------- degenerate shapes
def test_n2_and_empty():
    w = synth.random_small(14, 101, 2, 30, 5, 4, 1, dup=True, coeff_hi=1000)
    out = oracle.eval_direct(101, 2, w.coeffs, w.exps, w.alpha, 1, 4)
    want = {}
    for c, e in zip(w.coeffs, w.exps):
        want[(int(e[0]), int(e[1]))] = want.get((int(e[0]), int(e[1])), 0) + int(c)
    rows = _rows_ref(w.exps)
    for k in range(4):
        assert out[:, k].tolist() == [want[r] % 101 for r in rows]
    e = oracle.eval_direct(101, 4, np.zeros(0, np.uint64), np.zeros((0, 4), np.uint32), [2, 3], 1, 4)
    assert e.shape == (0, 4)


def test_duplicates_equal_merged():
    w = synth.random_small(15, P62, 5, 50, 2, 4, 1)
    dup_e = np.concatenate([w.exps, w.exps[:10]])
    dup_c = np.concatenate([w.coeffs, w.coeffs[:10]])
    merged_c = w.coeffs.copy()
    merged_c[:10] = [(2 * int(c)) % P62 for c in w.coeffs[:10]]
    a = oracle.eval_direct(P62, 5, dup_c, dup_e, w.alpha, 1, 4)
    b = oracle.eval_direct(P62, 5, merged_c, w.exps, w.alpha, 1, 4)
    assert np.array_equal(a, b)


def test_scalar_core_random():
    rng = np.random.default_rng(16)
    for p in (P62, P50, (1 << 63) - 25, 13):
        for _ in range(200):
            a, b = (int(x) for x in rng.integers(0, 1 << 63, 2, dtype=np.uint64))
            e = int(rng.integers(0, 1 << 62))
            assert oracle.mulmod(a, b, p) == a * b % p
            assert oracle.powmod(a, e, p) == pow(a, e, p)


# ---------------------------------------------------------------- Berlekamp-Massey oracle pins
from oracle.bm import berlekamp_massey  # noqa: E402


def _expand_prod_1_minus(ms, p):
    c = [1]
    for r in ms:                      # multiply by (1 - r z)
        nc = c + [0]
        for i in range(len(c)):
            nc[i + 1] = (nc[i + 1] - r * c[i]) % p
        c = nc
    return c


def test_bm_closed_forms():
    p = 1_000_003
    # Fibonacci: s_n = s_{n-1} + s_{n-2}  ->  C = 1 - z - z^2
    fib = [0, 1]
    for _ in range(30):
        fib.append((fib[-1] + fib[-2]) % p)
    assert berlekamp_massey(fib, p) == (2, [1, p - 1, p - 1])
    # geometric c r^n -> C = 1 - r z
    assert berlekamp_massey([5 * pow(7, n, p) % p for n in range(10)], p) == (1, [1, p - 7])
    # zero sequence -> L = 0
    assert berlekamp_massey([0] * 9, p) == (0, [1])
    # impulse at the last position -> L = T (no shorter LFSR generates it)
    L, C = berlekamp_massey([0] * 7 + [3], p)
    assert L == 8


def test_bm_power_sums_give_product():
    """s_n = sum a_i m_i^n (distinct m_i, a_i != 0), T = 2r: C = prod (1 - m_i z)."""
    p = (1 << 61) - 1
    import random
    rnd = random.Random(11)
    for r in (1, 2, 5, 17):
        ms = rnd.sample(range(2, p), r)
        a = [rnd.randrange(1, p) for _ in range(r)]
        seq = [sum(ai * pow(mi, n, p) for ai, mi in zip(a, ms)) % p for n in range(2 * r)]
        L, C = berlekamp_massey(seq, p)
        assert L == r and C == _expand_prod_1_minus(ms, p)


def test_bm_on_oracle_output_matches_monomials():
    """P9 through BM: every bucket of an oracle evaluation at j = 0.. (T >= 2 r_g) has connection
    polynomial prod over its distinct m_i of (1 - m_i z)."""
    p, n, T = (1 << 62) - 57, 5, 24
    w = synth.random_small(31, p, n, 60, 3, T, 0)
    w.exps[:, 0] = np.arange(60) % 9                    # 9 buckets of <= 7 terms
    w.exps[:, 1] = 0
    out = oracle.eval_direct(p, n, w.coeffs, w.exps, w.alpha, 0, T)
    rows = oracle.buckets(w.exps, n).tolist()
    for g, r in enumerate(rows):
        members = [i for i in range(60) if int(w.exps[i, 0]) == r[0]]
        coef = {}
        for i in members:
            m = _m_python(w.alpha, w.exps[i, 2:], p)
            coef[m] = (coef.get(m, 0) + int(w.coeffs[i])) % p
        ms = sorted(m for m, c in coef.items() if c)
        L, C = berlekamp_massey(out[g].tolist(), p)
        assert L == len(ms)
        assert C == _expand_prod_1_minus(ms, p)
