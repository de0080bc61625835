"""Pin P12: the sm_100a modular core (csrc/modcore.cuh) against exact integer arithmetic.

Exhaustive over all operand pairs for every odd prime p <= 509 (SPEC.md:97 shape), random
operands for 24 primes of 20..63 bits, lazy inputs up to 2^64, edge operands, and the FP64
signed-zero properties of PAPER.md:924-946 (x*0 never gives -0.0; nonzero x nonzero != 0).
"""
import numpy as np
import pytest

import paper_2004_11571_b200 as pe
import synth

pytestmark = pytest.mark.gpu

SMALL_PRIMES = [q for q in range(3, 510) if all(q % d for d in range(2, int(q**0.5) + 1))]


def _rand_primes():
    import sympy
    ps = [int(sympy.prevprime(1 << k)) for k in (20, 24, 28, 31, 32, 33, 36, 40, 44, 48, 49, 50)]
    ps += [int(sympy.prevprime(1 << k)) for k in (51, 52, 54, 56, 58, 60, 61, 62, 63)]
    ps += [(1 << 62) - 57, (1 << 50) - 27, int(sympy.nextprime(1 << 62))]
    return sorted(set(ps))


def _expect(a, b, p):
    return np.array([(x * y) % p for x, y in zip(a.tolist(), b.tolist())], dtype=np.uint64)


@pytest.mark.parametrize("variant", [pe.CORE_SHOUP4, pe.CORE_SHOUP2, pe.CORE_MONT, pe.CORE_FP64, pe.CORE_HYB])
def test_exhaustive_small_primes(variant):
    for p in SMALL_PRIMES:
        a, b = np.meshgrid(np.arange(p, dtype=np.uint64), np.arange(p, dtype=np.uint64))
        a, b = a.ravel(), b.ravel()
        out = pe.test_core(variant, p, a, b)
        assert np.array_equal(out, (a * b) % np.uint64(p)), (variant, p)


def test_exhaustive_small_primes_add_fp():
    for p in SMALL_PRIMES:
        a, b = np.meshgrid(np.arange(p, dtype=np.uint64), np.arange(p, dtype=np.uint64))
        a, b = a.ravel(), b.ravel()
        out = pe.test_core(pe.CORE_FP64ADD, p, a, b)
        assert np.array_equal(out, (a + b) % np.uint64(p)), p


def test_random_operands_all_primes():
    rng = np.random.default_rng(12)
    for p in _rand_primes():
        N = 200_000
        a = rng.integers(0, p, N, dtype=np.uint64)
        b = rng.integers(0, p, N, dtype=np.uint64)
        want = _expect(a, b, p)
        for v in (pe.CORE_SHOUP4, pe.CORE_SHOUP2, pe.CORE_MONT, pe.CORE_FP64, pe.CORE_HYB):
            if (v == pe.CORE_SHOUP4 and p >= 1 << 62) or (v == pe.CORE_FP64 and p >= 1 << 50):
                continue
            assert np.array_equal(pe.test_core(v, p, a, b), want), (v, p)


def test_lazy_inputs_and_raw_range():
    """SHOUP4 accepts any a < 2^64 and returns r == a*b (mod p) with r < 4p (p < 2^62);
    the PTX core equals its plain-C form (probe returns 2^64-2 on mismatch)."""
    rng = np.random.default_rng(13)
    for p in [q for q in _rand_primes() if q < (1 << 62)] + [13, 509]:
        N = 100_000
        a = rng.integers(0, np.iinfo(np.uint64).max, N, dtype=np.uint64, endpoint=True)
        b = rng.integers(0, p, N, dtype=np.uint64)
        edge_a = np.array([0, 1, p - 1, p, 2 * p - 1, 4 * p - 1 if 4 * p < 2**64 else p,
                           2**64 - 1, 2**63, 2**62], dtype=np.uint64)
        edge_b = np.array([0, 1, p - 1, p - 2, 1, p - 1, p - 1, p - 1, p - 1], dtype=np.uint64)
        a = np.concatenate([a, edge_a])
        b = np.concatenate([b, edge_b])
        raw = pe.test_core(pe.CORE_SHOUP4RAW, p, a, b)
        assert not np.any(raw == np.uint64(2**64 - 2)), "PTX core != C core"
        assert np.all(raw < np.uint64(4 * p)), p
        assert np.array_equal(raw % np.uint64(p), _expect(a, b, p)), p
        s2 = pe.test_core(pe.CORE_SHOUP2, p, a, b)
        assert np.array_equal(s2, _expect(a, b, p)), p


def test_hybrid_lazy_range_all_primes():
    """mul_hyb (FP64 quotient + integer remainder) returns r in (0, 2p), r == a*b (mod p), for
    any a < 2^64 and every odd p < 2^63 (DESIGN.md "Hybrid core" error bound)."""
    rng = np.random.default_rng(17)
    for p in _rand_primes() + [3, 13, 509, (1 << 63) - 25]:
        N = 200_000
        a = rng.integers(0, np.iinfo(np.uint64).max, N, dtype=np.uint64, endpoint=True)
        b = rng.integers(0, p, N, dtype=np.uint64)
        edge_a = np.array([0, 1, p - 1, p, 2 * p - 1, 2**64 - 1, 2**63, 2**62, 2**32 - 1, 2**32], dtype=np.uint64)
        edge_b = np.array([0, 1, p - 1, p - 2, 1, p - 1, p - 1, p - 1, p - 1, (p - 1) // 2], dtype=np.uint64)
        a = np.concatenate([a, edge_a])
        b = np.concatenate([b, edge_b])
        raw = pe.test_core(pe.CORE_HYBRAW, p, a, b)
        assert np.all(raw > 0) and np.all(raw < np.uint64(2 * p)), p
        assert np.array_equal(raw % np.uint64(p), _expect(a, b, p)), p


def test_edge_operands_62bit():
    for p in ((1 << 62) - 57, (1 << 63) - 25, (1 << 50) - 27):
        vals = [0, 1, 2, p - 1, p - 2, (p - 1) // 2, 1 << 31, (1 << 32) - 1, 1 << 32]
        a, b = np.meshgrid(np.array(vals, np.uint64), np.array(vals, np.uint64))
        a, b = a.ravel(), b.ravel()
        want = _expect(a, b, p)
        for v in (pe.CORE_SHOUP2, pe.CORE_MONT, pe.CORE_HYB) + ((pe.CORE_SHOUP4,) if p < 1 << 62 else ()) + \
                ((pe.CORE_FP64,) if p < 1 << 50 else ()):
            assert np.array_equal(pe.test_core(v, p, a, b), want), (v, p)
        assert pe.test_core(pe.CORE_MONT, p, np.array([p - 1], np.uint64), np.array([p - 1], np.uint64))[0] == 1


def test_fp64_signed_zero_and_nonzero_products():
    """for prime p no -0.0 appears, and x, y != 0 => x*y != 0 mod p.
    The probe maps a -0.0 result to 2^64-1, so equality with the exact product covers both."""
    rng = np.random.default_rng(14)
    p = (1 << 50) - 27
    a = rng.integers(1, p, 100_000, dtype=np.uint64)
    b = rng.integers(1, p, 100_000, dtype=np.uint64)
    out = pe.test_core(pe.CORE_FP64, p, a, b)
    assert np.all(out != 0)
    z = np.zeros(1000, np.uint64)
    assert np.all(pe.test_core(pe.CORE_FP64, p, z, b[:1000]) == 0)
    assert np.all(pe.test_core(pe.CORE_FP64, p, a[:1000], z) == 0)
    neg = (p - a[:1000]).astype(np.uint64)                  # x + (p - x) = 0 via the subtract branch
    assert np.all(pe.test_core(pe.CORE_FP64ADD, p, a[:1000], neg) == 0)


def test_seed_pow():
    rng = np.random.default_rng(15)
    for p in ((1 << 62) - 57, (1 << 63) - 25, 13, (1 << 50) - 27):
        N = 20_000
        c = rng.integers(0, np.iinfo(np.uint64).max, N, dtype=np.uint64, endpoint=True)
        m = rng.integers(1, p, N, dtype=np.uint64)
        e = rng.integers(0, np.iinfo(np.uint64).max, N, dtype=np.uint64, endpoint=True)
        e[:4] = [0, 1, 2, p - 1]
        out = pe.test_core(pe.CORE_POW, p, c, m, e)
        want = [(int(x) * pow(int(y), int(z), p)) % p for x, y, z in zip(c, m, e)]
        assert out.tolist() == want, p


def test_shoup_constant_fast_form():
    """shoup_w_fast (w = (m 2^64 mod p) * (-p^-1) mod 2^64, used by k_setup and k_tc_setup) equals
    the bit-loop division floor(m 2^64 / p) on every residue of small primes and on random and edge
    residues of 20- to 63-bit primes."""
    rng = np.random.default_rng(77)
    for p in (3, 5, 7, 13, 251, 509):
        b = np.arange(p, dtype=np.uint64)
        assert not np.any(pe.test_core(pe.CORE_SHOUPW, p, b, b))
    for p in (1_000_003, (1 << 31) - 1, (1 << 50) - 27, (1 << 62) - 57, (1 << 62) + 135, (1 << 63) - 25):
        b = np.concatenate([synth.uniform_mod(rng, 0, p, 20000),
                            np.array([0, 1, 2, p - 2, p - 1, p // 2, p // 2 + 1], np.uint64)])
        assert not np.any(pe.test_core(pe.CORE_SHOUPW, p, b, b)), p
