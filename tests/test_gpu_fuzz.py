"""Randomised differential parity: every hot kernel (k_step through PE_PATH_INT / FP64, k_tc through
PE_PATH_TC in both tensor-core forms for p >= 2^31, the fast product-tree method through PE_PATH_FAST, and the automatic choice) against
the direct CPU oracle on seeded random shapes -- primes across every arithmetic mode (p < 2^31,
the 7-digit range, p < 2^50, lazy-4 and exact-quotient 62/63-bit), n from 2 to 10, 1 to 3000 terms
with repeated (x, y) buckets, T from 1 to 2500 with ragged tails, j0 from 0 to near 2^64."""
import numpy as np
import pytest

import oracle
import paper_2004_11571_b200 as pe
import synth

pytestmark = pytest.mark.gpu

PRIMES = [3, 13, 65521, (1 << 31) - 1, (1 << 31) + 11, (1 << 50) - 27, (1 << 54) - 33, synth.P62,
          (1 << 62) + 135, (1 << 63) - 25]


def _case(seed):
    r = np.random.default_rng(900_000 + seed)
    p = int(PRIMES[r.integers(len(PRIMES))])
    n = int(r.integers(2, 11))
    t = int(r.integers(1, 3001))
    maxdeg = int(r.integers(1, 13))
    T = int(r.choice([1, 2, 31, 33, 64, 129, 500, 1000, 2047, 2500]))
    j0 = int(r.choice([0, 1, int(r.integers(2, 1 << 40)), (1 << 64) - T - 1]))
    w = synth.random_small(1000 + seed, p, n, t, maxdeg, T, j0, coeff_hi=2**64 - 1)
    if n >= 3 and r.random() < 0.5:                # few buckets, many terms each
        w.exps[:, :2] %= np.uint32(int(r.integers(1, 4)))
    return w


@pytest.mark.parametrize("seed", range(24))
def test_random_shapes_all_kernels(seed):
    w = _case(seed)
    ref = oracle.eval_workload(w)
    paths = [pe.PATH_AUTO, pe.PATH_INT, pe.PATH_TC, pe.PATH_FAST]
    if w.p < (1 << 50):
        paths.append(pe.PATH_FP64)
    variants = [(path, False, pe.TC_FORM_AUTO) for path in paths] + [(pe.PATH_AUTO, True, pe.TC_FORM_AUTO)]   # + uint8 exponents
    if w.p >= (1 << 31):   # both tensor-core forms of the 7- and 8-digit modes
        variants.append((pe.PATH_TC, False, pe.TC_FORM_PLAIN))
        variants.append((pe.PATH_TC, False, pe.TC_FORM_SWAPPED))
    for path, compact, form in variants:
        with pe.Context.from_workload(w, path=path, compact=compact, tc_form=form) as ctx:
            out = ctx.eval(w.j0, w.T)
            kern = ctx.eval_kernel(w.T)
        bad = np.argwhere(out != ref)
        assert bad.size == 0, (f"p={w.p} n={w.n} t={w.t} T={w.T} j0={w.j0} path={path} compact={compact} form={form} ({kern}): "
                               f"{len(bad)} mismatches, first {bad[:3].tolist()}")
