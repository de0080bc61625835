"""Python big-integer brute force -- TEST INFRASTRUCTURE ONLY (tiny inputs).

Literal substitution of beta^j = (alpha_1^j, ..., alpha_{n-2}^j) into every term of
f = sum_i c_i x^{dx_i} y^{dy_i} z_1^{e_i1} ... z_{n-2}^{e_i,n-2}  (PAPER.md:246-266 and
Eq. e:def_f), with Python's arbitrary-precision integers: each term's
value is computed as an exact integer product c_i * prod_l (alpha_l^j)^{e_il} and only the
final per-row sum is reduced mod p.  No modular shortcut, no identity m_i^t, no '%' inside
the product -- independent of oracle.c's __int128 arithmetic.
"""
from __future__ import annotations


def brute_eval(p, n, coeffs, exps, alpha, j0, T):
    """Returns (rows, out): rows = sorted distinct (dx,dy) descending; out[g][k] ints."""
    coeffs = [int(c) for c in coeffs]
    exps = [[int(e) for e in row] for row in exps]
    alpha = [int(a) for a in alpha]
    rows = sorted({(r[0], r[1]) for r in exps}, reverse=True)
    index = {r: g for g, r in enumerate(rows)}
    out = [[0] * T for _ in rows]
    for k in range(T):
        j = j0 + k
        beta = [a ** j for a in alpha]                       # exact integers, unreduced
        sums = [0] * len(rows)
        for c, r in zip(coeffs, exps):
            v = c
            for l in range(n - 2):
                v *= beta[l] ** r[2 + l]
            sums[index[(r[0], r[1])]] += v
        for g in range(len(rows)):
            out[g][k] = sums[g] % p
    return rows, out
