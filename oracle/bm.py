"""Berlekamp–Massey over F_p -- TEST INFRASTRUCTURE ONLY.

Textbook Massey (1969) with modular inverses on Python integers: for s_0 .. s_{T-1} returns the
shortest connection polynomial C(z) = 1 + c_1 z + ... + c_L z^L with
    s_n + c_1 s_{n-1} + ... + c_L s_{n-L} = 0   for L <= n < T.
For s_n = sum_i a_i m_i^n with distinct nonzero m_i and a_i != 0, and T >= 2r, C(z) =
prod_i (1 - m_i z) (Ben-Or/Tiwari, the transposed-Vandermonde structure of PAPER.md:279-285,
465-478, 765-773).  Pinned in tests/test_oracle_pins.py against closed forms.
"""
from __future__ import annotations


def berlekamp_massey(seq, p):
    s = [int(x) % p for x in seq]
    C, B = [1], [1]
    L, m, b = 0, 1, 1
    for n in range(len(s)):
        d = s[n]
        for i in range(1, L + 1):
            d = (d + C[i] * s[n - i]) % p
        if d == 0:
            m += 1
            continue
        coef = d * pow(b, p - 2, p) % p
        T = C[:]
        if len(C) < len(B) + m:
            C = C + [0] * (len(B) + m - len(C))
        for i, bi in enumerate(B):
            C[i + m] = (C[i + m] - coef * bi) % p
        if 2 * L <= n:
            L, B, b, m = n + 1 - L, T, d, 1
        else:
            m += 1
    C = (C + [0] * (L + 1))[: L + 1]
    return L, C
