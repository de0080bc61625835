"""Seeded synthetic workloads for the partial-evaluation hot path.

This module is shared by the tests, ``bench.py`` and ``__graft_entry__``: it feeds the
same inputs to the CPU oracle (``oracle/``) and to the CUDA path
(``paper_2004_11571_b200``).  It holds NONE of the method's arithmetic -- it only draws
random integers (coefficients, alpha, exponent vectors) with the shapes of
``BASELINE.json:configs`` and DESIGN.md "Input recipe".  It imports neither the oracle nor
the product package.

Workload shapes (BASELINE.json ``configs[0..4]`` plus the paper's default E1 shape,
PAPER.md:546-552 "s = 5x10^5 terms; n = 6 variables ... d=10 ... T ... 10000"):

====  ===  =========  =====  ==========  ==========================================
cfg    n       t        T     p           exponent recipe (readings R15-R18)
====  ===  =========  =====  ==========  ==========================================
1      6      1 000      64   2^62-57     each of the 6 exponents uniform on 0..5
2      8    100 000    1000   2^62-57     uniform on {e in N^8 : sum e <= 20}
3      9  1 000 000    4096   2^62-57     (dx,dy) uniform [0,15]^2; 7 evaluated exps
                                          uniform on {sum <= 30}
4      9  1 000 000    4096   2^50-27     config 3's exponents, coefficients mod p4
5     12 10 000 000   16384   2^62-57     (dx,dy) Zipf(s=1) over a seeded ranking of
                                          [0,30]^2; 10 evaluated exps uniform {sum<=40}
6      6    500 000   10000   2^50-27     paper E1 shape: exps uniform 0..10, coeffs
                                          in [1,p)
====  ===  =========  =====  ==========  ==========================================

All draws use ``numpy.random.Generator(PCG64(seed))`` with ``seed = 2004115710 + cfg``
unless a seed is given.  Full exponent vectors are deduplicated; the surviving terms keep
their (random) draw order so that the library's sort is exercised.
"""
from __future__ import annotations

import dataclasses
import numpy as np

P62 = (1 << 62) - 57          # largest prime below 2^62 (BASELINE.json configs 1,2,3,5)
P50 = (1 << 50) - 27          # largest prime below 2^50 (BASELINE.json config 4)
SEED_BASE = 2004115710


@dataclasses.dataclass
class Workload:
    name: str
    p: int
    n: int
    coeffs: np.ndarray        # uint64 [t]
    exps: np.ndarray          # uint32 [t, n]; col 0 = deg x, col 1 = deg y, cols 2.. = z_1..z_{n-2}
    alpha: np.ndarray         # uint64 [n-2]
    j0: int
    T: int

    @property
    def t(self) -> int:
        return int(self.coeffs.shape[0])

    def term_points(self) -> int:
        return self.t * self.T


CONFIGS = {
    1: dict(n=6, t=1_000, T=64, p=P62),
    2: dict(n=8, t=100_000, T=1000, p=P62),
    3: dict(n=9, t=1_000_000, T=4096, p=P62),
    4: dict(n=9, t=1_000_000, T=4096, p=P50),
    5: dict(n=12, t=10_000_000, T=16384, p=P62),
    6: dict(n=6, t=500_000, T=10_000, p=P50),
}


def uniform_mod(rng: np.random.Generator, lo: int, p: int, size) -> np.ndarray:
    """Uniform integers in [lo, p) as uint64 (p < 2^63)."""
    return rng.integers(lo, p, size=size, dtype=np.uint64)


def simplex(rng: np.random.Generator, N: int, k: int, D: int) -> np.ndarray:
    """N vectors uniform on {e in N^k : sum(e) <= D} (stars and bars).

    A uniformly random k-subset {q_1 < ... < q_k} of {0..D+k-1} (Floyd's algorithm,
    vectorised over rows) maps bijectively to e_1 = q_1, e_i = q_i - q_{i-1} - 1.
    """
    n = D + k
    S = np.empty((N, k), dtype=np.int64)
    for i, j in enumerate(range(n - k, n)):
        r = rng.integers(0, j + 1, size=N)
        hit = (S[:, :i] == r[:, None]).any(axis=1) if i else np.zeros(N, bool)
        S[:, i] = np.where(hit, j, r)
    S.sort(axis=1)
    e = np.empty_like(S)
    e[:, 0] = S[:, 0]
    e[:, 1:] = np.diff(S, axis=1) - 1
    return e.astype(np.uint8)


def _draw_rows(rng, cfg: int, N: int, n: int, zipf_rank=None) -> np.ndarray:
    if cfg == 1:
        return rng.integers(0, 6, size=(N, n), dtype=np.uint8)
    if cfg == 2:
        return simplex(rng, N, n, 20)
    if cfg in (3, 4):
        xy = rng.integers(0, 16, size=(N, 2), dtype=np.uint8)
        return np.concatenate([xy, simplex(rng, N, n - 2, 30)], axis=1)
    if cfg == 5:
        # Zipf s=1 over a seeded ranking of the 31x31 (dx,dy) pairs.
        w = 1.0 / np.arange(1, 962)
        pick = rng.choice(961, size=N, p=w / w.sum())
        pair = zipf_rank[pick]
        xy = np.stack([pair // 31, pair % 31], axis=1).astype(np.uint8)
        return np.concatenate([xy, simplex(rng, N, n - 2, 40)], axis=1)
    if cfg == 6:
        return rng.integers(0, 11, size=(N, n), dtype=np.uint8)
    raise ValueError(cfg)


def distinct_rows(rng, cfg: int, t: int, n: int) -> np.ndarray:
    """Exactly t distinct exponent rows, in random draw order."""
    zipf_rank = rng.permutation(961) if cfg == 5 else None
    have = np.zeros((0, n), np.uint8)
    while have.shape[0] < t:
        need = t - have.shape[0]
        cand = np.concatenate([have, _draw_rows(rng, cfg, int(need * 1.3) + 64, n, zipf_rank)])
        v = np.ascontiguousarray(cand).view(np.dtype((np.void, n))).ravel()
        _, first = np.unique(v, return_index=True)
        first.sort()                          # keep draw order (existing rows first)
        have = cand[first[:t]]
    return have


def gen_config(cfg: int, seed: int | None = None, t: int | None = None,
               T: int | None = None, j0: int = 1) -> Workload:
    """Seeded synthetic workload for BASELINE config ``cfg`` (1..5) or the paper shape (6).

    ``t``/``T`` override the term / point count (same recipe, smaller instance) for tests.
    Point indexing follows DESIGN.md reading R1: column k <-> j = j0 + k, j0 = 1.
    """
    c = CONFIGS[cfg]
    n, p = c["n"], c["p"]
    t = c["t"] if t is None else t
    T = c["T"] if T is None else T
    if cfg == 4:
        # config 4 = config 3's exponent structure with the 50-bit prime
        rng = np.random.Generator(np.random.PCG64(SEED_BASE + 3 if seed is None else seed))
        exps = distinct_rows(rng, 3, t, n)
        rng = np.random.Generator(np.random.PCG64((SEED_BASE + 4 if seed is None else seed) + 10**6))
    else:
        rng = np.random.Generator(np.random.PCG64(SEED_BASE + cfg if seed is None else seed))
        exps = distinct_rows(rng, cfg, t, n)
    lo = 1 if cfg == 6 else 0
    coeffs = uniform_mod(rng, lo, p, t)
    alpha = uniform_mod(rng, 1, p, n - 2)
    return Workload(f"config{cfg}", p, n, coeffs, exps.astype(np.uint32), alpha, j0, T)


def random_small(seed: int, p: int, n: int, t: int, maxdeg: int, T: int, j0: int = 1,
                 dup: bool = False, coeff_hi: int | None = None) -> Workload:
    """Small random instance (any prime p, any n >= 2) for parity / edge-case tests.

    ``dup`` allows repeated full monomials (reading R7); ``coeff_hi`` draws
    coefficients in [0, coeff_hi) (may exceed p: reading R5, reduced by the callee).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    if dup or t == 0:
        exps = rng.integers(0, maxdeg + 1, size=(t, n), dtype=np.uint32)
    else:
        space = (maxdeg + 1) ** n
        t = min(t, space)
        exps = np.zeros((0, n), np.uint32)
        while exps.shape[0] < t:
            cand = np.concatenate([exps, rng.integers(0, maxdeg + 1, size=(2 * t, n), dtype=np.uint32)])
            v = np.ascontiguousarray(cand).view(np.dtype((np.void, 4 * n))).ravel()
            _, first = np.unique(v, return_index=True)
            first.sort()
            exps = cand[first[:t]]
    hi = p if coeff_hi is None else coeff_hi
    coeffs = rng.integers(0, hi, size=t, dtype=np.uint64)
    alpha = rng.integers(1, p, size=max(n - 2, 0), dtype=np.uint64)
    return Workload(f"small{seed}", p, n, coeffs, exps.astype(np.uint32), alpha, j0, T)
