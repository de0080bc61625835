"""CPU checks of the arithmetic the tensor-core path rests on (csrc/tc.cuh), from
the definitions -- not from the kernel:

* byte-diagonal identity: for 64-bit L, R split into bytes L = sum_s 2^{8s} L_s,
  sum_i L_i R_i = sum_d 2^{8d} D_d with D_d = sum_i sum_{s+t=d} L_{i,s} R_{i,t} (exact integers);
* the accumulator bound: D_d <= 8 * 255^2 * 8192 < 2^32 for a piece of 8192 terms, so a
  wrapping u32/s32 accumulator holds it exactly;
* the round split: X mod p = (X_0 + X_1) mod p with X_g = sum over round g's diagonals
  (d = 0..7, d = 8..14), so each round can be reduced on its own;
* the epilogue reduction: the 160-bit X is cut into 32-bit words x0..x4, x2..x4 are folded with
  2^{32k} mod p into a 128-bit (hi, lo) with hi < p, and one Montgomery REDC gives X 2^-64 mod p --
  which is sum_i L_i m_i^v when the baby-step factors are Montgomery residues m^v 2^64 mod p.
"""
import random

import pytest

P62 = (1 << 62) - 57


def bytes_of(x):
    return [(x >> (8 * s)) & 0xFF for s in range(8)]


def diagonals(Ls, Rs):
    D = [0] * 15
    for L, R in zip(Ls, Rs):
        lb, rb = bytes_of(L), bytes_of(R)
        for s in range(8):
            for t in range(8):
                D[s + t] += lb[s] * rb[t]
    return D


def redc(hi, lo, p):
    """Montgomery reduction of hi*2^64 + lo (hi < p): returns (hi*2^64 + lo) * 2^-64 mod p."""
    assert hi < p
    pinv = (-pow(p, -1, 1 << 64)) % (1 << 64)
    u = (lo * pinv) % (1 << 64)
    t = (hi * (1 << 64) + lo + u * p) >> 64
    return t - p if t >= p else t


@pytest.mark.parametrize("seed", range(4))
def test_byte_diagonal_identity(seed):
    rng = random.Random(seed)
    n = 97
    Ls = [rng.getrandbits(64) for _ in range(n)]
    Rs = [rng.getrandbits(64) for _ in range(n)]
    D = diagonals(Ls, Rs)
    assert sum(a * b for a, b in zip(Ls, Rs)) == sum(D[d] << (8 * d) for d in range(15))


def test_accumulator_bound_at_piece_size():
    """All-0xFF bytes maximise every diagonal: the 8-pair diagonal over 8192 terms stays < 2^32."""
    npairs = [min(d, 14 - d) + 1 for d in range(15)]
    assert max(npairs) == 8
    worst = 8 * 255 * 255 * 8192
    assert worst < (1 << 32) and worst >= (1 << 31)     # tight: read as u32, not s32
    D = diagonals([2**64 - 1] * 3, [2**64 - 1] * 3)
    assert D == [3 * 255 * 255 * k for k in npairs]


@pytest.mark.parametrize("seed", range(3))
def test_round_split_and_epilogue_reduction(seed):
    rng = random.Random(100 + seed)
    p = P62
    R64 = (1 << 64) % p
    n = 64
    c = [rng.randrange(p) for _ in range(n)]
    m = [rng.randrange(1, p) for _ in range(n)]
    j, v = rng.randrange(1, 1 << 40), rng.randrange(64)
    # giant-step values (lazy representatives < 4p, as the Shoup chains leave them) and
    # Montgomery baby-step residues m^v 2^64 mod p
    Ls = [(ci * pow(mi, j, p)) % p + rng.randrange(4) * p for ci, mi in zip(c, m)]
    Ls = [x if x < (1 << 64) else x - p for x in Ls]
    Rs = [(pow(mi, v, p) * R64) % p for mi in m]
    want = sum(ci * pow(mi, j + v, p) for ci, mi in zip(c, m)) % p
    D = diagonals(Ls, Rs)
    parts = []
    for rnd in (range(0, 8), range(8, 15)):
        X = sum(D[d] << (8 * d) for d in rnd)
        assert X < (1 << 145)
        x = [(X >> (32 * k)) & 0xFFFFFFFF for k in range(5)]
        lo, hi = x[0] | (x[1] << 32), 0
        acc = lo
        for k, xk in ((2, x[2]), (3, x[3]), (4, x[4])):
            acc += xk * pow(2, 32 * k, p)                  # x_k * (2^{32k} mod p), 128-bit sum
        hi, lo = acc >> 64, acc & ((1 << 64) - 1)
        parts.append(redc(hi % p, lo, p))                  # = X_g 2^-64 mod p
    assert (parts[0] + parts[1]) % p == want


def test_shoup_constant_identity():
    """The identity behind shoup_w_fast (csrc/modcore.cuh): for m < p, floor(m 2^64 / p) equals
    (m 2^64 mod p) * (-p^-1 mod 2^64) mod 2^64 (m 2^64 = w p + rem, so w p == -rem mod 2^64, and
    0 <= w < 2^64 makes the congruence an equality).  Python integers, no kernel code."""
    import random
    rnd = random.Random(5)
    for p in (3, 13, 509, 1_000_003, (1 << 31) - 1, (1 << 62) - 57, (1 << 63) - 25):
        ninv = (-pow(p, -1, 1 << 64)) % (1 << 64)
        for m in [0, 1, p - 1] + [rnd.randrange(p) for _ in range(200)]:
            rem = (m << 64) % p
            assert (rem * ninv) % (1 << 64) == (m << 64) // p


@pytest.mark.parametrize("seed", range(3))
def test_swapped_form_reduction(seed):
    """The swapped form (tc.cuh MODE 4 / 5): A = giant steps G[u] = m^{64u} as Montgomery residues
    m^{64u} 2^64 mod p (point-independent, built per handle), B = baby steps R'[v] = c m^{j_s + v}
    (lazy representatives < 4p from the Shoup chains).  The same diagonals, round split and
    REDC give sum_i c_i m_i^{j_s + 64u + v} mod p: the byte identity does not care which side
    carries the point-dependent factor."""
    rng = random.Random(200 + seed)
    p = P62
    R64 = (1 << 64) % p
    n = 48
    c = [rng.randrange(p) for _ in range(n)]
    m = [rng.randrange(1, p) for _ in range(n)]
    js, u, v = rng.randrange(1, 1 << 40), rng.randrange(128), rng.randrange(64)
    Gs = [(pow(mi, 64 * u, p) * R64) % p for mi in m]
    Bs = [(ci * pow(mi, js + v, p)) % p + rng.randrange(4) * p for ci, mi in zip(c, m)]
    Bs = [x if x < (1 << 64) else x - p for x in Bs]
    want = sum(ci * pow(mi, js + 64 * u + v, p) for ci, mi in zip(c, m)) % p
    D = diagonals(Gs, Bs)
    total = 0
    for rnd in (range(0, 8), range(8, 15)):
        X = sum(D[d] << (8 * d) for d in rnd)
        x = [(X >> (32 * k)) & 0xFFFFFFFF for k in range(5)]
        acc = x[0] | (x[1] << 32)
        for k in (2, 3, 4):
            acc += x[k] * pow(2, 32 * k, p)
        total += redc((acc >> 64) % p, acc & ((1 << 64) - 1), p)
    assert total % p == want


def issue_all32_emulated(Lbytes, Rbytes, nkb):
    """Emulates tc.cuh issue_all32 over nkb K-blocks on byte planes: per K-block, L plane s times
    the 8 baby-step planes t is ONE MMA into slots s .. s + 7 (slot d = s + t); at K-block 0 plane 0
    overwrites slots 0..7, plane 7 goes second split into t = 0 (accumulates slot 7) and t = 1..7
    (overwrites slots 8..14), planes 1..6 accumulate.  Slots start as garbage, as TMEM does.
    Lbytes[s][i], Rbytes[t][i]: byte s / t of term i; a K-block is 32 consecutive terms."""
    rng = random.Random(7)
    slot = [rng.getrandbits(32) for _ in range(15)]          # uninitialised TMEM

    def mma(s, t_lo, t_hi, kb, acc):
        for t in range(t_lo, t_hi + 1):
            part = sum(Lbytes[s][i] * Rbytes[t][i] for i in range(32 * kb, 32 * kb + 32))
            slot[s + t] = ((slot[s + t] if acc else 0) + part) % (1 << 32)

    for kb in range(nkb):
        first = kb == 0
        mma(0, 0, 7, kb, not first)
        if first:
            mma(7, 0, 0, kb, True)
            mma(7, 1, 7, kb, False)
        else:
            mma(7, 0, 7, kb, True)
        for s in range(1, 7):
            mma(s, 0, 7, kb, True)
    return slot


@pytest.mark.parametrize("seed,swapped", [(0, False), (1, False), (2, True), (3, True)])
def test_single_round_v32_schedule_and_reduction(seed, swapped):
    """The V = 32 geometry of the 8-digit modes (tc.cuh issue_all32 / epi_drain5 / fold_row<5, 32>):
    the emulated kb-0 initialisation scheme reproduces every diagonal D_d of the byte-diagonal
    identity exactly (mod 2^32, as the s32 TMEM accumulator), and ONE fold of all 15 diagonals
    (X < 2^145) plus one REDC gives sum_i c_i m_i^{j_s + 32u + v} mod p -- plain form (lazy giant
    steps c m^{j_s + 32u} x Montgomery baby steps m^v 2^64) and swapped form (Montgomery giant steps
    m^{32u} 2^64 x lazy baby steps c m^{j_s + v}) alike.  Python integers, no kernel code."""
    rng = random.Random(300 + seed)
    p = P62
    R64 = (1 << 64) % p
    nkb = 3
    n = 32 * nkb
    c = [rng.randrange(p) for _ in range(n)]
    m = [rng.randrange(1, p) for _ in range(n)]
    js, u, v = rng.randrange(1, 1 << 40), rng.randrange(128), rng.randrange(32)
    if swapped:
        A = [(pow(mi, 32 * u, p) * R64) % p for mi in m]
        B = [(ci * pow(mi, js + v, p)) % p + rng.randrange(4) * p for ci, mi in zip(c, m)]
        B = [x if x < (1 << 64) else x - p for x in B]
    else:
        A = [(ci * pow(mi, js + 32 * u, p)) % p + rng.randrange(4) * p for ci, mi in zip(c, m)]
        A = [x if x < (1 << 64) else x - p for x in A]
        B = [(pow(mi, v, p) * R64) % p for mi in m]
    want = sum(ci * pow(mi, js + 32 * u + v, p) for ci, mi in zip(c, m)) % p
    Ab = [[(x >> (8 * s)) & 0xFF for x in A] for s in range(8)]
    Bb = [[(x >> (8 * t)) & 0xFF for x in B] for t in range(8)]
    slots = issue_all32_emulated(Ab, Bb, nkb)
    assert slots == diagonals(A, B)                          # every D_d < 2^32 here: exact
    X = sum(slots[d] << (8 * d) for d in range(15))
    assert X < (1 << 145)
    x = [(X >> (32 * k)) & 0xFFFFFFFF for k in range(5)]
    acc = x[0] | (x[1] << 32)
    for k in (2, 3, 4):
        acc += x[k] * pow(2, 32 * k, p)
    assert (acc >> 64) < p                                   # REDC's precondition without the fallback
    assert redc(acc >> 64, acc & ((1 << 64) - 1), p) == want


def issue_all32_7_emulated(Lbytes, Rbytes, nkb):
    """tc.cuh issue_all32_7 (7 digits): per K-block L plane s < 7 times the baby-step planes t < 7
    is one MMA into slots s .. s + 6; at K-block 0 plane 0 overwrites slots 0..6 and plane 6 goes
    second, split into t = 0 (accumulates slot 6) and t = 1..6 (overwrites slots 7..12)."""
    rng = random.Random(8)
    slot = [rng.getrandbits(32) for _ in range(13)]

    def mma(s, t_lo, t_hi, kb, acc):
        for t in range(t_lo, t_hi + 1):
            part = sum(Lbytes[s][i] * Rbytes[t][i] for i in range(32 * kb, 32 * kb + 32))
            slot[s + t] = ((slot[s + t] if acc else 0) + part) % (1 << 32)

    for kb in range(nkb):
        first = kb == 0
        mma(0, 0, 6, kb, not first)
        if first:
            mma(6, 0, 0, kb, True)
            mma(6, 1, 6, kb, False)
        else:
            mma(6, 0, 6, kb, True)
        for s in range(1, 6):
            mma(s, 0, 6, kb, True)
    return slot


@pytest.mark.parametrize("seed", range(3))
def test_single_round_v32_seven_digits(seed):
    """The 7-digit mode (2^31 <= p < 2^54) on the V = 32 geometry: lazy giant steps < 4p < 2^56 and
    Montgomery baby steps < p have 7 bytes; the emulated issue_all32_7 schedule reproduces the 13
    byte diagonals, and one 13-diagonal fold + REDC gives sum_i c_i m_i^{j_s + 32u + v} mod p."""
    rng = random.Random(400 + seed)
    p = (1 << 50) - 27
    R64 = (1 << 64) % p
    nkb = 3
    n = 32 * nkb
    c = [rng.randrange(p) for _ in range(n)]
    m = [rng.randrange(1, p) for _ in range(n)]
    js, u, v = rng.randrange(1, 1 << 40), rng.randrange(128), rng.randrange(32)
    A = [(ci * pow(mi, js + 32 * u, p)) % p + rng.randrange(4) * p for ci, mi in zip(c, m)]
    B = [(pow(mi, v, p) * R64) % p for mi in m]
    assert max(A) < (1 << 56) and max(B) < (1 << 56)
    want = sum(ci * pow(mi, js + 32 * u + v, p) for ci, mi in zip(c, m)) % p
    Ab = [[(x >> (8 * s)) & 0xFF for x in A] for s in range(7)]
    Bb = [[(x >> (8 * t)) & 0xFF for x in B] for t in range(7)]
    slots = issue_all32_7_emulated(Ab, Bb, nkb)
    assert slots == diagonals(A, B)[:13] and diagonals(A, B)[13:] == [0, 0]
    X = sum(slots[d] << (8 * d) for d in range(13))
    x = [(X >> (32 * k)) & 0xFFFFFFFF for k in range(5)]
    acc = x[0] | (x[1] << 32)
    for k in (2, 3, 4):
        acc += x[k] * pow(2, 32 * k, p)
    assert redc(acc >> 64, acc & ((1 << 64) - 1), p) == want
