/*
 * oracle/oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this.  It shares no code, header, table or constant with the CUDA path
 * (paper_2004_11571_b200/csrc); the two meet only through the seeded inputs of synth/.
 *
 * What it computes (§2.1 "Presentation", §2.3 Eq. e:def_f,
 * read coefficient-wise; DESIGN.md §"Readings" R1-R10):
 *
 *   out[g][k] = sum_{i : (dx_i,dy_i) = B_g} (c_i mod p) * prod_{l=1}^{n-2} ((alpha_l^{j} mod p)^{e_{i,l}} mod p)  (mod p)
 *   with j = j0 + k, and rows B_g = the distinct (dx,dy) of the input, descending lex order.
 *
 * It is the plain definition written out: for every point j it forms beta = alpha^j
 * ("beta^t = (beta_3^t, ..., beta_n^t)") and substitutes it into every term
 * by square-and-multiply with unsigned __int128 products reduced by '%'.  It does NOT use
 * the identity M_i(beta^t) = m_i^t that the GPU path exploits.
 *
 * Companion: incr_eval() is Alg. 1 ("Compute kernel of the matrix
 * method"): a <- a (x) m, c <- c (+) a, over runs of equal (d_i, e_i) in sorted order.
 * It uses the identity and is used only as the pin P7 (incremental == direct) and as a
 * fast full-output checker for large configs.
 *
 * Parity pins for every function here: tests/test_oracle_pins.py (P1-P12).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* (a*b) mod p by a double-width product and the '%' operator ("c = a x b"
 * denoting c = a*b mod p). */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)a * b) % p); }

/* (a+b) mod p for a, b < p. */
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t p) {
    u128 s = (u128)a + b;
    return (uint64_t)(s % p);
}

/* b^e mod p, left-to-right square and multiply ("exponentiations by squaring"). */
uint64_t oracle_powmod(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    b %= p;
    int started = 0;                       /* skip the leading zero bits of e */
    for (int bit = 63; bit >= 0; --bit) {
        if (started) r = mulmod(r, r, p);
        if ((e >> bit) & 1) { r = mulmod(r, b, p); started = 1; }
    }
    return r;
}

uint64_t oracle_mulmod(uint64_t a, uint64_t b, uint64_t p) { return mulmod(a % p, b % p, p); }

/* ---- bucket list: distinct (dx,dy), descending lexicographic order (PAPER.md:495-500,
 *      DESIGN.md reading R2) ---------------------------------------------------------- */
static int cmp_desc(const void* x, const void* y) {
    uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return a < b ? 1 : (a > b ? -1 : 0);
}

/* Returns G; writes dxdy[2g], dxdy[2g+1] for row g if dxdy != NULL and row[i] for each term. */
static uint64_t build_rows(uint64_t t, uint32_t n, const uint32_t* exps, uint64_t** keys_out,
                           uint64_t* row) {
    uint64_t* keys = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < t; ++i)
        keys[i] = ((uint64_t)exps[i * n + 0] << 32) | exps[i * n + 1];
    uint64_t* sorted = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    memcpy(sorted, keys, t * sizeof(uint64_t));
    qsort(sorted, t, sizeof(uint64_t), cmp_desc);
    uint64_t G = 0;
    for (uint64_t i = 0; i < t; ++i)
        if (i == 0 || sorted[i] != sorted[G - 1]) sorted[G++] = sorted[i];
    if (row) {
        for (uint64_t i = 0; i < t; ++i) {          /* binary search in the descending list */
            uint64_t lo = 0, hi = G;
            while (hi - lo > 1) {
                uint64_t mid = (lo + hi) / 2;
                if (sorted[mid] >= keys[i]) lo = mid; else hi = mid;
            }
            row[i] = lo;
        }
    }
    free(keys);
    *keys_out = sorted;
    return G;
}

/* Number of rows G and their (dx,dy) (dxdy may be NULL). */
uint64_t oracle_buckets(uint64_t t, uint32_t n, const uint32_t* exps, uint32_t* dxdy) {
    uint64_t* keys;
    uint64_t G = build_rows(t, n, exps, &keys, NULL);
    if (dxdy)
        for (uint64_t g = 0; g < G; ++g) { dxdy[2 * g] = (uint32_t)(keys[g] >> 32); dxdy[2 * g + 1] = (uint32_t)keys[g]; }
    free(keys);
    return G;
}

/*
 * Direct oracle.  Columns: ks == NULL -> k = 0..nk-1; else k = ks[0..nk-1] (sampled mode).
 * out is [G][nk] row-major, column c holds point j = j0 + (ks ? ks[c] : c).
 * Parallel over columns with OpenMP (each thread owns its column; the arithmetic per column
 * is the sequential definition above).
 */
int oracle_eval(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs, const uint32_t* exps,
                const uint64_t* alpha, uint64_t j0, const uint64_t* ks, uint64_t nk, uint64_t* out) {
    if (p < 2 || n < 2) return -1;
    uint64_t* keys;
    uint64_t* row = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    uint64_t G = build_rows(t, n, exps, &keys, row);
    free(keys);
    memset(out, 0, G * nk * sizeof(uint64_t));
    const uint32_t nz = n - 2;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < (int64_t)nk; ++c) {
        uint64_t j = j0 + (ks ? ks[c] : (uint64_t)c);
        uint64_t beta[64];
        for (uint32_t l = 0; l < nz; ++l) beta[l] = oracle_powmod(alpha[l] % p, j, p);   /* beta_l = alpha_l^j */
        for (uint64_t i = 0; i < t; ++i) {
            uint64_t v = coeffs[i] % p;                                          /* a_i in F_p (R5) */
            for (uint32_t l = 0; l < nz; ++l)
                v = mulmod(v, oracle_powmod(beta[l], exps[i * n + 2 + l], p), p);   /* (beta_l)^{e_il} */
            uint64_t* o = &out[row[i] * nk + c];
            *o = addmod(*o, v, p);
        }
    }
    free(row);
    return 0;
}

/*
 * Incremental checker, Alg. 1 with the a-vector seeded at j0:
 *   m_i = prod_l alpha_l^{e_il}                       ("m_i = M_i(beta)")
 *   a_i = c_i * m_i^{j0}                              (seed; PAPER.md:562-565 Lambda idea)
 *   for each point: c <- sum over the run of equal (d_i,e_i) of a_i  (line "c <- c (+) a[j]")
 *                   a_i <- a_i * m_i                  (line "a[j] <- a[j] (x) m[j]")
 * (reading R12: add-then-multiply order, Alg. 7.)
 * Terms are processed in the sorted order of their (dx,dy) row; out is [G][T].
 */
int incr_eval(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs, const uint32_t* exps,
              const uint64_t* alpha, uint64_t j0, uint64_t T, uint64_t* out) {
    if (p < 2 || n < 2) return -1;
    uint64_t* keys;
    uint64_t* row = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    uint64_t G = build_rows(t, n, exps, &keys, row);
    free(keys);
    /* order terms by row (counting sort) so each row is a contiguous run, as in Alg. 1 */
    uint64_t* start = (uint64_t*)calloc(G + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < t; ++i) start[row[i] + 1]++;
    for (uint64_t g = 0; g < G; ++g) start[g + 1] += start[g];
    uint64_t* fill = (uint64_t*)malloc((G + 1) * sizeof(uint64_t));
    memcpy(fill, start, (G + 1) * sizeof(uint64_t));
    uint64_t* a = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    uint64_t* m = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < t; ++i) {
        uint64_t mi = 1 % p;
        for (uint32_t l = 0; l + 2 < n; ++l) mi = mulmod(mi, oracle_powmod(alpha[l], exps[i * n + 2 + l], p), p);
        uint64_t pos = fill[row[i]]++;
        m[pos] = mi;
        a[pos] = mulmod(coeffs[i] % p, oracle_powmod(mi, j0, p), p);
    }
    free(fill);
    free(row);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t g = 0; g < (int64_t)G; ++g) {      /* runs are independent; points are sequential */
        for (uint64_t k = 0; k < T; ++k) {
            uint64_t c = 0;
            for (uint64_t i = start[g]; i < start[g + 1]; ++i) {
                c = addmod(c, a[i], p);
                a[i] = mulmod(a[i], m[i], p);
            }
            out[g * T + k] = c;
        }
    }
    free(start); free(a); free(m);
    return 0;
}

/*
 * Same Alg. 1 checker, with the points cut into blocks of `block` columns so that the work
 * is spread over (row, block) pairs rather than rows alone (a Zipf-skewed config-5 row of
 * 1.3M terms would otherwise run 16384 points on one thread).  Each (row, block) task seeds its
 * a-vector at its first point, a_i = c_i * m_i^{j0+k0} -- the seed incr_eval uses at j0, i.e. the
 * Lambda/Gamma seeding of PAPER.md:559-565 -- then runs Alg. 1 over the block.
 * Only the task split differs from incr_eval; the arithmetic per point is the same.
 */
int incr_eval_blocked(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs, const uint32_t* exps,
                      const uint64_t* alpha, uint64_t j0, uint64_t T, uint64_t block, uint64_t* out) {
    if (p < 2 || n < 2 || block == 0) return -1;
    uint64_t* keys;
    uint64_t* row = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    uint64_t G = build_rows(t, n, exps, &keys, row);
    free(keys);
    uint64_t* start = (uint64_t*)calloc(G + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < t; ++i) start[row[i] + 1]++;
    for (uint64_t g = 0; g < G; ++g) start[g + 1] += start[g];
    uint64_t* fill = (uint64_t*)malloc((G + 1) * sizeof(uint64_t));
    memcpy(fill, start, (G + 1) * sizeof(uint64_t));
    uint64_t* c = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    uint64_t* m = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < t; ++i) {                 /* m_i = prod_l alpha_l^{e_il} */
        uint64_t mi = 1 % p;
        for (uint32_t l = 0; l + 2 < n; ++l) mi = mulmod(mi, oracle_powmod(alpha[l], exps[i * n + 2 + l], p), p);
        uint64_t pos = fill[row[i]]++;
        m[pos] = mi;
        c[pos] = coeffs[i] % p;
    }
    free(fill);
    free(row);
    const uint64_t nb = (T + block - 1) / block;
    int fail = 0;
#pragma omp parallel
    {
        uint64_t cap = 0;
        uint64_t* a = NULL;
#pragma omp for schedule(dynamic, 1)
        for (int64_t task = 0; task < (int64_t)(G * nb); ++task) {
            const uint64_t g = (uint64_t)task / nb, b = (uint64_t)task % nb;
            const uint64_t k0 = b * block, k1 = k0 + block < T ? k0 + block : T;
            const uint64_t s0 = start[g], len = start[g + 1] - s0;
            if (len > cap) {
                free(a);
                cap = len;
                a = (uint64_t*)malloc(cap * sizeof(uint64_t));
                if (!a) { fail = 1; cap = 0; continue; }
            }
            for (uint64_t i = 0; i < len; ++i)         /* a_i = c_i m_i^{j0 + k0} */
                a[i] = mulmod(c[s0 + i], oracle_powmod(m[s0 + i], j0 + k0, p), p);
            for (uint64_t k = k0; k < k1; ++k) {
                uint64_t acc = 0;
                for (uint64_t i = 0; i < len; ++i) {
                    acc = addmod(acc, a[i], p);        /* c <- c (+) a[j] */
                    a[i] = mulmod(a[i], m[s0 + i], p); /* a[j] <- a[j] (x) m[j] */
                }
                out[g * T + k] = acc;
            }
        }
        free(a);
    }
    free(start); free(c); free(m);
    return fail ? -2 : 0;
}
