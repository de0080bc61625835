// fast.cu -- the asymptotically fast evaluation (HL13's
// "asymptotically fast method" that MW17 found to beat the matrix method serially from T = 504).
//
// Per (x,y) bucket g the T outputs are the first T coefficients of a rational power series: with
// a_i = c_i m_i^{j0} (the same seed as the matrix method),
//
//     sum_k out[g][k] z^k = sum_{i in g} a_i / (1 - m_i z)  =  N_g(z) / D_g(z)   (mod z^T),
//     D_g = prod_i (1 - m_i z),   N_g = sum_i a_i prod_{l != i} (1 - m_l z),
//
// i.e. the transposed Vandermonde product of PAPER.md:465-478 (rows m_i^k) computed by a product
// tree and one power-series division instead of T Hadamard steps.  O(s log^2 T) products.
//
//   leaves -> level 5   k_fast_leaf: 32 terms per warp, schoolbook merges mod p in shared memory
//   level l -> l+1      (N1,E1),(N2,E2) -> N = N1 + N2 + z(N1 E2 + N2 E1), E = E1 + E2 + z E1 E2,
//                       D = 1 + zE kept implicitly (E = (D-1)/z), every length capped at T2 =
//                       next_pow2(T) (N/D mod z^T2 only needs N, D mod z^T2)
//   root (N, E)         Y = D^-1 mod z^T2 by Newton (Y <- Y (2 - D Y), precision doubling), then
//                       out = N Y mod z^T.
//
// Polynomial products over F_p (any p < 2^63) are exact integer convolutions recovered by CRT from
// 5 NTT primes q_j < 2^30 (q_j = c 2^20 + 1; prod q_j > 2^149 > 2 L p^2 = 2^147 for L <= 2^20); operands
// longer than 4096 are cut into 4096-coefficient blocks whose 8192-point transforms are multiplied
// block-pairwise in the transform domain (a + b = c) and overlap-added -- so one shared-memory NTT
// of at most 8192 points serves every length.  Three batched kernels per product call:
//   k_fast_fwd    operand blocks mod q_j -> forward DIF NTT (bit-reversed spectra)
//   k_fast_pwinv  sum of block-pair pointwise products (32-bit Montgomery) -> inverse DIT NTT
//   k_fast_crt    overlap-add, Garner CRT over the 5 primes -> mod p, the call's epilogue
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/pe.h"
#include "fast.h"
#include "modcore.cuh"

namespace pe {
namespace fast {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- NTT primes (q < 2^30, 2^20 | q-1)
static const u32 kQ[kNP] = {1053818881u, 1051721729u, 1045430273u, 1012924417u, 1007681537u};
static const u32 kGen[kNP] = {7u, 6u, 3u, 5u, 3u};   // primitive roots

struct PrimeC {
  u32 q;
  u32 qinv_neg;   // -q^{-1} mod 2^32 (Montgomery)
  u64 bar;        // floor(2^64 / q)
};
struct Consts {
  PrimeC pr[kNP];
  uint2 ginv[kNP][kNP];   // Garner: q_i^{-1} mod q_j (i < j) and its Shoup companion
  u64 qmodp[kNP];         // q_i 2^64 mod p (Montgomery form of q_i mod p)
};

// ---------------------------------------------------------------- 32-bit modular helpers
// Shoup product with a fixed multiplier (w, ws = floor(w 2^32 / q)): any x < 2^32 -> [0, 2q).
__device__ __forceinline__ u32 shoup32(u32 x, u32 w, u32 ws, u32 q) {
  const u32 t = __umulhi(x, ws);
  return x * w - t * q;
}
// Montgomery product a b 2^-32 mod q for a, b < 2q (q < 2^30): result in [0, 2q).
__device__ __forceinline__ u32 mont32(u32 a, u32 b, u32 q, u32 qinv_neg) {
  const u64 ab = (u64)a * b;
  const u32 m = (u32)ab * qinv_neg;
  return (u32)((ab + (u64)m * q) >> 32);
}
__device__ __forceinline__ u32 red2q(u32 x, u32 q2) { return x >= q2 ? x - q2 : x; }
// x mod q for x < 2^64 (Barrett with floor(2^64/q)): result in [0, 2q).
__device__ __forceinline__ u32 reduce_q(u64 x, const PrimeC& P) {
  const u64 qh = __umul64hi(x, P.bar);
  return (u32)(x - qh * P.q);
}

// ---------------------------------------------------------------- shared-memory NTTs
// X holds transforms of S = 2^lg points each (npts points in all), values in [0, 2q), stored with
// one pad word per 32 (phys): every pass below reads each thread's elements at a power-of-two stride,
// and the pad makes the warp's 32 accesses hit 32 distinct banks for every stride.
// Forward: DIF (Gentleman-Sande), natural order in, bit-reversed out, twiddles tw[len + i] =
// w_{2len}^i.  Inverse: DIT (Cooley-Tukey), bit-reversed in, natural out, inverse twiddles.
// Stages run in passes of up to 4: a thread loads 16 elements (indices base + c 2^{s_bot}), does the
// pass's stages in registers and stores them back -- 4 shared-memory round trips and barriers for
// an 8192-point transform instead of 13.
__device__ __forceinline__ u32 phys(u32 i) { return i + (i >> 5); }
constexpr u32 padded(u32 n) { return n + (n >> 5); }

template <int R, bool FWD>
__device__ __forceinline__ void ntt_pass(u32* X, int s_bot, u32 npts, const uint2* __restrict__ tw, u32 q) {
  constexpr int E = 1 << R;
  const u32 q2 = 2 * q;
  const u32 ngroups = npts >> R;
  for (u32 gi = threadIdx.x; gi < ngroups; gi += blockDim.x) {
    const u32 lo = gi & ((1u << s_bot) - 1);
    const u32 base = ((gi >> s_bot) << (s_bot + R)) | lo;   // R zero bits inserted at s_bot
    u32 v[E];
#pragma unroll
    for (int c = 0; c < E; ++c) v[c] = X[phys(base + ((u32)c << s_bot))];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int st = FWD ? R - 1 - k : k;               // DIF: top stage first; DIT: bottom first
      const int s = s_bot + st;
      const u32 len = 1u << s;
#pragma unroll
      for (int c = 0; c < E; ++c) {
        if (c & (1 << st)) continue;
        const int c2 = c | (1 << st);
        const u32 i = (base + ((u32)c << s_bot)) & (len - 1);
        const uint2 w = tw[len + i];
        const u32 u = v[c], x = v[c2];
        if (FWD) {
          v[c] = red2q(u + x, q2);
          v[c2] = shoup32(u - x + q2, w.x, w.y, q);
        } else {
          const u32 t = shoup32(x, w.x, w.y, q);
          v[c] = red2q(u + t, q2);
          v[c2] = red2q(u - t + q2, q2);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < E; ++c) X[phys(base + ((u32)c << s_bot))] = v[c];
  }
  __syncthreads();
}
template <bool FWD>
__device__ __forceinline__ void ntt_run(u32* X, int s_bot, int R, u32 npts, const uint2* tw, u32 q) {
  switch (R) {
    case 4: ntt_pass<4, FWD>(X, s_bot, npts, tw, q); break;
    case 3: ntt_pass<3, FWD>(X, s_bot, npts, tw, q); break;
    case 2: ntt_pass<2, FWD>(X, s_bot, npts, tw, q); break;
    default: ntt_pass<1, FWD>(X, s_bot, npts, tw, q); break;
  }
}
__device__ __forceinline__ void ntt_dif(u32* X, int lg, u32 npts, const uint2* __restrict__ tw, u32 q) {
  for (int top = lg - 1; top >= 0;) {
    const int R = top + 1 < 4 ? top + 1 : 4;
    ntt_run<true>(X, top - R + 1, R, npts, tw, q);
    top -= R;
  }
}
__device__ __forceinline__ void ntt_dit(u32* X, int lg, u32 npts, const uint2* __restrict__ tw, u32 q) {
  for (int bot = 0; bot < lg;) {
    const int R = lg - bot < 4 ? lg - bot : 4;
    ntt_run<false>(X, bot, R, npts, tw, q);
    bot += R;
  }
}

// ---------------------------------------------------------------- kernel arguments
struct Call {
  // operands: op o of job j = base[o] + idx[j * nidx + (o >> ish)] * rstride (idx NULL: the job index);
  // an index of kNone reads as the zero polynomial
  const u64* base[4];
  const u32* idx;
  u32 nidx, ish;
  u64 rstride;
  u32 nops, nouts, njobs;
  u32 Lc, Lo, Bk, nb, nbo, lg;          // operand length, output length, block, blocks, out blocks, log2 S
  u32 lgnb, lgnops, lgnouts, lgnbo, lgLo, lgBk;   // the same as shifts (all powers of two)
  u32 nbz[4];           // op o has nonzero coefficients only in its first nbz[o] blocks (others: skipped)
  const u32* len0;      // optional [njobs]: op 0 of job j has only len0[j] nonzero coefficients (Newton's
                        // D and N: a bucket of s terms has deg D = s, so its upper blocks are zero)
  u32 keep;             // bit o: op o's spectra are already in place from the previous call (not redone)
  int kind;                             // kMerge / kMul / kTwoMinus
  // outputs
  u64* dst[2];
  u64 dstride;
  u32* spec;                            // [kNP][njobs][nops][nb][S]
  u32* res;                             // [kNP][njobs][nouts][nbo][S]
  const uint2* twf;                     // [kNP][kSmax] forward twiddles
  const uint2* twi;                     // [kNP][kSmax] inverse twiddles
  const uint2* scale;                   // [kNP][kLgMax + 1]: 2^(32 - lg) mod q and Shoup companion
  Consts C;
  ModParams mp;
};
enum { kMerge = 0, kMul = 1, kTwoMinus = 2 };
constexpr u32 kNone = 0xffffffffu;

__device__ __forceinline__ const u64* op_ptr(const Call& a, u32 job, u32 o) {
  const u32 ix = a.idx ? a.idx[(u64)job * a.nidx + (o >> a.ish)] : job;
  return ix == kNone ? nullptr : a.base[o] + (u64)ix * a.rstride;
}

// Forward transforms: unit = (job, op, block) of prime blockIdx.y; a CTA holds kTile / S units.
constexpr u32 kNttThreads = 256;
__global__ void __launch_bounds__(kNttThreads, 4) k_fast_fwd(Call a) {
  extern __shared__ u32 X[];
  const int j = blockIdx.y;
  const PrimeC P = a.C.pr[j];
  const u32 S = 1u << a.lg, per = kTile >> a.lg < 1 ? 1 : kTile >> a.lg;
  const u32 nunits = a.njobs * a.nops * a.nb;
  const u32 u0 = blockIdx.x * per;
  const u32 nu = min(per, nunits - u0), npts = nu * S;
  auto skipped = [&](u32 u) {
    const u32 blk = u & (a.nb - 1), o = (u >> a.lgnb) & (a.nops - 1);
    if (o == 0 && a.len0 && blk >= ((a.len0[u >> (a.lgnb + a.lgnops)] + a.Bk - 1) >> a.lgBk)) return true;
    return ((a.keep >> o) & 1u) || blk >= a.nbz[o];
  };
  if (nu == 1 && skipped(u0)) return;          // whole CTA (one 8192-point unit) not needed
  // 4 independent loads in flight per thread before any reduction (the loads are the latency)
  for (u32 x0 = threadIdx.x; x0 < npts; x0 += 4 * blockDim.x) {
    u64 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const u32 x = x0 + k * blockDim.x;
      v[k] = 0;
      const u32 u = u0 + (x >> a.lg), i = x & (S - 1);
      if (x < npts && i < a.Bk) {
        const u32 blk = u & (a.nb - 1), o = (u >> a.lgnb) & (a.nops - 1), job = u >> (a.lgnb + a.lgnops);
        const u64* src = op_ptr(a, job, o);
        if (src) v[k] = __ldg(src + (u64)blk * a.Bk + i);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const u32 x = x0 + k * blockDim.x;
      if (x < npts) X[phys(x)] = reduce_q(v[k], P);
    }
  }
  __syncthreads();
  ntt_dif(X, a.lg, npts, a.twf + (u64)j * kSmax, P.q);
  u32* out = a.spec + ((u64)j * nunits + u0) * S;
  for (u32 x = threadIdx.x; x < npts; x += blockDim.x)
    if (!skipped(u0 + (x >> a.lg))) out[x] = X[phys(x)];
}

// Pointwise products + inverse: unit = (job, out, out block c) of prime blockIdx.y.
// out 0 of kMerge: N1 E2 + N2 E1 (ops 0,3 and 2,1); out 1: E1 E2 (ops 1,3); kMul: op0 op1.
__global__ void __launch_bounds__(kNttThreads, 4) k_fast_pwinv(Call a) {
  extern __shared__ u32 X[];
  const int j = blockIdx.y;
  const PrimeC P = a.C.pr[j];
  const u32 q2 = 2 * P.q;
  const u32 S = 1u << a.lg, per = kTile >> a.lg < 1 ? 1 : kTile >> a.lg;
  const u32 nunits = a.njobs * a.nouts * a.nbo;
  const u32 u0 = blockIdx.x * per;
  const u32 nu = min(per, nunits - u0), npts = nu * S;
  const u64 opstride = (u64)a.nb * S;                       // one operand's spectra
  const u32* spec = a.spec + (u64)j * a.njobs * a.nops * opstride;
  for (u32 x = threadIdx.x; x < npts; x += blockDim.x) {
    const u32 u = u0 + (x >> a.lg), i = x & (S - 1);
    const u32 c = u & (a.nbo - 1), out = (u >> a.lgnbo) & (a.nouts - 1), job = u >> (a.lgnbo + a.lgnouts);
    const u32* J = spec + (u64)job * a.nops * opstride + i;
    u32 acc = 0;
    const int npair = (a.kind == kMerge && out == 0) ? 2 : 1;
    for (int pr = 0; pr < npair; ++pr) {
      u32 oa, ob;
      if (a.kind == kMerge) {
        oa = out == 0 ? (pr == 0 ? 0u : 2u) : 1u;
        ob = out == 0 ? (pr == 0 ? 3u : 1u) : 3u;
      } else {
        oa = 0u; ob = 1u;
      }
      u32 na = a.nbz[oa], nbb = a.nbz[ob];              // blocks beyond nbz are zero: no product
      if (a.len0) {
        const u32 n0 = (a.len0[job] + a.Bk - 1) >> a.lgBk;
        if (oa == 0) na = min(na, n0);
        if (ob == 0) nbb = min(nbb, n0);
      }
      if (na == 0 || nbb == 0 || c + 1 > na + nbb - 1) continue;
      const u32 blo = c + 1 > nbb ? c + 1 - nbb : 0, bhi = min(c, na - 1);
      for (u32 ba = blo; ba <= bhi; ++ba) {
        const u32 bb = c - ba;
        const u32 A = J[(u64)oa * opstride + (u64)ba * S], B = J[(u64)ob * opstride + (u64)bb * S];
        acc = red2q(acc + mont32(A, B, P.q, P.qinv_neg), q2);
      }
    }
    X[phys(x)] = acc;
  }
  __syncthreads();
  ntt_dit(X, a.lg, npts, a.twi + (u64)j * kSmax, P.q);
  const uint2 sc = a.scale[j * (kLgMax + 1) + a.lg];       // S^-1 2^32: undoes the transform and mont32
  u32* out = a.res + ((u64)j * nunits + u0) * S;
  for (u32 x = threadIdx.x; x < npts; x += blockDim.x) {
    u32 v = red2q(shoup32(X[phys(x)], sc.x, sc.y, P.q), P.q);
    out[x] = v;
  }
}

// Garner over the 5 primes -> the exact integer (< prod q) reduced mod p.
__device__ __forceinline__ u64 crt_modp(const u32 (&r)[kNP], const Consts& C, const ModParams& mp) {
  u32 v[kNP];
#pragma unroll
  for (int jj = 0; jj < kNP; ++jj) {
    const u32 q = C.pr[jj].q;
    u32 t = r[jj];
#pragma unroll
    for (int i = 0; i < jj; ++i) {
      // t <- (t - v_i) q_i^{-1} mod q_j
      const u32 d = t + q - (v[i] >= q ? v[i] - q : v[i]);   // v_i < q_i < 2 q_j: d in (0, 2q)
      t = red2q(shoup32(d, C.ginv[jj][i].x, C.ginv[jj][i].y, q), q);
    }
    v[jj] = t;
  }
  // x = v0 + q0 (v1 + q1 (v2 + q2 (v3 + q3 v4)))  mod p
  u64 y = v[kNP - 1] < mp.p ? v[kNP - 1] : v[kNP - 1] % mp.p;
#pragma unroll
  for (int i = kNP - 2; i >= 0; --i) {
    y = mont_mul(y, C.qmodp[i], mp);   // y q_i mod p (qmodp in Montgomery form)
    const u64 vi = v[i] < mp.p ? v[i] : v[i] % mp.p;
    y += vi;
    y = y >= mp.p ? y - mp.p : y;
  }
  return y;
}
__device__ __forceinline__ u64 addp(u64 x, u64 y, u64 p) {
  const u64 s = x + y;   // x, y < p < 2^63: no wrap
  return s >= p ? s - p : s;
}

// Overlap-add + CRT + epilogue: thread = (job, output coefficient k < Lo).
__global__ void k_fast_crt(Call a) {
  const u64 total = (u64)a.njobs * a.Lo;
  const u32 S = 1u << a.lg;
  const u64 p = a.mp.p;
  for (u64 x = blockIdx.x * (u64)blockDim.x + threadIdx.x; x < total; x += (u64)gridDim.x * blockDim.x) {
    const u32 job = (u32)(x >> a.lgLo), k = (u32)(x & (a.Lo - 1));
    u64 conv[2];
    const int shift = a.kind == kMerge ? 1 : 0;
    for (u32 o = 0; o < a.nouts; ++o) {
      if ((int)k - shift < 0) { conv[o] = 0; continue; }
      const u32 K = k - shift;
      u32 r[kNP];
#pragma unroll
      for (int jj = 0; jj < kNP; ++jj) {
        const u32 q = a.C.pr[jj].q;
        const u32* R = a.res + (((u64)jj * a.njobs + job) * a.nouts + o) * a.nbo * S;
        const u32 c = K >> a.lgBk;
        u32 acc = 0;
        if (c < a.nbo) acc = R[(u64)c * S + (K - (c << a.lgBk))];
        if (c >= 1 && c - 1 < a.nbo) {
          acc += R[(u64)(c - 1) * S + (K - ((c - 1) << a.lgBk))];
          acc = acc >= q ? acc - q : acc;
        }
        r[jj] = acc;
      }
      conv[o] = crt_modp(r, a.C, a.mp);
    }
    if (a.kind == kMerge) {
      // N = N1 + N2 + z P, E = E1 + E2 + z Q (child coefficients beyond Lc are 0)
      const u64* N1 = op_ptr(a, job, 0);
      const u64* E1 = op_ptr(a, job, 1);
      const u64* N2 = op_ptr(a, job, 2);
      const u64* E2 = op_ptr(a, job, 3);
      u64 n = conv[0], e = conv[1];
      if (k < a.Lc) {
        if (N1) { n = addp(n, N1[k], p); e = addp(e, E1[k], p); }
        if (N2) { n = addp(n, N2[k], p); e = addp(e, E2[k], p); }
      }
      a.dst[0][(u64)job * a.dstride + k] = n;
      a.dst[1][(u64)job * a.dstride + k] = e;
    } else if (a.kind == kMul) {
      a.dst[0][(u64)job * a.dstride + k] = conv[0];
    } else {   // kTwoMinus: W = 2 - conv (Newton: Y <- Y (2 - D Y))
      const u64 two = 2 % p;
      const u64 c0 = k == 0 ? two : 0;
      a.dst[0][(u64)job * a.dstride + k] = c0 >= conv[0] ? c0 - conv[0] : c0 + p - conv[0];
    }
  }
}

// Fused tree merge for short operands (S = 2 Lc <= kFusedS): a CTA holds kFusedS / S jobs and runs
// the whole product in shared memory -- per prime the 4 operands mod q (one array of 4 x npts
// points: DIF over every S-point unit at once), pointwise P = N1 E2 + N2 E1 and Q = E1 E2, the 2
// inverse transforms, residues kept in shared memory -- then Garner CRT and the merge epilogue
// straight into the next level.  Global traffic: the children (L2-resident across the 5 primes)
// and the parents, instead of spectra and residues.
constexpr u32 kFusedS = 1024;
constexpr u32 kFusedThreads = 256;
// W (padded) + residues of P, Q for the 5 primes + the 4 operands as u64 (read from global once)
constexpr u32 kFusedSmem = (padded(4 * kFusedS) + 2 * kNP * kFusedS) * sizeof(u32) + 4 * (kFusedS / 2) * sizeof(u64);
__global__ void __launch_bounds__(kFusedThreads, 3) k_fast_merge_fused(Call a) {
  extern __shared__ u32 sm[];
  u32* W = sm;                       // [4][npts]: N1, E1, N2, E2 of the CTA's jobs (P, Q after the products)
  u32* Rz = sm + padded(4 * kFusedS);   // [kNP][2][npts] residues of P and Q (W is padded: phys)
  u64* Op = (u64*)(Rz + 2 * kNP * kFusedS);   // [4][nj * Lc] the operands, canonical mod p
  const u32 S = 1u << a.lg, per = kFusedS >> a.lg;
  const u32 job0 = blockIdx.x * per;
  const u32 nj = min(per, a.njobs - job0), npts = nj * S;
  const u32 lgLc = a.lg - 1, nop = nj << lgLc;     // Lc = S / 2 coefficients per operand
  for (u32 x = threadIdx.x; x < 4 * nop; x += blockDim.x) {
    const u32 o = x / nop, r = x - o * nop, jj = r >> lgLc, i = r & (a.Lc - 1);
    const u64* src = op_ptr(a, job0 + jj, o);
    Op[x] = src ? src[i] : 0;
  }
  __syncthreads();
  for (int jp = 0; jp < kNP; ++jp) {
    const PrimeC P = a.C.pr[jp];
    for (u32 x = threadIdx.x; x < 4 * npts; x += blockDim.x) {
      const u32 unit = x >> a.lg, i = x & (S - 1);            // unit = o * nj + jj
      W[phys(x)] = i < a.Lc ? reduce_q(Op[(unit << lgLc) + i], P) : 0u;
    }
    __syncthreads();
    ntt_dif(W, a.lg, 4 * npts, a.twf + (u64)jp * kSmax, P.q);
    const u32 q2 = 2 * P.q;
    for (u32 x = threadIdx.x; x < npts; x += blockDim.x) {
      const u32 n1 = W[phys(x)], e1 = W[phys(npts + x)], n2 = W[phys(2 * npts + x)], e2 = W[phys(3 * npts + x)];
      W[phys(x)] = red2q(mont32(n1, e2, P.q, P.qinv_neg) + mont32(n2, e1, P.q, P.qinv_neg), q2);
      W[phys(npts + x)] = mont32(e1, e2, P.q, P.qinv_neg);
    }
    __syncthreads();
    ntt_dit(W, a.lg, 2 * npts, a.twi + (u64)jp * kSmax, P.q);
    const uint2 sc = a.scale[jp * (kLgMax + 1) + a.lg];
    for (u32 x = threadIdx.x; x < 2 * npts; x += blockDim.x)
      Rz[(u32)jp * 2 * kFusedS + x] = red2q(shoup32(W[phys(x)], sc.x, sc.y, P.q), P.q);
    __syncthreads();
  }
  const u64 p = a.mp.p;
  for (u32 x = threadIdx.x; x < nj * a.Lo; x += blockDim.x) {
    const u32 jj = x >> a.lgLo, k = x & (a.Lo - 1), job = job0 + jj;
    u64 conv[2] = {0, 0};
    if (k >= 1) {
      for (int o = 0; o < 2; ++o) {
        u32 r[kNP];
#pragma unroll
        for (int jp = 0; jp < kNP; ++jp) r[jp] = Rz[(u32)jp * 2 * kFusedS + (u32)o * npts + jj * S + k - 1];
        conv[o] = crt_modp(r, a.C, a.mp);
      }
    }
    u64 n = conv[0], e = conv[1];
    if (k < a.Lc) {   // children from the shared-memory copy (absent children read as zero)
      const u32 b = (jj << lgLc) + k;
      n = addp(addp(n, Op[b], p), Op[2 * nop + b], p);
      e = addp(addp(e, Op[nop + b], p), Op[3 * nop + b], p);
    }
    a.dst[0][(u64)job * a.dstride + k] = n;
    a.dst[1][(u64)job * a.dstride + k] = e;
  }
}

// Leaves to level 5: warp w of the CTA owns padded terms 32 g .. 32 g + 31 (g = global group); a_i =
// c_i m_i^{j0}, leaf (N, E) = (a_i, -m_i); five levels of pairwise merges in shared memory by
// schoolbook products mod p; the level-5 node (length min(32, T2)) goes to N5[g], E5[g].
__global__ void __launch_bounds__(128) k_fast_leaf(const u64* __restrict__ c, const u64* __restrict__ m, u64 ngroups,
                                                   u64 j0, u32 L5, u64* __restrict__ N5, u64* __restrict__ E5,
                                                   ModParams mp) {
  __shared__ u64 sN[4][2][32], sE[4][2][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u64 p = mp.p;
  for (u64 g = blockIdx.x * 4ull + w; g < ngroups; g += (u64)gridDim.x * 4) {
    const u64 q = g * 32 + lane;
    const u64 mi = m[q];
    // Montgomery form inside the warp (one REDC per product), normal form out
    sN[w][0][lane] = to_mont(seed_pow(c[q], mi, j0, mp), mp);
    sE[w][0][lane] = to_mont(mi == 0 ? 0 : p - mi, mp);
    __syncwarp();
    int cur = 0;
    for (int lc = 1; lc < 32; lc <<= 1) {   // child length lc, output length 2 lc
      const int lo = 2 * lc;
      const int node = lane / lo, k = lane % lo;
      const u64* n1 = &sN[w][cur][node * lo];
      const u64* e1 = &sE[w][cur][node * lo];
      const u64* n2 = n1 + lc;
      const u64* e2 = e1 + lc;
      u64 n = 0, e = 0;
      if (k < lc) { n = addp(n1[k], n2[k], p); e = addp(e1[k], e2[k], p); }
      for (int x = 0; x < lc && x <= k - 1; ++x) {
        const int y = k - 1 - x;
        if (y >= lc) continue;
        n = addp(n, mont_mul(n1[x], e2[y], mp), p);
        n = addp(n, mont_mul(n2[x], e1[y], mp), p);
        e = addp(e, mont_mul(e1[x], e2[y], mp), p);
      }
      sN[w][cur ^ 1][lane] = n;
      sE[w][cur ^ 1][lane] = e;
      __syncwarp();
      cur ^= 1;
    }
    if ((u32)lane < L5) {
      N5[g * L5 + lane] = from_mont(sN[w][cur][lane], mp);
      E5[g * L5 + lane] = from_mont(sE[w][cur][lane], mp);
    }
    __syncwarp();
  }
}

// Copy finished bucket roots (node rows of length L) into the [G][T2] root arrays (zero tail).
__global__ void k_fast_root_copy(const uint2* __restrict__ roots, u32 nroots, const u64* __restrict__ N,
                                 const u64* __restrict__ E, u32 L, u64* __restrict__ RN, u64* __restrict__ RE,
                                 u32 T2) {
  const u64 total = (u64)nroots * T2;
  for (u64 x = blockIdx.x * (u64)blockDim.x + threadIdx.x; x < total; x += (u64)gridDim.x * blockDim.x) {
    const uint2 r = roots[x / T2];
    const u32 k = (u32)(x % T2);
    RN[(u64)r.x * T2 + k] = k < L ? N[(u64)r.y * L + k] : 0;
    RE[(u64)r.x * T2 + k] = k < L ? E[(u64)r.y * L + k] : 0;
  }
}

// D = 1 + z E (rows of length T2), Y = 1.
__global__ void k_fast_newton_init(const u64* __restrict__ RE, u64 G, u32 T2, u64* __restrict__ D, u64* __restrict__ Y,
                                   u64 p) {
  const u64 total = G * T2;
  for (u64 x = blockIdx.x * (u64)blockDim.x + threadIdx.x; x < total; x += (u64)gridDim.x * blockDim.x) {
    const u32 k = (u32)(x % T2);
    D[x] = k == 0 ? 1 % p : RE[x - 1];
    Y[x] = k == 0 ? 1 % p : 0;
  }
}

// out[g][k] = B[g][k] for k < T (B rows of length T2).
__global__ void k_fast_store(const u64* __restrict__ B, u64 G, u32 T2, u64 T, u64* __restrict__ out, u64 ld) {
  const u64 total = G * T;
  for (u64 x = blockIdx.x * (u64)blockDim.x + threadIdx.x; x < total; x += (u64)gridDim.x * blockDim.x) {
    const u64 g = x / T, k = x % T;
    out[g * ld + k] = B[g * T2 + k];
  }
}

// ---------------------------------------------------------------- host
static u64 hpow(u64 b, u64 e, u64 q) {
  u64 r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = (u64)((u128)r * b % q);
    b = (u64)((u128)b * b % q);
    e >>= 1;
  }
  return r;
}
static uint2 shoup_pair(u64 w, u32 q) { return make_uint2((u32)w, (u32)(((u64)w << 32) / q)); }

static unsigned grid_for(u64 n, unsigned block) {
  u64 b = (n + block - 1) / block;
  return (unsigned)std::max<u64>(1, std::min<u64>(b, 148ull * 32));
}

#define FCU(call)                                                                 \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      if (getenv("PE_DEBUG")) fprintf(stderr, "pe fast: %s:%d %s: %s\n", __FILE__, \
                                      __LINE__, #call, cudaGetErrorString(_e));   \
      return _e == cudaErrorMemoryAllocation ? PE_ENOMEM : PE_ECUDA;              \
    }                                                                             \
  } while (0)

struct Level {
  u32 nnodes;              // nodes at this level
  u32 njobs;               // merge jobs producing it (== nnodes for l > 5)
  std::vector<u32> kids;   // [njobs][2] child node indices at level l - 1 (kNone: absent)
  std::vector<uint2> roots;   // buckets whose tree ends here: (g, node)
  u32* d_kids = nullptr;
  uint2* d_roots = nullptr;
};

struct Plan {
  u64 G = 0, t_pad = 0, ngroups = 0;
  std::vector<Level> lv;   // lv[0] = level 5 (leaf groups), lv[i] = level 5 + i
  u64 max_nodes = 0;
  uint2 *d_twf = nullptr, *d_twi = nullptr, *d_scale = nullptr;
  Consts C{};
  // workspace (stream-ordered pools, grown on demand)
  u64* d_nodes = nullptr;     // 4 x node_cap: N[0], N[1], E[0], E[1] (ping-pong by level)
  u64 node_cap = 0;
  u64* d_rows = nullptr;      // 5 x row_cap: RN, RE, D, Y, W  ([G][T2] each)
  u64 row_cap = 0;
  u32 *d_spec = nullptr, *d_res = nullptr;
  u64 spec_elems = 0, res_elems = 0;
  u32* d_rootlen = nullptr;    // [G]: a bucket of s padded terms has deg D = s, deg N < s -> s + 1
};

static void free_ws(Plan* P, cudaStream_t s) {
  for (void* q : {(void*)P->d_nodes, (void*)P->d_rows, (void*)P->d_spec, (void*)P->d_res})
    if (q) cudaFreeAsync(q, s);
  P->d_nodes = P->d_rows = nullptr;
  P->d_spec = P->d_res = nullptr;
  P->node_cap = P->row_cap = P->spec_elems = P->res_elems = 0;
}

void destroy(Plan* P, cudaStream_t s) {
  if (!P) return;
  free_ws(P, s);
  for (auto& L : P->lv) {
    if (L.d_kids) cudaFreeAsync(L.d_kids, s);
    if (L.d_roots) cudaFreeAsync(L.d_roots, s);
  }
  for (void* q : {(void*)P->d_twf, (void*)P->d_twi, (void*)P->d_scale, (void*)P->d_rootlen})
    if (q) cudaFreeAsync(q, s);
  delete P;
}

int create(const std::vector<u64>& poff, const ModParams& mp, cudaStream_t s, Plan** out) {
  *out = nullptr;
  Plan* P = new Plan();
  P->G = poff.size() - 1;
  P->t_pad = poff.back();
  P->ngroups = P->t_pad / 32;
  // tree shape: level 5 = one node per 32 padded terms (bucket ranges are multiples of 32)
  std::vector<u64> cnt(P->G), off(P->G);
  Level L5;
  L5.nnodes = (u32)P->ngroups;
  L5.njobs = 0;
  std::vector<u32> rootlen(P->G);
  for (u64 g = 0; g < P->G; ++g) {
    cnt[g] = (poff[g + 1] - poff[g]) / 32;
    rootlen[g] = (u32)std::min<u64>(poff[g + 1] - poff[g] + 1, 1ull << 30);   // > kTMax: no skipping
    off[g] = poff[g] / 32;
    if (cnt[g] == 1) L5.roots.push_back(make_uint2((u32)g, (u32)off[g]));
  }
  P->lv.push_back(std::move(L5));
  P->max_nodes = P->ngroups;
  for (;;) {
    Level L;
    std::vector<u64> ncnt(P->G, 0), noff(P->G, 0);
    u32 nn = 0;
    for (u64 g = 0; g < P->G; ++g) {
      noff[g] = nn;
      if (cnt[g] < 2) continue;
      ncnt[g] = (cnt[g] + 1) / 2;
      for (u64 i = 0; i < ncnt[g]; ++i) {
        L.kids.push_back((u32)(off[g] + 2 * i));
        L.kids.push_back(2 * i + 1 < cnt[g] ? (u32)(off[g] + 2 * i + 1) : kNone);
      }
      if (ncnt[g] == 1) L.roots.push_back(make_uint2((u32)g, nn));
      nn += (u32)ncnt[g];
    }
    if (nn == 0) break;
    L.nnodes = L.njobs = nn;
    cnt = ncnt;
    off = noff;
    P->lv.push_back(std::move(L));
  }
  int rc = PE_OK;
  for (auto& L : P->lv) {
    if (!L.kids.empty()) {
      if (cudaMallocAsync((void**)&L.d_kids, L.kids.size() * sizeof(u32), s) != cudaSuccess) rc = PE_ENOMEM;
      else if (cudaMemcpyAsync(L.d_kids, L.kids.data(), L.kids.size() * sizeof(u32), cudaMemcpyHostToDevice, s) !=
               cudaSuccess) rc = PE_ECUDA;
    }
    if (rc == PE_OK && !L.roots.empty()) {
      if (cudaMallocAsync((void**)&L.d_roots, L.roots.size() * sizeof(uint2), s) != cudaSuccess) rc = PE_ENOMEM;
      else if (cudaMemcpyAsync(L.d_roots, L.roots.data(), L.roots.size() * sizeof(uint2), cudaMemcpyHostToDevice,
                               s) != cudaSuccess) rc = PE_ECUDA;
    }
    if (rc != PE_OK) break;
  }
  // NTT tables and CRT constants
  std::vector<uint2> twf((size_t)kNP * kSmax), twi((size_t)kNP * kSmax), sc((size_t)kNP * (kLgMax + 1));
  for (int j = 0; j < kNP; ++j) {
    const u32 q = kQ[j];
    const u64 wmax = hpow(kGen[j], (q - 1) / kSmax, q);    // primitive kSmax-th root
    for (u32 len = 1; len < kSmax; len <<= 1) {
      const u64 w = hpow(wmax, kSmax / (2 * len), q), wi = hpow(w, q - 2, q);
      u64 x = 1, xi = 1;
      for (u32 i = 0; i < len; ++i) {
        twf[(size_t)j * kSmax + len + i] = shoup_pair(x, q);
        twi[(size_t)j * kSmax + len + i] = shoup_pair(xi, q);
        x = x * w % q;
        xi = xi * wi % q;
      }
    }
    twf[(size_t)j * kSmax] = twi[(size_t)j * kSmax] = make_uint2(0, 0);
    for (int lg = 0; lg <= kLgMax; ++lg) {
      const u64 sinv = hpow(hpow(2, lg, q), q - 2, q);
      sc[(size_t)j * (kLgMax + 1) + lg] = shoup_pair(sinv * (((u64)1 << 32) % q) % q, q);
    }
    PrimeC& pc = P->C.pr[j];
    pc.q = q;
    u32 inv = q;
    for (int i = 0; i < 5; ++i) inv *= 2 - q * inv;
    pc.qinv_neg = (u32)0 - inv;
    pc.bar = (u64)(((u128)1 << 64) / q);
    for (int i = 0; i < j; ++i) P->C.ginv[j][i] = shoup_pair(hpow(kQ[i] % q, q - 2, q), q);
    P->C.qmodp[j] = (u64)((((u128)(kQ[j] % mp.p)) << 64) % mp.p);
  }
  if (rc == PE_OK) {
    if (cudaMallocAsync((void**)&P->d_twf, twf.size() * sizeof(uint2), s) != cudaSuccess ||
        cudaMallocAsync((void**)&P->d_twi, twi.size() * sizeof(uint2), s) != cudaSuccess ||
        cudaMallocAsync((void**)&P->d_scale, sc.size() * sizeof(uint2), s) != cudaSuccess ||
        cudaMallocAsync((void**)&P->d_rootlen, std::max<u64>(P->G, 1) * sizeof(u32), s) != cudaSuccess)
      rc = PE_ENOMEM;
    else if (cudaMemcpyAsync(P->d_twf, twf.data(), twf.size() * sizeof(uint2), cudaMemcpyHostToDevice, s) ||
             cudaMemcpyAsync(P->d_twi, twi.data(), twi.size() * sizeof(uint2), cudaMemcpyHostToDevice, s) ||
             cudaMemcpyAsync(P->d_scale, sc.data(), sc.size() * sizeof(uint2), cudaMemcpyHostToDevice, s) ||
             cudaMemcpyAsync(P->d_rootlen, rootlen.data(), P->G * sizeof(u32), cudaMemcpyHostToDevice, s))
      rc = PE_ECUDA;
  }
  if (rc == PE_OK && cudaStreamSynchronize(s) != cudaSuccess) rc = PE_ECUDA;   // host vectors die here
  if (rc != PE_OK) {
    cudaGetLastError();
    destroy(P, s);
    return rc;
  }
  *out = P;
  return PE_OK;
}

template <class T>
static int grow(T** p, u64& have, u64 need, cudaStream_t s) {
  if (need <= have) return PE_OK;
  if (*p) cudaFreeAsync(*p, s);
  *p = nullptr;
  have = 0;
  FCU(cudaMallocAsync((void**)p, std::max<u64>(need, 1) * sizeof(T), s));
  have = need;
  return PE_OK;
}

static u32 ilog2(u64 x) { u32 r = 0; while ((1ull << r) < x) ++r; return r; }

// One batched product call: transforms, pointwise + inverse, CRT + epilogue.
static int run_call(Plan* P, Call& a, cudaStream_t s) {
  a.Bk = std::min<u32>(a.Lc, kBkMax);
  a.nb = a.Lc / a.Bk;
  a.lg = ilog2(2ull * a.Bk);
  const u32 S = 1u << a.lg;
  // output blocks: the block-pair sums a + b = c needed for coefficients < Lo (c <= 2nb - 2; a
  // power of two so the kernels split unit indices with shifts -- an extra c = 2nb - 1 has no pairs)
  if (a.nb == 1) a.nbo = 1;
  else a.nbo = std::min<u32>((a.Lo + a.Bk - 1) / a.Bk, 2 * a.nb);
  a.lgnb = ilog2(a.nb); a.lgnops = ilog2(a.nops); a.lgnouts = ilog2(a.nouts); a.lgnbo = ilog2(a.nbo);
  a.lgLo = ilog2(a.Lo); a.lgBk = ilog2(a.Bk);
  for (int o = 0; o < 4; ++o)   // callers give nonzero lengths in coefficients (0: the whole operand)
    a.nbz[o] = a.nbz[o] ? std::min<u32>(a.nb, (a.nbz[o] + a.Bk - 1) / a.Bk) : a.nb;
  a.twf = P->d_twf;
  a.twi = P->d_twi;
  a.scale = P->d_scale;
  a.C = P->C;
  if (a.kind == kMerge && S <= kFusedS && !getenv("PE_FAST_NOFUSE")) {   // short operands: one fused kernel
    if (a.njobs == 0) return PE_OK;
    const u32 per = kFusedS / S;
    FCU(cudaFuncSetAttribute(k_fast_merge_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem));
    k_fast_merge_fused<<<(a.njobs + per - 1) / per, kFusedThreads, kFusedSmem, s>>>(a);
    FCU(cudaGetLastError());
    return PE_OK;
  }

  if (a.njobs == 0) return PE_OK;
  const u64 nspec = (u64)kNP * a.njobs * a.nops * a.nb * S;
  const u64 nres = (u64)kNP * a.njobs * a.nouts * a.nbo * S;
  if (grow(&P->d_spec, P->spec_elems, nspec, s) || grow(&P->d_res, P->res_elems, nres, s)) return PE_ENOMEM;
  a.spec = P->d_spec;
  a.res = P->d_res;
  const u32 per = std::max<u32>(1, kTile >> a.lg);
  const u32 smem = padded(per * S) * sizeof(u32);
  const u32 threads = std::min<u32>(kNttThreads, std::max<u32>(32, per * S / 2));
  FCU(cudaFuncSetAttribute(k_fast_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, padded(kTile) * 4));
  FCU(cudaFuncSetAttribute(k_fast_pwinv, cudaFuncAttributeMaxDynamicSharedMemorySize, padded(kTile) * 4));
  const u32 nu_f = a.njobs * a.nops * a.nb, nu_i = a.njobs * a.nouts * a.nbo;
  k_fast_fwd<<<dim3((nu_f + per - 1) / per, kNP), threads, smem, s>>>(a);
  FCU(cudaGetLastError());
  k_fast_pwinv<<<dim3((nu_i + per - 1) / per, kNP), threads, smem, s>>>(a);
  FCU(cudaGetLastError());
  k_fast_crt<<<grid_for((u64)a.njobs * a.Lo, 256), 256, 0, s>>>(a);
  FCU(cudaGetLastError());
  return PE_OK;
}

int eval(Plan* P, const u64* d_c, const u64* d_m, const ModParams& mp, u64 j0, u64 T, u64* d_out, u64 ld,
         cudaStream_t s) {
  if (T == 0 || P->G == 0) return PE_OK;
  if (T > kTMax) return PE_ERANGE;   // CRT bound (prod q_j > 2 T2 p^2)
  const u32 T2 = 1u << ilog2(T);
  auto len_of = [&](size_t i) { return (u32)std::min<u64>(32ull << std::min<size_t>(i, 40), T2); };
  u64 need = 0;
  for (size_t i = 0; i < P->lv.size(); ++i) need = std::max<u64>(need, (u64)P->lv[i].nnodes * len_of(i));
  if (grow(&P->d_nodes, P->node_cap, 4 * need, s) || grow(&P->d_rows, P->row_cap, 5 * P->G * T2, s)) return PE_ENOMEM;
  u64* Nb[2] = {P->d_nodes, P->d_nodes + need};
  u64* Eb[2] = {P->d_nodes + 2 * need, P->d_nodes + 3 * need};
  const u64 GT = P->G * T2;
  u64 *RN = P->d_rows, *RE = RN + GT, *D = RE + GT, *Y = D + GT, *W = Y + GT;

  // leaves -> level 5
  int cur = 0;
  k_fast_leaf<<<grid_for(P->ngroups, 4), 128, 0, s>>>(d_c, d_m, P->ngroups, j0, len_of(0), Nb[0], Eb[0], mp);
  FCU(cudaGetLastError());
  auto copy_roots = [&](size_t i) -> int {
    const Level& L = P->lv[i];
    if (L.roots.empty()) return PE_OK;
    k_fast_root_copy<<<grid_for((u64)L.roots.size() * T2, 256), 256, 0, s>>>(L.d_roots, (u32)L.roots.size(), Nb[cur],
                                                                             Eb[cur], len_of(i), RN, RE, T2);
    FCU(cudaGetLastError());
    return PE_OK;
  };
  if (copy_roots(0)) return PE_ECUDA;
  // the product tree, level by level over all buckets at once
  for (size_t i = 1; i < P->lv.size(); ++i) {
    Call a{};
    a.base[0] = Nb[cur]; a.base[1] = Eb[cur]; a.base[2] = Nb[cur]; a.base[3] = Eb[cur];
    a.idx = P->lv[i].d_kids; a.nidx = 2; a.ish = 1;
    a.rstride = len_of(i - 1);
    a.nops = 4; a.nouts = 2; a.njobs = P->lv[i].njobs;
    a.Lc = len_of(i - 1); a.Lo = len_of(i);
    a.kind = kMerge;
    a.dst[0] = Nb[cur ^ 1]; a.dst[1] = Eb[cur ^ 1]; a.dstride = a.Lo;
    a.mp = mp;
    if (int rc = run_call(P, a, s)) return rc;
    cur ^= 1;
    if (copy_roots(i)) return PE_ECUDA;
  }
  // Y = D^-1 mod z^T2 by Newton: Y <- Y (2 - D Y) mod z^{2k}
  k_fast_newton_init<<<grid_for(GT, 256), 256, 0, s>>>(RE, P->G, T2, D, Y, mp.p);
  FCU(cudaGetLastError());
  for (u32 k = 1; k < T2; k <<= 1) {
    Call a{};
    a.base[0] = D; a.base[1] = Y; a.idx = nullptr; a.nidx = 1; a.ish = 0; a.rstride = T2;
    a.nops = 2; a.nouts = 1; a.njobs = (u32)P->G; a.Lc = 2 * k; a.Lo = 2 * k;
    a.kind = kTwoMinus; a.dst[0] = W; a.dstride = T2; a.mp = mp;
    a.nbz[0] = 0; a.nbz[1] = k;               // Y has k coefficients: its upper blocks are zero
    a.len0 = P->d_rootlen;                    // D's upper blocks are zero for buckets shorter than 2k
    if (int rc = run_call(P, a, s)) return rc;
    // Y <- Y W: op 1 is Y again, same length: its spectra from the call above are reused
    Call b{};
    b.base[0] = W; b.base[1] = Y; b.idx = nullptr; b.nidx = 1; b.ish = 0; b.rstride = T2;
    b.nops = 2; b.nouts = 1; b.njobs = (u32)P->G; b.Lc = 2 * k; b.Lo = 2 * k;
    b.kind = kMul; b.dst[0] = Y; b.dstride = T2; b.mp = mp;
    b.nbz[0] = 0; b.nbz[1] = k; b.keep = 2u;
    if (int rc = run_call(P, b, s)) return rc;
  }
  // out = N Y mod z^T
  Call f{};
  f.base[0] = RN; f.base[1] = Y; f.idx = nullptr; f.nidx = 1; f.ish = 0; f.rstride = T2;
  f.nops = 2; f.nouts = 1; f.njobs = (u32)P->G; f.Lc = T2; f.Lo = T2;
  f.kind = kMul; f.dst[0] = W; f.dstride = T2; f.mp = mp;
  f.len0 = P->d_rootlen;                      // N: deg < s
  if (int rc = run_call(P, f, s)) return rc;
  k_fast_store<<<grid_for(P->G * T, 256), 256, 0, s>>>(W, P->G, T2, T, d_out, ld);
  FCU(cudaGetLastError());
  return PE_OK;
}

}  // namespace fast
}  // namespace pe
