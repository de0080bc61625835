// modcore.cuh -- sm_100a modular-arithmetic core (device, header-only).
//
// The paper's operators (x) and (+) (§3.1) on a chip with no 64x64-bit
// multiplier: every 64-bit product is built from 32-bit IMAD / IMAD.WIDE / IMAD.HI.
//
//   * Shoup "fixed multiplier" product (Barrett family): m_i is fixed per
//     term across all points (a <- a o m), so w_i = floor(m_i 2^64 / p)
//     is precomputed once and every step costs one approximate 64x64-high product plus two
//     64x64-low products.
//       - mul_shoup4: p < 2^62, quotient from 3 of the 4 partial products (drops only the
//         a0*w0 term => q in [q_shoup-1, q_shoup]), result lazily in [0, 3p) subset [0, 4p)
//         for ANY input a < 2^64.  4p < 2^64 so the remainder computed mod 2^64 is exact.
//       - mul_shoup2: p < 2^63, exact Shoup quotient, one conditional subtract, output in
//         [0, 2p) for input a < 2^64.
//   * Montgomery REDC for general products (seeding by exponentiation,
//     monomial setup, final reductions).  p odd, p < 2^63.
//   * FP64-FMA Alg. 2 and Alg. 3, p < 2^50, with
//     explicit round-to-nearest intrinsics so nvcc never contracts or reorders (R11).
#pragma once
#include <stdint.h>

namespace pe {

typedef uint64_t u64;
typedef unsigned int u32;

__device__ __forceinline__ u32 lo32(u64 x) { return (u32)x; }
__device__ __forceinline__ u32 hi32(u64 x) { return (u32)(x >> 32); }

struct ModParams {
  u64 p;      // prime, 3 <= p < 2^63
  u64 np;     // 2^64 - p
  u64 pinv;   // -p^{-1} mod 2^64 (Montgomery)
  u64 r1;     // 2^64 mod p   (Montgomery one)
  u64 r2;     // 2^128 mod p
  double pd;  // (double)p  (exact when p < 2^53)
  double u;   // RN(1/p)     (Alg. 2 "u stores 1/(double) p")
  u64 hc;     // mul_hyb constant C = K*p mod 2^64
};

// ---------------------------------------------------------------- 32-bit building blocks
__device__ __forceinline__ u64 mul_wide(u32 a, u32 b) { return (u64)a * b; }   // IMAD.WIDE.U32
__device__ __forceinline__ u32 mul_hi(u32 a, u32 b) { return __umulhi(a, b); } // IMAD.HI.U32

// Full 64x64 -> 128 product (hi, lo).
__device__ __forceinline__ void mul128(u64 a, u64 b, u64& hi, u64& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

// ---------------------------------------------------------------- Shoup products
// w = floor(m * 2^64 / p), m < p.
// Lazy-4: p < 2^62, any a < 2^64 -> r == a*m (mod p), r in [0, 3p) (contract: [0, 4p)).
//   q = a1*w1 + floor((a1*w0 + a0*w1) / 2^32) (deficit <= 1 vs Shoup's q = floor(a*w/2^64))
//   r = a*m - q*p = a*m + q*(2^64 - p)  (mod 2^64)
// PTX chosen by SASS slot count (scripts/core_variants.cu, scripts/sass_slots.py): 5 full-width
// products (IMAD.WIDE, 2 IMAD-pipe slots each) + 4 low IMADs = the 14-slot minimum, with the
// cross-term sum and the carries on the ALU pipe and no zero-register pairs.
__device__ __forceinline__ u64 mul_shoup4(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t"
      ".reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, x1l, x1h, x2l, x2h, z, s, c, q0, q1, r0, r1;\n\t"
      ".reg .u64 rr, x1, x2;\n\t"
      "mov.b64 {a0, a1}, %1;\n\t"
      "mov.b64 {m0, m1}, %2;\n\t"
      "mov.b64 {w0, w1}, %3;\n\t"
      "mov.b64 {n0, n1}, %4;\n\t"
      // cross terms as full products; s:c = floor((a1*w0 + a0*w1) / 2^32) on the ALU
      "mul.wide.u32 x1, a1, w0;\n\t"
      "mul.wide.u32 x2, a0, w1;\n\t"
      "mov.b64 {x1l, x1h}, x1;\n\t"
      "mov.b64 {x2l, x2h}, x2;\n\t"
      "add.cc.u32 z, x1l, x2l;\n\t"
      "addc.cc.u32 s, x1h, x2h;\n\t"
      "addc.u32 c, 0, 0;\n\t"
      // q = a1*w1 + s + c*2^32 with carry chains (no 64-bit addend pairs -> no predicate spills)
      "mad.lo.cc.u32 q0, a1, w1, s;\n\t"
      "madc.hi.u32 q1, a1, w1, c;\n\t"
      "mul.wide.u32 rr, a0, m0;\n\t"
      "mov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.cc.u32 r0, q0, n0, r0;\n\t"
      "madc.hi.u32 r1, q0, n0, r1;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\t"
      "mad.lo.u32 r1, a1, m0, r1;\n\t"
      "mad.lo.u32 r1, q0, n1, r1;\n\t"
      "mad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t"
      "}"
      : "=l"(r)
      : "l"(a), "l"(m), "l"(w), "l"(np));
  return r;
}

// Reference (plain C) form of mul_shoup4, used by the probe to cross-check the PTX.
__device__ __forceinline__ u64 mul_shoup4_c(u64 a, u64 m, u64 w, u64 np) {
  const u32 a0 = lo32(a), a1 = hi32(a), w0 = lo32(w), w1 = hi32(w);
  const unsigned __int128 cross = (unsigned __int128)mul_wide(a1, w0) + mul_wide(a0, w1);
  u64 q = mul_wide(a1, w1) + (u64)(cross >> 32);   // floor((a*w - a0*w0) / 2^64)
  return a * m + q * np;
}

// ---------------------------------------------------------------- hybrid FP64-quotient product
// "mul_hyb": the IMAD pipe (fmaheavy) is the bottleneck of the Shoup step while the FP64 pipe
// is idle, so the quotient is estimated in FP64 (the paper's FP-FMA idea, PAPER.md:679-699,
// applied to the quotient only).  With a = a1*2^32 + a0 and the per-term constants
//     ms = m * 2^32 mod p,  mp = RN(m/p),  msp = RN(ms/p)    (m fixed per term)
// X = a1*ms + a0*m == a*m (mod p) has X/p < 2^33, and e = a1*msp + a0*mp is within
// delta <= 9*2^-21 of X/p (a1, a0 < 2^32 exact in FP64; |msp - ms/p|, |mp - m/p| <= 3u;
// DMUL/DFMA rounding <= 2^-21 + 2^-20).  With q = round(e) - 1:
//     X/p - q in [0.5 - delta, 1.5 + delta]   =>   r = X - q*p in (0, 2p)   for any a < 2^64.
// round(e) is read from the bits of t = e + 1.5*2^52 (exact, |e| < 2^51); with
// T = bits(t) and K = bits(1.5*2^52) + 1, q = T - K, so
//     r = a1*ms + a0*m + T*np + C  (mod 2^64),   np = 2^64 - p,  C = K*p mod 2^64.
// Integer pipe: 3 IMAD.WIDE + 4 IMAD; FP64 pipe: 2 exact u32->f64 (magic DADD), DMUL, DFMA,
// DADD.  Valid for every odd p < 2^63 (r < 2p < 2^64).
__device__ __forceinline__ u64 mul_hyb(u64 a, u64 m, u64 ms, double mp, double msp, u64 np, u64 C) {
  u64 r;
  asm("{\n\t"
      ".reg .u32 a0, a1, m0, m1, s0, s1, n0, n1, t0, t1, r0, r1, hb;\n\t"
      ".reg .f64 d0, d1, e, t;\n\t"
      ".reg .u64 rr;\n\t"
      "mov.u32 hb, 0x43300000;\n\t"
      "mov.b64 {a0, a1}, %1;\n\t"
      "mov.b64 {m0, m1}, %2;\n\t"
      "mov.b64 {s0, s1}, %3;\n\t"
      "mov.b64 {n0, n1}, %6;\n\t"
      // exact u32 -> f64: bits {x, 0x43300000} = 2^52 + x
      "mov.b64 d1, {a1, hb};\n\t"
      "mov.b64 d0, {a0, hb};\n\t"
      "sub.rn.f64 d1, d1, 0d4330000000000000;\n\t"
      "sub.rn.f64 d0, d0, 0d4330000000000000;\n\t"
      "mul.rn.f64 e, d1, %5;\n\t"
      "fma.rn.f64 e, d0, %4, e;\n\t"
      "add.rn.f64 t, e, 0d4338000000000000;\n\t"
      "mov.b64 {t0, t1}, t;\n\t"
      "mad.wide.u32 rr, a1, s0, %7;\n\t"
      "mad.wide.u32 rr, a0, m0, rr;\n\t"
      "mad.wide.u32 rr, t0, n0, rr;\n\t"
      "mov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.u32 r1, a1, s1, r1;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\t"
      "mad.lo.u32 r1, t0, n1, r1;\n\t"
      "mad.lo.u32 r1, t1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t"
      "}"
      : "=l"(r)
      : "l"(a), "l"(m), "l"(ms), "d"(mp), "d"(msp), "l"(np), "l"(C));
  return r;
}
// Host/device constant C for mul_hyb.
__host__ __device__ __forceinline__ u64 hyb_C(u64 p) { return 0x4338000000000001ull * p; }

// 32-bit Shoup ("a few less bits"): p < 2^31,
// w32 = floor(m 2^32 / p), any a < 2^32 -> r == a*m (mod p), r in [0, 2p) (2p < 2^32).
// One IMAD.HI + two IMADs = 4 IMAD slots instead of 14.
__device__ __forceinline__ u32 mul_shoup32(u32 a, u32 m, u32 w32, u32 p) {
  const u32 q = __umulhi(a, w32);
  return a * m - q * p;
}

// Lazy-2: p < 2^63, exact Shoup quotient, any a < 2^64 -> r in [0, 2p).
__device__ __forceinline__ u64 mul_shoup2(u64 a, u64 m, u64 w, u64 np) {
  u64 q = __umul64hi(a, w);
  return a * m + q * np;
}

// Conditional subtract: x in [0, 2p) -> [0, p).
__device__ __forceinline__ u64 csub(u64 x, u64 p) { return x >= p ? x - p : x; }

// ---------------------------------------------------------------- Montgomery
// REDC(hi:lo) = (hi*2^64 + lo) * 2^-64 mod p, valid when hi:lo < p * 2^64; output in [0, p).
__device__ __forceinline__ u64 redc(u64 hi, u64 lo, const ModParams& mp) {
  u64 u = lo * mp.pinv;
  u64 uh = __umul64hi(u, mp.p);
  // lo + lo(u*p) == 0 mod 2^64, carry-out == (lo != 0)
  u64 t = hi + uh + (lo != 0 ? 1ull : 0ull);
  // t < 2p < 2^64 since p < 2^63
  return csub(t, mp.p);
}
// a*b*2^-64 mod p, a*b < p*2^64 (e.g. a < p, b < 2^64 or a,b < p).
__device__ __forceinline__ u64 mont_mul(u64 a, u64 b, const ModParams& mp) {
  u64 hi, lo;
  mul128(a, b, hi, lo);
  return redc(hi, lo, mp);
}
__device__ __forceinline__ u64 to_mont(u64 a, const ModParams& mp) { return mont_mul(a, mp.r2, mp); }
__device__ __forceinline__ u64 from_mont(u64 a, const ModParams& mp) { return redc(0, a, mp); }
// Plain a*b mod p for a, b < p.
__device__ __forceinline__ u64 mulmod(u64 a, u64 b, const ModParams& mp) {
  return mont_mul(mont_mul(a, b, mp), mp.r2, mp);
}

// x^e in Montgomery form: xm = mont(x); returns mont(x^e).  Left-to-right square-and-multiply
// ("exponentiations by squaring").
__device__ __forceinline__ u64 mont_pow(u64 xm, u64 e, const ModParams& mp) {
  u64 r = mp.r1;  // mont(1)
  if (e == 0) return r;
  int top = 63 - __clzll(e);
  r = xm;
  for (int b = top - 1; b >= 0; --b) {
    r = mont_mul(r, r, mp);
    if ((e >> b) & 1) r = mont_mul(r, xm, mp);
  }
  return r;
}

// c * m^e mod p for c < 2^64 (any), m < p.  Returns canonical [0, p).
__device__ __forceinline__ u64 seed_pow(u64 c, u64 m, u64 e, const ModParams& mp) {
  u64 xm = mont_pow(to_mont(m, mp), e, mp);   // m^e * R
  // xm * c * R^-1 = c * m^e; needs xm * c < p * 2^64: xm < p, c < 2^64 ok.
  return mont_mul(xm, c, mp);
}

// (hi * 2^64 + lo) mod p for any hi, lo.
__device__ __forceinline__ u64 reduce128(u64 hi, u64 lo, const ModParams& mp) {
  u64 h = hi < mp.p ? hi : hi % mp.p;
  return mont_mul(redc(h, lo, mp), mp.r2, mp);
}

// floor(m * 2^64 / p) for m < p: restoring long division, 64 quotient bits.
__device__ __forceinline__ u64 shoup_w(u64 m, u64 p) {
  u64 r = m, q = 0;
  #pragma unroll 1
  for (int i = 0; i < 64; ++i) {
    // r < p < 2^63 so (r << 1) does not overflow
    r <<= 1;
    q <<= 1;
    if (r >= p) { r -= p; q |= 1; }
  }
  return q;
}

// floor(m * 2^64 / p) for m < p without the bit loop: with rem = m 2^64 mod p (= to_mont(m)),
// m 2^64 = w p + rem, so w p == -rem (mod 2^64) and w = rem * (-p^{-1}) mod 2^64 = rem * mp.pinv --
// exact because 0 <= w < 2^64.  One Montgomery product and one 64-bit multiply.
__device__ __forceinline__ u64 shoup_w_fast(u64 m, const ModParams& mp) {
  return to_mont(m, mp) * mp.pinv;
}

// ---------------------------------------------------------------- FP64 Alg. 2 / Alg. 3
// Alg. 2, p < 2^50, x,y in [0,p) as exact doubles; returns [0,p).
__device__ __forceinline__ double mul_fp(double x, double y, double p, double u) {
  double h = __dmul_rn(x, y);            // line 1: h <- x*y
  double l = __fma_rn(x, y, -h);         // line 2: l <- fma(x, y, -h)   (h + l == x*y exactly)
  double b = __dmul_rn(h, u);            // line 3: b <- h*u
  double c = floor(b);                   // line 4: c <- floor(b)  (quotient +-1)
  double d = __fma_rn(-c, p, h);         // line 5: d <- fma(-c, p, h)
  double g = __dadd_rn(d, l);            // line 6: g <- d + l      (remainder +-p)
  // lines 7-9 as selects (no divergent branches): g >= p -> g - p; g < 0 -> g + p; else g
  const double gm = __dsub_rn(g, p), gp = __dadd_rn(g, p);
  g = (g >= p) ? gm : g;                 // line 7
  g = (g < 0.0) ? gp : g;                // line 8 (exclusive with line 7 for g in (-p, 2p))
  return g;                              // line 9
}
// Alg. 3
__device__ __forceinline__ double add_fp(double x, double y, double p) {
  double s = __dadd_rn(x, y);
  return s >= p ? __dsub_rn(s, p) : s;
}

}  // namespace pe
