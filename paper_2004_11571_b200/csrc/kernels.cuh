// kernels.cuh -- device kernels of the partial-evaluation path (sm_100a).
//
//   k_keys        a2: bucket key (dx<<32 | dy) per term
//   k_max_exp     max evaluated exponent (power-table size d)
//   k_power_table a3: beta_k^e tables, Montgomery form
//   k_setup       a3: m_i, Shoup w_i in the padded tile layout (k_setup_c: reduced c_i)
//   k_step        a4+a5+a6: seed a_i = c_i m_i^{j_s}, then per point acc += a_i, a_i <- a_i m_i
//                 with the per-(x,y) segmented reduction
//   k_fixup       a6: cross-CTA carries of one bucket -> canonical out
#pragma once
#include "modcore.cuh"

namespace pe {

constexpr int kMaxWarps = 16;
constexpr int kSuper = 32;   // points per shared-memory super-group (one lane per point)

// Scalar cores of k_step (the hybrid FP64-quotient and the mixed FP64/IMAD variants measured in
// round 1 were not faster and live only in the test library, csrc/probe.cu).
enum PathKind { kInt4 = 0, kInt2 = 1, kFp64 = 2, kInt32 = 5 };
// Max threads per CTA of k_step<PATH, R> (register budget: 65536 / threads per thread).
__host__ __device__ constexpr int step_max_threads(int path, int R) {
  return R >= 16 ? 256 : 512;
}

// ---------------------------------------------------------------- 96-bit accumulators
struct U96 { u32 w0, w1, w2; };

__device__ __forceinline__ void add96_64(U96& x, u64 v) {
  asm("add.cc.u32 %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32 %2, %2, 0;"
      : "+r"(x.w0), "+r"(x.w1), "+r"(x.w2)
      : "r"(lo32(v)), "r"(hi32(v)));
}
// x = u + v (65 bits) without zero-initialising x.
__device__ __forceinline__ void set96_sum(U96& x, u64 u, u64 v) {
  asm("add.cc.u32 %0, %3, %5;\n\t"
      "addc.cc.u32 %1, %4, %6;\n\t"
      "addc.u32 %2, 0, 0;"
      : "=r"(x.w0), "=r"(x.w1), "=r"(x.w2)
      : "r"(lo32(u)), "r"(hi32(u)), "r"(lo32(v)), "r"(hi32(v)));
}
__device__ __forceinline__ void add96(U96& x, const U96& y) {
  asm("add.cc.u32 %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32 %2, %2, %5;"
      : "+r"(x.w0), "+r"(x.w1), "+r"(x.w2)
      : "r"(y.w0), "r"(y.w1), "r"(y.w2));
}

template <int NW>
__device__ __forceinline__ U96 shfl_xor96(const U96& x, int off) {
  U96 r;
  r.w0 = __shfl_xor_sync(0xffffffffu, x.w0, off);
  r.w1 = __shfl_xor_sync(0xffffffffu, x.w1, off);
  r.w2 = NW == 3 ? __shfl_xor_sync(0xffffffffu, x.w2, off) : 0u;
  return r;
}
__device__ __forceinline__ U96 sel96(bool c, const U96& a, const U96& b) {
  U96 r;
  r.w0 = c ? a.w0 : b.w0;
  r.w1 = c ? a.w1 : b.w1;
  r.w2 = c ? a.w2 : b.w2;
  return r;
}
template <int NW>
__device__ __forceinline__ void add96n(U96& x, const U96& y) {
  if (NW == 3) {
    add96(x, y);
  } else {
    asm("add.cc.u32 %0, %0, %2;\n\t"
        "addc.u32 %1, %1, %3;"
        : "+r"(x.w0), "+r"(x.w1)
        : "r"(y.w0), "r"(y.w1));
  }
}

// Transpose-reduce 8 points over the 32 lanes of a warp (the GPU analogue of the paper's
// SIMD tree reduction with shuffles): lanes exchange halves of their
// 8 per-point partial sums at xor-distance 16, 8, 4 (each lane keeps the half matching its
// lane bit), then butterfly at 2, 1.  Afterwards lane l holds the warp total of point
// (l >> 2) & 7.  9 exchanges per lane for 8 points instead of 40 for 8 plain butterflies.
// NW = 32-bit words carried (2 when every partial sum fits 64 bits, else 3).
template <int NW>
__device__ __forceinline__ U96 xpose_reduce8(U96 (&v)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  U96 t4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    U96 send = sel96(b4, v[i], v[i + 4]);
    t4[i] = sel96(b4, v[i + 4], v[i]);
    add96n<NW>(t4[i], shfl_xor96<NW>(send, 16));
  }
  U96 t2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    U96 send = sel96(b3, t4[i], t4[i + 2]);
    t2[i] = sel96(b3, t4[i + 2], t4[i]);
    add96n<NW>(t2[i], shfl_xor96<NW>(send, 8));
  }
  U96 send = sel96(b2, t2[0], t2[1]);
  U96 t1 = sel96(b2, t2[1], t2[0]);
  add96n<NW>(t1, shfl_xor96<NW>(send, 4));
  add96n<NW>(t1, shfl_xor96<NW>(t1, 2));
  add96n<NW>(t1, shfl_xor96<NW>(t1, 1));
  return t1;
}

// ---------------------------------------------------------------- setup kernels
// Terms [a, b) (one upload chunk): bucket key and input index.  E: exponent type of the input
// (u32, or u8 for pe_create_compact).
template <class E>
static __global__ void k_keys(const E* __restrict__ exps, u64 a, u64 b, u32 n, u64* __restrict__ key,
                       u32* __restrict__ idx, u32* __restrict__ kmax) {
  u32 mx = 0, my = 0;
  for (u64 i = a + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < b; i += (u64)gridDim.x * blockDim.x) {
    const u32 dx = exps[i * n + 0], dy = exps[i * n + 1];
    key[i] = ((u64)dx << 32) | dy;
    idx[i] = (u32)i;
    mx = max(mx, dx);
    my = max(my, dy);
  }
  for (int o = 16; o; o >>= 1) {   // the largest degrees in x and y (the sort's key width)
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    my = max(my, __shfl_xor_sync(0xffffffffu, my, o));
  }
  __shared__ u32 bx, by;            // one atomic per block, not per warp (they all hit one address)
  if (threadIdx.x == 0) { bx = 0; by = 0; }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) { atomicMax(&bx, mx); atomicMax(&by, my); }
  __syncthreads();
  if (threadIdx.x == 0) { atomicMax(kmax, bx); atomicMax(kmax + 1, by); }
}
// Keys (dx << 32 | dy) -> (dx << bd | dy) with dy < 2^bd: the same order in bx + bd bits, so the
// radix sort runs ceil((bx + bd) / 8) passes instead of 8 (config 5: 2).
static __global__ void k_pack_keys(u64* __restrict__ key, u64 t, u32 bd) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < t; i += (u64)gridDim.x * blockDim.x) {
    const u64 k = key[i];
    key[i] = ((k >> 32) << bd) | (k & 0xffffffffull);
  }
}

// Batched polynomials: polynomial id of every (key-sorted) term, from
// the term offsets poly_off[npoly+1]; iota[j] = j for the stable re-sort by polynomial.
static __global__ void k_poly_of(const u32* __restrict__ idx_sorted, u64 t, const u64* __restrict__ poly_off,
                                 u32 npoly, u32* __restrict__ pid, u32* __restrict__ iota) {
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < t; j += (u64)gridDim.x * blockDim.x) {
    const u64 i = idx_sorted[j];
    u32 lo = 0, hi = npoly;
    while (hi - lo > 1) {
      u32 mid = (lo + hi) >> 1;
      if (poly_off[mid] <= i) lo = mid; else hi = mid;
    }
    pid[j] = lo;
    iota[j] = (u32)j;
  }
}
static __global__ void k_apply_perm(const u32* __restrict__ perm, u64 t, const u64* __restrict__ key_in,
                                    const u32* __restrict__ idx_in, u64* __restrict__ key_out,
                                    u32* __restrict__ idx_out) {
  for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < t; k += (u64)gridDim.x * blockDim.x) {
    const u32 j = perm[k];
    key_out[k] = key_in[j];
    idx_out[k] = idx_in[j];
  }
}
// Run starts of equal (polynomial, dx, dy) in the sorted order (pid may be NULL: one polynomial).
static __global__ void k_run_flags(const u64* __restrict__ key, const u32* __restrict__ pid, u64 t,
                                   unsigned char* __restrict__ flags) {
  for (u64 k = blockIdx.x * (u64)blockDim.x + threadIdx.x; k < t; k += (u64)gridDim.x * blockDim.x)
    flags[k] = (k == 0 || key[k] != key[k - 1] || (pid && pid[k] != pid[k - 1])) ? 1 : 0;
}
static __global__ void k_gather_runs(const u32* __restrict__ starts, u32 G, const u64* __restrict__ key,
                                     const u32* __restrict__ pid, u64* __restrict__ ukey, u32* __restrict__ upid) {
  for (u32 g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
    ukey[g] = key[starts[g]];
    upid[g] = pid ? pid[starts[g]] : 0;
  }
}

// table[l*(D+1) + e] = mont(alpha_l^e), one thread per entry (independent exponentiations); D + 1 =
// kTab entries per variable (exponents beyond take direct powers in k_monomials).
constexpr u32 kTab = 256;
static __global__ void k_power_table(const u64* __restrict__ alpha, u32 nz, u32 D, u64* __restrict__ table,
                              ModParams mp) {
  u64 total = (u64)nz * (D + 1);
  for (u64 q = blockIdx.x * (u64)blockDim.x + threadIdx.x; q < total; q += (u64)gridDim.x * blockDim.x) {
    u32 l = (u32)(q / (D + 1)), e = (u32)(q % (D + 1));
    table[q] = mont_pow(to_mont(alpha[l], mp), e, mp);
  }
}

// m_i = prod_l alpha_l^{e_il} mod p for the input terms [a, b) of one upload chunk (input order), with
// n-3 Montgomery products from the power tables ("n-3 multiplications for each m_i
// thanks to the tables of powers"); an exponent beyond the table takes a direct power.  Runs while
// later chunks are still crossing PCIe.
template <class E>
static __global__ void k_monomials(const E* __restrict__ exps, u64 a, u64 b, u32 n,
                                   const u64* __restrict__ table, const u64* __restrict__ alpha,
                                   u64* __restrict__ m_in, ModParams mp) {
  for (u64 i = a + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < b; i += (u64)gridDim.x * blockDim.x) {
    const E* e = exps + i * n;
    u64 acc = mp.r1;   // Montgomery 1
    for (u32 l = 0; l + 2 < n; ++l) {
      const u32 x = e[2 + l];
      const u64 f = x < kTab ? table[(u64)l * kTab + x] : mont_pow(to_mont(alpha[l], mp), x, mp);
      acc = l == 0 ? f : mont_mul(acc, f, mp);
    }
    m_in[i] = from_mont(acc, mp);
  }
}

// One thread per padded slot q.  Bucket g of the padded layout owns [poff[g], poff[g+1]); its first
// cnt[g] slots are the sorted terms bstart[g] .. bstart[g]+cnt[g]-1, the rest are padding (c = 0,
// m = 1: contributes 0 at every point).  Coefficients reduced mod p (reading R5), m_i from
// k_monomials, Shoup constant w_i = floor(m_i 2^64 / p).
static __global__ void k_setup(const u64* __restrict__ m_in,
                        const u32* __restrict__ sorted_idx, const u64* __restrict__ poff,
                        const u64* __restrict__ bstart, u32 G, u64 t_pad,
                        u64* __restrict__ m_out, u64* __restrict__ w_out,
                        u32* __restrict__ perm_out, ModParams mp) {
  for (u64 q = blockIdx.x * (u64)blockDim.x + threadIdx.x; q < t_pad; q += (u64)gridDim.x * blockDim.x) {
    u32 lo = 0, hi = G;   // bucket g: poff[g] <= q < poff[g+1]
    while (hi - lo > 1) {
      u32 mid = (lo + hi) >> 1;
      if (poff[mid] <= q) lo = mid; else hi = mid;
    }
    const u32 g = lo;
    const u64 r = q - poff[g];
    const u64 cnt = bstart[g + 1] - bstart[g];
    u64 m = 1 % mp.p;
    u32 src = 0xffffffffu;
    if (r < cnt) {
      src = sorted_idx[bstart[g] + r];
      m = m_in[src];
    }
    m_out[q] = m;
    w_out[q] = shoup_w_fast(m, mp);
    perm_out[q] = src;
  }
}

// The coefficients in the same layout, reduced mod p (padding: c = 0).  Separate from k_setup so
// that pe_create uploads them last, while the sort and the tensor-path setup (which need only the
// exponents) run.
static __global__ void k_setup_c(const u64* __restrict__ coeffs, const u32* __restrict__ perm, u64 t_pad,
                                 u64* __restrict__ c_out, u64 p) {
  for (u64 q = blockIdx.x * (u64)blockDim.x + threadIdx.x; q < t_pad; q += (u64)gridDim.x * blockDim.x) {
    const u32 src = perm[q];
    c_out[q] = src != 0xffffffffu ? coeffs[src] % p : 0;
  }
}

static __global__ void k_scatter_m(const u64* __restrict__ m_pad, const u32* __restrict__ perm, u64 t_pad,
                            u64* __restrict__ m_orig) {
  for (u64 q = blockIdx.x * (u64)blockDim.x + threadIdx.x; q < t_pad; q += (u64)gridDim.x * blockDim.x) {
    u32 s = perm[q];
    if (s != 0xffffffffu) m_orig[s] = m_pad[q];
  }
}

// ---------------------------------------------------------------- the hot kernel
struct StepArgs {
  const u64* c;          // [t_pad] reduced coefficients (tile layout)
  const u64* m;          // [t_pad] m_i
  const u64* w;          // [t_pad] floor(m_i 2^64 / p)           (Shoup paths)
  const uint2* wt_info;  // [n_wt] x = partial slot, y = run length if run leader else 0
  u64* partial;          // [n_slots][ldp]
  u64 ldp;               // leading dimension of partial (points of this pass)
  u64 js0;               // j of column 0 of this pass
  u32 n_wt;              // warp tiles
  u32 npts;              // points of this pass
  u32 chunk;             // points per CTA (multiple of kSuper)
  ModParams mp;
};

// One warp owns a tile of 32*R terms of ONE (x,y) bucket (buckets are padded to whole
// tiles); lane l holds terms tile + r*32 + l (r < R) in registers for the CTA's whole point
// chunk: a_i is read from HBM once per chunk, the GPU form of the paper's T_d dependent
// evaluations, and the R independent chains per lane are its T_i / M
// ILP without the T_i copies of a (the no-extra-memory variant,
// PAPER.md:1979-2046).
//
// Per 8 points each lane accumulates acc[k] += a_r (Alg. 7 order: reduce, then multiply,
// PAPER.md:1642-1643), then a warp transpose-reduce leaves one 96-bit total per point; per
// 32 points the totals of the warps of one bucket inside the CTA are summed in shared
// memory, reduced mod p and written as one partial per (CTA run, point).
template <int PATH, int R>
__global__ void __launch_bounds__(step_max_threads(PATH, R))
k_step(StepArgs args) {
  __shared__ U96 sacc[2][kMaxWarps][kSuper];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int W = blockDim.x >> 5;
  const u32 wt = blockIdx.x * W + warp;
  const bool active = wt < args.n_wt;
  const u32 k_begin = blockIdx.y * args.chunk;
  const u32 cnt = min(args.chunk, args.npts - k_begin);
  const u64 js = args.js0 + k_begin;
  const ModParams mp = args.mp;

  // ---- load the lane's R terms and seed a_r = c_r * m_r^{js} (each
  //      independent chain seeded by exponentiation)
  u64 a[R], m[R], w[R];
  double ad[R], md[R];   // FP64 path: a, m
  u32 a32[R], m32[R], w32[R];   // kInt32 path
  uint2 info = make_uint2(0, 0);
  if (active) {
    info = args.wt_info[wt];
    const u64 base = (u64)wt * (32 * R) + lane;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const u64 q = base + (u64)r * 32;
      const u64 c = __ldg(args.c + q);
      m[r] = __ldg(args.m + q);
      a[r] = seed_pow(c, m[r], js, mp);
      if (PATH == kFp64) { ad[r] = (double)a[r]; md[r] = (double)m[r]; }
      if (PATH == kInt4 || PATH == kInt2) w[r] = __ldg(args.w + q);
      if (PATH == kInt32) { a32[r] = (u32)a[r]; m32[r] = (u32)m[r]; w32[r] = hi32(__ldg(args.w + q)); }
    }
  }

  int buf = 0;
  for (u32 k0 = 0; k0 < cnt; k0 += kSuper, buf ^= 1) {
    if (active) {
#pragma unroll 1
      for (int s = 0; s < kSuper / 8; ++s) {
        U96 acc[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (PATH == kFp64) {
            double sum = 0.0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
              sum = __dadd_rn(sum, ad[r]);                   // exact: R*p < 2^53
              ad[r] = mul_fp(ad[r], md[r], mp.pd, mp.u);     // Alg. 2
            }
            const u64 si = __double2ull_rn(sum);
            acc[k].w0 = lo32(si); acc[k].w1 = hi32(si); acc[k].w2 = 0;
          } else if (PATH == kInt32) {
            u64 s64 = a32[0];                                  // R values < 2^32: no overflow
#pragma unroll
            for (int r = 1; r < R; ++r) s64 += a32[r];
            acc[k].w0 = lo32(s64); acc[k].w1 = hi32(s64); acc[k].w2 = 0;
            const u32 p32 = (u32)mp.p;
#pragma unroll
            for (int r = 0; r < R; ++r) a32[r] = mul_shoup32(a32[r], m32[r], w32[r], p32);
          } else {
            if (R == 1) {
              acc[k].w0 = lo32(a[0]); acc[k].w1 = hi32(a[0]); acc[k].w2 = 0;
            } else {
              set96_sum(acc[k], a[0], a[1]);
            }
#pragma unroll
            for (int r = 2; r < R; ++r) add96_64(acc[k], a[r]);
#pragma unroll
            for (int r = 0; r < R; ++r)
              a[r] = PATH == kInt4 ? mul_shoup4(a[r], m[r], w[r], mp.np) : mul_shoup2(a[r], m[r], w[r], mp.np);
          }
        }
        const U96 tot = (PATH == kFp64 || PATH == kInt32) ? xpose_reduce8<2>(acc, lane)
                                                           : xpose_reduce8<3>(acc, lane);
        if ((lane & 3) == 0) sacc[buf][warp][s * 8 + (lane >> 2)] = tot;
      }
    }
    __syncthreads();
    // run leaders: lane = point within the super-group
    if (active && info.y) {
      U96 x = sacc[buf][warp][lane];
      for (u32 v = 1; v < info.y; ++v) add96(x, sacc[buf][warp + v][lane]);
      const u32 k = k0 + lane;
      if (k < cnt) {
        const u64 lo = ((u64)x.w1 << 32) | x.w0;
        args.partial[(u64)info.x * args.ldp + k_begin + k] = reduce128(x.w2, lo, mp);
      }
    }
    // double-buffered sacc: the next super-group writes the other buffer; the barrier of
    // the next iteration orders the reads above before buffer reuse two groups later.
  }
}

// out[g*ld + k] = sum over the bucket's partial slots, mod p.  One thread per (g, k).
// skip1: rows with a single slot were written to `out` by k_tc directly (TcArgs::direct)
static __global__ void k_fixup(const u64* __restrict__ partial, u64 ldp, const u32* __restrict__ slot_start,
                        u32 G, u32 npts, u32 nkb, u64* __restrict__ out, u64 ld, ModParams mp, int skip1) {
  const u32 g = blockIdx.x / nkb;
  const u32 k = (blockIdx.x % nkb) * blockDim.x + threadIdx.x;
  if (g >= G || k >= npts) return;
  if (skip1 && slot_start[g + 1] - slot_start[g] == 1) return;
  u64 lo = 0, hi = 0;
  for (u32 s = slot_start[g]; s < slot_start[g + 1]; ++s) {
    const u64 v = partial[(u64)s * ldp + k];
    lo += v;
    hi += (lo < v);
  }
  out[(u64)g * ld + k] = reduce128(hi, lo, mp);
}

// The same for rows with many slots (k_tc pieces of a large bucket; one term shard of config 5 is a
// single 300-slot row): a 256-thread block covers (g, 32 points), warp w sums slots w, w + 8, ... with
// coalesced 256-byte loads, and the 8 partial 128-bit sums meet in shared memory.
static __global__ void __launch_bounds__(256) k_fixup_wide(const u64* __restrict__ partial, u64 ldp,
                                                           const u32* __restrict__ slot_start, u32 G, u32 npts,
                                                           u32 nkb, u64* __restrict__ out, u64 ld, ModParams mp,
                                                           int skip1) {
  __shared__ u64 slo[8][32], shi[8][32];
  const u32 g = blockIdx.x / nkb;
  if (g < G && skip1 && slot_start[g + 1] - slot_start[g] == 1) return;   // whole block: uniform exit
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const u32 k = (blockIdx.x % nkb) * 32 + lane;
  u64 lo = 0, hi = 0;
  if (g < G && k < npts) {
    for (u32 s = slot_start[g] + warp; s < slot_start[g + 1]; s += 8) {
      const u64 v = partial[(u64)s * ldp + k];
      lo += v;
      hi += (lo < v);
    }
  }
  slo[warp][lane] = lo;
  shi[warp][lane] = hi;
  __syncthreads();
  if (warp == 0 && g < G && k < npts) {
    for (int w = 1; w < 8; ++w) {
      const u64 v = slo[w][lane];
      lo += v;
      hi += shi[w][lane] + (lo < v);
    }
    out[(u64)g * ld + k] = reduce128(hi, lo, mp);
  }
}

// Multi-GPU assembly (pe_rows_addmod): dst[r][k] = (dst[r][k] + src[r][k]) mod p for canonical
// residues (< p < 2^63, so the u64 sum cannot wrap) -- the root's sum of a bucket split between
// two term ranges, i.e. the coefficient reduction of PAPER.md:489-503 across ranks.
static __global__ void k_rows_addmod(u64* __restrict__ dst, u64 ldd, const u64* __restrict__ src, u64 lds, u64 rows,
                                     u64 cols, u64 p) {
  const u64 n = rows * cols;
  for (u64 x = blockIdx.x * (u64)blockDim.x + threadIdx.x; x < n; x += (u64)gridDim.x * blockDim.x) {
    const u64 r = x / cols, k = x - r * cols;
    const u64 s = dst[r * ldd + k] + src[r * lds + k];
    dst[r * ldd + k] = s >= p ? s - p : s;
  }
}

}  // namespace pe
