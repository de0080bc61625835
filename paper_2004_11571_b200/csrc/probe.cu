// probe.cu -- modular-core probes (pin P12) and register-resident roofline microbenchmarks
// (SURVEY.md §8(d) "K5"): include/pe_test.h.
#include <cuda_runtime.h>

#include <cstdlib>

#include "../../include/pe.h"
#include "../../include/pe_test.h"
#include "kernels.cuh"
#include "tc.cuh"

using namespace pe;

typedef unsigned __int128 u128;

static ModParams probe_params(u64 p) {
  ModParams mp;
  mp.p = p;
  mp.np = (u64)0 - p;
  u64 inv = p;
  for (int i = 0; i < 6; ++i) inv *= 2 - p * inv;
  mp.pinv = (u64)0 - inv;
  mp.r1 = (u64)(((u128)1 << 64) % p);
  mp.r2 = (u64)(((u128)mp.r1 * mp.r1) % p);
  mp.pd = (double)p;
  mp.u = 1.0 / (double)p;
  mp.hc = hyb_C(p);
  return mp;
}

__global__ void k_probe(int variant, u64 N, const u64* a, const u64* b, const u64* x, u64* out, ModParams mp) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < N; i += (u64)gridDim.x * blockDim.x) {
    const u64 ai = a[i], bi = b[i];
    u64 r = 0;
    switch (variant) {
      case PE_CORE_SHOUP4: {
        u64 v = mul_shoup4(ai, bi, shoup_w(bi, mp.p), mp.np);
        r = v % mp.p;
        break;
      }
      case PE_CORE_SHOUP4RAW: {
        const u64 w = shoup_w(bi, mp.p);
        r = mul_shoup4(ai, bi, w, mp.np);
        if (r != mul_shoup4_c(ai, bi, w, mp.np)) r = 0xfffffffffffffffeull;  // PTX != C form
        break;
      }
      case PE_CORE_SHOUP2: r = csub(mul_shoup2(ai, bi, shoup_w(bi, mp.p), mp.np), mp.p); break;
      case PE_CORE_SHOUPW: r = shoup_w_fast(bi, mp) ^ shoup_w(bi, mp.p); break;   // 0 iff the two agree
      case PE_CORE_MONT: r = mulmod(ai, bi, mp); break;
      case PE_CORE_FP64: {
        double g = mul_fp((double)ai, (double)bi, mp.pd, mp.u);
        r = __double_as_longlong(g) < 0 ? 0xffffffffffffffffull : __double2ull_rn(g);  // flag -0.0
        break;
      }
      case PE_CORE_FP64ADD: {
        double g = add_fp((double)ai, (double)bi, mp.pd);
        r = __double_as_longlong(g) < 0 ? 0xffffffffffffffffull : __double2ull_rn(g);
        break;
      }
      case PE_CORE_POW: r = seed_pow(ai, bi, x[i], mp); break;
      case PE_CORE_HYB:
      case PE_CORE_HYBRAW: {
        const u64 ms = mulmod(bi, (u64)(((unsigned __int128)1 << 32) % mp.p), mp);
        const double mpd = __ddiv_rn(__ull2double_rn(bi), __ull2double_rn(mp.p));
        const double mspd = __ddiv_rn(__ull2double_rn(ms), __ull2double_rn(mp.p));
        r = mul_hyb(ai, bi, ms, mpd, mspd, mp.np, mp.hc);
        if (variant == PE_CORE_HYB) r %= mp.p;
        break;
      }
    }
    out[i] = r;
  }
}

extern "C" int pe_test_core(int variant, uint64_t p, uint64_t N, const uint64_t* a, const uint64_t* b,
                            const uint64_t* extra, uint64_t* out) {
  if (p < 3 || p >= (1ull << 63) || (p & 1) == 0) return PE_ERANGE;
  if ((variant == PE_CORE_SHOUP4 || variant == PE_CORE_SHOUP4RAW) && p >= (1ull << 62)) return PE_ENOTSUP;
  if ((variant == PE_CORE_FP64 || variant == PE_CORE_FP64ADD) && p >= (1ull << 50)) return PE_ENOTSUP;
  if (variant < 0 || variant > 9 || (N && (!a || !b || !out)) || (variant == PE_CORE_POW && N && !extra))
    return PE_EINVAL;
  if (N == 0) return PE_OK;
  u64 *da, *db, *dx = nullptr, *dout;
  if (cudaMalloc(&da, N * 8) || cudaMalloc(&db, N * 8) || cudaMalloc(&dout, N * 8)) return PE_ECUDA;
  if (variant == PE_CORE_POW && cudaMalloc(&dx, N * 8)) return PE_ECUDA;
  int rc = PE_OK;
  if (cudaMemcpy(da, a, N * 8, cudaMemcpyHostToDevice) || cudaMemcpy(db, b, N * 8, cudaMemcpyHostToDevice) ||
      (dx && cudaMemcpy(dx, extra, N * 8, cudaMemcpyHostToDevice)))
    rc = PE_ECUDA;
  if (rc == PE_OK) {
    unsigned blocks = (unsigned)((N + 255) / 256 < 148 * 32 ? (N + 255) / 256 : 148 * 32);
    k_probe<<<blocks, 256>>>(variant, N, da, db, dx, dout, probe_params(p));
    if (cudaGetLastError() != cudaSuccess || cudaMemcpy(out, dout, N * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = PE_ECUDA;
  }
  cudaFree(da); cudaFree(db); cudaFree(dout); cudaFree(dx);
  return rc;
}

// ---------------------------------------------------------------- K5 microbenchmarks
// The hot loop body without memory or reduction: acc += a_r; a_r <- a_r * m_r, R chains.
template <int V, int R>
__global__ void k_bench(int iters, u64* sink, long long* cyc, ModParams mp) {
  const u64 tid = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  long long t0 = clock64();
  if (V == PE_CORE_FP64) {
    double a[R], m[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      a[r] = (double)((tid * 7919 + r * 104729 + 1) % mp.p);
      m[r] = (double)((tid * 31337 + r * 7 + 3) % mp.p);
    }
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc = __dadd_rn(acc, a[r]);
        a[r] = mul_fp(a[r], m[r], mp.pd, mp.u);
      }
      if (acc >= 4503599627370496.0) acc = __dsub_rn(acc, 4503599627370496.0);
    }
    u64 x = __double2ull_rn(acc);
#pragma unroll
    for (int r = 0; r < R; ++r) x ^= __double2ull_rn(a[r]);
    sink[tid] = x;
  } else if (V == PE_CORE_HYB || V == 20) {
    u64 a[R], m[R], ms[R];
    double mpd[R], mspd[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      a[r] = (tid * 7919 + r * 104729 + 1) % mp.p;
      m[r] = (tid * 31337 + r * 7 + 3) % mp.p;
      ms[r] = mulmod(m[r], (u64)(((unsigned __int128)1 << 32) % mp.p), mp);
      mpd[r] = __ddiv_rn(__ull2double_rn(m[r]), __ull2double_rn(mp.p));
      mspd[r] = __ddiv_rn(__ull2double_rn(ms[r]), __ull2double_rn(mp.p));
    }
    U96 acc{0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (V < 20) add96_64(acc, a[r]);
        a[r] = mul_hyb(a[r], m[r], ms[r], mpd[r], mspd[r], mp.np, mp.hc);
      }
    }
    u64 x = acc.w0 ^ ((u64)acc.w1 << 32) ^ acc.w2;
#pragma unroll
    for (int r = 0; r < R; ++r) x ^= a[r];
    sink[tid] = x;
  } else if (V == PE_CORE_SHOUP4 || V == PE_CORE_SHOUP2 || V == 21) {
    u64 a[R], m[R], w[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      a[r] = (tid * 7919 + r * 104729 + 1) % mp.p;
      m[r] = (tid * 31337 + r * 7 + 3) % mp.p;
      w[r] = shoup_w(m[r], mp.p);
    }
    // same accumulation structure as k_step: 8 points per group, per point one 96-bit sum of
    // the R chains (set96_sum + add96_64), `iters` counts points
    U96 acc{0, 0, 0};
    for (int it = 0; it < iters; it += 8) {
      U96 pa[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (V < 20) {
          if (R == 1) { pa[k].w0 = lo32(a[0]); pa[k].w1 = hi32(a[0]); pa[k].w2 = 0; }
          else set96_sum(pa[k], a[0], a[1]);
#pragma unroll
          for (int r = 2; r < R; ++r) add96_64(pa[k], a[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
          a[r] = (V == PE_CORE_SHOUP4 || V == 21) ? mul_shoup4(a[r], m[r], w[r], mp.np) : mul_shoup2(a[r], m[r], w[r], mp.np);
      }
      if (V < 20) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { acc.w0 ^= pa[k].w0; acc.w1 += pa[k].w1; acc.w2 ^= pa[k].w2; }
      }
    }
    u64 x = acc.w0 ^ ((u64)acc.w1 << 32) ^ acc.w2;
#pragma unroll
    for (int r = 0; r < R; ++r) x ^= a[r];
    sink[tid] = x;
  } else {
    // bare instruction chains: R independent chains, one instruction per chain per iteration
    u32 x[R], y = (u32)tid | 1;
    u64 xw[R];
    double xd[R];
#pragma unroll
    for (int r = 0; r < R; ++r) { x[r] = (u32)tid + r; xw[r] = tid + r; xd[r] = (double)(tid + r); }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (V == 10) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(xw[r]) : "r"((u32)xw[r]), "r"(y));
        if (V == 11) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[r]) : "r"(y), "r"(y));
        if (V == 12) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(xd[r]) : "d"(1.0000001));
        if (V == 13) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[r]) : "r"(y), "r"(y));
        if (V == 14) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[r]) : "r"(y));
      }
    }
    u64 s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += x[r] + xw[r] + (u64)xd[r];
    sink[tid] = s;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
static void launch_bench_v(int R, int blocks, int threads, int iters, u64* sink, long long* cyc, ModParams mp) {
  switch (R) {
    case 1: k_bench<V, 1><<<blocks, threads>>>(iters, sink, cyc, mp); break;
    case 2: k_bench<V, 2><<<blocks, threads>>>(iters, sink, cyc, mp); break;
    case 4: k_bench<V, 4><<<blocks, threads>>>(iters, sink, cyc, mp); break;
    case 8: k_bench<V, 8><<<blocks, threads>>>(iters, sink, cyc, mp); break;
    case 16: k_bench<V, 16><<<blocks, threads>>>(iters, sink, cyc, mp); break;
  }
}

extern "C" int pe_bench_core(int variant, uint64_t p, int R, int blocks, int threads, int iters, float* ms,
                             double* steps, double* cycles) {
  if (R != 1 && R != 2 && R != 4 && R != 8 && R != 16) return PE_EINVAL;
  if (blocks < 1 || threads < 32 || threads > 1024 || iters < 1) return PE_EINVAL;
  if (p < 3 || p >= (1ull << 63)) return PE_ERANGE;
  ModParams mp = probe_params(p);
  u64* sink;
  long long* cyc;
  if (cudaMalloc(&sink, (size_t)blocks * threads * 8) || cudaMalloc(&cyc, blocks * sizeof(long long)))
    return PE_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int rc = PE_OK;
  for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
    cudaEventRecord(e0);
    switch (variant) {
      case PE_CORE_SHOUP4: launch_bench_v<PE_CORE_SHOUP4>(R, blocks, threads, iters, sink, cyc, mp); break;
      case PE_CORE_SHOUP2: launch_bench_v<PE_CORE_SHOUP2>(R, blocks, threads, iters, sink, cyc, mp); break;
      case PE_CORE_FP64: launch_bench_v<PE_CORE_FP64>(R, blocks, threads, iters, sink, cyc, mp); break;
      case PE_CORE_HYB: launch_bench_v<PE_CORE_HYB>(R, blocks, threads, iters, sink, cyc, mp); break;
      case 20: launch_bench_v<20>(R, blocks, threads, iters, sink, cyc, mp); break;
      case 21: launch_bench_v<21>(R, blocks, threads, iters, sink, cyc, mp); break;
      case 10: launch_bench_v<10>(R, blocks, threads, iters, sink, cyc, mp); break;
      case 11: launch_bench_v<11>(R, blocks, threads, iters, sink, cyc, mp); break;
      case 12: launch_bench_v<12>(R, blocks, threads, iters, sink, cyc, mp); break;
      case 13: launch_bench_v<13>(R, blocks, threads, iters, sink, cyc, mp); break;
      case 14: launch_bench_v<14>(R, blocks, threads, iters, sink, cyc, mp); break;
      default: rc = PE_EINVAL;
    }
    cudaEventRecord(e1);
  }
  if (rc == PE_OK && (cudaGetLastError() != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess)) rc = PE_ECUDA;
  if (rc == PE_OK) {
    cudaEventElapsedTime(ms, e0, e1);
    *steps = (double)blocks * threads * R * (double)iters;
    long long* hc = (long long*)malloc(blocks * sizeof(long long));
    cudaMemcpy(hc, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int b = 0; b < blocks; ++b) s += (double)hc[b];
    *cycles = s / blocks;
    free(hc);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaFree(cyc);
  return rc;
}

// ---------------------------------------------------------------- int8 tcgen05 issue-rate probe
// One CTA per SM issues `iters` M=128 x N x K=32 kind::i8 MMAs (u8 x u8 -> s32) from a fixed
// shared-memory tile into 4 rotating TMEM accumulators: the same-run tensor ceiling that
// bench.py quotes beside k_tc (the tc.cuh MMA shape is N = tc::kV = 64).
__global__ void k_bench_mma(int iters, u32 idesc, u32 ncols, int nacc) {
  extern __shared__ uint8_t dsm[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dsm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ u32 tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * (int)tc::kPlaneA; i += blockDim.x) sm[i] = (uint8_t)(i * 13);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(tc::smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const u32 tb = tmem_base;
  if (threadIdx.x == 0) {
    const uint64_t ad = tc::smem_desc(tc::smem_u32(sm), tc::kLBOA),
                   bd = tc::smem_desc(tc::smem_u32(sm) + tc::kPlaneA, tc::kLBOA);
    u32 acc_col = 0;
    const u32 acc_end = (u32)nacc * ncols;
    for (int it = 0; it < iters; ++it, acc_col = (acc_col + ncols == acc_end) ? 0u : acc_col + ncols)
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "setp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
          :: "r"(tb + acc_col), "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
    tc::mma_commit(&bar);
  }
  __shared__ u32 abort_flag;
  abort_flag = 0;
  tc::mbar_wait(&bar, 0, tc::Abort{&abort_flag, nullptr});
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
  }
}

extern "C" int pe_bench_mma(int N, int iters, float* ms, double* macs) {
  if ((N != 16 && N != 32 && N != 64 && N != 128) || iters < 1 || !ms || !macs) return PE_EINVAL;
  const int nacc = (512 / N) < 16 ? 512 / N : 16;   // rotating independent accumulators
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return PE_ECUDA;
  const u32 idesc = (2u << 4) | ((u32)(N >> 3) << 17) | ((u32)(128 >> 4) << 24);
  const int smem = 2 * tc::kPlaneA + 1024;
  if (cudaFuncSetAttribute(k_bench_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return PE_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
    cudaEventRecord(e0);
    k_bench_mma<<<nsm, 128, smem>>>(iters, idesc, (u32)N, nacc);
    cudaEventRecord(e1);
  }
  int rc = PE_OK;
  if (cudaGetLastError() != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess) rc = PE_ECUDA;
  if (rc == PE_OK) {
    cudaEventElapsedTime(ms, e0, e1);
    *macs = (double)nsm * iters * 128.0 * N * 32.0;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return rc;
}
