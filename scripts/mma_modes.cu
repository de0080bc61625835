// Development probe: per-MMA cost of tcgen05.mma kind::i8 (M=128, K=32) for N = 64 / 128 under
// the issue patterns k_tc can use.  One CTA per SM, clock64 around the issue + completion.
//   mode 0: one thread, A and B re-read from smem by every MMA
//   mode 1: one thread, runs of 4 MMAs sharing A through the collector (fill/use/use/lastuse)
//   mode 2: two warps issue mode-1 runs concurrently on disjoint accumulators
//   mode 3: two warps issue mode-0 MMAs concurrently on disjoint accumulators
//   mode 4: k_tc's issue_round<0> + issue_round<1> (64 MMAs, N = 64) from one elected thread
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2004_11571_b200/csrc \
//        scripts/mma_modes.cu -o scripts/mma_modes
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace pe;
using namespace pe::tc;

__device__ __forceinline__ void mma_mode(u32 dt, uint64_t ad, uint64_t bd, u32 idesc, int col) {
  if (col == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" :: "r"(dt), "l"(ad), "l"(bd), "r"(idesc));
  else if (col == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n\t}\n" :: "r"(dt), "l"(ad), "l"(bd), "r"(idesc));
  else if (col == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n\t}\n" :: "r"(dt), "l"(ad), "l"(bd), "r"(idesc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}\n" :: "r"(dt), "l"(ad), "l"(bd), "r"(idesc));
}

__global__ void k_modes(int iters, int N, int mode, long long* cyc) {
  extern __shared__ uint8_t dsm[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dsm + 127) & ~(uintptr_t)127);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ u32 tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 16 * 4096; i += blockDim.x) sm[i] = (uint8_t)(i * 13);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const u32 tb = tmem_base;
  const u32 idesc = (2u << 4) | ((u32)(N >> 3) << 17) | ((u32)(128 >> 4) << 24);
  const int nacc = 512 / N;
  const bool two = mode == 2 || mode == 3;
  const int nw = two ? 2 : 1;
  long long t0 = clock64();
  if (warp < nw && (threadIdx.x & 31) == 0) {
    const int acc0 = two ? warp * (nacc / 2) : 0, nac = two ? nacc / 2 : nacc;
    const bool col = mode == 1 || mode == 2;
    const u32 base = smem_u32(sm);
    const uint64_t ad0 = smem_desc(base, 2048), bd0 = smem_desc(base + 32768, 2048);
    const u32 dt0 = tb + (u32)(acc0 * N);
    const u32 nN = (u32)N, nacm = (u32)nac - 1;   // nac is a power of 2
    for (int blk = 0; blk < iters / nw / 32; ++blk) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int plane = (j >> 2) & 7, k = j & 3;
        const uint64_t ad = ad0 + (uint64_t)(plane * 256);            // 4096 B >> 4
        const uint64_t bd = bd0 + (uint64_t)(((j + warp) & 7) * 256);
        const u32 dt = dt0 + ((u32)j & nacm) * nN;
        if (col) mma_mode(dt, ad, bd, idesc, k == 0 ? 1 : k == 3 ? 3 : 2);
        else mma_mode(dt, ad, bd, idesc, 0);
      }
    }
    mma_commit(&bar[warp]);
  }
  if (mode == 4 && threadIdx.x < 32) {   // k_tc's own issue sequence (rounds 0 and 1 alternately)
    const uint64_t da = smem_desc(uni(smem_u32(sm)), kLBOA);
    const uint64_t db = smem_desc(uni(smem_u32(sm)) + 8 * kPlaneA, kLBOB);
    const u32 tbu = uni(tb);
    __syncwarp();
    if (elect_one()) {
      for (int blk = 0; blk < iters / 64; ++blk) {
        issue_round<0>(tbu, da, db, false);
        issue_round<1>(tbu, da, db, false);
      }
      mma_commit(&bar[0]);
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) { mbar_wait(&bar[0], 0); if (two && mode < 4) mbar_wait(&bar[1], 0); }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, nsm * sizeof(long long));
  const int smem = 16 * 4096 + 256;
  cudaFuncSetAttribute(k_modes, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 8192;
  for (int N : {64, 128})
    for (int mode = 0; mode < 5; ++mode) {
      if (mode == 4 && N != 64) continue;
      for (int rep = 0; rep < 2; ++rep) k_modes<<<nsm, 128, smem>>>(iters, N, mode, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[256];
      cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
      double s = 0;
      for (int b = 0; b < nsm; ++b) s += (double)h[b];
      s /= nsm;
      printf("N=%3d mode=%d  clk/MMA %.1f  (%s)\n", N, mode, s / iters, cudaGetErrorString(e));
    }
  return 0;
}
