// Development probe: the 2-CTA (cta_group::2) int8 MMA that a CTA-pair k_tc would use.
// Cluster of 2 CTAs; CTA r holds A rows 128r..128r+127 (128 x 32 u8) and B rows 32r..32r+31
// (N = 64 total, 32 x 32 u8), both no-swizzle K-major; the leader issues
// tcgen05.mma.cta_group::2.kind::i8 (M = 256, N = 64, K = 32) and a multicast commit; each CTA
// reads its 128 TMEM lanes back.  Checks D = A B^T exactly against the host, then times `iters`
// MMAs issued back to back (clk per MMA on the leader).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2004_11571_b200/csrc \
//        scripts/mma2_probe.cu -o scripts/mma2_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace pe;
using namespace pe::tc;

__device__ __forceinline__ u32 cluster_rank() {
  u32 r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr u32 kA = 2048, kB = 512;   // LBO of A (128 rows) and B (32 rows) planes

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
k_mma2(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B, u32* __restrict__ D, int iters,
       long long* cyc) {
  __shared__ __align__(1024) uint8_t sa[4096];
  __shared__ __align__(1024) uint8_t sb[1024];
  __shared__ __align__(8) uint64_t bar;
  __shared__ u32 tmem_base;
  const u32 rank = cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // A rows 128r + row, K byte k  -> sa[(k/16)*kA + (row/8)*128 + (row%8)*16 + k%16]
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int row = i / 32, k = i % 32;
    sa[(k / 16) * kA + (row / 8) * 128 + (row % 8) * 16 + k % 16] = A[(128 * rank + row) * 32 + k];
  }
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
    const int row = i / 32, k = i % 32;
    sb[(k / 16) * kB + (row / 8) * 128 + (row % 8) * 16 + k % 16] = B[(32 * rank + row) * 32 + k];
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const u32 tb = tmem_base;
  const u32 idesc = (2u << 4) | ((u32)(64 >> 3) << 17) | ((u32)(256 >> 4) << 24);
  long long t0 = clock64();
  if (rank == 0 && warp == 0) {
    const uint64_t ad = smem_desc(smem_u32(sa), kA), bd = smem_desc(smem_u32(sb), kB);
    __syncwarp();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
        const u32 acc = it == 0 ? 0u : 1u;
        const u32 dt = tb + (u32)((it & 7) * 64);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(it < 8 ? tb + (u32)(it * 64) : dt), "l"(ad), "l"(bd), "r"(idesc), "r"(it < 8 ? 0u : acc));
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   :: "r"(smem_u32(&bar)), "h"((unsigned short)3) : "memory");
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  long long t1 = clock64();
  tc_fence_after();
  // accumulator 0 (columns 0..63): each iteration it = 8k writes accumulator 0 (k = 0 overwrites)
  const u32 row = (u32)(warp * 32 + lane);
  for (int c = 0; c < 64; c += 8) {
    u32 v[8];
    tmem_ld8(tb + ((u32)(warp * 32) << 16) + (u32)c, v);
    tmem_wait_ld();
    tmem_reg_fence(v);
    for (int j = 0; j < 8; ++j) D[(128 * rank + row) * 64 + c + j] = v[j];
  }
  if (threadIdx.x == 0 && rank == 0) *cyc = t1 - t0;
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tb));
  }
}

int main() {
  std::vector<uint8_t> A(256 * 32), B(64 * 32);
  srand(7);
  for (auto& x : A) x = (uint8_t)(rand() & 255);
  for (auto& x : B) x = (uint8_t)(rand() & 255);
  uint8_t *dA, *dB;
  u32* dD;
  long long* dc;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 256 * 64 * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  for (int iters : {1, 8, 9, 4096}) {
    cudaMemset(dD, 0, 256 * 64 * 4);
    k_mma2<<<2, 128>>>(dA, dB, dD, iters, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<u32> D(256 * 64);
    long long c = 0;
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    // accumulator 0 receives iterations 0, 8, 16, ... : count k = ceil(iters / 8)
    const u32 times = (u32)((iters + 7) / 8);
    long bad = 0;
    for (int i = 0; i < 256; ++i)
      for (int j = 0; j < 64; ++j) {
        u32 ref = 0;
        for (int k = 0; k < 32; ++k) ref += (u32)A[i * 32 + k] * B[j * 32 + k];
        ref *= times;
        if (D[i * 64 + j] != ref) {
          if (bad < 4) printf("  mismatch D[%d][%d] = %u, want %u\n", i, j, D[i * 64 + j], ref);
          ++bad;
        }
      }
    printf("iters %5d: %s, mismatches %ld, clk/MMA %.1f\n", iters, cudaGetErrorString(e), bad, (double)c / iters);
  }
  return 0;
}
