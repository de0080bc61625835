// dsmem_probe.cu -- bandwidth of TMA bulk copies shared::cta -> peer shared::cluster within a CTA pair
// (cluster of 2), both directions at once, 64 KB per copy, completion on the peer's mbarrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/dsmem_probe scripts/dsmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}

constexpr int kBytes = 16384, kSlots = 4;
__global__ void __cluster_dims__(2, 1, 1) k_copy(int iters, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* src = sm;
  uint8_t* dst0 = sm + kBytes;           // the peer writes into kSlots slots here
  __shared__ __align__(8) uint64_t fullb[kSlots], readyb[kSlots];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const uint32_t peer = rank ^ 1;
  for (int i = threadIdx.x; i < kBytes; i += blockDim.x) src[i] = (uint8_t)i;
  if (threadIdx.x == 0) {
    for (int k = 0; k < kSlots; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&fullb[k])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&readyb[k])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    // every slot starts free: arm all my slots and release them to the peer
    for (int k = 0; k < kSlots; ++k) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&fullb[k])), "r"(kBytes) : "memory");
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa(smem_u32(&readyb[k]), peer)) : "memory");
    }
    for (int it = 0; it < iters; ++it) {
      const int k = it % kSlots;
      const uint32_t ph = (it / kSlots) & 1;
      // peer slot k free -> copy into it
      while (!try_wait(smem_u32(&readyb[k]), ph)) {}
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(mapa(smem_u32(dst0 + k * kBytes), peer)), "r"(smem_u32(src)), "r"(kBytes),
                      "r"(mapa(smem_u32(&fullb[k]), peer)) : "memory");
      // my slot k filled by the peer -> consume, re-arm and release it
      while (!try_wait(smem_u32(&fullb[k]), ph)) {}
      if (it + kSlots < iters) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&fullb[k])), "r"(kBytes) : "memory");
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa(smem_u32(&readyb[k]), peer)) : "memory");
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 8000, grid = nsm / 2 * 2;
  long long* cyc;
  cudaMalloc(&cyc, grid * 8);
  cudaFuncSetAttribute(k_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, (1 + kSlots) * kBytes);
  k_copy<<<grid, 128, (1 + kSlots) * kBytes>>>(10, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_copy<<<grid, 128, (1 + kSlots) * kBytes>>>(iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  std::vector<long long> c(grid);
  cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
  long long mx = 0; for (auto x : c) mx = x > mx ? x : mx;
  printf("{\"probe\":\"dsmem_bulk_copy\",\"bytes_per_copy\":%d,\"iters\":%d,\"ms\":%.3f,\"bytes_per_clk_per_sm_each_way\":%.1f,"
         "\"GBps_per_sm_each_way\":%.1f}\n", kBytes, iters, ms, (double)kBytes * iters / mx,
         (double)kBytes * iters / (ms * 1e-3) / 1e9);
  return 0;
}
