// tc_probe.cu -- tcgen05.mma kind::i8 probe for sm_100a: (1) correctness of the hand-built
// shared-memory / instruction descriptors (no-swizzle K-major canonical layout) against a CPU
// int8 GEMM, for M = 128 and several N; (2) issue-rate microbenchmark (MMA from a fixed smem
// tile, no data movement) to measure the int8 tensor rate per SM for each N.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o scripts/tc_probe scripts/tc_probe.cu
//   scripts/tc_probe
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

// byte offset of element (r, k) of an R-row, K-major int8 operand tile in the no-swizzle canonical
// layout: core matrix = 8 rows x 16 bytes (128 B contiguous); core matrices ordered K-chunk-major:
// offset(core (g, c)) = (c * R/8 + g) * 128.  LBO (next 16 B K-chunk) = R/8*128, SBO (next 8 rows) = 128.
__host__ __device__ inline uint32_t kmaj_off(uint32_t r, uint32_t k, uint32_t R) {
  return ((k >> 4) * (R >> 3) + (r >> 3)) * 128u + (r & 7u) * 16u + (k & 15u);
}

__device__ inline uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_i8(uint32_t M, uint32_t N) {
  return (2u << 4)           // D format S32
       | (1u << 7)           // A signed int8
       | (1u << 10)          // B signed int8
       | ((N >> 3) << 17)    // N
       | ((M >> 4) << 24);   // M
}

__device__ inline void mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(dtmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ inline void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

__device__ inline void mbar_init(uint64_t* bar, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(cnt));
}

__device__ inline void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n"
      :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase) : "memory");
}

// one CTA, 128 threads: D[128 x N] = A[128 x K] * B[N x K]^T (both K-major int8)
template <int N>
__global__ void k_gemm_check(const int8_t* A, const int8_t* B, int K, int32_t* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB = sm + 128 * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int idx = tid; idx < 128 * K; idx += blockDim.x) {
    int r = idx / K, k = idx % K;
    sA[kmaj_off(r, k, 128)] = (uint8_t)A[idx];
  }
  for (int idx = tid; idx < N * K; idx += blockDim.x) {
    int r = idx / K, k = idx % K;
    sB[kmaj_off(r, k, N)] = (uint8_t)B[idx];
  }
  constexpr uint32_t ncols = N < 32 ? 32 : N;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  if (tid == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sA), b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int ks = 0; ks < K / 32; ++ks) {
      uint64_t ad = smem_desc(a0 + ks * 2 * (128 / 8) * 128, (128 / 8) * 128, 128);
      uint64_t bd = smem_desc(b0 + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
      mma_i8(tb, ad, bd, idesc_i8(128, N), ks > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tb + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "n"(ncols));
}

// throughput: each CTA issues `iters` x (K/32) MMAs of 128 x N x 32 on fixed smem tiles into
// `nacc` rotating accumulators; one commit at the end.
template <int N>
__global__ void k_gemm_rate(int iters, int K, int nacc, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB = sm + 128 * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int idx = tid; idx < (128 + N) * K; idx += blockDim.x) sm[idx] = (uint8_t)(idx * 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_base)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  long long t0 = clock64();
  if (tid == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sA), b0 = (uint32_t)__cvta_generic_to_shared(sB);
    for (int it = 0; it < iters; ++it) {
      for (int ks = 0; ks < K / 32; ++ks) {
        uint64_t ad = smem_desc(a0 + ks * 2 * (128 / 8) * 128, (128 / 8) * 128, 128);
        uint64_t bd = smem_desc(b0 + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        mma_i8(tb + (uint32_t)((it % nacc) * N), ad, bd, idesc_i8(128, N), 1);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tb), "n"(512));
}

template <int N>
static bool check(int K) {
  std::vector<int8_t> A(128 * K), B(N * K);
  std::vector<int32_t> D(128 * N), R(128 * N, 0);
  srand(N * 1000 + K);
  for (auto& x : A) x = (int8_t)(rand() & 0xff);
  for (auto& x : B) x = (int8_t)(rand() & 0xff);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      int32_t s = 0;
      for (int k = 0; k < K; ++k) s += (int32_t)A[m * K + k] * (int32_t)B[n * K + k];
      R[m * N + n] = s;
    }
  int8_t *dA, *dB;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0x55, D.size() * 4));
  size_t sm = (128 + N) * K;
  CK(cudaFuncSetAttribute(k_gemm_check<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_gemm_check<N><<<1, 128, sm>>>(dA, dB, K, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (size_t i = 0; i < D.size(); ++i) bad += D[i] != R[i];
  printf("{\"probe\":\"check\",\"M\":128,\"N\":%d,\"K\":%d,\"mismatches\":%d,\"D00\":%d,\"R00\":%d}\n", N, K, bad, D[0], R[0]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad == 0;
}

template <int N>
static void rate(int K, int ctas_per_sm) {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int iters = 4096, nacc = 512 / N > 8 ? 8 : 512 / N;
  size_t sm = (128 + N) * K;
  CK(cudaFuncSetAttribute(k_gemm_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  long long* cyc;
  CK(cudaMalloc(&cyc, 8 * nsm * ctas_per_sm));
  k_gemm_rate<N><<<nsm * ctas_per_sm, 128, sm>>>(16, K, nacc, cyc);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_gemm_rate<N><<<nsm * ctas_per_sm, 128, sm>>>(iters, K, nacc, cyc);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> c(nsm * ctas_per_sm);
  CK(cudaMemcpy(c.data(), cyc, 8 * c.size(), cudaMemcpyDeviceToHost));
  long long mx = 0;
  for (auto x : c) mx = x > mx ? x : mx;
  double macs = (double)nsm * ctas_per_sm * iters * (K / 32) * 128.0 * N * 32.0;
  double mac_per_clk_sm = (double)ctas_per_sm * iters * (K / 32) * 128.0 * N * 32.0 / (double)mx;
  printf("{\"probe\":\"rate\",\"M\":128,\"N\":%d,\"K\":%d,\"ctas_per_sm\":%d,\"ms\":%.3f,\"TOPS\":%.1f,"
         "\"mac_per_clk_sm\":%.0f,\"clk_per_mma\":%.2f}\n",
         N, K, ctas_per_sm, ms, 2.0 * macs / (ms * 1e-3) / 1e12, mac_per_clk_sm,
         (double)mx / (iters * (K / 32)) / ctas_per_sm);
  cudaFree(cyc);
}

int main() {
  bool ok = true;
  ok &= check<16>(64);
  ok &= check<32>(32);
  ok &= check<32>(128);
  ok &= check<64>(96);
  ok &= check<128>(64);
  ok &= check<256>(64);
  if (!ok) { printf("{\"probe\":\"check\",\"ok\":false}\n"); return 1; }
  rate<16>(128, 1);
  rate<32>(128, 1);
  rate<32>(128, 2);
  rate<64>(128, 1);
  rate<128>(128, 1);
  rate<256>(128, 1);
  return 0;
}
