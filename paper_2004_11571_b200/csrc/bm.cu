// bm.cu -- Berlekamp-Massey per bucket on the GPU (the consumer right
// after the path).  For each output row g (a bucket's sequence S_g(k) = sum_i c_i m_i^{j0+k},
// PAPER.md:420-427) it finds the shortest connection polynomial
//     C_g(z) = 1 + c_1 z + ... + c_L z^L,   S_g(k) + sum_{i=1..L} c_i S_g(k-i) = 0  (L <= k < T),
// which for T >= 2 r_g is prod_i (1 - m_i z) over the bucket's r_g distinct monomial values with
// nonzero coefficient (Ben-Or/Tiwari; the transposed-Vandermonde view PAPER.md:279-285,
// 465-478, 765-773).  Division-free Massey iteration: C <- b*C - d*z^m*B keeps every update
// inversion-free; C is normalised by C_0^{-1} once at the end.  One CTA per sequence; C, B and a
// spare live in global scratch (they can exceed shared memory for T ~ 16k); the discrepancy is
// a block reduction of Montgomery products.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "../../include/pe.h"
#include "kernels.cuh"

using namespace pe;

namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u64 addm(u64 a, u64 b, u64 p) {
  u64 s = a + b;  // a, b < p < 2^63: no overflow
  return s >= p ? s - p : s;
}
__device__ __forceinline__ u64 subm(u64 a, u64 b, u64 p) { return a >= b ? a - b : a + p - b; }

__device__ u64 block_sum_mod(u64 v, u64 p, u64* red) {
  for (int o = 16; o; o >>= 1) v = addm(v, __shfl_xor_sync(0xffffffffu, v, o), p);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  u64 s = 0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < nw ? red[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) s = addm(s, __shfl_xor_sync(0xffffffffu, s, o), p);
  }
  return s;  // valid in thread 0
}

// All values of C, B are kept in Montgomery form; S is read in normal form (mont_mul(C~, S) = C*S).
__global__ void k_bm(const u64* __restrict__ seq, u64 ld, u32 T, u64* __restrict__ lam, u64 ldl,
                     u32* __restrict__ len_out, u64* __restrict__ scratch, ModParams mp) {
  __shared__ u64 red[32];
  __shared__ u64 sh_d;
  const u64 p = mp.p;
  const u64 g = blockIdx.x;
  const u64* S = seq + g * ld;
  u64* X = scratch + g * 3ull * (T + 1);  // C
  u64* Y = X + (T + 1);                   // B
  u64* Z = Y + (T + 1);                   // spare
  for (u32 i = threadIdx.x; i <= T; i += blockDim.x) {
    X[i] = i == 0 ? mp.r1 : 0;
    Y[i] = i == 0 ? mp.r1 : 0;
  }
  u32 L = 0, m = 1, degC = 0, degB = 0;
  u64 bm = mp.r1;  // b in Montgomery form
  __syncthreads();
  for (u32 n = 0; n < T; ++n) {
    // discrepancy d = sum_{i=0}^{L} C_i S_{n-i}  (normal form)
    u64 part = 0;
    const u32 top = min(L, degC);
    for (u32 i = threadIdx.x; i <= top; i += blockDim.x) part = addm(part, mont_mul(X[i], S[n - i], mp), p);
    const u64 d = block_sum_mod(part, p, red);
    if (threadIdx.x == 0) sh_d = d;
    __syncthreads();
    const u64 dn = sh_d;
    if (dn == 0) {
      ++m;
      continue;
    }
    const u64 dm = to_mont(dn, mp);
    // Z = b*C - d*z^m*B
    const u32 newdeg = max(degC, m + degB);
    for (u32 i = threadIdx.x; i <= newdeg && i <= T; i += blockDim.x) {
      const u64 c = i <= degC ? mont_mul(bm, X[i], mp) : 0;
      const u64 bb = (i >= m && i - m <= degB) ? mont_mul(dm, Y[i - m], mp) : 0;
      Z[i] = subm(c, bb, p);
    }
    __syncthreads();
    if (2 * L <= n) {
      // B <- old C, C <- Z, spare <- old B
      u64* oldY = Y;
      Y = X;
      X = Z;
      Z = oldY;
      degB = degC;
      L = n + 1 - L;
      bm = dm;
      m = 1;
    } else {
      u64* oldX = X;  // C <- Z, spare <- old C (B unchanged)
      X = Z;
      Z = oldX;
      ++m;
    }
    degC = min(newdeg, T);
    // zero the spare beyond its live range is unnecessary: reads are bounded by degC / degB
    __syncthreads();
  }
  // normalise: C_0^{-1} (C_0 = product of the b's, nonzero); write normal form
  __shared__ u64 inv_m;
  if (threadIdx.x == 0) {
    const u64 c0 = from_mont(X[0], mp);
    const u64 inv = from_mont(mont_pow(to_mont(c0, mp), p - 2, mp), mp);  // Fermat
    inv_m = to_mont(inv, mp);
    len_out[g] = L;
  }
  __syncthreads();
  for (u32 i = threadIdx.x; i <= T && i < ldl; i += blockDim.x)
    lam[g * ldl + i] = i <= L && i <= degC ? from_mont(mont_mul(X[i], inv_m, mp), mp) : 0;
}

ModParams bm_params(u64 p) {
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
  return mp;
}

}  // namespace

namespace pe {
int set_last_error(int e);   // pe.cu: thread-local code read by pe_last_error
}

extern "C" int pe_bm_device(uint64_t p, uint64_t G, uint64_t T, const uint64_t* d_seq, uint64_t ld,
                            uint64_t* d_lambda, uint64_t ldl, uint32_t* d_len, void* stream) {
  set_last_error(PE_OK);
  if (p < 3 || p >= (1ull << 63) || (p & 1) == 0) return set_last_error(PE_ERANGE);
  if (G == 0 || T == 0) return PE_OK;
  if (!d_seq || !d_lambda || !d_len || ld < T || ldl < T + 1 || T >= 0xffffffffull || G >= 0x7fffffffull)
    return set_last_error(PE_EINVAL);
  cudaStream_t s = (cudaStream_t)stream;
  u64* scratch = nullptr;
  if (cudaMallocAsync((void**)&scratch, G * 3 * (T + 1) * sizeof(u64), s) != cudaSuccess) {
    cudaGetLastError();
    return set_last_error(PE_ENOMEM);
  }
  k_bm<<<(unsigned)G, 256, 0, s>>>(d_seq, ld, (u32)T, d_lambda, ldl, d_len, scratch, bm_params(p));
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  return e == cudaSuccess ? PE_OK : set_last_error(PE_ECUDA);
}

extern "C" int pe_bm(uint64_t p, uint64_t G, uint64_t T, const uint64_t* seq, uint64_t* lambda, uint32_t* len) {
  set_last_error(PE_OK);
  if (G == 0 || T == 0) return PE_OK;
  if (!seq || !lambda || !len) return set_last_error(PE_EINVAL);
  u64 *ds = nullptr, *dl = nullptr;
  u32* dn = nullptr;
  int rc = PE_OK;
  if (cudaMalloc(&ds, G * T * 8) != cudaSuccess || cudaMalloc(&dl, G * (T + 1) * 8) != cudaSuccess ||
      cudaMalloc(&dn, G * 4) != cudaSuccess) {
    cudaGetLastError();
    rc = PE_ENOMEM;
  }
  if (rc == PE_OK && cudaMemcpy(ds, seq, G * T * 8, cudaMemcpyHostToDevice) != cudaSuccess) rc = PE_ECUDA;
  if (rc == PE_OK) rc = pe_bm_device(p, G, T, ds, T, dl, T + 1, dn, nullptr);
  if (rc == PE_OK && (cudaMemcpy(lambda, dl, G * (T + 1) * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
                      cudaMemcpy(len, dn, G * 4, cudaMemcpyDeviceToHost) != cudaSuccess))
    rc = PE_ECUDA;
  if (ds) cudaFree(ds);   // also on the failure paths: no partial allocation leaks
  if (dl) cudaFree(dl);
  if (dn) cudaFree(dn);
  return rc == PE_OK ? PE_OK : set_last_error(rc);
}
