// fast.h -- internal interface of the asymptotically fast evaluation (fast.cu; SURVEY.md §8(f)
// NEXT-4) used by pe.cu.  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "modcore.cuh"

namespace pe {
namespace fast {

constexpr int kNP = 5;              // NTT primes q_j < 2^30, 2^20 | q_j - 1
constexpr int kLgMax = 13;          // largest shared-memory transform: 2^13 points
constexpr unsigned kSmax = 1u << kLgMax;
constexpr unsigned kBkMax = kSmax / 2;   // operand block (block convolution above this length)
constexpr unsigned kTile = kSmax;        // points per CTA in the transform kernels
constexpr unsigned long long kTMax = 1ull << 20;   // CRT bound: prod q_j (2^149.7) > 2 T2 p^2 (< 2^147)

struct Plan;
// Tree shape from the padded bucket offsets (multiples of 32), any p < 2^63: PE_OK / PE_ENOMEM /
// PE_ECUDA.
int create(const std::vector<u64>& poff, const ModParams& mp, cudaStream_t s, Plan** out);
// out[g*ld + k] = sum_{i in g} c_i m_i^{j0+k}, k < T (padded-layout c, m on the device).
int eval(Plan* P, const u64* d_c, const u64* d_m, const ModParams& mp, u64 j0, u64 T, u64* d_out, u64 ld,
         cudaStream_t s);
void destroy(Plan* P, cudaStream_t s);

}  // namespace fast
}  // namespace pe
