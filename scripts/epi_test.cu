// Unit check of the k_tc epilogue math without tensor cores: random D (u32 < 2^31) for the 4
// rounds' diagonals, folded per round through tc.cuh's fold_add (scratch in global memory, like
// epi_round), reduced once as in k_tc, vs the per-round W_d = 2^{8d} mod p path.
#include <cstdio>
#include <cstdlib>
#include "../paper_2004_11571_b200/csrc/tc.cuh"
using namespace pe;
using namespace pe::tc;
typedef unsigned __int128 u128;
static u64 hpow(u64 b, u64 e, u64 p) { u64 r = 1 % p; b %= p; while (e) { if (e & 1) r = (u128)r * b % p; b = (u128)b * b % p; e >>= 1; } return r; }

template <int G>
__device__ void fold_round(u32 (&x)[5], const u32* D) {
  if (group_diag(G, 0) >= 0) fold_add<8 * (group_diag(G, 0) < 0 ? 0 : group_diag(G, 0))>(x, D[0]);
  if (group_diag(G, 1) >= 0) fold_add<8 * (group_diag(G, 1) < 0 ? 0 : group_diag(G, 1))>(x, D[1]);
  if (group_diag(G, 2) >= 0) fold_add<8 * (group_diag(G, 2) < 0 ? 0 : group_diag(G, 2))>(x, D[2]);
  if (group_diag(G, 3) >= 0) fold_add<8 * (group_diag(G, 3) < 0 ? 0 : group_diag(G, 3))>(x, D[3]);
}
__global__ void k(const u32* D, u64* out, int n, ModParams mp, u64 C64, u64 C96, u64 C128) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u32 x[5] = {0, 0, 0, 0, 0};
  fold_round<0>(x, D + i * 16 + 0);
  fold_round<1>(x, D + i * 16 + 4);
  fold_round<2>(x, D + i * 16 + 8);
  fold_round<3>(x, D + i * 16 + 12);
  u64 lo = ((u64)x[1] << 32) | x[0], hi = 0;
  const u64 terms[3][2] = {{x[2], C64}, {x[3], C96}, {x[4], C128}};
  for (int q = 0; q < 3; ++q) {
    const u64 p0 = terms[q][0] * lo32(terms[q][1]);
    const u64 p1 = terms[q][0] * hi32(terms[q][1]);
    const u64 add_lo = p0 + (p1 << 32);
    const u64 add_hi = (p1 >> 32) + (add_lo < p0 ? 1ull : 0ull);
    lo += add_lo;
    hi += add_hi + (lo < add_lo ? 1ull : 0ull);
  }
  out[i] = reduce128(hi, lo, mp);
  if (i == 0) printf("dev x: %u %u %u %u %u  hi=%llu lo=%llu\n", x[0], x[1], x[2], x[3], x[4], (unsigned long long)hi, (unsigned long long)lo);
}
int main(int argc, char** argv) {
  const u64 p = argc > 1 ? strtoull(argv[1], 0, 10) : 4611686018427387847ull;
  ModParams mp;
  mp.p = p; mp.np = 0 - p;
  u64 inv = p; for (int i = 0; i < 6; ++i) inv *= 2 - p * inv;
  mp.pinv = 0 - inv; mp.r1 = (u64)(((u128)1 << 64) % p); mp.r2 = (u128)mp.r1 * mp.r1 % p;
  const int n = 4096;
  u32* D; u64* O;
  cudaMallocManaged(&D, n * 16 * 4);
  cudaMallocManaged(&O, n * 8);
  srand(2);
  for (int i = 0; i < n * 16; ++i) D[i] = ((u32)rand() << 16 ^ (u32)rand()) & 0x7fffffffu;
  k<<<n / 128, 128>>>(D, O, n, mp, hpow(2, 64, p), hpow(2, 96, p), hpow(2, 128, p));
  cudaDeviceSynchronize();
  const int groups[4][4] = {{7, 6, 0, -1}, {8, 5, 1, 14}, {9, 4, 2, 13}, {10, 3, 11, 12}};
  int bad = 0;
  for (int i = 0; i < n; ++i) {
    u64 r = 0;
    for (int g = 0; g < 4; ++g)
      for (int di = 0; di < 4; ++di)
        if (groups[g][di] >= 0) r = (u64)(((u128)r + (u128)D[i * 16 + 4 * g + di] * hpow(2, 8 * groups[g][di], p)) % p);
    bad += r != O[i];
    if (i == 0) {
      u128 X[2] = {0, 0};  // 256-bit as two u128
      for (int g = 0; g < 4; ++g) for (int di = 0; di < 4; ++di) if (groups[g][di] >= 0) {
        int s8 = 8 * groups[g][di]; u128 v = D[4 * g + di];
        if (s8 < 128) { u128 add = v << s8; u128 old = X[0]; X[0] += add; X[1] += (X[0] < old) + (s8 ? (v >> (128 - s8)) : 0); }
      }
      printf("host x: %u %u %u %u %u\n", (u32)X[0], (u32)(X[0] >> 32), (u32)(X[0] >> 64), (u32)(X[0] >> 96), (u32)X[1]);
    }
    if (i < 2) printf("%llu %llu\n", (unsigned long long)O[i], (unsigned long long)r);
  }
  printf("p=%llu epilogue bad: %d of %d\n", (unsigned long long)p, bad, n);
  return 0;
}
