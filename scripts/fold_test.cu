// Unit check of tc.cuh fold_add<8d>: X += D << 8d over random D, all 15 d, vs host 128-bit math.
#include <cstdio>
#include <cstdlib>
#include "../paper_2004_11571_b200/csrc/tc.cuh"
using namespace pe;
using namespace pe::tc;
template <int D8> __device__ void f(u32 (&x)[5], u32 v) { fold_add<D8>(x, v); }
__global__ void k(const u32* D, u32* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u32 x[5] = {0, 0, 0, 0, 0};
  const u32* d = D + i * 15;
  f<0>(x, d[0]); f<8>(x, d[1]); f<16>(x, d[2]); f<24>(x, d[3]); f<32>(x, d[4]); f<40>(x, d[5]);
  f<48>(x, d[6]); f<56>(x, d[7]); f<64>(x, d[8]); f<72>(x, d[9]); f<80>(x, d[10]); f<88>(x, d[11]);
  f<96>(x, d[12]); f<104>(x, d[13]); f<112>(x, d[14]);
  for (int w = 0; w < 5; ++w) out[i * 5 + w] = x[w];
}
int main() {
  const int n = 1000;
  u32 *D, *O;
  cudaMallocManaged(&D, n * 15 * 4);
  cudaMallocManaged(&O, n * 5 * 4);
  srand(1);
  for (int i = 0; i < n * 15; ++i) D[i] = ((u32)rand() << 16 ^ (u32)rand()) & 0x7fffffffu;
  k<<<(n + 127) / 128, 128>>>(D, O, n);
  cudaDeviceSynchronize();
  int bad = 0;
  for (int i = 0; i < n; ++i) {
    // host: 160-bit as 5 words via 64-bit accumulation per word with carries
    unsigned long long acc[6] = {0};
    for (int d = 0; d < 15; ++d) {
      unsigned __int128 v = (unsigned __int128)D[i * 15 + d] << (8 * d % 64);
      int w64 = 8 * d / 64;
      // add v (up to 95 bits) at 64-bit word w64
      unsigned __int128 lo = (unsigned __int128)acc[w64] + (unsigned long long)v;
      acc[w64] = (unsigned long long)lo;
      unsigned __int128 hi = (unsigned __int128)acc[w64 + 1] + (unsigned long long)(v >> 64) + (unsigned long long)(lo >> 64);
      acc[w64 + 1] = (unsigned long long)hi;
      acc[w64 + 2] += (unsigned long long)(hi >> 64);
    }
    u32 ref[5] = {(u32)acc[0], (u32)(acc[0] >> 32), (u32)acc[1], (u32)(acc[1] >> 32), (u32)acc[2]};
    for (int w = 0; w < 5; ++w) bad += ref[w] != O[i * 5 + w];
    if (i < 2) printf("%u %u %u %u %u | %u %u %u %u %u\n", O[i*5], O[i*5+1], O[i*5+2], O[i*5+3], O[i*5+4], ref[0], ref[1], ref[2], ref[3], ref[4]);
  }
  printf("fold bad words: %d\n", bad);
  return 0;
}
