// pipe_bench.cu -- standalone SASS-level throughput probes for B200 (sm_100a).
// Measures warp-instructions per clock per SM for single instruction types and 1:1 mixes,
// with independent chains (no data dependence between chains, 8 chains x 16 warps / SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define IT 2048

template <int V>
__global__ void kb(uint64_t* sink, long long* cyc, uint32_t seed) {
  uint32_t x[CH], y[CH];
  uint64_t w[CH];
  double d[CH], e[CH];
  float f[CH];
  const uint32_t t = threadIdx.x + seed;
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    x[i] = t * (i + 3) + 1; y[i] = t ^ (i * 77); w[i] = (uint64_t)t << i; d[i] = t + i; e[i] = 1.0 + i * 1e-9; f[i] = (float)i;
  }
  const uint32_t k = seed | 1;
  const double c = 1.0000001;
  const uint64_t cw = ((uint64_t)seed << 33) | 12345;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      // every chain depends on itself through a multiplicand (no loop-invariant products)
      if (V == 0 || V == 8 || V == 10 || V == 14) {
        asm volatile("{.reg .u32 lo, hi, z; mov.b64 {lo, hi}, %0; xor.b32 z, lo, hi; mad.wide.u32 %0, z, %1, %2;}"
                     : "+l"(w[i]) : "r"(k), "l"(cw));
      }
      if (V == 1 || V == 12) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(y[i]) : "r"(k), "r"(x[i]));
      if (V == 2 || V == 7 || V == 9 || V == 10 || V == 13)
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[i]) : "r"(k), "r"(x[i]));
      if (V == 3 || V == 7 || V == 8 || V == 12) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(c), "d"(e[i]));
      if (V == 4) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(c));
      if (V == 5) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(e[i]));
      if (V == 6 || V == 9) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
      if (V == 11) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(e[i]), "d"(e[(i + 1) % CH]));
      if (V == 13) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f[i]) : "f"(1.0001f));
      if (V == 14) {
        asm volatile("add.u32 %0, %0, %1;" : "+r"(y[i]) : "r"(k));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(k));
      }
    }
  }
  long long t1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i] + y[i] + w[i] + (uint64_t)d[i] + (uint64_t)f[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int ops_per_chain_iter, int warps) {
  int nsm = 148, threads = 32 * warps;
  uint64_t* sink; long long* cyc;
  cudaMalloc(&sink, (size_t)nsm * threads * 8);
  cudaMalloc(&cyc, nsm * 8);
  kb<V><<<nsm, threads>>>(sink, cyc, 1);
  kb<V><<<nsm, threads>>>(sink, cyc, 3);
  long long hc[148];
  cudaMemcpy(hc, cyc, nsm * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < nsm; ++i) mx += hc[i];
  mx /= nsm;
  double warp_instr = (double)warps * CH * IT * ops_per_chain_iter;
  printf("{\"probe\": \"%s\", \"warps_per_sm\": %d, \"warp_instr_per_clk_sm\": %.3f, \"lanes_per_clk_sm\": %.1f}\n",
         name, warps, warp_instr / mx, 32 * warp_instr / mx);
  cudaFree(sink); cudaFree(cyc);
}

int main() {
  for (int warps : {8, 16, 32}) {
    run<0>("IMAD.WIDE.U32(+64b addend)", 1, warps);
    run<1>("IMAD.HI.U32", 1, warps);
    run<2>("IMAD(lo)", 1, warps);
    run<3>("DFMA", 1, warps);
    run<4>("DMUL", 1, warps);
    run<5>("DADD", 1, warps);
    run<6>("IADD3", 1, warps);
    run<7>("IMAD+DFMA", 2, warps);
    run<8>("IMAD.WIDE+DFMA", 2, warps);
    run<9>("IMAD+IADD3", 2, warps);
    run<10>("IMAD.WIDE+IMAD", 2, warps);
    run<11>("DFMA(3 reg pairs)", 1, warps);
    run<12>("IMAD.HI+DFMA", 2, warps);
    run<13>("FFMA+IMAD", 2, warps);
    run<14>("IMAD.WIDE+2xIADD3", 3, warps);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
