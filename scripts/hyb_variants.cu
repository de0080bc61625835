// hyb_variants.cu -- scratch harness: register-resident throughput of hybrid FP64-quotient step
// variants (k_step-like: R chains x 8 points, 96-bit per-point sums) vs the Shoup baseline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hyb_variants hyb_variants.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
typedef uint64_t u64;
typedef uint32_t u32;

struct U96 { u32 w0, w1, w2; };
__device__ __forceinline__ void add96_64(U96& x, u64 v) {
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, 0;"
      : "+r"(x.w0), "+r"(x.w1), "+r"(x.w2) : "r"((u32)v), "r"((u32)(v >> 32)));
}
__device__ __forceinline__ void set96_sum(U96& x, u64 u, u64 v) {
  asm("add.cc.u32 %0, %3, %5;\n\taddc.cc.u32 %1, %4, %6;\n\taddc.u32 %2, 0, 0;"
      : "=r"(x.w0), "=r"(x.w1), "=r"(x.w2)
      : "r"((u32)u), "r"((u32)(u >> 32)), "r"((u32)v), "r"((u32)(v >> 32)));
}

// Shoup v5 (library)
__device__ __forceinline__ u64 mul_shoup(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, x1l, x1h, x2l, x2h, z, s, c, q0, q1, r0, r1;\n\t.reg .u64 rr, x1, x2;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {w0, w1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.wide.u32 x1, a1, w0;\n\tmul.wide.u32 x2, a0, w1;\n\tmov.b64 {x1l, x1h}, x1;\n\tmov.b64 {x2l, x2h}, x2;\n\t"
      "add.cc.u32 z, x1l, x2l;\n\taddc.cc.u32 s, x1h, x2h;\n\taddc.u32 c, 0, 0;\n\t"
      "mad.lo.cc.u32 q0, a1, w1, s;\n\tmadc.hi.u32 q1, a1, w1, c;\n\t"
      "mul.wide.u32 rr, a0, m0;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.cc.u32 r0, q0, n0, r0;\n\tmadc.hi.u32 r1, q0, n0, r1;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, a1, m0, r1;\n\tmad.lo.u32 r1, q0, n1, r1;\n\tmad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(w), "l"(np));
  return r;
}

// H0: library mul_hyb
__device__ __forceinline__ u64 hyb0(u64 a, u64 m, u64 ms, double mp, double msp, u64 np, u64 C) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, s0, s1, n0, n1, t0, t1, r0, r1, hb;\n\t.reg .f64 d0, d1, e, t;\n\t.reg .u64 rr;\n\t"
      "mov.u32 hb, 0x43300000;\n\tmov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {s0, s1}, %3;\n\tmov.b64 {n0, n1}, %6;\n\t"
      "mov.b64 d1, {a1, hb};\n\tmov.b64 d0, {a0, hb};\n\t"
      "sub.rn.f64 d1, d1, 0d4330000000000000;\n\tsub.rn.f64 d0, d0, 0d4330000000000000;\n\t"
      "mul.rn.f64 e, d1, %5;\n\tfma.rn.f64 e, d0, %4, e;\n\tadd.rn.f64 t, e, 0d4338000000000000;\n\tmov.b64 {t0, t1}, t;\n\t"
      "mad.wide.u32 rr, a1, s0, %7;\n\tmad.wide.u32 rr, a0, m0, rr;\n\tmad.wide.u32 rr, t0, n0, rr;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.u32 r1, a1, s1, r1;\n\tmad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, t0, n1, r1;\n\tmad.lo.u32 r1, t1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(ms), "d"(mp), "d"(msp), "l"(np), "l"(C));
  return r;
}
// H1: r's low word via mul.wide + madc chains (no 64-bit addend pairs), + C folded at the end
__device__ __forceinline__ u64 hyb1(u64 a, u64 m, u64 ms, double mp, double msp, u64 np, u64 C) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, s0, s1, n0, n1, t0, t1, r0, r1, hb, c0, c1;\n\t.reg .f64 d0, d1, e, t;\n\t.reg .u64 rr;\n\t"
      "mov.u32 hb, 0x43300000;\n\tmov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {s0, s1}, %3;\n\tmov.b64 {n0, n1}, %6;\n\t"
      "mov.b64 {c0, c1}, %7;\n\t"
      "mov.b64 d1, {a1, hb};\n\tmov.b64 d0, {a0, hb};\n\t"
      "sub.rn.f64 d1, d1, 0d4330000000000000;\n\tsub.rn.f64 d0, d0, 0d4330000000000000;\n\t"
      "mul.rn.f64 e, d1, %5;\n\tfma.rn.f64 e, d0, %4, e;\n\tadd.rn.f64 t, e, 0d4338000000000000;\n\tmov.b64 {t0, t1}, t;\n\t"
      "mul.wide.u32 rr, a1, s0;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.cc.u32 r0, a0, m0, r0;\n\tmadc.hi.u32 r1, a0, m0, r1;\n\t"
      "mad.lo.cc.u32 r0, t0, n0, r0;\n\tmadc.hi.u32 r1, t0, n0, r1;\n\t"
      "add.cc.u32 r0, r0, c0;\n\taddc.u32 r1, r1, c1;\n\t"
      "mad.lo.u32 r1, a1, s1, r1;\n\tmad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, t0, n1, r1;\n\tmad.lo.u32 r1, t1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(ms), "d"(mp), "d"(msp), "l"(np), "l"(C));
  return r;
}
// H2: like H1 but the constant C folded into the hi word only (C's low word is K*p mod 2^32...)
//     -> keep H1; H2 uses cvt.rn.f64.u32 for the conversions (I2F.F64 on whatever pipe)
__device__ __forceinline__ u64 hyb2(u64 a, u64 m, u64 ms, double mp, double msp, u64 np, u64 C) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, s0, s1, n0, n1, t0, t1, r0, r1, c0, c1;\n\t.reg .f64 d0, d1, e, t;\n\t.reg .u64 rr;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {s0, s1}, %3;\n\tmov.b64 {n0, n1}, %6;\n\t"
      "mov.b64 {c0, c1}, %7;\n\t"
      "cvt.rn.f64.u32 d1, a1;\n\tcvt.rn.f64.u32 d0, a0;\n\t"
      "mul.rn.f64 e, d1, %5;\n\tfma.rn.f64 e, d0, %4, e;\n\tadd.rn.f64 t, e, 0d4338000000000000;\n\tmov.b64 {t0, t1}, t;\n\t"
      "mul.wide.u32 rr, a1, s0;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.cc.u32 r0, a0, m0, r0;\n\tmadc.hi.u32 r1, a0, m0, r1;\n\t"
      "mad.lo.cc.u32 r0, t0, n0, r0;\n\tmadc.hi.u32 r1, t0, n0, r1;\n\t"
      "add.cc.u32 r0, r0, c0;\n\taddc.u32 r1, r1, c1;\n\t"
      "mad.lo.u32 r1, a1, s1, r1;\n\tmad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, t0, n1, r1;\n\tmad.lo.u32 r1, t1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(ms), "d"(mp), "d"(msp), "l"(np), "l"(C));
  return r;
}

template <int V, int R, int MINB>
__global__ void __launch_bounds__(256, MINB) kh(const u64* __restrict__ in, u64 np, u64 C, int groups, u64* out) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  u64 a[R], m[R], w[R];
  double mp[R], msp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    a[r] = in[(tid * R + r) % 4096];
    m[r] = in[(tid * R + r + 7) % 4096];
    w[r] = in[(tid * R + r + 13) % 4096];
    mp[r] = (double)m[r] * 2.1684043449710089e-19;
    msp[r] = (double)w[r] * 2.1684043449710089e-19;
  }
  U96 tot{0, 0, 0};
#pragma unroll 1
  for (int g = 0; g < groups; ++g) {
    U96 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (R == 1) { acc[k].w0 = (u32)a[0]; acc[k].w1 = (u32)(a[0] >> 32); acc[k].w2 = 0; }
      else set96_sum(acc[k], a[0], a[1]);
#pragma unroll
      for (int r = 2; r < R; ++r) add96_64(acc[k], a[r]);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (V == 9) a[r] = mul_shoup(a[r], m[r], w[r], np);
        if (V == 0) a[r] = hyb0(a[r], m[r], w[r], mp[r], msp[r], np, C);
        if (V == 1) a[r] = hyb1(a[r], m[r], w[r], mp[r], msp[r], np, C);
        if (V == 2) a[r] = hyb2(a[r], m[r], w[r], mp[r], msp[r], np, C);
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) { tot.w0 ^= acc[k].w0; tot.w1 += acc[k].w1; tot.w2 ^= acc[k].w2; }
  }
  out[tid] = tot.w0 ^ ((u64)tot.w1 << 32) ^ tot.w2 ^ a[0];
}

template <int V, int R, int MINB>
void run(const char* nm, u64* in, u64* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * MINB * 4, threads = 256, groups = 512;
  const u64 p = (1ull << 62) - 57, np = 0 - p, C = 0x4338000000000001ull * p;
  kh<V, R, MINB><<<blocks, threads>>>(in, np, C, groups, out);
  cudaEventRecord(e0);
  kh<V, R, MINB><<<blocks, threads>>>(in, np, C, groups, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kh<V, R, MINB>);
  double tp = (double)blocks * threads * R * 8 * groups;
  printf("{\"variant\": \"%s\", \"R\": %d, \"minb\": %d, \"regs\": %d, \"ms\": %.3f, \"per_clk_sm_at_1965\": %.3f}\n",
         nm, R, MINB, fa.numRegs, ms, tp / (ms * 1e-3) / (148 * 1965e6));
}

int main() {
  const int N = 4096;
  u64 h[N];
  const u64 p = (1ull << 62) - 57;
  for (int i = 0; i < N; ++i) h[i] = (0x9E3779B97F4A7C15ull * (i + 1)) % p;
  u64 *in, *out;
  cudaMalloc(&in, N * 8); cudaMalloc(&out, 148 * 16 * 256 * 8);
  cudaMemcpy(in, h, N * 8, cudaMemcpyHostToDevice);
  run<9, 8, 1>("shoup", in, out);
  run<9, 4, 2>("shoup", in, out);
  run<0, 4, 1>("hyb0", in, out); run<0, 4, 2>("hyb0", in, out); run<0, 2, 2>("hyb0", in, out); run<0, 2, 3>("hyb0", in, out);
  run<1, 4, 1>("hyb1", in, out); run<1, 4, 2>("hyb1", in, out); run<1, 2, 2>("hyb1", in, out); run<1, 2, 3>("hyb1", in, out);
  run<1, 8, 1>("hyb1", in, out); run<1, 2, 4>("hyb1", in, out); run<1, 1, 4>("hyb1", in, out);
  run<2, 4, 2>("hyb2_cvt", in, out); run<2, 2, 3>("hyb2_cvt", in, out);
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
