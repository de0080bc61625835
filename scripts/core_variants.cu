// core_variants.cu -- scratch harness: alternative PTX forms of the Shoup-lazy step, compiled in a
// k_step-like loop (R chains x 8 points with 96-bit accumulators) to compare IMAD-pipe slots in
// SASS (scripts/sass_slots.py) and, on the GPU, throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o core_variants core_variants.cu
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


__device__ __forceinline__ void add96(U96& x, const U96& y) {
  asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
      : "+r"(x.w0), "+r"(x.w1), "+r"(x.w2) : "r"(y.w0), "r"(y.w1), "r"(y.w2));
}
__device__ __forceinline__ U96 shfl96(const U96& x, int off) {
  U96 r; r.w0 = __shfl_xor_sync(0xffffffffu, x.w0, off); r.w1 = __shfl_xor_sync(0xffffffffu, x.w1, off);
  r.w2 = __shfl_xor_sync(0xffffffffu, x.w2, off); return r;
}
__device__ __forceinline__ U96 sel96(bool c, const U96& a, const U96& b) {
  U96 r; r.w0 = c ? a.w0 : b.w0; r.w1 = c ? a.w1 : b.w1; r.w2 = c ? a.w2 : b.w2; return r;
}
__device__ __forceinline__ U96 xpose8(U96 (&v)[8], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  U96 t4[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) { U96 s = sel96(b4, v[i], v[i + 4]); t4[i] = sel96(b4, v[i + 4], v[i]); add96(t4[i], shfl96(s, 16)); }
  U96 t2[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) { U96 s = sel96(b3, t4[i], t4[i + 2]); t2[i] = sel96(b3, t4[i + 2], t4[i]); add96(t2[i], shfl96(s, 8)); }
  U96 s = sel96(b2, t2[0], t2[1]); U96 t1 = sel96(b2, t2[1], t2[0]); add96(t1, shfl96(s, 4));
  add96(t1, shfl96(t1, 2)); add96(t1, shfl96(t1, 1)); return t1;
}

// V0: current library form
__device__ __forceinline__ u64 mul_v0(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, t1, t2, q0, q1, r0, r1;\n\t.reg .u64 q, rr;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {w0, w1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.hi.u32 t1, a1, w0;\n\tmul.hi.u32 t2, a0, w1;\n\tmul.wide.u32 q, a1, w1;\n\tmov.b64 {q0, q1}, q;\n\t"
      "add.cc.u32 q0, q0, t1;\n\taddc.u32 q1, q1, 0;\n\tadd.cc.u32 q0, q0, t2;\n\taddc.u32 q1, q1, 0;\n\t"
      "mul.wide.u32 rr, a0, m0;\n\tmad.wide.u32 rr, q0, n0, rr;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, a1, m0, r1;\n\tmad.lo.u32 r1, q0, n1, r1;\n\tmad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(w), "l"(np));
  return r;
}
// V1: q via mad.lo.cc / madc.hi (no 64-bit addend pairs)
__device__ __forceinline__ u64 mul_v1(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, t1, t2, s, c, q0, q1, r0, r1;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {w0, w1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.hi.u32 t1, a1, w0;\n\tmul.hi.u32 t2, a0, w1;\n\t"
      "add.cc.u32 s, t1, t2;\n\taddc.u32 c, 0, 0;\n\t"
      "mad.lo.cc.u32 q0, a1, w1, s;\n\tmadc.hi.u32 q1, a1, w1, c;\n\t"
      "mad.lo.cc.u32 r0, a0, m0, 0;\n\tmadc.hi.u32 r1, a0, m0, 0;\n\t"
      "mad.lo.cc.u32 r0, q0, n0, r0;\n\tmadc.hi.u32 r1, q0, n0, r1;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, a1, m0, r1;\n\tmad.lo.u32 r1, q0, n1, r1;\n\tmad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(w), "l"(np));
  return r;
}
// V2: plain C (compiler's choice)
__device__ __forceinline__ u64 mul_v2(u64 a, u64 m, u64 w, u64 np) {
  const u32 a0 = (u32)a, a1 = (u32)(a >> 32), w0 = (u32)w, w1 = (u32)(w >> 32);
  u64 q = (u64)a1 * w1 + (u64)__umulhi(a1, w0) + (u64)__umulhi(a0, w1);
  return a * m + q * np;
}
// V3: q high via a single 64-bit-addend chain: q = a1*w1 + hi(a0*w1) as mad.wide with addend
//     {t2,0}; then + t1 with add.cc; r as V0.
__device__ __forceinline__ u64 mul_v3(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, t1, t2, q0, q1, r0, r1, z;\n\t.reg .u64 q, rr, tt;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {w0, w1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.hi.u32 t1, a1, w0;\n\tmul.hi.u32 t2, a0, w1;\n\tmov.u32 z, 0;\n\tmov.b64 tt, {t1, z};\n\t"
      "mad.wide.u32 q, a1, w1, tt;\n\tmov.b64 {q0, q1}, q;\n\t"
      "add.cc.u32 q0, q0, t2;\n\taddc.u32 q1, q1, 0;\n\t"
      "mul.wide.u32 rr, a0, m0;\n\tmad.wide.u32 rr, q0, n0, rr;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, a1, m0, r1;\n\tmad.lo.u32 r1, q0, n1, r1;\n\tmad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(w), "l"(np));
  return r;
}
// V4: like V1 but r's low products via mul.wide (pairs), q via madc
__device__ __forceinline__ u64 mul_v4(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, t1, t2, s, c, q0, q1, r0, r1;\n\t.reg .u64 rr;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {w0, w1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.hi.u32 t1, a1, w0;\n\tmul.hi.u32 t2, a0, w1;\n\t"
      "add.cc.u32 s, t1, t2;\n\taddc.u32 c, 0, 0;\n\t"
      "mad.lo.cc.u32 q0, a1, w1, s;\n\tmadc.hi.u32 q1, a1, w1, c;\n\t"
      "mul.wide.u32 rr, a0, m0;\n\tmad.wide.u32 rr, q0, n0, rr;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, a1, m0, r1;\n\tmad.lo.u32 r1, q0, n1, r1;\n\tmad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(w), "l"(np));
  return r;
}

// V5: cross terms as full products (pairs), high halves summed on the ALU (+ low-half carry)
__device__ __forceinline__ u64 mul_v5(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, x1l, x1h, x2l, x2h, s, c, z, q0, q1, r0, r1;\n\t.reg .u64 x1, x2, rr;\n\t"
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
// V6: library form (madc q, mul.wide r)
__device__ __forceinline__ u64 mul_v6(u64 a, u64 m, u64 w, u64 np) {
  u64 r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, w0, w1, n0, n1, t1, t2, s, c, q0, q1, r0, r1;\n\t.reg .u64 rr;\n\t"
      "mov.b64 {a0, a1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\tmov.b64 {w0, w1}, %3;\n\tmov.b64 {n0, n1}, %4;\n\t"
      "mul.hi.u32 t1, a1, w0;\n\tmul.hi.u32 t2, a0, w1;\n\tadd.cc.u32 s, t1, t2;\n\taddc.u32 c, 0, 0;\n\t"
      "mad.lo.cc.u32 q0, a1, w1, s;\n\tmadc.hi.u32 q1, a1, w1, c;\n\t"
      "mul.wide.u32 rr, a0, m0;\n\tmov.b64 {r0, r1}, rr;\n\t"
      "mad.lo.cc.u32 r0, q0, n0, r0;\n\tmadc.hi.u32 r1, q0, n0, r1;\n\t"
      "mad.lo.u32 r1, a0, m1, r1;\n\tmad.lo.u32 r1, a1, m0, r1;\n\tmad.lo.u32 r1, q0, n1, r1;\n\tmad.lo.u32 r1, q1, n0, r1;\n\t"
      "mov.b64 %0, {r0, r1};\n\t}" : "=l"(r) : "l"(a), "l"(m), "l"(w), "l"(np));
  return r;
}

template <int V>
__device__ __forceinline__ u64 mulv(u64 a, u64 m, u64 w, u64 np) {
  if (V == 0) return mul_v0(a, m, w, np);
  if (V == 1) return mul_v1(a, m, w, np);
  if (V == 2) return mul_v2(a, m, w, np);
  if (V == 3) return mul_v3(a, m, w, np);
  if (V == 5 || V == 105) return mul_v5(a, m, w, np);
  if (V == 6) return mul_v6(a, m, w, np);
  return mul_v4(a, m, w, np);
}

template <int V, int R>
__global__ void __launch_bounds__(256, 2) kv(const u64* __restrict__ in, u64 np, int groups, u64* out) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  u64 a[R], m[R], w[R];
#pragma unroll
  for (int r = 0; r < R; ++r) { a[r] = in[tid * 3 * R + r]; m[r] = in[tid * 3 * R + R + r]; w[r] = in[tid * 3 * R + 2 * R + r]; }
  U96 tot{0, 0, 0};
#pragma unroll 1
  for (int g = 0; g < groups; ++g) {
    U96 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      set96_sum(acc[k], a[0], a[1]);
#pragma unroll
      for (int r = 2; r < R; ++r) add96_64(acc[k], a[r]);
#pragma unroll
      for (int r = 0; r < R; ++r) a[r] = mulv<V>(a[r], m[r], w[r], np);
    }
    if (V >= 100) {
      U96 x = xpose8(acc, threadIdx.x & 31);
      tot.w0 ^= x.w0; tot.w1 += x.w1; tot.w2 ^= x.w2;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) { tot.w0 ^= acc[k].w0; tot.w1 += acc[k].w1; tot.w2 ^= acc[k].w2; }
    }
  }
  out[tid] = tot.w0 ^ ((u64)tot.w1 << 32) ^ tot.w2 ^ a[0];
}

template <int V>
void run(const char* nm, u64* in, u64* out, int groups) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 2, threads = 256;
  kv<V, 8><<<blocks, threads>>>(in, 0xC000000000000039ull, groups, out);
  cudaEventRecord(e0);
  kv<V, 8><<<blocks, threads>>>(in, 0xC000000000000039ull, groups, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double tp = (double)blocks * threads * 8 * 8 * groups;
  printf("{\"variant\": \"%s\", \"ms\": %.3f, \"Tterm_pt_s\": %.4f, \"per_clk_sm_at_1965\": %.3f}\n", nm, ms,
         tp / (ms * 1e-3) / 1e12, tp / (ms * 1e-3) / (148 * 1965e6));
}

int main() {
  const int N = 148 * 2 * 256 * 3 * 8;
  u64* h = new u64[N];
  const u64 p = (1ull << 62) - 57;
  for (int i = 0; i < N; ++i) h[i] = (0x9E3779B97F4A7C15ull * (i + 1)) % p;
  u64 *in, *out;
  cudaMalloc(&in, N * 8); cudaMalloc(&out, 148 * 2 * 256 * 8);
  cudaMemcpy(in, h, N * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; ++rep) {
    run<0>("v0_current", in, out, 2048);
    run<1>("v1_madc", in, out, 2048);
    run<2>("v2_plainC", in, out, 2048);
    run<3>("v3_pairaddend", in, out, 2048);
    run<4>("v4_madc_q_wide_r", in, out, 2048);
    run<5>("v5_wide_cross", in, out, 2048);
    run<6>("v6_library", in, out, 2048);
    run<105>("v5_plus_xpose", in, out, 2048);
  }
  printf("{\"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
