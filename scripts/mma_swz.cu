// Development probe: clk per K-block of k_tc's 22-MMA issue sequence (both diagonal rounds,
// 64 digit pairs, M = 128, K = 32, N = 64..256, A collector) with operands streamed through
// `nst` distinct shared-memory stages, for three operand layouts:
//   layout 0: no swizzle (k_tc today: 8-row x 16-B core matrices, LBO = K-half stride)
//   layout 6: SWIZZLE_32B K-major (rows of 32 B, 8-row atoms of 256 B, SBO = 256)
//   layout 2: SWIZZLE_128B K-major (8-row atoms of 1 KB holding 4 K-blocks; K step = +32 B)
// Optional `nprod` producer warps, paced by the issuer's K-block count, store `stb` bytes per K-block into a separate smem area to load the
// shared-memory port like k_tc's producers (32 KB per K-block and round in the plain form).
// Floor: 64 pairs x N=64 at N/2 clk = 2048 clk per K-block (both rounds).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2004_11571_b200/csrc \
//        scripts/mma_swz.cu -o scripts/mma_swz
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace pe;
using namespace pe::tc;

__device__ __forceinline__ uint64_t desc(u32 saddr, u32 lbo, u32 sbo, int layout) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// one K-block round G, k_tc's wide-MMA sequence with compile-time plane offsets (as in
// tc.cuh issue_round_wide): A plane s at da + s * PA, B plane t at db + t * PB (descriptor units)
template <int G, u32 PA, u32 PB, int DM = 0>
__device__ __forceinline__ void issue(u32 tb, uint64_t da, uint64_t db, bool nocol) {
  int cnt = 0;
  constexpr int d_lo = G == 0 ? 0 : 8, d_hi = G == 0 ? 7 : 14;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int sd = G == 0 ? k : 7 - k;
    const int t_lo = d_lo - sd > 0 ? d_lo - sd : 0;
    const int t_hi = d_hi - sd < 7 ? d_hi - sd : 7;
    if (t_lo > t_hi) continue;
    const int nmma = (t_hi - t_lo) / 4 + 1;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (c >= nmma) continue;
      const int ta = t_lo + 4 * c;
      const int tb2 = ta + 3 < t_hi ? ta + 3 : t_hi;
      const int n = 64 * (tb2 - ta + 1);
      const u32 dt = DM == 0 || DM >= 4 ? tb + (u32)((sd + ta - d_lo) * kV) : DM == 1 ? tb : DM == 2 ? tb + (u32)((cnt & 1) * 256) : tb + (u32)(((sd + ta - d_lo) * kV) & ~(n - 1) & 255);
      ++cnt;
      const uint64_t ad = DM == 5 ? da : da + (uint64_t)(sd * PA);
      const uint64_t bd = DM == 4 ? db : DM == 6 ? db + (uint64_t)((ta & ~(n / 64 - 1)) * PB) : db + (uint64_t)(ta * PB);
      if (nocol || nmma == 1) mma_u8n<0>(dt, ad, bd, idesc_n(n), 1u);
      else if (c == 0) mma_u8n<1>(dt, ad, bd, idesc_n(n), 1u);
      else mma_u8n<2>(dt, ad, bd, idesc_n(n), 1u);
    }
  }
}

// uniform patterns: 4096 / N MMAs of width N per K-block (floor 2048 clk); A plane changes every
// AR MMAs (collector inside a run); B planes cycle
template <int N, int AR, int SH = 0>
__device__ __forceinline__ void issue_uniform(u32 tb, uint64_t da, uint64_t db) {
  constexpr int nm = 4096 / N;
#pragma unroll
  for (int i = 0; i < nm; ++i) {
    const int sd = (i / AR) & 7, pos = i % AR;
    const u32 dt = SH ? tb + (u32)((i * SH) & 255) : tb + (u32)((i * N) & 511);
    const uint64_t ad = da + (uint64_t)(sd * 256);
    const uint64_t bd = db + (uint64_t)((((i * (N / 64)) & 7) & ~(N / 64 - 1)) * 64);
    if (AR == 1) mma_u8n<0>(dt, ad, bd, idesc_n(N), 1u);
    else if (pos == 0) mma_u8n<1>(dt, ad, bd, idesc_n(N), 1u);
    else if (pos == AR - 1) mma_u8n<2>(dt, ad, bd, idesc_n(N), 1u);
    else mma_u8n<3>(dt, ad, bd, idesc_n(N), 1u);
  }
}

// 8 MMAs of the listed widths, each with its own A plane (no collector), B planes from 0
template <int N0, int N1, int N2, int N3, int N4, int N5, int N6, int N7>
__device__ __forceinline__ void issue_list(u32 tb, uint64_t da, uint64_t db) {
  constexpr int Ns[8] = {N0, N1, N2, N3, N4, N5, N6, N7};
#pragma unroll
  for (int i = 0; i < 8; ++i)
    mma_u8n<0>(tb + (u32)((i & 1) * 256), da + (uint64_t)(i * 256), db, idesc_n(Ns[i]), 1u);
}

// the listed widths in order, A plane i & 7, B plane 0, D alternating 0 / 256
template <int... Ns>
__device__ __forceinline__ void issue_seq(u32 tb, uint64_t da, uint64_t db) {
  constexpr int n[] = {Ns...};
#pragma unroll
  for (int i = 0; i < (int)sizeof...(Ns); ++i)
    mma_u8n<0>(tb + (u32)((i & 1) * 256), da + (uint64_t)((i & 7) * 256), db, idesc_n(n[i]), 1u);
}

// k_tc's round-G sequence with four switches: DALT (D alternating 0 / 256 instead of the diagonal
// slots), ADIST (A plane = MMA index & 7 instead of the run's L plane), COL (collector), BCONST (B = plane 0)
template <int G, int DALT, int ADIST, int COL, int BCONST>
__device__ __forceinline__ void issue_x(u32 tb, uint64_t da, uint64_t db) {
  constexpr int d_lo = G == 0 ? 0 : 8, d_hi = G == 0 ? 7 : 14;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int sd = G == 0 ? k : 7 - k;
    const int t_lo = d_lo - sd > 0 ? d_lo - sd : 0;
    const int t_hi = d_hi - sd < 7 ? d_hi - sd : 7;
    if (t_lo > t_hi) continue;
    const int nmma = (t_hi - t_lo) / 4 + 1;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (c >= nmma) continue;
      const int ta = t_lo + 4 * c;
      const int tb2 = ta + 3 < t_hi ? ta + 3 : t_hi;
      const int n = 64 * (tb2 - ta + 1);
      const u32 dt = DALT ? tb + (u32)((cnt & 1) * 256) : tb + (u32)((sd + ta - d_lo) * kV);
      const uint64_t ad = da + (uint64_t)((ADIST ? (cnt & 7) : sd) * 256);
      const uint64_t bd = BCONST ? db : db + (uint64_t)(ta * 64);
      ++cnt;
      if (!COL || nmma == 1) mma_u8n<0>(dt, ad, bd, idesc_n(n), 1u);
      else if (c == 0) mma_u8n<1>(dt, ad, bd, idesc_n(n), 1u);
      else mma_u8n<2>(dt, ad, bd, idesc_n(n), 1u);
    }
  }
}

__global__ void k_swz(int kblocks, int layout, int nst, int nocol, int nprod, int stb, int un, int arun, int same, long long* cyc) {
  extern __shared__ uint8_t dsm[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dsm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar[1];
  __shared__ u32 tmem_base;
  __shared__ u32 no_abort;
  __shared__ volatile int issued;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    no_abort = 0;
    issued = 0;
    mbar_init(&bar[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const u32 tb = tmem_base;
  // stage bytes: layouts 0/6: 32 KB A + 16 KB B; layout 2: 4 K-blocks share 128 KB A + 64 KB B
  const u32 stage = layout == 2 ? 196608u : 49152u;
  const u32 base = smem_u32(sm);
  long long t0 = clock64();
  if (warp == 0) {
    const u32 tbu = uni(tb);
    const bool nc = nocol != 0;
    __syncwarp();
    if (elect_one()) {
      for (int kb = 0; kb < kblocks; ++kb) {
        const u32 st = base + (u32)(kb % nst) * stage;
        const uint64_t da0 = desc(st, 2048, 128, 0), db0 = desc(st + 32768, 8192, 128, 0);
        const uint64_t da6 = desc(st, 16, 256, 6), db6 = desc(st + 32768, 16, 256, 6);
        const u32 kbo = (u32)(kb & 3) * 32;
        const uint64_t da2 = desc(base + kbo, 16, 1024, 2), db2 = desc(base + 131072 + kbo, 16, 1024, 2);
        switch (un) {
          case 256: if (arun == 1) issue_uniform<256, 1>(tbu, da0, db0); else issue_uniform<256, 2>(tbu, da0, db0); break;
          case 128: if (arun == 1) issue_uniform<128, 1>(tbu, da0, db0); else issue_uniform<128, 4>(tbu, da0, db0); break;
          case 1: issue_uniform<256, 1, 64>(tbu, da0, db0); break;
          case 2: issue_uniform<128, 1, 64>(tbu, da0, db0); break;
          case 3: issue<0, 256, 64, 1>(tbu, da0, db0, nc); issue<1, 256, 64, 1>(tbu, da0, db0, nc); break;
          case 4: issue<0, 256, 64, 2>(tbu, da0, db0, nc); issue<1, 256, 64, 2>(tbu, da0, db0, nc); break;
          case 5: issue<0, 256, 64, 3>(tbu, da0, db0, nc); issue<1, 256, 64, 3>(tbu, da0, db0, nc); break;
          case 6: issue_uniform<256, 1, 128>(tbu, da0, db0); break;
          case 7: issue_list<192, 192, 192, 192, 192, 192, 192, 192>(tbu, da0, db0); issue_list<192, 192, 192, 192, 192, 192, 192, 192>(tbu, da0, db0); break;
          case 8: issue_list<256, 64, 256, 64, 256, 64, 256, 64>(tbu, da0, db0); issue_list<256, 64, 256, 64, 256, 64, 256, 64>(tbu, da0, db0); break;
          case 9: issue_list<64, 256, 64, 256, 64, 256, 64, 256>(tbu, da0, db0); issue_list<64, 256, 64, 256, 64, 256, 64, 256>(tbu, da0, db0); break;
          case 10: issue_list<128, 128, 128, 128, 128, 128, 128, 128>(tbu, da0, db0); issue_list<256, 256, 256, 256, 256, 256, 256, 256>(tbu, da0, db0); break;
          case 11: issue_list<256, 128, 256, 128, 256, 128, 256, 128>(tbu, da0, db0); issue_list<256, 128, 256, 128, 256, 128, 256, 128>(tbu, da0, db0); break;
          case 14: issue<0, 256, 64, 4>(tbu, da0, db0, nc); issue<1, 256, 64, 4>(tbu, da0, db0, nc); break;
          case 15: issue<0, 256, 64, 5>(tbu, da0, db0, nc); issue<1, 256, 64, 5>(tbu, da0, db0, nc); break;
          case 16: issue<0, 256, 64, 6>(tbu, da0, db0, nc); issue<1, 256, 64, 6>(tbu, da0, db0, nc); break;
          case 20: issue_seq<256,256,256,192,256,128,256,64,256,192,128,64>(tbu, da0, db0); break;
          case 21: issue_seq<256,256,256,256,256,256,192,192,128,128,64,64>(tbu, da0, db0); break;
          case 22: issue_seq<192,256,192,256,192,256,192,256>(tbu, da0, db0); break;
          case 23: issue_seq<128,64,128,64,128,64,128,64>(tbu, da0, db0); break;
          case 24: issue_seq<256,192,256,192,256,192,256,192>(tbu, da0, db0); break;
          case 25: issue_seq<64,128,192,256,256,64,256,128,256,192>(tbu, da0, db0); break;
          case 26: issue_seq<256,256,256,256,256,256,256,256>(tbu, da0, db0); break;
          case 27: issue_seq<192,192,192,192,192,192,192,192>(tbu, da0, db0); break;
          case 28: issue_seq<256,128,256,128,256,128,256,128>(tbu, da0, db0); break;
          case 100: issue_x<0,0,0,0,0>(tbu, da0, db0); issue_x<1,0,0,0,0>(tbu, da0, db0); break;
          case 101: issue_x<0,0,0,0,1>(tbu, da0, db0); issue_x<1,0,0,0,1>(tbu, da0, db0); break;
          case 102: issue_x<0,0,0,1,0>(tbu, da0, db0); issue_x<1,0,0,1,0>(tbu, da0, db0); break;
          case 103: issue_x<0,0,0,1,1>(tbu, da0, db0); issue_x<1,0,0,1,1>(tbu, da0, db0); break;
          case 104: issue_x<0,0,1,0,0>(tbu, da0, db0); issue_x<1,0,1,0,0>(tbu, da0, db0); break;
          case 105: issue_x<0,0,1,0,1>(tbu, da0, db0); issue_x<1,0,1,0,1>(tbu, da0, db0); break;
          case 108: issue_x<0,1,0,0,0>(tbu, da0, db0); issue_x<1,1,0,0,0>(tbu, da0, db0); break;
          case 109: issue_x<0,1,0,0,1>(tbu, da0, db0); issue_x<1,1,0,0,1>(tbu, da0, db0); break;
          case 110: issue_x<0,1,0,1,0>(tbu, da0, db0); issue_x<1,1,0,1,0>(tbu, da0, db0); break;
          case 111: issue_x<0,1,0,1,1>(tbu, da0, db0); issue_x<1,1,0,1,1>(tbu, da0, db0); break;
          case 112: issue_x<0,1,1,0,0>(tbu, da0, db0); issue_x<1,1,1,0,0>(tbu, da0, db0); break;
          case 113: issue_x<0,1,1,0,1>(tbu, da0, db0); issue_x<1,1,1,0,1>(tbu, da0, db0); break;
          case 12: issue<0, 256, 64>(tbu, da0, db0, nc); issue<0, 256, 64>(tbu, da0, db0, nc); break;
          case 13: issue<1, 256, 64>(tbu, da0, db0, nc); issue<1, 256, 64>(tbu, da0, db0, nc); break;
          case 64: if (arun == 1) issue_uniform<64, 1>(tbu, da0, db0); else issue_uniform<64, 8>(tbu, da0, db0); break;
          default:
            if (layout == 0) { issue<0, 256, 64>(tbu, da0, db0, nc); issue<1, 256, 64>(tbu, da0, db0, nc); }
            else if (layout == 6) { issue<0, 256, 128>(tbu, da6, db6, nc); issue<1, 256, 128>(tbu, da6, db6, nc); }
            else { issue<0, 1024, 512>(tbu, da2, db2, nc); issue<1, 1024, 512>(tbu, da2, db2, nc); }
        }
        issued = kb + 1;
      }
      mma_commit(&bar[0]);
    }
    __syncwarp();
  } else if (warp <= nprod) {   // synthetic producers: 16-B stores into a private 16 KB area
    const u32 area = base + (layout == 2 ? 196608u : (u32)nst * stage);
    const bool b32 = stb < 0;
    const int bytes = b32 ? -stb : stb;
    const int per_warp = bytes / nprod / (b32 ? 128 : 512);   // stores per lane
    uint4 v = make_uint4(warp, lane, 1, 2);
    for (int kb = 0; kb < kblocks; ++kb) {
      while (issued < kb) __nanosleep(32);   // paced by the issuer (its queue runs ahead of the tensor core)
      for (int i = 0; i < per_warp; ++i) {
        const u32 addr = area + (u32)(((warp * 7 + i) & 31) * 512 + lane * 16);
        if (b32) {
          const u32 a4 = area + (u32)(((warp * 7 + i) & 127) * 128 + lane * 4);
          asm volatile("st.shared.b32 [%0], %1;" :: "r"(a4), "r"(v.x) : "memory");
        } else {
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" :: "r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
        v.x += 1;
      }
    }
  }
  if (threadIdx.x == 0) mbar_wait(&bar[0], 0, Abort{&no_abort, nullptr}, 0);
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
  }
}

// k_tc's round-G sequence with the L planes in the order `ord` (the first plane still initialises every
// slot at K-block 0), and a plane's two MMAs issued narrow-first (fill / lastuse) so that each
// K-block ends on wide MMAs: the tensor core's queue then holds more work across the K-block boundary.
template <int G, int LO = 0, int HI = 99>
__device__ __forceinline__ void issue_y(u32 tb, uint64_t da, uint64_t db) {
  constexpr int d_lo = G == 0 ? 0 : 8, d_hi = G == 0 ? 7 : 14;
  int cnt = 0;
  constexpr int ord0[8] = {0, 7, 6, 5, 4, 3, 2, 1}, ord1[8] = {7, 1, 2, 3, 4, 5, 6, 0};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int sd = G == 0 ? ord0[k] : ord1[k];
    const int t_lo = d_lo - sd > 0 ? d_lo - sd : 0;
    const int t_hi = d_hi - sd < 7 ? d_hi - sd : 7;
    if (t_lo > t_hi) continue;
    const int nmma = (t_hi - t_lo) / 4 + 1;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      if (cc >= nmma) continue;
      const int c = (nmma == 2 && k > 0) ? 1 - cc : cc;
      const int me = cnt++;
      if (me < LO || me >= HI) continue;
      const int ta = t_lo + 4 * c;
      const int tb2 = ta + 3 < t_hi ? ta + 3 : t_hi;
      const int n = 64 * (tb2 - ta + 1);
      const u32 dt = tb + (u32)((sd + ta - d_lo) * kV);
      const uint64_t ad = da + (uint64_t)(sd * 256);
      const uint64_t bd = db + (uint64_t)(ta * 64);
      if (nmma == 1) mma_u8n<0>(dt, ad, bd, idesc_n(n), 1u);
      else if (cc == 0) mma_u8n<1>(dt, ad, bd, idesc_n(n), 1u);
      else mma_u8n<2>(dt, ad, bd, idesc_n(n), 1u);
    }
  }
}

// k_tc's stage handshake without generation (its PE_TC_DEBUG=6 path): 4 stages, 2 producer warps per
// stage that wait `empty`, optionally store `stb` bytes (b32 stores) into their stage's A half, and
// arrive on `full`; the MMA warp waits `full`, issues one round (units of 64 K-blocks alternate
// rounds 0 / 1) and commits `empty`.  sleep: poll back-off of the MMA warp / producers (ns).
__global__ void k_hs(int kblocks, int stb, int sl_mma, int sl_prod, int one_round, int nowait, int nocommit, int oneelect, int reord, int early, long long* cyc) {
  extern __shared__ uint8_t dsm[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)dsm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[4], empty[4], done;
  __shared__ u32 tmem_base, no_abort;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    no_abort = 0;
    for (int i = 0; i < 4; ++i) { mbar_init(&full[i], 64); mbar_init(&empty[i], 1); }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const Abort ab{&no_abort, nullptr};
  const u32 tb = tmem_base, base = smem_u32(sm);
  long long t0 = clock64();
  if (warp == 0) {
    const u32 tbu = uni(tb);
    const uint64_t dA0 = desc(uni(base), 2048, 128, 0), dB0 = desc(uni(base) + 32768, 8192, 128, 0);
    if (early) {   // lane 0: issue K-block i up to its last two MMAs, wait for stage i+1, finish i
      if (lane == 0) {
        mbar_wait(&full[0], 0, ab, (u32)sl_mma);
        tc_fence_after();
        for (int kb = 0; kb < kblocks; ++kb) {
          const int stage = kb & 3;
          const uint64_t da = dA0 + (uint64_t)((stage * 49152) >> 4), db = dB0 + (uint64_t)((stage * 49152) >> 4);
          const bool r0 = ((kb >> 6) & 1) == 0;
          const int nlast = r0 ? 10 : 8;   // round 0: 12 MMAs, round 1: 10
          if (r0) issue_y<0, 0, 10>(tbu, da, db); else issue_y<1, 0, 8>(tbu, da, db);
          if (kb + 1 < kblocks) { mbar_wait(&full[(kb + 1) & 3], ((kb + 1) >> 2) & 1, ab, (u32)sl_mma); tc_fence_after(); }
          if (r0) issue_y<0, 10, 99>(tbu, da, db); else issue_y<1, 8, 99>(tbu, da, db);
          (void)nlast;
          mma_commit(&empty[stage]);
          if (kb + 1 == kblocks) mma_commit(&done);
        }
      }
    } else
    for (int kb = 0; kb < kblocks; ++kb) {
      const int stage = kb & 3, use = kb >> 2;
      if (oneelect && lane != 0) break;
      if (!nowait) mbar_wait(&full[stage], use & 1, ab, (u32)sl_mma);
      tc_fence_after();
      const uint64_t da = dA0 + (uint64_t)((stage * 49152) >> 4), db = dB0 + (uint64_t)((stage * 49152) >> 4);
      if (oneelect) {   // lane 0 alone issues (no per-K-block converge / elect)
        if (lane == 0) {
          if (reord) {
            if (one_round || ((kb >> 6) & 1) == 0) issue_y<0>(tbu, da, db);
            else issue_y<1>(tbu, da, db);
          } else if (one_round || ((kb >> 6) & 1) == 0) issue_x<0, 0, 0, 1, 0>(tbu, da, db);
          else issue_x<1, 0, 0, 1, 0>(tbu, da, db);
          if (!nocommit) mma_commit(&empty[stage]);
          if (kb + 1 == kblocks) mma_commit(&done);
        }
        continue;
      }
      __syncwarp();
      if (elect_one()) {
        if (reord) {
          if (one_round || ((kb >> 6) & 1) == 0) issue_y<0>(tbu, da, db);
          else issue_y<1>(tbu, da, db);
        } else if (one_round || ((kb >> 6) & 1) == 0) issue_x<0, 0, 0, 1, 0>(tbu, da, db);
        else issue_x<1, 0, 0, 1, 0>(tbu, da, db);
        if (!nocommit) mma_commit(&empty[stage]);
        if (kb + 1 == kblocks) mma_commit(&done);
      }
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0) mbar_wait(&done, 0, ab, 0);
  } else if (warp <= 8 && !nowait) {
    const int pw = warp - 1, my_stage = pw >> 1, sub = pw & 1;
    const u32 area = base + (u32)my_stage * 49152 + (u32)sub * 16384;
    const int per_lane = stb / 2 / 128;
    for (int use = 0;; ++use) {
      const int kb = my_stage + 4 * use;
      if (kb >= kblocks) break;
      mbar_wait(&empty[my_stage], (use & 1) ^ 1, ab, (u32)sl_prod);
      for (int i = 0; i < per_lane; ++i)
        asm volatile("st.shared.b32 [%0], %1;" :: "r"(area + (u32)((i & 127) * 128 + lane * 4)), "r"(i) : "memory");
      fence_async_smem();
      mbar_arrive(&full[my_stage]);
    }
  }
  long long t1 = clock64();
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
  }
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  cudaMalloc(&cyc, nsm * sizeof(long long));
  const int smem = 215 * 1024;
  cudaFuncSetAttribute(k_swz, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int kblocks = 2048;
  struct Cfg { int layout, nst, nocol, nprod, stb, un, arun, same; };
  const Cfg cfgs[] = {
      {0, 4, 0, 0, 0, 102, 1, 0},
  };
  // floor clk per call (sum of N / 2)
  auto fl = [](int u) -> double {
    switch (u) { case 20: return 1152; case 21: return 1152; case 22: return 896; case 23: return 384; case 24: return 896;
                 case 25: return 832; case 26: return 1024; case 27: return 768; case 28: return 768; default: return 2048; }
  };
  const double floors[14] = {2048, 2048, 2048, 2048, 2048, 2048, 2048, 1536, 2560, 2560, 1536, 3072, 2304, 1792};
  for (const Cfg& c : cfgs) {
    for (int rep = 0; rep < 2; ++rep) k_swz<<<nsm, 288, smem>>>(kblocks, c.layout, c.nst, c.nocol, c.nprod, c.stb, c.un, c.arun, c.same, cyc);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int b = 0; b < nsm; ++b) s += (double)h[b];
    s /= nsm;
    printf("case=%3d (dalt adist col bconst = %d %d %d %d) uniformN=%3d arun=%d same=%d layout=%d stages=%d nocol=%d prod_warps=%d prod_bytes/kb=%6d  clk/K-block %.0f (floor 2048: %.2f)  %s\n",
           c.un, (c.un - 100) >> 3 & 1, (c.un - 100) >> 2 & 1, (c.un - 100) >> 1 & 1, (c.un - 100) & 1, c.un, c.arun, c.same, c.layout, c.nst, c.nocol, c.nprod, c.stb, s / kblocks, fl(c.un) * kblocks / s, cudaGetErrorString(e));
  }
  cudaFuncSetAttribute(k_hs, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  struct H { int stb, slm, slp, one, nw, nc, oe, ro, ea; };
  const H hs[] = {{0, 32, 64, 0, 0, 0, 0, 0, 0}, {0, 32, 64, 0, 0, 0, 0, 1, 0}, {0, 32, 64, 0, 0, 0, 1, 1, 1}, {0, 0, 64, 0, 0, 0, 1, 1, 1}, {32768, 32, 64, 0, 0, 0, 1, 1, 1}, {0, 32, 64, 0, 1, 0, 1, 1, 0}};
  for (const H& c : hs) {
    for (int rep = 0; rep < 2; ++rep) k_hs<<<nsm, 288, smem>>>(kblocks, c.stb, c.slm, c.slp, c.one, c.nw, c.nc, c.oe, c.ro, c.ea, cyc);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int b = 0; b < nsm; ++b) s += (double)h[b];
    s /= nsm;
    const double fl = c.one ? 1152.0 : 1024.0;
    printf("handshake: early=%d reorder=%d nocommit=%d lane0-only=%d nowait=%d stores/kb=%6d sleep mma/prod=%d/%d one_round=%d  clk/K-block-round %.0f (floor %.0f: %.2f)  %s\n",
           c.ea, c.ro, c.nc, c.oe, c.nw, c.stb, c.slm, c.slp, c.one, s / kblocks, fl, fl * kblocks / s, cudaGetErrorString(e));
  }
  return 0;
}
