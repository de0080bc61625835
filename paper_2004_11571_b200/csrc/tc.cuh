// tc.cuh -- tensor-core form of the step-and-reduce (rows a5 + a6) for p < 2^63 (sm_100a).
//
// The matrix method's T x s evaluation matrix has the Vandermonde structure V[j][i] = m_i^j
// ("M_i(beta^t) = m_i^t"; PAPER.md:465-478 transposed Vandermonde).  Writing a
// chunk's points as j = j_s + u*V + v (u < U, v < V) factors every bucket's block of outputs
// into one dense product per bucket g (baby-step / giant-step):
//
//     out[g][j_s + uV + v] = sum_{i in g} L[u][i] * R[i][v]   (mod p),
//     L[u][i] = c_i m_i^{j_s + uV}   (giant steps: a_i <- a_i * m_i^V),
//     R[i][v] = m_i^v                (baby steps:  a_i <- a_i * m_i),
//
// i.e. U + V modular products per term give U*V term-points, and the remaining work --
// U*V*s multiply-adds -- is a dense contraction over the terms of a bucket, which is what
// the 5th-generation tensor cores do.  Exactness: L and R are split into their 8 unsigned
// bytes (L = sum_s 2^{8s} L_s), every byte product L_s R_t is an exact int8 MMA with int32
// accumulation in TMEM, and the 64 (s, t) products are summed by diagonal d = s + t:
//     X = sum_d 2^{8d} D_d,   D_d = sum_{s+t=d} L_s R_t,   D_d < 8192 * 8 * 255^2 < 2^32
// for <= 8192 terms per accumulation (a "piece"; the s32 TMEM accumulator wraps mod 2^32 without
// saturation, so its bits read as u32 are exact).  X mod p = sum_d D_d (2^{8d} mod p) mod p.
//
// Shapes: U = M = 128 (TMEM lanes), K-block = 32 terms (one kind::i8 MMA K step), V by mode
// (mode_v):
//   V = 32 (8-digit modes, p >= 2^54 -- config 5 -- and 7-digit modes, 2^31 <= p < 2^54): all 15
//     (13) diagonals fit TMEM at once (15 x 32 = 480 of 512 columns), so a unit is (piece, chunk
//     of 128 x 32 points) in ONE round: per K-block, L plane s against the 8 (7) consecutive R
//     planes is ONE MMA of N = 256 (224) into slots s .. s + 7 (issue_all32 / issue_all32_7), one
//     fold + REDC per point (epi_drain5<5 / 6>, fold_row<5 / 6, 32>).
//   V = 64 (the 4-digit mode, p < 2^31: 7 diagonals, one round of 5 MMAs; and the two-round forms
//     kept for reference -- issue_round_wide, issue_round7_*): with 8 digits 15 x 64 columns do
//     not fit, so a piece ran in 2 rounds (d = 0..7 and 8..14, slot = d - d_lo) and a unit was
//     (piece, chunk, round) reducing its own part X_g into its own partial row (X mod p = sum of
//     the parts); a round's partners t of one L plane s are consecutive, so each (s, run of t) is
//     ONE MMA with N = 64k <= 256.
// The baby-step planes R = m^v do not depend on the points: they are built once per handle and
// streamed into the stages by TMA, so per evaluation only the giant steps are generated (1
// modular product per 32 term-points).
//
// Warp roles (one CTA per SM, 12 warps = 3 per SMSP, persistent; units are piece-major and dealt
// to the CTAs in snake order or by the host's LPT schedule):
//   warps 0-3  epilogue: tcgen05.ld the unit's diagonals (TMEM lane = u) into the unit's raw
//              buffer (per-CTA, L2-resident), release TMEM; then an exact 160-bit fold of the
//              unit's diagonals and one reduction mod p per point (warps 1-3; warps 2 / 3 also
//              cover warp 0's rows) -> partial[slot][chunk * 128 V + u V + v].  Warp 0 issues
//              every unit's MMAs (tcgen05.mma.cta_group::1.kind::i8, elect.sync leader) and
//              allocates TMEM.
//   warps 4-11 producers, 2 per smem stage: each generates 16 terms x 128 giant-step rows of one
//              K-block with Shoup products (4 chains per lane, seeded from the chunk seed) and
//              writes their 8 byte planes in the no-swizzle K-major UMMA layout; one warp's first
//              lane copies the K-block's baby-step planes into the stage with TMA, the other's
//              prefetches the group's next K-block of per-term records.
//
// Swapped form (MODE 4 / 5, 8-digit p >= 2^54; the automatic form, pe_config.tc_form): the
// point-dependent factor c m^{j_s} is folded into the baby steps instead, R'[i][v] =
// c_i m_i^{j_s + v}, and the giant steps G[u][i] = m_i^{uV} become the point-independent factor,
// built once per handle (k_tc_gplanes, Montgomery residues, 1 KB per term) and streamed into the
// A half of the stages by TMA.  The producers then generate only the V = 32 baby-step rows per
// term and unit (a quarter of the plain form's 128 giant-step rows) into the B half; the MMAs,
// the TMEM layout and the epilogue are the same (sum_i G R' = 2^64 X, one REDC).  On config 5 the
// tensor core then binds: 91 % tensor-pipe utilisation (profiles/r02_ktc_summary.json).
#pragma once
#include "modcore.cuh"

namespace pe {
namespace tc {

constexpr int kU = 128;                   // giant steps per chunk  (MMA M / TMEM lanes)
constexpr int kV = 64;                    // baby steps per chunk of the V = 64 modes (mode_v)
constexpr u32 kChunk = kU * kV;           // points per chunk
constexpr int kKB = 32;                   // terms per K-block (one i8 MMA K step)
constexpr int kStages = 4;
constexpr u32 kPieceMax = 8192;           // terms per accumulation: 8192 * 8 * 255^2 < 2^32 (the s32
                                          // accumulator wraps mod 2^32, saturate = 0; read as u32)
// Digit planes in the no-swizzle K-major UMMA layout: 8-row x 16-byte core matrices, rows of a
// core-matrix column 128 B apart (SBO), the two 16-byte K halves LBO apart.
constexpr u32 kLBOA = 2048;               // L planes (A, 128 rows): writes are conflict-free unpadded
constexpr u32 kPlaneA = kLBOA + 2048;
// R planes (B, 64 rows, written by TMA only): [K half][plane t][64 rows x 16 B], so planes
// t .. t+k-1 are one B operand of N = 64k rows (SBO 128) -- one MMA covers k diagonals
constexpr u32 kPlaneB = kV * 16;          // one plane's rows in one K half (1 KB)
constexpr u32 kLBOB = 8 * kPlaneB;        // K-half stride (8 KB)
constexpr u32 kStageBytes = 8 * kPlaneA + 2 * kLBOB;     // 8 L planes + 8 R planes (49152 B)
constexpr u32 kGBytes = 8 * kPlaneA;      // one K-block's giant-step planes in the A layout (32 KB)
// Per-term records (array of structs, so one K-block's data is two contiguous bulk copies):
//   LS record (per chunk, 1 u64): the chunk seed c m^{j_s}
//   C  record (10 u64): the giant-step chain multiplier m^{8V} and its Shoup constant, and the
//      Montgomery residues of m^{rr V} (rr < 8) that turn the chunk seed into the 8 chain seeds
// The baby-step factors R[i][v] = m_i^v do not depend on the points: pe_create writes their byte
// planes once per handle, in the stage's R-plane layout ([t_pad / 32][kRBytes], k_tc_rplanes),
// and each K-block's 16.5 KB is one TMA bulk copy into the stage.
constexpr int kLSRec = 1, kCRec = 10;
enum { kC_mL = 0, kC_wL = 1, kC_g0 = 2 };
constexpr u32 kRBytes = 2 * kLBOB;                    // one K-block's R planes (16384 B)
// Geometry of a mode: V baby steps per chunk, a chunk = kU * V points.  Every mode but the 4-digit
// one uses V = 32: all 15 (7 digits: 13) diagonals then fit TMEM at once (15 x 32 = 480 columns), so
// a unit is (piece, chunk) in ONE round -- 8 MMAs of N = 256 per K-block (L plane s against the 8
// baby-step planes, slots s .. s + 7) -- with half the baby-step plane bytes per term (256 B) and
// one fold + REDC per point instead of one per round; the plain and swapped 8-digit forms alike.
// The 4-digit mode (p < 2^31: 7 diagonals, one round at V = 64) keeps V = 64, where V = 32 would
// double its generation per point.
__host__ __device__ constexpr int mode_v(int MODE) { return MODE == 2 ? 64 : 32; }
__host__ __device__ constexpr u32 plane_b(int V) { return (u32)V * 16; }      // one R plane, one K half
__host__ __device__ constexpr u32 lbo_b(int V) { return 8 * plane_b(V); }     // R planes' K-half stride
__host__ __device__ constexpr u32 r_bytes(int V) { return 2 * lbo_b(V); }     // one K-block's R planes
__host__ __device__ constexpr u32 chunk_pts(int V) { return (u32)kU * (u32)V; }
constexpr u32 kDataLS = kKB * kLSRec * 8;             // 256 B
constexpr u32 kDataSlot = kDataLS + kKB * kCRec * 8;  // 2816 B
constexpr int kDataSlots = 2 * kStages;               // 2 per producer group: current + next K-block
constexpr u32 kSmemBytes = kStages * kStageBytes + kDataSlots * kDataSlot + 128;
constexpr int kRounds = 2;
constexpr int kDiag = 8;                  // diagonal accumulators per round: 8 x 64 TMEM columns
constexpr int kProdPerStage = 2;          // L terms 0-15, L terms 16-31 (128 rows each)
constexpr int kEpiWarps = 4, kMmaWarp = 0, kProdWarp0 = 4;   // warp 0: epilogue + MMA issue
constexpr int kThreads = (kProdWarp0 + kStages * kProdPerStage) * 32;   // 12 warps: 3 per SMSP
static_assert(kRounds <= kEpiWarps, "round g's MMAs are issued by epilogue warp g");
static_assert(kDiag * kV == 512, "a round's accumulators fill TMEM");
static_assert(kSmemBytes + 256 <= 232448, "shared memory");
// diagonal rounds: d = 0..7 and d = 8..14 (36 + 28 digit pairs); accumulator slot = d - d_lo, so
// for one L plane s the round's pairs (s, t) have consecutive t and land in consecutive slots:
// one wide MMA (B = planes t..t+k-1, N = 64k <= 256) covers k of them
// group 2: the single round of the 4-digit mode (p < 2^31: values < 2^32), d = 0..6
// group 4: the 7-digit mode's second round, d = 8..12
// group 5: the single round of the V = 32 geometry, d = 0..14 in slots 0..14 (8 digits);
// group 6: the same for 7 digits (2^31 <= p < 2^54), d = 0..12 in slots 0..12
__host__ __device__ constexpr int group_diag(int g, int di) {
  return g == 0 ? (di < 8 ? di : -1) : g == 1 ? (di < 7 ? 8 + di : -1) : g == 2 ? (di < 7 ? di : -1)
       : g == 5 ? (di < 15 ? di : -1) : g == 6 ? (di < 13 ? di : -1) : (di < 5 ? 8 + di : -1);
}
__host__ __device__ constexpr int nslots(int g) { return g == 5 ? 15 : g == 6 ? 13 : kDiag; }

struct TcArgs {
  const u64* LS;         // [nch][t_pad] chunk seeds c m^{j_s}
  const u64* C;          // [t_pad][10] C records (giant-step chain multiplier, m^{rr V} table)
  const uint8_t* Rp;     // [t_pad / 32][kRBytes] baby-step byte planes (k_tc_rplanes), MODE 0-3
  const uint8_t* Gp;     // [t_pad / 32][kGBytes] giant-step byte planes (k_tc_gplanes), MODE 4-5
  const uint4* piece;    // x = first padded term, y = K-blocks, z = partial slot (sorted by size desc)
  const u32* sched;      // units of CTA b: sched[sched_off[b] .. sched_off[b+1])  (host LPT schedule)
  const u32* sched_off;  // [gridDim.x + 1]
  u64* partial;          // [n_slots][ldp]
  u64* out;              // output row of the launch's first bucket, at the pass's first point
  u64 ldo;               // its leading dimension
  int direct;            // 1: a bucket's sole piece (piece.w = 1 + row) writes its row of out directly
  u64 ldp, t_pad;
  u32 npieces, nunits, npts, nch;
  u32 rounds;            // diagonal rounds per (piece, chunk): 2 (8-byte digits) or 1 (4-byte, p < 2^31)
  u64 Wd[15];            // 2^{8d} mod p  (Wd[8] = 2^64, Wd[12] = 2^96, Wd[14] -> see C128)
  u64 C128;              // 2^128 mod p
  u32* scratch;          // per CTA: 2 (ping-pong by unit) x kDiag accumulators x kChunk u32 drained diagonal sums
  ModParams mp;
  int discard;           // 1: discard the raw scratch lines from L2 once folded (PE_TC_DISCARD, default 1)
  u32 sleep_ns[3];       // poll back-off (ns) of the MMA warp's stage wait, the producers' stage wait and
                         // the epilogue's accumulator wait (32 / 64 / 64; env PE_TC_SLEEP=a,b,c)
  u32* status;           // mapped host word (pe_ctx::h_status): set to 1 if a pipeline wait timed out
  unsigned long long* prof;  // optional phase timers [gridDim][warps][4] (PE_TC_PROF=1), else null
  int dbg;                   // development only (PE_TC_DEBUG, PROF build): 1 = skip the MMAs,
                             // 2 = producers skip generation, 3 = the TMEM drain skips its stores,
                             // 4 = no baby-step plane copies, 6 = 2 + 4, 7 = 6 without the A collector
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t smem_desc(u32 saddr, u32 lbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;    // leading (K) byte offset
  d |= (uint64_t)((128u >> 4) & 0x3FFF) << 32;   // stride (8-row group) byte offset
  d |= (uint64_t)1 << 46;                        // sm_100 descriptor version; no swizzle
  return d;
}
// kind::i8, D s32, A u8, B u8, both K-major, M = kU = 128, N = kV = 64
constexpr u32 kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | ((u32)(kV >> 3) << 17) | ((u32)(kU >> 4) << 24);

__device__ __forceinline__ void mma_u8(u32 dtmem, uint64_t ad, uint64_t bd, u32 acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(dtmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ bool elect_one() {
  u32 pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
// warp-uniform value (lets the compiler keep it in the uniform datapath for tcgen05 operands)
__device__ __forceinline__ u32 uni(u32 x) { return __shfl_sync(0xffffffffu, x, 0); }

// MMA with an A-operand collector mode: 0 = read A (no keep), 1 = read A and keep it in the
// collector buffer (fill), 2 = reuse the collector's A and keep it (use), 3 = reuse and release
// (lastuse).  Reusing A removes its 4 KB shared-memory read from all but the first MMA of a run.
template <int COL>
__device__ __forceinline__ void mma_u8c(u32 dtmem, uint64_t ad, uint64_t bd, u32 acc) {
  if (COL == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
  else if (COL == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
  else if (COL == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
}

template <int COL>
__device__ __forceinline__ void mma_u8n(u32 dtmem, uint64_t ad, uint64_t bd, u32 idesc, u32 acc) {
  if (COL == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
  else if (COL == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::fill [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
  else if (COL == 2)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8.collector::a::use [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__host__ __device__ constexpr u32 idesc_n(int n) {
  return (2u << 4) | ((u32)(n >> 3) << 17) | ((u32)(kU >> 4) << 24);
}

// Round G on one stage as wide MMAs: for each L plane s the round's partners t form one range
// [t_lo, t_hi]; it is issued as MMAs of <= 4 consecutive R planes (N = 64k), D = slots
// s + t - d_lo ...  The plane whose range covers every slot of the round (s = 0 for d = 0..7,
// s = 7 for d = 8..14) goes first, so at K-block 0 it initialises all accumulators (acc = 0) and
// every later MMA accumulates.  A plane issued as two MMAs keeps A in the collector.
// Order (wide_ord: planes 0, 7, 6, .., 1 for round 0 and 7, 1, 2, .., 6 for round 1): after the
// initialising plane, the planes with the fewest partners come first and a plane's narrow MMA
// precedes its wide one, so every K-block ends on wide MMAs and the tensor core's queue still holds
// ~250 clk of work while the issuing warp crosses the K-block boundary (stage wait, commit, loop).
// Measured: the stage handshake alone (scripts/mma_swz.cu k_hs) 0.72 -> 0.80 of the MMA floor;
// whole k_tc on config 5 (ncu sm__cycles_elapsed) 13.47 M -> 13.20 M clk, bench +1.3 % burst and
// +1 % sustained at the power cap (profiles/r02_ktc_issue_order.txt).  Moving the next stage's
// wait in front of the last two MMAs as well took the MMA path alone to 0.86 of its floor, but
// the whole kernel to 13.89 M clk (the producers then lose more to the tensor core's shared-
// memory reads), so it is not used.  MMAs LO <= i < HI of the order are issued.
__host__ __device__ constexpr int wide_ord(int g, int k) { return g == 0 ? (k == 0 ? 0 : 8 - k) : (k == 0 ? 7 : k == 7 ? 0 : k); }
template <int G, int LO = 0, int HI = 16>
__device__ __forceinline__ void issue_round_wide(u32 tb, uint64_t da, uint64_t db, bool first_kb) {
  constexpr int d_lo = G == 0 ? 0 : 8, d_hi = G == 0 ? 7 : 14;
  int idx = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int sd = wide_ord(G, k);
    const int t_lo = d_lo - sd > 0 ? d_lo - sd : 0;
    const int t_hi = d_hi - sd < 7 ? d_hi - sd : 7;
    if (t_lo > t_hi) continue;
    const int nmma = (t_hi - t_lo) / 4 + 1;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      if (cc >= nmma) continue;
      const int me = idx++;
      if (me < LO || me >= HI) continue;
      const int c = (nmma == 2 && k > 0) ? 1 - cc : cc;   // narrow part first (c = 1 is the tail run)
      const int ta = t_lo + 4 * c;
      const int tb2 = ta + 3 < t_hi ? ta + 3 : t_hi;
      const int n = 64 * (tb2 - ta + 1);
      const u32 acc = (!first_kb || k > 0) ? 1u : 0u;
      const u32 dt = tb + (u32)((sd + ta - d_lo) * kV);
      const uint64_t ad = da + (uint64_t)((u32)sd * (kPlaneA >> 4));
      const uint64_t bd = db + (uint64_t)((u32)ta * (kPlaneB >> 4));
      if (nmma == 1) mma_u8n<0>(dt, ad, bd, idesc_n(n), acc);
      else if (cc == 0) mma_u8n<1>(dt, ad, bd, idesc_n(n), acc);
      else mma_u8n<2>(dt, ad, bd, idesc_n(n), acc);
    }
  }
}

// Single-round geometry (V = 32): L plane s against all 8 baby-step planes is ONE MMA of N = 256
// into slots s .. s + 7 (TMEM columns 32 s ..); 8 MMAs per K-block, all 256 wide.  At K-block 0
// plane 0 initialises slots 0..7 and plane 7 goes second, split so that its t = 1..7 part
// initialises slots 8..14 (its t = 0 part accumulates into slot 7); planes 1..6 then accumulate.
__device__ __forceinline__ void issue_all32(u32 tb, uint64_t da, uint64_t db, bool first_kb) {
  constexpr u32 V = 32, PB = plane_b(32) >> 4, PA = kPlaneA >> 4;
  mma_u8n<0>(tb, da, db, idesc_n(256), first_kb ? 0u : 1u);
  if (first_kb) {
    mma_u8n<1>(tb + 7 * V, da + 7 * PA, db, idesc_n(32), 1u);
    mma_u8n<2>(tb + 8 * V, da + 7 * PA, db + PB, idesc_n(224), 0u);
  } else {
    mma_u8n<0>(tb + 7 * V, da + 7 * PA, db, idesc_n(256), 1u);
  }
#pragma unroll
  for (int sd = 1; sd < 7; ++sd) mma_u8n<0>(tb + (u32)sd * V, da + (uint64_t)(sd * PA), db, idesc_n(256), 1u);
}

// The 7-digit modes (2^31 <= p < 2^54: lazy values < 4p < 2^56) on the V = 32 geometry: L plane s
// (s < 7) against the 7 baby-step planes t < 7 is one MMA of N = 224 into slots s .. s + 6 (13
// slots, 416 columns); at K-block 0 plane 0 initialises slots 0..6 and plane 6, split, initialises
// slots 7..12 (its t = 0 part accumulates into slot 6).
__device__ __forceinline__ void issue_all32_7(u32 tb, uint64_t da, uint64_t db, bool first_kb) {
  constexpr u32 V = 32, PB = plane_b(32) >> 4, PA = kPlaneA >> 4;
  mma_u8n<0>(tb, da, db, idesc_n(224), first_kb ? 0u : 1u);
  if (first_kb) {
    mma_u8n<1>(tb + 6 * V, da + 6 * PA, db, idesc_n(32), 1u);
    mma_u8n<2>(tb + 7 * V, da + 6 * PA, db + PB, idesc_n(192), 0u);
  } else {
    mma_u8n<0>(tb + 6 * V, da + 6 * PA, db, idesc_n(224), 1u);
  }
#pragma unroll
  for (int sd = 1; sd < 6; ++sd) mma_u8n<0>(tb + (u32)sd * V, da + (uint64_t)(sd * PA), db, idesc_n(224), 1u);
}

// The 4-digit mode (p < 2^31): 16 digit pairs, diagonals 0..6 in one round, as 5 MMAs.  No L plane
// meets every diagonal, so at K-block 0 the two MMAs that overwrite cover disjoint slots
// (s = 0: slots 0..3; s = 3, t = 1..3: slots 4..6) and every later MMA accumulates.
__device__ __forceinline__ void issue_round4(u32 tb, uint64_t da, uint64_t db, bool first_kb) {
  const u32 ini = first_kb ? 0u : 1u;
  mma_u8n<0>(tb + 0 * kV, da + 0 * (kPlaneA >> 4), db + 0 * (kPlaneB >> 4), idesc_n(256), ini);
  mma_u8n<1>(tb + 4 * kV, da + 3 * (kPlaneA >> 4), db + 1 * (kPlaneB >> 4), idesc_n(192), ini);
  mma_u8n<2>(tb + 3 * kV, da + 3 * (kPlaneA >> 4), db + 0 * (kPlaneB >> 4), idesc_n(64), 1u);
  mma_u8n<0>(tb + 1 * kV, da + 1 * (kPlaneA >> 4), db + 0 * (kPlaneB >> 4), idesc_n(256), 1u);
  mma_u8n<0>(tb + 2 * kV, da + 2 * (kPlaneA >> 4), db + 0 * (kPlaneB >> 4), idesc_n(256), 1u);
}

// The 7-digit mode (p < 2^54: lazy values < 4p < 2^56): 49 pairs, rounds d = 0..7 (34 pairs, 12
// MMAs) and d = 8..12 (15 pairs, 6 MMAs).  Round 0 has no L plane meeting all 8 diagonals: the MMAs
// that overwrite at K-block 0 cover disjoint slots (s=0: 0..3 and 4..6, s=1 t=6: 7); in round 1,
// s = 6 meets all five and goes first.  Runs of one L plane keep A in the collector.
#define TC7(COL, S, T0, N, SLOT, ACC) \
  mma_u8n<COL>(tb + (SLOT) * kV, da + (S) * (kPlaneA >> 4), db + (T0) * (kPlaneB >> 4), idesc_n(N), ACC)
__device__ __forceinline__ void issue_round7_0(u32 tb, uint64_t da, uint64_t db, bool first_kb) {
  const u32 ini = first_kb ? 0u : 1u;
  TC7(1, 0, 0, 256, 0, ini); TC7(2, 0, 4, 192, 4, ini);
  TC7(1, 1, 6, 64, 7, ini);  TC7(3, 1, 0, 256, 1, 1u); TC7(2, 1, 4, 128, 5, 1u);
  TC7(1, 2, 0, 256, 2, 1u);  TC7(2, 2, 4, 128, 6, 1u);
  TC7(1, 3, 0, 256, 3, 1u);  TC7(2, 3, 4, 64, 7, 1u);
  TC7(0, 4, 0, 256, 4, 1u);  TC7(0, 5, 0, 192, 5, 1u);  TC7(0, 6, 0, 128, 6, 1u);
}
__device__ __forceinline__ void issue_round7_1(u32 tb, uint64_t da, uint64_t db, bool first_kb) {
  const u32 ini = first_kb ? 0u : 1u;
  TC7(1, 6, 2, 256, 0, ini); TC7(2, 6, 6, 64, 4, ini);
  TC7(0, 5, 3, 256, 0, 1u);  TC7(0, 4, 4, 192, 0, 1u);  TC7(0, 3, 5, 128, 0, 1u);  TC7(0, 2, 6, 64, 0, 1u);
}
#undef TC7

// digit pair (s, t = d - s) of diagonal slot di exists in round G
__host__ __device__ constexpr bool pair_ok(int G, int di, int sd) {
  return group_diag(G, di) >= 0 && group_diag(G, di) - sd >= 0 && group_diag(G, di) - sd <= 7;
}
__host__ __device__ constexpr int run_len(int G, int sd) {
  int n = 0;
  for (int di = 0; di < kDiag; ++di) n += pair_ok(G, di, sd) ? 1 : 0;
  return n;
}
// position of the k-th visited slot inside the run of plane sd (slots visited in the rotated
// order di = (sd + k) mod kDiag, which keeps consecutive MMAs on different accumulators)
__host__ __device__ constexpr int run_pos(int G, int sd, int k) {
  int n = 0;
  for (int j = 0; j < k; ++j) n += pair_ok(G, (sd + j) % kDiag, sd) ? 1 : 0;
  return n;
}

// The digit-pair MMAs of round G on one smem stage (da / db = descriptors of L plane 0 / R plane
// 0), grouped by L plane s so the A operand (L_s) is read from shared memory once per K-block and
// reused from the collector buffer.  Fully unrolled: every operand offset and collector mode is a
// compile-time constant.
template <int G, bool NOCOL = false>
__device__ __forceinline__ void issue_round(u32 tb, uint64_t da, uint64_t db, bool first_kb) {
#pragma unroll
  for (int sd = 0; sd < 8; ++sd) {
#pragma unroll
    for (int k = 0; k < kDiag; ++k) {
      const int di = (sd + k) % kDiag;
      if (pair_ok(G, di, sd)) {
        const int d = group_diag(G, di);
        const int n = run_len(G, sd), pos = run_pos(G, sd, k);
        const int s0 = d > 7 ? d - 7 : 0;
        const u32 acc = (!first_kb || sd > s0) ? 1u : 0u;   // first pair of diagonal d at kb 0 overwrites
        const u32 dt = tb + (u32)di * kV;
        const uint64_t ad = da + (uint64_t)((u32)sd * (kPlaneA >> 4));
        const uint64_t bd = db + (uint64_t)((u32)(d - sd) * (kPlaneB >> 4));
        if (n == 1 || NOCOL) mma_u8c<0>(dt, ad, bd, acc);
        else if (pos == 0) mma_u8c<1>(dt, ad, bd, acc);
        else if (pos == n - 1) mma_u8c<3>(dt, ad, bd, acc);
        else mma_u8c<2>(dt, ad, bd, acc);
      }
    }
  }
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, u32 cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(cnt));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, u32 parity) {
  u32 ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
// Bounded wait.  A wait that has not completed after kWaitTimeoutNs of %globaltimer (far beyond any
// legitimate stall: a whole config-5 launch takes ~9 ms) marks the CTA aborted and the handle's
// status word failed, and returns; once a CTA is aborted every wait returns at once, so all its
// warps run out of their loops (producing garbage, never hanging) and the host reports PE_ECUDA
// (pe.cu tc_failed) instead of a trapped context.  SLEEP_NS > 0 backs off between polls so a
// waiting warp stops taking issue slots from the producers on its SMSP.
constexpr unsigned long long kWaitTimeoutNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct Abort {
  volatile u32* cta;   // shared word: this CTA gave up
  u32* status;         // mapped host word
};
template <int SLEEP_NS = 0>
__device__ __forceinline__ void mbar_wait(uint64_t* bar, u32 parity, const Abort& ab, u32 sleep_ns = SLEEP_NS) {
  if (mbar_try(bar, parity) || *ab.cta) return;
  const unsigned long long t0 = gtimer();
  for (u32 n = 1;; ++n) {
    if (sleep_ns) __nanosleep(sleep_ns);
    if (mbar_try(bar, parity)) return;
    if ((n & 255) == 0) {
      if (*ab.cta) return;
      if (gtimer() - t0 > kWaitTimeoutNs) {
        *ab.cta = 1;
        if (ab.status) atomicExch(ab.status, 1u);
        return;
      }
    }
  }
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (complete_tx)
__device__ __forceinline__ void bulk_g2s(u32 dst, const void* src, u32 bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ u64 lds64(u32 addr) {
  u64 v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void lds2(u32 addr, u64& a, u64& b) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr) : "memory");
}
__device__ __forceinline__ void lds4(u32 addr, u64 (&v)[4]) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%4];\n\tld.shared.v2.u64 {%2, %3}, [%4+16];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "r"(addr) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld8(u32 taddr, u32 (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Redefine registers written by tcgen05.ld after tcgen05.wait::ld: later (non-volatile) uses then
// depend on this volatile statement and cannot be scheduled above the wait.
__device__ __forceinline__ void tmem_reg_fence(u32 (&v)[8]) {
  asm volatile("" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
               :: "memory");
}

__device__ __forceinline__ u32 prmt(u32 a, u32 b, u32 sel) {
  u32 r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Byte-transpose 4 values (terms tq*4 + e, e < 4) into 8 digit-plane words (word s = byte s of
// each value, value e in byte e = K position) and store them at row `row` of the stage.
__device__ __forceinline__ void sts32(u32 addr, u32 v) {
  asm volatile("st.shared.b32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
// values < 2^32 (4-digit mode): only the low 4 byte planes
template <u32 PS>
__device__ __forceinline__ void store_digits4(u32 planes, const u64 (&x)[4]) {
  const u32 l0 = lo32(x[0]), l1 = lo32(x[1]), l2 = lo32(x[2]), l3 = lo32(x[3]);
  const u32 a = prmt(l0, l1, 0x5140), b = prmt(l2, l3, 0x5140);
  const u32 c = prmt(l0, l1, 0x7362), d = prmt(l2, l3, 0x7362);
  sts32(planes + 0 * PS, prmt(a, b, 0x5410));
  sts32(planes + 1 * PS, prmt(a, b, 0x7632));
  sts32(planes + 2 * PS, prmt(c, d, 0x5410));
  sts32(planes + 3 * PS, prmt(c, d, 0x7632));
}
template <u32 PS>
__device__ __forceinline__ void store_digits(u32 planes, const u64 (&x)[4]) {
  const u32 l0 = lo32(x[0]), l1 = lo32(x[1]), l2 = lo32(x[2]), l3 = lo32(x[3]);
  const u32 h0 = hi32(x[0]), h1 = hi32(x[1]), h2 = hi32(x[2]), h3 = hi32(x[3]);
  u32 a = prmt(l0, l1, 0x5140), b = prmt(l2, l3, 0x5140);
  u32 c = prmt(l0, l1, 0x7362), d = prmt(l2, l3, 0x7362);
  sts32(planes + 0 * PS, prmt(a, b, 0x5410));
  sts32(planes + 1 * PS, prmt(a, b, 0x7632));
  sts32(planes + 2 * PS, prmt(c, d, 0x5410));
  sts32(planes + 3 * PS, prmt(c, d, 0x7632));
  a = prmt(h0, h1, 0x5140); b = prmt(h2, h3, 0x5140);
  c = prmt(h0, h1, 0x7362); d = prmt(h2, h3, 0x7362);
  sts32(planes + 4 * PS, prmt(a, b, 0x5410));
  sts32(planes + 5 * PS, prmt(a, b, 0x7632));
  sts32(planes + 6 * PS, prmt(c, d, 0x5410));
  sts32(planes + 7 * PS, prmt(c, d, 0x7632));
}

template <u32 LBO>
__device__ __forceinline__ u32 plane_off(u32 row, u32 kbyte) {
  return (kbyte >> 4) * LBO + (row >> 3) * 128u + (row & 7u) * 16u + (kbyte & 15u);
}

// X (5 x 32-bit words, little endian) += sum over the round's diagonals of D_d << 8d, exactly
// (X < 2^145 < 2^160 for the sum over all 15 diagonals: D < 2^31, 8d <= 112).  The low 128 bits
// are composed once per point; plain C 128-bit arithmetic lets the compiler own the carry chain
// (carry flags are not preserved between separate inline-asm statements).
typedef unsigned __int128 u128_t;
template <int D8>
__device__ __forceinline__ void fold_one(u128_t& lo, u32& x4, u32 Dv) {
  if (D8 < 0) return;
  constexpr int s = D8 < 0 ? 0 : D8;
  const u128_t add = (u128_t)Dv << s;                                 // low 128 bits of D << 8d
  const u32 spill = s > 96 ? (u32)(Dv >> (128 - s > 31 ? 31 : 128 - s)) : 0u;   // bits >= 2^128
  lo += add;
  x4 += spill + (lo < add ? 1u : 0u);
}
// single-diagonal form (unit tests: scripts/fold_test.cu)
template <int D8>
__device__ __forceinline__ void fold_add(u32 (&X)[5], u32 Dv) {
  u128_t lo = ((u128_t)(((u64)X[3] << 32) | X[2]) << 64) | (((u64)X[1] << 32) | X[0]);
  u32 x4 = X[4];
  fold_one<D8>(lo, x4, Dv);
  X[0] = (u32)lo;
  X[1] = (u32)(lo >> 32);
  X[2] = (u32)(lo >> 64);
  X[3] = (u32)(lo >> 96);
  X[4] = x4;
}

// Epilogue critical part: drain round G's diagonals of thread row u from TMEM into the unit's raw
// buffer (raw[slot][v/4][u][v%4], u32: the diagonal sums themselves) and release TMEM (acce) as soon as the
// last block is in registers -- only tcgen05.ld and fire-and-forget stores, so the MMA warp can
// start the next round almost at once.  Four accumulators (32 registers) per tcgen05.wait.
template <int G, int H, int V = kV>
__device__ __forceinline__ void drain_ld(u32 tl, u32 v0, u32 (&D)[4][8]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (group_diag(G, 4 * H + j) >= 0) tmem_ld8(tl + (u32)(4 * H + j) * V + v0, D[j]);
}
template <int G, int H>
__device__ __forceinline__ void drain_fence(u32 (&D)[4][8]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (group_diag(G, 4 * H + j) >= 0) tmem_reg_fence(D[j]);
}
template <int G, int H, int V = kV>
__device__ __forceinline__ void drain_st(u32 v0, u32* __restrict__ raw_u, const u32 (&D)[4][8]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (group_diag(G, 4 * H + j) >= 0) {
      // raw[d][v / 4][u][v % 4]: a warp's 16-byte stores cover 512 contiguous bytes
      uint4* p4 = (uint4*)(raw_u + (u32)(4 * H + j) * (kU * (u32)V) + (v0 >> 2) * (kU * 4));
      p4[0] = make_uint4(D[j][0], D[j][1], D[j][2], D[j][3]);
      p4[kU] = make_uint4(D[j][4], D[j][5], D[j][6], D[j][7]);
    }
  }
}
// Software-pipelined: the tcgen05.ld of the next 4 accumulators x 8 columns is in flight while
// the previous block is stored; TMEM is released (acce) right after the last load completes.
template <int G>
__device__ __forceinline__ void epi_drain(u32 tl, u32* __restrict__ raw_u, uint64_t* acce, bool st = true) {
  u32 A[4][8], B[4][8];
  drain_ld<G, 0>(tl, 0, A);
  tmem_wait_ld();
  drain_fence<G, 0>(A);
#pragma unroll 1
  for (u32 v0 = 0; v0 < (u32)kV; v0 += 8) {
    drain_ld<G, 1>(tl, v0, B);
    if (st) drain_st<G, 0>(v0, raw_u, A);
    tmem_wait_ld();
    drain_fence<G, 1>(B);
    if (v0 + 8 < (u32)kV) {
      drain_ld<G, 0>(tl, v0 + 8, A);
    } else {   // TMEM drained: the MMA may start the next round
      tc_fence_before();
      mbar_arrive(acce);
    }
    if (st) drain_st<G, 1>(v0, raw_u, B);
    if (v0 + 8 < (u32)kV) {
      tmem_wait_ld();
      drain_fence<G, 0>(A);
    }
  }
}

// The single-round geometry (G = 5, V = 32): 15 diagonals x 32 columns as 16 blocks of 4 diagonals
// x 8 columns (block b: v0 = 8 (b / 4), diagonals 4 (b % 4) ..), each block's tcgen05.ld in flight
// while the previous block is stored.
template <int G, int H>
__device__ __forceinline__ void drain5_ld(u32 tl, int b, u32 (&D)[4][8]) { drain_ld<G, H, 32>(tl, (u32)(b / 4) * 8, D); }
template <int G>
__device__ __forceinline__ void epi_drain5(u32 tl, u32* __restrict__ raw_u, uint64_t* acce, bool st = true) {
  u32 A[4][8], B[4][8];
  drain5_ld<G, 0>(tl, 0, A);
  tmem_wait_ld();
  drain_fence<G, 0>(A);
#pragma unroll
  for (int b = 0; b < 16; b += 2) {   // A holds block b (H = 0 or 2), B gets block b + 1 (H = 1 or 3)
    const u32 v0 = (u32)(b / 4) * 8;
    const bool lo = (b % 4) == 0;
    if (lo) drain5_ld<G, 1>(tl, b + 1, B); else drain5_ld<G, 3>(tl, b + 1, B);
    if (st) { if (lo) drain_st<G, 0, 32>(v0, raw_u, A); else drain_st<G, 2, 32>(v0, raw_u, A); }
    tmem_wait_ld();
    if (lo) drain_fence<G, 1>(B); else drain_fence<G, 3>(B);
    if (b + 2 < 16) {
      if (lo) drain5_ld<G, 2>(tl, b + 2, A); else drain5_ld<G, 0>(tl, b + 2, A);
    } else {   // TMEM drained: the MMA may start the next unit
      tc_fence_before();
      mbar_arrive(acce);
    }
    if (st) { if (lo) drain_st<G, 1, 32>(v0, raw_u, B); else drain_st<G, 3, 32>(v0, raw_u, B); }
    if (b + 2 < 16) {
      tmem_wait_ld();
      if (lo) drain_fence<G, 2>(A); else drain_fence<G, 0>(A);
    }
  }
}

// X (160-bit, 5 x u32) = sum_{d<15} D_d 2^{8d}, exactly (< 2^145): composed in 128-bit C
// arithmetic (the compiler owns the carries) + a top word.
template <int D8>
__device__ __forceinline__ void fold_in(u128_t& lo, u32& x4, u32 Dv) {
  const u128_t add = (u128_t)Dv << D8;
  const u32 spill = D8 > 96 ? (u32)(Dv >> (128 - D8 > 31 ? 31 : 128 - D8)) : 0u;
  lo += add;
  x4 += spill + (lo < add ? 1u : 0u);
}

// X_G += sum over round G's accumulator slots DI.. of D[slot] << 8 d(slot)  (compile-time shifts)
template <int G, int DI, int NS>
__device__ __forceinline__ void fold_group(u128_t& acc, u32& x4, const u32 (&D)[NS][4], int j) {
  if constexpr (DI < NS) {
    if constexpr (group_diag(G, DI) >= 0) fold_in<8 * group_diag(G, DI)>(acc, x4, D[DI][j]);
    fold_group<G, DI + 1, NS>(acc, x4, D, j);
  }
}

// One TMEM row (giant step ur) of a unit: fold round G's diagonals of each of the kV points into
// X_G (< 2^145), reduce the 2^64..2^128 words with 2^{32k} mod p into 128 bits, and finish with
// one REDC into the unit's partial row.
// discard.global.L2: drop a 128-byte L2 line without writing it back (a weak write of an undefined
// value, ordered by the same release/acquire as a store).  The drained diagonal sums are dead once
// folded; without this the dirty scratch lines are evicted to DRAM by the streaming baby-step
// planes before the ping-pong rewrites them (round 1: ~1.8 GB of the 8.5 GB per config-5 launch).
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" :: "l"(p) : "memory");
}

template <int G, int V = kV>
__device__ __forceinline__ void fold_row(const u32* __restrict__ rr_, u64* __restrict__ prow, u64 kbase, u32 npts,
                                         u64 C64, u64 C96, u64 C128, const ModParams& mp, u32 vbeg, u32 vend,
                                         bool disc) {
  const bool line_head = (threadIdx.x & 7) == 0;   // 8 consecutive rows x 16 B = one 128-B line
#pragma unroll 1
  for (u32 v0 = vbeg; v0 < vend; v0 += 4) {
    constexpr int NS = nslots(G);
    u32 D[NS][4];
#pragma unroll
    for (int di = 0; di < NS; ++di) {
      if (group_diag(G, di) >= 0) {
        const uint4 q = *(const uint4*)(rr_ + (u32)di * (kU * (u32)V) + (v0 >> 2) * (kU * 4));
        D[di][0] = q.x; D[di][1] = q.y; D[di][2] = q.z; D[di][3] = q.w;
      }
    }
    u64 res[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      u128_t acc = 0;
      u32 x4 = 0;
      fold_group<G, 0, NS>(acc, x4, D, j);
      // X mod p = (x0 + x1 2^32) + x2 (2^64 mod p) + x3 (2^96 mod p) + x4 (2^128 mod p)  (< 2^98)
      u64 lo = (u64)acc, hi = 0;
      const u64 x2 = (u64)(acc >> 64) & 0xffffffffull, x3 = (u64)(acc >> 96);
      const u64 terms[3][2] = {{x2, C64}, {x3, C96}, {(u64)x4, C128}};
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const u64 p0 = terms[q][0] * lo32(terms[q][1]);
        const u64 p1 = terms[q][0] * hi32(terms[q][1]);
        const u64 add_lo = p0 + (p1 << 32);
        const u64 add_hi = (p1 >> 32) + (add_lo < p0 ? 1ull : 0ull);
        lo += add_lo;
        hi += add_hi + (lo < add_lo ? 1ull : 0ull);
      }
      // the baby-step planes hold Montgomery residues m^v 2^64 (k_tc_rplanes), so the sum is
      // 2^64 X: one REDC (x 2^-64) is the reduction; REDC needs its high word < p
      res[j] = redc(hi < mp.p ? hi : hi % mp.p, lo, mp);
    }
    if (disc) {
      // every lane's loads of this v0 group were consumed above; once the warp has converged, the
      // warp's 4 lines per diagonal (its 32 rows x 16 B) are dead
      __syncwarp();
      if (line_head) {
#pragma unroll
        for (int di = 0; di < NS; ++di)
          if (group_diag(G, di) >= 0) discard_l2(rr_ + (u32)di * (kU * (u32)V) + (v0 >> 2) * (kU * 4));
      }
    }
    if (kbase + v0 + 4 <= npts) {
      ulonglong2* dst = (ulonglong2*)(prow + kbase + v0);
      dst[0] = make_ulonglong2(res[0], res[1]);
      dst[1] = make_ulonglong2(res[2], res[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (kbase + v0 + j < npts) prow[kbase + v0 + j] = res[j];
    }
  }
}

__device__ __forceinline__ long long clk() { return clock64(); }

// unit -> (piece, chunk, diagonal round g), piece-major over the size-sorted pieces: the
// kRounds x nch units of one piece run at the same time on neighbouring CTAs, so all but the
// first reader of a K-block's baby-step planes and C records find them in L2.  X mod p is the
// sum of the rounds' parts (X = sum_g X_g), so each unit reduces its own part into its own
// partial row (slot = piece slot * rounds + g) and k_fixup adds them.
// The i-th unit of this CTA, from the host's schedule (pe.cu tc_schedule: longest-processing-time
// dealing of the size-sorted units over the CTAs, so a launch with few units per CTA -- a shard of
// a multi-GPU run -- stays balanced); past the CTA's list it returns 0xffffffff (>= nunits).
__device__ __forceinline__ u32 unit_id(const TcArgs& a, u32 i) {
  const u32 o = a.sched_off[blockIdx.x] + i;
  return o < a.sched_off[blockIdx.x + 1] ? a.sched[o] : 0xffffffffu;
}
__device__ __forceinline__ void unit_of(const TcArgs& a, u32 unit, uint4& pc, u32& chunk, u32& g) {
  g = unit % a.rounds;
  const u32 r = unit / a.rounds;
  chunk = r % a.nch;
  pc = a.piece[r / a.nch];
}

// PROF: per-warp phase timers (clock64) into a.prof -- a development build of the same kernel
// (PE_TC_PROF=1); the production instantiation has no timers.
// Walks one CTA's K-block sequence: units unit_id(0), unit_id(1), ...; per unit the piece's K-blocks.
struct KIter {
  u32 ord, unit, kb, nkb, q0, chunk;
  bool valid;
  __device__ __forceinline__ void load(const TcArgs& a) {
    unit = unit_id(a, ord);
    valid = unit < a.nunits;
    if (valid) {
      uint4 pc;
      u32 g;
      unit_of(a, unit, pc, chunk, g);
      nkb = pc.y;
      q0 = pc.x;
    }
  }
  __device__ __forceinline__ void init(const TcArgs& a) { ord = 0; kb = 0; load(a); }
  // n K-blocks ahead (a producer group's next K-block is kStages ahead): one add and compare
  // unless a unit boundary is crossed
  __device__ __forceinline__ void advance(const TcArgs& a, u32 n) {
    kb += n;
    while (valid && kb >= nkb) {
      kb -= nkb;
      ++ord;
      load(a);
    }
  }
};

// The two TMA bulk copies of one K-block's per-term records into a data slot.
__device__ __forceinline__ void load_kblock(const TcArgs& a, const KIter& k, u32 dst, uint64_t* bar) {
  const u64 q = (u64)k.q0 + (u64)k.kb * kKB;
  mbar_expect_tx(bar, kDataSlot);
  bulk_g2s(dst, a.LS + ((u64)k.chunk * a.t_pad + q) * kLSRec, kDataLS, bar);
  bulk_g2s(dst + kDataLS, a.C + q * kCRec, kDataSlot - kDataLS, bar);
}

// MODE 0: p < 2^62, lazy Shoup chains (values < 4p < 2^64), 8 byte digits, 2 rounds.
// MODE 1: 2^62 <= p < 2^63, exact-quotient chains (values < 2p < 2^64), 8 digits, 2 rounds.
// MODE 2: p < 2^31, exact-quotient chains (values < 2p < 2^32), 4 digits, 1 round of 5 MMAs.
// MODE 3: 2^31 <= p < 2^54, lazy chains (values < 4p < 2^56), 7 digits, one round of 7 MMAs (V = 32).
// MODE 4 / 5 / 6: the swapped forms of modes 0 / 1 / 3 (giant-step planes per handle, baby steps generated).
template <bool PROF, int MODE>
static __global__ void __launch_bounds__(kThreads, 1) k_tc(TcArgs a) {   // 12 warps: <= 168 regs/thread
  constexpr bool SEVEN = MODE == 3 || MODE == 6;   // 7-digit modes (plain / swapped)
  unsigned long long g_entry = 0;
  if (PROF) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
  extern __shared__ uint8_t dsm[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)dsm + 127) & ~(uintptr_t)127);   // kSmemBytes holds 128 B of slack
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], accf, acce, dfull[kDataSlots];
  __shared__ u32 tmem_base;
  __shared__ u32 abort_flag;
  const Abort ab{&abort_flag, a.status};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    // full: the group's threads + the leader's expect_tx arrival for the R planes
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 32 * kProdPerStage + 1); mbar_init(&empty[s], 1); }
    mbar_init(&accf, 1);
    mbar_init(&acce, 32 * kEpiWarps);
    for (int s = 0; s < kDataSlots; ++s) mbar_init(&dfull[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    abort_flag = 0;
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const u32 tb = tmem_base;
  unsigned long long g_alloc = 0;
  if (PROF) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_alloc));
  long long T[4] = {0, 0, 0, 0};   // phase timers (a.prof)
  const long long t_start = clk();
  const u32 data0 = smem_u32(smem) + kStages * kStageBytes;

  if (warp >= kProdWarp0) {
    // ------------------------------------------------------------ producers
    // 2 warps per stage generate the 128 giant-step rows of 16 terms each: lane = (tq < 4,
    // rr < 8), terms sub*16 + tq*4 .. +3, rows rr + 8k (k < 16) -- 4 Shoup chains of stride 8 per
    // lane; one store instruction covers 8 rows x 16 bytes = all 32 banks.  The group's first
    // lane brings in, with TMA, the K-block's baby-step planes (straight into the stage, counted
    // on its full barrier) and the group's NEXT K-block's per-term records (two data slots).
    const int pw = warp - kProdWarp0;
    const int my_stage = pw / kProdPerStage, sub = pw % kProdPerStage;
    const bool leader = sub == 0 && lane == 0;            // issues the baby-step plane copies
    const bool loader = sub == 1 && lane == 0;            // issues the per-term record prefetches
    const u32 tq = (u32)(lane >> 3), rr = (u32)(lane & 7);
    const u32 term0 = (u32)sub * 16 + tq * 4;     // first of the lane's 4 terms
    const u32 stage0 = smem_u32(smem) + (u32)my_stage * kStageBytes;
    constexpr bool SW = MODE >= 4;                        // swapped form: generate R' into the B half
    const u32 planes0 = SW ? stage0 + 8 * kPlaneA + plane_off<lbo_b(mode_v(MODE))>(rr, term0) : stage0 + plane_off<kLBOA>(rr, term0);
    const u32 seed_off = term0 * kLSRec * 8;
    const u32 mul_off = kDataLS + (term0 * kCRec + kC_mL) * 8;
    const u32 g_off = kDataLS + (term0 * kCRec + kC_g0 + rr) * 8;
    const ModParams mp = a.mp;
    const u32 slot0 = (u32)my_stage * 2;
    const u64 np = a.mp.np;
    // the group owns K-blocks my_stage, my_stage + kStages, ... of the CTA's sequence
    KIter cur, ahead;
    cur.init(a);
    cur.advance(a, (u32)my_stage);                                   // the group's first K-block
    ahead = cur;
    ahead.advance(a, kStages);                                       // ... and its second
    if (loader && cur.valid) load_kblock(a, cur, data0 + slot0 * kDataSlot, &dfull[slot0]);
    u32 guse = 0;
    // the lane's chain seeds and multipliers of the group's K-block number g (data slot g & 1)
    u64 x[4], sm[4], sw[4];
    auto fetch = [&](u32 g) {
      const u32 dslot = data0 + (slot0 + (g & 1)) * kDataSlot;
      const long long f0 = clk();
      mbar_wait<64>(&dfull[slot0 + (g & 1)], (g >> 1) & 1, ab);
      if (PROF) T[0] += clk() - f0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // chain seed of row rr: c m^{j_s} (normal) x Montgomery m^{rr V} -> c m^{j_s + rr V}
        x[e] = mont_mul(lds64(dslot + seed_off + (u32)e * kLSRec * 8), lds64(dslot + g_off + (u32)e * kCRec * 8), mp);
        lds2(dslot + mul_off + (u32)e * kCRec * 8, sm[e], sw[e]);
      }
    };
    if (cur.valid) fetch(0);
    for (; cur.valid; cur = ahead, ahead.advance(a, kStages)) {
      const u32 stage = (u32)my_stage;
      const u32 use = guse;
      long long c0 = clk();
      mbar_wait<64>(&empty[stage], (use & 1) ^ 1, ab, a.sleep_ns[1]);
      long long c1 = clk();
      if (PROF) T[1] += c1 - c0;
      // the other slot held K-block guse-1, which every warp of the group read (at the end of
      // K-block guse-2) before arriving on that stage fill: refill it with the group's next K-block
      if (leader) {
        if (PROF && (a.dbg == 4 || a.dbg == 6 || a.dbg == 7)) {
          mbar_arrive(&full[stage]);
        } else if (SW) {
          mbar_expect_tx(&full[stage], kGBytes);
          bulk_g2s(stage0, a.Gp + ((u64)cur.q0 / kKB + cur.kb) * kGBytes, kGBytes, &full[stage]);
        } else {
          constexpr u32 RB = r_bytes(mode_v(MODE));
          mbar_expect_tx(&full[stage], RB);
          bulk_g2s(stage0 + 8 * kPlaneA, a.Rp + ((u64)cur.q0 / kKB + cur.kb) * RB, RB, &full[stage]);
        }
      }
      if (loader && ahead.valid)
        load_kblock(a, ahead, data0 + (slot0 + ((guse + 1) & 1)) * kDataSlot, &dfull[slot0 + ((guse + 1) & 1)]);
      if (SW && !(PROF && (a.dbg == 2 || a.dbg >= 6))) {
        // baby-step rows rr + 8k (k < V / 8) of R' = c m^{j_s + v}
        constexpr int VV8 = mode_v(MODE) / 8;
        constexpr u32 PB = plane_b(mode_v(MODE));
#pragma unroll
        for (int k = 0; k < VV8 - 1; ++k) {
          store_digits<PB>(planes0 + (u32)k * 128u, x);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            x[e] = MODE == 5 ? mul_shoup2(x[e], sm[e], sw[e], np) : mul_shoup4(x[e], sm[e], sw[e], np);
        }
        store_digits<PB>(planes0 + (u32)(VV8 - 1) * 128u, x);
      } else if (!(PROF && (a.dbg == 2 || a.dbg >= 6))) {
#pragma unroll 3
        for (int k = 0; k < 15; ++k) {
          // row rr + 8k: the next 8-row core-matrix group, +128 bytes
          if (MODE == 2) store_digits4<kPlaneA>(planes0 + (u32)k * 128u, x);
          else store_digits<kPlaneA>(planes0 + (u32)k * 128u, x);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // p < 2^31: 32-bit Shoup (3 IMADs instead of the 64-bit form's ~10); its constant
            // floor(m 2^32 / p) is the high word of the record's floor(m 2^64 / p), and values stay
            // < 2p < 2^32 (4 digits)
            if (MODE == 2) x[e] = mul_shoup32((u32)x[e], (u32)sm[e], (u32)(sw[e] >> 32), (u32)mp.p);
            else x[e] = MODE == 1 ? mul_shoup2(x[e], sm[e], sw[e], np) : mul_shoup4(x[e], sm[e], sw[e], np);
          }
        }
        if (MODE == 2) store_digits4<kPlaneA>(planes0 + 15u * 128u, x);   // last row: no product after it
        else store_digits<kPlaneA>(planes0 + 15u * 128u, x);
      }
      fence_async_smem();
      mbar_arrive(&full[stage]);
      if (PROF) T[2] += clk() - c1;
      if (PROF) T[3] += 1;
      ++guse;
      // next K-block's seeds while this stage is being consumed (its data arrived during this
      // K-block); the product latency hides in the wait for the stage
      if (ahead.valid) fetch(guse);
    }
  } else {
    // ------------------------------------------------------------ epilogue (+ MMA issue in warp 0)
    // MMA issue and TMEM drain alternate (TMEM holds one round), so warp 0 issues a round's MMAs
    // (converged warp, elect.sync leader) and then drains its lane quarter.  Per round every
    // epilogue warp only moves its rows of the round's diagonals from TMEM to the unit's raw buffer (ping-pong by
    // unit) and releases TMEM.  After the unit's last round warps 1-3 fold all 15 diagonals
    // exactly (X = sum D_d 2^{8d}) and reduce mod p into the piece's partial row -- warps 2 and 3 also
    // for warp 0's rows -- while warp 0 is already issuing the next unit's MMAs.
    const u32 u = (u32)(warp * 32 + lane);
    const u32 tl = tb + ((u32)(warp * 32) << 16);
    const ModParams mp = a.mp;
    u32* raw_cta = a.scratch + (u64)blockIdx.x * 2 * kDiag * (kU * kV);
    const u64 C64 = a.Wd[8], C96 = a.Wd[12], C128 = a.C128;
    const u32 tbu = uni(tb);
    const uint64_t dA0 = smem_desc(uni(smem_u32(smem)), kLBOA);
    constexpr int VV = mode_v(MODE);   // baby steps per chunk (32: single-round geometry)
    const uint64_t dB0 = smem_desc(uni(smem_u32(smem)) + 8 * kPlaneA, lbo_b(VV));
    u32 it = 0;
    for (u32 nunit = 0, unit = unit_id(a, 0); unit < a.nunits; unit = unit_id(a, ++nunit)) {
      uint4 pc; u32 chunk, g;
      unit_of(a, unit, pc, chunk, g);
      const u32 nkb = uni(pc.y);
      g = uni(g);
      u64* prow = a.partial + ((u64)pc.z * a.rounds + g) * a.ldp;
      if (a.direct && pc.w) prow = a.out + (u64)(pc.w - 1) * a.ldo;   // sole piece: the final row
      if (MODE == 2) g = 2;   // the 4-digit mode's single round
      if (VV == 32) g = SEVEN ? 6 : 5;   // the V = 32 geometry's single round (7 / 8 digits)
      u32* raw = raw_cta + (u64)(nunit & 1) * kDiag * (kU * kV);
      if (warp == kMmaWarp) {
        // (this raw buffer was last read two units ago by warps 2 / 3's fold of warp 0's rows;
        // that fold precedes their drain of the previous unit, which this warp has waited for
        // through acce -- no extra barrier needed)
        long long c0 = clk();
        mbar_wait<32>(&acce, (nunit & 1) ^ 1, ab);
        if (PROF) T[2] += clk() - c0;
        tc_fence_after();
        for (u32 kb = 0; kb < nkb; ++kb, ++it) {
          const u32 stage = it % kStages, use = it / kStages;
          c0 = clk();
          mbar_wait<32>(&full[stage], use & 1, ab, a.sleep_ns[0]);
          if (PROF) T[kb < (u32)kStages ? 0 : 1] += clk() - c0;   // unit start vs steady state
          tc_fence_after();
          const uint64_t da = dA0 + (uint64_t)((stage * kStageBytes) >> 4);
          const uint64_t db = dB0 + (uint64_t)((stage * kStageBytes) >> 4);
          // converge first so elect.sync picks the same leader (lane 0) every time: a
          // tcgen05.commit tracks the MMAs its own thread issued
          __syncwarp();
          if (elect_one()) {
            if (VV == 32) {
              if (PROF && a.dbg == 1) {
              } else if (SEVEN) issue_all32_7(tbu, da, db, kb == 0);
              else issue_all32(tbu, da, db, kb == 0);
            } else if (PROF && a.dbg == 7) {   // one N = 64 MMA per digit pair (the previous issue form)
              if (g == 0) issue_round<0, true>(tbu, da, db, kb == 0);
              else issue_round<1, true>(tbu, da, db, kb == 0);
            } else if (!(PROF && a.dbg == 1)) {
              if (MODE == 2) issue_round4(tbu, da, db, kb == 0);
              else if (MODE == 3) {
                if (g == 0) issue_round7_0(tbu, da, db, kb == 0);
                else issue_round7_1(tbu, da, db, kb == 0);
              } else if (g == 0) issue_round_wide<0>(tbu, da, db, kb == 0);
              else issue_round_wide<1>(tbu, da, db, kb == 0);
            }
            if (kb + 1 == nkb) mma_commit(&accf);   // accumulators complete after this K-block
            mma_commit(&empty[stage]);
          }
          __syncwarp();
        }
      }
      long long c0 = clk();
      mbar_wait<64>(&accf, nunit & 1, ab, a.sleep_ns[2]);
      long long c1 = clk();
      if (PROF) T[0] += c1 - c0;
      tc_fence_after();
      u32* raw_u = raw + (u64)u * 4;
      const bool st = !(PROF && a.dbg == 3);
      if (VV == 32 && SEVEN) epi_drain5<6>(tl, raw_u, &acce, st);
      else if (VV == 32) epi_drain5<5>(tl, raw_u, &acce, st);
      else if (MODE == 2) epi_drain<2>(tl, raw_u, &acce, st);
      else if (MODE == 3 && g == 1) epi_drain<4>(tl, raw_u, &acce, st);
      else if (g == 0) epi_drain<0>(tl, raw_u, &acce, st);
      else epi_drain<1>(tl, raw_u, &acce, st);
      if (PROF && warp != kMmaWarp) T[1] += clk() - c1;
      if (PROF) T[3] += 1;
      // warps 1-3 fold the unit while warp 0 issues the next one's MMAs; warp 0's rows are
      // split by v between warps 2 and 3 (1.5 row-sets each on SMSPs 2 / 3, 1 on SMSP 1: the fold
      // shares those SMSPs with producer warps)
      long long c2 = clk();
      for (int pass = 0; pass < (warp == kMmaWarp ? 0 : (warp == 1 ? 1 : 2)); ++pass) {
        u32 ur = u, vbeg = 0, vend = (u32)VV;
        if (pass == 1) {                 // warp 0's rows, once all 4 warps drained the unit
          mbar_wait<32>(&acce, nunit & 1, ab);
          ur = (u32)lane;
          vbeg = warp == 2 ? 0u : (u32)VV / 2;
          vend = vbeg + (u32)VV / 2;
        }
        const u32* rr_ = raw + (u64)ur * 4;
        const u64 kbase = (u64)chunk * chunk_pts(VV) + (u64)ur * VV;   // multiple of 8; ldp multiple of 8
        if (VV == 32 && SEVEN) fold_row<6, 32>(rr_, prow, kbase, a.npts, C64, C96, C128, mp, vbeg, vend, a.discard);
        else if (VV == 32) fold_row<5, 32>(rr_, prow, kbase, a.npts, C64, C96, C128, mp, vbeg, vend, a.discard);
        else if (MODE == 2) fold_row<2>(rr_, prow, kbase, a.npts, C64, C96, C128, mp, vbeg, vend, a.discard);
        else if (MODE == 3 && g == 1) fold_row<4>(rr_, prow, kbase, a.npts, C64, C96, C128, mp, vbeg, vend, a.discard);
        else if (g == 0) fold_row<0>(rr_, prow, kbase, a.npts, C64, C96, C128, mp, vbeg, vend, a.discard);
        else fold_row<1>(rr_, prow, kbase, a.npts, C64, C96, C128, mp, vbeg, vend, a.discard);
      }
      if (PROF) T[2] += clk() - c2;
    }
  }
  if (PROF && a.prof && lane == 0) {
    unsigned long long* o = a.prof + ((u64)blockIdx.x * (kThreads / 32) + warp) * 5;
    for (int i = 0; i < 4; ++i) o[i] = (unsigned long long)T[i];
    o[4] = (unsigned long long)(clk() - t_start);
    if (warp == 0) {   // wall-clock stamps (ns): entry, after TMEM alloc, exit of this CTA
      unsigned long long g_exit;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
      unsigned long long* gt = a.prof + (u64)gridDim.x * (kThreads / 32) * 5 + (u64)blockIdx.x * 3;
      gt[0] = g_entry; gt[1] = g_alloc; gt[2] = g_exit;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tb));
  }
}

// ---------------------------------------------------------------- setup kernels
// Per padded term (pe_create): the C record -- the giant-step chain multiplier m^{8V} (stride 8
// rows of L), its Shoup constant and the Montgomery table m^{rr V} (rr < 8) -- and, for the
// per-pass chunk seeds, Montgomery m^V and m^{kChunk}.
// (The swapped form's records -- chain multiplier m^8, table m^{rr} -- are written by k_tc_gplanes.)
template <int V>
static __global__ void k_tc_setup(const u64* __restrict__ m, u64 t_pad, u64* __restrict__ C, u64* __restrict__ MS,
                                  ModParams mp) {
  for (u64 q = blockIdx.x * (u64)blockDim.x + threadIdx.x; q < t_pad; q += (u64)gridDim.x * blockDim.x) {
    const u64 mm = to_mont(m[q], mp);
    const u64 mV = mont_pow(mm, V, mp);
    u64 g = mp.r1;                                     // Montgomery m^{rr V}
    for (int rr = 0; rr < 8; ++rr) {
      C[q * kCRec + kC_g0 + rr] = g;
      g = mont_mul(g, mV, mp);
    }
    const u64 aL = from_mont(g, mp);                   // m^{8V}
    C[q * kCRec + kC_mL] = aL;
    C[q * kCRec + kC_wL] = shoup_w_fast(aL, mp);
    MS[2 * q] = mV;
    MS[2 * q + 1] = mont_pow(mV, kU, mp);              // m^{kChunk}
  }
}

// Per handle (pe_create): the baby-step byte planes R_t[i][v] = byte t of the Montgomery residue
// m_i^v 2^64 mod p (v < V) in the stage layout of each K-block (any representative < 2^64 gives
// exact byte products; the epilogue's REDC removes the 2^64).  Warp task = (K-block, K half):
// lane = (ql: 4 terms, r: rows r + 8j, j < 8); a warp's store of one plane word covers 8 rows x 16
// bytes = one 128-byte line, so the planes go straight to global memory.  m, m^2, m^3, m^4 and the
// normal m^8 with its Shoup constant are computed once per term (lane r < 4 of the term's group) and
// shuffled to the group's 8 lanes, so each lane's row start m^r costs at most one product.
// The stride-8 chain of a lane (rows r, r + 8, ...) multiplies by the fixed m^8 with Shoup products
// (its constant is m8_mont * (-p^-1) mod 2^64, modcore.cuh shoup_w_fast): any representative below
// 2^digits is exact for the MMAs, so LAZY chains (values < 4p) serve 2^31 <= p < 2^62 (8 digits, or 7
// when p < 2^54: 4p < 2^56) and exact-quotient ones (< 2p) the 4-digit (p < 2^31) and p >= 2^62 modes.
constexpr int kRpThreads = 256;
template <bool LAZY, int V>
static __global__ void __launch_bounds__(kRpThreads) k_tc_rplanes(const u64* __restrict__ m, u64 t_pad,
                                                                  uint8_t* __restrict__ Rp, ModParams mp) {
  const u64 nkb = 2 * ((t_pad + 2 * kKB - 1) / (2 * kKB));   // Rp is allocated for whole pairs of K-blocks
  const u64 ntask = 2 * nkb;
  const int lane = threadIdx.x & 31;
  const u32 ql = (u32)(lane >> 3), r = (u32)(lane & 7);
  const u64 nwarp = (u64)gridDim.x * (kRpThreads / 32);
  for (u64 task = (u64)blockIdx.x * (kRpThreads / 32) + (threadIdx.x >> 5); task < ntask; task += nwarp) {
    const u64 blk = task >> 1;
    const u32 h = (u32)(task & 1);
    const u64 q0 = blk * kKB + (u64)h * 16 + ql * 4;
    const u64 q = q0 + (r & 3);
    const u64 mm = to_mont(q < t_pad ? m[q] : 0ull, mp);
    const u64 m2 = mont_mul(mm, mm, mp), m4 = mont_mul(m2, m2, mp);
    const u64 m8m = mont_mul(m4, m4, mp);                // Montgomery m^8 = m^8 2^64 mod p
    const u64 m3 = mont_mul(m2, mm, mp);
    const u64 n8 = from_mont(m8m, mp), s8 = m8m * mp.pinv;   // normal m^8 and its Shoup constant
    u64 y[4], m8[4], w8[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int src = (int)(ql * 8) + e;
      const u64 v1 = __shfl_sync(0xffffffffu, mm, src), v2 = __shfl_sync(0xffffffffu, m2, src);
      const u64 v3 = __shfl_sync(0xffffffffu, m3, src), v4 = __shfl_sync(0xffffffffu, m4, src);
      m8[e] = __shfl_sync(0xffffffffu, n8, src);         // normal m^8: the chain's fixed multiplier
      w8[e] = __shfl_sync(0xffffffffu, s8, src);         // its Shoup constant floor(m^8 2^64 / p)
      const u32 r2 = r & 3;                              // one product at most: m^{r&3} [x m^4]
      u64 x = r2 == 0 ? mp.r1 : r2 == 1 ? v1 : r2 == 2 ? v2 : v3;
      if (r & 4) x = mont_mul(x, v4, mp);
      y[e] = x;                                          // m^r (Montgomery residue, canonical)
    }
    uint8_t* dst = Rp + blk * r_bytes(V) + h * lbo_b(V) + r * 16u + ql * 4u;
#pragma unroll 1
    for (u32 j = 0; j < (u32)V / 8; ++j) {               // row r + 8j
      const u32 l0 = lo32(y[0]), l1 = lo32(y[1]), l2 = lo32(y[2]), l3 = lo32(y[3]);
      const u32 h0 = hi32(y[0]), h1 = hi32(y[1]), h2 = hi32(y[2]), h3 = hi32(y[3]);
      u32 wd[8];
      u32 a = prmt(l0, l1, 0x5140), b = prmt(l2, l3, 0x5140), c = prmt(l0, l1, 0x7362), d = prmt(l2, l3, 0x7362);
      wd[0] = prmt(a, b, 0x5410); wd[1] = prmt(a, b, 0x7632); wd[2] = prmt(c, d, 0x5410); wd[3] = prmt(c, d, 0x7632);
      a = prmt(h0, h1, 0x5140); b = prmt(h2, h3, 0x5140); c = prmt(h0, h1, 0x7362); d = prmt(h2, h3, 0x7362);
      wd[4] = prmt(a, b, 0x5410); wd[5] = prmt(a, b, 0x7632); wd[6] = prmt(c, d, 0x5410); wd[7] = prmt(c, d, 0x7632);
#pragma unroll
      for (int t = 0; t < 8; ++t) *(u32*)(dst + (u32)t * plane_b(V) + j * 128u) = wd[t];
      if (j + 1 < (u32)V / 8) {                         // row r + 8(j+1) = row r + 8j times m^8
#pragma unroll
        for (int e = 0; e < 4; ++e)
          y[e] = LAZY ? mul_shoup4(y[e], m8[e], w8[e], mp.np) : mul_shoup2(y[e], m8[e], w8[e], mp.np);
      }
    }
  }
}

// Per handle, swapped form (MODE 4 / 5): the giant-step byte planes G_s[i][u] = byte s of the
// Montgomery residue m_i^{uV} 2^64 mod p (u < U) in the A layout of each K-block's stage (32 KB).
// Warp task = (K-block, K half): lane = (ql: 4 terms, r: rows r + 8j, j < 16), 4 chains of stride 8
// with the fixed multiplier m^{8V} (Shoup).  A warp's store of one plane word covers 8 rows x 16
// bytes = one 128-byte line, so the planes go straight to global memory.  The per-term powers
// m^V, m^{2V}, m^{4V}, m^{8V} are computed once per term (lane r < 4 of the term's group) and
// shuffled to the group's 8 lanes; the same lane also writes the term's C record (the swapped
// chain's m^8, its Shoup constant, Montgomery m^{rr} for rr < 8) and seed powers (m^V, m^{kChunk}).
constexpr int kGpThreads = 256;
template <bool LAZY, int V>
static __global__ void __launch_bounds__(kGpThreads) k_tc_gplanes(const u64* __restrict__ m, u64 t_pad,
                                                                  uint8_t* __restrict__ Gp, u64* __restrict__ C,
                                                                  u64* __restrict__ MS, ModParams mp) {
  const u64 ntask = 2 * ((t_pad + kKB - 1) / kKB);
  const int lane = threadIdx.x & 31;
  const u32 ql = (u32)(lane >> 3), r = (u32)(lane & 7);
  const u64 nwarp = (u64)gridDim.x * (kGpThreads / 32);
  for (u64 task = (u64)blockIdx.x * (kGpThreads / 32) + (threadIdx.x >> 5); task < ntask; task += nwarp) {
    const u64 blk = task >> 1;
    const u32 h = (u32)(task & 1);
    const u64 q0 = blk * kKB + (u64)h * 16 + ql * 4;
    // lane (ql, r): powers of term q0 + (r & 3)
    static_assert(V == 32, "the shared 8-step prologue below assumes log2(V) + 3 == 8");
    const u64 q = q0 + (r & 3);
    const u64 mm = to_mont(q < t_pad ? m[q] : 0ull, mp);
    // One 8-step chain, branch-free across the two lanes of a term: lanes r < 4 square
    // (m -> m^V -> m^{2V} -> m^{4V} -> m^{8V}), lanes r >= 4 walk the C record's Montgomery
    // m^{rr}, rr < 8 (ending at m^8).
    const bool sq = r < 4;
    const bool rec = !sq && q < t_pad;
    u64 x = sq ? mm : mp.r1, mV = 0, m2V = 0, m4V = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (rec) C[q * kCRec + kC_g0 + k] = x;             // Montgomery m^{k}
      x = mont_mul(x, sq ? x : mm, mp);
      if (k == 4) mV = x;
      if (k == 5) m2V = x;
      if (k == 6) m4V = x;
    }
    // x = m^{8V} (r < 4) or m^8 (r >= 4), Montgomery: normal form and Shoup constant for both
    const u64 nx = from_mont(x, mp), wx = x * mp.pinv;
    if (rec) {
      C[q * kCRec + kC_mL] = nx;                         // m^8
      C[q * kCRec + kC_wL] = wx;                         // shoup_w_fast(m^8)
    }
    const u64 m3V = mont_mul(m2V, mV, mp);               // lanes r < 4 (unused elsewhere)
    if (sq && q < t_pad) {                               // seed powers
      u64 mC = x;                                        // m^{kChunk} = (m^{8V})^16
#pragma unroll 1
      for (int i = 0; i < 4; ++i) mC = mont_mul(mC, mC, mp);
      MS[2 * q] = mV;
      MS[2 * q + 1] = mC;
    }
    u64 y[4], mS[4], wS[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int src = (int)(ql * 8) + e;                 // lane r = e < 4: term q0 + e's powers
      const u64 v1 = __shfl_sync(0xffffffffu, mV, src), v2 = __shfl_sync(0xffffffffu, m2V, src);
      const u64 v3 = __shfl_sync(0xffffffffu, m3V, src), v4 = __shfl_sync(0xffffffffu, m4V, src);
      mS[e] = __shfl_sync(0xffffffffu, nx, src);         // normal m^{8V}: the chain's fixed multiplier
      wS[e] = __shfl_sync(0xffffffffu, wx, src);         // its Shoup constant
      const u32 r2 = r & 3;                              // one product at most: m^{(r&3)V} [x m^{4V}]
      u64 x = r2 == 0 ? mp.r1 : r2 == 1 ? v1 : r2 == 2 ? v2 : v3;
      if (r & 4) x = mont_mul(x, v4, mp);
      y[e] = x;                                          // m^{rV} (Montgomery residue, canonical)
    }
    uint8_t* dst = Gp + blk * kGBytes + plane_off<kLBOA>(r, h * 16 + ql * 4);
#pragma unroll 1
    for (u32 j = 0; j < (u32)kU / 8; ++j) {              // row r + 8j
      const u32 l0 = lo32(y[0]), l1 = lo32(y[1]), l2 = lo32(y[2]), l3 = lo32(y[3]);
      const u32 h0 = hi32(y[0]), h1 = hi32(y[1]), h2 = hi32(y[2]), h3 = hi32(y[3]);
      u32 wd[8];
      u32 a = prmt(l0, l1, 0x5140), b = prmt(l2, l3, 0x5140), c = prmt(l0, l1, 0x7362), d = prmt(l2, l3, 0x7362);
      wd[0] = prmt(a, b, 0x5410); wd[1] = prmt(a, b, 0x7632); wd[2] = prmt(c, d, 0x5410); wd[3] = prmt(c, d, 0x7632);
      a = prmt(h0, h1, 0x5140); b = prmt(h2, h3, 0x5140); c = prmt(h0, h1, 0x7362); d = prmt(h2, h3, 0x7362);
      wd[4] = prmt(a, b, 0x5410); wd[5] = prmt(a, b, 0x7632); wd[6] = prmt(c, d, 0x5410); wd[7] = prmt(c, d, 0x7632);
#pragma unroll
      for (int t = 0; t < 8; ++t) *(u32*)(dst + (u32)t * kPlaneA + j * 128u) = wd[t];
      if (j + 1 < (u32)kU / 8) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          y[e] = LAZY ? mul_shoup4(y[e], mS[e], wS[e], mp.np) : mul_shoup2(y[e], mS[e], wS[e], mp.np);
      }
    }
  }
}

// Per evaluation pass: the chunk seeds LS[c][q] = c_q m_q^{js0 + c*kChunk}.  Thread = (term,
// kSeedChunks consecutive chunks): one exponentiation, then products with m^{kChunk}.
constexpr u32 kSeedChunks = 4;
// Terms [q0, q1) only (a row block of pe_eval); LS keeps its [nch][t_pad] layout.
static __global__ void k_tc_seed(const u64* __restrict__ c, const u64* __restrict__ m, const u64* __restrict__ MS,
                                 u64 t_pad, u64 q0, u64 q1, u32 nch, u32 chunk, u64 js0, u64* __restrict__ LS,
                                 ModParams mp) {
  const u32 ngrp = (nch + kSeedChunks - 1) / kSeedChunks;
  const u64 nq = q1 - q0, total = nq * ngrp;
  for (u64 x = blockIdx.x * (u64)blockDim.x + threadIdx.x; x < total; x += (u64)gridDim.x * blockDim.x) {
    const u64 grp = x / nq, q = q0 + (x - grp * nq);
    const u32 ch0 = (u32)grp * kSeedChunks, ch1 = min(nch, ch0 + kSeedChunks);
    const u64 mC = MS[2 * q + 1];                        // Montgomery m^{kChunk}
    u64 s = seed_pow(c[q], m[q], js0 + (u64)ch0 * chunk, mp);   // normal form, < p
    for (u32 ch = ch0; ch < ch1; ++ch) {
      LS[(u64)ch * t_pad + q] = s;
      s = mont_mul(s, mC, mp);                           // normal x Montgomery -> normal
    }
  }
}

}  // namespace tc
}  // namespace pe
