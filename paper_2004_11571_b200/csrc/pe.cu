// pe.cu -- C ABI (include/pe.h) and host planner of the B200 partial-evaluation library.
//
// pe_create: validate on the host (before any CUDA call), upload, then on the device:
//   keys -> CUB radix sort (descending lex on (dx,dy)) -> run-length
//   encode (the G buckets and their sizes) -> [host: tile plan from the G sizes] ->
//   power tables -> k_setup (m_i, w_i, c_i in the padded tile layout).
// pe_eval_device: per pass of points, k_step (seed + hot loop + in-CTA reduction) then
//   k_fixup (cross-CTA sums -> canonical out).
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/pe.h"
#include "fast.h"
#include "kernels.cuh"
#include "tc.cuh"

using namespace pe;

// ---------------------------------------------------------------- errors
static thread_local int g_last_error = PE_OK;
static int set_err(int e) { g_last_error = e; return e; }
namespace pe {
int set_last_error(int e) { return set_err(e); }   // bm.cu's calls report through pe_last_error too
}

#define CU(call)                                                                  \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      if (getenv("PE_DEBUG")) fprintf(stderr, "pe: %s:%d %s: %s\n", __FILE__,     \
                                      __LINE__, #call, cudaGetErrorString(_e));   \
      return set_err(_e == cudaErrorMemoryAllocation ? PE_ENOMEM : PE_ECUDA);     \
    }                                                                             \
  } while (0)

// ---------------------------------------------------------------- host number theory
typedef unsigned __int128 u128;
static u64 h_mulmod(u64 a, u64 b, u64 p) { return (u64)(((u128)a * b) % p); }
static u64 h_powmod(u64 b, u64 e, u64 p) {
  u64 r = 1 % p;
  b %= p;
  while (e) {
    if (e & 1) r = h_mulmod(r, b, p);
    b = h_mulmod(b, b, p);
    e >>= 1;
  }
  return r;
}
// Deterministic Miller-Rabin for 64-bit n with the 12 prime bases <= 37.
static bool h_is_prime(u64 n) {
  if (n < 2) return false;
  static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (u64 b : bases) {
    if (n == b) return true;
    if (n % b == 0) return false;
  }
  u64 d = n - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; ++s; }
  for (u64 b : bases) {
    u64 x = h_powmod(b, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < s; ++i) {
      x = h_mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}
static ModParams h_mod_params(u64 p) {
  ModParams mp;
  mp.p = p;
  mp.np = (u64)0 - p;
  // p^{-1} mod 2^64 by Newton iteration, then negate
  u64 inv = p;  // correct to 3 bits for odd p
  for (int i = 0; i < 6; ++i) inv *= 2 - p * inv;
  mp.pinv = (u64)0 - inv;
  mp.r1 = (u64)(((u128)1 << 64) % p);
  mp.r2 = h_mulmod(mp.r1, mp.r1, p);
  mp.pd = (double)p;
  mp.u = 1.0 / (double)p;  // RN(1/p) (host IEEE division, default rounding)
  return mp;
}

// ---------------------------------------------------------------- handle
struct pe_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;  // handle's own stream (pe_create, pe_eval)
  u64 p = 0, t = 0;
  u32 n = 0;
  ModParams mp{};
  int path = kInt4;
  int R = 8, W = 8, chunk_req = 0;
  u64 G = 0, t_pad = 0;
  u32 n_wt = 0, n_slots = 0;
  std::vector<u32> dxdy;  // host copy [2G]
  std::vector<u64> poly_off{0, 0};   // term offsets of the batched polynomials [npoly+1]
  std::vector<u64> poly_rows{0, 0};  // first output row of each polynomial [npoly+1]
  // device
  u64 *d_c = nullptr, *d_m = nullptr, *d_w = nullptr;
  u32* d_perm = nullptr;
  uint2* d_wt_info = nullptr;
  u32* d_slot_start = nullptr;
  u64* d_partial = nullptr;
  size_t partial_elems = 0;
  u64* d_out_scratch = nullptr;
  size_t out_scratch_elems = 0;
  // tensor-core path (tc.cuh): 0 off, 1 auto (T >= tc_min_T(t_pad)), 2 forced
  int tc_mode = 0;
  bool tc_ok = false;
  bool tc_swap = false;   // swapped form (tc.cuh MODE 4 / 5): giant-step planes per handle, baby steps generated
  int tc_form_req = 0;    // pe_config.tc_form
  u32 tc_rounds = 2;
  u32 tc_v = 64, tc_chunk = 8192;   // baby steps and points per chunk of the handle's k_tc geometry (tc.cuh mode_v)
  int n_sm = 148;
  u64* d_tcC = nullptr;   // [t_pad][2] tensor-core path C records (tc.cuh)
  u64* d_tcMS = nullptr;  // [t_pad][2] Montgomery m^V, m^{kChunk} (k_tc_seed)
  uint8_t* d_tcR = nullptr;   // [t_pad / 32][tc::kRBytes] baby-step byte planes m^v, v < 64 (tc.cuh)
  u64* d_seed = nullptr;
  size_t seed_elems = 0;
  u32* d_tc_scratch = nullptr;   // k_tc per-CTA drained diagonal sums (n_sm x 2 x kDiag x kChunk u32)
  u32* h_status = nullptr;       // mapped host word: k_tc sets it when a pipeline wait times out
  u32* d_status = nullptr;       // its device address
  // caller streams pe_eval_device(_rows) enqueued work on, with an event after the latest such
  // work: pe_destroy waits for these instead of synchronising the whole device
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> used;
  // k_tc piece plans, one per chunk count of a pass (tc_plan): pieces, partial slots, unit schedule
  struct TcPlan {
    u32 npieces = 0, nslots = 0, grid = 0, max_slots = 0;   // max_slots: most partial rows of one bucket
    std::vector<uint4> pieces;       // x = first padded term, y = K-blocks, z = slot (size-sorted)
    std::vector<u32> slot_start;     // [G+1] partial slots of bucket g (x rounds)
    std::vector<u32> sched;          // [nunits] units per CTA, then [grid + 1] offsets
    uint4* d_piece = nullptr;
    u32* d_slot_start = nullptr;
    u32* d_sched = nullptr;
    cudaEvent_t uploaded = nullptr;  // the device copies are complete (any stream may wait on it)
  };
  u64 split_g1 = 0;                  // pe_eval's row split for the tensor path (0: no split)
  // lazily built cache (also from const queries), keyed by (chunks per pass, first row, end row)
  mutable std::map<std::tuple<u32, u64, u64>, TcPlan> tc_plans;
  // asymptotically fast method (fast.cu, NEXT-4): 0 off, 1 automatic (T >= fast_min_T), 2 forced
  int fast_mode = 0;
  u64 fast_min_T = 0;
  fast::Plan* fast = nullptr;
  std::vector<u64> h_poff;       // padded bucket offsets [G+1] (the fast path's tree shape)
  size_t partial_cap_bytes = (size_t)1 << 30;
  cudaStream_t copy_stream = nullptr;   // pe_eval: device->host copy of a column block
  cudaEvent_t copy_done = nullptr;
  // kernel timing (pe_set_timing / pe_kernel_stats)
  bool timing = false;
  struct Rec { cudaEvent_t e0, e1, e2; double tp; };
  std::vector<Rec> recs;
};

static void drop_recs(pe_ctx* h) {
  for (auto& r : h->recs) { cudaEventDestroy(r.e0); cudaEventDestroy(r.e1); cudaEventDestroy(r.e2); }
  h->recs.clear();
}

// k_tc status words: mapped, portable pinned host memory handed out from 4-KB slabs that live for
// the process -- cudaHostAlloc / cudaFreeHost per handle would serialise with (and cudaFreeHost
// synchronise against) work other threads have in flight on the device
static std::mutex g_status_mu;
static std::vector<std::pair<u32*, u32*>> g_status_free;   // (host, device) words
static int status_get(u32** host, u32** dev) {
  std::lock_guard<std::mutex> lk(g_status_mu);
  if (g_status_free.empty()) {
    const int kWords = 1024;
    u32* base = nullptr;
    u32* dbase = nullptr;
    if (cudaHostAlloc((void**)&base, kWords * sizeof(u32), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
      return PE_ENOMEM;
    if (cudaHostGetDevicePointer((void**)&dbase, base, 0) != cudaSuccess) return PE_ECUDA;   // slab kept
    for (int i = kWords - 1; i >= 0; --i) g_status_free.emplace_back(base + i, dbase + i);
  }
  *host = g_status_free.back().first;
  *dev = g_status_free.back().second;
  g_status_free.pop_back();
  **host = 0;
  return PE_OK;
}
static void status_put(u32* host, u32* dev) {
  std::lock_guard<std::mutex> lk(g_status_mu);
  g_status_free.emplace_back(host, dev);
}

static int note_use(pe_ctx* h, cudaStream_t s) {
  for (auto& u : h->used)
    if (u.first == s) return cudaEventRecord(u.second, s) == cudaSuccess ? PE_OK : PE_ECUDA;
  cudaEvent_t e;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return PE_ECUDA;
  h->used.emplace_back(s, e);
  return cudaEventRecord(e, s) == cudaSuccess ? PE_OK : PE_ECUDA;
}

static void free_all(pe_ctx* h) {
  if (!h) return;
  drop_recs(h);
  // stream-ordered frees back into the (retained) device memory pool
  cudaStream_t s = h->stream;
  for (void* q : {(void*)h->d_c, (void*)h->d_m, (void*)h->d_w, (void*)h->d_perm, (void*)h->d_wt_info, (void*)h->d_slot_start, (void*)h->d_partial,
                  (void*)h->d_out_scratch, (void*)h->d_tcC, (void*)h->d_tcR, (void*)h->d_tcMS,
                  (void*)h->d_tc_scratch, (void*)h->d_seed})
    if (q) cudaFreeAsync(q, s);
  for (auto& kv : h->tc_plans) {
    for (void* q : {(void*)kv.second.d_piece, (void*)kv.second.d_slot_start, (void*)kv.second.d_sched})
      if (q) cudaFreeAsync(q, s);
    if (kv.second.uploaded) cudaEventDestroy(kv.second.uploaded);
  }
  h->tc_plans.clear();
  if (s) cudaStreamSynchronize(s);
  if (h->copy_stream) cudaStreamSynchronize(h->copy_stream), cudaStreamDestroy(h->copy_stream);
  if (h->copy_done) cudaEventDestroy(h->copy_done);
  if (h->h_status) status_put(h->h_status, h->d_status), h->h_status = h->d_status = nullptr;
  if (h->fast) fast::destroy(h->fast, s), h->fast = nullptr;
  if (h->stream) cudaStreamDestroy(h->stream);
}

// All device buffers are stream-ordered allocations from the device's default memory pool,
// whose release threshold is raised once per device so that repeated create / eval / destroy
// cycles reuse memory instead of paying cudaMalloc / cudaFree each time.
static thread_local cudaStream_t g_alloc_stream = nullptr;
static void retain_pool_once(int dev) {
  static bool done[64] = {};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}
template <class T>
static int dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  CU(cudaMallocAsync((void**)p, n * sizeof(T), g_alloc_stream));
  return PE_OK;
}

static int env_int(const char* k, int dflt) {
  const char* v = getenv(k);
  return v && *v ? atoi(v) : dflt;
}

// ---------------------------------------------------------------- kernel dispatch
template <int PATH>
static cudaError_t launch_step_path(int R, dim3 grid, dim3 block, cudaStream_t s, const StepArgs& a) {
  switch (R) {
    case 1: k_step<PATH, 1><<<grid, block, 0, s>>>(a); break;
    case 2: k_step<PATH, 2><<<grid, block, 0, s>>>(a); break;
    case 4: k_step<PATH, 4><<<grid, block, 0, s>>>(a); break;
    case 8: k_step<PATH, 8><<<grid, block, 0, s>>>(a); break;
    case 16:
      if (PATH == kFp64) return cudaErrorInvalidValue;
      k_step<PATH == kFp64 ? kInt4 : PATH, 16><<<grid, block, 0, s>>>(a);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
static cudaError_t launch_step(int path, int R, dim3 grid, dim3 block, cudaStream_t s, const StepArgs& a) {
  if (path == kInt32) return launch_step_path<kInt32>(R, grid, block, s, a);
  if (path == kInt4) return launch_step_path<kInt4>(R, grid, block, s, a);
  if (path == kInt2) return launch_step_path<kInt2>(R, grid, block, s, a);
  return launch_step_path<kFp64>(R, grid, block, s, a);
}

// automatic tensor-core path from this many points (a chunk is 8192 points, 4096 in the V = 32
// geometry of p >= 2^54): k_tc
// costs a flat ~0.11 ms + 0.42 ns per padded term for any T <= 8192, k_step grows with t * T.
// Measured crossovers (scripts/tc_threshold.py, profiles/r01_tc_threshold.jsonl): T ~ 860 for
// 10^5 terms, ~480 for 10^6 (k_step INT), 512 vs FP64 Alg. 2 -- i.e. T* ~ 8.6e7 / t_pad, >= 512.
// p < 2^31 competes with the 4-IMAD-slot 32-bit Shoup k_step instead: crossovers T ~ 770 (10^6
// terms) and ~930 (10^5) against k_tc's 4-digit mode (scripts/tc_threshold_p31.py).
// p >= 2^54 (the V = 32 geometry, 4096-point chunks; scripts/tc_threshold_v32.py,
// profiles/r02_tc_threshold_v32.jsonl): crossovers T ~ 540 / 380 / 280 / 235 at 1.3e4 / 1.0e5 /
// 3.1e5 / 1.0e6 padded terms, fitted by T* = max(3400 t_pad^-0.19, 7.3e6 / t_pad) (the second term:
// tiny handles, where k_step's cost is ~flat while k_tc keeps its ~0.045 ms floor), in [192, 8192].
// The 7-digit mode (2^31 <= p < 2^54, V = 32 since session 2) against the FP64 Alg. 2 k_step
// (scripts/tc_threshold_v32.py --p50, profiles/r02_tc_threshold_v32_p50.jsonl): crossovers T ~ 510 /
// 420 / 330 / 270 at the same term counts, fitted by max(2200 t_pad^-0.144, 7.3e6 / t_pad).
static u64 tc_min_T_v32(u64 t_pad, double a, double b) {
  const double tp = (double)std::max<u64>(t_pad, 1);
  const double t = std::max(a * std::pow(tp, -b), 7.3e6 / tp);
  return std::min<u64>(8192, std::max<u64>(192, (u64)std::ceil(t)));
}
static u64 tc_min_T(u64 t_pad, u64 p) {
  const u64 tp = std::max<u64>(t_pad, 1);
  if (p >= (1ull << 54)) return tc_min_T_v32(t_pad, 3400.0, 0.19);
  if (p >= (1ull << 31)) return tc_min_T_v32(t_pad, 2200.0, 0.144);
  // p < 2^31: the 4-digit mode with 32-bit Shoup producers against the 32-bit Shoup k_step
  // (scripts/tc_threshold_v32.py --p31, profiles/r02_tc_threshold_p31_shoup32.jsonl): crossovers
  // T ~ 850 / 780 / 750 / 730 at 1.3e4 / 1.0e5 / 3.1e5 / 1.0e6 padded terms
  if (p < (1ull << 31)) {
    const double t = std::max(1350.0 * std::pow((double)tp, -0.045), 1.1e7 / (double)tp);
    return std::min<u64>(8192, std::max<u64>(512, (u64)std::ceil(t)));
  }
  if (t_pad >= 500000) return 512;
  return std::min<u64>(8192, std::max<u64>(512, 86000000ull / tp));
}

// automatic fast-method threshold against the scalar matrix method (points; profiles/
// r02_fast_sweep_*.jsonl): fast/k_step = 1.05 at T = 4096 and 0.72 at 8192 on config 3 (3.9k terms
// per bucket), 0.81 at 4096 on config 5 (10k per bucket).  Its per-bucket Newton inversion costs
// O(T log T) whatever the bucket size, so it also needs >= kFastMinTermsPerBucket terms per bucket.
static const u64 kFastMinT = 8192;
static const u64 kFastMinTermsPerBucket = 2048;

static unsigned grid_for(u64 n, unsigned block) {
  u64 b = (n + block - 1) / block;
  if (b == 0) b = 1;
  return (unsigned)std::min<u64>(b, 148ull * 64);
}

// ---------------------------------------------------------------- create
static int tc_plan(const pe_ctx* h, u32 nch, u64 g0, u64 g1, bool upload, cudaStream_t s, pe_ctx::TcPlan** out);


// pe_eval's row split for the tensor path: rows [0, G1) then [G1, G), the first block's device->host
// copy overlapping the second's evaluation.  G1 minimises E1 + max(E2, D1) + D2 under a simple model
// -- evaluation ~ padded terms x T at ~2e13 term-points/s, copy ~ rows x T x 8 B at ~50 GB/s (PCIe 5)
// -- in which T cancels, so the split is a property of the handle (config 5: ~22 % of the terms in
// the second block, whose copy, the exposed tail, is ~1/4 of the result).  0 = no split.
static u64 tc_row_split(const pe_ctx* h) {
  if (h->G < 2) return 0;
  // ce: k_tc seconds per padded term-point (config 5 runs at ~2.4e13; env PE_SPLIT_RATE_T in units of
  // 1e12 for experiments -- 20 / 24 / 30 measure the same e2e within noise), cd: D2H seconds per byte-point
  const double ce = 1.0 / (env_int("PE_SPLIT_RATE_T", 24) * 1e12), cd = 8.0 / 5e10, tp = (double)h->t_pad;
  double best = tp * ce + (double)h->G * cd;   // no split
  u64 G1 = 0;
  for (u64 g = 1; g < h->G; ++g) {
    const double e1 = (double)h->h_poff[g] * ce, e2 = (tp - (double)h->h_poff[g]) * ce;
    const double d1 = (double)g * cd, d2 = (double)(h->G - g) * cd;
    const double tot = e1 + std::max(e2, d1) + d2;
    if (tot < best) { best = tot; G1 = g; }
  }
  return G1;
}

// Development: env PE_CREATE_PROF=1 prints the device time between pe_create's phases (CUDA events on
// the handle stream; host waits show up as gaps).
struct CreateProf {
  bool on = false;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  std::vector<double> host_ms;   // host clock when each mark was issued
  static double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  void mark(const char* what, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back({what, e});
    host_ms.push_back(now_ms());
  }
  ~CreateProf() {
    if (!on || ev.empty()) return;
    cudaEventSynchronize(ev.back().second);
    for (size_t i = 1; i < ev.size(); ++i) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
      fprintf(stderr, "pe_create %-28s device %8.3f ms  host %8.3f ms\n", ev[i].first, ms, host_ms[i] - host_ms[i - 1]);
    }
    for (auto& x : ev) cudaEventDestroy(x.second);
  }
};

template <class E>
static int create_impl(pe_ctx* h, const u64* coeffs, const E* exps, const u64* alpha) {
  const u64 t = h->t;
  const u32 n = h->n;
  const u32 nz = n - 2;
  CU(cudaGetDevice(&h->device));
  CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  cudaStream_t s = h->stream;
  retain_pool_once(h->device);
  g_alloc_stream = s;
  CreateProf prof;
  prof.on = env_int("PE_CREATE_PROF", 0) != 0;
  prof.mark("start", s);
  if (t == 0) {
    h->G = 0;
    return PE_OK;
  }

  // ---- upload (a1)
  u64* d_coeffs; E* d_exps; u64* d_alpha;
  if (dalloc(&d_coeffs, t) || dalloc(&d_exps, t * n) || dalloc(&d_alpha, nz + 1)) return g_last_error;
  struct Tmp {
    std::vector<void*> v;
    cudaStream_t s = nullptr;
    ~Tmp() { for (void* p : v) if (p) cudaFreeAsync(p, s); }
  } tmp;
  tmp.v = {d_coeffs, d_exps, d_alpha};
  tmp.s = s;
  std::vector<u64> alpha_red(nz + 1, 1);
  for (u32 l = 0; l < nz; ++l) alpha_red[l] = alpha[l] % h->p;
  CU(cudaMemcpyAsync(d_alpha, alpha_red.data(), (nz + 1) * sizeof(u64), cudaMemcpyHostToDevice, s));
  // power tables alpha_l^e, e < kTab (a3), ready before the first chunk lands
  u64* d_table = nullptr;
  if (nz) {
    if (dalloc(&d_table, (size_t)nz * kTab)) return g_last_error;
    tmp.v.push_back(d_table);
    k_power_table<<<grid_for((u64)nz * kTab, 128), 128, 0, s>>>(d_alpha, nz, kTab - 1, d_table, h->mp);
    CU(cudaGetLastError());
  }

  // ---- upload in chunks on a copy stream; keys (a2) and monomials (a3) of each chunk run on the
  // handle's stream as soon as it lands, while the next chunks are still crossing PCIe.  The
  // exponents go first: the sort, the plan and the tensor-path setup need only them, and run while
  // the coefficients (needed by k_setup_c alone) follow.
  u64 *d_key, *d_key2, *d_m_in; u32 *d_idx, *d_idx2, *d_kmax;
  if (dalloc(&d_key, t) || dalloc(&d_key2, t) || dalloc(&d_idx, t) || dalloc(&d_idx2, t) || dalloc(&d_m_in, t) ||
      dalloc(&d_kmax, 2))
    return g_last_error;
  tmp.v.insert(tmp.v.end(), {d_key, d_key2, d_idx, d_idx2, d_m_in, d_kmax});
  CU(cudaMemsetAsync(d_kmax, 0, 2 * sizeof(u32), s));
  // the coefficients are on the device; on every exit the handle stream waits for them before the
  // temporaries (freed on that stream after this guard) can be reused
  struct EvGuard {
    cudaEvent_t& e;
    cudaStream_t s;
    ~EvGuard() { if (e) cudaStreamWaitEvent(s, e, 0), cudaEventDestroy(e); }
  };
  cudaEvent_t c_landed = nullptr;
  EvGuard c_guard{c_landed, s};
  {
    cudaStream_t cs = nullptr;
    CU(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    const u64 nchunk = t >= (1u << 20) ? 8 : 1;
    std::vector<cudaEvent_t> ev(nchunk, nullptr);
    int rc = PE_OK;
    if (cudaEventCreateWithFlags(&c_landed, cudaEventDisableTiming) != cudaSuccess) rc = PE_ECUDA;
    cudaEvent_t ready = nullptr;   // the copy stream starts after the handle stream's allocations
    if (cudaEventCreateWithFlags(&ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ready, s) != cudaSuccess || cudaStreamWaitEvent(cs, ready, 0) != cudaSuccess)
      rc = PE_ECUDA;
    for (u64 k = 0; k < nchunk && rc == PE_OK; ++k) {
      const u64 a = t * k / nchunk, b = t * (k + 1) / nchunk;
      if (cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming) != cudaSuccess ||
          cudaMemcpyAsync(d_exps + a * n, exps + a * n, (b - a) * n * sizeof(E), cudaMemcpyHostToDevice, cs) !=
              cudaSuccess ||
          cudaEventRecord(ev[k], cs) != cudaSuccess || cudaStreamWaitEvent(s, ev[k], 0) != cudaSuccess) {
        rc = PE_ECUDA;
        break;
      }
      k_keys<<<grid_for(b - a, 256), 256, 0, s>>>(d_exps, a, b, n, d_key, d_idx, d_kmax);
      k_monomials<<<grid_for(b - a, 256), 256, 0, s>>>(d_exps, a, b, n, d_table, d_alpha, d_m_in, h->mp);
      if (cudaGetLastError() != cudaSuccess) rc = PE_ECUDA;
    }
    if (rc == PE_OK &&
        (cudaMemcpyAsync(d_coeffs, coeffs, t * sizeof(u64), cudaMemcpyHostToDevice, cs) != cudaSuccess ||
         cudaEventRecord(c_landed, cs) != cudaSuccess))
      rc = PE_ECUDA;
    for (auto e : ev) if (e) cudaEventDestroy(e);   // destruction is deferred until the events complete
    if (ready) cudaEventDestroy(ready);
    cudaStreamDestroy(cs);                           // likewise: returns at once, the copies still run
    if (rc != PE_OK) return set_err(rc);
  }
  prof.mark("upload+keys+monomials", s);
  // key width: the largest x and y degrees (the host waits here for the upload it cannot pass)
  u32 kmax[2] = {0, 0};
  CU(cudaMemcpyAsync(kmax, d_kmax, 2 * sizeof(u32), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  auto nbits = [](u32 x) { int b = 0; while (b < 32 && (x >> b)) ++b; return b; };
  const int bd = nbits(kmax[1]), key_bits = std::max(1, nbits(kmax[0]) + bd);
  k_pack_keys<<<grid_for(t, 256), 256, 0, s>>>(d_key, t, (u32)bd);
  CU(cudaGetLastError());
  const u32 npoly = (u32)h->poly_off.size() - 1;
  size_t sort_bytes = 0, sort2_bytes = 0, sel_bytes = 0;
  unsigned char* d_flags;
  u32 *d_starts, *d_nruns, *d_pid = nullptr, *d_pid2 = nullptr, *d_iota = nullptr, *d_perm = nullptr;
  if (dalloc(&d_flags, t) || dalloc(&d_starts, t + 1) || dalloc(&d_nruns, 1)) return g_last_error;
  tmp.v.insert(tmp.v.end(), {d_flags, d_starts, d_nruns});
  cub::CountingInputIterator<u32> counting(0);
  CU(cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, d_key, d_key2, d_idx, d_idx2, (int)t, 0, 64, s));
  CU(cub::DeviceSelect::Flagged(nullptr, sel_bytes, counting, d_flags, d_starts, d_nruns, (int)t, s));
  if (npoly > 1) {
    if (dalloc(&d_pid, t) || dalloc(&d_pid2, t) || dalloc(&d_iota, t) || dalloc(&d_perm, t)) return g_last_error;
    tmp.v.insert(tmp.v.end(), {d_pid, d_pid2, d_iota, d_perm});
    CU(cub::DeviceRadixSort::SortPairs(nullptr, sort2_bytes, d_pid, d_pid2, d_iota, d_perm, (int)t, 0, 32, s));
  }
  void* d_cub;
  if (dalloc((char**)&d_cub, std::max(std::max(sort_bytes, sort2_bytes), sel_bytes))) return g_last_error;
  tmp.v.push_back(d_cub);
  CU(cub::DeviceRadixSort::SortPairsDescending(d_cub, sort_bytes, d_key, d_key2, d_idx, d_idx2, (int)t, 0,
                                               key_bits, s));
  u64* d_keyS = d_key2;   // final order: (polynomial asc, dx desc, dy desc)
  u32* d_idxS = d_idx2;
  if (npoly > 1) {
    u64* d_poff;
    if (dalloc(&d_poff, npoly + 1)) return g_last_error;
    tmp.v.push_back(d_poff);
    CU(cudaMemcpyAsync(d_poff, h->poly_off.data(), (npoly + 1) * sizeof(u64), cudaMemcpyHostToDevice, s));
    k_poly_of<<<grid_for(t, 256), 256, 0, s>>>(d_idx2, t, d_poff, npoly, d_pid, d_iota);
    CU(cudaGetLastError());
    // LSD radix sort is stable: equal polynomial ids keep their (dx,dy)-descending order
    CU(cub::DeviceRadixSort::SortPairs(d_cub, sort2_bytes, d_pid, d_pid2, d_iota, d_perm, (int)t, 0, 32, s));
    k_apply_perm<<<grid_for(t, 256), 256, 0, s>>>(d_perm, t, d_key2, d_idx2, d_key, d_idx);
    CU(cudaGetLastError());
    d_keyS = d_key;
    d_idxS = d_idx;
  }
  k_run_flags<<<grid_for(t, 256), 256, 0, s>>>(d_keyS, npoly > 1 ? d_pid2 : nullptr, t, d_flags);
  CU(cudaGetLastError());
  CU(cub::DeviceSelect::Flagged(d_cub, sel_bytes, counting, d_flags, d_starts, d_nruns, (int)t, s));

  prof.mark("sort+runs", s);
  u32 nruns = 0;
  CU(cudaMemcpyAsync(&nruns, d_nruns, sizeof(u32), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  const u64 G = nruns;
  h->G = G;
  u64* d_ukeys; u32* d_upid;
  if (dalloc(&d_ukeys, G) || dalloc(&d_upid, G)) return g_last_error;
  tmp.v.insert(tmp.v.end(), {d_ukeys, d_upid});
  k_gather_runs<<<grid_for(G, 256), 256, 0, s>>>(d_starts, (u32)G, d_keyS, npoly > 1 ? d_pid2 : nullptr,
                                                 d_ukeys, d_upid);
  CU(cudaGetLastError());
  std::vector<u64> ukeys(G);
  std::vector<u32> starts(G + 1), upid(G), counts(G);
  CU(cudaMemcpyAsync(ukeys.data(), d_ukeys, G * sizeof(u64), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(starts.data(), d_starts, G * sizeof(u32), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(upid.data(), d_upid, G * sizeof(u32), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  starts[G] = (u32)t;
  for (u64 g = 0; g < G; ++g) counts[g] = starts[g + 1] - starts[g];
  h->dxdy.resize(2 * G);
  const u64 ymask = bd >= 64 ? ~0ull : ((1ull << bd) - 1);
  for (u64 g = 0; g < G; ++g) { h->dxdy[2 * g] = (u32)(ukeys[g] >> bd); h->dxdy[2 * g + 1] = (u32)(ukeys[g] & ymask); }
  h->poly_rows.assign(npoly + 1, G);
  for (u64 g = G; g-- > 0;) h->poly_rows[upid[g]] = g;            // first row of each polynomial
  for (u32 k = npoly; k-- > 0;) h->poly_rows[k] = std::min(h->poly_rows[k], h->poly_rows[k + 1]);

  // ---- host tile plan from the G bucket sizes
  const int maxR = h->path == kFp64 ? 8 : 16;
  int R = h->R;
  if (R == 0) {
    // largest R whose per-bucket padding wastes <= 6% of the terms (and R <= 8 by default)
    R = 1;
    for (int cand = 8; cand >= 1; cand >>= 1) {
      u64 tile = 32ull * cand, padded = 0;
      for (u64 g = 0; g < G; ++g) padded += (counts[g] + tile - 1) / tile * tile;
      if (padded - t <= t * 6 / 100 || cand == 1) { R = cand; break; }
    }
  }
  if (R != 1 && R != 2 && R != 4 && R != 8 && R != 16) return set_err(PE_EINVAL);
  if (R > maxR) return set_err(PE_ENOTSUP);
  if (32 * h->W > step_max_threads(h->path, R)) return set_err(PE_EINVAL);
  h->R = R;
  const u64 tile = 32ull * R;
  std::vector<u64> poff(G + 1), bstart(G + 1);
  poff[0] = bstart[0] = 0;
  for (u64 g = 0; g < G; ++g) {
    bstart[g + 1] = bstart[g] + counts[g];
    poff[g + 1] = poff[g] + (counts[g] + tile - 1) / tile * tile;
  }
  h->t_pad = poff[G];
  h->h_poff = poff;
  const u64 n_wt = h->t_pad / tile;
  if (n_wt >= 0x7fffffffull) return set_err(PE_ERANGE);
  h->n_wt = (u32)n_wt;
  // ---- padded layout + monomials
  u64 *d_poff, *d_bstart;
  if (dalloc(&d_poff, G + 1) || dalloc(&d_bstart, G + 1)) return g_last_error;
  tmp.v.insert(tmp.v.end(), {d_poff, d_bstart});
  CU(cudaMemcpyAsync(d_poff, poff.data(), (G + 1) * sizeof(u64), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(d_bstart, bstart.data(), (G + 1) * sizeof(u64), cudaMemcpyHostToDevice, s));
  if (dalloc(&h->d_c, h->t_pad) || dalloc(&h->d_m, h->t_pad) || dalloc(&h->d_w, h->t_pad) ||
      dalloc(&h->d_perm, h->t_pad) || dalloc(&h->d_wt_info, n_wt) || dalloc(&h->d_slot_start, G + 1))
    return g_last_error;
  prof.mark("host plan (+gaps)", s);
  k_setup<<<grid_for(h->t_pad, 256), 256, 0, s>>>(d_m_in, d_idxS, d_poff, d_bstart, (u32)G, h->t_pad,
                                                   h->d_m, h->d_w, h->d_perm, h->mp);
  CU(cudaGetLastError());

  // ---- tensor-core path (tc.cuh): per-term strides + the piece plan
  if (h->tc_mode != 0 && (h->path == kInt4 || h->path == kInt2 || h->path == kFp64 || h->path == kInt32)) {
    const u64 tp = h->t_pad;
    // handle memory of the tensor-core form: C records + seed powers + baby-step planes (DESIGN.md
    // §6, ~624 B per padded term).  If it does not fit (the device, or the env cap PE_TC_MEM_MB),
    // an automatic handle degrades to the scalar k_step; a forced one (PE_PATH_TC) fails.
    const u64 nrblk = (tp + 2 * tc::kKB - 1) / (2 * tc::kKB);
    // 8-digit primes (p >= 2^54): the swapped form (tc.cuh; giant-step planes per handle, 1 KB per
    // term; 7-digit primes may request it) unless pe_config.tc_form asks for the plain one; with PE_TC_FORM_AUTO the env override
    // PE_TC_SWAP=0/1 decides, and an automatic swapped handle whose planes do not fit (the device,
    // or PE_TC_MEM_MB) falls back to the plain form (256 B per term) before the scalar k_step.
    const bool auto_form = h->tc_form_req == PE_TC_FORM_AUTO;
    // automatic: swapped for 8 digits (config 5: 13-15 % faster evaluations); plain for 7 digits,
    // where the swapped form measured no gain on config 4 (0.276 vs 0.272 ms: one 4096-point chunk
    // per piece reads the 1-KB giant-step planes once, with no L2 reuse across chunk-units)
    const int form = !auto_form ? h->tc_form_req
                   : (env_int("PE_TC_SWAP", h->p >= (1ull << 54) ? 1 : 0) ? PE_TC_FORM_SWAPPED : PE_TC_FORM_PLAIN);
    h->tc_swap = h->p >= (1ull << 31) && form == PE_TC_FORM_SWAPPED;   // 7- and 8-digit modes
    // 7- and 8-digit modes (p >= 2^31), plain or swapped: the single-round V = 32 geometry (tc.cuh
    // mode_v); the 4-digit mode (p < 2^31) keeps V = 64 (its 7 diagonals already fit one round)
    h->tc_v = h->p >= (1ull << 31) ? 32u : 64u;
    h->tc_chunk = tc::chunk_pts((int)h->tc_v);
    const u64 cap = (u64)std::max(0, env_int("PE_TC_MEM_MB", 0)) << 20;
    int rc = PE_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {
      const u64 plane_bytes = h->tc_swap ? (tp + tc::kKB - 1) / tc::kKB * tc::kGBytes : nrblk * 2 * tc::r_bytes((int)h->tc_v);
      const u64 tc_bytes = (u64)tc::kCRec * 8 * tp + 16 * tp + plane_bytes;
      rc = PE_OK;
      if (cap && tc_bytes > cap) rc = PE_ENOMEM;
      if (rc == PE_OK && (dalloc(&h->d_tcC, (size_t)tc::kCRec * tp) || dalloc(&h->d_tcMS, (size_t)2 * tp) ||
                          dalloc(&h->d_tcR, (size_t)plane_bytes)))
        rc = g_last_error;
      if (rc == PE_OK) break;
      if (rc != PE_ENOMEM) return set_err(rc);
      for (void** q : {(void**)&h->d_tcC, (void**)&h->d_tcMS, (void**)&h->d_tcR})
        if (*q) { cudaFreeAsync(*q, s); *q = nullptr; }
      cudaGetLastError();               // allocation failures are not sticky; clear the record
      g_last_error = PE_OK;
      if (!(auto_form && h->tc_swap)) break;
      h->tc_swap = false;               // automatic form: retry with the plain form's smaller planes
    }
    if (rc != PE_OK) {
      if (h->tc_mode == 2) return set_err(rc);
      h->tc_mode = 0;                   // the rest of the tensor-path setup is skipped below
    }
  }
  if (h->tc_mode != 0 && (h->path == kInt4 || h->path == kInt2 || h->path == kFp64 || h->path == kInt32)) {
    const u64 tp = h->t_pad;
    prof.mark("k_setup (+copies)", s);
    // swapped form: one kernel writes the giant-step planes, the C records and the seed powers.
    // Plain form: the C records (k_tc_setup) and the baby-step planes (k_tc_rplanes) both depend
    // only on m; the former runs on a side stream beside the latter.
    if (h->tc_swap) {
      const u64 ngp = 2 * ((tp + tc::kKB - 1) / tc::kKB);        // warp tasks (K-block, K half)
      const unsigned gpg = (unsigned)std::max<u64>(1, std::min<u64>((ngp + 7) / 8, 148ull * 8));
      if (h->p < (1ull << 62))
        tc::k_tc_gplanes<true, 32><<<gpg, tc::kGpThreads, 0, s>>>(h->d_m, tp, h->d_tcR, h->d_tcC, h->d_tcMS, h->mp);
      else
        tc::k_tc_gplanes<false, 32><<<gpg, tc::kGpThreads, 0, s>>>(h->d_m, tp, h->d_tcR, h->d_tcC, h->d_tcMS, h->mp);
      CU(cudaGetLastError());
    } else {
      cudaStream_t s2 = nullptr;
      cudaEvent_t e_m = nullptr, e_done = nullptr;
      CU(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
      int rc = PE_OK;
      if (cudaEventCreateWithFlags(&e_m, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&e_done, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventRecord(e_m, s) != cudaSuccess || cudaStreamWaitEvent(s2, e_m, 0) != cudaSuccess)
        rc = PE_ECUDA;
      if (rc == PE_OK) {
        if (h->tc_v == 32) tc::k_tc_setup<32><<<grid_for(tp, 256), 256, 0, s2>>>(h->d_m, tp, h->d_tcC, h->d_tcMS, h->mp);
        else tc::k_tc_setup<64><<<grid_for(tp, 256), 256, 0, s2>>>(h->d_m, tp, h->d_tcC, h->d_tcMS, h->mp);
        const u64 nrp = 4 * ((tp + 2 * tc::kKB - 1) / (2 * tc::kKB));   // warp tasks (K-block, K half)
        const unsigned rpg = (unsigned)std::max<u64>(1, std::min<u64>((nrp + 7) / 8, 148ull * 8));
        const bool lazy = h->p >= (1ull << 31) && h->p < (1ull << 62);
        if (h->tc_v == 32 && lazy) tc::k_tc_rplanes<true, 32><<<rpg, tc::kRpThreads, 0, s>>>(h->d_m, tp, h->d_tcR, h->mp);
        else if (h->tc_v == 32) tc::k_tc_rplanes<false, 32><<<rpg, tc::kRpThreads, 0, s>>>(h->d_m, tp, h->d_tcR, h->mp);
        else if (lazy) tc::k_tc_rplanes<true, 64><<<rpg, tc::kRpThreads, 0, s>>>(h->d_m, tp, h->d_tcR, h->mp);
        else tc::k_tc_rplanes<false, 64><<<rpg, tc::kRpThreads, 0, s>>>(h->d_m, tp, h->d_tcR, h->mp);
        if (cudaGetLastError() != cudaSuccess || cudaEventRecord(e_done, s2) != cudaSuccess ||
            cudaStreamWaitEvent(s, e_done, 0) != cudaSuccess)
          rc = PE_ECUDA;
      }
      if (e_m) cudaEventDestroy(e_m);
      if (e_done) cudaEventDestroy(e_done);
      cudaStreamDestroy(s2);
      if (rc != PE_OK) return set_err(rc);
    }
    CU(cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, h->device));
    // 4-byte digits (7 diagonals) and the V = 32 geometry (15 x 32 columns): one round
    h->tc_rounds = (h->p < (1ull << 31) || h->tc_v == 32) ? 1 : tc::kRounds;
    if (int rc = status_get(&h->h_status, &h->d_status)) return set_err(rc);
    h->tc_ok = true;
  }
  // ---- k_step's warp-tile plan (host), computed while the setup kernels above run
  const int W = h->W;
  std::vector<uint2> wt_info(n_wt);
  std::vector<u32> wt_bucket(n_wt), slot_start(G + 1);
  for (u64 g = 0; g < G; ++g)
    for (u64 x = poff[g] / tile; x < poff[g + 1] / tile; ++x) wt_bucket[x] = (u32)g;
  u32 slot = 0;
  for (u64 x = 0; x < n_wt; ++x) {
    bool start = (x % W == 0) || wt_bucket[x] != wt_bucket[x - 1];
    if (start) {
      if (x == 0 || wt_bucket[x] != wt_bucket[x - 1]) slot_start[wt_bucket[x]] = slot;
      u32 len = 1;
      while ((x + len) % W != 0 && x + len < n_wt && wt_bucket[x + len] == wt_bucket[x]) ++len;
      wt_info[x] = make_uint2(slot, len);
      ++slot;
    } else {
      wt_info[x] = make_uint2(slot - 1, 0);
    }
  }
  slot_start[G] = slot;
  h->n_slots = slot;

  CU(cudaMemcpyAsync(h->d_wt_info, wt_info.data(), n_wt * sizeof(uint2), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(h->d_slot_start, slot_start.data(), (G + 1) * sizeof(u32), cudaMemcpyHostToDevice, s));

  // k_tc plans of the common evaluation shapes (8192- or 16384-point passes; all rows, and pe_eval's two
  // row blocks), built on the host while the setup kernels run and uploaded behind them
  if (h->tc_ok) {
    h->split_g1 = tc_row_split(h);
    const u64 ranges[3][2] = {{0, h->G}, {0, h->split_g1}, {h->split_g1, h->G}};
    for (u32 k = 1; k <= 2; ++k)   // passes of 8192 and 16384 points
      for (auto& r : ranges) {
        const u32 nch = k * (8192u / h->tc_chunk);
        if (r[0] >= r[1]) continue;
        pe_ctx::TcPlan* P = nullptr;
        if (tc_plan(h, nch, r[0], r[1], true, s, &P)) return g_last_error;
      }
  }
  if (h->fast_mode == 2) {
    const int rc = fast::create(h->h_poff, h->mp, s, &h->fast);
    if (rc != PE_OK) return set_err(rc);
  }
  prof.mark("tc setup + rplanes", s);
  CU(cudaStreamWaitEvent(s, c_landed, 0));
  k_setup_c<<<grid_for(h->t_pad, 256), 256, 0, s>>>(d_coeffs, h->d_perm, h->t_pad, h->d_c, h->mp.p);
  CU(cudaGetLastError());
  prof.mark("coefficients", s);
  CU(cudaStreamSynchronize(s));  // host vectors above must outlive the copies; tmp frees after
  return PE_OK;
}

template <class E>
static pe_ctx* create_common(uint64_t p, uint32_t npoly, const uint64_t* t_per_poly, uint32_t n,
                             const uint64_t* coeffs, const E* exps, const uint64_t* alpha,
                             const pe_config* cfg) {
  g_last_error = PE_OK;
  // ---- validation before any CUDA call
  if (npoly < 1 || !t_per_poly) { set_err(PE_EINVAL); return nullptr; }
  std::vector<u64> poly_off(npoly + 1, 0);
  for (u32 k = 0; k < npoly; ++k) {
    poly_off[k + 1] = poly_off[k] + t_per_poly[k];
    if (poly_off[k + 1] < poly_off[k]) { set_err(PE_ERANGE); return nullptr; }
  }
  const u64 t = poly_off[npoly];
  if (n < 2 || n > 66) { set_err(PE_EINVAL); return nullptr; }
  if (t > 0x7fffffffull) { set_err(PE_ERANGE); return nullptr; }   // CUB sort / select take int num_items
  if (t > 0 && (!coeffs || !exps)) { set_err(PE_EINVAL); return nullptr; }
  if (n > 2 && !alpha) { set_err(PE_EINVAL); return nullptr; }
  if (p < 3 || p >= (1ull << 63)) { set_err(PE_ERANGE); return nullptr; }
  if (!h_is_prime(p)) { set_err(PE_ENOTPRIME); return nullptr; }
  for (u32 l = 0; l + 2 < n; ++l)
    if (alpha[l] % p == 0) { set_err(PE_ERANGE); return nullptr; }
  int path_req = cfg ? cfg->path : PE_PATH_AUTO;
  if (path_req == PE_PATH_AUTO) {
    const char* e = getenv("PE_PATH");
    if (e && !strcmp(e, "int")) path_req = PE_PATH_INT;
    if (e && !strcmp(e, "fp64")) path_req = PE_PATH_FP64;
  }
  int path;
  if (path_req == PE_PATH_FP64) {
    if (p >= (1ull << 50)) { set_err(PE_ENOTSUP); return nullptr; }
    path = kFp64;
  } else if (path_req == PE_PATH_INT || path_req == PE_PATH_AUTO) {
    // INT64 family: the 32-bit-IMAD Shoup core (lazy-4 for p < 2^62, lazy-2 above)
    const char* core = getenv("PE_CORE");
    path = p < (1ull << 62) ? kInt4 : kInt2;
    if (path_req == PE_PATH_AUTO && p < (1ull << 50) && (!core || !strcmp(core, "auto"))) path = kFp64;
    // p < 2^31: 32-bit Shoup (4 IMAD slots per product instead of 14)
    if (p < (1ull << 31) && (!core || !strcmp(core, "auto") || !strcmp(core, "int32"))) path = kInt32;
    if (core && !strcmp(core, "fp64")) {
      if (p >= (1ull << 50)) { set_err(PE_ENOTSUP); return nullptr; }
      path = kFp64;
    }
  } else if (path_req == PE_PATH_TC) {
    path = p < (1ull << 62) ? kInt4 : kInt2;
  } else if (path_req == PE_PATH_FAST) {
    path = p < (1ull << 62) ? kInt4 : kInt2;
  } else {
    set_err(PE_EINVAL);
    return nullptr;
  }
  // tensor-core path: forced by PE_PATH_TC; automatic (large T) for the INT64 Shoup path when the
  // caller asked for PE_PATH_AUTO; env PE_TC=0|1|2 overrides the automatic choice.
  // (any p < 2^63: the automatic scalar core -- Shoup, FP64 Alg. 2 or 32-bit Shoup -- serves short
  // point ranges, the tensor-core form long ones)
  const bool tc_able = path == kInt4 || path == kInt2 || path == kFp64 || path == kInt32;
  int tc_mode = path_req == PE_PATH_TC ? 2 : (path_req == PE_PATH_AUTO && tc_able ? 1 : 0);
  // fast method: forced by PE_PATH_FAST; automatic (p < 2^62, T >= the measured crossover) unless
  // env PE_FAST=0; PE_FAST=2 forces it for PE_PATH_AUTO handles
  int fast_mode = path_req == PE_PATH_FAST ? 2 : 0;
  if (path_req == PE_PATH_AUTO) {
    const int e = env_int("PE_FAST", 1);
    fast_mode = e <= 0 ? 0 : (e >= 2 ? 2 : 1);
  }
  if (path_req == PE_PATH_AUTO && tc_able) {
    const int e = env_int("PE_TC", 1);
    tc_mode = e < 0 ? 0 : (e > 2 ? 2 : e);
  }
  int R = cfg && cfg->R ? cfg->R : env_int("PE_R", 0);
  int W = cfg && cfg->warps ? cfg->warps : env_int("PE_WARPS", 8);
  int chunk = cfg && cfg->chunk ? cfg->chunk : env_int("PE_CHUNK", 0);
  const int tc_form = cfg ? cfg->tc_form : PE_TC_FORM_AUTO;
  if (W < 1 || W > kMaxWarps || chunk < 0 || chunk % kSuper || tc_form < PE_TC_FORM_AUTO ||
      tc_form > PE_TC_FORM_SWAPPED) {
    set_err(PE_EINVAL);
    return nullptr;
  }
  pe_ctx* h = new (std::nothrow) pe_ctx();
  if (!h) { set_err(PE_ENOMEM); return nullptr; }
  h->p = p; h->t = t; h->n = n;
  h->mp = h_mod_params(p);
  h->path = path;
  h->tc_mode = tc_mode;
  h->fast_mode = fast_mode;
  h->R = R; h->W = W; h->chunk_req = chunk;
  h->tc_form_req = tc_form;
  h->partial_cap_bytes = (size_t)env_int("PE_PARTIAL_MB", 1024) << 20;
  h->poly_off = poly_off;
  h->poly_rows.assign(npoly + 1, 0);
  int rc = create_impl(h, coeffs, exps, alpha);
  if (rc != PE_OK) {
    int e = g_last_error != PE_OK ? g_last_error : rc;
    free_all(h);
    delete h;
    set_err(e);
    return nullptr;
  }
  return h;
}

extern "C" pe_ctx* pe_create_ex(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs,
                                const uint32_t* exps, const uint64_t* alpha, const pe_config* cfg) {
  return create_common(p, 1, &t, n, coeffs, exps, alpha, cfg);
}

extern "C" pe_ctx* pe_create(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs,
                             const uint32_t* exps, const uint64_t* alpha) {
  return pe_create_ex(p, t, n, coeffs, exps, alpha, nullptr);
}

extern "C" pe_ctx* pe_create_batch(uint64_t p, uint32_t npoly, const uint64_t* t_per_poly, uint32_t n,
                                   const uint64_t* coeffs, const uint32_t* exps, const uint64_t* alpha,
                                   const pe_config* cfg) {
  return create_common(p, npoly, t_per_poly, n, coeffs, exps, alpha, cfg);
}

extern "C" pe_ctx* pe_create_compact(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs,
                                     const uint8_t* exps, const uint64_t* alpha, const pe_config* cfg) {
  return create_common(p, 1, &t, n, coeffs, exps, alpha, cfg);
}

extern "C" uint32_t pe_num_polys(const pe_ctx* h) { return h ? (uint32_t)h->poly_off.size() - 1 : 0; }

extern "C" int pe_poly_rows(const pe_ctx* h, uint64_t* row_off) {
  if (!h || !row_off) return set_err(PE_EINVAL);
  memcpy(row_off, h->poly_rows.data(), h->poly_rows.size() * sizeof(u64));
  return PE_OK;
}

extern "C" void pe_destroy(pe_ctx* h) {
  if (!h) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(h->device);
  // the handle's own streams, and the latest work it enqueued on each caller stream; not the
  // whole device, so that destroying a handle does not wait for other handles' (threads') work
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->copy_stream) cudaStreamSynchronize(h->copy_stream);
  for (auto& u : h->used) cudaEventSynchronize(u.second), cudaEventDestroy(u.second);
  h->used.clear();
  free_all(h);
  cudaSetDevice(cur);
  delete h;
}

// ---------------------------------------------------------------- eval
static int ensure_partial(pe_ctx* h, size_t need, cudaStream_t s) {
  if (need > h->partial_elems) {
    if (h->d_partial) cudaFreeAsync(h->d_partial, s);
    h->d_partial = nullptr;
    h->partial_elems = 0;
    CU(cudaMallocAsync((void**)&h->d_partial, need * sizeof(u64), s));
    h->partial_elems = need;
  }
  return PE_OK;
}

// k_tc piece plan for a pass of nch chunks (host part cached per nch; device copies on first use).
// Pieces: each bucket's padded range cut into near-equal runs of whole K-blocks of at most maxkb
// K-blocks -- <= kPieceMax terms keeps every int32 diagonal sum exact (tc.cuh) -- with maxkb chosen
// so the launch has about kUnitsPerCta units (piece, chunk, round) per CTA: enough to balance a
// small launch (a 1/8 term shard of config 5), while a large one keeps the 8192-term maximum.
// Schedule (longest processing time first, by piece): pieces in decreasing size, the nch x rounds
// units of a piece dealt to the currently least-loaded CTAs (cost = K-blocks + ~4 for the unit's
// epilogue and pipeline fill), so the units sharing a piece's baby-step planes sit at the same
// load level of neighbouring CTAs and run side by side (one DRAM read of the planes, L2 for the
// rest -- the round-1 snake order's property).  env PE_TC_PIECE (terms) / PE_TC_UPC override.
static const u32 kUnitsPerCta = 6;
// Largest piece (K-blocks) of a plan for rows [g0, g1) and nch chunks.
static u64 tc_maxkb(const pe_ctx* h, u32 nch, u64 g0, u64 g1) {
  const u64 n_w = (u64)h->n_sm;
  const u64 tkb = (h->h_poff[g1] - h->h_poff[g0]) / tc::kKB;
  const u32 rounds = h->tc_rounds;
  u64 maxkb;
  const int pm_env = env_int("PE_TC_PIECE", 0), upc = env_int("PE_TC_UPC", (int)kUnitsPerCta);
  if (pm_env > 0) {
    maxkb = std::max<u64>(1, (u64)pm_env / tc::kKB);
  } else if (upc <= 0) {   // round-1 rule: pieces of up to twice the per-SM share
    maxkb = 2 * ((h->t_pad + n_w - 1) / n_w) / tc::kKB;
    maxkb = std::max<u64>(maxkb, 1024 / tc::kKB);
  } else {
    maxkb = (tkb * nch * rounds + n_w * upc - 1) / (n_w * upc);
    maxkb = std::max<u64>(maxkb, 1024 / tc::kKB);
  }
  return std::min<u64>(maxkb, tc::kPieceMax / tc::kKB);
}
// Partial rows (pieces x rounds) of that plan, without building it (O(rows)).
static u64 tc_nslots(const pe_ctx* h, u32 nch, u64 g0, u64 g1) {
  const u64 maxkb = tc_maxkb(h, nch, g0, g1);
  u64 n = 0;
  for (u64 g = g0; g < g1; ++g) n += ((h->h_poff[g + 1] - h->h_poff[g]) / tc::kKB + maxkb - 1) / maxkb;
  return n * h->tc_rounds;
}
// Rows [g0, g1) only (pe_eval's row blocks): pieces of those buckets, slots numbered from 0.
static int tc_plan(const pe_ctx* h, u32 nch, u64 g0, u64 g1, bool upload, cudaStream_t s, pe_ctx::TcPlan** out) {
  const auto key = std::make_tuple(nch, g0, g1);
  auto it = h->tc_plans.find(key);
  pe_ctx::TcPlan* P = nullptr;
  if (it == h->tc_plans.end()) {
    P = &h->tc_plans[key];
    const u64 G = g1 - g0;
    const u32 rounds = h->tc_rounds;
    const u64 maxkb = tc_maxkb(h, nch, g0, g1);
    std::vector<u32> slot(G + 1);
    for (u64 gg = 0; gg < G; ++gg) {
      const u64 g = g0 + gg;
      slot[gg] = (u32)P->pieces.size();
      const u64 nkb = (h->h_poff[g + 1] - h->h_poff[g]) / tc::kKB;   // poff multiples of 32R
      const u64 np_g = (nkb + maxkb - 1) / maxkb;
      u64 kb0 = 0;
      for (u64 k = 0; k < np_g; ++k) {
        const u64 len = nkb / np_g + (k < nkb % np_g ? 1 : 0);
        // w = 1 + the bucket's row (relative to g0) for a bucket's sole piece in a one-round geometry:
        // its partial row is already the canonical result, so k_tc may write it to the output row
        // directly (TcArgs::direct) and the fix-up skips that row
        const u32 sole = (np_g == 1 && rounds == 1) ? (u32)(gg + 1) : 0u;
        P->pieces.push_back(make_uint4((u32)(h->h_poff[g] + kb0 * tc::kKB), (u32)len, (u32)P->pieces.size(), sole));
        kb0 += len;
      }
    }
    slot[G] = (u32)P->pieces.size();
    std::stable_sort(P->pieces.begin(), P->pieces.end(), [](const uint4& x, const uint4& y) { return x.y > y.y; });
    // one partial row per (piece, diagonal round): k_tc reduces each round's part on its own
    P->npieces = (u32)P->pieces.size();
    P->nslots = P->npieces * rounds;
    for (auto& x : slot) x *= rounds;
    for (u64 gg = 0; gg < G; ++gg) P->max_slots = std::max(P->max_slots, slot[gg + 1] - slot[gg]);
    P->slot_start = std::move(slot);
    // schedule
    const u32 upp = nch * rounds, nunits = P->npieces * upp;
    const u32 grid = (u32)std::min<u64>(nunits, (u64)h->n_sm);
    P->grid = grid;
    std::vector<std::pair<u64, u32>> heap;   // (load, cta), min-heap
    for (u32 b = 0; b < grid; ++b) heap.push_back({0, b});
    auto cmp = [](const std::pair<u64, u32>& x, const std::pair<u64, u32>& y) {
      return x.first != y.first ? x.first > y.first : x.second > y.second;
    };
    std::make_heap(heap.begin(), heap.end(), cmp);
    // (a) snake: units in piece-major order, row r of `grid` units dealt left to right for even r,
    //     right to left for odd r (the round-1 order: with ~50 units per CTA its makespan is within
    //     0.5 % of the mean and a piece's units start together);
    // (b) LPT by piece (below).  The cost model picks (b) only when it shortens the makespan by > 3 %
    //     -- launches with few units per CTA, e.g. one term shard of a multi-GPU run.
    std::vector<std::vector<u32>> snake(grid), lists(grid);
    std::vector<u64> sload(grid, 0);
    for (u32 u = 0; u < nunits; ++u) {
      const u32 row = u / grid, col = u % grid, b = (row & 1) ? grid - 1 - col : col;
      snake[b].push_back(u);
      sload[b] += (u64)P->pieces[u / upp].y + 4;
    }
    std::vector<std::pair<u64, u32>> took;
    const int sch = env_int("PE_TC_SCHED", -1);   // testing: 0 snake, 1 LPT
    // with >= 16 units per CTA the snake order is already within a few % of the mean: skip LPT
    const bool try_lpt = sch == 1 || (sch < 0 && nunits < 16ull * grid);
    for (u32 pc = 0; try_lpt && pc < P->npieces; ++pc) {   // pieces are size-sorted: LPT order
      const u64 cost = (u64)P->pieces[pc].y + 4;
      took.clear();
      for (u32 k = 0; k < upp; ++k) {
        if (took.size() == grid) {              // more units than CTAs: reuse the least loaded again
          for (auto& x : took) { heap.push_back(x); std::push_heap(heap.begin(), heap.end(), cmp); }
          took.clear();
        }
        std::pop_heap(heap.begin(), heap.end(), cmp);
        auto top = heap.back();
        heap.pop_back();
        lists[top.second].push_back(pc * upp + k);   // unit = (piece * nch + chunk) * rounds + g
        top.first += cost;
        took.push_back(top);
      }
      for (auto& x : took) { heap.push_back(x); std::push_heap(heap.begin(), heap.end(), cmp); }
    }
    u64 lpt_max = 0, snake_max = 0;
    for (auto& x : heap) lpt_max = std::max(lpt_max, x.first);
    for (u64 x : sload) snake_max = std::max(snake_max, x);
    if (!try_lpt || sch == 0 || (sch < 0 && !(lpt_max * 100 < snake_max * 97))) lists.swap(snake);
    P->sched.assign(nunits + grid + 1, 0);
    u32 o = 0;
    for (u32 b = 0; b < grid; ++b) {
      P->sched[nunits + b] = o;
      for (u32 u : lists[b]) P->sched[o++] = u;
    }
    P->sched[nunits + grid] = o;
  } else {
    P = &it->second;
  }
  if (upload && !P->d_piece) {
    CU(cudaMallocAsync((void**)&P->d_piece, std::max<size_t>(1, P->pieces.size()) * sizeof(uint4), s));
    CU(cudaMallocAsync((void**)&P->d_slot_start, P->slot_start.size() * sizeof(u32), s));
    CU(cudaMallocAsync((void**)&P->d_sched, P->sched.size() * sizeof(u32), s));
    CU(cudaMemcpyAsync(P->d_piece, P->pieces.data(), P->pieces.size() * sizeof(uint4), cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(P->d_slot_start, P->slot_start.data(), P->slot_start.size() * sizeof(u32),
                       cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(P->d_sched, P->sched.data(), P->sched.size() * sizeof(u32), cudaMemcpyHostToDevice, s));
    // (pageable sources: each copy has left the host vector when it returns; the plan's host
    // vectors also live on in the cache.)  Later launches on any stream wait on this event.
    CU(cudaEventCreateWithFlags(&P->uploaded, cudaEventDisableTiming));
    CU(cudaEventRecord(P->uploaded, s));
  }
  *out = P;
  return PE_OK;
}

// Tensor-core evaluation (tc.cuh): per pass, chunk seeds -> k_tc (persistent, one CTA per SM)
// -> k_fixup over the pieces' partial rows.
// Rows [g0, g1) of the output (default: all): out row g is d_out + g * ld.
static int eval_tc(pe_ctx* h, u64 j0, u64 T, u64* d_out, u64 ld, cudaStream_t s, u64 g0 = 0, u64 g1 = ~0ull) {
  if (g1 > h->G) g1 = h->G;
  if (g0 >= g1) return PE_OK;
  const u64 q0 = h->h_poff[g0], q1 = h->h_poff[g1];   // the rows' padded terms
  // pass length from the one-chunk plan: it has the most pieces (plans with more chunks per pass
  // use larger pieces), so its slot count bounds every pass's partial rows
  const u64 nslots = tc_nslots(h, 1, g0, g1);
  const u64 CH = h->tc_chunk;   // points per chunk of the handle's geometry
  u64 Tp = h->partial_cap_bytes / 8 / std::max<u64>(nslots, 1) / CH * CH;
  Tp = std::max<u64>(Tp, CH);
  Tp = std::min<u64>(Tp, (T + CH - 1) / CH * CH);
  Tp = std::min<u64>(Tp, CH * 4096);
  // every allocation of the evaluation comes before its first launch, so an automatic handle can
  // still fall back to k_step on PE_ENOMEM (eval_device_impl)
  // partial rows padded to a multiple of 8 points (the epilogue's 64-byte vector accesses)
  if (ensure_partial(h, (size_t)nslots * ((std::min<u64>(Tp, T) + 7) / 8 * 8), s)) return g_last_error;
  const u32 nch_max = (u32)(Tp / CH);
  if ((size_t)h->t_pad * nch_max * tc::kLSRec > h->seed_elems) {
    if (h->d_seed) cudaFreeAsync(h->d_seed, s);
    h->d_seed = nullptr;
    h->seed_elems = 0;
    CU(cudaMallocAsync((void**)&h->d_seed, (size_t)h->t_pad * nch_max * tc::kLSRec * sizeof(u64), s));
    h->seed_elems = (size_t)h->t_pad * nch_max * tc::kLSRec;
  }
  if (!h->d_tc_scratch) CU(cudaMallocAsync((void**)&h->d_tc_scratch, (size_t)h->n_sm * 2 * tc::kDiag * tc::kChunk * sizeof(u32), s));
  u32* d_status = h->d_status;
  // kernel mode: 0 = lazy chains, 8 digits; 1 = p >= 2^62, exact chains, 8 digits; 2 = p < 2^31,
  // exact chains (values < 2^32), 4 digits, one round
  // 3 = 2^31 <= p < 2^54: lazy chains (values < 2^56), 7 digits, one round of 7 MMAs (V = 32)
  // 4 / 5: the swapped forms of 0 / 1 (giant-step planes per handle, baby steps generated)
  int mode = h->p < (1ull << 31) ? 2 : h->p < (1ull << 54) ? 3 : (h->p >= (1ull << 62) ? 1 : 0);
  if (h->tc_swap) mode = mode == 3 ? 6 : mode + 4;   // 6: the swapped 7-digit mode
  // k_tc's units are scheduled statically over its persistent CTAs, so every CTA must own its SM:
  // it asks for the whole of the SM's shared memory (default; PE_TC_EXCLUSIVE=0: only what it
  // uses), which keeps a concurrent kernel of another stream (e.g. a pe_create running beside this
  // evaluation) from co-residing with one of its CTAs and making that CTA the launch's straggler
  const void* tc_fns[9] = {(const void*)tc::k_tc<false, 6>, (const void*)tc::k_tc<false, 0>, (const void*)tc::k_tc<false, 1>,
                           (const void*)tc::k_tc<false, 2>, (const void*)tc::k_tc<false, 3>,
                           (const void*)tc::k_tc<false, 4>, (const void*)tc::k_tc<false, 5>,
                           (const void*)tc::k_tc<true, 0>, (const void*)tc::k_tc<true, 4>};
  static thread_local int smem_dev = -1, smem_dyn = 0;
  if (smem_dev != h->device) {
    int optin = 0;
    CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    size_t st = 0;
    for (const void* f : tc_fns) {
      cudaFuncAttributes fa;
      CU(cudaFuncGetAttributes(&fa, f));
      st = std::max(st, fa.sharedSizeBytes);
    }
    smem_dyn = std::max<int>((int)tc::kSmemBytes, optin - (int)st);
    smem_dev = h->device;
  }
  const int tc_smem = env_int("PE_TC_EXCLUSIVE", 1) ? smem_dyn : (int)tc::kSmemBytes;
  for (const void* f : tc_fns) CU(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem));
  for (u64 k0 = 0; k0 < T; k0 += Tp) {
    const u32 np = (u32)std::min<u64>(Tp, T - k0);
    const u32 nch = (u32)((np + CH - 1) / CH);
    const u64 nseed = (q1 - q0) * ((nch + tc::kSeedChunks - 1) / tc::kSeedChunks);
    tc::k_tc_seed<<<grid_for(nseed, 256), 256, 0, s>>>(h->d_c, h->d_m, h->d_tcMS, h->t_pad, q0, q1, nch, (u32)CH,
                                                       j0 + k0, h->d_seed, h->mp);
    CU(cudaGetLastError());
    pe_ctx::TcPlan* P = nullptr;
    if (tc_plan(h, nch, g0, g1, true, s, &P)) return g_last_error;
    CU(cudaStreamWaitEvent(s, P->uploaded, 0));
    tc::TcArgs a;
    a.LS = h->d_seed;
    a.C = h->d_tcC;
    a.Rp = h->tc_swap ? nullptr : h->d_tcR;
    a.Gp = h->tc_swap ? h->d_tcR : nullptr;
    a.piece = P->d_piece;
    a.partial = h->d_partial;
    a.ldp = (np + 7) / 8 * 8;
    // sole-piece rows straight into the output when its rows keep the epilogue's 16-B stores aligned
    a.out = d_out + g0 * ld + k0;
    a.ldo = ld;
    a.direct = (env_int("PE_TC_DIRECT", 1) && ld % 2 == 0 && ((uintptr_t)a.out & 15) == 0) ? 1 : 0;
    a.t_pad = h->t_pad;
    a.npieces = P->npieces;
    a.rounds = h->tc_rounds;
    a.nunits = P->npieces * nch * a.rounds;
    a.nch = nch;
    a.npts = np;
    for (int d = 0; d < 15; ++d) a.Wd[d] = h_powmod(2, 8 * (u64)d, h->p);
    a.C128 = h_powmod(2, 128, h->p);
    a.scratch = h->d_tc_scratch;
    a.mp = h->mp;
    a.status = d_status;
    a.discard = env_int("PE_TC_DISCARD", 1);
    a.sleep_ns[0] = 32; a.sleep_ns[1] = 64; a.sleep_ns[2] = 64;
    if (const char* e = getenv("PE_TC_SLEEP")) {
      unsigned x, y, z;
      if (sscanf(e, "%u,%u,%u", &x, &y, &z) == 3) { a.sleep_ns[0] = x; a.sleep_ns[1] = y; a.sleep_ns[2] = z; }
    }
    a.prof = nullptr;
    a.dbg = env_int("PE_TC_DEBUG", 0);
    const unsigned grid = P->grid;
    a.sched = P->d_sched;
    a.sched_off = P->d_sched + a.nunits;
    pe_ctx::Rec rec{};
    if (h->timing) {
      CU(cudaEventCreate(&rec.e0));
      CU(cudaEventCreate(&rec.e1));
      CU(cudaEventCreate(&rec.e2));
      rec.tp = (double)h->t_pad * np;
      CU(cudaEventRecord(rec.e0, s));
    }
    unsigned long long* d_prof = nullptr;
    const size_t nprof = (size_t)grid * (tc::kThreads / 32) * 5 + (size_t)grid * 3;
    a.prof = nullptr;
    if (env_int("PE_TC_PROF", 0)) {   // development: per-warp phase timers printed to stderr
      CU(cudaMalloc(&d_prof, nprof * sizeof(unsigned long long)));
      CU(cudaMemset(d_prof, 0, nprof * sizeof(unsigned long long)));
      a.prof = d_prof;
    }
    if (d_prof && mode == 0) tc::k_tc<true, 0><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else if (d_prof && mode == 4) tc::k_tc<true, 4><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else if (mode == 4) tc::k_tc<false, 4><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else if (mode == 5) tc::k_tc<false, 5><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else if (mode == 6) tc::k_tc<false, 6><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else if (mode == 1) tc::k_tc<false, 1><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else if (mode == 2) tc::k_tc<false, 2><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else if (mode == 3) tc::k_tc<false, 3><<<grid, tc::kThreads, tc_smem, s>>>(a);
    else tc::k_tc<false, 0><<<grid, tc::kThreads, tc_smem, s>>>(a);
    CU(cudaGetLastError());
    if (d_prof) {
      std::vector<unsigned long long> hp(nprof);
      CU(cudaMemcpyAsync(hp.data(), d_prof, nprof * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      cudaFree(d_prof);
      const int nw = tc::kThreads / 32;
      for (int wv = 0; wv < nw; ++wv) {
        double acc[5] = {0, 0, 0, 0, 0};
        for (unsigned b = 0; b < grid; ++b)
          for (int i = 0; i < 5; ++i) acc[i] += (double)hp[((size_t)b * nw + wv) * 5 + i] / grid;
        fprintf(stderr, "tcprof warp %2d: t0 %.0f t1 %.0f t2 %.0f n %.0f total %.0f\n", wv, acc[0], acc[1], acc[2],
                acc[3], acc[4]);
      }
      const unsigned long long* gt = hp.data() + (size_t)grid * nw * 5;
      unsigned long long e0 = ~0ull, e1 = 0, a0 = ~0ull, a1 = 0, x0 = ~0ull, x1 = 0;
      for (unsigned b = 0; b < grid; ++b) {
        e0 = std::min(e0, gt[3 * b]); e1 = std::max(e1, gt[3 * b]);
        a0 = std::min(a0, gt[3 * b + 1]); a1 = std::max(a1, gt[3 * b + 1]);
        x0 = std::min(x0, gt[3 * b + 2]); x1 = std::max(x1, gt[3 * b + 2]);
      }
      fprintf(stderr, "tcprof wall us: entry %.1f..%.1f  alloc-done %.1f..%.1f  exit %.1f..%.1f\n", 0.0,
              (e1 - e0) / 1e3, (a0 - e0) / 1e3, (a1 - e0) / 1e3, (x0 - e0) / 1e3, (x1 - e0) / 1e3);
    }
    if (h->timing) CU(cudaEventRecord(rec.e1, s));
    const u32 nkb = (np + 255) / 256;
    // few rows of many pieces (a term shard holding one huge bucket): the thread-per-point kernel
    // would leave most SMs idle, so split each row's slots over 8 warps instead
    if (P->max_slots >= 16 && (g1 - g0) * nkb < 8ull * h->n_sm) {
      const u32 nkw = (np + 31) / 32;
      k_fixup_wide<<<(unsigned)((g1 - g0) * nkw), 256, 0, s>>>(h->d_partial, a.ldp, P->d_slot_start, (u32)(g1 - g0),
                                                               np, nkw, d_out + g0 * ld + k0, ld, h->mp, a.direct);
    } else {
      k_fixup<<<(unsigned)((g1 - g0) * nkb), 256, 0, s>>>(h->d_partial, a.ldp, P->d_slot_start, (u32)(g1 - g0), np,
                                                          nkb, d_out + g0 * ld + k0, ld, h->mp, a.direct);
    }
    CU(cudaGetLastError());
    if (h->timing) {
      CU(cudaEventRecord(rec.e2, s));
      h->recs.push_back(rec);
    }
  }
  return PE_OK;
}

// Tensor-core form for this T?  Forced handles always; automatic ones from the measured threshold,
// and only while one chunk's partial rows (one per piece and diagonal round, T_pass >= one chunk)
// fit the partial-buffer cap -- a handle with very many buckets stays on k_step, whose partial
// rows are per CTA run and need far less.
static bool use_tc(const pe_ctx* h, u64 T) {
  if (!h->tc_ok) return false;
  if (h->tc_mode == 2) return true;
  if (h->tc_mode != 1 || T < tc_min_T(h->t_pad, h->p)) return false;
  const u64 row = (std::min<u64>(T, h->tc_chunk) + 7) / 8 * 8;
  return tc_nslots(h, 1, 0, h->G) * row * sizeof(u64) <= h->partial_cap_bytes;
}

// automatic fast-method threshold: the measured crossover against k_tc (fast method)
static u64 fast_min_T(const pe_ctx* h) {
  (void)h;
  const int e = env_int("PE_FAST_MIN_T", 0);
  return e > 0 ? (u64)e : kFastMinT;
}
// Automatic choice: the fast method beats the scalar matrix method (k_step) from T ~ kFastMinT on,
// but never the tensor-core form within its supported T (profiles/r02_fast_sweep*.jsonl, DESIGN.md
// §7), so an automatic handle takes it only when its tensor-core form is off (PE_TC=0, or it
// degraded for lack of memory).
static bool use_fast(const pe_ctx* h, u64 T) {
  if (h->fast_mode == 2) return true;
  return h->fast_mode == 1 && !h->tc_ok && T >= fast_min_T(h) && T <= fast::kTMax &&
         h->t >= kFastMinTermsPerBucket * h->G;
}
enum { kKStep = 0, kKTc = 1, kKFast = 2 };
static int choose_kernel(const pe_ctx* h, u64 T) {
  if (use_fast(h, T)) return kKFast;
  return use_tc(h, T) ? kKTc : kKStep;
}

static int eval_fast(pe_ctx* h, u64 j0, u64 T, u64* d_out, u64 ld, cudaStream_t s) {
  if (!h->fast) {
    const int rc = fast::create(h->h_poff, h->mp, s, &h->fast);
    if (rc != PE_OK) return set_err(rc);
  }
  pe_ctx::Rec rec{};
  if (h->timing) {
    CU(cudaEventCreate(&rec.e0));
    CU(cudaEventCreate(&rec.e1));
    CU(cudaEventCreate(&rec.e2));
    rec.tp = (double)h->t_pad * T;
    CU(cudaEventRecord(rec.e0, s));
  }
  const int rc = fast::eval(h->fast, h->d_c, h->d_m, h->mp, j0, T, d_out, ld, s);
  if (rc != PE_OK) return set_err(rc);
  if (h->timing) {
    CU(cudaEventRecord(rec.e1, s));
    CU(cudaEventRecord(rec.e2, s));
    h->recs.push_back(rec);
  }
  return PE_OK;
}

static int eval_device_impl(pe_ctx* h, u64 j0, u64 T, u64* d_out, u64 ld, cudaStream_t s) {
  if (T == 0 || h->G == 0) return PE_OK;
  if (choose_kernel(h, T) == kKFast) {
    const int rc = eval_fast(h, j0, T, d_out, ld, s);
    if (rc != PE_ENOMEM || h->fast_mode == 2) return rc;
    cudaGetLastError();            // automatic handle: degrade to the matrix method
    g_last_error = PE_OK;
  }
  if (use_tc(h, T)) {
    const int rc = eval_tc(h, j0, T, d_out, ld, s);
    if (rc != PE_ENOMEM || h->tc_mode == 2) return rc;
    // automatic handle and the evaluation's scratch does not fit: degrade to k_step
    cudaGetLastError();
    g_last_error = PE_OK;
  }
  const u64 nslots = h->n_slots;
  // pass size bounded by the partial-buffer cap
  u64 Tp = std::max<u64>(kSuper, h->partial_cap_bytes / 8 / std::max<u64>(nslots, 1));
  Tp = std::min<u64>(Tp, T);
  Tp = std::min<u64>(Tp, 1u << 30);
  if (ensure_partial(h, (size_t)nslots * Tp, s)) return g_last_error;
  const int W = h->W;
  const u32 n_cta = (h->n_wt + W - 1) / W;
  for (u64 k0 = 0; k0 < T; k0 += Tp) {
    const u32 np = (u32)std::min<u64>(Tp, T - k0);
    u32 chunk = (u32)h->chunk_req;
    if (chunk == 0) {
      // cover the SMs: aim for >= 148 * 2 * 4 CTAs, but keep chunks long (seeding cost
      // ~ 2 log2(j) Montgomery products per term per chunk)
      // >= ~32 waves of 2 CTAs/SM keeps the last-wave tail small (config 5: 2 chunks, -1%);
      // chunks stay >= 1024 points so the seed (~2 log2 j Montgomery products) is amortised
      const u64 target = 148ull * 2 * 32;
      u64 nch = std::max<u64>(1, (target + n_cta - 1) / n_cta);
      nch = std::min<u64>(nch, std::max<u64>(1, np / 1024));
      chunk = (u32)((np + nch - 1) / nch);
      chunk = (chunk + kSuper - 1) / kSuper * kSuper;
    }
    StepArgs a;
    a.c = h->d_c; a.m = h->d_m; a.w = h->d_w; a.wt_info = h->d_wt_info;
    a.partial = h->d_partial; a.ldp = np; a.js0 = j0 + k0; a.n_wt = h->n_wt; a.npts = np;
    a.chunk = chunk; a.mp = h->mp;
    dim3 grid(n_cta, (np + chunk - 1) / chunk), block(32 * W);
    pe_ctx::Rec rec{};
    if (h->timing) {
      CU(cudaEventCreate(&rec.e0));
      CU(cudaEventCreate(&rec.e1));
      CU(cudaEventCreate(&rec.e2));
      rec.tp = (double)h->t_pad * np;
      CU(cudaEventRecord(rec.e0, s));
    }
    cudaError_t e = launch_step(h->path, h->R, grid, block, s, a);
    if (e != cudaSuccess) return set_err(PE_ECUDA);
    if (h->timing) CU(cudaEventRecord(rec.e1, s));
    const u32 nkb = (np + 255) / 256;
    k_fixup<<<(unsigned)(h->G * nkb), 256, 0, s>>>(h->d_partial, np, h->d_slot_start, (u32)h->G, np, nkb,
                                                   d_out + k0, ld, h->mp, 0);
    CU(cudaGetLastError());
    if (h->timing) {
      CU(cudaEventRecord(rec.e2, s));
      h->recs.push_back(rec);
    }
  }
  return PE_OK;
}

// A k_tc pipeline wait that timed out (bounded waits) leaves the handle's status
// word set; every later call on the handle reports PE_ECUDA.
static bool tc_failed(const pe_ctx* h) { return h->h_status && *(volatile u32*)h->h_status != 0; }

extern "C" int pe_eval_device(pe_ctx* h, uint64_t j0, uint64_t T, uint64_t* d_out, uint64_t ld,
                              void* stream) {
  g_last_error = PE_OK;
  if (!h) return set_err(PE_EINVAL);
  if (T && j0 + (T - 1) < j0) return set_err(PE_ERANGE);
  if (T && h->G && (!d_out || ld < T)) return set_err(PE_EINVAL);
  if (tc_failed(h)) return set_err(PE_ECUDA);
  int cur = 0;
  CU(cudaGetDevice(&cur));
  if (cur != h->device) CU(cudaSetDevice(h->device));   // kernels and stream-ordered allocations go to the handle's device
  int rc = eval_device_impl(h, j0, T, d_out, ld, (cudaStream_t)stream);
  if (note_use(h, (cudaStream_t)stream) != PE_OK && rc == PE_OK) rc = set_err(PE_ECUDA);
  if (cur != h->device) cudaSetDevice(cur);
  return rc;
}

extern "C" int pe_eval_device_rows(pe_ctx* h, uint64_t j0, uint64_t T, uint64_t g0, uint64_t g1, uint64_t* d_out,
                                   uint64_t ld, void* stream) {
  g_last_error = PE_OK;
  if (!h) return set_err(PE_EINVAL);
  if (g0 == 0 && g1 == h->G) return pe_eval_device(h, j0, T, d_out, ld, stream);
  if (g0 > g1 || g1 > h->G) return set_err(PE_EINVAL);
  if (T && j0 + (T - 1) < j0) return set_err(PE_ERANGE);
  if (T == 0 || g0 == g1) return PE_OK;
  if (!d_out || ld < T) return set_err(PE_EINVAL);
  if (choose_kernel(h, T) != kKTc) return set_err(PE_ENOTSUP);   // row ranges: tensor-core path only
  if (tc_failed(h)) return set_err(PE_ECUDA);
  int cur = 0;
  CU(cudaGetDevice(&cur));
  if (cur != h->device) CU(cudaSetDevice(h->device));
  int rc = eval_tc(h, j0, T, d_out, ld, (cudaStream_t)stream, g0, g1);
  if (note_use(h, (cudaStream_t)stream) != PE_OK && rc == PE_OK) rc = set_err(PE_ECUDA);
  if (cur != h->device) cudaSetDevice(cur);
  return rc;
}

extern "C" uint64_t pe_row_split(const pe_ctx* h) { return h && h->tc_ok ? h->split_g1 : 0; }

extern "C" int pe_eval(pe_ctx* h, uint64_t j0, uint64_t T, uint64_t* out) {
  g_last_error = PE_OK;
  if (!h) return set_err(PE_EINVAL);
  if (T && j0 + (T - 1) < j0) return set_err(PE_ERANGE);
  if (T == 0 || h->G == 0) return PE_OK;
  if (!out) return set_err(PE_EINVAL);
  int cur = 0;
  CU(cudaGetDevice(&cur));
  if (cur != h->device) CU(cudaSetDevice(h->device));
  const size_t need = (size_t)h->G * T;
  int rc = PE_OK;
  if (need > h->out_scratch_elems) {
    if (h->d_out_scratch) cudaFreeAsync(h->d_out_scratch, h->stream);
    h->d_out_scratch = nullptr;
    h->out_scratch_elems = 0;
    if (cudaMallocAsync((void**)&h->d_out_scratch, need * sizeof(u64), h->stream) != cudaSuccess)
      rc = set_err(PE_ENOMEM);
    else h->out_scratch_elems = need;
  }
  // Tensor-core path: two ROW blocks [0, G1) and [G1, G) over all T points (tc_row_split) -- each
  // launch keeps whole chunks -- with the first block's device->host copy (contiguous rows)
  // overlapping the second's evaluation.
  const u64 G1 = rc == PE_OK && choose_kernel(h, T) == kKTc ? h->split_g1 : 0;
  bool done = false;
  if (G1) {
    if (!h->copy_stream && cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
      rc = set_err(PE_ECUDA);
    if (rc == PE_OK && !h->copy_done && cudaEventCreateWithFlags(&h->copy_done, cudaEventDisableTiming) != cudaSuccess)
      rc = set_err(PE_ECUDA);
    const u64 blk[2][2] = {{0, G1}, {G1, h->G}};
    int b = 0;
    for (; b < 2 && rc == PE_OK; ++b) {
      rc = eval_tc(h, j0, T, h->d_out_scratch, T, h->stream, blk[b][0], blk[b][1]);
      if (rc != PE_OK) break;
      if (cudaEventRecord(h->copy_done, h->stream) != cudaSuccess ||
          cudaStreamWaitEvent(h->copy_stream, h->copy_done, 0) != cudaSuccess ||
          cudaMemcpyAsync(out + blk[b][0] * T, h->d_out_scratch + blk[b][0] * T, (blk[b][1] - blk[b][0]) * T * sizeof(u64),
                          cudaMemcpyDeviceToHost, h->copy_stream) != cudaSuccess)
        rc = set_err(PE_ECUDA);
    }
    if (cudaStreamSynchronize(h->copy_stream) != cudaSuccess || cudaStreamSynchronize(h->stream) != cudaSuccess)
      if (rc == PE_OK) rc = set_err(PE_ECUDA);
    done = rc == PE_OK;
    if (rc == PE_ENOMEM && b == 0 && h->tc_mode != 2) {   // automatic handle short of memory: whole path
      cudaGetLastError();
      rc = g_last_error = PE_OK;
    }
  }
  if (!done && rc == PE_OK) {
    rc = eval_device_impl(h, j0, T, h->d_out_scratch, T, h->stream);
    if (rc == PE_OK) {
      if (cudaMemcpyAsync(out, h->d_out_scratch, need * sizeof(u64), cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
          cudaStreamSynchronize(h->stream) != cudaSuccess)
        rc = set_err(PE_ECUDA);
    }
  }
  if (rc == PE_OK && tc_failed(h)) rc = set_err(PE_ECUDA);
  if (cur != h->device) cudaSetDevice(cur);
  return rc;
}

// ---------------------------------------------------------------- introspection
extern "C" uint64_t pe_num_buckets(const pe_ctx* h) { return h ? h->G : 0; }

extern "C" int pe_bucket_exps(const pe_ctx* h, uint32_t* dxdy) {
  if (!h || (h->G && !dxdy)) return set_err(PE_EINVAL);
  if (h->G) memcpy(dxdy, h->dxdy.data(), 2 * h->G * sizeof(u32));
  return PE_OK;
}

extern "C" int pe_info(const pe_ctx* h, int32_t* path, int32_t* R, int32_t* warps, uint64_t* t_padded,
                       uint64_t* n_slots) {
  if (!h) return set_err(PE_EINVAL);
  if (path)
    *path = h->path == kFp64 ? PE_PATH_FP64 : h->path == kInt32 ? PE_PATH_INT32 : PE_PATH_INT;
  if (R) *R = h->R;
  if (warps) *warps = h->W;
  if (t_padded) *t_padded = h->t_pad;
  if (n_slots) *n_slots = h->n_slots;
  return PE_OK;
}

extern "C" int pe_tc_info(const pe_ctx* h, int32_t* mode, uint64_t* pieces, uint64_t* min_T) {
  if (!h) return set_err(PE_EINVAL);
  if (mode) *mode = h->tc_ok ? h->tc_mode : 0;
  if (pieces) {
    *pieces = h->tc_ok ? tc_nslots(h, 1, 0, h->G) / h->tc_rounds : 0;
  }
  if (min_T) *min_T = h->tc_ok ? (h->tc_mode == 2 ? 1 : tc_min_T(h->t_pad, h->p)) : 0;
  return PE_OK;
}

extern "C" int pe_tc_form(const pe_ctx* h) {
  if (!h) return set_err(PE_EINVAL);
  return h->tc_ok ? (h->tc_swap ? PE_TC_FORM_SWAPPED : PE_TC_FORM_PLAIN) : 0;
}

extern "C" int pe_eval_kernel(const pe_ctx* h, uint64_t T) {
  if (!h) return set_err(PE_EINVAL);
  return choose_kernel(h, T);
}

extern "C" int pe_monomials(const pe_ctx* h, uint64_t* m) {
  if (!h || (h->t && !m)) return set_err(PE_EINVAL);
  if (h->t == 0) return PE_OK;
  u64* d;
  CU(cudaMallocAsync((void**)&d, h->t * sizeof(u64), h->stream));
  k_scatter_m<<<grid_for(h->t_pad, 256), 256, 0, h->stream>>>(h->d_m, h->d_perm, h->t_pad, d);
  cudaError_t e = cudaMemcpyAsync(m, d, h->t * sizeof(u64), cudaMemcpyDeviceToHost, h->stream);
  cudaFreeAsync(d, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return set_err(PE_ECUDA);
  return PE_OK;
}

extern "C" int pe_set_timing(pe_ctx* h, int enable) {
  if (!h) return set_err(PE_EINVAL);
  h->timing = enable != 0;
  return PE_OK;
}

extern "C" int pe_kernel_stats(pe_ctx* h, uint64_t* step_launches, double* step_ms, double* fixup_ms,
                               double* term_points) {
  if (!h) return set_err(PE_EINVAL);
  double s_ms = 0, f_ms = 0, tp = 0;
  for (auto& r : h->recs) {
    float a = 0, b = 0;
    if (cudaEventSynchronize(r.e2) != cudaSuccess || cudaEventElapsedTime(&a, r.e0, r.e1) != cudaSuccess ||
        cudaEventElapsedTime(&b, r.e1, r.e2) != cudaSuccess)
      return set_err(PE_ECUDA);
    s_ms += a;
    f_ms += b;
    tp += r.tp;
  }
  if (step_launches) *step_launches = h->recs.size();
  if (step_ms) *step_ms = s_ms;
  if (fixup_ms) *fixup_ms = f_ms;
  if (term_points) *term_points = tp;
  drop_recs(h);
  return PE_OK;
}

// ---------------------------------------------------------------- multi-GPU assembly
extern "C" int pe_rows_addmod(uint64_t p, uint64_t* d_dst, uint64_t ld_dst, const uint64_t* d_src, uint64_t ld_src,
                              uint64_t rows, uint64_t cols, void* stream) {
  g_last_error = PE_OK;
  if (p < 3 || p >= (1ull << 63)) return set_err(PE_ERANGE);
  if (rows == 0 || cols == 0) return PE_OK;
  if (!d_dst || !d_src || ld_dst < cols || ld_src < cols) return set_err(PE_EINVAL);
  k_rows_addmod<<<grid_for(rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(d_dst, ld_dst, d_src, ld_src, rows,
                                                                            cols, p);
  CU(cudaGetLastError());
  return PE_OK;
}

extern "C" int pe_unshard_columns(uint64_t* d_out, uint64_t ld, const uint64_t* d_blocks, uint64_t P, uint64_t G,
                                  uint64_t Tr, uint64_t T, void* stream) {
  g_last_error = PE_OK;
  if (G == 0 || T == 0 || P == 0) return PE_OK;
  if (!d_out || !d_blocks || ld < T || Tr == 0 || P * Tr < T) return set_err(PE_EINVAL);
  for (u64 r = 0; r < P && r * Tr < T; ++r) {
    const u64 cnt = std::min<u64>(Tr, T - r * Tr);
    CU(cudaMemcpy2DAsync(d_out + r * Tr, ld * sizeof(u64), d_blocks + r * G * Tr, Tr * sizeof(u64),
                         cnt * sizeof(u64), G, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  }
  return PE_OK;
}

extern "C" int pe_last_error(void) { return g_last_error; }

extern "C" const char* pe_strerror(int code) {
  switch (code) {
    case PE_OK: return "ok";
    case PE_EINVAL: return "invalid argument";
    case PE_ENOTPRIME: return "p is not prime";
    case PE_ERANGE: return "value out of range";
    case PE_ENOMEM: return "out of memory";
    case PE_ECUDA: return "CUDA error";
    case PE_ENOTSUP: return "not supported for this p";
    default: return "unknown error";
  }
}

extern "C" int pe_interp_bound_ok(uint64_t p, uint64_t t) {
  u128 b = (u128)100 * t * t;
  return (u128)p > b ? 1 : 0;
}
