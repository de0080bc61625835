/*
 * pe_test.h -- C ABI of libpe.so's modular-core probes and roofline microbenchmarks.
 * Used by tests (pin P12: core vs __int128 on the host) and bench.py (the mulmod roofline,
 * SURVEY.md §8(d) "K5").  Not part of the evaluation path.
 */
#ifndef PE_TEST_H_
#define PE_TEST_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Core variants (see csrc/modcore.cuh). */
enum {
  PE_CORE_SHOUP4 = 0,  /* Shoup lazy [0,4p), p < 2^62; probe canonicalises the output       */
  PE_CORE_SHOUP2 = 1,  /* Shoup exact quotient, [0,2p), p < 2^63; probe canonicalises        */
  PE_CORE_MONT = 2,    /* Montgomery mulmod (a*b mod p via two REDCs), p < 2^63               */
  PE_CORE_FP64 = 3,    /* Alg. 2, p < 2^50, a,b < p                        */
  PE_CORE_FP64ADD = 4, /* Alg. 3, p < 2^50, a,b < p                        */
  PE_CORE_POW = 5,     /* a * b^e mod p via Montgomery square-and-multiply: e = extra[i]      */
  PE_CORE_SHOUP4RAW = 6, /* raw lazy output of SHOUP4 (must be < 4p and == a*b mod p)         */
  PE_CORE_HYB = 7,       /* hybrid FP64-quotient product, p < 2^63; probe canonicalises        */
  PE_CORE_HYBRAW = 8,    /* raw output of HYB (must be in (0, 2p) and == a*b mod p)            */
  PE_CORE_SHOUPW = 9     /* shoup_w_fast(b) XOR shoup_w(b): 0 iff the Montgomery form of the Shoup
                            constant floor(b 2^64 / p) agrees with the bit-loop division       */
};

/*
 * pe_test_core -- out[i] = core(a[i], b[i]) for i < N (HOST arrays; extra may be NULL unless
 * PE_CORE_POW).  Lazy variants take any a < 2^64 and b < p.  Returns PE_OK or a PE_E* code
 * (PE_ENOTSUP if p is out of the variant's range).  Synchronous.
 */
int pe_test_core(int variant, uint64_t p, uint64_t N, const uint64_t* a, const uint64_t* b,
                 const uint64_t* extra, uint64_t* out);

/*
 * pe_bench_core -- register-resident throughput of one step of the hot loop (acc += a;
 * a <- a*m), no memory traffic: blocks x threads threads, each with R independent chains,
 * `iters` steps.  Writes device time (ms) and the number of term-point steps executed.
 * variant: PE_CORE_SHOUP4 / PE_CORE_SHOUP2 / PE_CORE_FP64, or 10 = bare IMAD.WIDE chain,
 * 11 = bare IMAD (lo) chain, 12 = bare DFMA chain, 13 = IMAD.HI chain, 14 = IADD3 chain
 * (ops counted as "steps" = one instruction per chain per iteration).
 * Returns PE_OK / PE_ECUDA / PE_EINVAL.
 */
int pe_bench_core(int variant, uint64_t p, int R, int blocks, int threads, int iters,
                  float* ms, double* steps, double* cycles);
/* cycles: mean over blocks of the SM-clock cycles (clock64) the block ran; ms: CUDA-event
 * device time of the launch. */

/*
 * pe_bench_mma -- int8 tensor-core issue rate: one CTA per SM issues `iters` tcgen05.mma
 * kind::i8 (u8 x u8 -> s32, M = 128, N = 16, 32, 64 or 128, K = 32) from a fixed shared-memory tile
 * (the k_tc MMA shape, csrc/tc.cuh).  Writes the CUDA-event device time of the launch (ms) and
 * the multiply-accumulates executed.  Returns PE_OK / PE_EINVAL / PE_ECUDA.  Synchronous.
 */
int pe_bench_mma(int N, int iters, float* ms, double* macs);

#ifdef __cplusplus
}
#endif
#endif /* PE_TEST_H_ */
