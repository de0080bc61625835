/*
 * pe.h -- C ABI of the B200 partial-evaluation library (libpe.so).
 *
 * Computes T bivariate images of a sparse n-variate polynomial modulo a prime p at the
 * points beta^j = (alpha_1^j, ..., alpha_{n-2}^j), j = j0 .. j0+T-1:
 *
 *   f = sum_{i<t} c_i x^{dx_i} y^{dy_i} z_1^{e_i,1} ... z_{n-2}^{e_i,n-2}
 *   out[g*T + k] = coefficient of x^{dx_g} y^{dy_g} in f(x, y, beta^{j0+k})  mod p
 *
 * PAPER.md:246-266 (§2.1 "b_t(x1,x2) = f(x1,x2,beta^t)"), PAPER.md:408-419 (§2.3 Eq.
 * e:def_f), computed by the matrix method: m_i = M_i(alpha) once
 * (PAPER.md:428-442), a_i seeded at the chunk start by exponentiation,
 * then per point: coefficient reduction over equal (dx,dy) and a_i <- a_i * m_i
 * (Alg. 1, Alg. 7).
 *
 * Only POD types cross this boundary; all pointers are plain host or device pointers as
 * stated per call.  All functions are thread-safe across distinct handles; a single handle
 * is not re-entrant.
 *
 * Result contract (readings R1-R9):
 *   - rows g = 0..G-1 are the distinct (dx,dy) of the INPUT terms (zero-coefficient terms
 *     included), in descending lexicographic order; pe_bucket_exps()
 *     returns them;
 *   - every value is the canonical residue in [0, p); zero coefficients are stored (dense);
 *   - coefficients are reduced mod p; duplicate full monomials are summed; alpha_k is
 *     reduced mod p and must be non-zero mod p ("non-zero ... from F_p");
 *   - j0 = 0 is accepted (beta^0 = (1,...,1)); any j0 with j0+T-1 < 2^64.
 *   - bit-exact: the result is unique, independent of R / warps / chunk / stream.
 */
#ifndef PE_H_
#define PE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pe_ctx pe_ctx; /* opaque; owns its device buffers */

enum {
  PE_OK = 0,
  PE_EINVAL = -1,    /* NULL / inconsistent argument                                   */
  PE_ENOTPRIME = -2, /* p composite (deterministic Miller-Rabin, 12 prime bases <= 37)  */
  PE_ERANGE = -3,    /* p < 3, p >= 2^63, alpha_k == 0 mod p, j0+T-1 overflows, T*G huge  */
  PE_ENOMEM = -4,    /* host or device allocation failed                                */
  PE_ECUDA = -5,     /* CUDA runtime error (no device, launch failure, ...)             */
  PE_ENOTSUP = -6    /* requested path / option not supported for this p               */
};

enum { PE_PATH_AUTO = 0, PE_PATH_INT = 1, PE_PATH_FP64 = 2, PE_PATH_INT32 = 4, PE_PATH_TC = 5,
       PE_PATH_FAST = 6 };  /* 3: retired */
/* PE_PATH_FAST forces the asymptotically fast method (HL13)
 * for every T, any p < 2^63, T <= 2^20 (PE_ERANGE above): per bucket the T outputs
 * are the first T coefficients of sum_i a_i / (1 - m_i z) = N(z)/D(z), a_i = c_i m_i^{j0}, computed
 * by a product tree of (N, D) pairs and a Newton power-series inversion, with polynomial products
 * done exactly by NTTs over five 30-bit primes and CRT (O(s log^2 T) operations instead of s T).
 * PE_PATH_AUTO takes it only where the tensor-core form is off (env PE_TC=0, or degraded for lack
 * of memory), for T >= 8192 with >= 2048 terms per bucket -- its measured crossover with the scalar
 * k_step; it never beats the tensor-core form.  pe_eval_kernel reports the choice;
 * env PE_FAST=0 off, 2 always.  Bit-identical results. */
/* PE_PATH_TC forces the tensor-core form of the step (any p < 2^63; for 2^62 <= p the giant-step
 * chains use the exact-quotient Shoup product so every value keeps 8 bytes): each bucket's
 * block of T_c = 128 x V points is the product L * R of giant-step values c_i m_i^{j_s+Vu} and
 * baby-step values m_i^v, v < V (the Vandermonde structure M_i(beta^t) = m_i^t, PAPER.md:420-427,
 * 465-478), computed exactly as 64 byte-by-byte int8 tcgen05 MMAs; V = 32 for
 * p >= 2^54 (4096-point chunks, all 15 byte diagonals in one round), V = 64 below; the baby-step
 * planes are built once per handle (about 260 B per padded term of device memory at V = 32,
 * 530 B at V = 64).
 * PE_PATH_AUTO selects it for any p < 2^63 once T reaches the handle's measured threshold
 * (pe_tc_info): for p >= 2^54 (V = 32), T >= max(3400 t_pad^-0.19, 7.3e6 / t_pad) clamped to
 * [192, 8192]; for 2^31 <= p < 2^54, T >= max(2200 t_pad^-0.144, 7.3e6 / t_pad) clamped to
 * [192, 8192]; for p < 2^31 (against the 32-bit scalar core) T >= max(1350 t_pad^-0.045,
 * 1.1e7 / t_pad) clamped to [512, 8192].  It also needs one chunk of partial rows (8 B x pieces x rounds per point)
 * to fit the partial-buffer cap (env PE_PARTIAL_MB, default 1024), and its handle memory to fit the
 * device (and env PE_TC_MEM_MB if set): otherwise an automatic handle degrades to the scalar
 * k_step (same results).  env PE_TC=0 off, 1 auto, 2 always; PE_PATH_INT never uses it; PE_TC_DIRECT=0
 * makes every output row go through the fix-up (default: a bucket's sole piece writes its row directly).  Results
 * are bit-identical either way. */
/* PE_PATH_INT32 is reported by pe_info only: every p < 2^31 (any requested path except FP64)
 * uses 32-bit Shoup products. */

/* Tuning knobs (0 = automatic).  They never change the result (pin P13). */
typedef struct pe_config {
  int32_t path;  /* PE_PATH_AUTO: scalar core = 32-bit Shoup if p < 2^31, FP64 Alg. 2 if p < 2^50, else
                    INT64 Shoup; the tensor-core form instead for T >= the handle's threshold (any
                    p < 2^63).  PE_PATH_FP64 / PE_PATH_INT / PE_PATH_TC force one.
                    env PE_PATH=int|fp64, PE_CORE=fp64|shoup|int32               */
  int32_t R;     /* terms per lane: 1,2,4,8,16 (FP64: <= 8); auto picks by bucket sizes    */
  int32_t warps; /* warps per CTA, 1..16 (auto 8)                                          */
  int32_t chunk; /* points per CTA (multiple of 32; auto by grid coverage)                 */
  int32_t tc_form; /* tensor-core path, 7- and 8-digit primes (p >= 2^31): PE_TC_FORM_SWAPPED
                      (giant-step planes m^{32u} per handle, 1 KB per term, the 32 baby steps
                      c m^{j+v} per term and chunk generated -- a quarter of the plain form's
                      generation; config 5 evaluates 13-15 % faster; the automatic choice for
                      p >= 2^54) or PE_TC_FORM_PLAIN (baby-step planes m^v per handle, 256 B per term,
                      the 128 giant steps generated; 3x less DRAM per evaluation; the automatic
                      choice for 2^31 <= p < 2^54, where the swapped form measured no gain).  Same
                      results.  Below 2^31 always plain.  An automatic handle whose swapped planes
                      do not fit the device (or env PE_TC_MEM_MB) takes the plain form; env
                      PE_TC_SWAP=0/1 overrides the automatic (0) choice. */
} pe_config;
enum { PE_TC_FORM_AUTO = 0, PE_TC_FORM_PLAIN = 1, PE_TC_FORM_SWAPPED = 2 };

/*
 * pe_create -- build an evaluation handle on the CUDA device current at the call.
 *   p       prime, 3 <= p < 2^63.
 *   t       number of terms (0 allowed: G = 0).
 *   n       number of variables, n >= 2 (columns 0,1 are x,y; 2..n-1 are z_1..z_{n-2}).
 *   coeffs  HOST uint64[t], any values (reduced mod p).
 *   exps    HOST uint32[t*n], row-major: exps[i*n + 0] = deg_x, [i*n+1] = deg_y,
 *           [i*n + 2 + l] = deg of z_{l+1}.
 *   alpha   HOST uint64[n-2] (may be NULL iff n == 2), reduced mod p, must be != 0 mod p.
 * Deep-copies everything; the caller may free its arrays on return.
 * Returns NULL on error and sets pe_last_error() (PE_EINVAL / PE_ENOTPRIME / PE_ERANGE /
 * PE_ENOMEM / PE_ECUDA).  Validation happens before any CUDA call.  t <= 2^31 - 1 (PE_ERANGE).
 */
pe_ctx* pe_create(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs,
                  const uint32_t* exps, const uint64_t* alpha);
/* Same, with tuning knobs (cfg may be NULL = all automatic). */
pe_ctx* pe_create_ex(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs,
                     const uint32_t* exps, const uint64_t* alpha, const pe_config* cfg);

/*
 * pe_create_compact -- pe_create_ex with exponents as HOST uint8[t*n] (same row-major layout; every
 * degree < 256, which covers every BASELINE config and the paper's workloads).
 * A quarter of the bytes to move over PCIe for the same polynomial: the upload is most of an
 * end-to-end evaluation.  Same results, errors and ownership as pe_create_ex.
 */
pe_ctx* pe_create_compact(uint64_t p, uint64_t t, uint32_t n, const uint64_t* coeffs, const uint8_t* exps,
                          const uint64_t* alpha, const pe_config* cfg);

/*
 * pe_create_batch -- several polynomials f_0..f_{npoly-1} evaluated at the SAME points beta^j in
 * one launch (the gcd workload: images of f and h at the same beta^t;
 * SURVEY.md §8(f) NEXT-1).  Polynomial k owns terms [sum_{q<k} t_per_poly[q], ... + t_per_poly[k])
 * of coeffs / exps (same layouts as pe_create).  Output rows are ordered by polynomial, then by
 * descending (dx,dy) within it; pe_poly_rows gives the row range of each polynomial.
 * npoly >= 1; a polynomial may have zero terms (zero rows).  Errors as pe_create.
 */
pe_ctx* pe_create_batch(uint64_t p, uint32_t npoly, const uint64_t* t_per_poly, uint32_t n,
                        const uint64_t* coeffs, const uint32_t* exps, const uint64_t* alpha,
                        const pe_config* cfg);
uint32_t pe_num_polys(const pe_ctx* h);                       /* npoly (1 for pe_create)        */
int pe_poly_rows(const pe_ctx* h, uint64_t* row_off);         /* HOST uint64[npoly+1]: rows of f_k
                                                                 are [row_off[k], row_off[k+1]) */

/*
 * pe_eval -- T images into HOST memory out[G*T] (row g, column k <-> j = j0 + k).
 * Synchronous.  T == 0 or G == 0 is a no-op returning PE_OK.
 * Errors: PE_EINVAL (h NULL, out NULL with G*T > 0), PE_ERANGE (j0 + T - 1 >= 2^64),
 *         PE_ENOMEM, PE_ECUDA.
 */
int pe_eval(pe_ctx* h, uint64_t j0, uint64_t T, uint64_t* out);

/*
 * pe_eval_device -- T images into DEVICE memory: d_out[g*ld + k], ld >= T (elements).
 * Asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream): returns after
 * enqueueing.  The handle's scratch is reused by the next call on the same handle, so calls
 * on one handle must be stream-ordered (same stream, or synchronised).  Runs on the handle's
 * device whatever device is current (restored on return).  If an earlier tensor-core launch of
 * the handle timed out in a pipeline wait (a protocol fault, never a legitimate stall), every
 * later call returns PE_ECUDA.
 */
int pe_eval_device(pe_ctx* h, uint64_t j0, uint64_t T, uint64_t* d_out, uint64_t ld,
                   void* stream);

/*
 * pe_eval_device_rows -- rows [g0, g1) of the result only, into d_out[g*ld + k] for g0 <= g < g1
 * (the other rows untouched).  Asynchronous on `stream` like pe_eval_device.  A strict sub-range
 * needs the tensor-core path for this T (pe_eval_kernel == 1), else PE_ENOTSUP; g0 = 0, g1 = G is
 * plain pe_eval_device.  Used to overlap a row block's transfer with the next block's evaluation.
 * Errors: PE_EINVAL (h NULL, g0 > g1 or g1 > G, d_out NULL, ld < T), PE_ERANGE, PE_ENOTSUP, PE_ECUDA.
 */
int pe_eval_device_rows(pe_ctx* h, uint64_t j0, uint64_t T, uint64_t g0, uint64_t g1, uint64_t* d_out,
                        uint64_t ld, void* stream);
/* The handle's row split G1 for such overlap (pe_eval uses rows [0, G1) then [G1, G); chosen so the
 * second block's evaluation covers the first block's transfer); 0 = no split
 * (no tensor-core path, or G < 2). */
uint64_t pe_row_split(const pe_ctx* h);

/* NULL-safe.  Waits for the handle's own streams and for the latest work each pe_eval_device(_rows)
 * call enqueued on a caller stream, then frees the handle (stream-ordered); it does not synchronise
 * the whole device, so other handles' work (e.g. another thread's pe_create) keeps running. */
void pe_destroy(pe_ctx* h);

uint64_t pe_num_buckets(const pe_ctx* h);                   /* G (0 if h NULL) */
int pe_bucket_exps(const pe_ctx* h, uint32_t* dxdy);        /* HOST uint32[2G]: row g -> (dx,dy) */

/* Introspection: values chosen at create. Any pointer may be NULL. */
int pe_info(const pe_ctx* h, int32_t* path, int32_t* R, int32_t* warps, uint64_t* t_padded,
            uint64_t* n_slots);

/* Tensor-core path state: *mode = 0 (not built for this handle, or degraded for lack of memory), 1
 * (automatic: used by evaluations with T >= *min_T), 2 (forced, every T); *pieces = accumulation
 * pieces (<= 8192 terms of one bucket each; env PE_TC_PIECE caps them lower, for tests).  Any
 * pointer may be NULL.  Errors: PE_EINVAL (h NULL). */
int pe_tc_info(const pe_ctx* h, int32_t* mode, uint64_t* pieces, uint64_t* min_T);
/* The handle's tensor-core form: PE_TC_FORM_PLAIN or PE_TC_FORM_SWAPPED, 0 if it has no tensor-core
 * path (pe_config.tc_form).  PE_EINVAL if h is NULL. */
int pe_tc_form(const pe_ctx* h);

/* Which hot kernel an evaluation of T points on this handle runs: 0 = the scalar k_step, 1 = the
 * tensor-core k_tc, 2 = the fast product-tree method (the automatic choice: thresholds,
 * partial-buffer cap, memory).  PE_EINVAL if h is NULL. */
int pe_eval_kernel(const pe_ctx* h, uint64_t T);

/* m_i = prod_l alpha_l^{e_i,l} mod p for every input term i (HOST uint64[t], input order). */
int pe_monomials(const pe_ctx* h, uint64_t* m);

/*
 * Kernel timing (for bench.py's roofline): when enabled, pe_eval_device records CUDA events
 * on its stream around every hot-loop launch (k_step, or k_tc on the tensor-core path) and the
 * k_fixup that follows it.  pe_kernel_stats waits for the recorded events, returns the
 * accumulated launch count, device milliseconds of the hot kernel and of k_fixup, and the
 * term-points processed (padded terms x points), then resets them.
 */
int pe_set_timing(pe_ctx* h, int enable);
int pe_kernel_stats(pe_ctx* h, uint64_t* step_launches, double* step_ms, double* fixup_ms,
                    double* term_points);

/*
 * Berlekamp-Massey per sequence (the sparse-interpolation step after the
 * path; Ben-Or/Tiwari).  For each of the G sequences
 * s_g(k) = d_seq[g*ld + k], k < T, values canonical in [0, p) (e.g. pe_eval_device output),
 * computes the shortest connection polynomial C_g(z) = 1 + c_1 z + ... + c_L z^L with
 * s_g(k) + sum_{i=1..L} c_i s_g(k-i) = 0 for L <= k < T:
 *   d_lambda[g*ldl + i] = c_i (c_0 = 1, zeros beyond L), ldl >= T+1;   d_len[g] = L.
 * For T >= 2 r_g it equals prod (1 - m_i z) over the bucket's distinct m_i with nonzero
 * coefficient sum.  p prime, 3 <= p < 2^63.  Asynchronous on `stream` (device pointers);
 * pe_bm is the synchronous host-array form.  Errors: PE_EINVAL, PE_ERANGE, PE_ENOMEM, PE_ECUDA.
 */
int pe_bm_device(uint64_t p, uint64_t G, uint64_t T, const uint64_t* d_seq, uint64_t ld,
                 uint64_t* d_lambda, uint64_t ldl, uint32_t* d_len, void* stream);
int pe_bm(uint64_t p, uint64_t G, uint64_t T, const uint64_t* seq /*[G*T]*/,
          uint64_t* lambda /*[G*(T+1)]*/, uint32_t* len /*[G]*/);

/*
 * Multi-GPU assembly (BASELINE.json north_star "sharding ... one gather"), so the
 * Python plumbing does no modular arithmetic and no per-rank copy loops.  Device pointers,
 * asynchronous on `stream`.
 *
 * pe_rows_addmod -- d_dst[r*ld_dst + k] = (d_dst[r*ld_dst + k] + d_src[r*ld_src + k]) mod p for
 *   r < rows, k < cols.  Both operands canonical residues in [0, p), 3 <= p < 2^63 (the u64 sum
 *   cannot wrap).  The root's coefficient reduction of a bucket whose terms two ranks share
 *   (PAPER.md:489-503 across ranks).  Errors: PE_ERANGE (p), PE_EINVAL (NULL, ld < cols), PE_ECUDA.
 *
 * pe_unshard_columns -- point-range shards back into rows: d_blocks is [P][G][Tr] (rank r's
 *   columns r*Tr .. r*Tr + Tr - 1, the gathered buffer), d_out is [G][ld] with ld >= T;
 *   d_out[g*ld + r*Tr + k] = d_blocks[(r*G + g)*Tr + k] for r*Tr + k < T.  Errors: PE_EINVAL
 *   (NULL, ld < T, P*Tr < T), PE_ECUDA.
 */
int pe_rows_addmod(uint64_t p, uint64_t* d_dst, uint64_t ld_dst, const uint64_t* d_src, uint64_t ld_src,
                   uint64_t rows, uint64_t cols, void* stream);
int pe_unshard_columns(uint64_t* d_out, uint64_t ld, const uint64_t* d_blocks, uint64_t P, uint64_t G,
                       uint64_t Tr, uint64_t T, void* stream);

int pe_last_error(void);            /* thread-local code of the last failing call */
const char* pe_strerror(int code);

/* Advisory: 1 iff p > 100 t^2 (distinct m_i likely); never enforced. */
int pe_interp_bound_ok(uint64_t p, uint64_t t);

#ifdef __cplusplus
}
#endif
#endif /* PE_H_ */
