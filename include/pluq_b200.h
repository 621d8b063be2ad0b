/* pluq_b200.h — C ABI of the B200-native PLUQ-mod-p hot path.
 *
 * Drop-in boundary for the reference package `pluq` (/root/reference/pkg/src/pluq).
 * Every entry point names the reference interface it replaces.  No torch or C++
 * types cross this boundary: plain pointers, sizes and int status codes.
 *
 * Conventions
 *  - Matrices are row-major; `ld` is the row pitch in ELEMENTS.  Device-side
 *    storage is uint32 canonical residues in [0, p), p prime, 2 <= p < 2^31.
 *  - Permutations are returned as int64 "sigma" arrays with the reference
 *    convention Mat(sigma)[i, sigma(i)] = 1 (matrix.py:3-11).
 *  - counts[4] = {field_mul, field_add, field_inv, modular_reductions}, i.e.
 *    OpCounts (matrix.py:22-43); they are ADDED to, never reset.
 *  - Return value: PLUQ_OK or a PLUQ_E* code; the Python wrapper maps
 *    PLUQ_EINVAL -> ValueError and PLUQ_EZERODIV -> ZeroDivisionError
 *    (recursive.py:171-172, field.py:44-45, kernels.py:93-95).
 *  - All device work is ordered on the context's stream.  A context is not
 *    thread-safe; use one context per host thread (a
 *    decomposition is single-threaded, distinct decompositions may run
 *    concurrently).
 */
#ifndef PLUQ_B200_H
#define PLUQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PLUQ_OK = 0,
  PLUQ_EINVAL = 1,
  PLUQ_EZERODIV = 2,
  PLUQ_ECUDA = 3,
  PLUQ_ENOMEM = 4,
  PLUQ_EUNSUPPORTED = 5
};

typedef struct pluq_ctx pluq_ctx;

/* Context: device, stream (cudaStream_t as void*, NULL = legacy default stream)
 * and the reusable workspace (replaces the Workspace hook, recursive.py:36-48). */
int pluq_create(pluq_ctx** ctx, int device, void* stream);
int pluq_destroy(pluq_ctx* ctx);
int pluq_set_stream(pluq_ctx* ctx, void* stream);
/* Frees the context's kept device workspace: the node backup of the speculative LU
 * (m*n*2 bytes for p < 2^16, else m*n*4, kept between calls) and the pool's free blocks. */
int pluq_release_workspace(pluq_ctx* ctx);
/* Tuning knobs (0 = keep default): largest node m*n handled whole by one CTA in
 * shared memory, and whether the tensor-core GEMM may be used (1/0). */
int pluq_set_option(pluq_ctx* ctx, const char* key, int64_t value);
/* Current value of an option (PLUQ_EINVAL for an unknown key). */
int pluq_get_option(pluq_ctx* ctx, const char* key, int64_t* value);
const char* pluq_last_error(pluq_ctx* ctx);

/* pluq(a, threshold) — recursive.py:159-183 (+ _pluq_rec :186-256).
 * dA: device uint32 m x n (pitch ld), overwritten in place by [L\U, V; M, 0].
 * Entries must be canonical residues in [0, p): otherwise PLUQ_EINVAL and dA is left
 * untouched (field.py:140-147; option check_inputs).  The same holds for the batched and
 * host-buffer entry points (the batched host one raises after the fact: see below).
 * p_sigma (m) / q_sigma (n): HOST int64 outputs. rank: host output. */
int pluq_factor(pluq_ctx* ctx, uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t p,
                int64_t threshold, int64_t* p_sigma, int64_t* q_sigma, int64_t* rank,
                int64_t* counts);

/* pluq_iterative(a) — iterative.py:23-27 (Algorithm 2 on the whole matrix). */
int pluq_factor_iterative(pluq_ctx* ctx, uint32_t* dA, int64_t ld, int64_t m, int64_t n,
                          int64_t p, int64_t* p_sigma, int64_t* q_sigma, int64_t* rank,
                          int64_t* counts);

/* Batched pluq over `batch` independent m x n blocks at dA + b*stride (device).
 * The reference loops pluq() per matrix; here one CTA factors one matrix.
 * Outputs are DEVICE int32: d_p (batch*m), d_q (batch*n), d_rank (batch);
 * d_counts (batch*4 uint64) may be NULL.  Requires the block to fit in shared
 * memory (see pluq_batched_max_elems). */
int pluq_factor_batched(pluq_ctx* ctx, uint32_t* dA, int64_t stride, int64_t batch, int64_t m,
                        int64_t n, int64_t p, int64_t threshold, int32_t* d_p, int32_t* d_q,
                        int32_t* d_rank, uint64_t* d_counts);
int64_t pluq_batched_max_elems(pluq_ctx* ctx, int64_t m, int64_t n);

/* Host-buffer entry points (end-to-end path of `pluq(DenseMatrix)`): the matrix
 * is read from and written back to HOST memory in the reference's storage dtype
 * (float64 when (p-1)^2*8192 <= 2^53, else int64; field.py:75-81). */
int pluq_factor_host_f64(pluq_ctx* ctx, double* hA, int64_t m, int64_t n, int64_t p,
                         int64_t threshold, int64_t* p_sigma, int64_t* q_sigma, int64_t* rank,
                         int64_t* counts);
int pluq_factor_host_i64(pluq_ctx* ctx, int64_t* hA, int64_t m, int64_t n, int64_t p,
                         int64_t threshold, int64_t* p_sigma, int64_t* q_sigma, int64_t* rank,
                         int64_t* counts);
/* Non-canonical entries (outside [0, p), non-integral, NaN) give PLUQ_EINVAL after the
 * pipelined call; the buffer's contents are then unspecified. */
int pluq_factor_batched_host_f64(pluq_ctx* ctx, double* hA, int64_t batch, int64_t m, int64_t n,
                                 int64_t p, int64_t threshold, int64_t* p_sigma,
                                 int64_t* q_sigma, int64_t* ranks);

/* Kernel strategy (kernels.py:30-120, ClassicalKernels) on device views. */
/* mm_acc: C <- C - A B mod p (kernels.py:38-55). */
int pluq_modgemm_sub(pluq_ctx* ctx, uint32_t* dC, int64_t ldc, const uint32_t* dA, int64_t lda,
                     const uint32_t* dB, int64_t ldb, int64_t m, int64_t n, int64_t k, int64_t p);
/* trsm_left_unit_lower: B <- L^-1 B, L r x r unit lower (kernels.py:59-83). */
int pluq_trsm_llu(pluq_ctx* ctx, const uint32_t* dL, int64_t ldl, uint32_t* dB, int64_t ldb,
                  int64_t r, int64_t n, int64_t p);
/* trsm_right_upper: B <- B U^-1, U r x r upper (kernels.py:85-120); PLUQ_EZERODIV
 * if diag(U) has a zero. */
int pluq_trsm_ru(pluq_ctx* ctx, uint32_t* dB, int64_t ldb, const uint32_t* dU, int64_t ldu,
                 int64_t m, int64_t r, int64_t p);
/* apply_rows(X, perm) / apply_cols(X, perm) (matrix.py:249-283): gather form,
 * new_row[i] = old_row[g[i]] / new_col[j] = old_col[g[j]]; g is HOST int64. */
int pluq_permute_rows(pluq_ctx* ctx, uint32_t* dX, int64_t ld, int64_t rows, int64_t cols,
                      const int64_t* g);
int pluq_permute_cols(pluq_ctx* ctx, uint32_t* dX, int64_t ld, int64_t rows, int64_t cols,
                      const int64_t* g);

/* Tensor-core modular GEMM only (tcgen05 kind::i8 limb path); used by tests and
 * the bench to time the dominant kernel.  Returns PLUQ_EUNSUPPORTED if the shape
 * is below the tensor-core tile. */
int pluq_modgemm_sub_tc(pluq_ctx* ctx, uint32_t* dC, int64_t ldc, const uint32_t* dA,
                        int64_t lda, const uint32_t* dB, int64_t ldb, int64_t m, int64_t n,
                        int64_t k, int64_t p);

/* OpCounts the reference charges on an m x n matrix with a GENERIC rank profile of rank
 * `rank` (leading principal minors 1..rank nonzero), where P = Q = I.  Host-only. */
int pluq_generic_counts(int64_t m, int64_t n, int64_t rank, int64_t threshold, int64_t* counts);

/* *out = 1 if the device view (uint32, pitch ld) has a nonzero entry, else 0.  Used by the
 * multi-GPU driver for the "Schur complement vanishes" test (recursive.py:188-189 zero blocks). */
int pluq_nonzero(pluq_ctx* ctx, const uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t* out);

/* Algorithm 1 with the Algorithm 2 base case (recursive.py:186-256, iterative.py:23-91)
 * replayed symbolically on the m x n rank profile matrix with ones at (prow[k], pcol[k]),
 * k < r: the P.sigma (m), Q.sigma (n) and OpCounts (counts[4], may be NULL; SET, not added)
 * that pluq() returns for ANY matrix with that rank profile matrix (pluq_rpm.cuh facts).
 * Host-only (no device work); PLUQ_EINVAL unless the pairs form a partial permutation. */
int pluq_rank_profile_replay(int64_t m, int64_t n, int64_t threshold, int64_t r, const int64_t* prow,
                             const int64_t* pcol, int64_t* p_sigma, int64_t* q_sigma, int64_t* counts);

/* PLUQ_OK iff every entry of the device view (uint32, pitch ld) is a canonical residue in
 * [0, p); PLUQ_EINVAL otherwise.  The check field.asarray makes when a DenseMatrix is built
 * (field.py:140-147), for device-resident matrices; one HBM read of the view. */
int pluq_check_residues(pluq_ctx* ctx, const uint32_t* dA, int64_t ld, int64_t m, int64_t n, int64_t p);

/* Microbenchmarked peaks of this device (SURVEY §8d roofline denominators):
 * out[0] = tcgen05 kind::i8 dense TOP/s (128x256x32 MMAs, one CTA per SM),
 * out[1] = FP64 DMMA (mma.sync m8n8k4) TFLOP/s.  Diagnostics; not on the factorization path. */
int pluq_measure_peaks(pluq_ctx* ctx, double* out, int64_t nout);

/* Statistics of the last call: launches, host syncs, nodes, small-node kernels, base-case
 * kernels, tensor-core / SIMT GEMMs, zero-block skips, generic leaves, speculative ok/fail,
 * generic- and fallback-kernel ns of a batch (option time_kernels), the MMA-kernel ns of
 * the last tensor-core GEMM (option tc_time), and — option tc_time, summed over the call —
 * MMA-kernel launches, their CUDA-event ns and their algorithmic int8 ops (2 m n k L^2), and
 * the zero pivots the speculative LU repaired by a column rotation, and the chunks of the
 * last host-buffer call that were downloaded while its factorization was still running. */
int pluq_last_stats(pluq_ctx* ctx, int64_t* out, int64_t nout);

#ifdef __cplusplus
}
#endif
#endif /* PLUQ_B200_H */
