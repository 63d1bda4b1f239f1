/* batchfact_b200 -- C ABI of the B200-native batched QR / Jacobi SVD / randomized SVD.
 *
 * Drop-in boundary for the reference's batched entry points (all of which route
 * through core.batch_apply, /root/reference/pkg/src/batchfact/core.py:97-123):
 *
 *   bf_qr_batched_*         replaces batch_qr        qr.py:98-100        (per entry: qr, qr.py:63-95)
 *   bf_svd_batched_*        replaces batch_svd       jacobi.py:287-290   (per entry: svd, jacobi.py:231-284)
 *   bf_block_svd_batched_*  replaces batch_block_svd blockjacobi.py:171-174 (block_svd, :84-168)
 *   bf_rsvd_batched_*       replaces batch_rsvd      rsvd.py:79-86       (rsvd, rsvd.py:56-76)
 *   bf_gaussian_batched_*   replaces gaussian_matrix rsvd.py:42-53 (numpy Philox4x64 + ziggurat, bitwise)
 *
 * Conventions (all of them the reference's):
 *   - every matrix is column-major with ld = rows; a batch is `batch` equally shaped
 *     matrices at a fixed stride (rows*cols elements); all pointers are DEVICE pointers;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); calls are asynchronous;
 *   - m >= n is required (qr.py:71-72, jacobi.py:242-243, blockjacobi.py:94-95),
 *     k + p <= min(m, n) for rsvd (rsvd.py:60-64): violations return BF_ERR_ARG before any
 *     launch, with the reference's message in bf_last_error();
 *   - non-convergence is never an error: per-entry `converged` flags and `sweeps` counts;
 *   - workspace: query bf_*_workspace_size() and pass at least that many device bytes;
 *   - the _f32 entry points keep float32 in / out and float32 semantics (default tolerances,
 *     numpy's float32 Gaussian stream) and compute on the float64 tiers where those cover the
 *     shape (QR, rr / register SVD, block direct, rsvd); their workspace query (es = 4)
 *     includes the widened copies. BF_F32_NATIVE=1 in the environment keeps float32 arithmetic.
 *
 * Return: BF_OK (0) or a negative BF_ERR_* code (or a positive cudaError_t value).
 */
#ifndef BATCHFACT_B200_H
#define BATCHFACT_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BF_API __attribute__((visibility("default")))
#else
#define BF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BF_OK 0
#define BF_ERR_ARG (-1)         /* precondition violation: the reference raises ValueError */
#define BF_ERR_WORKSPACE (-2)   /* workspace missing / too small */
#define BF_ERR_UNSUPPORTED (-3) /* shape/option outside what this build implements */

/* JacobiOptions (jacobi.py:30-48). tolerance <= 0 selects the per-dtype default
 * (1e-14 f64 / 1e-6 f32, jacobi.py:22-25). ordering: 0 serial, 1 round_robin.
 * tier: 0 auto, 1 register (warp per matrix, n <= 32), 2 shared memory. */
typedef struct bf_jacobi_opts {
  double tolerance;
  int32_t max_sweeps;
  int32_t ordering;
  int32_t accumulate_v;
  int32_t tier;
} bf_jacobi_opts;

/* BlockJacobiOptions (blockjacobi.py:27-48). method: 0 gram, 1 direct (reference default).
 * tolerance <= 0: 1e-13 f64 / 1e-5 f32 (blockjacobi.py:19-22). */
typedef struct bf_block_opts {
  double tolerance;
  int32_t block_width;
  int32_t method;
  int32_t max_sweeps;
  int32_t accumulate_v;
} bf_block_opts;

BF_API const char* bf_last_error(void);
BF_API const char* bf_version(void);

/* ---- batched Householder QR: q (m x n), r (n x n, exact zeros below the diagonal) */
BF_API size_t bf_qr_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t dtype_bytes);
BF_API int bf_qr_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* q, double* r,
                      int32_t panel_width, void* workspace, size_t workspace_bytes, void* stream);
BF_API int bf_qr_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* q, float* r,
                      int32_t panel_width, void* workspace, size_t workspace_bytes, void* stream);

/* ---- batched one-sided Jacobi SVD: u (m x n), sigma (n, descending), v (n x n, nullable
 * unless accumulate_v), sweeps/converged per entry, rotations (nullable) = total rotations. */
BF_API size_t bf_svd_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t dtype_bytes, const bf_jacobi_opts* opts);
BF_API int bf_svd_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* u, double* sigma, double* v,
                       int32_t* sweeps, uint8_t* converged, int64_t* rotations, const bf_jacobi_opts* opts,
                       void* workspace, size_t workspace_bytes, void* stream);
BF_API int bf_svd_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* u, float* sigma, float* v,
                       int32_t* sweeps, uint8_t* converged, int64_t* rotations, const bf_jacobi_opts* opts,
                       void* workspace, size_t workspace_bytes, void* stream);

/* ---- batched block Jacobi SVD; e_history (nullable): batch x max_sweeps, entry b's first
 * sweeps[b] values are its per-sweep max scaled off-diagonal (BlockSvdResult.e_history). */
BF_API size_t bf_block_svd_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t dtype_bytes,
                                   const bf_block_opts* opts);
BF_API int bf_block_svd_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* u, double* sigma,
                             double* v, int32_t* sweeps, uint8_t* converged, double* e_history,
                             const bf_block_opts* opts, void* workspace, size_t workspace_bytes, void* stream);
BF_API int bf_block_svd_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* u, float* sigma,
                             float* v, int32_t* sweeps, uint8_t* converged, float* e_history,
                             const bf_block_opts* opts, void* workspace, size_t workspace_bytes, void* stream);
/* Same, plus per-matrix work counters (stats: batch x 4 int64, nullable): [0] pair visits (Gram or
 * pair QR + e = scaled_offdiag), [1] rotated pairs (e > tol), [2] inner-SVD pair visits (inner
 * sweeps x 2k(2k-1)/2), [3] inner-SVD rotations -- the run's own counts behind the algorithmic
 * flop figure (no reference counterpart; measurement extension). */
BF_API int bf_block_svd_batched_ex_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* u, double* sigma,
                                double* v, int32_t* sweeps, uint8_t* converged, double* e_history, int64_t* stats,
                                const bf_block_opts* opts, void* workspace, size_t workspace_bytes, void* stream);
BF_API int bf_block_svd_batched_ex_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* u, float* sigma,
                                float* v, int32_t* sweeps, uint8_t* converged, float* e_history, int64_t* stats,
                                const bf_block_opts* opts, void* workspace, size_t workspace_bytes, void* stream);

/* ---- batched randomized SVD (Alg. 4): entry b uses seed ^ (index_base + b) (rsvd.py:79-86),
 * seed = seed_lo | seed_hi << 64. omega (nullable): batch x (n x (k+p)) sketch supplied by the
 * caller; NULL draws it on the device, bitwise equal to gaussian_matrix(n, k+p, seed ^ i, dtype)
 * (rsvd.py:52,65: the f32 entry point draws numpy's float32 stream).
 * u: m x (k+p), s: k+p, v: n x (k+p) -- all k+p triplets, not truncated (rsvd.py:35-39). */
BF_API size_t bf_rsvd_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t k, int32_t p, int32_t dtype_bytes);
BF_API int bf_rsvd_batched_f64(int64_t batch, int32_t m, int32_t n, int32_t k, int32_t p, uint64_t seed_lo,
                        uint64_t seed_hi, int64_t index_base, const double* a, const double* omega, double* u,
                        double* s, double* v, void* workspace, size_t workspace_bytes, void* stream);
BF_API int bf_rsvd_batched_f32(int64_t batch, int32_t m, int32_t n, int32_t k, int32_t p, uint64_t seed_lo,
                        uint64_t seed_hi, int64_t index_base, const float* a, const float* omega, float* u,
                        float* s, float* v, void* workspace, size_t workspace_bytes, void* stream);

/* ---- numpy-compatible Gaussian matrices: entry b uses key (seed_lo ^ (index_base + b), seed_hi)
 * when seed_mode == 0, (seed_lo + index_base + b, seed_hi) when seed_mode == 1. */
BF_API int bf_gaussian_batched_f64(int64_t batch, int32_t rows, int32_t cols, uint64_t seed_lo, uint64_t seed_hi,
                            int64_t index_base, int32_t seed_mode, double* out, void* stream);
BF_API int bf_gaussian_batched_f32(int64_t batch, int32_t rows, int32_t cols, uint64_t seed_lo, uint64_t seed_hi,
                            int64_t index_base, int32_t seed_mode, float* out, void* stream);

/* ---- testmat.make_matrix (testmat.py:83-94) on the device, geometric/arithmetic spectrum:
 * entry b uses seed_lo + index_base + b. Harness utility (input generation), not hot path. */
BF_API size_t bf_make_matrix_workspace_size(int64_t batch, int32_t m, int32_t n);
BF_API int bf_make_matrix_batched_f64(int64_t batch, int32_t m, int32_t n, int32_t mode, double cond, int32_t rank,
                               uint64_t seed_lo, uint64_t seed_hi, int64_t index_base, double* a, double* sigma,
                               void* workspace, size_t workspace_bytes, void* stream);

/* ---- strided batched GEMM, C_b = op(A_b) op(B_b) (column-major; op = transpose when t* != 0).
 * The batched matrix-matrix products of the H^2 compression ("After forming the TE
 * matrices using batched matrix-matrix multiplication"; "S~_ts = T_t S_ts T_s^T using
 * batched matrix-matrix multiplications"). op(A) is M x K, op(B) is K x N, C is M x N (ldc >= M).
 * f64 runs on the FP64 tensor cores (DMMA) when M <= 128, N <= 64 and the operands are 16-byte
 * aligned with even leading dimensions/strides; otherwise a tiled CUDA-core kernel. */
BF_API int bf_gemm_batched_f64(int64_t batch, int32_t M, int32_t N, int32_t K, const double* a, int32_t lda,
                        int64_t a_stride, int32_t ta, const double* b, int32_t ldb, int64_t b_stride, int32_t tb,
                        double* c, int32_t ldc, int64_t c_stride, void* stream);
BF_API int bf_gemm_batched_f32(int64_t batch, int32_t M, int32_t N, int32_t K, const float* a, int32_t lda,
                        int64_t a_stride, int32_t ta, const float* b, int32_t ldb, int64_t b_stride, int32_t tb,
                        float* c, int32_t ldc, int64_t c_stride, void* stream);

/* ---- the reference's public helper functions, batched over independent entries (the drop-in
 * calls them with batch = 1). All operands device pointers, column-major.
 *   bf_householder_batched_*      replaces householder_vector  qr.py:26-48
 *                                 (x, v: batch x len; tau: batch; v[0] = 1)
 *   bf_jacobi_rotation_batched_f64 replaces jacobi_rotation   jacobi.py:68-80 (c, s per entry)
 *   bf_off_orthogonality_batched_* replaces off_orthogonality jacobi.py:83-99 (a: m x n)
 *   bf_scaled_offdiag_batched_*   replaces scaled_offdiag     blockjacobi.py:57-76 (g: n x n)
 *   bf_syrk_batched_*             replaces syrk               core.py:68-78 (g = a^T a, mirrored)
 *   bf_frobenius_batched_*        replaces frobenius          core.py:81-86
 *   bf_axpby_*                    gemm's alpha/beta epilogue  core.py:36-65 (out = alpha p + beta c) */
BF_API int bf_householder_batched_f64(int64_t batch, int32_t len, const double* x, double* v, double* tau,
                               void* stream);
BF_API int bf_householder_batched_f32(int64_t batch, int32_t len, const float* x, float* v, float* tau, void* stream);
BF_API int bf_jacobi_rotation_batched_f64(int64_t batch, const double* g_pp, const double* g_pq, const double* g_qq,
                                   double* c, double* s, void* stream);
BF_API int bf_off_orthogonality_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* out,
                                     void* stream);
BF_API int bf_off_orthogonality_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* out,
                                     void* stream);
BF_API int bf_scaled_offdiag_batched_f64(int64_t batch, int32_t n, const double* g, double* out, void* stream);
BF_API int bf_scaled_offdiag_batched_f32(int64_t batch, int32_t n, const float* g, float* out, void* stream);
BF_API int bf_syrk_batched_f64(int64_t batch, int32_t m, int32_t k, const double* a, double* g, void* stream);
BF_API int bf_syrk_batched_f32(int64_t batch, int32_t m, int32_t k, const float* a, float* g, void* stream);
BF_API int bf_frobenius_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* out, void* stream);
BF_API int bf_frobenius_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* out, void* stream);
BF_API int bf_axpby_f64(int64_t n, double alpha, const double* p, double beta, const double* c, double* out,
                 void* stream);
BF_API int bf_axpby_f32(int64_t n, float alpha, const float* p, float beta, const float* c, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BATCHFACT_B200_H */
