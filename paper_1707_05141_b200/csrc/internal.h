// Internal launch interface between the C-ABI layer (api.cu) and the kernel TUs.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace bf {

template <typename T>
struct Tol;
template <>
struct Tol<double> {
  // jacobi.py:22-25, blockjacobi.py:19-22
  static constexpr double svd = 1e-14;
  static constexpr double block = 1e-13;
};
template <>
struct Tol<float> {
  static constexpr double svd = 1e-6;
  static constexpr double block = 1e-5;
};

struct SvdLaunch {
  int64_t batch;
  int m, n;
  const void* a;     // batch x (m x n) column-major, stride m*n
  int64_t a_stride;  // elements between consecutive matrices
  void* u;           // batch x (m x n)
  int64_t u_stride;
  void* s;  // batch x n
  int64_t s_stride;
  void* v;  // batch x (n x n) or null
  int64_t v_stride;
  int32_t* sweeps;
  uint8_t* converged;
  int64_t* rotations;
  double tol;
  int max_sweeps, ordering, tier;
  bool transpose_a;  // read A^T (a is n x m column-major) -- used by rsvd for R_B^T
  const uint8_t* active = nullptr;  // optional per-entry mask: inactive entries are skipped
  bool accumulate = false;          // add to sweeps / rotations instead of storing (block inner SVDs)
};

struct GemmLaunch {
  int64_t batch;
  int M, N, K;
  const void* a;
  int lda;
  int64_t a_stride;
  bool ta;  // op(A) = A^T (A stored K x M)
  const void* b;
  int ldb;
  int64_t b_stride;
  bool tb;
  void* c;
  int ldc;
  int64_t c_stride;
};

// Opt a kernel into `need` bytes of dynamic shared memory. The attribute is process-wide state per
// function and device, so concurrent host threads launching the same kernel with different sizes
// must not lower it under each other: it is only ever raised (under a mutex).
cudaError_t smem_optin(const void* func, size_t need);

// all return 0 or a CUDA error code; dtype 0 = f64, 1 = f32
size_t svd_global_ws_bytes(int dtype, int64_t batch, int m, int n, int ordering, bool accv, int tier, int max_sweeps);
int launch_svd(int dtype, const SvdLaunch& L, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_qr(int dtype, int64_t batch, int m, int n, const void* a, int64_t a_stride, void* q, int64_t q_stride,
              void* r, int64_t r_stride, void* ws, cudaStream_t st);
size_t qr_global_ws_bytes(int dtype, int64_t batch, int m, int n);
int launch_gemm(int dtype, const GemmLaunch& L, cudaStream_t st);
// c_order: store the C-order fill contiguously (row-major rows x cols) instead of column-major
int launch_gaussian_f64(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, int64_t index_base,
                        int seed_mode, uint64_t xor_mask, double* out, int64_t out_stride, cudaStream_t st,
                        int c_order = 0);
int launch_gaussian_f32(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, int64_t index_base,
                        int seed_mode, uint64_t xor_mask, float* out, int64_t out_stride, cudaStream_t st,
                        int c_order = 0);
int launch_sign_fix_f64(int64_t batch, int m, int n, double* q, const double* r, cudaStream_t st);
int launch_scale_cols_f64(int64_t batch, int m, int n, double* q, const double* sigma, cudaStream_t st);

// reference helper functions (helpers.cu)
template <typename T>
int launch_householder(int64_t batch, int len, const T* x, T* v, T* tau, cudaStream_t st);
int launch_rotation(int64_t batch, const double* gpp, const double* gpq, const double* gqq, double* c, double* s,
                    cudaStream_t st);
template <typename T>
int launch_offdiag(int64_t batch, int m, int n, const T* a, int gram, T* out, cudaStream_t st);
template <typename T>
int launch_syrk(int64_t batch, int m, int k, const T* a, T* g, cudaStream_t st);
template <typename T>
int launch_frobenius(int64_t batch, int64_t count, const T* a, T* out, cudaStream_t st);
template <typename T>
int launch_axpby(int64_t n, T alpha, const T* p, T beta, const T* c, T* out, cudaStream_t st);
template <typename S, typename D>
int launch_cast(int64_t n, const S* src, D* dst, cudaStream_t st);
// float64 fast tiers covering a shape (the float32 entry points compute on them, api.cu)
bool qr_reg_covers(int m, int n);
bool svd_rr_covers(const SvdLaunch& L);
bool svd_reg_covers(const SvdLaunch& L);

struct BlockLaunch {
  int64_t batch;
  int m, n;
  const void* a;
  void* u;
  void* s;
  void* v;
  int32_t* sweeps;
  uint8_t* converged;
  void* e_history;  // batch x max_sweeps or null
  int block_width, method, max_sweeps;
  double tol;
  // optional per-matrix work counters (batch x 4): pair visits (Gram / pair QR + e), rotated pairs,
  // inner-SVD pair visits (inner sweeps x 2k(2k-1)/2), inner-SVD rotations -- the run's own counts
  // behind the algorithmic flop figure
  int64_t* stats = nullptr;
};
size_t block_ws_bytes(int dtype, int64_t batch, int m, int n, int block_width, int method, bool accv);
int launch_block_svd(int dtype, const BlockLaunch& L, void* ws, cudaStream_t st);

}  // namespace bf
