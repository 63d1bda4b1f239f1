// Device kernels behind the reference's public helper functions (the names batchfact re-exports,
// /root/reference/pkg/src/batchfact/__init__.py:3-23, plus blockjacobi.scaled_offdiag):
//   householder_vector   qr.py:26-48        jacobi_rotation     jacobi.py:68-80
//   off_orthogonality    jacobi.py:83-99    scaled_offdiag      blockjacobi.py:57-76
//   syrk                 core.py:68-78      frobenius           core.py:81-86
//   gemm (alpha/beta)    core.py:36-65      (the product itself is bf_gemm_batched_*)
// All batched over B independent entries (one CTA or thread per entry); the drop-in calls them
// with B = 1. These are not on the factorisation hot path; the hot kernels inline the same
// formulas (common.cuh, jacobi_cta.cuh).
#include <math.h>

#include "common.cuh"
#include "internal.h"

namespace bf {

template <typename T>
BF_DEV T block_sum(T v, T* red) {
  v = warp_allreduce_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T t = T(0);
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}

template <typename T>
BF_DEV T block_max(T v, T* red) {
  v = warp_allreduce_max(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T t = red[0];
  for (int w = 1; w < nw; ++w) t = red[w] > t ? red[w] : t;
  return t;
}

// householder_vector (qr.py:26-48): v[0] = 1, v[1:] = x[1:] / (alpha - beta),
// beta = -copysign(hypot(alpha, ||x[1:]||), alpha), tau = (beta - alpha) / beta; a zero or
// empty tail gives the identity reflector (tau = 0, v = x with v[0] = 1).
template <typename T>
__global__ void __launch_bounds__(256) householder_kernel(int64_t batch, int len, const T* x, T* v, T* tau) {
  __shared__ T red[32];
  const int64_t b = blockIdx.x;
  if (b >= batch) return;
  const T* xb = x + b * (int64_t)len;
  T* vb = v + b * (int64_t)len;
  T ts = T(0);
  for (int i = 1 + threadIdx.x; i < len; i += blockDim.x) ts = fma(xb[i], xb[i], ts);
  const T tail_sq = block_sum(ts, red);
  const T alpha = xb[0];
  if (len == 1 || tail_sq == T(0)) {
    for (int i = threadIdx.x; i < len; i += blockDim.x) vb[i] = i == 0 ? T(1) : xb[i];
    if (threadIdx.x == 0) tau[b] = T(0);
    return;
  }
  const T beta = -copysign(hypot(alpha, sqrt(tail_sq)), alpha);
  const T denom = alpha - beta;
  for (int i = threadIdx.x; i < len; i += blockDim.x) vb[i] = i == 0 ? T(1) : xb[i] / denom;
  if (threadIdx.x == 0) tau[b] = (beta - alpha) / beta;
}

// jacobi_rotation (jacobi.py:68-80), the reference's formula with IEEE operations:
// g_pq == 0 -> (1, 0); zeta = (g_qq - g_pp) / (2 g_pq); t = sign(zeta) / (|zeta| + hypot(1, zeta));
// c = 1 / hypot(1, t); s = c t.
__global__ void rotation_kernel(int64_t batch, const double* gpp, const double* gpq, const double* gqq, double* c,
                                double* s) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const double q = gpq[b];
  if (q == 0.0) {
    c[b] = 1.0;
    s[b] = 0.0;
    return;
  }
  const double zeta = (gqq[b] - gpp[b]) / (2.0 * q);
  const double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
  const double cc = 1.0 / hypot(1.0, t);
  c[b] = cc;
  s[b] = cc * t;
}

// max over i != j of |g_ij| / (d_i d_j) with d_i = sqrt(|g_ii|), g = A^T A (off_orthogonality:
// zero columns contribute 0, jacobi.py:83-99) or g given (scaled_offdiag: 0/0 -> 0, x/0 -> +inf,
// blockjacobi.py:57-76). One CTA per entry; gram = 1 forms g_ij = a_i . a_j on the fly.
template <typename T>
__global__ void __launch_bounds__(256) offdiag_kernel(int64_t batch, int m, int n, const T* a, int gram, T* out) {
  __shared__ T red[32];
  const int64_t b = blockIdx.x;
  if (b >= batch) return;
  const T* ab = a + b * (int64_t)m * n;  // gram: m x n columns; else n x n
  auto g = [&](int i, int j) -> T {
    if (!gram) return ab[(int64_t)j * n + i];
    T acc = T(0);
    for (int r = 0; r < m; ++r) acc = fma(ab[(int64_t)i * m + r], ab[(int64_t)j * m + r], acc);
    return acc;
  };
  T best = T(0);
  for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    if (i == j) continue;
    const T di = sqrt(fabs(g(i, i))), dj = sqrt(fabs(g(j, j)));
    const T den = di * dj, num = fabs(g(i, j));
    T r;
    if (den > T(0))
      r = num / den;
    else
      r = (!gram && num > T(0)) ? T(INFINITY) : T(0);
    best = r > best ? r : best;
  }
  best = block_max(best, red);
  if (threadIdx.x == 0) out[b] = best;
}

// syrk (core.py:68-78): G = A^T A with the upper triangle mirrored -- G[i,j] and G[j,i] bitwise
// equal. One thread per (i <= j) element.
template <typename T>
__global__ void syrk_kernel(int64_t batch, int m, int k, const T* a, T* g) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)k * k;
  if (e >= batch * per) return;
  const int64_t b = e / per;
  const int i = (int)((e % per) % k), j = (int)((e % per) / k);
  if (i > j) return;
  const T* ab = a + b * (int64_t)m * k;
  T acc = T(0);
  for (int r = 0; r < m; ++r) acc = fma(ab[(int64_t)i * m + r], ab[(int64_t)j * m + r], acc);
  T* gb = g + b * per;
  gb[(int64_t)j * k + i] = acc;
  gb[(int64_t)i * k + j] = acc;
}

// frobenius (core.py:81-86): scaled two-pass norm (max |a| first), overflow- and underflow-safe
// like the LAPACK norm numpy uses; 0 for an empty matrix.
template <typename T>
__global__ void __launch_bounds__(256) frobenius_kernel(int64_t batch, int64_t count, const T* a, T* out) {
  __shared__ T red[32];
  const int64_t b = blockIdx.x;
  if (b >= batch) return;
  const T* ab = a + b * count;
  T mx = T(0), nan = T(0);
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    const T x = fabs(ab[i]);
    mx = x > mx ? x : mx;
    nan += x != x ? T(1) : T(0);
  }
  mx = block_max(mx, red);
  nan = block_sum(nan, red);
  if (nan > T(0) || !(mx > T(0)) || isinf(mx)) {  // nan -> nan, inf -> inf, all zero -> 0
    if (threadIdx.x == 0) out[b] = nan > T(0) ? T(NAN) : mx;
    return;
  }
  const T inv = T(1) / mx;
  T acc = T(0);
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    const T y = ab[i] * inv;
    acc = fma(y, y, acc);
  }
  acc = block_sum(acc, red);
  if (threadIdx.x == 0) out[b] = mx * sqrt(acc);
}

// gemm epilogue (core.py:36-65): out = alpha * P + beta * C (beta == 0 ignores C entirely, so no
// NaN/Inf leaks from it; alpha == 0 gives exact zeros)
template <typename T>
__global__ void axpby_kernel(int64_t n, T alpha, const T* p, T beta, const T* c, T* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T r = alpha == T(0) ? T(0) : (alpha == T(1) ? p[i] : alpha * p[i]);
  if (beta != T(0)) r = r + (beta == T(1) ? c[i] : beta * c[i]);
  out[i] = r;
}

// float32 <-> float64 widening / rounding for the float32 entry points that compute on the float64
// tiers (api.cu); grid-stride, 2 elements per thread per iteration
template <typename S, typename D>
__global__ void __launch_bounds__(256) cast_kernel(int64_t n, const S* __restrict__ src, D* __restrict__ dst) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = (D)src[i];
}

static unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

template <typename S, typename D>
int launch_cast(int64_t n, const S* src, D* dst, cudaStream_t st) {
  if (n <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256, cap = (int64_t)sms * 8;
  cast_kernel<S, D><<<(unsigned)(want < cap ? want : cap), 256, 0, st>>>(n, src, dst);
  return (int)cudaGetLastError();
}
template int launch_cast<float, double>(int64_t, const float*, double*, cudaStream_t);
template int launch_cast<double, float>(int64_t, const double*, float*, cudaStream_t);

template <typename T>
int launch_householder(int64_t batch, int len, const T* x, T* v, T* tau, cudaStream_t st) {
  if (batch == 0 || len == 0) return 0;
  householder_kernel<T><<<(unsigned)batch, 256, 0, st>>>(batch, len, x, v, tau);
  return (int)cudaGetLastError();
}
template int launch_householder<double>(int64_t, int, const double*, double*, double*, cudaStream_t);
template int launch_householder<float>(int64_t, int, const float*, float*, float*, cudaStream_t);

int launch_rotation(int64_t batch, const double* gpp, const double* gpq, const double* gqq, double* c, double* s,
                    cudaStream_t st) {
  if (batch == 0) return 0;
  rotation_kernel<<<blocks_for(batch, 128), 128, 0, st>>>(batch, gpp, gpq, gqq, c, s);
  return (int)cudaGetLastError();
}

template <typename T>
int launch_offdiag(int64_t batch, int m, int n, const T* a, int gram, T* out, cudaStream_t st) {
  if (batch == 0) return 0;
  offdiag_kernel<T><<<(unsigned)batch, 256, 0, st>>>(batch, m, n, a, gram, out);
  return (int)cudaGetLastError();
}
template int launch_offdiag<double>(int64_t, int, int, const double*, int, double*, cudaStream_t);
template int launch_offdiag<float>(int64_t, int, int, const float*, int, float*, cudaStream_t);

template <typename T>
int launch_syrk(int64_t batch, int m, int k, const T* a, T* g, cudaStream_t st) {
  if (batch == 0 || k == 0) return 0;
  syrk_kernel<T><<<blocks_for(batch * (int64_t)k * k, 128), 128, 0, st>>>(batch, m, k, a, g);
  return (int)cudaGetLastError();
}
template int launch_syrk<double>(int64_t, int, int, const double*, double*, cudaStream_t);
template int launch_syrk<float>(int64_t, int, int, const float*, float*, cudaStream_t);

template <typename T>
int launch_frobenius(int64_t batch, int64_t count, const T* a, T* out, cudaStream_t st) {
  if (batch == 0) return 0;
  if (count == 0) return (int)cudaMemsetAsync(out, 0, sizeof(T) * (size_t)batch, st);
  frobenius_kernel<T><<<(unsigned)batch, 256, 0, st>>>(batch, count, a, out);
  return (int)cudaGetLastError();
}
template int launch_frobenius<double>(int64_t, int64_t, const double*, double*, cudaStream_t);
template int launch_frobenius<float>(int64_t, int64_t, const float*, float*, cudaStream_t);

template <typename T>
int launch_axpby(int64_t n, T alpha, const T* p, T beta, const T* c, T* out, cudaStream_t st) {
  if (n == 0) return 0;
  axpby_kernel<T><<<blocks_for(n, 256), 256, 0, st>>>(n, alpha, p, beta, c, out);
  return (int)cudaGetLastError();
}
template int launch_axpby<double>(int64_t, double, const double*, double, const double*, double*, cudaStream_t);
template int launch_axpby<float>(int64_t, float, const float*, float, const float*, float*, cudaStream_t);

}  // namespace bf
