// CTA-cooperative Householder QR building block (matrix staged in shared memory).
//
// Semantics of the reference qr() (qr.py:63-95): reflector j from column j
// (householder_vector, qr.py:26-48; beta = -copysign(hypot(alpha, ||tail||), alpha),
// tau = (beta - alpha)/beta, v = x/(alpha - beta), v_0 = 1), applied to column j
// itself and to every trailing column in order (the panel width only reorders
// independent column updates, so any blocking gives the same column recurrences);
// explicit reduced Q = H_0 ... H_{n-1} I (qr.py:90-94).
#pragma once
#include "common.cuh"

namespace bf {

// Factor R (m x n, ld) in place: on exit the upper triangle holds R, rows below the
// diagonal hold v (v_0 = 1 implicit), tau[j] the reflector scalars.
template <typename T, int PB>
BF_DEV void qr_factor_cta(T* R, int ldr, int m, int n, T* tau) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int j = 0; j < n; ++j) {
    T* x = R + (size_t)j * ldr;
    if (warp == 0) {
      T ts = 0;
      for (int i = j + 1 + lane; i < m; i += 32) ts = fma(x[i], x[i], ts);
      double tail_sq = (double)warp_allreduce_sum(ts);
      double alpha = (double)x[j];
      double tj = 0.0;
      if (j + 1 < m && tail_sq != 0.0) {
        double beta = -copysign(hypot(alpha, sqrt(tail_sq)), alpha);
        tj = (beta - alpha) / beta;
        const T denom = (T)(alpha - beta);
        T acc = 0;
        for (int i = j + 1 + lane; i < m; i += 32) {
          T xi = x[i];
          T vi = xi / denom;
          acc = fma(vi, xi, acc);
          x[i] = vi;
        }
        // reflector applied to its own column: w = tau * (v . x); R_jj = alpha - w
        T w = (x[j] + warp_allreduce_sum(acc)) * (T)tj;
        __syncwarp();
        if (lane == 0) x[j] = x[j] - w;
      }
      if (lane == 0) tau[j] = (T)tj;
    }
    __syncthreads();
    const T tj = tau[j];
    if (tj != T(0)) {
      const int ncols = n - j - 1;
      for (int base = warp; base < ncols; base += nwarps * PB) {
        T d[PB];
#pragma unroll
        for (int b = 0; b < PB; ++b) {
          int c = j + 1 + base + b * nwarps;
          d[b] = 0;
          if (base + b * nwarps < ncols) {
            const T* col = R + (size_t)c * ldr;
            for (int i = j + 1 + lane; i < m; i += 32) d[b] = fma(x[i], col[i], d[b]);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int b = 0; b < PB; ++b) d[b] += shfl_xor(d[b], o);
T w[PB];
#pragma unroll
        for (int b = 0; b < PB; ++b)
          w[b] = base + b * nwarps < ncols ? (R[(size_t)(j + 1 + base + b * nwarps) * ldr + j] + d[b]) * tj : T(0);
        __syncwarp();
#pragma unroll
        for (int b = 0; b < PB; ++b) {
          if (base + b * nwarps >= ncols) continue;
          T* col = R + (size_t)(j + 1 + base + b * nwarps) * ldr;
          for (int i = j + 1 + lane; i < m; i += 32) col[i] = fma(-x[i], w[b], col[i]);
          if (lane == 0) col[j] -= w[b];
        }
      }
    }
    __syncthreads();
  }
}

// Explicit Q (m x n, ld) from the factored storage: Q = H_0 ... H_{n-1} [I; 0].
template <typename T, int PB>
BF_DEV void qr_form_q_cta(const T* R, int ldr, const T* tau, T* Q, int ldq, int m, int n) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int c = warp; c < n; c += nwarps)
    for (int i = lane; i < m; i += 32) Q[(size_t)c * ldq + i] = (i == c) ? T(1) : T(0);
  __syncthreads();
  for (int j = n - 1; j >= 0; --j) {
    const T tj = tau[j];
    if (tj == T(0)) continue;  // uniform across the CTA
    const T* v = R + (size_t)j * ldr;
    const int ncols = n - j;
    for (int base = warp; base < ncols; base += nwarps * PB) {
      T d[PB];
#pragma unroll
      for (int b = 0; b < PB; ++b) {
        d[b] = 0;
        if (base + b * nwarps < ncols) {
          const T* col = Q + (size_t)(j + base + b * nwarps) * ldq;
          for (int i = j + 1 + lane; i < m; i += 32) d[b] = fma(v[i], col[i], d[b]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int b = 0; b < PB; ++b) d[b] += shfl_xor(d[b], o);
T w[PB];
#pragma unroll
      for (int b = 0; b < PB; ++b)
        w[b] = base + b * nwarps < ncols ? (Q[(size_t)(j + base + b * nwarps) * ldq + j] + d[b]) * tj : T(0);
      __syncwarp();
#pragma unroll
      for (int b = 0; b < PB; ++b) {
        if (base + b * nwarps >= ncols) continue;
        T* col = Q + (size_t)(j + base + b * nwarps) * ldq;
        for (int i = j + 1 + lane; i < m; i += 32) col[i] = fma(-v[i], w[b], col[i]);
        if (lane == 0) col[j] -= w[b];
      }
    }
    __syncthreads();
  }
}

}  // namespace bf
