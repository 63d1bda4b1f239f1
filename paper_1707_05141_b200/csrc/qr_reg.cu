// Register-resident batched Householder QR (reference: qr() qr.py:63-95, batch_qr :98-100).
//
// One CTA of WW warps per matrix, lane = row (R rows per lane, rows >= m are zero), the whole
// m x N matrix in registers with compile-time column indices (the reflector loop is fully
// unrolled, N compile-time).
//   R phase: reflector j from column j (householder_vector, qr.py:26-48), applied to column j
//     itself (R_jj = alpha - tau (v . x)) and to every trailing column (the panel width only
//     reorders independent column updates: the column recurrences are the reference's).
//     The trailing dot products v . a_c are reduced across rows through a shared-memory
//     transpose (each lane writes its partials as a row, each lane sums one column).
//   Q phase (LAPACK dorg2r order, in place over the reflectors): for j = N-1..0 apply H_j to
//     the already-formed columns j+1.. and set column j = H_j e_j  -- the same product
//     H_0 ... H_{N-1} [I; 0] as the reference's backward accumulation (qr.py:90-94).
#include "common.cuh"
#include "internal.h"

namespace bf {

namespace {


// barrier of the WW warps holding one matrix; with several matrices per CTA (kernel template
// G) each group of WW warps uses its own named barrier 1 + group
BF_DEV void wbar(int ww) {
  if (ww > 1) {
    const int id = 1 + (int)(threadIdx.x >> 5) / ww;
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(ww * 32) : "memory");
  } else {
    __syncwarp();
  }
}

// Sum over all rows (all lanes of all WW warps) of K per-lane partials; result in p[] on every
// lane. tb: (WW*32) x TS doubles, wsum: K doubles.
// TS: transpose row stride in doubles (odd, > K) so rows and columns are both conflict-free
template <int K, int WW, int TS>
BF_DEV void rows_allreduce(double (&p)[K > 0 ? K : 1], double* tb, double* wsum, int tid) {
  if (K == 0) return;
  constexpr int ROWS = WW * 32;
#pragma unroll
  for (int c = 0; c < K; ++c) tb[tid * TS + c] = p[c];
  wbar(WW);
  if (K <= 16) {
    // two threads per column, each over half of the rows
    const int c = tid & 15, h = (tid >> 4) & 1;
    if (tid < 32) {
      double a0 = 0, a1 = 0;
      if (c < K) {
#pragma unroll
        for (int r = 0; r < ROWS / 2; r += 2) {
          a0 += tb[(h * (ROWS / 2) + r) * TS + c];
          a1 += tb[(h * (ROWS / 2) + r + 1) * TS + c];
        }
      }
      double v = a0 + a1;
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (h == 0 && c < K) wsum[c] = v;
    }
  } else {
    if (tid < K) {
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int r = 0; r < ROWS; r += 4) {
        a0 += tb[r * TS + tid];
        a1 += tb[(r + 1) * TS + tid];
        a2 += tb[(r + 2) * TS + tid];
        a3 += tb[(r + 3) * TS + tid];
      }
      wsum[tid] = (a0 + a1) + (a2 + a3);
    }
  }
  wbar(WW);
#pragma unroll
  for (int c = 0; c < K; ++c) p[c] = wsum[c];
  wbar(WW);  // tb / wsum reuse
}

template <int WW>
BF_DEV double rows_allreduce1(double x, double* wsum, int tid) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (WW == 1) return x;
  if ((tid & 31) == 0) wsum[40 + (tid >> 5)] = x;
  wbar(WW);
  double t = 0;
#pragma unroll
  for (int q = 0; q < WW; ++q) t += wsum[40 + q];
  wbar(WW);
  return t;
}

}  // namespace

template <int N, int R, int WW>
struct QrReg {
  static constexpr int TSN = N < 32 ? 33 : (N % 2 == 0 ? N + 1 : N + 2);
  template <int J>
  static BF_DEV void factor_col(double (&a)[R][N], double* tau_s, double* tb, double* wsum, int tid, int m) {
    // ---- householder_vector of column J (rows J..m-1)
    double ts = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = tid + r * WW * 32;
      if (row > J && row < m) ts = fma(a[r][J], a[r][J], ts);
    }
    const double tail_sq = rows_allreduce1<WW>(ts, wsum, tid);
    // alpha = a[J][J]: row J lives in thread J % (WW*32), register J / (WW*32)
    constexpr int rJ = J / (WW * 32);
    if (tid == J % (WW * 32)) wsum[48] = a[rJ][J];
    wbar(WW);
    const double alpha = wsum[48];
    wbar(WW);
    double tj = 0.0;
    if (J + 1 < m && tail_sq != 0.0) {  // uniform
      double beta, denom, rden;
      householder_scalars(alpha, tail_sq, beta, tj, denom, rden);
      double acc = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int row = tid + r * WW * 32;
        if (row > J && row < m) {
          const double vi = div_by(a[r][J], denom, rden);
          acc = fma(vi, a[r][J], acc);
          a[r][J] = vi;  // reflector stored below the diagonal
        }
      }
      // reflector applied to its own column: w = tau (v . x); R_JJ = alpha - w
      const double w = (alpha + rows_allreduce1<WW>(acc, wsum, tid)) * tj;
      if (tid == J % (WW * 32)) a[rJ][J] = alpha - w;
      // ---- trailing columns J+1..N-1
      constexpr int K = N - 1 - J;
      if (K > 0) {
        double p[K > 0 ? K : 1];
#pragma unroll
        for (int c = 0; c < K; ++c) {
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int row = tid + r * WW * 32;
            const double v = row == J ? 1.0 : (row > J && row < m ? a[r][J] : 0.0);
            s = fma(v, a[r][J + 1 + c], s);
          }
          p[c] = s;
        }
        rows_allreduce<K, WW, TSN>(p, tb, wsum, tid);
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double wc = p[c] * tj;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int row = tid + r * WW * 32;
            const double v = row == J ? 1.0 : (row > J && row < m ? a[r][J] : 0.0);
            a[r][J + 1 + c] = fma(-v, wc, a[r][J + 1 + c]);
          }
        }
      }
    }
    if (tid == 0) tau_s[J] = tj;
  }

  template <int J>
  static BF_DEV void factor_from(double (&a)[R][N], double* tau_s, double* tb, double* wsum, int tid, int m) {
    if constexpr (J < N) {
      factor_col<J>(a, tau_s, tb, wsum, tid, m);
      factor_from<J + 1>(a, tau_s, tb, wsum, tid, m);
    }
  }

  // dorg2r: column J of Q from H_J, after columns J+1.. are formed
  template <int J>
  static BF_DEV void form_col(double (&a)[R][N], const double* tau_s, double* tb, double* wsum, int tid, int m) {
    const double tj = tau_s[J];
    constexpr int K = N - 1 - J;
    // reflector v_J (unit at row J) from the stored lower part of column J
    double v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = tid + r * WW * 32;
      v[r] = row == J ? 1.0 : (row > J && row < m ? a[r][J] : 0.0);
    }
    if (K > 0 && tj != 0.0) {  // uniform
      double p[K > 0 ? K : 1];
#pragma unroll
      for (int c = 0; c < K; ++c) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) s = fma(v[r], a[r][J + 1 + c], s);
        p[c] = s;
      }
      rows_allreduce<K, WW, TSN>(p, tb, wsum, tid);
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const double wc = p[c] * tj;
#pragma unroll
        for (int r = 0; r < R; ++r) a[r][J + 1 + c] = fma(-v[r], wc, a[r][J + 1 + c]);
      }
    }
    // Q[:, J] = e_J - tau v (rows < J are zero)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = tid + r * WW * 32;
      a[r][J] = row < J ? 0.0 : (row == J ? 1.0 - tj : -tj * v[r]);
    }
  }

  template <int J>
  static BF_DEV void form_from(double (&a)[R][N], const double* tau_s, double* tb, double* wsum, int tid, int m) {
    if constexpr (J >= 0) {
      form_col<J>(a, tau_s, tb, wsum, tid, m);
      form_from<J - 1>(a, tau_s, tb, wsum, tid, m);
    }
  }
};

// G > 1: G independent groups of WW warps per CTA, each on its own matrix with its own
// shared-memory slice (and named barrier). The unrolled kernel is tens of thousands of
// instructions long; warps launched together walk it roughly in step and share i-cache lines.
#ifndef BF_QR40_G
#define BF_QR40_G 1  // measured: G = 2 is slower for 128x40 (1.98 vs 1.93 ms)
#endif
#ifndef BF_QR_MINB
#define BF_QR_MINB 1
#endif
#ifndef BF_QR_G
#define BF_QR_G 4  // measured: 64x32 x10000 0.590 -> 0.571 ms (G = 2: 0.580)
#endif
template <int N, int R, int WW, int G = 1>
__global__ void __launch_bounds__(WW * 32 * G, BF_QR_MINB) qr_reg_kernel(int64_t batch, int m, const double* A, int64_t as,
                                                             double* Q, int64_t qs, double* Rout, int64_t rs) {
  static_assert(G * WW <= 15, "one named barrier per matrix group");
  __shared__ double tb_all[G][WW * 32 * QrReg<N, R, WW>::TSN];
  __shared__ double wsum_all[G][64];
  __shared__ double tau_all[G][N];
  const int grp = G > 1 ? (int)(threadIdx.x / (WW * 32)) : 0;
  double* tb = tb_all[grp];
  double* wsum = wsum_all[grp];
  double* tau_s = tau_all[grp];
  const int tid = G > 1 ? (int)(threadIdx.x % (WW * 32)) : (int)threadIdx.x;
  for (int64_t b = (int64_t)blockIdx.x * G + grp; b < batch; b += (int64_t)gridDim.x * G) {
    const double* Ab = A + b * as;
    double a[R][N];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = tid + r * WW * 32;
#pragma unroll
      for (int c = 0; c < N; ++c) a[r][c] = row < m ? Ab[(size_t)c * m + row] : 0.0;
    }
    QrReg<N, R, WW>::template factor_from<0>(a, tau_s, tb, wsum, tid, m);
    // R: n x n upper triangle with exact zeros below (qr.py:84-85, :95)
    double* Rb = Rout + b * rs;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = tid + r * WW * 32;
      if (row < N) {
#pragma unroll
        for (int c = 0; c < N; ++c) Rb[(size_t)c * N + row] = c >= row ? a[r][c] : 0.0;
      }
    }
    wbar(WW);
    QrReg<N, R, WW>::template form_from<N - 1>(a, tau_s, tb, wsum, tid, m);
    double* Qb = Q + b * qs;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = tid + r * WW * 32;
      if (row < m) {
#pragma unroll
        for (int c = 0; c < N; ++c) Qb[(size_t)c * m + row] = a[r][c];
      }
    }
    wbar(WW);
  }
}

template <int N, int R, int WW, int G = 1>
static int launch_qr_reg_t(int64_t batch, int m, const double* a, int64_t as, double* q, int64_t qs, double* r,
                           int64_t rs, cudaStream_t st) {
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qr_reg_kernel<N, R, WW, G>, WW * 32 * G, 0);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)per_sm * sms;
  const int64_t need = (batch + G - 1) / G;
  const int grid = (int)(need < cap ? need : cap);
  qr_reg_kernel<N, R, WW, G><<<grid, WW * 32 * G, 0, st>>>(batch, m, a, as, q, qs, r, rs);
  return (int)cudaGetLastError();
}

bool qr_reg_covers(int m, int n) { return ((n == 32 || n == 16) && m <= 64) || (n == 40 && m <= 128); }

// Returns -1 if no register configuration covers (m, n).
int launch_qr_reg(int dtype, int64_t batch, int m, int n, const void* a, int64_t as, void* q, int64_t qs, void* r,
                  int64_t rs, cudaStream_t st) {
  if (dtype != 0) return -1;
  const double* A = (const double*)a;
  double* Q = (double*)q;
  double* Rr = (double*)r;
  if (!qr_reg_covers(m, n)) return -1;
  if (n == 32 && m <= 64) return launch_qr_reg_t<32, 2, 1, BF_QR_G>(batch, m, A, as, Q, qs, Rr, rs, st);
  if (n == 16 && m <= 64) return launch_qr_reg_t<16, 2, 1>(batch, m, A, as, Q, qs, Rr, rs, st);
  if (n == 40 && m <= 128) return launch_qr_reg_t<40, 2, 2, BF_QR40_G>(batch, m, A, as, Q, qs, Rr, rs, st);
  return -1;
}

}  // namespace bf
