// Batched one-sided block Jacobi SVD: global-memory tier.
//
// Reference: block_svd blockjacobi.py:84-168, batch_block_svd :171-174.
// W (m x n_pad) and V (n_pad x n_pad) live in a global (L2-resident) workspace.
// Each round-robin step over the n_blocks block columns is one kernel launch with
// one CTA per (matrix, block pair); pairs of a step are disjoint, so running them
// concurrently is exactly the reference's serial order (blockjacobi.py:110-111,120).
//   gram  : G = pair^T pair (syrk, core.py:68-78), e = scaled_offdiag(G); if e > tol the
//           inner round-robin SVD of G (no V) gives the rotation U_G; pair <- pair U_G with
//           exactly-null directions zeroed (blockjacobi.py:124-134).
//   direct: QR of the pair, e = scaled_offdiag(R); inner SVD of R with V; pair <-
//           Q U_R diag(sigma) (applied as H_0..H_{2k-1} [U_R diag(sigma); 0]), rotation V_R
//           (blockjacobi.py:135-143).
// A per-sweep finalize kernel records e_history, counts the sweep and retires converged
// matrices (blockjacobi.py:150-154); converged matrices simply stop (per-matrix, :171-174).
#include <mutex>
#include <utility>
#include <vector>

#include <cudaTypedefs.h>

#include "internal.h"
#include "jacobi_cta.cuh"
#include "qr_cta.cuh"
#include "block_gemm.cuh"

namespace bf {

template <typename T>
struct BJArgs {
  int64_t batch;
  int m, n, n_pad, k, nb;  // k = block width, nb = n_pad / k
  T* W;                    // batch x m x n_pad
  T* V;                    // batch x n_pad x n_pad or null
  T* P;                    // direct method: per-CTA pair scratch (batch*nb/2 x m x 2k) when not in smem
  double* e_sweep;         // batch
  uint8_t* active;         // batch
  int32_t* sweeps;
  uint8_t* conv;
  T* e_hist;
  int max_sweeps;
  double tol, tol_inner;
  bool p_in_smem;
  int64_t* stats;   // batch x 4 work counters or null (BlockLaunch::stats)
  int32_t* in_sw;   // batched pipelines: per-slot accumulated inner-SVD sweeps
  int64_t* in_rot;  // ... and inner-SVD rotations
};

BF_DEV void atomic_max_pos(double* addr, double v) {
  // non-negative doubles (incl. +inf) order like their bit patterns
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}

// scaled_offdiag (blockjacobi.py:57-76) of a square 2k x 2k matrix in smem, CTA-wide.
template <typename T>
BF_DEV double scaled_offdiag_cta(const T* G, int ld, int nn, double* red) {
  if (threadIdx.x == 0) *red = 0.0;
  __syncthreads();
  double best = 0.0;
  for (int e = threadIdx.x; e < nn * nn; e += blockDim.x) {
    int j = e / nn, i = e % nn;
    if (i == j) continue;
    T di = (T)sqrt((double)fabs((double)G[(size_t)i * ld + i]));
    T dj = (T)sqrt((double)fabs((double)G[(size_t)j * ld + j]));
    T den = di * dj;
    T num = G[(size_t)j * ld + i];
    num = num < T(0) ? -num : num;
    double rt = den > T(0) ? (double)(num / den) : (num > T(0) ? __longlong_as_double(0x7ff0000000000000LL) : 0.0);
    best = rt > best ? rt : best;
  }
  best = warp_allreduce_max(best);
  if ((threadIdx.x & 31) == 0 && best > 0.0) atomic_max_pos(red, best);
  __syncthreads();
  double r = *red;
  __syncthreads();
  return r;
}

// column c (0..2k-1) of the block pair -> global column
BF_DEV int pair_col(int c, int k, int bi, int bj) { return c < k ? bi * k + c : bj * k + (c - k); }

// rows x 2k panel of M (ld) times R (2k x 2k, smem): out = panel @ R, in place, row chunks
// through smem. zero_sig: zero output columns whose sigma == 0 (gram path).
template <typename T>
BF_DEV void pair_times_rot(T* M, int ld, int rows, int k, int bi, int bj, const T* R, T* chunk, const T* sig,
                           bool zero_null) {
  const int kk = 2 * k;
  const int CH = 32;
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int r0 = 0; r0 < rows; r0 += CH) {
    int nr = rows - r0 < CH ? rows - r0 : CH;
    for (int e = tid; e < kk * CH; e += nth) {
      int c = e / CH, r = e % CH;
      chunk[c * CH + r] = r < nr ? M[(size_t)pair_col(c, k, bi, bj) * ld + r0 + r] : T(0);
    }
    __syncthreads();
    for (int e = tid; e < kk * CH; e += nth) {
      int t = e / CH, r = e % CH;
      if (r >= nr) continue;
      T acc = 0;
      for (int u = 0; u < kk; ++u) acc = fma(chunk[u * CH + r], R[(size_t)t * kk + u], acc);
      if (zero_null && !(sig[t] != T(0))) acc = T(0);
      M[(size_t)pair_col(t, k, bi, bj) * ld + r0 + r] = acc;
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void __launch_bounds__(256) bj_gram_step(BJArgs<T> a, int step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  if (b >= a.batch || !a.active[b]) return;
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, kk = 2 * k, m = a.m, tid = threadIdx.x;
  T* G = reinterpret_cast<T*>(smem_raw);  // kk x kk; inner W
  T* U = G + kk * kk;                     // kk x kk rotation
  T* chunk = U + kk * kk;                 // kk x 32
  T* sig = chunk + kk * 32;               // kk
  T* cand = sig + kk;                     // 2 kk
  int* order = reinterpret_cast<int*>(cand + 2 * kk);
  int* counters = order + kk;
  double* red = reinterpret_cast<double*>(((uintptr_t)(counters + 4) + 7) & ~(uintptr_t)7);
  T* Wb = a.W + b * (int64_t)m * a.n_pad;

  // ---- G = pair^T pair, rows streamed in chunks of 32 (syrk, core.py:68-78)
  for (int e = tid; e < kk * kk; e += blockDim.x) G[e] = T(0);
  T acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = T(0);
  const int ne = kk * kk;
  for (int r0 = 0; r0 < m; r0 += 32) {
    int nr = m - r0 < 32 ? m - r0 : 32;
    __syncthreads();
    for (int e = tid; e < kk * 32; e += blockDim.x) {
      int c = e / 32, r = e % 32;
      chunk[c * 32 + r] = r < nr ? Wb[(size_t)pair_col(c, k, bi, bj) * m + r0 + r] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      int e = tid + q * 256;
      if (e < ne) {
        int j = e / kk, i = e % kk;
        if (i <= j) {
          T s = acc[q];
          for (int r = 0; r < 32; ++r) s = fma(chunk[i * 32 + r], chunk[j * 32 + r], s);
          acc[q] = s;
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    int e = tid + q * 256;
    if (e < ne) {
      int j = e / kk, i = e % kk;
      if (i <= j) {
        G[(size_t)j * kk + i] = acc[q];
        G[(size_t)i * kk + j] = acc[q];
      }
    }
  }
  __syncthreads();
  // ---- convergence measure before the update (blockjacobi.py:126-129)
  double e = scaled_offdiag_cta<T>(G, kk, kk, red);
  if (tid == 0) {
    atomic_max_pos(a.e_sweep + b, e);
    bj_count(a.stats, b, e > a.tol);
  }
  if (e <= a.tol) return;
  // ---- inner round-robin SVD of G without V (blockjacobi.py:130, _inner_options :79-81)
  const SweepStats ist = jacobi_sweeps<T, 4>(G, kk, (T*)nullptr, kk, kk, kk, kk, 1, a.tol_inner, 30, counters);
  if (tid == 0 && a.stats) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + 4 * b + 2),
              (unsigned long long)ist.sweeps * (unsigned long long)(kk * (kk - 1) / 2));
    atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + 4 * b + 3), (unsigned long long)ist.rotations);
  }
  extract_svd_cta<T>(G, kk, (const T*)nullptr, kk, kk, kk, kk, 0, U, kk, sig, (T*)nullptr, kk, chunk, order, cand,
                     counters + 2);
  // (extract used `chunk` as its unsorted-norm scratch; `sig` holds the sorted sigma)
  pair_times_rot<T>(Wb, m, m, k, bi, bj, U, chunk, sig, true);
  if (a.V) pair_times_rot<T>(a.V + b * (int64_t)a.n_pad * a.n_pad, a.n_pad, a.n_pad, k, bi, bj, U, chunk, sig, false);
}

template <typename T>
__global__ void __launch_bounds__(256) bj_direct_step(BJArgs<T> a, int step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  if (b >= a.batch || !a.active[b]) return;
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, kk = 2 * k, m = a.m, tid = threadIdx.x;
  T* Rw = reinterpret_cast<T*>(smem_raw);  // kk x kk inner W (R)
  T* Vi = Rw + kk * kk;                    // kk x kk inner V
  T* Vr = Vi + kk * kk;                    // kk x kk rotation V_R
  T* Ur = Vr + kk * kk;                    // kk x kk U_R (scaled later)
  T* sig = Ur + kk * kk;                   // kk
  T* sig2 = sig + kk;                      // kk (sorted sigma)
  T* tau = sig2 + kk;                      // kk
  T* cand = tau + kk;                      // 2 kk
  int* order = reinterpret_cast<int*>(cand + 2 * kk);
  int* counters = order + kk;
  double* red = reinterpret_cast<double*>(((uintptr_t)(counters + 4) + 7) & ~(uintptr_t)7);
  T* Pm = a.p_in_smem ? reinterpret_cast<T*>(red + 2) : a.P + (int64_t)blockIdx.x * m * kk;
  T* Wb = a.W + b * (int64_t)m * a.n_pad;

  for (int e = tid; e < m * kk; e += blockDim.x) {
    int c = e / m, r = e % m;
    Pm[e] = Wb[(size_t)pair_col(c, k, bi, bj) * m + r];
  }
  __syncthreads();
  qr_factor_cta<T, 4>(Pm, m, m, kk, tau);  // qr(pair) (blockjacobi.py:136)
  for (int e = tid; e < kk * kk; e += blockDim.x) {
    int j = e / kk, i = e % kk;
    Rw[e] = i <= j ? Pm[(size_t)j * m + i] : T(0);
    Vi[e] = i == j ? T(1) : T(0);
  }
  __syncthreads();
  double e = scaled_offdiag_cta<T>(Rw, kk, kk, red);
  if (tid == 0) {
    atomic_max_pos(a.e_sweep + b, e);
    bj_count(a.stats, b, e > a.tol);
  }
  if (e <= a.tol) return;
  const SweepStats ist = jacobi_sweeps<T, 4>(Rw, kk, Vi, kk, kk, kk, kk, 1, a.tol_inner, 30, counters);
  if (tid == 0 && a.stats) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + 4 * b + 2),
              (unsigned long long)ist.sweeps * (unsigned long long)(kk * (kk - 1) / 2));
    atomicAdd(reinterpret_cast<unsigned long long*>(a.stats + 4 * b + 3), (unsigned long long)ist.rotations);
  }
  extract_svd_cta<T>(Rw, kk, Vi, kk, kk, kk, kk, kk, Ur, kk, sig2, Vr, kk, sig, order, cand, counters + 2);
  // new pair = H_0 ... H_{kk-1} [U_R diag(sigma); 0]  (== (Q @ U_R) * sigma, blockjacobi.py:143)
  for (int e2 = tid; e2 < m * kk; e2 += blockDim.x) {
    int c = e2 / m, r = e2 % m;
    Wb[(size_t)pair_col(c, k, bi, bj) * m + r] = r < kk ? Ur[(size_t)c * kk + r] * sig2[c] : T(0);
  }
  __syncthreads();
  {
    const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int j = kk - 1; j >= 0; --j) {
      const T tj = tau[j];
      if (tj == T(0)) continue;
      const T* v = Pm + (size_t)j * m;
      for (int c = warp; c < kk; c += nwarps) {
        T* col = Wb + (size_t)pair_col(c, k, bi, bj) * m;
        T d = 0;
        for (int i = j + 1 + lane; i < m; i += 32) d = fma(v[i], col[i], d);
        d = warp_allreduce_sum(d);
        T w = (col[j] + d) * tj;
        __syncwarp();
        for (int i = j + 1 + lane; i < m; i += 32) col[i] = fma(-v[i], w, col[i]);
        if (lane == 0) col[j] -= w;
      }
      __syncthreads();
    }
  }
  if (a.V) pair_times_rot<T>(a.V + b * (int64_t)a.n_pad * a.n_pad, a.n_pad, a.n_pad, k, bi, bj, Vr, Ur, sig2, false);
}

// ---- batched direct method (fp64, 2k <= 64): bj_dqr -> register-tier inner SVD of R with V ->
// bj_dapply (+ bj_rot_mma on the V pair). Same operations as bj_direct_step, with the inner SVD
// taken out of the per-pair CTA and run batched over all active pairs of the step.
struct BDArgs {
  double* P;    // slots x m x kk: the factored pair (reflectors below the diagonal)
  double* tau;  // slots x kk
  double* G;    // slots x kk x kk: R (inner SVD input)
  double* U;    // slots x kk x kk: U_R (sorted)
  double* S;    // slots x kk: sigma (sorted)
  uint8_t* pact;
};

// qr(pair) (blockjacobi.py:136), e = scaled_offdiag(R) (:137), skip e <= tol (:139-140)
__global__ void __launch_bounds__(256) bj_dqr(BJArgs<double> a, BDArgs d, int step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  const int64_t slot = blockIdx.x;
  if (b >= a.batch) return;
  if (!a.active[b]) {
    if (threadIdx.x == 0) d.pact[slot] = 0;
    return;
  }
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, kk = 2 * k, m = a.m, tid = threadIdx.x;
  double* Pm = reinterpret_cast<double*>(smem_raw);  // m x kk
  double* tau = Pm + (size_t)m * kk;                 // kk
  double* red = tau + kk;                            // 2
  const double* Wb = a.W + b * (int64_t)m * a.n_pad;
  for (int e = tid; e < m * kk; e += blockDim.x) {
    const int c = e / m, r = e % m;
    Pm[e] = Wb[(size_t)pair_col(c, k, bi, bj) * m + r];
  }
  __syncthreads();
  qr_factor_cta<double, 4>(Pm, m, m, kk, tau);
  double* G = d.G + slot * kk * kk;
  for (int e = tid; e < kk * kk; e += blockDim.x) {
    const int j = e / kk, i = e % kk;
    G[e] = i <= j ? Pm[(size_t)j * m + i] : 0.0;
  }
  double* Pg = d.P + slot * (int64_t)m * kk;
  for (int e = tid; e < m * kk; e += blockDim.x) Pg[e] = Pm[e];
  if (tid < kk) d.tau[slot * kk + tid] = tau[tid];
  __syncthreads();
  // scaled_offdiag of R (read back from the smem copy: rows < kk of Pm, upper triangle)
  double best = 0.0;
  for (int e = tid; e < kk * kk; e += blockDim.x) {
    const int j = e / kk, i = e % kk;
    if (i == j) continue;
    const double gij = i <= j ? Pm[(size_t)j * m + i] : 0.0;
    const double den = sqrt(fabs(Pm[(size_t)i * m + i])) * sqrt(fabs(Pm[(size_t)j * m + j]));
    const double num = fabs(gij);
    const double rt = den > 0.0 ? num / den : (num > 0.0 ? __longlong_as_double(0x7ff0000000000000LL) : 0.0);
    best = rt > best ? rt : best;
  }
  best = warp_allreduce_max(best);
  if (tid == 0) red[0] = 0.0;
  __syncthreads();
  if ((tid & 31) == 0 && best > 0.0) atomic_max_pos(red, best);
  __syncthreads();
  if (tid == 0) {
    atomic_max_pos(a.e_sweep + b, red[0]);
    d.pact[slot] = red[0] > a.tol ? 1 : 0;
    bj_count(a.stats, b, red[0] > a.tol);
  }
}

// Register-resident pair QR for m <= 256 (same contract and outputs as bj_dqr): 256 threads,
// thread r owns row r of the m x 64 pair in registers, the reflector loop unrolled so column
// indices are compile-time. Per reflector J: the tail norm and alpha (one CTA reduction), the
// scalars of householder_vector (qr.py:26-48), the dots v . a_c for c = J..63 in one pass (c = J
// is v . x, giving R_JJ = alpha - tau (v . x) as the reference applies the reflector to its own
// column, qr.py:84), reduced per warp through a shared-memory transpose and across the 8 warps
// through a partial-sum row, then the rank-1 update of columns J+1..63. The shared-memory
// qr_factor_cta it replaces ran each reflector's scalars on one warp while seven waited.
constexpr int kDqrTS = 65;  // transpose row stride (odd: conflict-free rows and columns)
constexpr size_t kDqrRegSmem = (size_t)(8 * 32 * kDqrTS + 8 * 64 + 64 + 64 + 32) * sizeof(double);

struct DqrReg {
  double* tb;    // 8 warps x 32 rows x kDqrTS
  double* part;  // 8 x 64 warp partial sums
  double* tot;   // 64: tau * (v . a_c)
  double* taus;  // 64
  double* misc;  // 2 x 16 (double-buffered by J parity): [0..7] warp norms, [8] alpha
  int tid, lane, warp, m;

  template <int J>
  BF_DEV void col(double (&a)[64]) {
    const bool live = tid < m;
    double* ms = misc + 16 * (J & 1);
    double ts = (tid > J && live) ? a[J] * a[J] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ts += __shfl_xor_sync(0xffffffffu, ts, o);
    if (lane == 0) ms[warp] = ts;
    if (tid == J) ms[8] = a[J];
    __syncthreads();
    double tail_sq = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tail_sq += ms[w];
    const double alpha = ms[8];
    double tj = 0.0;
    if (J + 1 < m && tail_sq != 0.0) {  // uniform
      double beta, denom, rden;
      householder_scalars(alpha, tail_sq, beta, tj, denom, rden);
      double v = 0.0, pj = 0.0;
      if (tid == J) {
        v = 1.0;
        pj = alpha;
      } else if (tid > J && live) {
        const double x = a[J];
        v = div_by(x, denom, rden);
        pj = v * x;
        a[J] = v;  // reflector stored below the diagonal
      }
      constexpr int K = 64 - J;
      double* row = tb + (warp * 32 + lane) * kDqrTS;
      row[0] = pj;
#pragma unroll
      for (int c = 1; c < K; ++c) row[c] = v * a[J + c];
      __syncwarp();
      const double* wt = tb + warp * 32 * kDqrTS;
      if (lane < K) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
        for (int r = 0; r < 32; r += 2) {
          s0 += wt[r * kDqrTS + lane];
          s1 += wt[(r + 1) * kDqrTS + lane];
        }
        part[warp * 64 + lane] = s0 + s1;
      }
      if (lane + 32 < K) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
        for (int r = 0; r < 32; r += 2) {
          s0 += wt[r * kDqrTS + lane + 32];
          s1 += wt[(r + 1) * kDqrTS + lane + 32];
        }
        part[warp * 64 + lane + 32] = s0 + s1;
      }
      __syncthreads();
      if (tid < K) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += part[w * 64 + tid];
        tot[tid] = t * tj;
      }
      __syncthreads();
      if (tid == J) a[J] = alpha - tot[0];
#pragma unroll
      for (int c = 1; c < K; ++c) a[J + c] = fma(-v, tot[c], a[J + c]);
    }
    if (tid == 0) taus[J] = tj;
  }

  template <int J>
  BF_DEV void from(double (&a)[64]) {
    if constexpr (J < 64) {
      col<J>(a);
      from<J + 1>(a);
    }
  }
};

__global__ void __launch_bounds__(256, 1) bj_dqr_reg(BJArgs<double> a, BDArgs d, int step) {
  extern __shared__ __align__(16) double dq_smem[];
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  const int64_t slot = blockIdx.x;
  if (b >= a.batch) return;
  if (!a.active[b]) {
    if (threadIdx.x == 0) d.pact[slot] = 0;
    return;
  }
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, m = a.m, tid = threadIdx.x;
  DqrReg q;
  q.tb = dq_smem;
  q.part = q.tb + 8 * 32 * kDqrTS;
  q.tot = q.part + 8 * 64;
  q.taus = q.tot + 64;
  q.misc = q.taus + 64;
  q.tid = tid;
  q.lane = tid & 31;
  q.warp = tid >> 5;
  q.m = m;
  const double* Wb = a.W + b * (int64_t)m * a.n_pad;
  double x[64];
#pragma unroll
  for (int c = 0; c < 64; ++c) x[c] = tid < m ? Wb[(size_t)pair_col(c, k, bi, bj) * m + tid] : 0.0;
  q.from<0>(x);
  // outputs: R (upper triangle, kk x kk) -> G, the factored pair -> P, tau
  double* G = d.G + slot * 64 * 64;
  if (tid < 64) {
#pragma unroll
    for (int c = 0; c < 64; ++c) G[(size_t)c * 64 + tid] = c >= tid ? x[c] : 0.0;
  }
  double* Pg = d.P + slot * (int64_t)m * 64;
  if (tid < m) {
#pragma unroll
    for (int c = 0; c < 64; ++c) Pg[(size_t)c * m + tid] = x[c];
  }
  __syncthreads();
  if (tid < 64) d.tau[slot * 64 + tid] = q.taus[tid];
  // scaled_offdiag of R (blockjacobi.py:57-76): diagonal to shared memory, row tid vs c > tid
  double* diag = q.part;  // 64 (free after the loop)
  double* red = q.tot;
  if (tid < 64) {
#pragma unroll
    for (int c = 0; c < 64; ++c)
      if (c == tid) diag[c] = x[c];
  }
  if (tid == 0) red[0] = 0.0;
  __syncthreads();
  double best = 0.0;
  if (tid < 64) {
    const double di = sqrt(fabs(diag[tid]));
#pragma unroll
    for (int c = 1; c < 64; ++c) {
      if (c > tid) {
        const double den = di * sqrt(fabs(diag[c]));
        const double num = fabs(x[c]);
        const double rt = den > 0.0 ? num / den : (num > 0.0 ? __longlong_as_double(0x7ff0000000000000LL) : 0.0);
        best = rt > best ? rt : best;
      }
    }
  }
  best = warp_allreduce_max(best);
  if ((tid & 31) == 0 && best > 0.0) atomic_max_pos(red, best);
  __syncthreads();
  if (tid == 0) {
    atomic_max_pos(a.e_sweep + b, red[0]);
    d.pact[slot] = red[0] > a.tol ? 1 : 0;
    bj_count(a.stats, b, red[0] > a.tol);
  }
}

// new pair = H_0 ... H_{kk-1} [U_R diag(sigma); 0] (== (Q @ U_R) * sigma, blockjacobi.py:143).
// Same product in compact-WY form on the FP64 tensor cores: with the reflectors Y (unit lower
// trapezoidal, m x 64) and tau, H_0 ... H_63 = I - Y T Y^T (LAPACK dlarft, forward / columnwise:
// T_jj = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] (Y^T Y)[0:j, j]), so the new pair
// Q [X1; 0] = [X1; 0] - Y (T (Y1^T X1)) with X1 = U_R diag(sigma) and Y1 the top 64 rows of Y.
// Every product is a 64-wide DMMA GEMM (warp w: a 16 x 32 block of the 64 x 64 output).
constexpr int kWyLD = 64 + 4;  // 64 x 64 smem matrices and Y chunks: element (r, c) at [c * LD + r]
constexpr int kWyCH = 64;      // Y rows per staged chunk
constexpr size_t kWySmem = (size_t)(5 * 64 * kWyLD + 64) * sizeof(double);

BF_DEV void wy_dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
BF_DEV void wy_cp16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
BF_DEV void wy_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
BF_DEV void wy_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__global__ void __launch_bounds__(256) bj_dapply_wy(BJArgs<double> a, BDArgs d, int step) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int KK = 64, LD = kWyLD, CH = kWyCH;
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  const int64_t slot = blockIdx.x;
  if (b >= a.batch || !d.pact[slot]) return;
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, m = a.m, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp >> 1) * 16, c0 = (warp & 1) * 32;  // this warp's 16 x 32 output block
  double* bufA = reinterpret_cast<double*>(smem_raw);
  double* bufB = bufA + 64 * LD;
  double* bufC = bufB + 64 * LD;
  double* const Ybase = bufC + 64 * LD;  // double-buffered raw Y chunks at Ybase + buf * 64 * LD
  double* taus = bufC + 3 * 64 * LD;
  const double* Pg = d.P + slot * (int64_t)m * KK;
  const double* U = d.U + slot * KK * KK;
  const double* S = d.S + slot * KK;
  if (tid < KK) taus[tid] = d.tau[slot * KK + tid];
  const int nch = (m + CH - 1) / CH;
  // raw rows rc..rc+63 of the factored pair, column-major, 16-byte cp.async (rows >= m zero)
  auto load = [&](int buf, int rc) {
    double* Y = Ybase + buf * (64 * LD);
    for (int e = tid; e < KK * (CH / 2); e += 256) {
      const int c = e / (CH / 2), rr = 2 * (e % (CH / 2)), r = rc + rr;
      double* dst = &Y[c * LD + rr];
      const double* src = Pg + (size_t)c * m + r;
      if (r + 1 < m && ((m & 1) == 0)) {
        wy_cp16(dst, src);
      } else {
        dst[0] = r < m ? src[0] : 0.0;
        dst[1] = r + 1 < m ? src[1] : 0.0;
      }
    }
    wy_commit();
  };
  // Y[r][c] (unit lower trapezoidal): the stored reflector below the diagonal, 1 on it, 0 above;
  // only the first chunk has rows <= c
  auto yv = [&](const double* Y, int rl, int c, int rg) {
    const double raw = Y[c * LD + rl];
    return rg > c ? raw : (rg == c ? 1.0 : 0.0);
  };
  double acc[2][4][2];
  auto zero = [&]() {
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  };
  auto store = [&](double* M) {  // fragments -> M (column-major 64 x 64, ld LD)
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y)
#pragma unroll
        for (int q = 0; q < 2; ++q) M[(c0 + 8 * y + 2 * t + q) * LD + r0 + 8 * x + g] = acc[x][y][q];
  };
  // ---- G_Y = Y^T Y, accumulated over double-buffered row chunks of Y
  zero();
  load(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      load((ch + 1) & 1, (ch + 1) * CH);
      wy_wait<1>();
    } else {
      wy_wait<0>();
    }
    __syncthreads();
    const double* Y = Ybase + (ch & 1) * (64 * LD);
    const int rc = ch * CH;
#pragma unroll 4
    for (int k0 = 0; k0 < CH; k0 += 4) {
      double av[2], bv[4];
      const int rl = k0 + t, rg = rc + rl;
#pragma unroll
      for (int x = 0; x < 2; ++x) av[x] = yv(Y, rl, r0 + 8 * x + g, rg);  // A[i][k] = Y[k][i]
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = yv(Y, rl, c0 + 8 * y + g, rg);  // B[k][j] = Y[k][j]
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) wy_dmma(acc[x][y], av[x], bv[y]);
    }
    __syncthreads();
  }
  store(bufA);  // G_Y
  // chunk 0 (Y1, and the first chunk of the final product) into the buffer not holding the
  // last chunk; it streams in while T is formed
  const int z = nch & 1;
  load(z, 0);
  // ---- X1 = U_R diag(sigma) -> bufC
  for (int e = tid; e < KK * KK; e += 256) {
    const int c = e / KK, r = e % KK;
    bufC[c * LD + r] = U[(size_t)c * KK + r] * S[c];
  }
  __syncthreads();
  // ---- T (upper triangular) -> bufB, column by column; the dot of row i is split over the 4
  // threads (i, q) (l = i + q mod 4) and summed by two shuffles, so all 256 threads work
  {
    const int i = tid >> 2, q = tid & 3;
    for (int j = 0; j < KK; ++j) {
      double zz = 0.0;
      if (i < j)
        for (int l = i + q; l < j; l += 4) zz = fma(bufB[l * LD + i], bufA[j * LD + l], zz);
      zz += __shfl_xor_sync(0xffffffffu, zz, 1);
      zz += __shfl_xor_sync(0xffffffffu, zz, 2);
      if (q == 0) bufB[j * LD + i] = i < j ? -taus[j] * zz : (i == j ? taus[j] : 0.0);
      __syncthreads();
    }
  }
  wy_wait<0>();
  __syncthreads();
  // ---- W1 = Y1^T X1 (Y1 = top 64 rows of Y) -> bufA
  zero();
  {
    const double* Y = Ybase + z * (64 * LD);
#pragma unroll 4
    for (int k0 = 0; k0 < KK; k0 += 4) {
      double av[2], bv[4];
#pragma unroll
      for (int x = 0; x < 2; ++x) av[x] = yv(Y, k0 + t, r0 + 8 * x + g, k0 + t);  // Y1[k][i]
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = bufC[(c0 + 8 * y + g) * LD + k0 + t];  // X1[k][j]
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) wy_dmma(acc[x][y], av[x], bv[y]);
    }
  }
  __syncthreads();
  store(bufA);  // W1 (G_Y no longer needed)
  if (nch > 1) load(z ^ 1, CH);  // the final product's second chunk
  __syncthreads();
  // ---- W2 = T W1 -> bufC (X1 is re-read from U, S below)
  zero();
#pragma unroll 4
  for (int k0 = 0; k0 < KK; k0 += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int x = 0; x < 2; ++x) av[x] = bufB[(k0 + t) * LD + r0 + 8 * x + g];  // T[i][k]
#pragma unroll
    for (int y = 0; y < 4; ++y) bv[y] = bufA[(c0 + 8 * y + g) * LD + k0 + t];  // W1[k][j]
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) wy_dmma(acc[x][y], av[x], bv[y]);
  }
  __syncthreads();
  store(bufC);
  // ---- new pair = [X1; 0] - Y W2, 64-row chunks of Y (double-buffered), written to W
  double* Wb = a.W + b * (int64_t)m * a.n_pad;
  for (int ch = 0; ch < nch; ++ch) {
    const int buf = (z + ch) & 1, rc = ch * CH;
    if (ch + 1 < nch) {
      wy_wait<1>();
    } else {
      wy_wait<0>();
    }
    __syncthreads();
    const double* Y = Ybase + buf * (64 * LD);
    zero();
#pragma unroll 4
    for (int k0 = 0; k0 < KK; k0 += 4) {
      double av[2], bv[4];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int rl = r0 + 8 * x + g;
        av[x] = yv(Y, rl, k0 + t, rc + rl);  // Y[i][k]
      }
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = bufC[(c0 + 8 * y + g) * LD + k0 + t];  // W2[k][j]
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) wy_dmma(acc[x][y], av[x], bv[y]);
    }
    __syncthreads();  // buffer `buf` is free
    if (ch + 2 < nch) load(buf, (ch + 2) * CH);
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int r = rc + r0 + 8 * x + g;
      if (r < m) {
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int c = c0 + 8 * y + 2 * t + q;
            const double x1 = r < KK ? U[(size_t)c * KK + r] * S[c] : 0.0;
            Wb[(size_t)pair_col(c, k, bi, bj) * m + r] = x1 - acc[x][y][q];
          }
      }
    }
  }
}

template <typename T>
__global__ void bj_init(BJArgs<T> a, const T* A) {
  const int64_t b = blockIdx.x;
  if (b >= a.batch) return;
  const int m = a.m, n = a.n, np = a.n_pad;
  T* Wb = a.W + b * (int64_t)m * np;
  const T* Ab = A + b * (int64_t)m * n;
  for (int64_t e = threadIdx.x; e < (int64_t)m * np; e += blockDim.x) Wb[e] = e < (int64_t)m * n ? Ab[e] : T(0);
  if (a.V) {
    T* Vb = a.V + b * (int64_t)np * np;
    for (int64_t e = threadIdx.x; e < (int64_t)np * np; e += blockDim.x) Vb[e] = (e / np == e % np) ? T(1) : T(0);
  }
  if (threadIdx.x == 0) {
    a.active[b] = 1;
    a.e_sweep[b] = 0.0;
    a.sweeps[b] = 0;
    a.conv[b] = 0;
  }
  if (a.stats && threadIdx.x < 4) a.stats[4 * b + threadIdx.x] = 0;
  if (a.in_sw)  // per-slot inner counters of this matrix's pairs
    for (int p = threadIdx.x; p < a.nb / 2; p += blockDim.x) {
      a.in_sw[b * (a.nb / 2) + p] = 0;
      a.in_rot[b * (a.nb / 2) + p] = 0;
    }
}

// fold the per-slot inner-SVD counters of the batched pipelines into the per-matrix stats
template <typename T>
__global__ void bj_stats_reduce(BJArgs<T> a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.batch) return;
  const int P = a.nb / 2, kk = 2 * a.k;
  long long sw = 0, rot = 0;
  for (int p = 0; p < P; ++p) {
    sw += a.in_sw[b * P + p];
    rot += a.in_rot[b * P + p];
  }
  a.stats[4 * b + 2] += sw * (long long)(kk * (kk - 1) / 2);
  a.stats[4 * b + 3] += rot;
}

template <typename T>
__global__ void bj_finalize_sweep(BJArgs<T> a, int* still_active) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool act = false;
  if (b < a.batch && a.active[b]) {
    double e = a.e_sweep[b];
    int s = a.sweeps[b];
    if (a.e_hist) a.e_hist[b * a.max_sweeps + s] = (T)e;
    s += 1;
    a.sweeps[b] = s;
    if (e < a.tol) {
      a.conv[b] = 1;
      a.active[b] = 0;
    } else if (s >= a.max_sweeps) {
      a.active[b] = 0;
    } else {
      act = true;
    }
    a.e_sweep[b] = 0.0;
  }
  // matrices still sweeping after this sweep: the host stops enqueueing sweeps at zero
  const unsigned bal = __ballot_sync(0xffffffffu, act);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(still_active, __popc(bal));
}

// Host-side sweep control: after each sweep the count of still-active matrices is copied to
// pinned memory; the host, running up to kSweepLag sweeps ahead of the device, stops enqueueing
// once a completed sweep reports zero (blockjacobi.py:150-154: converged matrices stop; the
// batch stops when all have). The device never waits on the host. A call's counters may still be
// in flight when it returns (asynchronous stream semantics), so each call takes a ring that no
// pending copy targets: rings are pooled per device and reused once their events have completed.
constexpr int kSweepLag = 2, kCtlRing = 4;
struct SweepCtl {
  int* host = nullptr;  // pinned, kCtlRing counters
  cudaEvent_t ev[kCtlRing] = {};
  bool recorded[kCtlRing] = {};
  bool in_use = false;  // a call is enqueueing with this ring
  bool idle() {
    if (in_use) return false;
    for (int i = 0; i < kCtlRing; ++i)
      if (recorded[i] && cudaEventQuery(ev[i]) != cudaSuccess) return false;
    return true;
  }
};
static std::mutex g_ctl_mu;
static SweepCtl* sweep_ctl_acquire() {
  static std::vector<std::pair<int, SweepCtl*>> pool;  // (device, ring); rings live for the process
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_ctl_mu);
  for (auto& e : pool)
    if (e.first == dev && e.second->idle()) {
      cudaGetLastError();  // clear cudaErrorNotReady from the queries
      for (int i = 0; i < kCtlRing; ++i) e.second->recorded[i] = false;
      e.second->in_use = true;
      return e.second;
    }
  cudaGetLastError();
  SweepCtl* c = new SweepCtl();
  bool good = cudaMallocHost((void**)&c->host, sizeof(int) * kCtlRing) == cudaSuccess;
  for (int i = 0; good && i < kCtlRing; ++i)
    good = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) == cudaSuccess;
  if (!good) {
    cudaGetLastError();
    return nullptr;  // fall back to max_sweeps launches
  }
  c->in_use = true;
  pool.emplace_back(dev, c);
  return c;
}
static void sweep_ctl_release(SweepCtl* c) {
  if (!c) return;
  std::lock_guard<std::mutex> lk(g_ctl_mu);
  c->in_use = false;
}

template <typename T>
__global__ void __launch_bounds__(256) bj_extract(BJArgs<T> a, T* U, T* S, T* Vout, T* cand_g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t b = blockIdx.x;
  if (b >= a.batch) return;
  const int m = a.m, n = a.n, np = a.n_pad;
  T* sig = reinterpret_cast<T*>(smem_raw);
  int* order = reinterpret_cast<int*>(sig + np);
  int* flag = order + np;
  extract_svd_cta<T>(a.W + b * (int64_t)m * np, m, a.V ? a.V + b * (int64_t)np * np : nullptr, np, m, np, n, n,
                     U + b * (int64_t)m * n, m, S + b * (int64_t)n, Vout ? Vout + b * (int64_t)n * n : nullptr, n,
                     sig, order, cand_g + b * 2 * (int64_t)m, flag);
}

// ---- wide block pairs (2k > 64, any block_width: blockjacobi.py:98-104 accepts every width).
// The pair is staged into a contiguous per-slot copy and the step runs as batched launches over
// all slots of the step: gather -> (Gram: G = P^T P | direct: P = Q R) -> e = scaled_offdiag
// (pairs at e <= tol skipped, blockjacobi.py:128-129,139-140) -> inner round-robin SVD (batched,
// masked by the pair flags) -> P U (Gram, null directions zeroed, :132-134) or (Q U_R) sigma
// (direct, :143) and the V pair times the rotation (:146-149) -> scatter of the active pairs.
template <typename T>
struct BWArgs {
  T *P, *PV, *G, *Q, *U, *S, *VR, *Pn, *PVn;
  uint8_t* pact;
};

template <typename T>
__global__ void __launch_bounds__(256) bw_gather(BJArgs<T> a, BWArgs<T> w, int step) {
  const int P = a.nb / 2;
  const int64_t slot = blockIdx.x, b = slot / P;
  if (b >= a.batch) return;
  if (!a.active[b]) {
    if (threadIdx.x == 0) w.pact[slot] = 0;
    return;
  }
  int bi, bj;
  rr_pair(a.nb, step, (int)(slot % P), bi, bj);
  const int k = a.k, kk = 2 * k, m = a.m, np = a.n_pad;
  const T* Wb = a.W + b * (int64_t)m * np;
  T* Ps = w.P + slot * (int64_t)m * kk;
  for (int64_t e = threadIdx.x; e < (int64_t)m * kk; e += blockDim.x) {
    const int c = (int)(e / m), r = (int)(e % m);
    Ps[e] = Wb[(int64_t)pair_col(c, k, bi, bj) * m + r];
  }
  if (a.V) {
    const T* Vb = a.V + b * (int64_t)np * np;
    T* Vs = w.PV + slot * (int64_t)np * kk;
    for (int64_t e = threadIdx.x; e < (int64_t)np * kk; e += blockDim.x) {
      const int c = (int)(e / np), r = (int)(e % np);
      Vs[e] = Vb[(int64_t)pair_col(c, k, bi, bj) * np + r];
    }
  }
}

// e = scaled_offdiag of G (Gram: mirrored upper triangle first, syrk core.py:68-78) or R (direct)
template <typename T>
__global__ void __launch_bounds__(256) bw_offdiag(BJArgs<T> a, BWArgs<T> w, int gram) {
  __shared__ double red;
  const int P = a.nb / 2;
  const int64_t slot = blockIdx.x, b = slot / P;
  if (b >= a.batch || !a.active[b]) return;
  const int kk = 2 * a.k;
  T* M = w.G + slot * (int64_t)kk * kk;
  if (gram) {
    for (int e = threadIdx.x; e < kk * kk; e += blockDim.x) {
      const int j = e / kk, i = e % kk;  // row i, column j
      if (i > j) M[(size_t)j * kk + i] = M[(size_t)i * kk + j];
    }
    __syncthreads();
  }
  const double e = scaled_offdiag_cta<T>(M, kk, kk, &red);
  if (threadIdx.x == 0) {
    atomic_max_pos(a.e_sweep + b, e);
    w.pact[slot] = e > a.tol ? 1 : 0;
    bj_count(a.stats, b, e > a.tol);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) bw_scatter(BJArgs<T> a, BWArgs<T> w, int step, int gram) {
  const int P = a.nb / 2;
  const int64_t slot = blockIdx.x, b = slot / P;
  if (b >= a.batch || !w.pact[slot]) return;
  int bi, bj;
  rr_pair(a.nb, step, (int)(slot % P), bi, bj);
  const int k = a.k, kk = 2 * k, m = a.m, np = a.n_pad;
  T* Wb = a.W + b * (int64_t)m * np;
  const T* Pn = w.Pn + slot * (int64_t)m * kk;
  const T* S = w.S + slot * (int64_t)kk;
  for (int64_t e = threadIdx.x; e < (int64_t)m * kk; e += blockDim.x) {
    const int c = (int)(e / m), r = (int)(e % m);
    const T sg = S[c];
    T x = Pn[e];
    if (gram)
      x = sg != T(0) ? x : T(0);  // exactly-null directions stay null (blockjacobi.py:133-134)
    else
      x = x * sg;  // (Q @ U_R) * sigma (blockjacobi.py:143)
    Wb[(int64_t)pair_col(c, k, bi, bj) * m + r] = x;
  }
  if (a.V) {
    T* Vb = a.V + b * (int64_t)np * np;
    const T* Vs = w.PVn + slot * (int64_t)np * kk;
    for (int64_t e = threadIdx.x; e < (int64_t)np * kk; e += blockDim.x) {
      const int c = (int)(e / np), r = (int)(e % np);
      Vb[(int64_t)pair_col(c, k, bi, bj) * np + r] = Vs[e];
    }
  }
}

static void bj_geometry(int m, int n, int bw, int method, int& k, int& n_pad, int& nb) {
  k = bw;
  if (method == 1) {
    k = m / 2 < k ? m / 2 : k;
    if (k < 1) k = 1;
  }
  n_pad = ((n + 2 * k - 1) / (2 * k)) * (2 * k);
  if (n_pad < 2 * k) n_pad = 2 * k;
  nb = n_pad / k;
}

template <typename T>
static size_t direct_smem(int m, int kk, bool p_in) {
  size_t b = (size_t)4 * kk * kk * sizeof(T) + (size_t)5 * kk * sizeof(T) + (size_t)kk * sizeof(int) + 64;
  if (p_in) b += (size_t)m * kk * sizeof(T);
  return (b + 15) & ~(size_t)15;
}

template <typename T>
struct BJLayout {
  size_t w, v, p, e, act, cand, g, u, s, pact, iws, dp, dtau, dvr, isw, irot, ring, total;
  // wide pairs (2k > 64)
  size_t xp, xpv, xq, xvr, xpn, xpvn, xqws;
};

// 2k > 64: the staged wide-pair pipeline (any block width)
static bool bj_wide(int kk) { return kk > 64; }

// batched direct pipeline: fp64, 2k in {16, 32, 48, 64} (register-tier inner SVD with V), the
// pair plus the reflector stage fitting one CTA's shared memory
static bool bj_batched_direct(int method, int m, int kk, bool f64) {
  return f64 && method == 1 && kk == 64 &&
         (size_t)m * kk * 8 + (size_t)8 * m * 8 + 64 * 8 <= 200 * 1024;
}

// batched Gram pipeline (bj_gram -> register-tier inner SVD -> bj_rot) covers 2k in {16,32,48,64}
static bool bj_batched_gram(int method, int kk) { return method == 0 && kk % 16 == 0 && kk <= 64; }

template <typename T>
static BJLayout<T> bj_layout(int64_t batch, int m, int n, int bw, int method, bool accv) {
  int k, np, nb;
  bj_geometry(m, n, bw, method, k, np, nb);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  BJLayout<T> L;
  size_t off = 0;
  L.w = off;
  off += al((size_t)batch * m * np * sizeof(T));
  L.v = off;
  off += accv ? al((size_t)batch * np * np * sizeof(T)) : 0;
  L.p = off;
  bool p_in = direct_smem<T>(m, 2 * k, true) <= 227 * 1024;
  off += (method == 1 && !p_in) ? al((size_t)batch * (nb / 2) * m * 2 * k * sizeof(T)) : 0;
  L.e = off;
  off += al((size_t)batch * sizeof(double));
  L.act = off;
  off += al((size_t)batch);
  L.cand = off;
  off += al((size_t)batch * 2 * m * sizeof(T));
  const int kk = 2 * k;
  const int64_t slots = batch * (nb / 2);
  const bool bg = bj_batched_gram(method, kk);
  const bool bd = bj_batched_direct(method, m, kk, sizeof(T) == 8);
  const bool bt = bg || bd;
  L.g = off;
  off += bt ? al((size_t)slots * kk * kk * sizeof(T)) : 0;
  L.u = off;
  off += bt ? al((size_t)slots * kk * kk * sizeof(T)) : 0;
  L.s = off;
  off += bt ? al((size_t)slots * kk * sizeof(T)) : 0;
  L.pact = off;
  off += bt ? al((size_t)slots) : 0;
  L.dp = off;
  off += bd ? al((size_t)slots * m * kk * sizeof(T)) : 0;
  L.dtau = off;
  off += bd ? al((size_t)slots * kk * sizeof(T)) : 0;
  L.dvr = off;
  off += bd ? al((size_t)slots * kk * kk * sizeof(T)) : 0;
  const bool wide = bj_wide(kk);
  const size_t es = sizeof(T);
  if (wide) {  // G doubles as R (direct); U, S, pact as above
    L.g = off;
    off += al((size_t)slots * kk * kk * es);
    L.u = off;
    off += al((size_t)slots * kk * kk * es);
    L.s = off;
    off += al((size_t)slots * kk * es);
    L.pact = off;
    off += al((size_t)slots);
    L.xp = off;
    off += al((size_t)slots * m * kk * es);
    L.xpn = off;
    off += al((size_t)slots * m * kk * es);
    L.xq = off;
    off += method == 1 ? al((size_t)slots * m * kk * es) : 0;
    L.xpv = off;
    off += accv ? al((size_t)slots * np * kk * es) : 0;
    L.xpvn = off;
    off += accv ? al((size_t)slots * np * kk * es) : 0;
    L.xvr = off;
    off += (method == 1 && accv) ? al((size_t)slots * kk * kk * es) : 0;
    L.xqws = off;
    off += method == 1 ? al(qr_global_ws_bytes(es == 8 ? 0 : 1, slots, m, kk)) : 0;
  }
  L.ring = off;
  off += al(sizeof(int) * 4);
  L.isw = off;
  off += al((size_t)slots * sizeof(int32_t));
  L.irot = off;
  off += al((size_t)slots * sizeof(int64_t));
  L.iws = off;
  off += (bt || wide) ? al(svd_global_ws_bytes(es == 8 ? 0 : 1, slots, kk, kk, 1, bd || (wide && method == 1 && accv),
                                               0, 30))
                      : 0;
  L.total = off;
  return L;
}

size_t block_ws_bytes(int dtype, int64_t batch, int m, int n, int block_width, int method, bool accv) {
  return dtype == 0 ? bj_layout<double>(batch, m, n, block_width, method, accv).total
                    : bj_layout<float>(batch, m, n, block_width, method, accv).total;
}

// fp64 with 2k = 64: Gram and rotation products on the FP64 tensor cores (bj_*_mma)
template <typename T>
static constexpr bool kUseMma(int TT) {
  return sizeof(T) == 8 && TT == 4;
}

// Tensor map for the 2-D TMA staging of bj_gram_tma: W as a column-major (m rows) x (B n_pad
// columns) float64 tensor, box 8 x 32, 64-byte swizzle (block_gemm.cuh, tma_load_2d). The encoder
// is the driver's cuTensorMapEncodeTiled, reached through the runtime (no libcuda link).
static bool make_col_tmap(CUtensorMap* map, const double* base, int rows, int64_t cols) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!enc || (rows & 1) || ((uintptr_t)base & 15) || cols > 0x7fffffff) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  const cuuint64_t strides[1] = {(cuuint64_t)rows * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)kTmaBoxRows, (cuuint32_t)kTmaBoxCols};
  const cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)base, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T>
static int launch_block_t(const BlockLaunch& L, void* ws, cudaStream_t st) {
  BJArgs<T> a;
  int k, np, nb;
  bj_geometry(L.m, L.n, L.block_width, L.method, k, np, nb);
  BJLayout<T> lay = bj_layout<T>(L.batch, L.m, L.n, L.block_width, L.method, L.v != nullptr);
  char* base = (char*)ws;
  a.batch = L.batch;
  a.m = L.m;
  a.n = L.n;
  a.n_pad = np;
  a.k = k;
  a.nb = nb;
  a.W = (T*)(base + lay.w);
  a.V = L.v ? (T*)(base + lay.v) : nullptr;
  a.P = (T*)(base + lay.p);
  a.e_sweep = (double*)(base + lay.e);
  a.active = (uint8_t*)(base + lay.act);
  a.sweeps = L.sweeps;
  a.conv = L.converged;
  a.e_hist = (T*)L.e_history;
  a.max_sweeps = L.max_sweeps;
  a.tol = L.tol;
  a.tol_inner = sizeof(T) == 8 ? Tol<double>::svd : Tol<float>::svd;
  a.stats = L.stats;
  a.in_sw = L.stats ? (int32_t*)(base + lay.isw) : nullptr;
  a.in_rot = L.stats ? (int64_t*)(base + lay.irot) : nullptr;
  const int kk = 2 * k;
  a.p_in_smem = direct_smem<T>(L.m, kk, true) <= 227 * 1024;
  cudaError_t e;
  bj_init<T><<<(unsigned)L.batch, 256, 0, st>>>(a, (const T*)L.a);
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  const unsigned grid = (unsigned)(L.batch * (nb / 2));
  size_t smem = 0;
  if (!bj_wide(kk)) {  // the one-CTA-per-pair step kernels (the wide pipeline needs no large smem)
    if (L.method == 0) {
      smem = (size_t)(2 * kk * kk + kk * 32 + 3 * kk) * sizeof(T) + (size_t)kk * sizeof(int) + 64;
      e = smem_optin((const void*)bj_gram_step<T>, (size_t)(smem));
    } else {
      smem = direct_smem<T>(L.m, kk, a.p_in_smem);
      e = smem_optin((const void*)bj_direct_step<T>, (size_t)(smem));
    }
    if (e != cudaSuccess) return (int)e;
  }
  const bool bg = bj_batched_gram(L.method, kk);
  BJGemmArgs<T> g;
  // TMA staging of the DMMA block kernels (bit 0 Gram, bit 1 rotation); BF_BLOCK_TMA overrides
  static const int tma_sel = [] {
    const char* e = getenv("BF_BLOCK_TMA");
    return e ? atoi(e) : kBlockTmaDefault;
  }();
  g.tma = tma_sel;
  // tensor-map TMA kernels (bits 4 / 8); fall back to the cp.async kernels if a map can't be encoded
  CUtensorMap tm_w{}, tm_v{};
  int tma_sel_gram = tma_sel & 4, tma_sel_rot = tma_sel & 8;
  if ((tma_sel & 12) && sizeof(T) == 8 && k == 32) {
    if (!make_col_tmap(&tm_w, (const double*)a.W, L.m, L.batch * np)) tma_sel_gram = tma_sel_rot = 0;
    if (a.V && !make_col_tmap(&tm_v, (const double*)a.V, np, L.batch * np)) tma_sel_rot = 0;
  }
  SvdLaunch in{};
  size_t rot_smem = 0;
  if (bg) {
    g.batch = L.batch;
    g.m = L.m;
    g.n_pad = np;
    g.k = k;
    g.nb = nb;
    g.W = a.W;
    g.V = a.V;
    g.G = (T*)(base + lay.g);
    g.U = (T*)(base + lay.u);
    g.S = (T*)(base + lay.s);
    g.pair_act = (uint8_t*)(base + lay.pact);
    g.active = a.active;
    g.e_sweep = a.e_sweep;
    g.tol = L.tol;
    // inner SVD of every active G: round robin, no V, default tolerance (blockjacobi.py:79-81)
    in.batch = L.batch * (nb / 2);
    in.m = kk;
    in.n = kk;
    in.a = g.G;
    in.a_stride = (int64_t)kk * kk;
    in.u = g.U;
    in.u_stride = (int64_t)kk * kk;
    in.s = g.S;
    in.s_stride = kk;
    in.v = nullptr;
    in.v_stride = 0;
    in.sweeps = nullptr;
    in.converged = nullptr;
    in.rotations = nullptr;
    in.tol = a.tol_inner;
    in.max_sweeps = 30;
    in.ordering = 1;
    in.tier = 0;
    in.transpose_a = false;
    in.active = g.pair_act;
    in.sweeps = a.in_sw;  // per-slot work counters, accumulated over the run
    in.rotations = a.in_rot;
    in.accumulate = true;
    g.stats = L.stats;
    rot_smem = (size_t)2 * kk * (kk + 1) * sizeof(T);
    const int TT = kk / 16;
    if (TT == 1) e = smem_optin((const void*)bj_rot<T, 1>, rot_smem);
    if (TT == 2) e = smem_optin((const void*)bj_rot<T, 2>, rot_smem);
    if (TT == 3) e = smem_optin((const void*)bj_rot<T, 3>, rot_smem);
    if (TT == 4) e = smem_optin((const void*)bj_rot<T, 4>, rot_smem);
    if (e == cudaSuccess && kUseMma<T>(TT))
      e = smem_optin((const void*)bj_rot_mma, (size_t)(kRotSmem));
    if (e == cudaSuccess && kUseMma<T>(TT) && tma_sel_rot) e = smem_optin((const void*)bj_rot_tma, kRotTmaSmem);
    if (e != cudaSuccess) return (int)e;
  }
  // batched direct pipeline (fp64, 2k = 64)
  const bool bd = bj_batched_direct(L.method, L.m, kk, sizeof(T) == 8);
  BDArgs dd{};
  BJGemmArgs<T> gv{};
  gv.tma = tma_sel;
  size_t dqr_smem = 0, dap_smem = 0;
  bool dqr_reg = false;
  if (bd) {
    dd.P = (double*)(base + lay.dp);
    dd.tau = (double*)(base + lay.dtau);
    dd.G = (double*)(base + lay.g);
    dd.U = (double*)(base + lay.u);
    dd.S = (double*)(base + lay.s);
    dd.pact = (uint8_t*)(base + lay.pact);
    // inner SVD of every active R: round robin with V (blockjacobi.py:141)
    in.batch = L.batch * (nb / 2);
    in.m = kk;
    in.n = kk;
    in.a = dd.G;
    in.a_stride = (int64_t)kk * kk;
    in.u = dd.U;
    in.u_stride = (int64_t)kk * kk;
    in.s = dd.S;
    in.s_stride = kk;
    in.v = base + lay.dvr;
    in.v_stride = (int64_t)kk * kk;
    in.sweeps = nullptr;
    in.converged = nullptr;
    in.rotations = nullptr;
    in.tol = a.tol_inner;
    in.max_sweeps = 30;
    in.ordering = 1;
    in.tier = 0;
    in.transpose_a = false;
    in.active = dd.pact;
    in.sweeps = a.in_sw;
    in.rotations = a.in_rot;
    in.accumulate = true;
    // V pair <- V pair @ V_R on the FP64 tensor cores (blockjacobi.py:146-149)
    gv.batch = L.batch;
    gv.m = L.m;
    gv.n_pad = np;
    gv.k = k;
    gv.nb = nb;
    gv.W = a.W;
    gv.V = a.V;
    gv.U = (T*)(base + lay.dvr);
    gv.S = (T*)dd.S;
    gv.pair_act = dd.pact;
    gv.active = a.active;
    gv.only_v = 1;
    dqr_reg = L.m <= 256;
    dqr_smem = dqr_reg ? kDqrRegSmem : ((size_t)L.m * kk + kk + 2) * sizeof(double);
    dap_smem = kWySmem;
    e = smem_optin((const void*)(dqr_reg ? bj_dqr_reg : bj_dqr), (size_t)(dqr_smem));
    if (e == cudaSuccess)
      e = smem_optin((const void*)bj_dapply_wy, (size_t)(dap_smem));
    if (e == cudaSuccess) e = smem_optin((const void*)bj_rot_mma, (size_t)(kRotSmem));
    if (e == cudaSuccess && tma_sel_rot) e = smem_optin((const void*)bj_rot_tma, kRotTmaSmem);
    if (e != cudaSuccess) return (int)e;
  }
  // wide pairs (2k > 64): staged pipeline over batched QR / GEMM / SVD launches
  const bool wide = bj_wide(kk);
  BWArgs<T> wa{};
  SvdLaunch win{};
  if (wide) {
    wa.P = (T*)(base + lay.xp);
    wa.Pn = (T*)(base + lay.xpn);
    wa.Q = L.method == 1 ? (T*)(base + lay.xq) : nullptr;
    wa.PV = L.v ? (T*)(base + lay.xpv) : nullptr;
    wa.PVn = L.v ? (T*)(base + lay.xpvn) : nullptr;
    wa.VR = (L.method == 1 && L.v) ? (T*)(base + lay.xvr) : nullptr;
    wa.G = (T*)(base + lay.g);
    wa.U = (T*)(base + lay.u);
    wa.S = (T*)(base + lay.s);
    wa.pact = (uint8_t*)(base + lay.pact);
    // inner SVD (blockjacobi.py:79-81): round robin, default tolerance; V only for the direct
    // method's rotation (:141, :145)
    win.batch = L.batch * (nb / 2);
    win.m = kk;
    win.n = kk;
    win.a = wa.G;
    win.a_stride = (int64_t)kk * kk;
    win.u = wa.U;
    win.u_stride = (int64_t)kk * kk;
    win.s = wa.S;
    win.s_stride = kk;
    win.v = wa.VR;
    win.v_stride = (int64_t)kk * kk;
    win.sweeps = nullptr;
    win.converged = nullptr;
    win.rotations = nullptr;
    win.tol = a.tol_inner;
    win.max_sweeps = 30;
    win.ordering = 1;
    win.tier = 0;
    win.transpose_a = false;
    win.active = wa.pact;
    win.sweeps = a.in_sw;
    win.rotations = a.in_rot;
    win.accumulate = true;
  }
  void* iws = base + lay.iws;
  const size_t iws_bytes = lay.total - lay.iws;
  // sweep control (see SweepCtl): inside a stream capture the host cannot observe the device,
  // so the graph gets all max_sweeps sweeps (converged matrices exit each kernel at once)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  SweepCtl* ctl = cap == cudaStreamCaptureStatusNone ? sweep_ctl_acquire() : nullptr;
  struct CtlGuard {
    SweepCtl* c;
    ~CtlGuard() { sweep_ctl_release(c); }
  } ctl_guard{ctl};
  int* ring = (int*)(base + lay.ring);
  for (int sw = 0; sw < L.max_sweeps; ++sw) {
    if (ctl && sw >= kSweepLag) {
      const int r = (sw - kSweepLag) % kCtlRing;
      if (cudaEventSynchronize(ctl->ev[r]) == cudaSuccess && ctl->host[r] == 0) break;
    }
    for (int s = 0; s < nb - 1; ++s) {
      if (wide) {
        const int dt = sizeof(T) == 8 ? 0 : 1;
        const int64_t slots = L.batch * (nb / 2);
        const int64_t mk = (int64_t)L.m * kk, k2 = (int64_t)kk * kk, vk = (int64_t)np * kk;
        bw_gather<T><<<grid, 256, 0, st>>>(a, wa, s);
        int rc;
        GemmLaunch gl;
        if (L.method == 0) {  // G = P^T P (upper triangle mirrored in bw_offdiag)
          gl = GemmLaunch{slots, kk, kk, L.m, wa.P, L.m, mk, true, wa.P, L.m, mk, false, wa.G, kk, k2};
          if ((rc = launch_gemm(dt, gl, st))) return rc;
        } else {  // (Q, R) = qr(P)
          if ((rc = launch_qr(dt, slots, L.m, kk, wa.P, mk, wa.Q, mk, wa.G, k2, base + lay.xqws, st))) return rc;
        }
        bw_offdiag<T><<<grid, 256, 0, st>>>(a, wa, L.method == 0);
        if ((rc = launch_svd(dt, win, iws, iws_bytes, st))) return rc;
        // Gram: P U_G; direct: Q U_R (sigma applied in the scatter)
        gl = GemmLaunch{slots, L.m, kk, kk, L.method == 0 ? wa.P : wa.Q, L.m, mk, false, wa.U, kk, k2, false,
                        wa.Pn, L.m, mk};
        if ((rc = launch_gemm(dt, gl, st))) return rc;
        if (L.v) {  // V pair @ rot (rot = U_G | V_R)
          gl = GemmLaunch{slots, np, kk, kk, wa.PV, np, vk, false, L.method == 0 ? wa.U : wa.VR, kk, k2, false,
                          wa.PVn, np, vk};
          if ((rc = launch_gemm(dt, gl, st))) return rc;
        }
        bw_scatter<T><<<grid, 256, 0, st>>>(a, wa, s, L.method == 0);
      } else if (bd) {
        if (dqr_reg)
          bj_dqr_reg<<<grid, 256, dqr_smem, st>>>(*reinterpret_cast<BJArgs<double>*>(&a), dd, s);
        else
          bj_dqr<<<grid, 256, dqr_smem, st>>>(*reinterpret_cast<BJArgs<double>*>(&a), dd, s);
        int rc = launch_svd(0, in, iws, iws_bytes, st);
        if (rc) return rc;
        bj_dapply_wy<<<grid, 256, dap_smem, st>>>(*reinterpret_cast<BJArgs<double>*>(&a), dd, s);
        if (a.V && tma_sel_rot)
          bj_rot_tma<<<grid, 256, kRotTmaSmem, st>>>(*reinterpret_cast<BJGemmArgs<double>*>(&gv), s, tm_w, tm_v);
        else if (a.V)
          bj_rot_mma<<<grid, 256, kRotSmem, st>>>(*reinterpret_cast<BJGemmArgs<double>*>(&gv), s);
      } else if (bg) {
        const int TT = kk / 16;
        if (TT == 1) bj_gram<T, 1><<<grid, 256, 0, st>>>(g, s);
        if (TT == 2) bj_gram<T, 2><<<grid, 256, 0, st>>>(g, s);
        if (TT == 3) bj_gram<T, 3><<<grid, 256, 0, st>>>(g, s);
        if (kUseMma<T>(TT) && tma_sel_gram)
          bj_gram_tma<<<grid, 256, 0, st>>>(*reinterpret_cast<BJGemmArgs<double>*>(&g), s, tm_w);
        else if (kUseMma<T>(TT))
          bj_gram_mma<<<grid, 256, 0, st>>>(*reinterpret_cast<BJGemmArgs<double>*>(&g), s);
        else if (TT == 4)
          bj_gram<T, 4><<<grid, 256, 0, st>>>(g, s);
        int rc = launch_svd(sizeof(T) == 8 ? 0 : 1, in, iws, iws_bytes, st);
        if (rc) return rc;
        if (TT == 1) bj_rot<T, 1><<<grid, 256, rot_smem, st>>>(g, s);
        if (TT == 2) bj_rot<T, 2><<<grid, 256, rot_smem, st>>>(g, s);
        if (TT == 3) bj_rot<T, 3><<<grid, 256, rot_smem, st>>>(g, s);
        if (kUseMma<T>(TT) && tma_sel_rot)
          bj_rot_tma<<<grid, 256, kRotTmaSmem, st>>>(*reinterpret_cast<BJGemmArgs<double>*>(&g), s, tm_w, tm_v);
        else if (kUseMma<T>(TT))
          bj_rot_mma<<<grid, 256, kRotSmem, st>>>(*reinterpret_cast<BJGemmArgs<double>*>(&g), s);
        else if (TT == 4)
          bj_rot<T, 4><<<grid, 256, rot_smem, st>>>(g, s);
      } else if (L.method == 0) {
        bj_gram_step<T><<<grid, 256, smem, st>>>(a, s);
      } else {
        bj_direct_step<T><<<grid, 256, smem, st>>>(a, s);
      }
    }
    int* cnt = ring + sw % kCtlRing;
    cudaMemsetAsync(cnt, 0, sizeof(int), st);
    bj_finalize_sweep<T><<<(unsigned)((L.batch + 255) / 256), 256, 0, st>>>(a, cnt);
    if (ctl) {
      cudaMemcpyAsync(ctl->host + sw % kCtlRing, cnt, sizeof(int), cudaMemcpyDeviceToHost, st);
      cudaEventRecord(ctl->ev[sw % kCtlRing], st);
      ctl->recorded[sw % kCtlRing] = true;
    }
  }
  if (L.stats && (bg || bd || wide)) bj_stats_reduce<T><<<(unsigned)((L.batch + 255) / 256), 256, 0, st>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  size_t xs = (size_t)np * (sizeof(T) + sizeof(int)) + 16;
  e = smem_optin((const void*)bj_extract<T>, (size_t)(xs));
  if (e != cudaSuccess) return (int)e;
  bj_extract<T><<<(unsigned)L.batch, 256, xs, st>>>(a, (T*)L.u, (T*)L.s, (T*)L.v, (T*)(base + lay.cand));
  return (int)cudaGetLastError();
}

int launch_block_svd(int dtype, const BlockLaunch& L, void* ws, cudaStream_t st) {
  if (L.batch == 0) return 0;
  return dtype == 0 ? launch_block_t<double>(L, ws, st) : launch_block_t<float>(L, ws, st);
}

}  // namespace bf
