// Block-Jacobi Gram path kernels (blockjacobi.py:124-134), batched over (matrix, block pair):
//   bj_gram: G = pair^T pair (syrk, core.py:68-78, mirrored exactly symmetric), the scaled
//            off-diagonal e (blockjacobi.py:57-76) -> per-sweep max, and the activity mask
//            (e > tol) that drives the batched inner SVD;
//   bj_rot:  pair <- pair @ U_G with exactly-null directions zeroed, V pair <- V pair @ U_G.
// The inner SVD of every active G runs in between as ONE batched call of the register-tier
// Jacobi kernel (round robin, no V; blockjacobi.py:79-81, :130).
// Tiles: 256 threads, thread (ti, tj) owns entries (ti + 16a, tj + 16b), a, b < TT (kk = 16*TT),
// so every shared-memory read in the inner loop is a broadcast or a 128-byte contiguous row.
#pragma once
#include "common.cuh"

namespace bf {

template <typename T>
struct BJGemmArgs {
  int64_t batch;
  int m, n_pad, k, nb;
  T* W;
  T* V;
  T* G;               // batch * P x kk x kk
  T* U;               // batch * P x kk x kk (inner U, sorted)
  T* S;               // batch * P x kk (inner sigma, sorted)
  uint8_t* pair_act;  // batch * P
  const uint8_t* active;
  double* e_sweep;
  double tol;
};

BF_DEV int bj_pair_col(int c, int k, int bi, int bj) { return c < k ? bi * k + c : bj * k + (c - k); }

BF_DEV void bj_atomic_max_pos(double* addr, double v) {
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}

template <typename T, int TT>
__global__ void __launch_bounds__(256) bj_gram(BJGemmArgs<T> a, int step) {
  constexpr int KK = 16 * TT, LD = KK + 1, CH = 32;
  __shared__ T buf[(KK > CH ? KK : CH) * LD];
  T* chunk = buf;  // row chunk during the accumulation
  T* Gs = buf;     // G afterwards
  __shared__ double red;
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  const int64_t slot = blockIdx.x;
  if (b >= a.batch) return;
  if (!a.active[b]) {
    if (threadIdx.x == 0) a.pair_act[slot] = 0;
    return;
  }
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, m = a.m, tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const T* Wb = a.W + b * (int64_t)m * a.n_pad;
  T acc[TT][TT];
#pragma unroll
  for (int x = 0; x < TT; ++x)
#pragma unroll
    for (int y = 0; y < TT; ++y) acc[x][y] = T(0);
  for (int r0 = 0; r0 < m; r0 += CH) {
    const int nr = m - r0 < CH ? m - r0 : CH;
    __syncthreads();
    for (int e = tid; e < KK * CH; e += 256) {
      const int c = e / CH, r = e % CH;
      chunk[r * LD + c] = r < nr ? Wb[(size_t)bj_pair_col(c, k, bi, bj) * m + r0 + r] : T(0);
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < CH; ++r) {
      T av[TT], bv[TT];
#pragma unroll
      for (int x = 0; x < TT; ++x) {
        av[x] = chunk[r * LD + ti + 16 * x];
        bv[x] = chunk[r * LD + tj + 16 * x];
      }
#pragma unroll
      for (int x = 0; x < TT; ++x)
#pragma unroll
        for (int y = 0; y < TT; ++y) acc[x][y] = fma(av[x], bv[y], acc[x][y]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int x = 0; x < TT; ++x)
#pragma unroll
    for (int y = 0; y < TT; ++y) Gs[(ti + 16 * x) * LD + tj + 16 * y] = acc[x][y];
  if (tid == 0) red = 0.0;
  __syncthreads();
  // exactly symmetric (core.py:75-77: upper triangle mirrored), column-major out; e on the fly
  T* Gout = a.G + slot * KK * KK;
  double best = 0.0;
  for (int e = tid; e < KK * KK; e += 256) {
    const int j = e / KK, i = e % KK;  // G[i][j]
    const T g = i <= j ? Gs[i * LD + j] : Gs[j * LD + i];
    Gout[e] = g;
    if (i != j) {
      const T di = (T)sqrt((double)fabs((double)Gs[i * LD + i]));
      const T dj = (T)sqrt((double)fabs((double)Gs[j * LD + j]));
      const T den = di * dj;
      const T num = g < T(0) ? -g : g;
      const double rt =
          den > T(0) ? (double)(num / den) : (num > T(0) ? __longlong_as_double(0x7ff0000000000000LL) : 0.0);
      best = rt > best ? rt : best;
    }
  }
  best = warp_allreduce_max(best);
  if ((tid & 31) == 0 && best > 0.0) bj_atomic_max_pos(&red, best);
  __syncthreads();
  if (tid == 0) {
    const double e = red;
    bj_atomic_max_pos(a.e_sweep + b, e);
    a.pair_act[slot] = e > a.tol ? 1 : 0;  // pairs at e <= tol are skipped (blockjacobi.py:128-129)
  }
}

template <typename T, int TT>
__global__ void __launch_bounds__(256) bj_rot(BJGemmArgs<T> a, int step) {
  constexpr int KK = 16 * TT, LD = KK + 1, CH = 16 * TT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* Us = reinterpret_cast<T*>(smem_raw);  // KK x LD (row k, col c)
  T* X = Us + KK * LD;                     // CH x LD rows of the panel
  __shared__ T sig[KK];
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  const int64_t slot = blockIdx.x;
  if (b >= a.batch || !a.pair_act[slot]) return;
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, m = a.m, tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const T* Ug = a.U + slot * KK * KK;
  for (int e = tid; e < KK * KK; e += 256) {
    const int c = e / KK, r = e % KK;  // U column-major: U[r][c]
    Us[r * LD + c] = Ug[e];
  }
  if (tid < KK) sig[tid] = a.S[slot * KK + tid];
  for (int pass = 0; pass < 2; ++pass) {
    T* M = pass == 0 ? a.W + b * (int64_t)m * a.n_pad : (a.V ? a.V + b * (int64_t)a.n_pad * a.n_pad : nullptr);
    if (!M) break;
    const int rows = pass == 0 ? m : a.n_pad, ld = rows;
    for (int r0 = 0; r0 < rows; r0 += CH) {
      const int nr = rows - r0 < CH ? rows - r0 : CH;
      __syncthreads();
      for (int e = tid; e < KK * CH; e += 256) {
        const int c = e / CH, r = e % CH;
        X[r * LD + c] = r < nr ? M[(size_t)bj_pair_col(c, k, bi, bj) * ld + r0 + r] : T(0);
      }
      __syncthreads();
      T acc[TT][TT];
#pragma unroll
      for (int x = 0; x < TT; ++x)
#pragma unroll
        for (int y = 0; y < TT; ++y) acc[x][y] = T(0);
#pragma unroll 4
      for (int kq = 0; kq < KK; ++kq) {
        T xv[TT], uv[TT];
#pragma unroll
        for (int x = 0; x < TT; ++x) {
          xv[x] = X[(ti + 16 * x) * LD + kq];
          uv[x] = Us[kq * LD + tj + 16 * x];
        }
#pragma unroll
        for (int x = 0; x < TT; ++x)
#pragma unroll
          for (int y = 0; y < TT; ++y) acc[x][y] = fma(xv[x], uv[y], acc[x][y]);
      }
#pragma unroll
      for (int x = 0; x < TT; ++x) {
        const int r = ti + 16 * x;
        if (r < nr) {
#pragma unroll
          for (int y = 0; y < TT; ++y) {
            const int c = tj + 16 * y;
            // keep exactly-null directions exactly null (blockjacobi.py:133-134)
            const T val = (pass == 0 && !(sig[c] != T(0))) ? T(0) : acc[x][y];
            M[(size_t)bj_pair_col(c, k, bi, bj) * ld + r0 + r] = val;
          }
        }
      }
    }
  }
}

}  // namespace bf
