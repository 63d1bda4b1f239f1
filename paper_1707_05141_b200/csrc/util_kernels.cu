// Small batched helpers: tiled GEMM, numpy-compatible Gaussian sampler, column fixes.
#include "common.cuh"
#include "internal.h"

#define BF_ZIG_QUAL static __device__ const
#include "ziggurat_tables.h"

namespace bf {

// ------------------------------------------------------------------ batched GEMM
// C (M x N) = op(A) (M x K) * op(B) (K x N), column-major, 64x64 tile per CTA,
// 256 threads x (4x4) register micro-tiles, K staged through shared memory.
template <typename T>
__global__ void __launch_bounds__(256) gemm_kernel(GemmLaunch g) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tiles_m = (g.M + BM - 1) / BM;
  const int tm = blockIdx.x % tiles_m, tn = blockIdx.x / tiles_m;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  for (int64_t b = blockIdx.y; b < g.batch; b += gridDim.y) {
    const T* A = (const T*)g.a + b * g.a_stride;
    const T* B = (const T*)g.b + b * g.b_stride;
    T* C = (T*)g.c + b * g.c_stride;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    for (int k0 = 0; k0 < g.K; k0 += BK) {
      for (int e = threadIdx.x; e < BK * BM; e += 256) {
        int kk = e / BM, ii = e % BM;
        int gi = tm * BM + ii, gk = k0 + kk;
        T val = 0;
        if (gi < g.M && gk < g.K) val = g.ta ? A[(size_t)gi * g.lda + gk] : A[(size_t)gk * g.lda + gi];
        As[kk][ii] = val;
      }
      for (int e = threadIdx.x; e < BK * BN; e += 256) {
        int kk = e % BK, jj = e / BK;
        int gj = tn * BN + jj, gk = k0 + kk;
        T val = 0;
        if (gj < g.N && gk < g.K) val = g.tb ? B[(size_t)gk * g.ldb + gj] : B[(size_t)gj * g.ldb + gk];
        Bs[kk][jj] = val;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        T av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[kk][tx + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][ty + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int gi = tm * BM + tx + 16 * i, gj = tn * BN + ty + 16 * j;
        if (gi < g.M && gj < g.N) C[(size_t)gj * g.ldc + gi] = acc[i][j];
      }
  }
}

int launch_gemm(int dtype, const GemmLaunch& g, cudaStream_t st) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return 0;
  int tiles = ((g.M + 63) / 64) * ((g.N + 63) / 64);
  unsigned gy = (unsigned)(g.batch < 65535 ? g.batch : 65535);
  if (dtype == 0)
    gemm_kernel<double><<<dim3(tiles, gy), 256, 0, st>>>(g);
  else
    gemm_kernel<float><<<dim3(tiles, gy), 256, 0, st>>>(g);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ Gaussian sampler
// numpy Generator(Philox(key=seed)).standard_normal((rows, cols)) (rsvd.py:42-53):
// Philox4x64-10 stream (counter incremented before each 4-word block), float64
// ziggurat (numpy random_standard_normal), C-order fill, stored column-major.
// One warp per matrix: lanes test 32 consecutive stream words against the
// ziggurat fast path in parallel; the rare slow path is walked by lane 0.

BF_DEV uint64_t philox_word(uint64_t k0, uint64_t k1, uint64_t pos) {
  uint64_t c0 = (pos >> 2) + 1, c1 = 0, c2 = 0, c3 = 0;
  if (c0 == 0) c1 = 1;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  switch (pos & 3) {
    case 0: return c0;
    case 1: return c1;
    case 2: return c2;
    default: return c3;
  }
}

BF_DEV double u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

__global__ void gaussian_kernel(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi,
                                int64_t index_base, int seed_mode, uint64_t xor_mask, double* out,
                                int64_t out_stride) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= batch) return;
  uint64_t gi = (uint64_t)(index_base + b);
  const uint64_t k0 = (seed_mode == 0 ? (seed_lo ^ gi) : (seed_lo + gi)) ^ xor_mask;
  const uint64_t k1 = seed_hi;
  double* o = out + b * out_stride;
  const int64_t total = (int64_t)rows * cols;
  int64_t k = 0;
  uint64_t pos = 0;
  while (k < total) {
    uint64_t r = philox_word(k0, k1, pos + lane);
    int idx = (int)(r & 0xff);
    uint64_t rr = r >> 8;
    int sign = (int)(rr & 1);
    uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * bf_zig_wi[idx];
    if (sign) x = -x;
    bool fast = rabs < bf_zig_ki[idx];
    unsigned bal = __ballot_sync(FULL, !fast);
    int L = bal ? __ffs(bal) - 1 : 32;
    if (lane < L && k + lane < total) {
      int64_t kk = k + lane;
      o[(kk % cols) * rows + kk / cols] = x;
    }
    if (L == 32) {
      k += 32;
      pos += 32;
      continue;
    }
    // slow path for the candidate at stream position pos + L (lane L holds it)
    double xs = __shfl_sync(FULL, x, L);
    uint64_t rabs_s = __shfl_sync(FULL, rabs, L);
    int idx_s = __shfl_sync(FULL, idx, L);
    uint64_t p = pos + L + 1;
    int produced = 0;
    double val = 0.0;
    if (lane == 0) {
      if (idx_s == 0) {
        for (;;) {
          double xx = -BF_ZIG_NOR_INV_R * log1p(-u01(philox_word(k0, k1, p)));
          double yy = -log1p(-u01(philox_word(k0, k1, p + 1)));
          p += 2;
          if (yy + yy > xx * xx) {
            val = ((rabs_s >> 8) & 0x1) ? -(BF_ZIG_NOR_R + xx) : BF_ZIG_NOR_R + xx;
            produced = 1;
            break;
          }
        }
      } else {
        double u = u01(philox_word(k0, k1, p));
        p += 1;
        if (((bf_zig_fi[idx_s - 1] - bf_zig_fi[idx_s]) * u + bf_zig_fi[idx_s]) < exp(-0.5 * xs * xs)) {
          val = xs;
          produced = 1;
        }
      }
      if (produced && k + L < total) {
        int64_t kk = k + L;
        o[(kk % cols) * rows + kk / cols] = val;
      }
    }
    produced = __shfl_sync(FULL, produced, 0);
    p = __shfl_sync(FULL, p, 0);
    k += L + produced;
    pos = p;
  }
}

int launch_gaussian_f64(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, int64_t index_base,
                        int seed_mode, uint64_t xor_mask, double* out, int64_t out_stride, cudaStream_t st) {
  if (batch == 0 || rows == 0 || cols == 0) return 0;
  const int wpb = 4;
  unsigned grid = (unsigned)((batch + wpb - 1) / wpb);
  gaussian_kernel<<<grid, wpb * 32, 0, st>>>(batch, rows, cols, seed_lo, seed_hi, index_base, seed_mode, xor_mask,
                                               out, out_stride);
  return (int)cudaGetLastError();
}

// random_orthonormal sign fix (testmat.py:68-80): flip column j where R_jj < 0.
__global__ void sign_fix_kernel(int64_t batch, int m, int n, double* q, const double* r) {
  int64_t b = blockIdx.x;
  if (b >= batch) return;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    int j = e / m;
    if (r[b * n * n + (size_t)j * n + j] < 0) q[b * m * n + e] = -q[b * m * n + e];
  }
}

int launch_sign_fix_f64(int64_t batch, int m, int n, double* q, const double* r, cudaStream_t st) {
  if (batch == 0) return 0;
  sign_fix_kernel<<<(unsigned)batch, 256, 0, st>>>(batch, m, n, q, r);
  return (int)cudaGetLastError();
}

__global__ void scale_cols_kernel(int64_t batch, int m, int n, double* q, const double* sigma) {
  int64_t b = blockIdx.x;
  if (b >= batch) return;
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) q[b * m * n + e] *= sigma[e / m];
}

int launch_scale_cols_f64(int64_t batch, int m, int n, double* q, const double* sigma, cudaStream_t st) {
  if (batch == 0) return 0;
  scale_cols_kernel<<<(unsigned)batch, 256, 0, st>>>(batch, m, n, q, sigma);
  return (int)cudaGetLastError();
}

}  // namespace bf
