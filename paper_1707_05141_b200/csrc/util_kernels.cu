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

// FP64 tensor-core (DMMA m8n8k4) batched GEMM for the tall-skinny products of the randomized SVD
// (Y = A Omega, B^T = A^T Q, U = Q U_R, V = Q_B V_R: M <= 128, N <= 64): one CTA of 8 warps per
// matrix, warp w owns row tiles 2w, 2w+1 and all NT column tiles of C. K is staged in chunks of
// 16 by 16-byte cp.async (zero-filled past M / N / K), double buffered; each operand keeps its
// global contiguity in shared memory (A: k-major when not transposed, i-major when transposed;
// B likewise), with padded strides so a fragment load is two wavefronts.
// Fragments: lane = 4 g + t holds A[g][t], B[t][g], D[g][2t + q].
BF_DEV void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
BF_DEV void cpa16z(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(n) : "memory");
}

constexpr int kGmKC = 16;          // K chunk
constexpr int kGmLDAk = 128 + 8;   // A, not transposed: As[k * LDAk + i]
constexpr int kGmLDAi = kGmKC + 4; // A, transposed:     As[i * LDAi + k]
constexpr int kGmLDBk = kGmKC + 4; // B, not transposed: Bs[j * LDBk + k]
constexpr int kGmLDBj = 64 + 8;    // B, transposed:     Bs[k * LDBj + j]
constexpr int kGmAStage = 128 * (kGmLDAk > kGmLDAi * 8 ? kGmLDAk : kGmLDAi * 8);  // >= both layouts
constexpr int kGmAStageD = (kGmKC * kGmLDAk > 128 * kGmLDAi ? kGmKC * kGmLDAk : 128 * kGmLDAi);
constexpr int kGmBStageD = (64 * kGmLDBk > kGmKC * kGmLDBj ? 64 * kGmLDBk : kGmKC * kGmLDBj);
constexpr size_t kGmSmem = (size_t)2 * (kGmAStageD + kGmBStageD) * sizeof(double);

template <int NT, bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_mma_kernel(GemmLaunch g) {
  extern __shared__ __align__(16) double gsm[];
  double* As0 = gsm;
  double* Bs0 = gsm + 2 * kGmAStageD;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, t = lane & 3;
  const int i0 = warp * 16;
  const int nk = (g.K + kGmKC - 1) / kGmKC;
  for (int64_t b = blockIdx.x; b < g.batch; b += gridDim.x) {
    const double* A = (const double*)g.a + b * g.a_stride;
    const double* B = (const double*)g.b + b * g.b_stride;
    double* C = (double*)g.c + b * g.c_stride;
    auto stage = [&](int buf, int k0) {
      double* As = As0 + buf * kGmAStageD;
      double* Bs = Bs0 + buf * kGmBStageD;
      if (!TA) {  // A column-major M x K: 2 consecutive rows i per 16 B
        for (int e = tid; e < kGmKC * 64; e += 256) {
          const int kk = e >> 6, ii = 2 * (e & 63), gk = k0 + kk;
          const bool ok = ii < g.M && gk < g.K;
          cpa16z(&As[kk * kGmLDAk + ii], ok ? A + (size_t)gk * g.lda + ii : A, ok);
        }
      } else {  // A stored K x M: 2 consecutive k per 16 B
        for (int e = tid; e < 128 * (kGmKC / 2); e += 256) {
          const int ii = e / (kGmKC / 2), kk = 2 * (e % (kGmKC / 2)), gk = k0 + kk;
          const bool ok = ii < g.M && gk < g.K;
          cpa16z(&As[ii * kGmLDAi + kk], ok ? A + (size_t)ii * g.lda + gk : A, ok);
        }
      }
      if (!TB) {  // B column-major K x N: 2 consecutive k per 16 B
        for (int e = tid; e < 8 * NT * (kGmKC / 2); e += 256) {
          const int jj = e / (kGmKC / 2), kk = 2 * (e % (kGmKC / 2)), gk = k0 + kk;
          const bool ok = jj < g.N && gk < g.K;
          cpa16z(&Bs[jj * kGmLDBk + kk], ok ? B + (size_t)jj * g.ldb + gk : B, ok);
        }
      } else {  // B stored N x K (row-major K x N): 2 consecutive j per 16 B
        for (int e = tid; e < kGmKC * 4 * NT; e += 256) {
          const int kk = e / (4 * NT), jj = 2 * (e % (4 * NT)), gk = k0 + kk;
          const bool ok = jj < g.N && gk < g.K;
          cpa16z(&Bs[kk * kGmLDBj + jj], ok ? B + (size_t)gk * g.ldb + jj : B, ok);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[2][NT][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < NT; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    __syncthreads();  // previous matrix done with the stages
    stage(0, 0);
    for (int kc = 0; kc < nk; ++kc) {
      if (kc + 1 < nk) {
        stage((kc + 1) & 1, (kc + 1) * kGmKC);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double* As = As0 + (kc & 1) * kGmAStageD;
      const double* Bs = Bs0 + (kc & 1) * kGmBStageD;
#pragma unroll
      for (int kq = 0; kq < kGmKC; kq += 4) {
        double av[2], bv[NT];
#pragma unroll
        for (int x = 0; x < 2; ++x)
          av[x] = TA ? As[(i0 + 8 * x + gq) * kGmLDAi + kq + t] : As[(kq + t) * kGmLDAk + i0 + 8 * x + gq];
#pragma unroll
        for (int y = 0; y < NT; ++y)
          bv[y] = TB ? Bs[(kq + t) * kGmLDBj + 8 * y + gq] : Bs[(8 * y + gq) * kGmLDBk + kq + t];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < NT; ++y) dmma884(acc[x][y], av[x], bv[y]);
      }
      __syncthreads();  // this stage is refilled two chunks later
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int i = i0 + 8 * x + gq;
      if (i < g.M) {
#pragma unroll
        for (int y = 0; y < NT; ++y)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int j = 8 * y + 2 * t + q;
            if (j < g.N) C[(size_t)j * g.ldc + i] = acc[x][y][q];
          }
      }
    }
  }
}

template <int NT, bool TA, bool TB>
static void launch_gemm_mma_t(const GemmLaunch& g, cudaStream_t st) {
  cudaFuncSetAttribute(gemm_mma_kernel<NT, TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGmSmem);
  int dev = 0, sms = 148, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, gemm_mma_kernel<NT, TA, TB>, 256, kGmSmem);
  if (per < 1) per = 1;
  const int64_t cap = (int64_t)sms * per;
  const unsigned grid = (unsigned)(g.batch < cap ? g.batch : cap);
  gemm_mma_kernel<NT, TA, TB><<<grid, 256, kGmSmem, st>>>(g);
}

template <int NT>
static void launch_gemm_mma(const GemmLaunch& g, cudaStream_t st) {
  if (!g.ta && !g.tb) launch_gemm_mma_t<NT, false, false>(g, st);
  if (!g.ta && g.tb) launch_gemm_mma_t<NT, false, true>(g, st);
  if (g.ta && !g.tb) launch_gemm_mma_t<NT, true, false>(g, st);
  if (g.ta && g.tb) launch_gemm_mma_t<NT, true, true>(g, st);
}

// 16-byte cp.async needs 16-byte aligned rows: even leading dimensions and strides
static bool gemm_mma_ok(const GemmLaunch& g) {
  auto even = [](int64_t x) { return (x & 1) == 0; };
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  return g.M <= 128 && g.N <= 64 && even(g.lda) && even(g.ldb) && even(g.a_stride) && even(g.b_stride) &&
         al16(g.a) && al16(g.b);
}

int launch_gemm(int dtype, const GemmLaunch& g, cudaStream_t st) {
  if (g.batch == 0 || g.M == 0 || g.N == 0) return 0;
  if (dtype == 0 && gemm_mma_ok(g)) {
    switch ((g.N + 7) / 8) {
      case 1: launch_gemm_mma<1>(g, st); break;
      case 2: launch_gemm_mma<2>(g, st); break;
      case 3: launch_gemm_mma<3>(g, st); break;
      case 4: launch_gemm_mma<4>(g, st); break;
      case 5: launch_gemm_mma<5>(g, st); break;
      case 6: launch_gemm_mma<6>(g, st); break;
      case 7: launch_gemm_mma<7>(g, st); break;
      default: launch_gemm_mma<8>(g, st); break;
    }
    return (int)cudaGetLastError();
  }
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
// ziggurat (numpy random_standard_normal), C-order fill.
// One warp per matrix: each lane computes one Philox block (4 consecutive stream words), so a
// warp tests 128 words against the ziggurat fast path at once; accepted samples are compacted
// by a warp prefix sum and stored contiguously (C order) or transposed (column-major). The rare
// slow path (~1.2% of words: wedge / tail) is walked by lane 0 and the warp resumes after it.

BF_DEV void philox_block(uint64_t k0, uint64_t k1, uint64_t blk, uint64_t (&w)[4]) {
  uint64_t c0 = blk + 1, c1 = 0, c2 = 0, c3 = 0;
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
  w[0] = c0;
  w[1] = c1;
  w[2] = c2;
  w[3] = c3;
}

BF_DEV uint64_t philox_word(uint64_t k0, uint64_t k1, uint64_t pos) {
  uint64_t w[4];
  philox_block(k0, k1, pos >> 2, w);
  switch (pos & 3) {
    case 0: return w[0];
    case 1: return w[1];
    case 2: return w[2];
    default: return w[3];
  }
}

BF_DEV double u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

__global__ void gaussian_kernel(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi,
                                int64_t index_base, int seed_mode, uint64_t xor_mask, double* out,
                                int64_t out_stride, int c_order) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= batch) return;
  uint64_t gi = (uint64_t)(index_base + b);
  const uint64_t k0 = (seed_mode == 0 ? (seed_lo ^ gi) : (seed_lo + gi)) ^ xor_mask;
  const uint64_t k1 = seed_hi;
  double* o = out + b * out_stride;
  const int64_t total = (int64_t)rows * cols;
  auto store = [&](int64_t kk, double v) {
    if (kk < total) {
      if (c_order)
        o[kk] = v;
      else
        o[(kk % cols) * rows + kk / cols] = v;
    }
  };
  int64_t k = 0;
  uint64_t pos = 0;
  while (k < total) {
    // one batch: lane l holds stream words 4 (blk + l) .. 4 (blk + l) + 3
    const uint64_t blk = pos >> 2;
    const uint64_t bend = (blk + 32) * 4;
    uint64_t w[4];
    philox_block(k0, k1, blk + lane, w);
    double x[4];
    bool fast[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t r = w[q];
      const int idx = (int)(r & 0xff);
      const uint64_t rr = r >> 8;
      const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
      const double v = (double)rabs * bf_zig_wi[idx];
      x[q] = (rr & 1) ? -v : v;
      fast[q] = rabs < bf_zig_ki[idx];
    }
    // the batch is consumed from `pos` on; every slow-path event is resolved inside it (its
    // extra words come from the batch's registers when they lie in it), so Philox runs once
    // per 128 words instead of once per event
    while (k < total && pos < bend) {
      const uint64_t lane0 = (blk + lane) * 4;  // stream position of this lane's word 0
      int rej = 4;
      int first = 4;  // first unconsumed word of this lane
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool live = lane0 + q >= pos;
        first = (live && first == 4) ? q : first;
        if (live && rej == 4 && !fast[q]) rej = q;
      }
      const unsigned bal = __ballot_sync(FULL, rej < 4);
      const int L = bal ? __ffs(bal) - 1 : 32;
      const int cnt = lane < L ? 4 - first : (lane == L ? rej - first : 0);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, d);
        if (lane >= d) incl += y;
      }
      const int start = incl - cnt;
      const int tot = __shfl_sync(FULL, incl, 31);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q >= first && q - first < cnt) store(k + start + (q - first), x[q]);
      k += tot;
      if (L == 32) {
        pos = bend;
        break;
      }
      // slow path for the first failing word (lane L, word q_s) at stream position ps
      const int q_s = __shfl_sync(FULL, rej, L);
      uint64_t r_s = w[0];
#pragma unroll
      for (int q = 1; q < 4; ++q) r_s = q == q_s ? w[q] : r_s;
      r_s = __shfl_sync(FULL, r_s, L);
      uint64_t p = (blk + L) * 4 + q_s + 1;
      // the wedge test's uniform is the next word: from the batch when it is in it
      const int lw = (int)((p >> 2) - blk), qw = (int)(p & 3);
      uint64_t r_u = w[0];
#pragma unroll
      for (int q = 1; q < 4; ++q) r_u = q == qw ? w[q] : r_u;
      r_u = __shfl_sync(FULL, r_u, lw < 32 ? lw : 0);
      int produced = 0;
      if (lane == 0 && k < total) {
        const int idx_s = (int)(r_s & 0xff);
        const uint64_t rr = r_s >> 8;
        const uint64_t rabs_s = (rr >> 1) & 0x000fffffffffffffULL;
        double xs = (double)rabs_s * bf_zig_wi[idx_s];
        if (rr & 1) xs = -xs;
        double val = 0.0;
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
          const double u = u01(lw < 32 ? r_u : philox_word(k0, k1, p));
          p += 1;
          if (((bf_zig_fi[idx_s - 1] - bf_zig_fi[idx_s]) * u + bf_zig_fi[idx_s]) < exp(-0.5 * xs * xs)) {
            val = xs;
            produced = 1;
          }
        }
        if (produced) store(k, val);
      }
      produced = __shfl_sync(FULL, produced, 0);
      p = __shfl_sync(FULL, p, 0);
      k += produced;
      pos = p;
    }
  }
}

int launch_gaussian_f64(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, int64_t index_base,
                        int seed_mode, uint64_t xor_mask, double* out, int64_t out_stride, cudaStream_t st,
                        int c_order) {
  if (batch == 0 || rows == 0 || cols == 0) return 0;
  const int wpb = 4;
  unsigned grid = (unsigned)((batch + wpb - 1) / wpb);
  gaussian_kernel<<<grid, wpb * 32, 0, st>>>(batch, rows, cols, seed_lo, seed_hi, index_base, seed_mode, xor_mask,
                                               out, out_stride, c_order);
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
