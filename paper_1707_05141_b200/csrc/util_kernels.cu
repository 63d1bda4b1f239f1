// Small batched helpers: tiled GEMM, numpy-compatible Gaussian sampler, column fixes.
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "internal.h"

#define BF_ZIG_QUAL static __device__ const
#include "ziggurat_tables.h"
#include "libm_log1p.h"

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
  smem_optin((const void*)gemm_mma_kernel<NT, TA, TB>, kGmSmem);
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
// numpy Generator(Philox(key=seed)).standard_normal((rows, cols), dtype) (rsvd.py:42-53; the
// reference passes dtype=a.dtype, rsvd.py:65): Philox4x64-10 stream (counter incremented before
// each 4-word block), C-order fill, and numpy's ziggurat for the dtype:
//   float64: random_standard_normal   -- one 64-bit word per draw, 52-bit rabs;
//   float32: random_standard_normal_f -- one 32-bit draw per try (next_uint32: the low half of a
//            word, then its high half), 23-bit rabs, float tables, double-precision wedge test.
// Bitwise equal to numpy: the tables are numpy's own (tools/gen_ziggurat_tables.py), every
// operation is an explicitly rounded IEEE op in numpy's order (no FMA contraction), and the tail
// uses log1p/log1pf restated from the host libm (libm_log1p.h). The wedge's exp() only decides
// accept/reject: CUDA's and glibc's exp differ by <= 1-2 ulp, which flips the decision only if
// the left side lands inside that ulp window (probability ~1e-14 per wedge event).
//
// One warp per matrix: each lane computes one Philox block (4 words = D draws), so a warp tests
// 32 D draws against the ziggurat fast path at once; accepted samples are compacted by a warp
// prefix sum and stored contiguously (C order) or transposed (column-major). The rare slow path
// (wedge / tail: ~1.2% of f64 draws) is walked by lane 0 and the warp resumes after it.

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

template <typename T>
struct Zig;

template <>
struct Zig<double> {
  using U = uint64_t;
  static constexpr int D = 4;  // draws per Philox block
  static BF_DEV void split(const uint64_t (&w)[4], U (&d)[D]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = w[q];
  }
  static BF_DEV U draw(uint64_t k0, uint64_t k1, uint64_t p) { return philox_word(k0, k1, p); }
  static BF_DEV double uni(U r) { return __dmul_rn((double)(r >> 11), 1.0 / 9007199254740992.0); }  // next_double
  // fast path: x = rabs * wi[idx] (sign from bit 8), accepted iff rabs < ki[idx]
  static BF_DEV bool fast(U r, double& x) {
    const int idx = (int)(r & 0xff);
    const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
    const double v = __dmul_rn((double)rabs, bf_zig_wi[idx]);
    x = ((r >> 8) & 1) ? -v : v;
    return rabs < bf_zig_ki[idx];
  }
  // slow path of draw r (numpy random_standard_normal after the fast test fails); the next draw
  // is `nxt` when the caller has it (has_nxt), else read from the stream at p. Advances p.
  static BF_DEV bool slow(U r, U nxt, bool has_nxt, uint64_t k0, uint64_t k1, uint64_t& p, double& val) {
    const int idx = (int)(r & 0xff);
    const uint64_t rabs = (r >> 9) & 0x000fffffffffffffULL;
    double xs = __dmul_rn((double)rabs, bf_zig_wi[idx]);
    if ((r >> 8) & 1) xs = -xs;
    if (idx == 0) {
      for (;;) {
        const double xx = __dmul_rn(-BF_ZIG_NOR_INV_R, bf_libm::log1p_d(-uni(draw(k0, k1, p))));
        const double yy = -bf_libm::log1p_d(-uni(draw(k0, k1, p + 1)));
        p += 2;
        if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
          const double t = __dadd_rn(xx, BF_ZIG_NOR_R);
          val = ((rabs >> 8) & 0x1) ? -t : t;
          return true;
        }
      }
    }
    const double u = uni(has_nxt ? nxt : draw(k0, k1, p));
    p += 1;
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(bf_zig_fi[idx - 1], bf_zig_fi[idx]), u), bf_zig_fi[idx]);
    val = xs;
    return lhs < exp(__dmul_rn(__dmul_rn(-0.5, xs), xs));
  }
};

template <>
struct Zig<float> {
  using U = uint32_t;
  static constexpr int D = 8;
  static BF_DEV void split(const uint64_t (&w)[4], U (&d)[D]) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      d[2 * q] = (uint32_t)(w[q] & 0xffffffffu);
      d[2 * q + 1] = (uint32_t)(w[q] >> 32);
    }
  }
  static BF_DEV U draw(uint64_t k0, uint64_t k1, uint64_t p) {
    const uint64_t w = philox_word(k0, k1, p >> 1);
    return (p & 1) ? (uint32_t)(w >> 32) : (uint32_t)(w & 0xffffffffu);
  }
  static BF_DEV float uni(U r) { return __fmul_rn((float)(r >> 8), 1.0f / 16777216.0f); }  // next_float
  static BF_DEV bool fast(U r, float& x) {
    const int idx = (int)(r & 0xff);
    const uint32_t rabs = r >> 9;
    const float v = __fmul_rn((float)rabs, bf_zig_wi_f[idx]);
    x = ((r >> 8) & 1) ? -v : v;
    return rabs < bf_zig_ki_f[idx];
  }
  static BF_DEV bool slow(U r, U nxt, bool has_nxt, uint64_t k0, uint64_t k1, uint64_t& p, float& val) {
    const int idx = (int)(r & 0xff);
    const uint32_t rabs = r >> 9;
    float xs = __fmul_rn((float)rabs, bf_zig_wi_f[idx]);
    if ((r >> 8) & 1) xs = -xs;
    if (idx == 0) {
      for (;;) {
        const float xx = __fmul_rn(-BF_ZIG_NOR_INV_R_F, bf_libm::log1p_f(-uni(draw(k0, k1, p))));
        const float yy = -bf_libm::log1p_f(-uni(draw(k0, k1, p + 1)));
        p += 2;
        if (__fadd_rn(yy, yy) > __fmul_rn(xx, xx)) {
          const float t = __fadd_rn(xx, BF_ZIG_NOR_R_F);
          val = ((rabs >> 8) & 0x1) ? -t : t;
          return true;
        }
      }
    }
    const float u = uni(has_nxt ? nxt : draw(k0, k1, p));
    p += 1;
    const float lhs = __fadd_rn(__fmul_rn(u, __fsub_rn(bf_zig_fi_f[idx - 1], bf_zig_fi_f[idx])), bf_zig_fi_f[idx]);
    val = xs;
    const double xd = (double)xs;
    return (double)lhs < exp(__dmul_rn(__dmul_rn(-0.5, xd), xd));
  }
};

template <typename T>
BF_DEV typename Zig<T>::U shfl_draw(typename Zig<T>::U v, int src) {
  return __shfl_sync(FULL, v, src);
}

// maps {0,1} -> {0,1} as 2-bit codes (bit s = f(s)); fn_comp(g, f) = g o f
constexpr int kFnZero = 0, kFnNot = 1, kFnId = 2, kFnOne = 3;
BF_DEV int fn_comp(int g, int f) { return ((g >> (f & 1)) & 1) | (((g >> ((f >> 1) & 1)) & 1) << 1); }

#ifndef BF_GAUSS_SERIAL_SLOW
#define BF_GAUSS_SERIAL_SLOW 0
#endif
#ifndef BF_GAUSS_NB
#define BF_GAUSS_NB 1
#endif

template <typename T>
__global__ void gaussian_kernel(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi,
                                int64_t index_base, int seed_mode, uint64_t xor_mask, T* out, int64_t out_stride,
                                int c_order) {
  using Z = Zig<T>;
  using U = typename Z::U;
  constexpr int NB = BF_GAUSS_NB;  // Philox blocks per lane per batch
  constexpr int D = Z::D * NB;     // draws per lane per batch
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= batch) return;
  uint64_t gi = (uint64_t)(index_base + b);
  const uint64_t k0 = (seed_mode == 0 ? (seed_lo ^ gi) : (seed_lo + gi)) ^ xor_mask;
  const uint64_t k1 = seed_hi;
  T* o = out + b * out_stride;
  const int64_t total = (int64_t)rows * cols;
  auto store = [&](int64_t kk, T v) {
    if (kk < total) {
      if (c_order)
        o[kk] = v;
      else
        o[(kk % cols) * rows + kk / cols] = v;
    }
  };
  int64_t k = 0;
  uint64_t pos = 0;  // stream position in draws
  while (k < total) {
    // one batch: lane l holds draws D (blk + l) .. D (blk + l) + D - 1
    const uint64_t blk = pos / D;
    const uint64_t bend = (blk + 32) * D;
    U d[D];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
      uint64_t w[4];
      philox_block(k0, k1, (blk + lane) * NB + nb, w);
      U dd[Z::D];
      Z::split(w, dd);
#pragma unroll
      for (int q = 0; q < Z::D; ++q) d[nb * Z::D + q] = dd[q];
    }
    T x[D];
    bool fast[D];
#pragma unroll
    for (int q = 0; q < D; ++q) fast[q] = Z::fast(d[q], x[q]);
#if BF_GAUSS_SERIAL_SLOW
    // (previous design, kept for A/B) the batch is consumed from `pos` on; every slow-path event
    // is resolved inside it by lane 0 while the warp waits, splitting the batch at each event
    while (k < total && pos < bend) {
      const uint64_t lane0 = (blk + lane) * D;  // stream position of this lane's draw 0
      int rej = D;
      int first = D;  // first unconsumed draw of this lane
#pragma unroll
      for (int q = 0; q < D; ++q) {
        const bool live = lane0 + q >= pos;
        first = (live && first == D) ? q : first;
        if (live && rej == D && !fast[q]) rej = q;
      }
      const unsigned bal = __ballot_sync(FULL, rej < D);
      const int L = bal ? __ffs(bal) - 1 : 32;
      const int cnt = lane < L ? D - first : (lane == L ? rej - first : 0);
      int incl = cnt;
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, dd);
        if (lane >= dd) incl += y;
      }
      const int start = incl - cnt;
      const int tot = __shfl_sync(FULL, incl, 31);
#pragma unroll
      for (int q = 0; q < D; ++q)
        if (q >= first && q - first < cnt) store(k + start + (q - first), x[q]);
      k += tot;
      if (L == 32) {
        pos = bend;
        break;
      }
      // slow path for the first failing draw (lane L, draw q_s) at stream position ps
      const int q_s = __shfl_sync(FULL, rej, L);
      U r_s = d[0];
#pragma unroll
      for (int q = 1; q < D; ++q) r_s = q == q_s ? d[q] : r_s;
      r_s = shfl_draw<T>(r_s, L);
      uint64_t p = (blk + L) * D + q_s + 1;
      // the wedge test's uniform is the next draw: from the batch when it is in it
      const int lw = (int)(p / D - blk), qw = (int)(p % D);
      U r_u = d[0];
#pragma unroll
      for (int q = 1; q < D; ++q) r_u = q == qw ? d[q] : r_u;
      r_u = shfl_draw<T>(r_u, lw < 32 ? lw : 0);
      int produced = 0;
      if (lane == 0 && k < total) {
        T val;
        if (Z::slow(r_s, r_u, lw < 32, k0, k1, p, val)) {
          store(k, val);
          produced = 1;
        }
      }
      produced = __shfl_sync(FULL, produced, 0);
      p = __shfl_sync(FULL, p, 0);
      k += produced;
      pos = p;
    }
#else
    // One pass per batch. Which positions start a draw is a linear recurrence -- position P
    // starts a draw unless P - 1 started one that failed the fast test (its wedge test consumes
    // P as the uniform) -- so each position's transition start[P-1] -> start[P] is one of
    // {const 0 (before pos), const 1, NOT}; composing them is a warp scan. Every wedge test of
    // the batch then runs in parallel on its own lane, and one more scan packs the accepted
    // draws in stream order. Only a tail event (idx 0, an unbounded number of words) ends the
    // batch early and is resolved by lane 0.
    const uint64_t P0 = (blk + lane) * D;  // stream position of this lane's draw 0
    bool rej[D];
#pragma unroll
    for (int q = 0; q < D; ++q) rej[q] = !fast[q];
    const bool prev_rej = __shfl_up_sync(FULL, (int)rej[D - 1], 1) != 0;
    int tr[D], F = kFnId;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      const uint64_t P = P0 + q;
      tr[q] = P < pos ? kFnZero : (P == pos ? kFnOne : ((q == 0 ? prev_rej : rej[q - 1]) ? kFnNot : kFnOne));
      F = fn_comp(tr[q], F);
    }
    int h = F;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const int y = __shfl_up_sync(FULL, h, dd);
      if (lane >= dd) h = fn_comp(h, y);
    }
    int S = __shfl_up_sync(FULL, h, 1);
    int sv = lane == 0 ? 0 : (S & 1);  // start[P0 - 1]
    bool st[D];
    int qt = D;  // first draw of this lane that starts a tail event
#pragma unroll
    for (int q = 0; q < D; ++q) {
      sv = (tr[q] >> sv) & 1;
      st[q] = sv != 0;
      if (st[q] && rej[q] && (d[q] & 0xff) == 0 && qt == D) qt = q;
    }
    const unsigned tball = __ballot_sync(FULL, qt < D);
    const int Lt = tball ? __ffs(tball) - 1 : 32;
    const int qlim = lane < Lt ? D : (lane == Lt ? qt : 0);  // this lane's draws before the tail
    const U nxt0 = shfl_draw<T>(d[0], lane < 31 ? lane + 1 : lane);
    T val[D];
    bool prod[D];
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < D; ++q) {
      prod[q] = false;
      val[q] = x[q];
      if (q < qlim && st[q]) {
        if (fast[q]) {
          prod[q] = true;
        } else {  // wedge test with the next position's word as the uniform
          uint64_t p = P0 + q + 1;
          const U nx = q + 1 < D ? d[(q + 1) % D] : nxt0;
          T v;
          if (Z::slow(d[q], nx, q + 1 < D || lane < 31, k0, k1, p, v)) {
            prod[q] = true;
            val[q] = v;
          }
        }
      }
      cnt += prod[q] ? 1 : 0;
    }
    int incl = cnt;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const int y = __shfl_up_sync(FULL, incl, dd);
      if (lane >= dd) incl += y;
    }
    int off = incl - cnt;
#pragma unroll
    for (int q = 0; q < D; ++q)
      if (prod[q]) store(k + off++, val[q]);
    k += __shfl_sync(FULL, incl, 31);
    if (Lt < 32) {  // tail event at lane Lt, draw qt: lane 0 runs it, the next batch starts after it
      U r_t = d[0];
      const int q_t = __shfl_sync(FULL, qt, Lt);
#pragma unroll
      for (int q = 1; q < D; ++q) r_t = q == q_t ? d[q] : r_t;
      r_t = shfl_draw<T>(r_t, Lt);
      uint64_t p = (blk + Lt) * D + q_t + 1;
      if (lane == 0 && k < total) {
        T v;
        if (Z::slow(r_t, r_t, false, k0, k1, p, v)) store(k, v);
      }
      p = __shfl_sync(FULL, p, 0);
      k += 1;
      pos = p;
    } else {
      // a wedge event on the batch's last position consumed the next batch's first word
      const bool last = __shfl_sync(FULL, (int)(st[D - 1] && rej[D - 1]), 31) != 0;
      pos = bend + (last ? 1 : 0);
    }
#endif
  }
}

template <typename T>
int launch_gaussian(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, int64_t index_base,
                    int seed_mode, uint64_t xor_mask, T* out, int64_t out_stride, cudaStream_t st, int c_order) {
  if (batch == 0 || rows == 0 || cols == 0) return 0;
  const int wpb = 4;
  unsigned grid = (unsigned)((batch + wpb - 1) / wpb);
  gaussian_kernel<T><<<grid, wpb * 32, 0, st>>>(batch, rows, cols, seed_lo, seed_hi, index_base, seed_mode,
                                                  xor_mask, out, out_stride, c_order);
  return (int)cudaGetLastError();
}

int launch_gaussian_f64(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, int64_t index_base,
                        int seed_mode, uint64_t xor_mask, double* out, int64_t out_stride, cudaStream_t st,
                        int c_order) {
  return launch_gaussian<double>(batch, rows, cols, seed_lo, seed_hi, index_base, seed_mode, xor_mask, out,
                                 out_stride, st, c_order);
}

int launch_gaussian_f32(int64_t batch, int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, int64_t index_base,
                        int seed_mode, uint64_t xor_mask, float* out, int64_t out_stride, cudaStream_t st,
                        int c_order) {
  return launch_gaussian<float>(batch, rows, cols, seed_lo, seed_hi, index_base, seed_mode, xor_mask, out,
                                out_stride, st, c_order);
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

cudaError_t smem_optin(const void* func, size_t need) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(func, dev);
  const auto it = granted.find(key);
  if (it != granted.end() && it->second >= need) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
  if (e == cudaSuccess) granted[key] = need;
  return e;
}

}  // namespace bf
