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
#include <cuda.h>  // CUtensorMap (the tensor-map TMA variant; encoded on the host, block_kernels.cu)

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
  int only_v = 0;
  int64_t* stats = nullptr;  // batch x 4 work counters (BlockLaunch::stats) or null
  int tma = 3;  // bit 0: bj_gram_mma, bit 1: bj_rot_mma stage with TMA bulk copies (even ld)  // bj_rot_mma: update the V pair only (direct method)
};

BF_DEV int bj_pair_col(int c, int k, int bi, int bj) { return c < k ? bi * k + c : bj * k + (c - k); }

// per-matrix work counters: one pair visit (Gram / pair QR + e), and whether it rotated
BF_DEV void bj_count(int64_t* stats, int64_t b, bool rotated) {
  if (!stats) return;
  atomicAdd(reinterpret_cast<unsigned long long*>(stats + 4 * b), 1ull);
  if (rotated) atomicAdd(reinterpret_cast<unsigned long long*>(stats + 4 * b + 1), 1ull);
}

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
    bj_count(a.stats, b, e > a.tol);
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

// ------------------------------------------------------------------------------------------
// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) versions for 2k = 64, the BASELINE block width.
// Tensor-core fragments (PTX m8n8k4 .f64): lane = 4 g + t holds A[g][t], B[t][g] and
// D[g][2t], D[g][2t+1]. A CTA of 8 warps owns one (matrix, block pair); warp w computes a 16 x 32
// block (2 x 4 tiles) of the 64-wide output so each k-step issues 6 fragment loads per 8 DMMAs.
// Operands are staged column-major in shared memory (row stride padded so the 4 k-rows x 8
// columns of a fragment load hit two wavefronts) by 16-byte cp.async, double buffered.
BF_DEV void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
BF_DEV void cpa16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
BF_DEV void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
BF_DEV void cpa_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}


// 1-D TMA (cp.async.bulk) staging: one bulk copy per column segment (the column-major blocks
// are contiguous per column), completion counted in bytes on an mbarrier (complete_tx).
BF_DEV unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
BF_DEV void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
BF_DEV void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
BF_DEV void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
      ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
BF_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
BF_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 2-D tensor-map TMA (cp.async.bulk.tensor): W viewed as a (rows = m) x (cols = B * n_pad)
// column-major tensor, box = 8 rows x 32 columns (one block's columns, 64 B of each), 64-byte
// swizzle. One elected thread issues 2 blocks x (chunk rows / 8) boxes per chunk; rows past m
// arrive as zeros (TMA out-of-bounds fill). In a [32 col][8 row] box the 16-byte chunk
// r / 2 of column c sits at chunk (r / 2) ^ ((c / 2) & 3) (64B pattern, 512 B period), which
// makes both fragment patterns below two wavefronts per warp load.
BF_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y) : "memory");
}
constexpr int kTmaBoxRows = 8, kTmaBoxCols = 32, kTmaBox = kTmaBoxRows * kTmaBoxCols;  // doubles per box
BF_DEV int swz64(int c, int r) { return c * kTmaBoxRows + ((((r >> 1) ^ ((c >> 1) & 3)) << 1) | (r & 1)); }

// BF_BLOCK_TMA bits: 1 / 2 = 1-D bulk staging of bj_gram_mma / bj_rot_mma, 4 / 8 = tensor-map
// TMA Gram / rotation kernels (bj_gram_tma / bj_rot_tma)
constexpr int kBlockTmaDefault = 12;  // tensor-map TMA kernels (measured: on par or 0.2-0.5 % faster than cp.async; 1-D bulk 1.4-3.5 % slower)
constexpr int kMmaKK = 64;   // pair width 2k
constexpr int kGramCH = 32;  // rows per staged chunk (8 k-steps)
constexpr int kGramLD = kGramCH + 4;

// G = P^T P for P = [W_bi W_bj] (m x 64), e = scaled_offdiag(G), activity mask (see bj_gram).
__global__ void __launch_bounds__(256) bj_gram_mma(BJGemmArgs<double> a, int step) {
  constexpr int KK = kMmaKK, CH = kGramCH, LDR = kGramLD, LDG = KK + 1;
  __shared__ __align__(16) double stage[2][KK * LDR];
  __shared__ double red;
  __shared__ __align__(8) uint64_t bars[2];
  double* Gs = &stage[0][0];  // 64 x 65 after the accumulation (fits in the two stages)
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
  const int k = a.k, m = a.m, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = (warp >> 1) * 16, j0 = (warp & 1) * 32;  // output rows (cols of P) / cols
  const double* Wb = a.W + b * (int64_t)m * a.n_pad;
  // even m: every column segment starts 16-byte aligned -> TMA bulk copies (warp 0 issues one
  // per column); odd m: 16-byte cp.async per 2 rows
  const bool tma = (a.tma & 1) && (m & 1) == 0;
  unsigned phase = 0u;  // bit b: parity of buffer b's next completion (a register, not a local array)
  if (tma) {
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
    }
    fence_proxy_async();
    __syncthreads();
  }
  auto load = [&](int buf, int r0) {
    if (tma) {
      const int rows = min(CH, m - r0);
      if (warp == 0) {
        fence_proxy_async();  // earlier generic reads of this buffer before the async writes
        if (lane == 0) mbar_expect_tx(&bars[buf], (unsigned)(KK * rows * sizeof(double)));
        __syncwarp();
        for (int c = lane; c < KK; c += 32)
          bulk_g2s(&stage[buf][c * LDR], Wb + (size_t)bj_pair_col(c, k, bi, bj) * m + r0,
                   (unsigned)(rows * sizeof(double)), &bars[buf]);
      }
      if (rows < CH)
        for (int e = tid; e < KK * (CH - rows); e += 256) stage[buf][(e / (CH - rows)) * LDR + rows + e % (CH - rows)] = 0.0;
      return;
    }
    // 64 columns x CH rows, 16 B (2 rows) per cp.async; rows past m are zero-filled; odd m
    // leaves every other column 8-byte aligned only -> plain loads
    for (int e = tid; e < KK * CH / 2; e += 256) {
      const int c = e / (CH / 2), r = 2 * (e % (CH / 2));
      double* dst = &stage[buf][c * LDR + r];
      if (r0 + r + 1 < m && (m & 1) == 0) {
        cpa16(dst, Wb + (size_t)bj_pair_col(c, k, bi, bj) * m + r0 + r);
      } else {
        const double* src = Wb + (size_t)bj_pair_col(c, k, bi, bj) * m + r0 + r;
        dst[0] = r0 + r < m ? src[0] : 0.0;
        dst[1] = r0 + r + 1 < m ? src[1] : 0.0;
      }
    }
    cpa_commit();
  };
  double acc[2][4][2];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int nch = (m + CH - 1) / CH;
  load(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) load((ch + 1) & 1, (ch + 1) * CH);
    if (tma) {
      mbar_wait(&bars[ch & 1], (phase >> (ch & 1)) & 1u);
      phase ^= 1u << (ch & 1);
    } else if (ch + 1 < nch) {
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    const double* S = stage[ch & 1];
#pragma unroll
    for (int k0 = 0; k0 < CH; k0 += 4) {
      double av[2], bv[4];
#pragma unroll
      for (int x = 0; x < 2; ++x) av[x] = S[(i0 + 8 * x + g) * LDR + k0 + t];  // A[g][t] = P[k][i]
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = S[(j0 + 8 * y + g) * LDR + k0 + t];  // B[t][g] = P[k][j]
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y], av[x], bv[y]);
    }
    __syncthreads();  // stage (ch & 1) is reloaded next iteration
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      Gs[(i0 + 8 * x + g) * LDG + j0 + 8 * y + 2 * t] = acc[x][y][0];
      Gs[(i0 + 8 * x + g) * LDG + j0 + 8 * y + 2 * t + 1] = acc[x][y][1];
    }
  if (tid == 0) red = 0.0;
  __syncthreads();
  // exactly symmetric (core.py:75-77: upper triangle mirrored), column-major out; e on the fly
  double* Gout = a.G + slot * KK * KK;
  double best = 0.0;
  for (int e = tid; e < KK * KK; e += 256) {
    const int j = e / KK, i = e % KK;  // G[i][j]
    const double gv = i <= j ? Gs[i * LDG + j] : Gs[j * LDG + i];
    Gout[e] = gv;
    if (i != j) {
      const double den = sqrt(fabs(Gs[i * LDG + i])) * sqrt(fabs(Gs[j * LDG + j]));
      const double num = fabs(gv);
      const double rt = den > 0.0 ? num / den : (num > 0.0 ? __longlong_as_double(0x7ff0000000000000LL) : 0.0);
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
    bj_count(a.stats, b, e > a.tol);
  }
}

// bj_gram_mma fed by 2-D tensor-map TMA (see tma_load_2d): same product, e and mask.
__global__ void __launch_bounds__(256) bj_gram_tma(BJGemmArgs<double> a, int step, const __grid_constant__ CUtensorMap tmW) {
  constexpr int KK = kMmaKK, CH = kGramCH, NS = CH / kTmaBoxRows, LDG = KK + 1;
  constexpr int STAGE = 2 * NS * kTmaBox;  // doubles per buffer (2 blocks x NS boxes)
  static_assert(2 * STAGE <= KK * LDG, "stages alias G");
  __shared__ __align__(1024) double sm[KK * LDG + 64];
  __shared__ double red;
  __shared__ __align__(8) uint64_t bars[2];
  double* Gs = sm;
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
  const int k = a.k, m = a.m, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int i0 = (warp >> 1) * 16, j0 = (warp & 1) * 32;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  fence_proxy_async();
  __syncthreads();
  const int yi = (int)(b * a.n_pad + (int64_t)bi * k), yj = (int)(b * a.n_pad + (int64_t)bj * k);
  auto load = [&](int buf, int r0) {
    if (tid == 0) {
      fence_proxy_async();
      mbar_expect_tx(&bars[buf], (unsigned)(STAGE * sizeof(double)));
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        tma_load_2d(sm + buf * STAGE + s * kTmaBox, &tmW, &bars[buf], r0 + s * kTmaBoxRows, yi);
        tma_load_2d(sm + buf * STAGE + (NS + s) * kTmaBox, &tmW, &bars[buf], r0 + s * kTmaBoxRows, yj);
      }
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  const int nch = (m + CH - 1) / CH;
  unsigned phase = 0u;  // bit b: parity of buffer b's next completion (a register, not a local array)
  load(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) load((ch + 1) & 1, (ch + 1) * CH);
    mbar_wait(&bars[ch & 1], (phase >> (ch & 1)) & 1u);
    phase ^= 1u << (ch & 1);
    const double* S = sm + (ch & 1) * STAGE;
#pragma unroll
    for (int k0 = 0; k0 < CH; k0 += 4) {
      const int kr = k0 + t, box = kr / kTmaBoxRows, rr = kr % kTmaBoxRows;
      double av[2], bv[4];
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int i = i0 + 8 * x + g;  // pair column: block i / 32, column i % 32
        av[x] = S[((i >> 5) * NS + box) * kTmaBox + swz64(i & 31, rr)];
      }
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int j = j0 + 8 * y + g;
        bv[y] = S[((j >> 5) * NS + box) * kTmaBox + swz64(j & 31, rr)];
      }
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y], av[x], bv[y]);
    }
    __syncthreads();  // buffer (ch & 1) is reloaded next iteration / aliased by G
  }
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      Gs[(i0 + 8 * x + g) * LDG + j0 + 8 * y + 2 * t] = acc[x][y][0];
      Gs[(i0 + 8 * x + g) * LDG + j0 + 8 * y + 2 * t + 1] = acc[x][y][1];
    }
  if (tid == 0) red = 0.0;
  __syncthreads();
  double* Gout = a.G + slot * KK * KK;
  double best = 0.0;
  for (int e = tid; e < KK * KK; e += 256) {
    const int j = e / KK, i = e % KK;
    const double gv = i <= j ? Gs[i * LDG + j] : Gs[j * LDG + i];
    Gout[e] = gv;
    if (i != j) {
      const double den = sqrt(fabs(Gs[i * LDG + i])) * sqrt(fabs(Gs[j * LDG + j]));
      const double num = fabs(gv);
      const double rt = den > 0.0 ? num / den : (num > 0.0 ? __longlong_as_double(0x7ff0000000000000LL) : 0.0);
      best = rt > best ? rt : best;
    }
  }
  best = warp_allreduce_max(best);
  if ((tid & 31) == 0 && best > 0.0) bj_atomic_max_pos(&red, best);
  __syncthreads();
  if (tid == 0) {
    const double e = red;
    bj_atomic_max_pos(a.e_sweep + b, e);
    a.pair_act[slot] = e > a.tol ? 1 : 0;
    bj_count(a.stats, b, e > a.tol);
  }
}

constexpr int kRotCH = 64;           // rows per chunk
constexpr int kRotLDX = kRotCH + 8;  // X chunk row stride (column-major, 64 rows)
constexpr int kRotLDU = kMmaKK + 4;  // U stride (column-major)
constexpr size_t kRotSmem = (size_t)(kMmaKK * kRotLDU + 2 * kMmaKK * kRotLDX + kMmaKK) * sizeof(double);

// pair <- pair @ U_G (null directions zeroed), V pair <- V pair @ U_G (see bj_rot).
__global__ void __launch_bounds__(256) bj_rot_mma(BJGemmArgs<double> a, int step) {
  constexpr int KK = kMmaKK, CH = kRotCH, LDX = kRotLDX, LDU = kRotLDU;
  extern __shared__ __align__(16) double sm_rot[];
  double* Us = sm_rot;                // U column-major: U[k][n] at Us[n * LDU + k]
  double* Xs = Us + KK * LDU;         // 2 chunks, column-major: X[r][c] at Xs[c * LDX + r]
  double* sig = Xs + 2 * KK * LDX;    // inner sigma (null directions)
  __shared__ __align__(8) uint64_t bars[2];
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  const int64_t slot = blockIdx.x;
  if (b >= a.batch || !a.pair_act[slot]) return;
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, m = a.m, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0w = (warp >> 1) * 16, c0w = (warp & 1) * 32;
  const double* Ug = a.U + slot * KK * KK;
  for (int e = tid; e < KK * KK / 2; e += 256) {
    const int c = e / (KK / 2), r = 2 * (e % (KK / 2));
    cpa16(&Us[c * LDU + r], Ug + (size_t)c * KK + r);
  }
  cpa_commit();
  if (tid < KK) sig[tid] = a.S[slot * KK + tid];
  // the chunk sequence runs over W (m rows) then V (n_pad rows)
  double* Wm = a.W + b * (int64_t)m * a.n_pad;
  double* Vm = a.V ? a.V + b * (int64_t)a.n_pad * a.n_pad : nullptr;
  const int nw_ch = a.only_v ? 0 : (m + CH - 1) / CH, nv_ch = Vm ? (a.n_pad + CH - 1) / CH : 0;
  const int nch = nw_ch + nv_ch;
  if (nch == 0) return;
  auto where = [&](int ch, double*& M, int& ld, int& rows, int& r0, bool& isw) {
    isw = ch < nw_ch;
    M = isw ? Wm : Vm;
    ld = isw ? m : a.n_pad;
    rows = ld;
    r0 = (isw ? ch : ch - nw_ch) * CH;
  };
  // even leading dimensions: TMA bulk copies, one per column segment, issued by warp 0
  const bool tma = (a.tma & 2) && (m & 1) == 0 && (a.n_pad & 1) == 0;
  unsigned phase = 0u;  // bit b: parity of buffer b's next completion (a register, not a local array)
  if (tma) {
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
    }
    fence_proxy_async();
    __syncthreads();
  }
  auto load = [&](int buf, int ch) {
    double* M;
    int ld, rows, r0;
    bool isw;
    where(ch, M, ld, rows, r0, isw);
    double* X = Xs + buf * KK * LDX;
    if (tma) {
      const int nr = min(CH, rows - r0);
      if (warp == 0) {
        fence_proxy_async();
        if (lane == 0) mbar_expect_tx(&bars[buf], (unsigned)(KK * nr * sizeof(double)));
        __syncwarp();
        for (int c = lane; c < KK; c += 32)
          bulk_g2s(&X[c * LDX], M + (size_t)bj_pair_col(c, k, bi, bj) * ld + r0, (unsigned)(nr * sizeof(double)),
                   &bars[buf]);
      }
      if (nr < CH)
        for (int e = tid; e < KK * (CH - nr); e += 256) X[(e / (CH - nr)) * LDX + nr + e % (CH - nr)] = 0.0;
      return;
    }
    for (int e = tid; e < KK * CH / 2; e += 256) {
      const int c = e / (CH / 2), r = 2 * (e % (CH / 2));
      double* dst = &X[c * LDX + r];
      const double* src = M + (size_t)bj_pair_col(c, k, bi, bj) * ld + r0 + r;
      if (r0 + r + 1 < rows && (ld & 1) == 0) {  // odd ld: 8-byte aligned columns only
        cpa16(dst, src);
      } else {
        dst[0] = r0 + r < rows ? src[0] : 0.0;
        dst[1] = r0 + r + 1 < rows ? src[1] : 0.0;
      }
    }
    cpa_commit();
  };
  load(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) load((ch + 1) & 1, ch + 1);
    if (tma) {
      if (ch == 0) cpa_wait<0>();  // U (cp.async)
      mbar_wait(&bars[ch & 1], (phase >> (ch & 1)) & 1u);
      phase ^= 1u << (ch & 1);
    } else if (ch + 1 < nch) {
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    const double* X = Xs + (ch & 1) * KK * LDX;
    double acc[2][4][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < KK; k0 += 4) {
      double av[2], bv[4];
#pragma unroll
      for (int x = 0; x < 2; ++x) av[x] = X[(k0 + t) * LDX + r0w + 8 * x + g];  // A[g][t] = X[r][k]
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = Us[(c0w + 8 * y + g) * LDU + k0 + t];  // B[t][g] = U[k][n]
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y], av[x], bv[y]);
    }
    double* M;
    int ld, rows, r0;
    bool isw;
    where(ch, M, ld, rows, r0, isw);
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int r = r0 + r0w + 8 * x + g;
      if (r < rows) {
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int c = c0w + 8 * y + 2 * t + q;
            // keep exactly-null directions exactly null (blockjacobi.py:133-134)
            const double val = (isw && !(sig[c] != 0.0)) ? 0.0 : acc[x][y][q];
            M[(size_t)bj_pair_col(c, k, bi, bj) * ld + r] = val;
          }
      }
    }
    __syncthreads();  // chunk buffer (ch & 1) is reloaded next iteration
  }
}


// bj_rot_mma fed by 2-D tensor-map TMA: the W and V chunks (64 rows x the pair's 64 columns)
// arrive as 2 blocks x 8 swizzled 8 x 32 boxes per chunk (block_gemm.cuh tma_load_2d); the
// A-fragment reads (rows g, column k0 + t) are two wavefronts under the 64B swizzle.
constexpr int kRotTmaStage = 2 * (kRotCH / kTmaBoxRows) * kTmaBox;  // doubles per chunk buffer
constexpr size_t kRotTmaSmem = (size_t)(2 * kRotTmaStage + kMmaKK * kRotLDU + kMmaKK) * sizeof(double) + 1024;

__global__ void __launch_bounds__(256) bj_rot_tma(BJGemmArgs<double> a, int step, const __grid_constant__ CUtensorMap tmW,
                                                  const __grid_constant__ CUtensorMap tmV) {
  constexpr int KK = kMmaKK, CH = kRotCH, NS = CH / kTmaBoxRows, LDU = kRotLDU, STAGE = kRotTmaStage;
  extern __shared__ double sm_rot_raw[];
  double* Xs = (double*)(((uintptr_t)sm_rot_raw + 1023) & ~(uintptr_t)1023);  // swizzle period alignment
  double* Us = Xs + 2 * STAGE;  // U column-major: U[k][n] at Us[n * LDU + k]
  double* sig = Us + KK * LDU;
  __shared__ __align__(8) uint64_t bars[2];
  const int P = a.nb / 2;
  const int64_t b = blockIdx.x / P;
  const int pk = blockIdx.x % P;
  const int64_t slot = blockIdx.x;
  if (b >= a.batch || !a.pair_act[slot]) return;
  int bi, bj;
  rr_pair(a.nb, step, pk, bi, bj);
  const int k = a.k, m = a.m, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int r0w = (warp >> 1) * 16, c0w = (warp & 1) * 32;
  const double* Ug = a.U + slot * KK * KK;
  for (int e = tid; e < KK * KK / 2; e += 256) {
    const int c = e / (KK / 2), r = 2 * (e % (KK / 2));
    cpa16(&Us[c * LDU + r], Ug + (size_t)c * KK + r);
  }
  cpa_commit();
  if (tid < KK) sig[tid] = a.S[slot * KK + tid];
  double* Wm = a.W + b * (int64_t)m * a.n_pad;
  double* Vm = a.V ? a.V + b * (int64_t)a.n_pad * a.n_pad : nullptr;
  const int nw_ch = a.only_v ? 0 : (m + CH - 1) / CH, nv_ch = Vm ? (a.n_pad + CH - 1) / CH : 0;
  const int nch = nw_ch + nv_ch;
  if (nch == 0) return;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
  }
  fence_proxy_async();
  __syncthreads();
  const int yi = (int)(b * a.n_pad + (int64_t)bi * k), yj = (int)(b * a.n_pad + (int64_t)bj * k);
  auto load = [&](int buf, int ch) {
    if (tid == 0) {
      const bool isw = ch < nw_ch;
      const CUtensorMap* map = isw ? &tmW : &tmV;
      const int r0 = (isw ? ch : ch - nw_ch) * CH;
      double* X = Xs + buf * STAGE;
      fence_proxy_async();
      mbar_expect_tx(&bars[buf], (unsigned)(STAGE * sizeof(double)));
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        tma_load_2d(X + s * kTmaBox, map, &bars[buf], r0 + s * kTmaBoxRows, yi);
        tma_load_2d(X + (NS + s) * kTmaBox, map, &bars[buf], r0 + s * kTmaBoxRows, yj);
      }
    }
  };
  unsigned phase = 0u;  // bit b: parity of buffer b's next completion (a register, not a local array)
  load(0, 0);
  cpa_wait<0>();  // U
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) load((ch + 1) & 1, ch + 1);
    mbar_wait(&bars[ch & 1], (phase >> (ch & 1)) & 1u);
    phase ^= 1u << (ch & 1);
    const double* X = Xs + (ch & 1) * STAGE;
    double acc[2][4][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < KK; k0 += 4) {
      const int c = k0 + t;  // pair column: block c / 32, column c % 32
      double av[2], bv[4];
#pragma unroll
      for (int x = 0; x < 2; ++x)
        av[x] = X[((c >> 5) * NS + ((r0w + 8 * x) >> 3)) * kTmaBox + swz64(c & 31, g)];  // A[g][t] = X[r][k]
#pragma unroll
      for (int y = 0; y < 4; ++y) bv[y] = Us[(c0w + 8 * y + g) * LDU + k0 + t];  // B[t][g] = U[k][n]
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) dmma_8x8x4(acc[x][y], av[x], bv[y]);
    }
    const bool isw = ch < nw_ch;
    double* M = isw ? Wm : Vm;
    const int ld = isw ? m : a.n_pad, rows = ld, r0 = (isw ? ch : ch - nw_ch) * CH;
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int r = r0 + r0w + 8 * x + g;
      if (r < rows) {
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int c = c0w + 8 * y + 2 * t + q;
            const double val = (isw && !(sig[c] != 0.0)) ? 0.0 : acc[x][y][q];  // blockjacobi.py:133-134
            M[(size_t)bj_pair_col(c, k, bi, bj) * ld + r] = val;
          }
      }
    }
    __syncthreads();  // chunk buffer (ch & 1) is reloaded next iteration
  }
}

}  // namespace bf
