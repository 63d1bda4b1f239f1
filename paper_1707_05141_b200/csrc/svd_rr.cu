// Tiled register tier of the batched one-sided Jacobi SVD, round-robin ordering.
//
// Reference: _round_robin_sweep jacobi.py:158-186 (skip rule :167, identity for skipped pairs
// :177-185), svd :231-284 (sweep until a rotation-free sweep :270-281, off_orthogonality
// fallback :282-283, _extract_svd :212-228), round_robin_schedule :102-115.
//
// Layout. The round-robin schedule pairs positions (k, NP-1-k) (slot k) and after every step
// moves positions 1..NP-1 one place on (idx = [idx0, idx[-1]] + idx[1:-1]). A thread owns an
// R-row x S-slot tile of W: for each of its rows the S "a" positions sg*S + j and the S "b"
// positions NP-1-(sg*S + j) of slot group sg. Lane = rgl * SG + sg (rgl = row group within the
// warp), so the SG slot groups of a row group are adjacent lanes:
//   * a step's data movement is a FIFO shift inside each thread (compile-time register renaming
//     with period S, no moves) plus ONE value per row and direction crossing to the neighbouring
//     slot group (shfl up/down within SG lanes); the fixed position 0 and the ring's turn at the
//     middle are two per-lane selects;
//   * g_pq is a per-thread R-row partial, a shuffle butterfly over the warp's row groups and, for
//     NWARP > 1, one shared-memory exchange between warps (the only barrier of a step);
//   * lane rgl == j of each slot group computes slot j's Rutishauser rotation
//     (jacobi.py:68-80) -- every warp redundantly, on identical inputs -- and the S (c, s) pairs
//     reach the group's lanes by shuffles.
// Shared-memory traffic per step is a few hundred bytes per matrix (the row-per-thread layout
// of svd_reg.cu moves ~64 KB through shared memory per 64 x 64 step).
// Column norms are tracked (dgesvj scheme, see jacobi_reg.cuh) and recomputed at sweep start
// and after cancellation. V is rebuilt from a rotation log replayed on the same tiles.
#include <cstdio>

#include "internal.h"
#include "jacobi_cta.cuh"
#include "jacobi_reg.cuh"

namespace bf {

template <int NP_, int S_, int R_, int NW_>
struct RRCfg {
  static constexpr int NP = NP_, S = S_, R = R_, NWARP = NW_;
  static constexpr int NPAIR = NP / 2;
  static constexpr int SG = NPAIR / S;     // slot groups
  static constexpr int RGW = 32 / SG;      // row groups per warp
  static constexpr int ROWS = RGW * NWARP * R;
  static constexpr int THREADS = 32 * NWARP;
  static_assert(NPAIR % S == 0, "S divides the pair count");
  static_assert(32 % SG == 0 && SG >= 2, "slot groups tile a warp");
  static_assert(RGW >= S, "one rotation lane per slot in every slot group");
};

#ifndef BF_RR_STAGE
#define BF_RR_STAGE 8
#endif
constexpr int kRRStage = BF_RR_STAGE;
// per-launch budget of the per-matrix rotation logs (the batch is chunked beyond it)
constexpr size_t kRRLogBudget = (size_t)6 << 30;

#ifndef BF_RR64_R
#define BF_RR64_R 8  // rows per thread for 64 x 64 (8 -> 2 warps, 4 -> 4 warps per matrix)
#endif

template <typename C>
struct RRShared {
  // carved out of the extraction work region (free during the sweeps)
  static constexpr int PART = 2 * C::NWARP * 2 * C::NPAIR;  // [parity][warp][2 * NPAIR]
  static constexpr int DN = C::NWARP * C::NP;               // tracked norms per warp
  static constexpr int FS = C::NWARP * C::NP;               // column scales per warp
  static constexpr int STAGE = 2 * kRRStage * C::NPAIR * 2; // V log staging (doubles)
  static constexpr int SWEEP = PART + DN + FS;
};

BF_DEV void rr_bar(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

// column held by position x at round-robin step t (jacobi.py:111-114)
template <int NP>
BF_DEV int rr_col(int x, int t) {
  if (x == 0) return 0;
  int v = x - 1 - t;
  v += v < 0 ? NP - 1 : 0;
  return 1 + v;
}

template <class C>
struct RRTile {
  static constexpr int S = C::S, R = C::R, SG = C::SG;
  double A[R][S], B[R][S];  // physical FIFO registers (W phase: scaled columns, true = stored * fs[col])

  // logical a[j] / b[j] at phase PH
  template <int PH>
  static BF_DEV constexpr int ia(int j) {
    return ((j - PH) % S + S) % S;
  }
  template <int PH>
  static BF_DEV constexpr int ib(int j) {
    return (j + PH) % S;
  }

  // Scaled rotation (the deferred-normalisation form of the rotation, cf. LAPACK dgesvj's
  // fast rotations): with true columns a = fa * ~a, b = fb * ~b the rotation
  // a' = c a - s b, b' = s a + c b is ~a' = ~a + al ~b, ~b' = ~b + be ~a with
  // al = -t fb / fa, be = t fa / fb and the scales multiplied by c -- 2 FMAs per element
  // instead of 2 multiplies + 2 FMAs. Skipped pairs have al = be = 0.
  template <int PH>
  BF_DEV void apply(const double (&al)[S], const double (&be)[S]) {
#pragma unroll
    for (int j = 0; j < S; ++j)
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const double a = A[i][ia<PH>(j)], b = B[i][ib<PH>(j)];
        A[i][ia<PH>(j)] = fma(al[j], b, a);
        B[i][ib<PH>(j)] = fma(be[j], a, b);
      }
  }
  // multiply columns by per-column factors (t == 0: position == column), phase PH
  template <int PH>
  BF_DEV void scale_cols(const double* f, int sg) {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const double fa = f[sg * S + j], fb = f[C::NP - 1 - (sg * S + j)];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        A[i][ia<PH>(j)] *= fa;
        B[i][ib<PH>(j)] *= fb;
      }
    }
  }

  // one round-robin move: positions 1..NP-1 advance one place; the tile goes from phase PH to PH+1
  template <int PH>
  static BF_DEV void move1(double (&a)[S], double (&b)[S], bool first, bool last) {
    constexpr int XA = ia<PH>(S - 1);  // exiting a register -> logical a[0] at PH+1
    constexpr int YA = ia<PH>(0);      // old a[0] -> logical a[1] at PH+1
    constexpr int XB = ib<PH>(0);      // exiting b register -> logical b[S-1] at PH+1
    const double a_exit = a[XA], b_exit = b[XB];
    const double ra = __shfl_up_sync(FULL, a_exit, 1, SG);
    const double rb = __shfl_down_sync(FULL, b_exit, 1, SG);
    // slot group 0: position 0 is fixed and position 1 takes position NP-1's value
    const double y = a[YA];
    a[XA] = first ? y : ra;
    a[YA] = first ? b_exit : y;
    // last slot group: the ring turns from position NP/2-1 to NP/2 inside the thread
    b[XB] = last ? a_exit : rb;
  }
  template <int PH>
  BF_DEV void move(int sg) {
    const bool first = sg == 0, last = sg == SG - 1;
#pragma unroll
    for (int i = 0; i < R; ++i) move1<PH>(A[i], B[i], first, last);
  }

  template <int PH>
  BF_DEV void partial_dots(double (&g)[S]) const {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      double acc = A[0][ia<PH>(j)] * B[0][ib<PH>(j)];
#pragma unroll
      for (int i = 1; i < R; ++i) acc = fma(A[i][ia<PH>(j)], B[i][ib<PH>(j)], acc);
      g[j] = acc;
    }
  }
  template <int PH>
  BF_DEV void partial_norms(double (&na)[S], double (&nb)[S]) const {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      double xa = A[0][ia<PH>(j)] * A[0][ia<PH>(j)], xb = B[0][ib<PH>(j)] * B[0][ib<PH>(j)];
#pragma unroll
      for (int i = 1; i < R; ++i) {
        xa = fma(A[i][ia<PH>(j)], A[i][ia<PH>(j)], xa);
        xb = fma(B[i][ib<PH>(j)], B[i][ib<PH>(j)], xb);
      }
      na[j] = xa;
      nb[j] = xb;
    }
  }

  // positions -> columns at t == 0 (identity): write the tile to column-major smem (ld rows)
  template <int PH>
  BF_DEV void store(double* M, int ld, int nrows, int ncols, int row0, int sg) const {
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int ca = sg * S + j, cb = C::NP - 1 - (sg * S + j);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int r = row0 + i;
        if (r < nrows) {
          if (ca < ncols) M[(size_t)ca * ld + r] = A[i][ia<PH>(j)];
          if (cb < ncols) M[(size_t)cb * ld + r] = B[i][ib<PH>(j)];
        }
      }
    }
  }
  BF_DEV void store_phase(int ph, double* M, int ld, int nrows, int ncols, int row0, int sg) const {
    switch (ph) {
      case 0: store<0>(M, ld, nrows, ncols, row0, sg); break;
      case 1: store<1 % S>(M, ld, nrows, ncols, row0, sg); break;
      case 2: store<2 % S>(M, ld, nrows, ncols, row0, sg); break;
      case 3: store<3 % S>(M, ld, nrows, ncols, row0, sg); break;
      case 4: store<4 % S>(M, ld, nrows, ncols, row0, sg); break;
      default: store<5 % S>(M, ld, nrows, ncols, row0, sg); break;
    }
  }
};

// lane-dependent pick of x[j] for j = idx (idx < S), uniform code
template <int S>
BF_DEV double pick(const double (&x)[S], int idx) {
  double r = x[0];
#pragma unroll
  for (int j = 1; j < S; ++j) r = idx == j ? x[j] : r;
  return r;
}

template <class C>
struct RRWork {
  static constexpr int S = C::S, SG = C::SG, NP = C::NP, NPAIR = C::NPAIR, NWARP = C::NWARP;
  int lane, warp, sg, rgl, n, max_sweeps;
  double tol2;
  double* part;  // [2][NWARP][2 * NPAIR]
  double* d;     // this warp's NP tracked norms
  double* fs;    // this warp's NP column scales (scaled rotations: true column = stored * fs[col])
  double2* log;  // global cursor (warp 0 writes): per step and slot (al, be)
  double* slog;  // global cursor (warp 0 writes): per sweep the NP column scales
  int ex, sweeps, conv, rot, recompute;
  long long rots;
#ifdef BF_RR_PHASE
  long long ph[6];
#endif

  BF_DEV bool rot_lane() const { return rgl < S; }
  BF_DEV int slot() const { return sg * S + rgl; }

  // sum over the warp's row groups (xor over the lane bits above the slot-group bits)
  template <int K>
  BF_DEV void warp_sum(double (&x)[K]) const {
#pragma unroll
    for (int o = SG; o < 32; o <<= 1)
#pragma unroll
      for (int j = 0; j < K; ++j) x[j] += __shfl_xor_sync(FULL, x[j], o);
  }
  // add the other warps' partials of this lane's slot value(s) (fixed warp order)
  template <int K>
  BF_DEV void cross_warp(double (&v)[K]) {
    if (NWARP == 1) return;
    double* buf = part + (ex & 1) * NWARP * 2 * NPAIR;
    ++ex;
    if (rot_lane())
#pragma unroll
      for (int q = 0; q < K; ++q) buf[warp * 2 * NPAIR + q * NPAIR + slot()] = v[q];
    rr_bar(C::THREADS);
    if (rot_lane()) {
#pragma unroll
      for (int q = 0; q < K; ++q) {
        double tot = buf[q * NPAIR + slot()];
#pragma unroll
        for (int w = 1; w < NWARP; ++w) tot += buf[w * 2 * NPAIR + q * NPAIR + slot()];
        v[q] = tot;
      }
    }
  }

  template <int PH>
  BF_DEV void norms(RRTile<C>& tile, int t) {
    double na[S], nb[S];
    tile.template partial_norms<PH>(na, nb);
    warp_sum(na);
    warp_sum(nb);
    double v[2] = {pick<S>(na, rgl), pick<S>(nb, rgl)};
    cross_warp(v);
    if (rot_lane()) {
      const int k = slot();
      const int ca = rr_col<NP>(k, t), cb = rr_col<NP>(NP - 1 - k, t);
      const double fa = fs[ca], fb = fs[cb];
      d[ca] = v[0] * (fa * fa);
      d[cb] = v[1] * (fb * fb);
    }
    __syncwarp();
    recompute = 0;
  }

  template <int PH>
  BF_DEV void sweep_start(RRTile<C>& tile, int t) {
    rot = 0;
    norms<PH>(tile, t);
  }

  template <int PH>
  BF_DEV void step(RRTile<C>& tile, int t) {
#ifdef BF_RR_PHASE
    long long c0 = clock64();
#endif
    if (recompute) norms<PH>(tile, t);
    double g[S];
    tile.template partial_dots<PH>(g);
    warp_sum(g);
    double v[1] = {pick<S>(g, rgl)};
#ifdef BF_RR_PHASE
    long long c1 = clock64();
#endif
    cross_warp(v);
#ifdef BF_RR_PHASE
    long long c2 = clock64();
#endif
    double al = 0.0, be = 0.0;
    int flag = 0;
    if (rot_lane()) {
      const int k = slot();
      const int ca = rr_col<NP>(k, t), cb = rr_col<NP>(NP - 1 - k, t);
      const double fa = fs[ca], fb = fs[cb];
      const bool rev = ca > cb;  // slot a holds the larger column: rotate with swapped roles
      const int p = rev ? cb : ca, q = rev ? ca : cb;
      const double dpp = d[p], dqq = d[q], gpq = v[0] * (fa * fb);
      if (gpq * gpq > tol2 * (dpp * dqq)) {  // skip rule (jacobi.py:167)
        double cc, sn, tt;
        jacobi_rotation_t(dpp, gpq, dqq, cc, sn, tt);
        const double np_ = dpp - tt * gpq, nq = dqq + tt * gpq;
        d[p] = np_ > 0.0 ? np_ : 0.0;
        d[q] = nq > 0.0 ? nq : 0.0;
        flag = (np_ < 1e-2 * dpp) | (nq < 1e-2 * dqq);  // cancellation -> recompute next step
        const double tp = rev ? -tt : tt;               // tangent in position order (a, b)
        const double rinv = rcp_fast(fa * fb);
        al = -tp * (fb * fb) * rinv;
        be = tp * (fa * fa) * rinv;
        fs[ca] = fa * cc;  // the rotation's cosine moves into the column scales
        fs[cb] = fb * cc;
        ++rot;
      }
      if (log != nullptr && warp == 0) log[k] = make_double2(al, be);
    }
    if (log != nullptr) log += NPAIR;
    // order this step's d updates before the next step's reads by other lanes (with several
    // warps the next step's cross-warp barrier already does; racecheck-clean either way)
    if (NWARP == 1) __syncwarp();
    recompute = __any_sync(FULL, flag);
#ifdef BF_RR_PHASE
    long long c3 = clock64();
#endif
    double a[S], b[S];
#pragma unroll
    for (int j = 0; j < S; ++j) {
      a[j] = __shfl_sync(FULL, al, j * SG + sg);
      b[j] = __shfl_sync(FULL, be, j * SG + sg);
    }
    tile.template apply<PH>(a, b);
#ifdef BF_RR_PHASE
    long long c4 = clock64();
#endif
    tile.template move<PH>(sg);
#ifdef BF_RR_PHASE
    long long c5 = clock64();
    ph[0] += c1 - c0;
    ph[1] += c2 - c1;
    ph[2] += c3 - c2;
    ph[3] += c4 - c3;
    ph[4] += c5 - c4;
    ph[5] += 1;
#endif
  }

  // end of a sweep (t == 0 again: positions are columns): fold the scales into W, log them
  // for the V replay, and decide convergence
  template <int PH>
  BF_DEV bool sweep_end(RRTile<C>& tile) {
    __syncwarp();  // this step's scale updates visible to the whole warp
    if (slog != nullptr) {
      if (warp == 0)
        for (int c = lane; c < NP; c += 32) slog[c] = fs[c];
      slog += NP;
    }
    // fold the scales into W (t == 0: positions are columns) and reset them
    tile.template scale_cols<PH>(fs, sg);
    __syncwarp();
    for (int c = lane; c < NP; c += 32) fs[c] = 1.0;
    __syncwarp();
    return sweep_end();
  }

  BF_DEV bool sweep_end() {
    const int r = __reduce_add_sync(FULL, rot);  // identical in every warp
    rots += r;
    ++sweeps;
    if (r == 0) conv = 1;
    return conv || sweeps >= max_sweeps;
  }
};

template <class C>
struct RRReplay {
  static constexpr int S = C::S, SG = C::SG, NPAIR = C::NPAIR;
  const double2* log;  // global cursor: next stage to prefetch
  double2* stage;      // 2 x kRRStage x NPAIR
  int sg, in_stage, cur, sweeps_left;

  BF_DEV void prefetch(int buf) {
    double2* dst = stage + buf * kRRStage * NPAIR;
    for (int e = threadIdx.x; e < kRRStage * NPAIR; e += C::THREADS) cp_async16(dst + e, log + e);
    cp_async_commit();
    log += kRRStage * NPAIR;
  }
  BF_DEV void start() {
    prefetch(0);
    cp_async_wait_all();
    prefetch(1);
    __syncthreads();
    cur = 0;
    in_stage = 0;
  }
  const double* slog;  // per sweep the NP column scales logged by the W phase
  template <int PH>
  BF_DEV void sweep_start(RRTile<C>&, int) {}
  template <int PH>
  BF_DEV bool sweep_end(RRTile<C>& tile) {
    tile.template scale_cols<PH>(slog, sg);
    slog += C::NP;
    return sweep_end();
  }
  template <int PH>
  BF_DEV void step(RRTile<C>& tile, int) {
    if (in_stage == kRRStage) {
      cp_async_wait_all();
      __syncthreads();
      prefetch(cur);
      cur ^= 1;
      in_stage = 0;
    }
    const double2* e = stage + (cur * kRRStage + in_stage) * NPAIR + sg * S;
    double c[S], s[S];
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const double2 x = e[j];
      c[j] = x.x;
      s[j] = x.y;
    }
    ++in_stage;
    tile.template apply<PH>(c, s);
    tile.template move<PH>(sg);
  }
  BF_DEV bool sweep_end() { return --sweeps_left <= 0; }
};

// Drives sweeps of NP-1 steps through the S-periodic register phases; returns the final phase.
template <class C, class Act>
struct RRDriver {
  static constexpr int S = C::S, NP = C::NP;
  template <int PH>
  static BF_DEV bool at(RRTile<C>& tile, Act& act, int& t) {
    act.template step<PH>(tile, t);
    if (++t == NP - 1) {
      t = 0;
      if (act.template sweep_end<(PH + 1) % S>(tile)) return true;
      act.template sweep_start<(PH + 1) % S>(tile, 0);
    }
    return false;
  }
  static BF_DEV int run(RRTile<C>& tile, Act& act) {
    int t = 0;
    act.template sweep_start<0>(tile, 0);
    for (;;) {
      if (at<0>(tile, act, t)) return 1 % S;
      if (at<1 % S>(tile, act, t)) return 2 % S;
      if (at<2 % S>(tile, act, t)) return 3 % S;
      if (at<3 % S>(tile, act, t)) return 4 % S;
      if constexpr (S > 4)
        if (at<4 % S>(tile, act, t)) return 5 % S;
      if constexpr (S > 5)
        if (at<5 % S>(tile, act, t)) return 6 % S;
    }
  }
};

template <typename T>
struct RRArgs {
  int64_t batch;
  int m, n, nw;
  const T* a;
  int64_t a_stride;
  bool ta;
  T* u;
  int64_t u_stride;
  T* s;
  int64_t s_stride;
  T* v;
  int64_t v_stride;
  int32_t* sweeps;
  uint8_t* conv;
  int64_t* rots;
  bool accum;  // += into sweeps / rots (block inner SVDs)
  double tol;
  int max_sweeps;
  double2* log;
  int64_t log_stride;
  double* slog;  // per CTA slot (or per matrix when split_v): max_sweeps x NP column scales
  int64_t slog_stride;
  const uint8_t* active;
  int split_v;      // V replayed by svd_rr_vkernel: logs per matrix, vmeta written
  int* queue;       // [0] W-kernel, [1] V-kernel work counters (zeroed before the launch) or null
  int32_t* vmeta;   // split_v: per matrix [replay sweeps, order[0..n)], stride nw + 1
};

// work region (extraction arrays; the sweep buffers and the V log stage alias its start)
template <class C>
__host__ __device__ static size_t rr_region_doubles(int m, int nw) {
  size_t r = (size_t)m * nw > (size_t)nw * nw ? (size_t)m * nw : (size_t)nw * nw;
  if ((size_t)RRShared<C>::SWEEP > r) r = RRShared<C>::SWEEP;
  if ((size_t)RRShared<C>::STAGE > r) r = RRShared<C>::STAGE;
  return r;
}

template <class C>
static size_t rr_smem_bytes(int m, int nw) {
  const size_t d = 8 + rr_region_doubles<C>(m, nw) + 2 * (size_t)m + nw + ((size_t)nw * 4 + 7) / 8;
  return (d * 8 + 15) & ~(size_t)15;
}

#ifndef BF_RR_MINB
#define BF_RR_MINB 1
#endif
// Dynamic matrix queue: a CTA's first matrix is blockIdx.x, later ones are claimed from a global
// counter, so CTAs that drew fast-converging matrices take more of them (sweep counts vary 7-11
// per matrix; a static b += gridDim.x split left the last wave ragged). Block-uniform result.
BF_DEV int64_t rr_claim(int* ctr, int64_t cur) {
  __shared__ long long next;
  __syncthreads();
  if (threadIdx.x == 0) next = ctr ? (long long)gridDim.x + atomicAdd(ctr, 1) : cur + gridDim.x;
  __syncthreads();
  return next;
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, BF_RR_MINB) svd_rr_kernel(RRArgs<double> a) {
  extern __shared__ __align__(16) double sm[];
  int* ctr = reinterpret_cast<int*>(sm);  // 16 ints: extraction counters
  double* Wsm = sm + 8;
  const int m = a.m, n = a.n, nw = a.nw;
  double* cand = Wsm + rr_region_doubles<C>(m, nw);
  double* sig = cand + 2 * m;
  int* order = reinterpret_cast<int*>(sig + nw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sg = lane % C::SG, rgl = lane / C::SG;
  const int row0 = (warp * C::RGW + rgl) * C::R;
  const bool accv = a.v != nullptr;

#ifdef BF_RR_PHASE
  long long phs[6] = {0, 0, 0, 0, 0, 0};
#endif
  for (int64_t b = blockIdx.x; b < a.batch; b = rr_claim(a.queue, b)) {
    if (a.active && !a.active[b]) continue;  // uniform across the CTA
    const double* Ab = a.a + b * a.a_stride;
    RRTile<C> tile;
#pragma unroll
    for (int j = 0; j < C::S; ++j) {
      const int ca = sg * C::S + j, cb = C::NP - 1 - (sg * C::S + j);
#pragma unroll
      for (int i = 0; i < C::R; ++i) {
        const int r = row0 + i;
        double xa = 0.0, xb = 0.0;
        if (r < m) {
          if (ca < n) xa = a.ta ? Ab[(size_t)r * n + ca] : Ab[(size_t)ca * m + r];
          if (cb < n) xb = a.ta ? Ab[(size_t)r * n + cb] : Ab[(size_t)cb * m + r];
        }
        tile.A[i][j] = xa;  // phase 0: logical == physical
        tile.B[i][j] = xb;
      }
    }
    RRWork<C> wk;
    wk.lane = lane;
    wk.warp = warp;
    wk.sg = sg;
    wk.rgl = rgl;
    wk.n = n;
    wk.max_sweeps = a.max_sweeps;
    wk.tol2 = a.tol * a.tol;
    wk.part = Wsm;
    wk.d = Wsm + RRShared<C>::PART + warp * C::NP;
    wk.fs = Wsm + RRShared<C>::PART + RRShared<C>::DN + warp * C::NP;
    const int64_t lslot = a.split_v ? b : (int64_t)blockIdx.x;
    wk.log = a.log ? a.log + lslot * a.log_stride : nullptr;
    wk.slog = a.log ? a.slog + lslot * a.slog_stride : nullptr;
    wk.ex = 0;
    wk.sweeps = 0;
    wk.conv = n < 2;
    wk.rot = 0;
    wk.recompute = 0;
    wk.rots = 0;
#ifdef BF_RR_PHASE
    if (b == blockIdx.x)
      for (int i = 0; i < 6; ++i) wk.ph[i] = 0;
    else
      for (int i = 0; i < 6; ++i) wk.ph[i] = phs[i];
#endif
    __syncthreads();  // previous matrix done with the shared region
    for (int c = lane; c < C::NP; c += 32) wk.fs[c] = 1.0;
    __syncwarp();
    int ph = 0;
    if (!wk.conv) ph = RRDriver<C, RRWork<C>>::run(tile, wk);
#ifdef BF_RR_PHASE
    for (int i = 0; i < 6; ++i) phs[i] = wk.ph[i];
#endif

    // ---- W -> shared memory (column-major m x nw), off-orthogonality fallback, extraction
    __syncthreads();
    tile.store_phase(ph, Wsm, m, m, nw, row0, sg);
    __syncthreads();
    int conv = wk.conv;
    if (!conv) {  // jacobi.py:282-283
      double off = off_orthogonality_cta<double>(Wsm, m, m, nw, sig, reinterpret_cast<double*>(ctr + 2));
      conv = off < a.tol;
    }
    extract_svd_cta<double>(Wsm, m, nullptr, nw, m, n, n, 0, a.u + b * a.u_stride, m, a.s + b * a.s_stride, nullptr, n,
                            sig, order, cand, ctr + 6);
    if (tid == 0) {
      if (a.sweeps) a.sweeps[b] = (a.accum ? a.sweeps[b] : 0) + wk.sweeps;
      if (a.conv) a.conv[b] = (uint8_t)conv;
      if (a.rots) a.rots[b] = (a.accum ? a.rots[b] : 0) + wk.rots;
    }
    if (accv && a.split_v) {
      int32_t* vm = a.vmeta + b * (int64_t)(nw + 1);
      if (tid == 0) vm[0] = wk.sweeps - (wk.conv ? 1 : 0);
      for (int r = tid; r < n; r += blockDim.x) vm[1 + r] = order[r];
    } else if (accv) {
      // ---- V: identity, replay the log on the same tiles, write in sorted order
#pragma unroll
      for (int j = 0; j < C::S; ++j) {
        const int ca = sg * C::S + j, cb = C::NP - 1 - (sg * C::S + j);
#pragma unroll
        for (int i = 0; i < C::R; ++i) {
          tile.A[i][j] = (row0 + i == ca) ? 1.0 : 0.0;
          tile.B[i][j] = (row0 + i == cb) ? 1.0 : 0.0;
        }
      }
      int vph = 0;
      __syncthreads();  // extraction done with the work region (stage lives there)
      if (wk.sweeps - (wk.conv ? 1 : 0) > 0) {
        RRReplay<C> rp;
        rp.log = a.log + (int64_t)blockIdx.x * a.log_stride;
        rp.slog = a.slog + (int64_t)blockIdx.x * a.slog_stride;
        rp.stage = reinterpret_cast<double2*>(Wsm);
        rp.sg = sg;
        // a converged run ends with a rotation-free sweep: identity rotations and unit scales,
        // and a full sweep returns every column to its position -- the replay can drop it
        rp.sweeps_left = wk.sweeps - (wk.conv ? 1 : 0);
        rp.start();
        vph = RRDriver<C, RRReplay<C>>::run(tile, rp);
        cp_async_wait_all();
      }
      __syncthreads();
      tile.store_phase(vph, Wsm, nw, nw, nw, row0, sg);
      __syncthreads();
      double* Vo = a.v + b * a.v_stride;
      for (int e = tid; e < n * n; e += blockDim.x) {
        const int r = e / n, i = e % n;
        Vo[(size_t)r * n + i] = Wsm[(size_t)order[r] * nw + i];
      }
    }
    __syncthreads();
  }
#ifdef BF_RR_PHASE
  if (threadIdx.x == 0 && blockIdx.x < 4)
    printf("rrphase blk %d steps %lld dots %lld xwarp %lld rot %lld apply %lld move %lld\n", blockIdx.x, phs[5], phs[0],
           phs[1], phs[2], phs[3], phs[4]);
#endif
}

// V replay as its own kernel (split_v): it needs no Gram or rotation state, so it runs at the
// occupancy its own registers allow instead of the W phase's (64 x 64: 230 vs 255 registers,
// 7.9 vs 8.3 ms for cfg3; 40 x 40: 4.3 vs 4.9 ms). The logs are then kept per matrix.

template <class C>
__global__ void __launch_bounds__(C::THREADS) svd_rr_vkernel(RRArgs<double> a) {
  extern __shared__ __align__(16) double sm[];
  const int n = a.n, nw = a.nw;
  double2* stage = reinterpret_cast<double2*>(sm);
  double* Vsm = sm + RRShared<C>::STAGE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sg = lane % C::SG, rgl = lane / C::SG;
  const int row0 = (warp * C::RGW + rgl) * C::R;
  for (int64_t b = blockIdx.x; b < a.batch; b = rr_claim(a.queue ? a.queue + 1 : nullptr, b)) {
    if (a.active && !a.active[b]) continue;
    const int32_t* vm = a.vmeta + b * (int64_t)(nw + 1);
    const int vs = vm[0];
    RRTile<C> tile;
#pragma unroll
    for (int j = 0; j < C::S; ++j) {
      const int ca = sg * C::S + j, cb = C::NP - 1 - (sg * C::S + j);
#pragma unroll
      for (int i = 0; i < C::R; ++i) {
        tile.A[i][j] = (row0 + i == ca) ? 1.0 : 0.0;
        tile.B[i][j] = (row0 + i == cb) ? 1.0 : 0.0;
      }
    }
    int vph = 0;
    __syncthreads();  // previous matrix done with the stage / V staging
    if (vs > 0) {
      RRReplay<C> rp;
      rp.log = a.log + b * a.log_stride;
      rp.slog = a.slog + b * a.slog_stride;
      rp.stage = stage;
      rp.sg = sg;
      rp.sweeps_left = vs;
      rp.start();
      vph = RRDriver<C, RRReplay<C>>::run(tile, rp);
      cp_async_wait_all();
    }
    tile.store_phase(vph, Vsm, nw, nw, nw, row0, sg);
    __syncthreads();
    double* Vo = a.v + b * a.v_stride;
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int r = e / n, i = e % n;
      Vo[(size_t)r * n + i] = Vsm[(size_t)vm[1 + r] * nw + i];
    }
  }
}

// V replay with FIXED columns: thread i holds row i of V (all NP columns in registers) and the
// whole sweep's 63 (NP - 1) steps are unrolled, so each slot's column pair
// (rr_col(k, t), rr_col(NP - 1 - k, t)) is a compile-time register pair. Nothing moves between
// threads: a step is S coefficient loads (broadcast) and 2 FMAs per slot per thread -- no
// shuffles and no FIFO selects (the tiled replay spent as many FSEL as DFMA on its moves).
// Coefficients stream through shared memory in VST-step stages (VST divides NP - 1, so a stage
// never straddles a sweep and every stage boundary is a compile-time step).
template <int NP>
struct VColCfg {
  static constexpr int NPAIR = NP / 2, L = NP - 1;
  static constexpr int THREADS = ((NP + 31) / 32) * 32;
  static constexpr int pick(int d) { return d < 6 ? (L * NPAIR * 16 <= 20 * 1024 ? L : 1) : (L % d == 0 ? d : pick(d - 1)); }
#ifdef BF_VCOL_VST
  static constexpr int VST = (L % BF_VCOL_VST == 0) ? BF_VCOL_VST : pick(16);  // A/B override
#else
  static constexpr int VST = pick(16);  // steps per coefficient stage
#endif
  static constexpr int STAGES = L / VST;
};

template <int NP>
BF_DEV constexpr int vcol_col(int x, int t) {  // column held by position x at step t (rr_col)
  return x == 0 ? 0 : 1 + ((x - 1 - t) % (NP - 1) + (NP - 1)) % (NP - 1);
}

template <int NP, int T0, int NS>
BF_DEV void vcol_steps(double (&v)[NP], const double2* st) {
  constexpr int NPAIR = NP / 2;
#pragma unroll
  for (int u = 0; u < NS; ++u) {
    const int t = T0 + u;  // compile-time after unrolling
#pragma unroll
    for (int k = 0; k < NPAIR; ++k) {
      const int ca = vcol_col<NP>(k, t), cb = vcol_col<NP>(NP - 1 - k, t);
      const double2 e = st[u * NPAIR + k];  // (al, be) in position order (a = slot k, b = NP-1-k)
      const double x = v[ca], y = v[cb];
      v[ca] = fma(e.x, y, x);
      v[cb] = fma(e.y, x, y);
    }
  }
}

// positions 1..NP-1 advance D places: new[x] = old[1 + (x - 1 - D) mod (NP - 1)] -- the data
// returns to "position order at the current step" so the next block reuses the same code
template <int NP, int D>
BF_DEV void vcol_rotate(double (&v)[NP]) {
  double tmp[NP];
#pragma unroll
  for (int x = 1; x < NP; ++x) tmp[x] = v[x];
#pragma unroll
  for (int x = 1; x < NP; ++x) v[x] = tmp[1 + ((x - 1 - D) % (NP - 1) + (NP - 1)) % (NP - 1)];
}

// One sweep: STAGES blocks of VST steps. Registers hold V's row in POSITION order as of the
// block's first step, so every block runs the same VST-step code (compile-time register pairs
// of steps 0..VST-1) followed by an in-register rotation by VST positions (NP - 1 moves per
// block instead of a 63-step unrolled body that thrashed the instruction cache: ncu
// no_instructions 41-52 %). After a sweep the ring is back at position == column.
template <int NP>
BF_DEV void vcol_sweep(double (&v)[NP], double2* stage, const double2*& log, int& cur) {
  using C = VColCfg<NP>;
#pragma unroll 1
  for (int g = 0; g < C::STAGES; ++g) {
    // stage cur holds this block's coefficients; prefetch the next block into cur ^ 1
    cp_async_wait_all();
    __syncthreads();
    {
      double2* dst = stage + (cur ^ 1) * C::VST * C::NPAIR;
      for (int e = threadIdx.x; e < C::VST * C::NPAIR; e += C::THREADS) cp_async16(dst + e, log + e);
      cp_async_commit();
      log += C::VST * C::NPAIR;
    }
    vcol_steps<NP, 0, C::VST>(v, stage + cur * C::VST * C::NPAIR);
    vcol_rotate<NP, C::VST>(v);
    cur ^= 1;
  }
}

// which widths replay V with fixed columns (measured, B200): 64 x 64 (cfg3) 7.83 -> 7.35 ms per
// step; 40 x 40 (rsvd's inner SVD) is faster on the tiled replay (two thirds of its 64 threads
// would hold no row)
#ifndef BF_RR_VTILE
template <int NP>
constexpr bool kVCol = NP == 64;
#else
template <int NP>
constexpr bool kVCol = false;
#endif

template <int NP>
__global__ void __launch_bounds__(VColCfg<NP>::THREADS) svd_rr_vcol_kernel(RRArgs<double> a) {
  using C = VColCfg<NP>;
  extern __shared__ __align__(16) double smv[];
  double2* stage = reinterpret_cast<double2*>(smv);      // 2 x VST x NPAIR
  double* Vsm = smv + 2 * C::VST * C::NPAIR * 2;          // NP x NP (column-major) for the sorted write
  const int n = a.n, nw = a.nw, row = threadIdx.x;
  for (int64_t b = blockIdx.x; b < a.batch; b = rr_claim(a.queue ? a.queue + 1 : nullptr, b)) {
    if (a.active && !a.active[b]) continue;
    const int32_t* vm = a.vmeta + b * (int64_t)(nw + 1);
    const int vs = vm[0];
    double v[NP];
#pragma unroll
    for (int c = 0; c < NP; ++c) v[c] = (c == row) ? 1.0 : 0.0;
    const double2* log = a.log + b * a.log_stride;
    const double* slog = a.slog + b * a.slog_stride;
    __syncthreads();  // previous matrix done with the stage / Vsm
    if (vs > 0) {
      // stage 0 of sweep 0
      for (int e = threadIdx.x; e < C::VST * C::NPAIR; e += C::THREADS) cp_async16(stage + e, log + e);
      cp_async_commit();
      log += C::VST * C::NPAIR;
      int cur = 0;
      for (int sw = 0; sw < vs; ++sw) {
        vcol_sweep<NP>(v, stage, log, cur);
        // sweep end: the W phase folded its column scales into W; apply them to V's columns
#pragma unroll
        for (int c = 0; c < NP; ++c) v[c] *= slog[c];
        slog += NP;
      }
      cp_async_wait_all();
    }
    if (row < nw) {
#pragma unroll
      for (int c = 0; c < NP; ++c) Vsm[(size_t)c * nw + row] = v[c];
    }
    __syncthreads();
    double* Vo = a.v + b * a.v_stride;
    for (int e = threadIdx.x; e < n * n; e += C::THREADS) {
      const int r = e / n, i = e % n;
      Vo[(size_t)r * n + i] = Vsm[(size_t)vm[1 + r] * nw + i];
    }
  }
}

// ------------------------------------------------------------------------------ dispatch

template <class C>
static int launch_rr(const SvdLaunch& L, int nw, void* ws, size_t ws_bytes, cudaStream_t st, size_t* need) {
  const size_t smem = rr_smem_bytes<C>(L.m, nw);
  if (smem > 227 * 1024) return -1;
  cudaError_t e = smem_optin((const void*)svd_rr_kernel<C>, (size_t)(smem));
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, svd_rr_kernel<C>, C::THREADS, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)per_sm * sms;
  // the replay prefetches up to two stages past the last logged step
  const int64_t log_stride = ((int64_t)L.max_sweeps * (C::NP - 1) + 2 * kRRStage + 1) * C::NPAIR;
  const int64_t slog_stride = (int64_t)L.max_sweeps * C::NP;
  const bool split = L.v != nullptr;
  // With V the logs are per matrix (split_v). They are sized for max_sweeps, so the batch runs in
  // chunks that keep the log workspace within kRRLogBudget (whole waves of CTAs per chunk);
  // without V there is no log.
  const size_t per_mat = (size_t)log_stride * sizeof(double2) + (size_t)slog_stride * 8 + (size_t)(nw + 1) * 4;
  int64_t chunk = L.batch;
  if (split) {
    int64_t fit = (int64_t)(kRRLogBudget / per_mat);
    fit = fit < cap ? cap : (fit / cap) * cap;
    chunk = L.batch < fit ? L.batch : fit;
  }
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t log_bytes = split ? al((size_t)chunk * log_stride * sizeof(double2)) +
                                       al((size_t)chunk * slog_stride * 8) + al((size_t)chunk * (nw + 1) * 4)
                                 : 0;
  const size_t need_bytes = log_bytes + 256;  // + the work-queue counters
  if (need) {
    *need = need_bytes;
    return 0;
  }
  if (!ws || ws_bytes < need_bytes) return -2;
  int* queue = (int*)((char*)ws + log_bytes);
  using CV = C;
  const size_t vsmem = ((size_t)RRShared<CV>::STAGE + (size_t)nw * nw) * 8;
  int vgrid_cap = 0;
  if (split) {
    e = smem_optin((const void*)svd_rr_vkernel<CV>, (size_t)(vsmem));
    if (e != cudaSuccess) return (int)e;
    int vper = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&vper, svd_rr_vkernel<CV>, CV::THREADS, vsmem);
    vgrid_cap = (vper < 1 ? 1 : vper) * sms;
  }
  using VC = VColCfg<C::NP>;
  const size_t vcol_smem = ((size_t)2 * VC::VST * VC::NPAIR * 2 + (size_t)C::NP * C::NP) * 8;
  int vcol_cap = 0;
  if constexpr (kVCol<C::NP>) {
    if (split) {
      e = smem_optin((const void*)svd_rr_vcol_kernel<C::NP>, vcol_smem);
      if (e != cudaSuccess) return (int)e;
      int vper = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&vper, svd_rr_vcol_kernel<C::NP>, VC::THREADS, vcol_smem);
      vcol_cap = (vper < 1 ? 1 : vper) * sms;
    }
  }
  for (int64_t c0 = 0; c0 < L.batch; c0 += chunk) {
    const int64_t cb = L.batch - c0 < chunk ? L.batch - c0 : chunk;
    RRArgs<double> a;
    a.batch = cb;
    a.m = L.m;
    a.n = L.n;
    a.nw = nw;
    a.a = (const double*)L.a + c0 * L.a_stride;
    a.a_stride = L.a_stride;
    a.ta = L.transpose_a;
    a.u = (double*)L.u + c0 * L.u_stride;
    a.u_stride = L.u_stride;
    a.s = (double*)L.s + c0 * L.s_stride;
    a.s_stride = L.s_stride;
    a.v = L.v ? (double*)L.v + c0 * L.v_stride : nullptr;
    a.v_stride = L.v_stride;
    a.sweeps = L.sweeps ? L.sweeps + c0 : nullptr;
    a.conv = L.converged ? L.converged + c0 : nullptr;
    a.rots = L.rotations ? L.rotations + c0 : nullptr;
    a.accum = L.accumulate;
    a.tol = L.tol;
    a.max_sweeps = L.max_sweeps;
    a.log = split ? (double2*)ws : nullptr;
    a.log_stride = log_stride;
    a.slog = split ? (double*)((char*)ws + al((size_t)chunk * log_stride * sizeof(double2))) : nullptr;
    a.slog_stride = slog_stride;
    a.active = L.active ? L.active + c0 : nullptr;
    a.split_v = split ? 1 : 0;
    a.vmeta = split ? (int32_t*)((char*)a.slog + al((size_t)chunk * slog_stride * 8)) : nullptr;
    a.queue = queue;
    cudaMemsetAsync(queue, 0, 2 * sizeof(int), st);
    const int grid = (int)(cb < cap ? cb : cap);
    svd_rr_kernel<C><<<grid, C::THREADS, smem, st>>>(a);
    if (split) {
      if constexpr (kVCol<C::NP>) {
        const int vgrid = (int)(cb < vcol_cap ? cb : vcol_cap);
        svd_rr_vcol_kernel<C::NP><<<vgrid, VColCfg<C::NP>::THREADS, vcol_smem, st>>>(a);
      } else {
        const int vgrid = (int)(cb < vgrid_cap ? cb : vgrid_cap);
        svd_rr_vkernel<CV><<<vgrid, CV::THREADS, vsmem, st>>>(a);
      }
    }
  }
  return (int)cudaGetLastError();
}

// -1: shape not covered by an instantiation
static int rr_dispatch(const SvdLaunch& L, void* ws, size_t wsb, cudaStream_t st, size_t* need) {
  const int nw = (L.n & 1) ? L.n + 1 : L.n;
  const int rows = L.m > nw ? L.m : nw;
  switch (nw) {
    case 16:
      if (rows <= 16) return launch_rr<RRCfg<16, 4, 1, 1>>(L, nw, ws, wsb, st, need);
      if (rows <= 32) return launch_rr<RRCfg<16, 4, 2, 1>>(L, nw, ws, wsb, st, need);
      if (rows <= 64) return launch_rr<RRCfg<16, 4, 4, 1>>(L, nw, ws, wsb, st, need);
      return -1;
    case 32:
      if (rows <= 32) return launch_rr<RRCfg<32, 4, 4, 1>>(L, nw, ws, wsb, st, need);
      if (rows <= 64) return launch_rr<RRCfg<32, 4, 4, 2>>(L, nw, ws, wsb, st, need);
      return -1;
    case 40:
      if (rows <= 40) return launch_rr<RRCfg<40, 5, 5, 1>>(L, nw, ws, wsb, st, need);
      if (rows <= 64) return launch_rr<RRCfg<40, 5, 4, 2>>(L, nw, ws, wsb, st, need);
      return -1;
    case 48:
      if (rows <= 48) return launch_rr<RRCfg<48, 6, 3, 2>>(L, nw, ws, wsb, st, need);
      if (rows <= 64) return launch_rr<RRCfg<48, 6, 4, 2>>(L, nw, ws, wsb, st, need);
      return -1;
    case 64:
      if (rows <= 64) return launch_rr<RRCfg<64, 4, BF_RR64_R, 64 / (4 * BF_RR64_R)>>(L, nw, ws, wsb, st, need);
      return -1;
    default:
      return -1;
  }
}

size_t svd_rr_ws_bytes(int dtype, const SvdLaunch& L) {
  if (dtype != 0 || L.ordering != 1 || L.tier == 2 || L.n < 2) return 0;
  size_t need = 0;
  return rr_dispatch(L, nullptr, 0, nullptr, &need) == 0 ? need : 0;
}

bool svd_rr_covers(const SvdLaunch& L) {
  if (L.ordering != 1 || L.tier == 2 || L.n < 2) return false;
  size_t need = 0;
  return rr_dispatch(L, nullptr, 0, nullptr, &need) == 0;
}

int launch_svd_rr(int dtype, const SvdLaunch& L, void* ws, size_t wsb, cudaStream_t st, bool* handled) {
  *handled = false;
  if (dtype != 0 || L.ordering != 1 || L.tier == 2 || L.n < 2) return 0;
  const int rc = rr_dispatch(L, ws, wsb, st, nullptr);
  if (rc == -1 || rc == -2) return 0;
  *handled = true;
  return rc;
}

}  // namespace bf
