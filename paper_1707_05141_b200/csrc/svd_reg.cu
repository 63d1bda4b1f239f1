// Register tier of the batched one-sided Jacobi SVD (csrc/jacobi_reg.cuh).
//
// Persistent CTAs of WW row-warps; per matrix:
//   1. W rows -> registers, sweeps until a rotation-free sweep (jacobi.py:270-281), every
//      step's (c, s) appended to this CTA's rotation log (global, L2-resident);
//   2. W -> shared memory; off_orthogonality fallback (jacobi.py:282-283); _extract_svd
//      (sigma, stable descending order, U, zero-column completion; jacobi.py:189-228);
//   3. V rows (lane = V row) start at I and replay the log with the same slot/move sequence,
//      then are written in the sorted order (jacobi.py:226-227).
#include "internal.h"
#include "jacobi_cta.cuh"
#include "jacobi_reg.cuh"

namespace bf {

template <typename T>
struct RegArgs {
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
  double2* log;  // gridDim.x slots of log_stride entries (null without V)
  int64_t log_stride;
  const uint8_t* active;  // optional: entries with active[b] == 0 are skipped
};

constexpr int kStage = 8;

template <class C>
__host__ __device__ constexpr size_t reg_fixed_smem_doubles() {
  // cs[32][2] + d[64] + stage[2][kStage][32][2] + ctr[16 ints]
  return 64 + 64 + 2 * kStage * 64 + 8;
}

// The work region holds the extraction arrays after the sweeps and the slot-product buffer
// (2 * pairs x rs doubles) during them.
template <class C>
static size_t reg_work_bytes(int m, int nw, int es) {
  size_t work = (size_t)m * nw > (size_t)nw * nw ? (size_t)m * nw : (size_t)nw * nw;
  size_t ext = (work + 2 * (size_t)m + nw) * es + (size_t)nw * 4;
  size_t prod = (size_t)2 * C::pairs * C::rs * 8;
  return ext > prod ? ext : prod;
}

template <class C>
static size_t reg_smem_bytes(int m, int nw, int es) {
  size_t b = reg_fixed_smem_doubles<C>() * 8 + reg_work_bytes<C>(m, nw, es) + 64;
  return (b + 15) & ~(size_t)15;
}

static int reg_steps_per_sweep(int np, int n, int ord) { return ord == 1 ? np - 1 : 2 * (n - 1); }

template <typename T, class C, int ORD>
#ifndef BF_REG_MINB
#define BF_REG_MINB 1
#endif
__global__ void __launch_bounds__(C::threads, BF_REG_MINB) svd_reg_kernel(RegArgs<T> a) {
  constexpr int NP = C::np, WW = C::ww;
  extern __shared__ __align__(16) double smem_d[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* cs_sh = smem_d;
  double* d_sh = cs_sh + 64;
  double2* stage = reinterpret_cast<double2*>(d_sh + 64);
  int* ctr = reinterpret_cast<int*>(stage + 2 * kStage * 32);  // [0..8) extraction, [8..10) sweep counters
  T* Wsm = reinterpret_cast<T*>(smem_d + reg_fixed_smem_doubles<C>());
  const int m = a.m, n = a.n, nw = a.nw;
  const bool accv = a.v != nullptr;
  const size_t work = (size_t)m * nw > (size_t)nw * nw ? (size_t)m * nw : (size_t)nw * nw;
  T* cand = Wsm + work;
  T* sig = cand + 2 * m;
  int* order = reinterpret_cast<int*>(sig + nw);
  const int off0 = ORD == 0 ? NP / 2 - 1 : 0;
  const int row = warp * 32 + lane;

  for (int64_t b = blockIdx.x; b < a.batch; b += gridDim.x) {
    if (a.active && !a.active[b]) continue;  // uniform across the CTA
    const T* A = a.a + b * a.a_stride;
    T w[NP];
#pragma unroll
    for (int x = 0; x < NP; ++x) {
      const int col = ORD == 0 ? ((x - off0) % NP + NP) % NP : x;
      T val = T(0);
      if (row < m && col < n) val = a.ta ? A[(size_t)row * n + col] : A[(size_t)col * m + row];
      w[x] = val;
    }
    if (tid == 0) ctr[8] = ctr[9] = 0;
    __syncthreads();
    WAction<T, C, ORD> act;
    act.tid = tid;
    act.n = n;
    act.max_sweeps = a.max_sweeps;
    act.tol2 = a.tol * a.tol;
    act.cs = cs_sh;
    act.d = d_sh;
    act.P = reinterpret_cast<double*>(Wsm);
    act.swrot = ctr + 8;
    act.log = a.log ? a.log + (int64_t)blockIdx.x * a.log_stride : nullptr;
    act.sweeps = 0;
    act.conv = n < 2;
    act.rot = 0;
    act.recompute = 0;
    static_assert(sizeof(T) == 8, "register tier is fp64");
    act.rots = 0;
    if (!act.conv) RegDriver<T, C, ORD>::run(w, n, act);

    // ---- W -> shared memory (column-major m x nw)
    __syncthreads();
    if (row < m) {
#pragma unroll
      for (int x = 0; x < NP; ++x) {
        const int col = ORD == 0 ? ((x - off0) % NP + NP) % NP : x;
        if (col < nw) Wsm[(size_t)col * m + row] = w[x];
      }
    }
    __syncthreads();
    int conv = act.conv;
    if (!conv) {  // jacobi.py:282-283
      double off = off_orthogonality_cta<T>(Wsm, m, m, nw, sig, reinterpret_cast<double*>(ctr + 2));
      conv = off < a.tol;
    }
    extract_svd_cta<T>(Wsm, m, nullptr, nw, m, n, n, 0, a.u + b * a.u_stride, m, a.s + b * a.s_stride, nullptr, n,
                       sig, order, cand, ctr + 6);
    if (tid == 0) {
      if (a.sweeps) a.sweeps[b] = (a.accum ? a.sweeps[b] : 0) + act.sweeps;
      if (a.conv) a.conv[b] = (uint8_t)conv;
      if (a.rots) a.rots[b] = (a.accum ? a.rots[b] : 0) + act.rots;
    }
    if (accv) {
      // ---- V: identity, replay the log, write in sorted order
      T v[NP];
#pragma unroll
      for (int x = 0; x < NP; ++x) {
        const int col = ORD == 0 ? ((x - off0) % NP + NP) % NP : x;
        v[x] = col == row ? T(1) : T(0);
      }
      // a converged run ends with a rotation-free sweep (identity rotations; a full sweep
      // realigns every column): the replay drops it
      const int vsweeps = act.sweeps - (act.conv ? 1 : 0);
      if (vsweeps > 0) {
        VAction<T, C, ORD, kStage> va;
        va.log = a.log + (int64_t)blockIdx.x * a.log_stride;
        va.stage = stage;
        va.sweeps_left = vsweeps;
        va.start();
        RegDriver<T, C, ORD>::run(v, n, va);
        cp_async_wait_all();  // the last prefetch (past the end of the log) must land before reuse
      }
      __syncthreads();  // everyone done with Wsm (extract) and the stage buffer
      if (row < nw) {
#pragma unroll
        for (int x = 0; x < NP; ++x) {
          const int col = ORD == 0 ? ((x - off0) % NP + NP) % NP : x;
          if (col < nw) Wsm[(size_t)col * nw + row] = v[x];
        }
      }
      __syncthreads();
      T* Vo = a.v + b * a.v_stride;
      for (int e = tid; e < n * n; e += blockDim.x) {
        const int r = e / n, i = e % n;
        Vo[(size_t)r * n + i] = Wsm[(size_t)order[r] * nw + i];
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ dispatch

struct RegPlan {
  int np = 0, ww = 0;
  bool ok = false;
};

static RegPlan reg_plan(const SvdLaunch& L, int dtype) {
  RegPlan p;
  if (dtype != 0 || L.tier == 2 || L.n < 2) return p;
  const int m = L.m, n = L.n;
  int nw;
  if (L.ordering == 1) {
    nw = (n & 1) ? n + 1 : n;
    if (nw != 16 && nw != 32 && nw != 40 && nw != 48 && nw != 64) return p;
    p.np = nw;
  } else {
    nw = n;
    if (n <= 16)
      p.np = 16;
    else if (n <= 32)
      p.np = 32;
    else if (n <= 64)
      p.np = 64;
    else
      return p;
  }
  const int rows = m > nw ? m : nw;
  p.ww = (rows + 31) / 32;
  if (p.ww > 2) return p;                   // instantiated for m <= 64
  if (p.np > 32 && p.ww < 2) p.ww = 2;      // the wide variants are instantiated with two row-warps
  p.ok = true;
  return p;
}

template <typename T, class C, int ORD>
static int launch_reg(const SvdLaunch& L, void* ws, size_t ws_bytes, cudaStream_t st, size_t* need) {
  const int nw = ORD == 1 ? C::np : L.n;
  const size_t smem = reg_smem_bytes<C>(L.m, nw, sizeof(T));
  if (smem > 227 * 1024) return -1;
  cudaError_t e = smem_optin((const void*)svd_reg_kernel<T, C, ORD>, smem);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0, dev = 0, sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, svd_reg_kernel<T, C, ORD>, C::threads, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)per_sm * sms;
  const int grid = (int)(L.batch < cap ? L.batch : cap);
  const int64_t log_stride =
      ((int64_t)L.max_sweeps * reg_steps_per_sweep(C::np, L.n, ORD) + 2 * kStage + 1) * C::pairs;
  const size_t log_bytes = L.v ? (size_t)grid * log_stride * sizeof(double2) : 0;
  if (need) {
    *need = log_bytes;
    return 0;
  }
  if (log_bytes && (!ws || ws_bytes < log_bytes)) return -2;
  RegArgs<T> a;
  a.batch = L.batch;
  a.m = L.m;
  a.n = L.n;
  a.nw = nw;
  a.a = (const T*)L.a;
  a.a_stride = L.a_stride;
  a.ta = L.transpose_a;
  a.u = (T*)L.u;
  a.u_stride = L.u_stride;
  a.s = (T*)L.s;
  a.s_stride = L.s_stride;
  a.v = (T*)L.v;
  a.v_stride = L.v_stride;
  a.sweeps = L.sweeps;
  a.conv = L.converged;
  a.rots = L.rotations;
  a.accum = L.accumulate;
  a.tol = L.tol;
  a.max_sweeps = L.max_sweeps;
  a.log = L.v ? (double2*)ws : nullptr;
  a.log_stride = log_stride;
  a.active = L.active;
  svd_reg_kernel<T, C, ORD><<<grid, C::threads, smem, st>>>(a);
  return (int)cudaGetLastError();
}

template <int ORD>
static int reg_dispatch(const RegPlan& p, const SvdLaunch& L, void* ws, size_t wsb, cudaStream_t st, size_t* need) {
  if (p.ww == 1) {
    if (p.np == 16) return launch_reg<double, RegCfg<16, 1>, ORD>(L, ws, wsb, st, need);
    if (p.np == 32) return launch_reg<double, RegCfg<32, 1>, ORD>(L, ws, wsb, st, need);
  } else {
    if (p.np == 16) return launch_reg<double, RegCfg<16, 2>, ORD>(L, ws, wsb, st, need);
    if (p.np == 32) return launch_reg<double, RegCfg<32, 2>, ORD>(L, ws, wsb, st, need);
    if (ORD == 1 && p.np == 40) return launch_reg<double, RegCfg<40, 2>, ORD>(L, ws, wsb, st, need);
    if (ORD == 1 && p.np == 48) return launch_reg<double, RegCfg<48, 2>, ORD>(L, ws, wsb, st, need);
    if (p.np == 64) return launch_reg<double, RegCfg<64, 2>, ORD>(L, ws, wsb, st, need);
  }
  return -1;
}

// Workspace (rotation log) the register tier needs for this launch, or 0 if it won't handle it.
size_t svd_reg_ws_bytes(int dtype, const SvdLaunch& L) {
  RegPlan p = reg_plan(L, dtype);
  if (!p.ok) return 0;
  size_t need = 0;
  int rc = L.ordering == 1 ? reg_dispatch<1>(p, L, nullptr, 0, nullptr, &need)
                           : reg_dispatch<0>(p, L, nullptr, 0, nullptr, &need);
  return rc == 0 ? need : 0;
}

bool svd_reg_covers(const SvdLaunch& L) {
  RegPlan p = reg_plan(L, 0);
  if (!p.ok) return false;
  size_t need = 0;
  return (L.ordering == 1 ? reg_dispatch<1>(p, L, nullptr, 0, nullptr, &need)
                          : reg_dispatch<0>(p, L, nullptr, 0, nullptr, &need)) == 0;
}

int launch_svd_reg(int dtype, const SvdLaunch& L, void* ws, size_t wsb, cudaStream_t st, bool* handled) {
  *handled = false;
  RegPlan p = reg_plan(L, dtype);
  if (!p.ok) return 0;
  int rc = L.ordering == 1 ? reg_dispatch<1>(p, L, ws, wsb, st, nullptr) : reg_dispatch<0>(p, L, ws, wsb, st, nullptr);
  if (rc == -1 || rc == -2) return 0;  // not instantiated / no workspace: shared tier handles it
  *handled = true;
  return rc;
}

#ifdef BF_PHASE_TIMING
extern "C" __attribute__((visibility("default"))) int bf_debug_phase_clk(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_phase_clk, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_phase_clk, z, sizeof(z));
  }
  return (int)cudaGetLastError();
}
#endif
}  // namespace bf
