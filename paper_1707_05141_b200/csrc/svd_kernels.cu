// Batched one-sided Jacobi SVD: shared-memory tier (one CTA per matrix).
//
// Reference: svd() jacobi.py:231-284, batch_svd jacobi.py:287-290.
// W and V are staged in shared memory when they fit (the paper's shared-memory
// kernel); larger matrices keep them in an L2-resident global
// workspace with the same code. The register tier (n <= 32) lives in svd_reg.cu.
#include "internal.h"
#include "jacobi_cta.cuh"

namespace bf {

template <typename T>
struct SvdArgs {
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
  int max_sweeps, ordering;
  bool in_smem;
  bool w_in_smem;  // !in_smem: W (+ candidates) still in shared memory, only V in global
  T* gws;  // per-matrix global workspace when !in_smem
  int64_t gws_stride;
  const uint8_t* active;
};

template <typename T>
__host__ __device__ static size_t svd_work_elems(int m, int nw, bool accv) {
  return (size_t)m * nw + (accv ? (size_t)nw * nw : 0) + 2 * (size_t)m;
}

template <typename T>
static size_t svd_smem_bytes(int m, int nw, bool accv, bool in_smem) {
  size_t b = 0;
  if (in_smem) b += svd_work_elems<T>(m, nw, accv) * sizeof(T);
  b += (size_t)nw * sizeof(T) + (size_t)nw * sizeof(int) + 4 * sizeof(int) + sizeof(double) + 16;
  return (b + 15) & ~(size_t)15;
}

#ifndef BF_CTA_MAXW
#define BF_CTA_MAXW 32  // warps per CTA (one matrix); 32 vs 16: 121x121 6.1 -> 5.4 ms
#endif
#ifndef BF_CTA_PB
#define BF_CTA_PB 2  // column pairs per warp per pass (2: 4-5 % faster than 4 and 3, measured)
#endif

// MODE 0: W, V, candidates in shared memory; 1: W + candidates in shared memory, V in global;
// 2: everything in the global workspace. Separate instantiations so the shared-memory operands
// are addressed as such (LDS/STS, not generic loads).
template <typename T, int MODE>
BF_DEV void svd_cta_body(const SvdArgs<T>& a, unsigned char* smem_raw, int64_t b) {
  const int m = a.m, n = a.n, nw = a.nw;
  const bool accv = a.v != nullptr;
  T* W;
  T* V;
  T* cand;
  size_t smem_elems;
  if (MODE == 0) {
    W = reinterpret_cast<T*>(smem_raw);
    V = accv ? W + (size_t)m * nw : nullptr;
    cand = W + (size_t)m * nw + (accv ? (size_t)nw * nw : 0);
    smem_elems = svd_work_elems<T>(m, nw, accv);
  } else if (MODE == 1) {
    W = reinterpret_cast<T*>(smem_raw);
    cand = W + (size_t)m * nw;
    V = accv ? a.gws + b * a.gws_stride : nullptr;
    smem_elems = svd_work_elems<T>(m, nw, false);
  } else {
    W = a.gws + b * a.gws_stride;
    V = accv ? W + (size_t)m * nw : nullptr;
    cand = W + (size_t)m * nw + (accv ? (size_t)nw * nw : 0);
    smem_elems = 0;
  }
  unsigned char* tail = smem_raw + smem_elems * sizeof(T);
  T* sig = reinterpret_cast<T*>(tail);
  int* order = reinterpret_cast<int*>(sig + nw);
  int* counters = order + nw;  // 4 ints
  double* red = reinterpret_cast<double*>(((uintptr_t)(counters + 4) + 7) & ~(uintptr_t)7);

  const T* A = a.a + b * a.a_stride;
  const int tid = threadIdx.x;
  if (!a.ta) {
    for (int64_t e = tid; e < (int64_t)m * nw; e += blockDim.x) W[e] = e < (int64_t)m * n ? A[e] : T(0);
  } else {  // A stored n x m column-major; W = A^T
    for (int64_t e = tid; e < (int64_t)m * nw; e += blockDim.x) {
      int j = (int)(e / m), i = (int)(e % m);
      W[e] = j < n ? A[(size_t)i * n + j] : T(0);
    }
  }
  if (accv)
    for (int64_t e = tid; e < (int64_t)nw * nw; e += blockDim.x) V[e] = (e / nw == e % nw) ? T(1) : T(0);
  __syncthreads();
  SweepStats st = jacobi_sweeps<T, BF_CTA_PB>(W, m, V, nw, m, n, nw, a.ordering, a.tol, a.max_sweeps, counters);
  if (!st.converged) {
    double off = off_orthogonality_cta<T>(W, m, m, nw, sig, red);
    st.converged = off < a.tol;
  }
  extract_svd_cta<T>(W, m, V, nw, m, n, n, n, a.u + b * a.u_stride, m, a.s + b * a.s_stride,
                     accv ? a.v + b * a.v_stride : nullptr, n, sig, order, cand, counters + 2);
  if (tid == 0) {
    if (a.sweeps) a.sweeps[b] = (a.accum ? a.sweeps[b] : 0) + st.sweeps;
    if (a.conv) a.conv[b] = (uint8_t)st.converged;
    if (a.rots) a.rots[b] = (a.accum ? a.rots[b] : 0) + st.rotations;
  }
}

static int working_cols(int n, int ordering) { return (ordering == 1 && (n & 1)) ? n + 1 : n; }

template <typename T>
__global__ void __launch_bounds__(BF_CTA_MAXW * 32) svd_cta_kernel(SvdArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t b = blockIdx.x;
  if (b >= a.batch) return;
  if (a.active && !a.active[b]) return;
  if (a.in_smem)
    svd_cta_body<T, 0>(a, smem_raw, b);
  else if (a.w_in_smem)
    svd_cta_body<T, 1>(a, smem_raw, b);
  else
    svd_cta_body<T, 2>(a, smem_raw, b);
}

static bool fits_smem(size_t bytes) { return bytes <= 227 * 1024; }

size_t svd_reg_ws_bytes(int dtype, const SvdLaunch& L);
size_t svd_rr_ws_bytes(int dtype, const SvdLaunch& L);

static size_t svd_shared_ws_bytes(int dtype, int64_t batch, int m, int n, int ordering, bool accv) {
  int nw = working_cols(n, ordering);
  size_t es = dtype == 0 ? 8 : 4;
  size_t smem = dtype == 0 ? svd_smem_bytes<double>(m, nw, accv, true) : svd_smem_bytes<float>(m, nw, accv, true);
  if (fits_smem(smem)) return 0;
  size_t per = (dtype == 0 ? svd_work_elems<double>(m, nw, accv) : svd_work_elems<float>(m, nw, accv)) * es;
  per = (per + 255) & ~(size_t)255;
  return per * (size_t)batch;
}

size_t svd_global_ws_bytes(int dtype, int64_t batch, int m, int n, int ordering, bool accv, int tier, int max_sweeps) {
  SvdLaunch L{};
  L.batch = batch;
  L.m = m;
  L.n = n;
  L.ordering = ordering;
  L.tier = tier;
  L.max_sweeps = max_sweeps;
  L.v = accv ? (void*)1 : nullptr;
  size_t r = svd_reg_ws_bytes(dtype, L);
  const size_t rr = svd_rr_ws_bytes(dtype, L);
  r = rr > r ? rr : r;
  size_t s = svd_shared_ws_bytes(dtype, batch, m, n, ordering, accv);
  return r > s ? r : s;
}

int launch_svd_reg(int dtype, const SvdLaunch& L, void* ws, size_t wsb, cudaStream_t st, bool* handled);
int launch_svd_rr(int dtype, const SvdLaunch& L, void* ws, size_t wsb, cudaStream_t st, bool* handled);

template <typename T>
static int launch_svd_t(const SvdLaunch& L, void* ws, cudaStream_t st) {
  SvdArgs<T> a;
  a.batch = L.batch;
  a.m = L.m;
  a.n = L.n;
  a.nw = working_cols(L.n, L.ordering);
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
  a.ordering = L.ordering;
  a.active = L.active;
  const bool accv = L.v != nullptr;
  size_t smem = svd_smem_bytes<T>(L.m, a.nw, accv, true);
  a.in_smem = fits_smem(smem);
  a.gws = (T*)ws;
  size_t per = svd_work_elems<T>(L.m, a.nw, accv) * sizeof(T);
  a.gws_stride = (int64_t)(((per + 255) & ~(size_t)255) / sizeof(T));
  a.w_in_smem = false;
  if (!a.in_smem) {
    const size_t wsm = svd_smem_bytes<T>(L.m, a.nw, false, true);  // W + candidates + tail
    a.w_in_smem = accv && fits_smem(wsm);
    smem = a.w_in_smem ? wsm : svd_smem_bytes<T>(L.m, a.nw, accv, false);
  }
  int pairs = a.nw / 2 > 0 ? a.nw / 2 : 1;
  int nwarps = (pairs + BF_CTA_PB - 1) / BF_CTA_PB;
  nwarps = nwarps < 2 ? 2 : (nwarps > BF_CTA_MAXW ? BF_CTA_MAXW : nwarps);
  cudaError_t e = smem_optin((const void*)svd_cta_kernel<T>, (size_t)(smem));
  if (e != cudaSuccess) return (int)e;
  svd_cta_kernel<T><<<(unsigned)L.batch, nwarps * 32, smem, st>>>(a);
  return (int)cudaGetLastError();
}

int launch_svd(int dtype, const SvdLaunch& L, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (L.batch == 0) return 0;
  if (L.tier != 2) {
    bool handled = false;
    int rc = launch_svd_rr(dtype, L, ws, ws_bytes, st, &handled);  // tiled round-robin register tier
    if (handled || rc) return rc;
    rc = launch_svd_reg(dtype, L, ws, ws_bytes, st, &handled);
    if (handled || rc) return rc;
  }
  return dtype == 0 ? launch_svd_t<double>(L, ws, st) : launch_svd_t<float>(L, ws, st);
}

}  // namespace bf
