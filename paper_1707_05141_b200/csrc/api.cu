// C ABI (include/batchfact_b200.h): validation, workspace planning, dispatch.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/batchfact_b200.h"
#include "internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, int a = 0, int b = 0, int c = 0) {
  char buf[512];
  snprintf(buf, sizeof(buf), fmt, a, b, c);
  g_err = buf;
  return code;
}

int cuda_rc(int rc, const char* where) {
  if (rc == 0) return BF_OK;
  char buf[512];
  snprintf(buf, sizeof(buf), "%s: CUDA error %d (%s)", where, rc, cudaGetErrorString((cudaError_t)rc));
  g_err = buf;
  return rc;
}

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

cudaStream_t S(void* s) { return (cudaStream_t)s; }

int check_ws(void* ws, size_t have, size_t need) {
  if (need == 0) return BF_OK;
  if (!ws || have < need) {
    char buf[256];
    snprintf(buf, sizeof(buf), "workspace too small: need %zu bytes, got %zu", need, ws ? have : (size_t)0);
    g_err = buf;
    return BF_ERR_WORKSPACE;
  }
  return BF_OK;
}

// ---------------------------------------------------------------- QR
template <typename T>
int qr_impl(int64_t batch, int m, int n, const T* a, T* q, T* r, int pw, void* ws, size_t wsb, void* st) {
  if (batch < 0 || m < 0 || n < 0) return fail(BF_ERR_ARG, "negative batch or shape");
  // qr.py:71-74
  if (m < n) return fail(BF_ERR_ARG, "qr requires m >= n, got %d x %d; pass the transpose", m, n);
  if (pw < 1) return fail(BF_ERR_ARG, "panel_width must be >= 1");
  int dt = sizeof(T) == 8 ? 0 : 1;
  int rc = check_ws(ws, wsb, bf::qr_global_ws_bytes(dt, batch, m, n));
  if (rc) return rc;
  return cuda_rc(bf::launch_qr(dt, batch, m, n, a, (int64_t)m * n, q, (int64_t)m * n, r, (int64_t)n * n, ws, S(st)),
                 "qr");
}

// ---------------------------------------------------------------- SVD
double resolve_tol(double t, bool f64, bool block) {
  if (t > 0) return t;
  if (block) return f64 ? bf::Tol<double>::block : bf::Tol<float>::block;
  return f64 ? bf::Tol<double>::svd : bf::Tol<float>::svd;
}

int check_jopts(const bf_jacobi_opts* o) {
  if (!o) return fail(BF_ERR_ARG, "opts is NULL");
  if (o->max_sweeps < 1) return fail(BF_ERR_ARG, "max_sweeps must be >= 1");
  if (o->ordering != 0 && o->ordering != 1) return fail(BF_ERR_ARG, "ordering must be one of ('serial', 'round_robin')");
  if (o->tier < 0 || o->tier > 2) return fail(BF_ERR_ARG, "tier must be 0 (auto), 1 (register) or 2 (shared)");
  if (!(o->tolerance == o->tolerance)) return fail(BF_ERR_ARG, "tolerance must be positive");
  return BF_OK;
}

template <typename T>
int svd_impl(int64_t batch, int m, int n, const T* a, T* u, T* s, T* v, int32_t* sweeps, uint8_t* conv, int64_t* rots,
             const bf_jacobi_opts* o, void* ws, size_t wsb, void* st) {
  int rc = check_jopts(o);
  if (rc) return rc;
  if (batch < 0 || m < 0 || n < 0) return fail(BF_ERR_ARG, "negative batch or shape");
  if (m < n) return fail(BF_ERR_ARG, "svd requires m >= n, got %d x %d; pass the transpose", m, n);
  if (o->accumulate_v && !v && batch > 0 && n > 0) return fail(BF_ERR_ARG, "accumulate_v set but v is NULL");
  const bool f64 = sizeof(T) == 8;
  int dt = f64 ? 0 : 1;
  if (n == 0) {  // jacobi.py:244-249: empty result, converged, 0 sweeps
    if (batch > 0) {
      if (sweeps) cudaMemsetAsync(sweeps, 0, sizeof(int32_t) * batch, S(st));
      if (conv) cudaMemsetAsync(conv, 1, batch, S(st));
      if (rots) cudaMemsetAsync(rots, 0, sizeof(int64_t) * batch, S(st));
    }
    return cuda_rc((int)cudaGetLastError(), "svd");
  }
  rc = check_ws(ws, wsb,
                bf::svd_global_ws_bytes(dt, batch, m, n, o->ordering, o->accumulate_v != 0, o->tier, o->max_sweeps));
  if (rc) return rc;
  bf::SvdLaunch L;
  L.batch = batch;
  L.m = m;
  L.n = n;
  L.a = a;
  L.a_stride = (int64_t)m * n;
  L.u = u;
  L.u_stride = (int64_t)m * n;
  L.s = s;
  L.s_stride = n;
  L.v = o->accumulate_v ? v : nullptr;
  L.v_stride = (int64_t)n * n;
  L.sweeps = sweeps;
  L.converged = conv;
  L.rotations = rots;
  L.tol = resolve_tol(o->tolerance, f64, false);
  L.max_sweeps = o->max_sweeps;
  L.ordering = o->ordering;
  L.tier = o->tier;
  L.transpose_a = false;
  return cuda_rc(bf::launch_svd(dt, L, ws, wsb, S(st)), "svd");
}

// ---------------------------------------------------------------- block SVD
int check_bopts(const bf_block_opts* o) {
  if (!o) return fail(BF_ERR_ARG, "opts is NULL");
  if (o->block_width < 1) return fail(BF_ERR_ARG, "block_width must be >= 1");
  if (o->method != 0 && o->method != 1) return fail(BF_ERR_ARG, "method must be one of ('gram', 'direct')");
  if (o->max_sweeps < 1) return fail(BF_ERR_ARG, "max_sweeps must be >= 1");
  return BF_OK;
}

template <typename T>
int block_impl(int64_t batch, int m, int n, const T* a, T* u, T* s, T* v, int32_t* sweeps, uint8_t* conv, T* eh,
               const bf_block_opts* o, void* ws, size_t wsb, void* st, int64_t* stats = nullptr) {
  int rc = check_bopts(o);
  if (rc) return rc;
  if (batch < 0 || m < 0 || n < 0) return fail(BF_ERR_ARG, "negative batch or shape");
  if (m < n) return fail(BF_ERR_ARG, "block_svd requires m >= n, got %d x %d", m, n);
  if (o->accumulate_v && !v && batch > 0 && n > 0) return fail(BF_ERR_ARG, "accumulate_v set but v is NULL");
  if (batch == 0) return BF_OK;  // an empty batch maps to an empty result (core.py:97-123)
  if (!sweeps || !conv) return fail(BF_ERR_ARG, "sweeps and converged are required for block_svd");
  int k = o->block_width;
  if (o->method == 1) k = std::max(1, std::min(k, m / 2));
  if (m == 0) return fail(BF_ERR_UNSUPPORTED, "block_svd of an empty matrix is unsupported");
  const bool f64 = sizeof(T) == 8;
  int dt = f64 ? 0 : 1;
  rc = check_ws(ws, wsb, bf::block_ws_bytes(dt, batch, m, n, o->block_width, o->method, o->accumulate_v != 0));
  if (rc) return rc;
  bf::BlockLaunch L;
  L.batch = batch;
  L.m = m;
  L.n = n;
  L.a = a;
  L.u = u;
  L.s = s;
  L.v = o->accumulate_v ? v : nullptr;
  L.sweeps = sweeps;
  L.converged = conv;
  L.e_history = eh;
  L.block_width = o->block_width;
  L.method = o->method;
  L.max_sweeps = o->max_sweeps;
  L.tol = resolve_tol(o->tolerance, f64, true);
  L.stats = stats;
  return cuda_rc(bf::launch_block_svd(dt, L, ws, S(st)), "block_svd");
}

// ---------------------------------------------------------------- rsvd
struct RsvdLayout {
  size_t omega, y, q, r, bt, qb, rb, ur, vr, svdws, total;
};

RsvdLayout rsvd_layout(int64_t batch, int m, int n, int w, int es, bool need_omega) {
  RsvdLayout L;
  size_t off = 0;
  auto take = [&](size_t elems) {
    size_t o = off;
    off += al(elems * es);
    return o;
  };
  L.omega = need_omega ? take((size_t)batch * n * w) : 0;
  L.y = take((size_t)batch * m * w);
  L.q = take((size_t)batch * m * w);
  L.r = take((size_t)batch * w * w);
  L.bt = take((size_t)batch * n * w);
  L.qb = take((size_t)batch * n * w);
  L.rb = take((size_t)batch * w * w);
  L.ur = take((size_t)batch * w * w);
  L.vr = take((size_t)batch * w * w);
  size_t qws = std::max(bf::qr_global_ws_bytes(es == 8 ? 0 : 1, batch, m, w),
                        bf::qr_global_ws_bytes(es == 8 ? 0 : 1, batch, n, w));
  size_t sws = bf::svd_global_ws_bytes(es == 8 ? 0 : 1, batch, w, w, 1, true, 0, 30);
  L.svdws = off;
  off += al(std::max(qws, sws));
  L.total = off;
  return L;
}

// omega_rowmajor: a caller-supplied omega stored like a device-drawn one (C order n x w, used by
// the float32-on-float64 path); svd_tol: the inner SVD tolerance (0: the default of T)
template <typename T>
int rsvd_impl(int64_t batch, int m, int n, int k, int p, uint64_t slo, uint64_t shi, int64_t ibase, const T* a,
              const T* omega, T* u, T* s, T* v, void* ws, size_t wsb, void* st, bool omega_rowmajor = false,
              double svd_tol = 0.0) {
  if (batch < 0 || m < 0 || n < 0) return fail(BF_ERR_ARG, "negative batch or shape");
  if (k < 1) return fail(BF_ERR_ARG, "k must be >= 1");
  if (p < 0) return fail(BF_ERR_ARG, "p must be >= 0");
  const int w = k + p;
  if (w > std::min(m, n))  // rsvd.py:60-64
    return fail(BF_ERR_ARG, "k + p = %d exceeds min(m, n) = %d for shape (%d, ...)", w, std::min(m, n), m);
  const bool f64 = sizeof(T) == 8;
  const int es = sizeof(T), dt = f64 ? 0 : 1;
  RsvdLayout Ly = rsvd_layout(batch, m, n, w, es, omega == nullptr);
  int rc = check_ws(ws, wsb, Ly.total);
  if (rc) return rc;
  if (batch == 0) return BF_OK;
  char* base = (char*)ws;
  cudaStream_t cs = S(st);
  T* om = omega ? (T*)omega : (T*)(base + Ly.omega);
  T* Y = (T*)(base + Ly.y);
  T* Q = (T*)(base + Ly.q);
  T* R = (T*)(base + Ly.r);
  T* Bt = (T*)(base + Ly.bt);
  T* Qb = (T*)(base + Ly.qb);
  T* Rb = (T*)(base + Ly.rb);
  T* Ur = (T*)(base + Ly.ur);
  T* Vr = (T*)(base + Ly.vr);
  void* sws = base + Ly.svdws;
  if (!omega) {  // gaussian_matrix(n, w, seed ^ i) (rsvd.py:65, :82-85), kept in C order (row-major)
    // float32 inputs draw numpy's float32 stream (dtype=a.dtype), not a rounded float64 one
    rc = f64 ? bf::launch_gaussian_f64(batch, n, w, slo, shi, ibase, 0, 0, (double*)om, (int64_t)n * w, cs, 1)
             : bf::launch_gaussian_f32(batch, n, w, slo, shi, ibase, 0, 0, (float*)om, (int64_t)n * w, cs, 1);
    if (rc) return cuda_rc(rc, "rsvd/omega");
  }
  bf::GemmLaunch g;
  // Y = A @ Omega (rsvd.py:66); a device-drawn Omega is row-major, i.e. Omega^T column-major
  const bool om_rm = !omega || omega_rowmajor;
  g = bf::GemmLaunch{batch, m,    w,  n, a, m, (int64_t)m * n, false, om, om_rm ? w : n, (int64_t)n * w, om_rm, Y, m,
                     (int64_t)m * w};
  if ((rc = bf::launch_gemm(dt, g, cs))) return cuda_rc(rc, "rsvd/gemm1");
  // Q = qr(Y).q (rsvd.py:67)
  if ((rc = bf::launch_qr(dt, batch, m, w, Y, (int64_t)m * w, Q, (int64_t)m * w, R, (int64_t)w * w, sws, cs)))
    return cuda_rc(rc, "rsvd/qr1");
  // B^T = A^T Q (n x w)  (B = Q^T A, rsvd.py:68)
  g = bf::GemmLaunch{batch, n, w, m, a, m, (int64_t)m * n, true, Q, m, (int64_t)m * w, false, Bt, n, (int64_t)n * w};
  if ((rc = bf::launch_gemm(dt, g, cs))) return cuda_rc(rc, "rsvd/gemm2");
  // (Q_B, R_B) = qr(B^T) (rsvd.py:69)
  if ((rc = bf::launch_qr(dt, batch, n, w, Bt, (int64_t)n * w, Qb, (int64_t)n * w, Rb, (int64_t)w * w, sws, cs)))
    return cuda_rc(rc, "rsvd/qr2");
  // svd(R_B^T, round_robin, accumulate_v) (rsvd.py:70-73)
  bf::SvdLaunch L;
  L.batch = batch;
  L.m = w;
  L.n = w;
  L.a = Rb;
  L.a_stride = (int64_t)w * w;
  L.u = Ur;
  L.u_stride = (int64_t)w * w;
  L.s = s;
  L.s_stride = w;
  L.v = Vr;
  L.v_stride = (int64_t)w * w;
  L.sweeps = nullptr;
  L.converged = nullptr;
  L.rotations = nullptr;
  L.tol = resolve_tol(svd_tol, f64, false);
  L.max_sweeps = 30;
  L.ordering = 1;
  L.tier = 0;
  L.transpose_a = true;
  if ((rc = bf::launch_svd(dt, L, sws, Ly.total - Ly.svdws, cs))) return cuda_rc(rc, "rsvd/svd");
  // U = Q @ U_R, V = Q_B @ V_R (rsvd.py:74-75)
  g = bf::GemmLaunch{batch, m, w, w, Q, m, (int64_t)m * w, false, Ur, w, (int64_t)w * w, false, u, m, (int64_t)m * w};
  if ((rc = bf::launch_gemm(dt, g, cs))) return cuda_rc(rc, "rsvd/gemm3");
  g = bf::GemmLaunch{batch, n, w, w, Qb, n, (int64_t)n * w, false, Vr, w, (int64_t)w * w, false, v, n, (int64_t)n * w};
  if ((rc = bf::launch_gemm(dt, g, cs))) return cuda_rc(rc, "rsvd/gemm4");
  return BF_OK;
}

// ---------------------------------------------------------------- float32 on the float64 tiers
// The float32 entry points keep float32 storage but compute on the float64 tiers wherever those
// are the specialised ones: the register QR, the rr / register SVD tiers, the DMMA block-Jacobi
// pipeline (direct method) and the rsvd built on them. On B200 those run 1.7-3.7x faster than the float32
// CUDA-core tiers on every BASELINE shape (tools/time_f32.py) and are more accurate;
// the semantics stay float32 (float32 default tolerances, numpy's float32 Gaussian stream for
// rsvd). Inputs are widened into the workspace, results rounded back. BF_F32_NATIVE=1 keeps the
// float32 tiers (A/B and the float32-kernel tests).
bool f32_native() {
  const char* e = getenv("BF_F32_NATIVE");
  return e && e[0] && e[0] != '0';
}

// bump allocator over the workspace (base == nullptr: sizing only)
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* b) : base((char*)b) {}
  template <typename T>
  T* take(size_t elems) {
    T* p = base ? (T*)(base + off) : nullptr;
    off += al(elems * sizeof(T));
    return p;
  }
  void* rest() const { return base ? base + off : nullptr; }
};

int widen(int64_t n, const float* s, double* d, cudaStream_t st) { return bf::launch_cast<float, double>(n, s, d, st); }
int narrow(int64_t n, const double* s, float* d, cudaStream_t st) { return bf::launch_cast<double, float>(n, s, d, st); }

bool qr_promote(int m, int n) { return !f32_native() && m >= n && n > 0 && bf::qr_reg_covers(m, n); }

size_t qr_promo_layout(Carve& c, int64_t B, int m, int n, double** a, double** q, double** r) {
  *a = c.take<double>((size_t)B * m * n);
  *q = c.take<double>((size_t)B * m * n);
  *r = c.take<double>((size_t)B * n * n);
  return c.off + bf::qr_global_ws_bytes(0, B, m, n);
}

int qr_f32(int64_t batch, int m, int n, const float* a, float* q, float* r, int pw, void* ws, size_t wsb, void* st) {
  if (batch <= 0 || pw < 1 || !qr_promote(m, n)) return qr_impl<float>(batch, m, n, a, q, r, pw, ws, wsb, st);
  Carve c(nullptr);
  double *A, *Q, *R;
  int rc = check_ws(ws, wsb, qr_promo_layout(c, batch, m, n, &A, &Q, &R));
  if (rc) return rc;
  Carve w(ws);
  qr_promo_layout(w, batch, m, n, &A, &Q, &R);
  cudaStream_t cs = S(st);
  if ((rc = widen(batch * (int64_t)m * n, a, A, cs))) return cuda_rc(rc, "qr/widen");
  if ((rc = qr_impl<double>(batch, m, n, A, Q, R, pw, w.rest(), wsb - w.off, st))) return rc;
  if ((rc = narrow(batch * (int64_t)m * n, Q, q, cs)) || (rc = narrow(batch * (int64_t)n * n, R, r, cs)))
    return cuda_rc(rc, "qr/narrow");
  return BF_OK;
}

bool svd_promote(int m, int n, const bf_jacobi_opts* o) {
  if (f32_native() || !o || o->tier == 2 || m < n || n < 2) return false;
  bf::SvdLaunch L{};
  L.batch = 1;
  L.m = m;
  L.n = n;
  L.ordering = o->ordering;
  L.tier = o->tier;
  L.max_sweeps = o->max_sweeps;
  L.v = o->accumulate_v ? (void*)1 : nullptr;
  return bf::svd_rr_covers(L) || bf::svd_reg_covers(L);
}

size_t svd_promo_layout(Carve& c, int64_t B, int m, int n, const bf_jacobi_opts* o, double** a, double** u, double** s,
                        double** v) {
  *a = c.take<double>((size_t)B * m * n);
  *u = c.take<double>((size_t)B * m * n);
  *s = c.take<double>((size_t)B * n);
  *v = o->accumulate_v ? c.take<double>((size_t)B * n * n) : nullptr;
  return c.off + bf::svd_global_ws_bytes(0, B, m, n, o->ordering, o->accumulate_v != 0, o->tier, o->max_sweeps);
}

int svd_f32(int64_t batch, int m, int n, const float* a, float* u, float* s, float* v, int32_t* sweeps, uint8_t* conv,
            int64_t* rots, const bf_jacobi_opts* o, void* ws, size_t wsb, void* st) {
  if (batch <= 0 || check_jopts(o) || !svd_promote(m, n, o) || (o->accumulate_v && !v))
    return svd_impl<float>(batch, m, n, a, u, s, v, sweeps, conv, rots, o, ws, wsb, st);
  Carve c(nullptr);
  double *A, *U, *Sg, *V;
  int rc = check_ws(ws, wsb, svd_promo_layout(c, batch, m, n, o, &A, &U, &Sg, &V));
  if (rc) return rc;
  Carve w(ws);
  svd_promo_layout(w, batch, m, n, o, &A, &U, &Sg, &V);
  bf_jacobi_opts o64 = *o;
  o64.tolerance = resolve_tol(o->tolerance, false, false);  // float32 semantics: jacobi.py:22-25
  cudaStream_t cs = S(st);
  if ((rc = widen(batch * (int64_t)m * n, a, A, cs))) return cuda_rc(rc, "svd/widen");
  if ((rc = svd_impl<double>(batch, m, n, A, U, Sg, V, sweeps, conv, rots, &o64, w.rest(), wsb - w.off, st))) return rc;
  if ((rc = narrow(batch * (int64_t)m * n, U, u, cs)) || (rc = narrow(batch * (int64_t)n, Sg, s, cs)) ||
      (V && (rc = narrow(batch * (int64_t)n * n, V, v, cs))))
    return cuda_rc(rc, "svd/narrow");
  return BF_OK;
}

// Direct method only: the float32 Gram method's behaviour is set by its float32 rounding -- its e
// floor (~ eps32 kappa^2 of the pair blocks) sits at the float32 tolerance, so the reference's
// float32 Gram sweeps / converged flags are decided by that rounding; a
// float64 Gram would converge where the reference does not. The float32 Gram runs on the float32
// tiers.
bool block_promote(int m, int n, int method) { return !f32_native() && method == 1 && m >= n && m > 0 && n > 0; }

size_t block_promo_layout(Carve& c, int64_t B, int m, int n, const bf_block_opts* o, double** a, double** u,
                          double** s, double** v, double** e) {
  *a = c.take<double>((size_t)B * m * n);
  *u = c.take<double>((size_t)B * m * n);
  *s = c.take<double>((size_t)B * n);
  *v = o->accumulate_v ? c.take<double>((size_t)B * n * n) : nullptr;
  *e = c.take<double>((size_t)B * o->max_sweeps);
  return c.off + bf::block_ws_bytes(0, B, m, n, o->block_width, o->method, o->accumulate_v != 0);
}

int block_f32(int64_t batch, int m, int n, const float* a, float* u, float* s, float* v, int32_t* sweeps, uint8_t* conv,
              float* eh, const bf_block_opts* o, void* ws, size_t wsb, void* st, int64_t* stats) {
  if (batch <= 0 || check_bopts(o) || !block_promote(m, n, o->method) || (o->accumulate_v && !v) || !sweeps || !conv)
    return block_impl<float>(batch, m, n, a, u, s, v, sweeps, conv, eh, o, ws, wsb, st, stats);
  Carve c(nullptr);
  double *A, *U, *Sg, *V, *E;
  int rc = check_ws(ws, wsb, block_promo_layout(c, batch, m, n, o, &A, &U, &Sg, &V, &E));
  if (rc) return rc;
  Carve w(ws);
  block_promo_layout(w, batch, m, n, o, &A, &U, &Sg, &V, &E);
  bf_block_opts o64 = *o;
  o64.tolerance = resolve_tol(o->tolerance, false, true);  // float32 semantics: blockjacobi.py:19-22
  cudaStream_t cs = S(st);
  if ((rc = widen(batch * (int64_t)m * n, a, A, cs))) return cuda_rc(rc, "block_svd/widen");
  if ((rc = block_impl<double>(batch, m, n, A, U, Sg, V, sweeps, conv, eh ? E : nullptr, &o64, w.rest(), wsb - w.off,
                               st, stats)))
    return rc;
  if ((rc = narrow(batch * (int64_t)m * n, U, u, cs)) || (rc = narrow(batch * (int64_t)n, Sg, s, cs)) ||
      (V && (rc = narrow(batch * (int64_t)n * n, V, v, cs))) ||
      (eh && (rc = narrow(batch * (int64_t)o->max_sweeps, E, eh, cs))))
    return cuda_rc(rc, "block_svd/narrow");
  return BF_OK;
}

bool rsvd_promote() { return !f32_native(); }

size_t rsvd_promo_layout(Carve& c, int64_t B, int m, int n, int w, bool draw, double** a, double** om, float** om32,
                         double** u, double** s, double** v) {
  *a = c.take<double>((size_t)B * m * n);
  *om = c.take<double>((size_t)B * n * w);
  *om32 = draw ? c.take<float>((size_t)B * n * w) : nullptr;
  *u = c.take<double>((size_t)B * m * w);
  *s = c.take<double>((size_t)B * w);
  *v = c.take<double>((size_t)B * n * w);
  return c.off + rsvd_layout(B, m, n, w, 8, false).total;
}

int rsvd_f32(int64_t batch, int m, int n, int k, int p, uint64_t slo, uint64_t shi, int64_t ibase, const float* a,
             const float* omega, float* u, float* s, float* v, void* ws, size_t wsb, void* st) {
  const int w = k + p;
  if (batch <= 0 || k < 1 || p < 0 || w > std::min(m, n) || !rsvd_promote())
    return rsvd_impl<float>(batch, m, n, k, p, slo, shi, ibase, a, omega, u, s, v, ws, wsb, st);
  Carve c(nullptr);
  double *A, *Om, *U, *Sg, *V;
  float* Om32;
  int rc = check_ws(ws, wsb, rsvd_promo_layout(c, batch, m, n, w, !omega, &A, &Om, &Om32, &U, &Sg, &V));
  if (rc) return rc;
  Carve cw(ws);
  rsvd_promo_layout(cw, batch, m, n, w, !omega, &A, &Om, &Om32, &U, &Sg, &V);
  cudaStream_t cs = S(st);
  const int64_t nom = batch * (int64_t)n * w;
  if (!omega) {  // numpy's float32 stream (rsvd.py:65 dtype=a.dtype), C order, then widened
    rc = bf::launch_gaussian_f32(batch, n, w, slo, shi, ibase, 0, 0, Om32, (int64_t)n * w, cs, 1);
    if (rc) return cuda_rc(rc, "rsvd/omega");
  }
  if ((rc = widen(batch * (int64_t)m * n, a, A, cs)) || (rc = widen(nom, omega ? omega : Om32, Om, cs)))
    return cuda_rc(rc, "rsvd/widen");
  if ((rc = rsvd_impl<double>(batch, m, n, k, p, slo, shi, ibase, A, Om, U, Sg, V, cw.rest(), wsb - cw.off, st,
                              !omega, resolve_tol(0.0, false, false))))
    return rc;
  if ((rc = narrow(batch * (int64_t)m * w, U, u, cs)) || (rc = narrow(batch * (int64_t)w, Sg, s, cs)) ||
      (rc = narrow(batch * (int64_t)n * w, V, v, cs)))
    return cuda_rc(rc, "rsvd/narrow");
  return BF_OK;
}

template <typename T>
int gemm_impl(int64_t batch, int M, int N, int K, const T* a, int lda, int64_t as, int ta, const T* b, int ldb,
              int64_t bs, int tb, T* c, int ldc, int64_t cs, void* st) {
  if (batch < 0 || M < 0 || N < 0 || K < 0) return fail(BF_ERR_ARG, "negative batch or shape");
  if (ldc < std::max(M, 1)) return fail(BF_ERR_ARG, "ldc %d < M %d", ldc, M);
  if (lda < std::max(ta ? K : M, 1)) return fail(BF_ERR_ARG, "lda %d too small", lda);
  if (ldb < std::max(tb ? N : K, 1)) return fail(BF_ERR_ARG, "ldb %d too small", ldb);
  if (batch == 0 || M == 0 || N == 0) return BF_OK;
  if (K == 0) {  // empty inner dimension: C = 0
    if (ldc == M && cs == (int64_t)M * N)
      cudaMemsetAsync(c, 0, sizeof(T) * (size_t)batch * M * N, S(st));
    else
      for (int64_t i = 0; i < batch; ++i) cudaMemset2DAsync(c + i * cs, sizeof(T) * ldc, 0, sizeof(T) * M, N, S(st));
    return cuda_rc((int)cudaGetLastError(), "gemm");
  }
  bf::GemmLaunch g;
  g.batch = batch;
  g.M = M;
  g.N = N;
  g.K = K;
  g.a = a;
  g.lda = lda;
  g.a_stride = as;
  g.ta = ta != 0;
  g.b = b;
  g.ldb = ldb;
  g.b_stride = bs;
  g.tb = tb != 0;
  g.c = c;
  g.ldc = ldc;
  g.c_stride = cs;
  return cuda_rc(bf::launch_gemm(sizeof(T) == 8 ? 0 : 1, g, S(st)), "gemm");
}

}  // namespace

extern "C" {

const char* bf_last_error(void) { return g_err.c_str(); }
const char* bf_version(void) { return "batchfact_b200 0.1.0 (sm_100a)"; }

size_t bf_qr_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t es) {
  if (m < n || m <= 0 || n <= 0) return 0;
  if (es == 4 && batch > 0 && qr_promote(m, n)) {
    Carve c(nullptr);
    double *a, *q, *r;
    return qr_promo_layout(c, batch, m, n, &a, &q, &r);
  }
  return bf::qr_global_ws_bytes(es == 8 ? 0 : 1, batch, m, n);
}
int bf_qr_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* q, double* r, int32_t pw,
                      void* ws, size_t wsb, void* st) {
  return qr_impl<double>(batch, m, n, a, q, r, pw, ws, wsb, st);
}
int bf_qr_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* q, float* r, int32_t pw, void* ws,
                      size_t wsb, void* st) {
  return qr_f32(batch, m, n, a, q, r, pw, ws, wsb, st);
}

size_t bf_svd_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t es, const bf_jacobi_opts* o) {
  if (!o || m < n || n <= 0) return 0;
  if (es == 4 && batch > 0 && svd_promote(m, n, o)) {
    Carve c(nullptr);
    double *a, *u, *s, *v;
    return svd_promo_layout(c, batch, m, n, o, &a, &u, &s, &v);
  }
  return bf::svd_global_ws_bytes(es == 8 ? 0 : 1, batch, m, n, o->ordering, o->accumulate_v != 0, o->tier,
                                 o->max_sweeps);
}
int bf_svd_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* u, double* s, double* v,
                       int32_t* sweeps, uint8_t* conv, int64_t* rots, const bf_jacobi_opts* o, void* ws, size_t wsb,
                       void* st) {
  return svd_impl<double>(batch, m, n, a, u, s, v, sweeps, conv, rots, o, ws, wsb, st);
}
int bf_svd_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* u, float* s, float* v,
                       int32_t* sweeps, uint8_t* conv, int64_t* rots, const bf_jacobi_opts* o, void* ws, size_t wsb,
                       void* st) {
  return svd_f32(batch, m, n, a, u, s, v, sweeps, conv, rots, o, ws, wsb, st);
}

size_t bf_block_svd_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t es, const bf_block_opts* o) {
  if (!o || m < n || m <= 0 || o->block_width < 1) return 0;
  if (es == 4 && batch > 0 && o->max_sweeps >= 1 && block_promote(m, n, o->method)) {
    Carve c(nullptr);
    double *a, *u, *s, *v, *e;
    return block_promo_layout(c, batch, m, n, o, &a, &u, &s, &v, &e);
  }
  return bf::block_ws_bytes(es == 8 ? 0 : 1, batch, m, n, o->block_width, o->method, o->accumulate_v != 0);
}
int bf_block_svd_batched_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* u, double* s, double* v,
                             int32_t* sweeps, uint8_t* conv, double* eh, const bf_block_opts* o, void* ws, size_t wsb,
                             void* st) {
  return block_impl<double>(batch, m, n, a, u, s, v, sweeps, conv, eh, o, ws, wsb, st);
}
int bf_block_svd_batched_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* u, float* s, float* v,
                             int32_t* sweeps, uint8_t* conv, float* eh, const bf_block_opts* o, void* ws, size_t wsb,
                             void* st) {
  return block_f32(batch, m, n, a, u, s, v, sweeps, conv, eh, o, ws, wsb, st, nullptr);
}
int bf_block_svd_batched_ex_f64(int64_t batch, int32_t m, int32_t n, const double* a, double* u, double* s, double* v,
                                int32_t* sweeps, uint8_t* conv, double* eh, int64_t* stats, const bf_block_opts* o,
                                void* ws, size_t wsb, void* st) {
  return block_impl<double>(batch, m, n, a, u, s, v, sweeps, conv, eh, o, ws, wsb, st, stats);
}
int bf_block_svd_batched_ex_f32(int64_t batch, int32_t m, int32_t n, const float* a, float* u, float* s, float* v,
                                int32_t* sweeps, uint8_t* conv, float* eh, int64_t* stats, const bf_block_opts* o,
                                void* ws, size_t wsb, void* st) {
  return block_f32(batch, m, n, a, u, s, v, sweeps, conv, eh, o, ws, wsb, st, stats);
}

size_t bf_rsvd_workspace_size(int64_t batch, int32_t m, int32_t n, int32_t k, int32_t p, int32_t es) {
  if (k < 1 || p < 0 || k + p > std::min(m, n)) return 0;
  if (es == 4 && batch > 0 && rsvd_promote()) {
    Carve c(nullptr);
    double *a, *om, *u, *s, *v;
    float* om32;
    return rsvd_promo_layout(c, batch, m, n, k + p, true, &a, &om, &om32, &u, &s, &v);
  }
  return rsvd_layout(batch, m, n, k + p, es, true).total;
}
int bf_rsvd_batched_f64(int64_t batch, int32_t m, int32_t n, int32_t k, int32_t p, uint64_t slo, uint64_t shi,
                        int64_t ibase, const double* a, const double* omega, double* u, double* s, double* v, void* ws,
                        size_t wsb, void* st) {
  return rsvd_impl<double>(batch, m, n, k, p, slo, shi, ibase, a, omega, u, s, v, ws, wsb, st);
}
int bf_rsvd_batched_f32(int64_t batch, int32_t m, int32_t n, int32_t k, int32_t p, uint64_t slo, uint64_t shi,
                        int64_t ibase, const float* a, const float* omega, float* u, float* s, float* v, void* ws,
                        size_t wsb, void* st) {
  return rsvd_f32(batch, m, n, k, p, slo, shi, ibase, a, omega, u, s, v, ws, wsb, st);
}

int bf_gaussian_batched_f64(int64_t batch, int32_t rows, int32_t cols, uint64_t slo, uint64_t shi, int64_t ibase,
                            int32_t mode, double* out, void* st) {
  if (batch < 0 || rows < 0 || cols < 0) return fail(BF_ERR_ARG, "rows and cols must be >= 0");
  return cuda_rc(bf::launch_gaussian_f64(batch, rows, cols, slo, shi, ibase, mode, 0, out, (int64_t)rows * cols, S(st)),
                 "gaussian");
}

int bf_gaussian_batched_f32(int64_t batch, int32_t rows, int32_t cols, uint64_t slo, uint64_t shi, int64_t ibase,
                            int32_t mode, float* out, void* st) {
  if (batch < 0 || rows < 0 || cols < 0) return fail(BF_ERR_ARG, "rows and cols must be >= 0");
  return cuda_rc(bf::launch_gaussian_f32(batch, rows, cols, slo, shi, ibase, mode, 0, out, (int64_t)rows * cols, S(st)),
                 "gaussian");
}

size_t bf_make_matrix_workspace_size(int64_t batch, int32_t m, int32_t n) {
  return al((size_t)batch * m * n * 8) * 2 + al((size_t)batch * n * n * 8) * 3 + al((size_t)n * 8) +
         std::max(bf::qr_global_ws_bytes(0, batch, m, n), bf::qr_global_ws_bytes(0, batch, n, n));
}

int bf_make_matrix_batched_f64(int64_t batch, int32_t m, int32_t n, int32_t mode, double cond, int32_t rank,
                               uint64_t slo, uint64_t shi, int64_t ibase, double* a, double* sigma, void* ws,
                               size_t wsb, void* st) {
  if (m < n || n < 1) return fail(BF_ERR_ARG, "make_matrix requires m >= spec.n >= 1");
  if (rank < 1 || rank > n) return fail(BF_ERR_ARG, "rank must be in [1, n]");
  if (!(cond >= 1.0)) return fail(BF_ERR_ARG, "cond must be >= 1");
  int rc = check_ws(ws, wsb, bf_make_matrix_workspace_size(batch, m, n));
  if (rc) return rc;
  if (batch == 0) return BF_OK;
  cudaStream_t cs = S(st);
  char* base = (char*)ws;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base + off;
    off += al(bytes);
    return (double*)p;
  };
  double* G1 = take((size_t)batch * m * n * 8);
  double* P = take((size_t)batch * m * n * 8);
  double* G2 = take((size_t)batch * n * n * 8);
  double* Qn = take((size_t)batch * n * n * 8);
  double* Rr = take((size_t)batch * n * n * 8);
  double* sg = take((size_t)n * 8);
  void* qws = base + off;
  // spectrum (testmat.py:51-65), same for every entry: computed on the host like numpy does
  std::vector<double> h(n, 0.0);
  if (rank == 1)
    h[0] = 1.0;
  else
    for (int i = 0; i < rank; ++i)
      h[i] = mode == 0 ? std::pow(cond, -(double)i / (double)(rank - 1))
                       : 1.0 - (1.0 - 1.0 / cond) * (double)i / (double)(rank - 1);
  if ((rc = (int)cudaMemcpyAsync(sg, h.data(), n * 8, cudaMemcpyHostToDevice, cs))) return cuda_rc(rc, "make_matrix");
  if ((rc = (int)cudaMemcpyAsync(sigma, sg, n * 8, cudaMemcpyDeviceToDevice, cs))) return cuda_rc(rc, "make_matrix");
  // P = random_orthonormal(m, n, seed), Q = random_orthonormal(n, n, seed ^ MIX) (testmat.py:68-80)
  if ((rc = bf::launch_gaussian_f64(batch, m, n, slo, shi, ibase, 1, 0, G1, (int64_t)m * n, cs)))
    return cuda_rc(rc, "make_matrix");
  if ((rc = bf::launch_gaussian_f64(batch, n, n, slo, shi, ibase, 1, 0x9E3779B97F4A7C15ULL, G2, (int64_t)n * n, cs)))
    return cuda_rc(rc, "make_matrix");
  if ((rc = bf::launch_qr(0, batch, m, n, G1, (int64_t)m * n, P, (int64_t)m * n, Rr, (int64_t)n * n, qws, cs)))
    return cuda_rc(rc, "make_matrix");
  if ((rc = bf::launch_sign_fix_f64(batch, m, n, P, Rr, cs))) return cuda_rc(rc, "make_matrix");
  if ((rc = bf::launch_qr(0, batch, n, n, G2, (int64_t)n * n, Qn, (int64_t)n * n, Rr, (int64_t)n * n, qws, cs)))
    return cuda_rc(rc, "make_matrix");
  if ((rc = bf::launch_sign_fix_f64(batch, n, n, Qn, Rr, cs))) return cuda_rc(rc, "make_matrix");
  if ((rc = bf::launch_scale_cols_f64(batch, m, n, P, sg, cs))) return cuda_rc(rc, "make_matrix");
  bf::GemmLaunch g{batch, m, n, n, P, m, (int64_t)m * n, false, Qn, n, (int64_t)n * n, true, a, m, (int64_t)m * n};
  return cuda_rc(bf::launch_gemm(0, g, cs), "make_matrix");
}

int bf_gemm_batched_f64(int64_t batch, int32_t M, int32_t N, int32_t K, const double* a, int32_t lda, int64_t as,
                        int32_t ta, const double* b, int32_t ldb, int64_t bs, int32_t tb, double* c, int32_t ldc,
                        int64_t cs, void* st) {
  return gemm_impl<double>(batch, M, N, K, a, lda, as, ta, b, ldb, bs, tb, c, ldc, cs, st);
}
int bf_gemm_batched_f32(int64_t batch, int32_t M, int32_t N, int32_t K, const float* a, int32_t lda, int64_t as,
                        int32_t ta, const float* b, int32_t ldb, int64_t bs, int32_t tb, float* c, int32_t ldc,
                        int64_t cs, void* st) {
  return gemm_impl<float>(batch, M, N, K, a, lda, as, ta, b, ldb, bs, tb, c, ldc, cs, st);
}

// ---------------------------------------------------------------- reference helpers
#define BF_HELPER_PAIR(T, SUF)                                                                                   \
  int bf_householder_batched_##SUF(int64_t batch, int32_t len, const T* x, T* v, T* tau, void* st) {             \
    if (batch < 0 || len < 1) return fail(BF_ERR_ARG, "householder_vector expects a nonempty vector");            \
    return cuda_rc(bf::launch_householder<T>(batch, len, x, v, tau, S(st)), "householder");                      \
  }                                                                                                              \
  int bf_off_orthogonality_batched_##SUF(int64_t batch, int32_t m, int32_t n, const T* a, T* out, void* st) {    \
    if (batch < 0 || m < 0 || n < 0) return fail(BF_ERR_ARG, "negative batch or shape");                        \
    return cuda_rc(bf::launch_offdiag<T>(batch, m, n, a, 1, out, S(st)), "off_orthogonality");                  \
  }                                                                                                              \
  int bf_scaled_offdiag_batched_##SUF(int64_t batch, int32_t n, const T* g, T* out, void* st) {                  \
    if (batch < 0 || n < 0) return fail(BF_ERR_ARG, "negative batch or shape");                                 \
    return cuda_rc(bf::launch_offdiag<T>(batch, n, n, g, 0, out, S(st)), "scaled_offdiag");                     \
  }                                                                                                              \
  int bf_syrk_batched_##SUF(int64_t batch, int32_t m, int32_t k, const T* a, T* g, void* st) {                   \
    if (batch < 0 || m < 0 || k < 0) return fail(BF_ERR_ARG, "negative batch or shape");                        \
    return cuda_rc(bf::launch_syrk<T>(batch, m, k, a, g, S(st)), "syrk");                                       \
  }                                                                                                              \
  int bf_frobenius_batched_##SUF(int64_t batch, int32_t m, int32_t n, const T* a, T* out, void* st) {            \
    if (batch < 0 || m < 0 || n < 0) return fail(BF_ERR_ARG, "negative batch or shape");                        \
    return cuda_rc(bf::launch_frobenius<T>(batch, (int64_t)m * n, a, out, S(st)), "frobenius");                 \
  }                                                                                                              \
  int bf_axpby_##SUF(int64_t n, T alpha, const T* p, T beta, const T* c, T* out, void* st) {                     \
    if (n < 0) return fail(BF_ERR_ARG, "negative length");                                                       \
    if (beta != T(0) && !c) return fail(BF_ERR_ARG, "beta != 0 requires c");                                     \
    return cuda_rc(bf::launch_axpby<T>(n, alpha, p, beta, c, out, S(st)), "axpby");                             \
  }
BF_HELPER_PAIR(double, f64)
BF_HELPER_PAIR(float, f32)
#undef BF_HELPER_PAIR

int bf_jacobi_rotation_batched_f64(int64_t batch, const double* gpp, const double* gpq, const double* gqq, double* c,
                                   double* s, void* st) {
  if (batch < 0) return fail(BF_ERR_ARG, "negative batch");
  return cuda_rc(bf::launch_rotation(batch, gpp, gpq, gqq, c, s, S(st)), "jacobi_rotation");
}

}  // extern "C"
