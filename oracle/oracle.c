/* batchfact CPU ORACLE -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference's hot path (/root/reference/pkg/src/batchfact,
 * pure Python + numpy) used ONLY by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs, as the CHECKER of the CUDA path and as the
 * CPU baseline. The product (paper_1707_05141_b200/) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this oracle against golden
 * fixtures produced by running the reference itself (tests/golden/make_golden.py).
 *
 * Restated functions (reference file:line):
 *   jacobi_rotation        jacobi.py:68-80        round_robin_schedule  jacobi.py:102-115
 *   householder_vector     qr.py:26-48            _apply_reflector      qr.py:51-60
 *   qr                     qr.py:63-95            off_orthogonality     jacobi.py:83-99
 *   _serial_sweep          jacobi.py:118-155      _round_robin_sweep    jacobi.py:158-186
 *   _complete_zero_rows    jacobi.py:189-209      _extract_svd          jacobi.py:212-228
 *   svd                    jacobi.py:231-284      syrk                  core.py:68-78
 *   scaled_offdiag         blockjacobi.py:57-76   block_svd             blockjacobi.py:84-168
 *   gaussian_matrix        rsvd.py:42-53 (numpy 2.3.5 Philox4x64-10 + float64 / float32 ziggurat)
 *   rsvd                   rsvd.py:56-76          batch_rsvd seed^i     rsvd.py:79-86
 *   spectrum / random_orthonormal / make_matrix   testmat.py:51-94
 *   batch_apply lowest-failing-index convention   core.py:97-123
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off: numpy never fuses a*b+c).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ziggurat_tables.h"

#define ORC_API __attribute__((visibility("default")))

/* ---------------------------------------------------------------- scalars */

/* jacobi_rotation (jacobi.py:68-80): Rutishauser; computed in double. */
static void orc_jacobi_rotation(double gpp, double gpq, double gqq, double* c, double* s) {
  if (gpq == 0.0) {
    *c = 1.0;
    *s = 0.0;
    return;
  }
  double zeta = (gqq - gpp) / (2.0 * gpq);
  double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
  double cc = 1.0 / hypot(1.0, t);
  *c = cc;
  *s = cc * t;
}

/* round_robin_schedule (jacobi.py:102-115): circle method, pairs normalised (min,max).
 * out: (n-1) steps x n/2 pairs x 2 ints. */
static void orc_round_robin_schedule(int n, int* out) {
  int* idx = (int*)malloc(sizeof(int) * n);
  int* nx = (int*)malloc(sizeof(int) * n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  for (int st = 0; st < n - 1; ++st) {
    for (int i = 0; i < n / 2; ++i) {
      int p = idx[i], q = idx[n - 1 - i];
      out[((size_t)st * (n / 2) + i) * 2 + 0] = p < q ? p : q;
      out[((size_t)st * (n / 2) + i) * 2 + 1] = p < q ? q : p;
    }
    nx[0] = idx[0];
    nx[1] = idx[n - 1];
    for (int j = 2; j < n; ++j) nx[j] = idx[j - 1];
    memcpy(idx, nx, sizeof(int) * n);
  }
  free(idx);
  free(nx);
}

static double orc_default_tol(size_t elem) { return elem == sizeof(double) ? 1e-14 : 1e-6; }

/* ------------------------------------------------- numpy Philox + ziggurat */

typedef struct {
  uint64_t ctr[4], key[2], buf[4];
  int pos;
} orc_philox;

static inline uint64_t orc_mulhilo(uint64_t a, uint64_t b, uint64_t* hi) {
  __uint128_t p = (__uint128_t)a * b;
  *hi = (uint64_t)(p >> 64);
  return (uint64_t)p;
}

/* Philox4x64-10 (Random123 constants), numpy bit_generator semantics: counter is
 * incremented BEFORE each block, 4 outputs buffered. */
static uint64_t orc_philox_next(orc_philox* st) {
  if (st->pos < 4) return st->buf[st->pos++];
  if (++st->ctr[0] == 0)
    if (++st->ctr[1] == 0)
      if (++st->ctr[2] == 0) ++st->ctr[3];
  uint64_t c0 = st->ctr[0], c1 = st->ctr[1], c2 = st->ctr[2], c3 = st->ctr[3];
  uint64_t k0 = st->key[0], k1 = st->key[1];
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    uint64_t hi0, hi1;
    uint64_t lo0 = orc_mulhilo(0xD2E7470EE14C6C93ULL, c0, &hi0);
    uint64_t lo1 = orc_mulhilo(0xCA5A826395121157ULL, c2, &hi1);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  st->buf[0] = c0;
  st->buf[1] = c1;
  st->buf[2] = c2;
  st->buf[3] = c3;
  st->pos = 1;
  return c0;
}

static inline double orc_next_double(orc_philox* st) {
  return (double)(orc_philox_next(st) >> 11) * (1.0 / 9007199254740992.0);
}

/* numpy random_standard_normal (float64 ziggurat) */
static double orc_standard_normal(orc_philox* st) {
  for (;;) {
    uint64_t r = orc_philox_next(st);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 0x1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * bf_zig_wi[idx];
    if (sign & 0x1) x = -x;
    if (rabs < bf_zig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -BF_ZIG_NOR_INV_R * log1p(-orc_next_double(st));
        double yy = -log1p(-orc_next_double(st));
        if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(BF_ZIG_NOR_R + xx) : BF_ZIG_NOR_R + xx;
      }
    } else {
      if (((bf_zig_fi[idx - 1] - bf_zig_fi[idx]) * orc_next_double(st) + bf_zig_fi[idx]) < exp(-0.5 * x * x))
        return x;
    }
  }
}

/* numpy's next_uint32 on Philox (bit_generator buffering): the low half of a fresh 64-bit
 * word, then its high half. */
typedef struct {
  orc_philox p;
  int has32;
  uint32_t hi32;
} orc_philox32;

static inline uint32_t orc_next_u32(orc_philox32* st) {
  if (st->has32) {
    st->has32 = 0;
    return st->hi32;
  }
  uint64_t w = orc_philox_next(&st->p);
  st->has32 = 1;
  st->hi32 = (uint32_t)(w >> 32);
  return (uint32_t)(w & 0xffffffffu);
}

static inline float orc_next_float(orc_philox32* st) {
  return (float)(orc_next_u32(st) >> 8) * (1.0f / 16777216.0f);
}

/* numpy random_standard_normal_f (float32 ziggurat on 23-bit halves). log1pf is the C
 * library's (npy_log1pf); the wedge test compares in double against exp(-0.5 x x). */
static float orc_standard_normal_f(orc_philox32* st) {
  for (;;) {
    uint32_t r = orc_next_u32(st);
    int idx = (int)(r & 0xff);
    int sign = (int)((r >> 8) & 0x1);
    uint32_t rabs = r >> 9;
    float x = (float)rabs * bf_zig_wi_f[idx];
    if (sign) x = -x;
    if (rabs < bf_zig_ki_f[idx]) return x;
    if (idx == 0) {
      for (;;) {
        float xx = -BF_ZIG_NOR_INV_R_F * log1pf(-orc_next_float(st));
        float yy = -log1pf(-orc_next_float(st));
        if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(BF_ZIG_NOR_R_F + xx) : BF_ZIG_NOR_R_F + xx;
      }
    } else {
      if (((bf_zig_fi_f[idx - 1] - bf_zig_fi_f[idx]) * orc_next_float(st) + bf_zig_fi_f[idx]) <
          exp(-0.5 * x * x))
        return x;
    }
  }
}

/* gaussian_matrix(rows, cols, seed, dtype=float32) (rsvd.py:42-53, dtype=a.dtype at :65) */
ORC_API int orc_gaussian_f32(int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, float* out) {
  if (rows < 0 || cols < 0) return -1;
  orc_philox32 st;
  memset(&st, 0, sizeof(st));
  st.p.key[0] = seed_lo;
  st.p.key[1] = seed_hi;
  st.p.pos = 4;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out[(size_t)j * rows + i] = orc_standard_normal_f(&st);
  return 0;
}

/* gaussian_matrix(rows, cols, seed) (rsvd.py:42-53): C-order fill, returned column-major */
ORC_API int orc_gaussian_f64(int rows, int cols, uint64_t seed_lo, uint64_t seed_hi, double* out) {
  if (rows < 0 || cols < 0) return -1;
  orc_philox st;
  memset(&st, 0, sizeof(st));
  st.key[0] = seed_lo;
  st.key[1] = seed_hi;
  st.pos = 4;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out[(size_t)j * rows + i] = orc_standard_normal(&st);
  return 0;
}

ORC_API void orc_philox_raw(uint64_t seed_lo, uint64_t seed_hi, int n, uint64_t* out) {
  orc_philox st;
  memset(&st, 0, sizeof(st));
  st.key[0] = seed_lo;
  st.key[1] = seed_hi;
  st.pos = 4;
  for (int i = 0; i < n; ++i) out[i] = orc_philox_next(&st);
}

/* ------------------------------------------------------- templated bodies */

#define T double
#define SUF _f64
#include "oracle_impl.h"
#undef T
#undef SUF
#define T float
#define SUF _f32
#include "oracle_impl.h"
#undef T
#undef SUF

/* ------------------------------------------------------------ exported */

ORC_API void orc_round_robin(int n, int* out) { orc_round_robin_schedule(n, out); }

ORC_API void orc_rotation(double gpp, double gpq, double gqq, double* cs) {
  orc_jacobi_rotation(gpp, gpq, gqq, &cs[0], &cs[1]);
}

ORC_API double orc_householder_f64(const double* x, int len, double* v) { return householder_f64(x, len, v); }
ORC_API double orc_off_orthogonality_f64(const double* a, int rows, int cols) {
  return off_orthogonality_f64(a, rows, cols);
}
ORC_API double orc_scaled_offdiag_f64(const double* g, int n) { return scaled_offdiag_f64(g, n); }
ORC_API void orc_syrk_f64(int m, int k, const double* a, double* g) { syrk_f64(m, k, a, g); }

/* Batch drivers: one worker per entry range, entries independent (core.py:97-123).
 * Every entry runs to completion; *bad_index receives the lowest failing index or -1. */

typedef struct {
  int kind, dtype;
  int64_t lo, hi;
  int m, n;
  const void* a;
  void *o1, *o2, *o3;
  int* sweeps;
  int* conv;
  long* rot;
  void* e_hist;
  int i1, i2, i3, i4;
  double tol;
  uint64_t seed_lo, seed_hi;
  int64_t index_base;
  const void* omega;
  int64_t first_bad;
} orc_job;

static void* orc_worker(void* arg) {
  orc_job* j = (orc_job*)arg;
  size_t es = j->dtype == 0 ? sizeof(double) : sizeof(float);
  int m = j->m, n = j->n;
  j->first_bad = -1;
  void* work = malloc(es * (size_t)2 * m * n + 64);
  for (int64_t b = j->lo; b < j->hi; ++b) {
    int rc = 0;
    const char* a = (const char*)j->a + es * (size_t)b * m * n;
    if (j->kind == 0) { /* qr */
      char* q = (char*)j->o1 + es * (size_t)b * m * n;
      char* r = (char*)j->o2 + es * (size_t)b * n * n;
      rc = j->dtype == 0 ? qr_f64(m, n, (const double*)a, (double*)q, (double*)r, j->i1, (double*)work)
                         : qr_f32(m, n, (const float*)a, (float*)q, (float*)r, j->i1, (float*)work);
    } else if (j->kind == 1) { /* svd */
      char* u = (char*)j->o1 + es * (size_t)b * m * n;
      char* s = (char*)j->o2 + es * (size_t)b * n;
      char* v = j->o3 ? (char*)j->o3 + es * (size_t)b * n * n : NULL;
      long* rot = j->rot ? j->rot + b : NULL;
      rc = j->dtype == 0 ? svd_f64(m, n, (const double*)a, (double*)u, (double*)s, (double*)v, j->sweeps + b,
                                   j->conv + b, rot, j->tol, j->i1, j->i2)
                         : svd_f32(m, n, (const float*)a, (float*)u, (float*)s, (float*)v, j->sweeps + b,
                                   j->conv + b, rot, j->tol, j->i1, j->i2);
    } else if (j->kind == 2) { /* block svd */
      char* u = (char*)j->o1 + es * (size_t)b * m * n;
      char* s = (char*)j->o2 + es * (size_t)b * n;
      char* v = j->o3 ? (char*)j->o3 + es * (size_t)b * n * n : NULL;
      char* eh = j->e_hist ? (char*)j->e_hist + es * (size_t)b * j->i3 : NULL;
      rc = j->dtype == 0 ? block_svd_f64(m, n, (const double*)a, (double*)u, (double*)s, (double*)v, j->sweeps + b,
                                         j->conv + b, (double*)eh, j->i1, j->i2, j->tol, j->i3)
                         : block_svd_f32(m, n, (const float*)a, (float*)u, (float*)s, (float*)v, j->sweeps + b,
                                         j->conv + b, (float*)eh, j->i1, j->i2, j->tol, j->i3);
    } else if (j->kind == 3) { /* rsvd: seed ^ (index_base + b) (rsvd.py:82-85) */
      int w = j->i1 + j->i2;
      char* u = (char*)j->o1 + es * (size_t)b * m * w;
      char* s = (char*)j->o2 + es * (size_t)b * w;
      char* v = (char*)j->o3 + es * (size_t)b * n * w;
      uint64_t idx = (uint64_t)(j->index_base + b);
      const char* om = j->omega ? (const char*)j->omega + es * (size_t)b * n * w : NULL;
      rc = j->dtype == 0 ? rsvd_f64(m, n, j->i1, j->i2, j->seed_lo ^ idx, j->seed_hi, (const double*)a,
                                    (const double*)om, (double*)u, (double*)s, (double*)v)
                         : rsvd_f32(m, n, j->i1, j->i2, j->seed_lo ^ idx, j->seed_hi, (const float*)a,
                                    (const float*)om, (float*)u, (float*)s, (float*)v);
    }
    if (rc != 0 && j->first_bad < 0) j->first_bad = b;
  }
  free(work);
  return NULL;
}

static int64_t orc_run(orc_job* tmpl, int64_t B, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > B) nthreads = B > 0 ? (int)B : 1;
  orc_job* jobs = (orc_job*)malloc(sizeof(orc_job) * nthreads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = *tmpl;
    jobs[t].lo = B * t / nthreads;
    jobs[t].hi = B * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, orc_worker, &jobs[t]);
  }
  int64_t bad = -1;
  for (int t = 0; t < nthreads; ++t) {
    pthread_join(th[t], NULL);
    if (jobs[t].first_bad >= 0 && (bad < 0 || jobs[t].first_bad < bad)) bad = jobs[t].first_bad;
  }
  free(jobs);
  free(th);
  return bad;
}

ORC_API int64_t orc_batch_qr(int dtype, int64_t B, int m, int n, const void* a, void* q, void* r, int pw,
                             int nthreads) {
  orc_job j;
  memset(&j, 0, sizeof(j));
  j.kind = 0; j.dtype = dtype; j.m = m; j.n = n; j.a = a; j.o1 = q; j.o2 = r; j.i1 = pw;
  return orc_run(&j, B, nthreads);
}

ORC_API int64_t orc_batch_svd(int dtype, int64_t B, int m, int n, const void* a, void* u, void* s, void* v,
                              int* sweeps, int* conv, long* rot, double tol, int max_sweeps, int ordering,
                              int nthreads) {
  orc_job j;
  memset(&j, 0, sizeof(j));
  j.kind = 1; j.dtype = dtype; j.m = m; j.n = n; j.a = a; j.o1 = u; j.o2 = s; j.o3 = v;
  j.sweeps = sweeps; j.conv = conv; j.rot = rot; j.tol = tol; j.i1 = max_sweeps; j.i2 = ordering;
  return orc_run(&j, B, nthreads);
}

ORC_API int64_t orc_batch_block_svd(int dtype, int64_t B, int m, int n, const void* a, void* u, void* s, void* v,
                                    int* sweeps, int* conv, void* e_hist, int bw, int method, double tol,
                                    int max_sweeps, int nthreads) {
  orc_job j;
  memset(&j, 0, sizeof(j));
  j.kind = 2; j.dtype = dtype; j.m = m; j.n = n; j.a = a; j.o1 = u; j.o2 = s; j.o3 = v;
  j.sweeps = sweeps; j.conv = conv; j.e_hist = e_hist; j.i1 = bw; j.i2 = method; j.i3 = max_sweeps; j.tol = tol;
  return orc_run(&j, B, nthreads);
}

ORC_API int64_t orc_batch_rsvd(int dtype, int64_t B, int m, int n, int k, int p, uint64_t seed_lo,
                               uint64_t seed_hi, int64_t index_base, const void* a, const void* omega, void* u,
                               void* s, void* v, int nthreads) {
  orc_job j;
  memset(&j, 0, sizeof(j));
  j.kind = 3; j.dtype = dtype; j.m = m; j.n = n; j.a = a; j.o1 = u; j.o2 = s; j.o3 = v; j.i1 = k; j.i2 = p;
  j.seed_lo = seed_lo; j.seed_hi = seed_hi; j.index_base = index_base; j.omega = omega;
  return orc_run(&j, B, nthreads);
}

/* testmat (testmat.py:51-94): geometric/arithmetic spectrum, A = P diag(sigma) Q^T */
static void orc_random_orthonormal(int m, int n, uint64_t seed_lo, uint64_t seed_hi, double* q) {
  double* g = (double*)malloc(sizeof(double) * (size_t)m * n);
  double* r = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* work = (double*)malloc(sizeof(double) * (size_t)2 * m * n);
  orc_gaussian_f64(m, n, seed_lo, seed_hi, g);
  qr_f64(m, n, g, q, r, 16, work);
  for (int j = 0; j < n; ++j)
    if (r[(size_t)j * n + j] < 0)
      for (int i = 0; i < m; ++i) q[(size_t)j * m + i] *= -1.0;
  free(g);
  free(r);
  free(work);
}

ORC_API int orc_make_matrix_f64(int m, int n, int mode /*0 geometric,1 arithmetic*/, double cond, int rank,
                                uint64_t seed_lo, uint64_t seed_hi, double* a, double* sigma) {
  if (m < n || rank < 1 || rank > n) return -1;
  for (int i = 0; i < n; ++i) sigma[i] = 0.0;
  if (rank == 1) {
    sigma[0] = 1.0;
  } else {
    for (int i = 0; i < rank; ++i)
      sigma[i] = mode == 0 ? pow(cond, -(double)i / (double)(rank - 1))
                           : 1.0 - (1.0 - 1.0 / cond) * (double)i / (double)(rank - 1);
  }
  double* p = (double*)malloc(sizeof(double) * (size_t)m * n);
  double* q = (double*)malloc(sizeof(double) * (size_t)n * n);
  orc_random_orthonormal(m, n, seed_lo, seed_hi, p);
  orc_random_orthonormal(n, n, seed_lo ^ 0x9E3779B97F4A7C15ULL, seed_hi, q);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += (p[(size_t)k * m + i] * sigma[k]) * q[(size_t)k * n + j];
      a[(size_t)j * m + i] = acc;
    }
  free(p);
  free(q);
  return 0;
}
