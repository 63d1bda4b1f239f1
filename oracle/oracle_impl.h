/* CPU oracle body, instantiated twice by oracle.c (T = double / float).
 *
 * TEST INFRASTRUCTURE ONLY -- see oracle.c's header. Every function restates the
 * reference algorithm (file:line cited) so the GPU path can be checked against it.
 * Layout: one column-major matrix (ld = rows). Scalars that the reference keeps
 * as Python floats (tau, beta, serial-ordering c/s) are double here too; array
 * arithmetic happens in T, as numpy does for a T array with a weak scalar.
 */

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define F(name) CAT(name, SUF)

/* dot product in T (BLAS xdot / einsum over a row) */
static T F(dot)(const T* x, const T* y, int n) {
  T s = 0;
  for (int i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

/* householder_vector (qr.py:26-48): v[0]=1, tau; beta = -copysign(hypot(alpha, ||tail||), alpha) */
static double F(householder)(const T* x, int len, T* v) {
  for (int i = 0; i < len; ++i) v[i] = x[i];
  v[0] = (T)1;
  double alpha = (double)x[0];
  if (len == 1) return 0.0;
  double tail_sq = (double)F(dot)(x + 1, x + 1, len - 1);
  if (tail_sq == 0.0) return 0.0;
  double beta = -copysign(hypot(alpha, sqrt(tail_sq)), alpha);
  double tau = (beta - alpha) / beta;
  T denom = (T)(alpha - beta);
  for (int i = 1; i < len; ++i) v[i] = x[i] / denom;
  return tau;
}

/* _apply_reflector (qr.py:51-60): block <- block - v (tau * v^T block), block is rows x cols, ld */
static void F(apply_reflector)(const T* v, double tau, T* block, int rows, int cols, int ld) {
  T tt = (T)tau;
  for (int c = 0; c < cols; ++c) {
    T* col = block + (size_t)c * ld;
    T w = F(dot)(v, col, rows);
    w *= tt;
    for (int i = 0; i < rows; ++i) col[i] -= v[i] * w;
  }
}

/* qr (qr.py:63-95): panel-ordered Householder, explicit reduced Q. q: m x n, r: n x n. */
static int F(qr)(int m, int n, const T* a, T* q, T* r_out, int pw, T* work /* m*n + m*n */) {
  if (m < n) return -1;
  if (pw < 1) return -2;
  T* r = work;                 /* m x n copy */
  T* vs = work + (size_t)m * n; /* reflectors: column j holds v_j in rows j.. */
  double* taus = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
  memcpy(r, a, sizeof(T) * (size_t)m * n);
  for (int p0 = 0; p0 < n; p0 += pw) {
    int p1 = p0 + pw < n ? p0 + pw : n;
    for (int j = p0; j < p1; ++j) {
      T* v = vs + (size_t)j * m + j;
      double tau = F(householder)(r + (size_t)j * m + j, m - j, v);
      taus[j] = tau;
      if (tau != 0.0) F(apply_reflector)(v, tau, r + (size_t)j * m + j, m - j, p1 - j, m);
      for (int i = j + 1; i < m; ++i) r[(size_t)j * m + i] = 0;
    }
    if (p1 < n) {
      for (int j = p0; j < p1; ++j)
        if (taus[j] != 0.0)
          F(apply_reflector)(vs + (size_t)j * m + j, taus[j], r + (size_t)p1 * m + j, m - j, n - p1, m);
    }
  }
  /* Q = H_0 ... H_{n-1} I, reflectors applied in reverse to q[j:, :] (qr.py:90-94) */
  memset(q, 0, sizeof(T) * (size_t)m * n);
  for (int i = 0; i < n; ++i) q[(size_t)i * m + i] = (T)1;
  for (int j = n - 1; j >= 0; --j)
    if (taus[j] != 0.0) F(apply_reflector)(vs + (size_t)j * m + j, taus[j], q + j, m - j, n, m);
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) r_out[(size_t)c * n + i] = r[(size_t)c * m + i];
  free(taus);
  return 0;
}

/* off_orthogonality (jacobi.py:83-99) on the columns of a (rows x cols, ld=rows) */
static double F(off_orthogonality)(const T* a, int rows, int cols) {
  if (cols < 2) return 0.0;
  T* d = (T*)malloc(sizeof(T) * cols);
  for (int j = 0; j < cols; ++j) {
    T g = F(dot)(a + (size_t)j * rows, a + (size_t)j * rows, rows);
    d[j] = (T)sqrt((double)(g < 0 ? -g : g));
  }
  T best = 0;
  for (int i = 0; i < cols; ++i)
    for (int j = 0; j < cols; ++j) {
      if (i == j) continue;
      T den = d[i] * d[j];
      if (!(den > 0)) continue;
      T g = F(dot)(a + (size_t)i * rows, a + (size_t)j * rows, rows);
      T rt = (g < 0 ? -g : g) / den;
      if (rt > best) best = rt;
    }
  free(d);
  return (double)best;
}

/* scaled_offdiag (blockjacobi.py:57-76) on a square g (n x n) */
static double F(scaled_offdiag)(const T* g, int n) {
  if (n < 2) return 0.0;
  double best = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      if (i == j) continue;
      T di = (T)sqrt((double)fabs((double)g[(size_t)i * n + i]));
      T dj = (T)sqrt((double)fabs((double)g[(size_t)j * n + j]));
      T den = di * dj;
      T num = g[(size_t)j * n + i];
      num = num < 0 ? -num : num;
      double rt;
      if (den > 0)
        rt = (double)(num / den);
      else
        rt = num > 0 ? INFINITY : 0.0;
      if (rt > best) best = rt;
    }
  return best;
}

/* _serial_sweep (jacobi.py:118-155). wt: nw rows of length m (row-major = A columns).
 * vt: nw x nw row-major or NULL. Returns the rotation count. */
static long F(serial_sweep)(T* wt, int nw, int m, T* vt, double tol2) {
  long rot = 0;
  for (int p = 0; p < nw - 1; ++p) {
    T* wp = wt + (size_t)p * m;
    for (int q = p + 1; q < nw; ++q) {
      T* wq = wt + (size_t)q * m;
      double gpp = (double)F(dot)(wp, wp, m);
      double gpq = (double)F(dot)(wp, wq, m);
      double gqq = (double)F(dot)(wq, wq, m);
      if (gpq * gpq <= tol2 * (gpp * gqq)) continue;
      double c, s;
      orc_jacobi_rotation(gpp, gpq, gqq, &c, &s);
      T ct = (T)c, st = (T)s;
      for (int i = 0; i < m; ++i) {
        T bp = wp[i] * ct, bq = wq[i] * st;
        T np_ = bp - bq;
        T a2 = wp[i] * st;
        T nq = wq[i] * ct;
        nq += a2;
        wp[i] = np_;
        wq[i] = nq;
      }
      if (vt) {
        T* vp = vt + (size_t)p * nw;
        T* vq = vt + (size_t)q * nw;
        for (int i = 0; i < nw; ++i) {
          T bp = vp[i] * ct, bq = vq[i] * st;
          T np_ = bp - bq;
          T a2 = vp[i] * st;
          T nq = vq[i] * ct;
          nq += a2;
          vp[i] = np_;
          vq[i] = nq;
        }
      }
      ++rot;
    }
  }
  return rot;
}

/* _round_robin_sweep (jacobi.py:158-186): all pairs of a step read the pre-step columns */
static long F(rr_sweep)(T* wt, int nw, int m, T* vt, double tol2, const int* sched /* (nw-1) x nw/2 x 2 */) {
  long rot = 0;
  int half = nw / 2;
  T tol2t = (T)tol2;
  for (int st = 0; st < nw - 1; ++st) {
    const int* pr = sched + (size_t)st * half * 2;
    for (int k = 0; k < half; ++k) {
      int p = pr[2 * k], q = pr[2 * k + 1];
      T* wp = wt + (size_t)p * m;
      T* wq = wt + (size_t)q * m;
      T gpp = F(dot)(wp, wp, m), gpq = F(dot)(wp, wq, m), gqq = F(dot)(wq, wq, m);
      if (!(gpq * gpq > tol2t * (gpp * gqq))) continue;
      ++rot;
      T den = (T)2 * gpq;
      T zeta = (gqq - gpp) / den;
      T t = (T)copysign(1.0, (double)zeta) / ((zeta < 0 ? -zeta : zeta) + (T)hypot(1.0, (double)zeta));
      T c = (T)1 / (T)hypot(1.0, (double)t);
      T s = c * t;
      for (int i = 0; i < m; ++i) {
        T a0 = wp[i], b0 = wq[i];
        wp[i] = c * a0 - s * b0;
        wq[i] = s * a0 + c * b0;
      }
      if (vt) {
        T* vp = vt + (size_t)p * nw;
        T* vq = vt + (size_t)q * nw;
        for (int i = 0; i < nw; ++i) {
          T a0 = vp[i], b0 = vq[i];
          vp[i] = c * a0 - s * b0;
          vq[i] = s * a0 + c * b0;
        }
      }
    }
  }
  return rot;
}

/* _complete_zero_rows (jacobi.py:189-209): ut is n x m row-major, zero rows listed in order */
static void F(complete_zero_rows)(T* ut, int n, int m, const int* zero, int nz) {
  int* done = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  int nd = 0;
  for (int i = 0; i < n; ++i) {
    int isz = 0;
    for (int k = 0; k < nz; ++k) isz |= (zero[k] == i);
    if (!isz) done[nd++] = i;
  }
  T* cand = (T*)malloc(sizeof(T) * m);
  T* best = (T*)malloc(sizeof(T) * m);
  for (int z = 0; z < nz; ++z) {
    double best_norm = -1.0;
    for (int j = 0; j < m; ++j) {
      for (int i = 0; i < m; ++i) cand[i] = 0;
      cand[j] = 1;
      for (int d = 0; d < nd; ++d) {
        const T* row = ut + (size_t)done[d] * m;
        T pr = F(dot)(row, cand, m);
        for (int i = 0; i < m; ++i) cand[i] -= row[i] * pr;
      }
      double nrm = sqrt((double)F(dot)(cand, cand, m));
      if (nrm > best_norm) {
        best_norm = nrm;
        memcpy(best, cand, sizeof(T) * m);
      }
    }
    for (int d = 0; d < nd; ++d) {
      const T* row = ut + (size_t)done[d] * m;
      T pr = F(dot)(row, best, m);
      for (int i = 0; i < m; ++i) best[i] -= row[i] * pr;
    }
    T nb = (T)sqrt((double)F(dot)(best, best, m));
    T* dst = ut + (size_t)zero[z] * m;
    for (int i = 0; i < m; ++i) dst[i] = best[i] / nb;
    done[nd++] = zero[z];
  }
  free(done);
  free(cand);
  free(best);
}

/* _extract_svd (jacobi.py:212-228): sigma = row norms of wt[:n], stable descending sort.
 * u: m x n col-major, s: n, v: n x n col-major (from vt rows, nw stride) or NULL. */
static void F(extract_svd)(const T* wt, int n, int m, const T* vt, int nw, T* u, T* s, T* v) {
  T* norms = (T*)malloc(sizeof(T) * (n > 0 ? n : 1));
  int* order = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  for (int j = 0; j < n; ++j) norms[j] = (T)sqrt((double)F(dot)(wt + (size_t)j * m, wt + (size_t)j * m, m));
  /* stable argsort of -norms: rank = #greater + #equal-before */
  for (int j = 0; j < n; ++j) {
    int rank = 0;
    for (int i = 0; i < n; ++i)
      if (norms[i] > norms[j] || (norms[i] == norms[j] && i < j)) ++rank;
    order[rank] = j;
  }
  int* zero = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
  int nz = 0;
  for (int r = 0; r < n; ++r) {
    int j = order[r];
    T sg = norms[j];
    s[r] = sg;
    for (int i = 0; i < m; ++i) u[(size_t)r * m + i] = wt[(size_t)j * m + i];
    if (sg > 0) {
      for (int i = 0; i < m; ++i) u[(size_t)r * m + i] /= sg;
    } else {
      zero[nz++] = r;
    }
  }
  /* u column r == ut row r, so the completion runs directly on u's columns */
  if (nz) F(complete_zero_rows)(u, n, m, zero, nz);
  if (v && vt) {
    for (int r = 0; r < n; ++r) {
      int j = order[r];
      for (int i = 0; i < n; ++i) v[(size_t)r * n + i] = vt[(size_t)j * nw + i];
    }
  }
  free(norms);
  free(order);
  free(zero);
}

/* svd (jacobi.py:231-284) */
static int F(svd)(int m, int n, const T* a, T* u, T* s, T* v, int* sweeps_out, int* conv_out, long* rot_out,
                  double tol, int max_sweeps, int ordering) {
  if (m < n) return -1;
  if (max_sweeps < 1) return -2;
  if (n == 0) {
    *sweeps_out = 0;
    *conv_out = 1;
    if (rot_out) *rot_out = 0;
    return 0;
  }
  double tol2 = tol * tol;
  int pad = (ordering == 1) && (n % 2 == 1);
  int nw = pad ? n + 1 : n;
  T* wt = (T*)calloc((size_t)nw * m, sizeof(T));
  memcpy(wt, a, sizeof(T) * (size_t)m * n); /* column j of a == row j of wt */
  T* vt = NULL;
  if (v) {
    vt = (T*)calloc((size_t)nw * nw, sizeof(T));
    for (int i = 0; i < nw; ++i) vt[(size_t)i * nw + i] = (T)1;
  }
  int* sched = NULL;
  if (ordering == 1 && nw >= 2) {
    sched = (int*)malloc(sizeof(int) * (size_t)(nw - 1) * nw);
    orc_round_robin_schedule(nw, sched);
  }
  int converged = n < 2;
  int sweeps = 0;
  long total = 0;
  for (int it = 0; it < max_sweeps; ++it) {
    if (converged) break;
    long r = ordering == 0 ? F(serial_sweep)(wt, nw, m, vt, tol2) : F(rr_sweep)(wt, nw, m, vt, tol2, sched);
    total += r;
    ++sweeps;
    if (r == 0) converged = 1;
  }
  if (!converged) converged = F(off_orthogonality)(wt, m, nw) < tol;
  F(extract_svd)(wt, n, m, vt, nw, u, s, v);
  *sweeps_out = sweeps;
  *conv_out = converged;
  if (rot_out) *rot_out = total;
  free(wt);
  free(vt);
  free(sched);
  return 0;
}

/* plain GEMM C (M x N) = A (M x K) * B (K x N), all column-major */
static void F(gemm_nn)(int M, int N, int K, const T* A, int lda, const T* B, int ldb, T* C, int ldc) {
  for (int j = 0; j < N; ++j) {
    T* c = C + (size_t)j * ldc;
    for (int i = 0; i < M; ++i) c[i] = 0;
    for (int k = 0; k < K; ++k) {
      T b = B[(size_t)j * ldb + k];
      const T* a = A + (size_t)k * lda;
      for (int i = 0; i < M; ++i) c[i] += a[i] * b;
    }
  }
}

/* syrk (core.py:68-78): G = A^T A, exactly symmetric */
static void F(syrk)(int m, int k, const T* a, T* g) {
  for (int j = 0; j < k; ++j)
    for (int i = 0; i <= j; ++i) {
      T d = F(dot)(a + (size_t)i * m, a + (size_t)j * m, m);
      g[(size_t)j * k + i] = d;
      g[(size_t)i * k + j] = d;
    }
}

/* block_svd (blockjacobi.py:84-168). method 0 = gram, 1 = direct. e_hist holds max_sweeps slots. */
static int F(block_svd)(int m, int n, const T* a, T* u, T* s, T* v, int* sweeps_out, int* conv_out, T* e_hist,
                        int bw, int method, double tol, int max_sweeps) {
  if (m < n) return -1;
  if (bw < 1 || max_sweeps < 1) return -2;
  int k = bw;
  if (method == 1) {
    k = m / 2 < k ? m / 2 : k;
    if (k < 1) k = 1;
  }
  int two_k = 2 * k;
  int n_pad = ((n + two_k - 1) / two_k) * two_k;
  if (n_pad < two_k) n_pad = two_k;
  T* w = (T*)calloc((size_t)m * n_pad, sizeof(T));
  memcpy(w, a, sizeof(T) * (size_t)m * n);
  T* vv = NULL;
  if (v) {
    vv = (T*)calloc((size_t)n_pad * n_pad, sizeof(T));
    for (int i = 0; i < n_pad; ++i) vv[(size_t)i * n_pad + i] = (T)1;
  }
  int n_blocks = n_pad / k;
  int* sched = (int*)malloc(sizeof(int) * (size_t)(n_blocks - 1) * n_blocks);
  orc_round_robin_schedule(n_blocks, sched);
  int n_pairs = (n_blocks - 1) * (n_blocks / 2);
  T* pair = (T*)malloc(sizeof(T) * (size_t)m * two_k);
  T* npair = (T*)malloc(sizeof(T) * (size_t)m * two_k);
  T* g = (T*)malloc(sizeof(T) * (size_t)two_k * two_k);
  T* iu = (T*)malloc(sizeof(T) * (size_t)(m > two_k ? m : two_k) * two_k);
  T* is = (T*)malloc(sizeof(T) * two_k);
  T* iv = (T*)malloc(sizeof(T) * (size_t)two_k * two_k);
  T* fq = (T*)malloc(sizeof(T) * (size_t)m * two_k);
  T* fr = (T*)malloc(sizeof(T) * (size_t)two_k * two_k);
  T* work = (T*)malloc(sizeof(T) * (size_t)2 * m * two_k);
  T* vpair = vv ? (T*)malloc(sizeof(T) * (size_t)n_pad * two_k) : NULL;
  T* nvpair = vv ? (T*)malloc(sizeof(T) * (size_t)n_pad * two_k) : NULL;
  int converged = 0, sweeps = 0;
  for (int it = 0; it < max_sweeps; ++it) {
    double e_sweep = 0.0;
    for (int pi = 0; pi < n_pairs; ++pi) {
      int bi = sched[2 * pi], bj = sched[2 * pi + 1];
      memcpy(pair, w + (size_t)bi * k * m, sizeof(T) * (size_t)m * k);
      memcpy(pair + (size_t)k * m, w + (size_t)bj * k * m, sizeof(T) * (size_t)m * k);
      const T* rot;
      if (method == 0) {
        F(syrk)(m, two_k, pair, g);
        double e = F(scaled_offdiag)(g, two_k);
        if (e > e_sweep) e_sweep = e;
        if (e <= tol) continue;
        int sw, cv;
        F(svd)(two_k, two_k, g, iu, is, NULL, &sw, &cv, NULL, orc_default_tol(sizeof(T)), 30, 1);
        F(gemm_nn)(m, two_k, two_k, pair, m, iu, two_k, npair, m);
        for (int j = 0; j < two_k; ++j)
          if (is[j] == 0)
            for (int i = 0; i < m; ++i) npair[(size_t)j * m + i] = 0;
        rot = iu;
      } else {
        F(qr)(m, two_k, pair, fq, fr, 16, work);
        double e = F(scaled_offdiag)(fr, two_k);
        if (e > e_sweep) e_sweep = e;
        if (e <= tol) continue;
        int sw, cv;
        F(svd)(two_k, two_k, fr, iu, is, iv, &sw, &cv, NULL, orc_default_tol(sizeof(T)), 30, 1);
        F(gemm_nn)(m, two_k, two_k, fq, m, iu, two_k, npair, m);
        for (int j = 0; j < two_k; ++j)
          for (int i = 0; i < m; ++i) npair[(size_t)j * m + i] *= is[j];
        rot = iv;
      }
      memcpy(w + (size_t)bi * k * m, npair, sizeof(T) * (size_t)m * k);
      memcpy(w + (size_t)bj * k * m, npair + (size_t)k * m, sizeof(T) * (size_t)m * k);
      if (vv) {
        memcpy(vpair, vv + (size_t)bi * k * n_pad, sizeof(T) * (size_t)n_pad * k);
        memcpy(vpair + (size_t)k * n_pad, vv + (size_t)bj * k * n_pad, sizeof(T) * (size_t)n_pad * k);
        F(gemm_nn)(n_pad, two_k, two_k, vpair, n_pad, rot, two_k, nvpair, n_pad);
        memcpy(vv + (size_t)bi * k * n_pad, nvpair, sizeof(T) * (size_t)n_pad * k);
        memcpy(vv + (size_t)bj * k * n_pad, nvpair + (size_t)k * n_pad, sizeof(T) * (size_t)n_pad * k);
      }
    }
    if (e_hist) e_hist[sweeps] = (T)e_sweep;
    ++sweeps;
    if (e_sweep < tol) {
      converged = 1;
      break;
    }
  }
  /* _extract_svd on the padded W (columns of w == rows of wt), then drop the padding */
  T* uu = (T*)malloc(sizeof(T) * (size_t)m * n_pad);
  T* ss = (T*)malloc(sizeof(T) * n_pad);
  T* vo = vv ? (T*)malloc(sizeof(T) * (size_t)n_pad * n_pad) : NULL;
  F(extract_svd)(w, n_pad, m, vv, n_pad, uu, ss, vo);
  for (int j = 0; j < n; ++j) {
    s[j] = ss[j];
    memcpy(u + (size_t)j * m, uu + (size_t)j * m, sizeof(T) * m);
    if (v)
      for (int i = 0; i < n; ++i) v[(size_t)j * n + i] = vo[(size_t)j * n_pad + i];
  }
  *sweeps_out = sweeps;
  *conv_out = converged;
  free(w); free(vv); free(sched); free(pair); free(npair); free(g); free(iu); free(is); free(iv);
  free(fq); free(fr); free(work); free(vpair); free(nvpair); free(uu); free(ss); free(vo);
  return 0;
}

/* rsvd (rsvd.py:56-76). omega: n x w col-major (NULL -> drawn with gaussian_matrix(n, w, seed)). */
static int F(rsvd)(int m, int n, int kk, int p, uint64_t seed_lo, uint64_t seed_hi, const T* a, const T* omega_in,
                   T* u, T* s, T* v) {
  int w = kk + p;
  if (w > (m < n ? m : n) || kk < 1 || p < 0) return -1;
  T* omega = (T*)malloc(sizeof(T) * (size_t)n * w);
  if (omega_in) {
    memcpy(omega, omega_in, sizeof(T) * (size_t)n * w);
  } else {
    /* the reference draws omega in the input's dtype (rsvd.py:65): float32 is its own stream */
    if (sizeof(T) == sizeof(double))
      orc_gaussian_f64(n, w, seed_lo, seed_hi, (double*)omega);
    else
      orc_gaussian_f32(n, w, seed_lo, seed_hi, (float*)omega);
  }
  T* y = (T*)malloc(sizeof(T) * (size_t)m * w);
  F(gemm_nn)(m, w, n, a, m, omega, n, y, m);
  T* q = (T*)malloc(sizeof(T) * (size_t)m * w);
  T* r = (T*)malloc(sizeof(T) * (size_t)w * w);
  T* work = (T*)malloc(sizeof(T) * (size_t)2 * (m > n ? m : n) * w);
  F(qr)(m, w, y, q, r, 16, work);
  /* B^T = A^T Q  (n x w); B = Q^T A */
  T* bt = (T*)malloc(sizeof(T) * (size_t)n * w);
  for (int j = 0; j < w; ++j)
    for (int i = 0; i < n; ++i) bt[(size_t)j * n + i] = F(dot)(a + (size_t)i * m, q + (size_t)j * m, m);
  T* qb = (T*)malloc(sizeof(T) * (size_t)n * w);
  T* rb = (T*)malloc(sizeof(T) * (size_t)w * w);
  F(qr)(n, w, bt, qb, rb, 16, work);
  T* rbt = (T*)malloc(sizeof(T) * (size_t)w * w);
  for (int j = 0; j < w; ++j)
    for (int i = 0; i < w; ++i) rbt[(size_t)j * w + i] = rb[(size_t)i * w + j];
  T* iu = (T*)malloc(sizeof(T) * (size_t)w * w);
  T* iv = (T*)malloc(sizeof(T) * (size_t)w * w);
  int sw, cv;
  F(svd)(w, w, rbt, iu, s, iv, &sw, &cv, NULL, orc_default_tol(sizeof(T)), 30, 1);
  F(gemm_nn)(m, w, w, q, m, iu, w, u, m);
  F(gemm_nn)(n, w, w, qb, n, iv, w, v, n);
  free(omega); free(y); free(q); free(r); free(work); free(bt); free(qb); free(rb); free(rbt); free(iu); free(iv);
  return 0;
}

#undef F
#undef CAT
#undef CAT2
