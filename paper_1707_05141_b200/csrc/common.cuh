// Shared device helpers for the batched factorisation kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

#define BF_DEV __device__ __forceinline__

namespace bf {

constexpr unsigned FULL = 0xffffffffu;

BF_DEV double shfl_xor(double v, int m) { return __shfl_xor_sync(FULL, v, m); }
BF_DEV float shfl_xor(float v, int m) { return __shfl_xor_sync(FULL, v, m); }

template <typename T>
BF_DEV T warp_allreduce_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += shfl_xor(v, o);
  return v;
}

template <typename T>
BF_DEV T warp_allreduce_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = shfl_xor(v, o);
    v = w > v ? w : v;
  }
  return v;
}

// Fast reciprocal / reciprocal square root: MUFU seed, one third-order correction and one Newton
// step (<= ~1 ulp; the final step's quadratic error term is far below an ulp, so only the
// round-to-nearest errors of the last operations remain). Only used on arguments in the normal
// range (callers fall back otherwise).
BF_DEV double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, fma(e, e, e), r);  // r (1 + e + e^2): error O(e^3)
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

BF_DEV double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // e = 1 - x y^2; y (1 + e/2 + 3 e^2 / 8) has error O(e^3)
  double e = fma(-x * y, y, 1.0);
  y = fma(y * e, fma(e, 0.375, 0.5), y);
  // Newton: y (1 + e/2)
  e = fma(-x * y, y, 1.0);
  return fma(y * 0.5, e, y);
}

// householder_vector's scalars (qr.py:26-48) on the fast reciprocal paths:
// beta = -copysign(hypot(alpha, sqrt(tail_sq)), alpha), tau = (beta - alpha) / beta, and
// 1 / (alpha - beta) for v = x / (alpha - beta); IEEE fallback outside [1e-150, 1e150].
BF_DEV void householder_scalars(double alpha, double tail_sq, double& beta, double& tau, double& denom,
                                double& rden) {
  const double q = fma(alpha, alpha, tail_sq);
  if (q > 1e-300 && q < 1e300) {
    const double h = q * rsqrt_fast(q);  // hypot(alpha, ||tail||)
    beta = -copysign(h, alpha);
    denom = alpha - beta;
    const double rb = rcp_fast(beta);
    const double tq = (beta - alpha) * rb;  // (beta - alpha) / beta, one Newton correction:
    tau = fma(fma(-tq, beta, beta - alpha), rb, tq);
    rden = rcp_fast(denom);
  } else {
    beta = -copysign(hypot(alpha, sqrt(tail_sq)), alpha);
    tau = (beta - alpha) / beta;
    denom = alpha - beta;
    rden = 1.0 / denom;
  }
}
// x / d from a reciprocal r ~ 1/d with one Newton correction of the quotient (<= 1 ulp).
BF_DEV double div_by(double x, double d, double r) {
  const double q = x * r;
  return fma(fma(-q, d, x), r, q);
}

// Norm-preserving cosine: given c0 ~ 1/sqrt(1 + t^2) (within a few ulp) and the tangent t that
// the caller applies (s = c t), return c with c^2 (1 + t^2) = 1 to second order: the residual
// rho = 1 - c0^2 - (c0 t)^2 is formed with FMAs (exact products) and c = c0 (1 + rho / 2).
// Without it, c = dd / hypot(dd, den) rounds independently of t and the rotations shrank the V
// columns on average (mean ||v_j||^2 - 1 of -1.9e-15 at 64 x 64 vs the reference's +1.7e-16;
// x56 V_R products in the block method). With it the drift is gone and ||V^T V - I|| falls below
// the reference's (whose c = 1 / hypot(1, t) is exactly 1 for |t| < 1e-8, an expansion).
BF_DEV double unit_cos(double c0, double t) {
  const double s0 = c0 * t;
  const double rho = fma(-s0, s0, fma(-c0, c0, 1.0));
  return fma(c0 * 0.5, rho, c0);
}

// Rutishauser rotation returning t as well (jacobi.py:68-80), g_pq != 0:
//   zeta = (g_qq - g_pp) / (2 g_pq), t = sign(zeta) / (|zeta| + hypot(1, zeta)),
//   c = 1 / hypot(1, t), s = c t.
// Evaluated without forming zeta: with den = 2 g_pq, diff = g_qq - g_pp and
// h = hypot(diff, den), dd = |diff| + h:  t = sign(zeta) |den| / dd,
// c = dd / hypot(dd, den), s = sign(zeta) |den| / hypot(dd, den) -- the same quantities
// multiplied through by |den|, which leaves two independent reciprocal chains (t and c, s)
// after h instead of four dependent ones. Exact IEEE fallback outside [1e-150, 1e150].
BF_DEV void jacobi_rotation_t(double gpp, double gpq, double gqq, double& c, double& s, double& t) {
  const double den = 2.0 * gpq, diff = gqq - gpp;
  const double aden = fabs(den), adiff = fabs(diff);
  const double big = aden > adiff ? aden : adiff;
  if (big > 1e-150 && big < 1e150) {
    // sign(zeta): zeta = diff / den carries the xor of both sign bits (signed zeros included)
    const unsigned long long sb =
        (unsigned long long)(__double_as_longlong(diff) ^ __double_as_longlong(den)) & 0x8000000000000000ULL;
    const double sden = __longlong_as_double(__double_as_longlong(aden) | (long long)sb);
    const double q = fma(diff, diff, den * den);
    const double h = q * rsqrt_fast(q);  // hypot(diff, den)
    const double dd = adiff + h;
    const double q2 = fma(dd, dd, den * den);
    const double r2 = rsqrt_fast(q2);  // 1 / hypot(dd, den)
    t = sden * rcp_fast(dd);
    c = unit_cos(dd * r2, t);
    s = c * t;
  } else {
    const double zeta = diff / den;
    t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
    c = 1.0 / hypot(1.0, t);
    s = c * t;
  }
}

// Rutishauser rotation (jacobi.py:68-80) for g_pq != 0:
//   zeta = (g_qq - g_pp) / (2 g_pq); t = sign(zeta) / (|zeta| + hypot(1, zeta));
//   c = 1 / hypot(1, t); s = c t.
// Fast path with MUFU+Newton reciprocals; exact IEEE path for extreme ranges.
BF_DEV void jacobi_rotation(double gpp, double gpq, double gqq, double& c, double& s) {
  double den = 2.0 * gpq;
  double diff = gqq - gpp;
  double aden = fabs(den);
  if (aden > 1e-290 && aden < 1e290 && fabs(diff) < 1e290) {
    double zeta = diff * rcp_fast(den);
    double az = fabs(zeta);
    double t;
    if (az < 1e150) {
      double x = fma(az, az, 1.0);
      double ry = rsqrt_fast(x);
      double h = x * ry;  // sqrt(1 + zeta^2)
      t = copysign(rcp_fast(az + h), zeta);
    } else {
      t = copysign(0.5 / az, zeta);  // az + hypot(1, az) == 2 az in double
    }
    c = unit_cos(rsqrt_fast(fma(t, t, 1.0)), t);
    s = c * t;
  } else {
    double zeta = diff / den;
    double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
    c = 1.0 / hypot(1.0, t);
    s = c * t;
  }
}

// Pair k of step st of the round-robin (circle method) schedule over nw columns
// (jacobi.py:102-115): idx_t[0] = 0, idx_t[j] = 1 + ((j - 1 - t) mod (nw - 1)),
// pair k = (idx_t[k], idx_t[nw-1-k]) normalised so p < q.
BF_DEV void rr_pair(int nw, int st, int k, int& p, int& q) {
  // circle method positions without integer division: 0 <= st < L, so both offsets lie in [-L, L)
  const int L = nw - 1;
  int x = k - 1 - st;
  x += x < 0 ? L : 0;
  const int a = (k == 0) ? 0 : 1 + x;
  int y = (nw - 1 - k) - 1 - st;
  y += y < 0 ? L : 0;
  const int b = 1 + y;
  p = a < b ? a : b;
  q = a < b ? b : a;
}

// Serial (row-cyclic) ordering executed as its anti-diagonal wavefront: step s
// (1 <= s <= 2nw-3) holds the disjoint pairs (p, s-p), p < s-p. Ordering pairs by
// p+q respects every column dependency of the serial sweep (jacobi.py:127-129), so
// the result is the serial sweep's, operation for operation.
BF_DEV int wf_count(int nw, int s) {
  int lo = s - (nw - 1);
  lo = lo < 0 ? 0 : lo;
  int hi = (s - 1) >> 1;
  return hi >= lo ? hi - lo + 1 : 0;
}
BF_DEV void wf_pair(int nw, int s, int k, int& p, int& q) {
  int lo = s - (nw - 1);
  lo = lo < 0 ? 0 : lo;
  p = lo + k;
  q = s - p;
}

}  // namespace bf
