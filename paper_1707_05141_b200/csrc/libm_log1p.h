// log1p / log1pf restated operation-for-operation from the algorithm the host libm uses
// (glibc 2.39 sysdeps/ieee754/dbl-64/s_log1p.c and flt-32/s_log1pf.c, both the Sun fdlibm
// log1p: argument reduction 1+x = 2^k (1+f), correction term c, s = f/(2+f), and the
// degree-7 odd polynomial in s^2).
//
// Why restated and not CUDA's log1p: numpy's ziggurat tail returns r + (-log1p(-U)/r)
// directly (numpy random_standard_normal / _f, see util_kernels.cu), so the sample is
// bitwise numpy's only if log1p is bitwise the host's. CUDA's log1p/log1pf are different
// (still ~1 ulp) polynomials. Every operation here is one IEEE-rounded op (explicit _rn
// intrinsics on the device: no FMA contraction, matching the SSE2 build of glibc), so the
// device result equals the host libm's for every input -- checked exhaustively for the
// 2^24 float tail arguments and on 2e7 + structured double arguments against the host
// libm by tests/test_libm_restatement.py (which compiles this same header with gcc).
//
// Usable from C++ (host, gcc -ffp-contract=off) and CUDA (device).
#pragma once
#include <stdint.h>
#include <string.h>
#if !defined(__CUDA_ARCH__)
#include <math.h>
#endif

#if defined(__CUDACC__)
#define BF_LM_FN __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define BF_LM_DADD(a, b) __dadd_rn((a), (b))
#define BF_LM_DSUB(a, b) __dsub_rn((a), (b))
#define BF_LM_DMUL(a, b) __dmul_rn((a), (b))
#define BF_LM_DDIV(a, b) __ddiv_rn((a), (b))
#define BF_LM_DFMA(a, b, c) __fma_rn((a), (b), (c))
#define BF_LM_FADD(a, b) __fadd_rn((a), (b))
#define BF_LM_FSUB(a, b) __fsub_rn((a), (b))
#define BF_LM_FMUL(a, b) __fmul_rn((a), (b))
#define BF_LM_FDIV(a, b) __fdiv_rn((a), (b))
#endif
#else
#define BF_LM_FN static inline
#endif
#ifndef BF_LM_DADD
#define BF_LM_DADD(a, b) ((a) + (b))
#define BF_LM_DSUB(a, b) ((a) - (b))
#define BF_LM_DMUL(a, b) ((a) * (b))
#define BF_LM_DDIV(a, b) ((a) / (b))
#define BF_LM_DFMA(a, b, c) fma((a), (b), (c))
#define BF_LM_FADD(a, b) ((a) + (b))
#define BF_LM_FSUB(a, b) ((a) - (b))
#define BF_LM_FMUL(a, b) ((a) * (b))
#define BF_LM_FDIV(a, b) ((a) / (b))
#endif

namespace bf_libm {

BF_LM_FN int32_t hi_word(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return (int32_t)(u >> 32);
}
BF_LM_FN double with_hi_word(double x, int32_t hi) {
  uint64_t u;
  memcpy(&u, &x, 8);
  u = (u & 0xffffffffULL) | ((uint64_t)(uint32_t)hi << 32);
  double r;
  memcpy(&r, &u, 8);
  return r;
}
BF_LM_FN int32_t f_word(float x) {
  int32_t u;
  memcpy(&u, &x, 4);
  return u;
}
BF_LM_FN float f_from_word(int32_t u) {
  float r;
  memcpy(&r, &u, 4);
  return r;
}

// double log1p, as glibc's FMA build computes it (the ifunc variant selected on every AVX2+FMA
// host -- what numpy calls there): the fdlibm algorithm with a*b+c contracted at the places the
// compiled code contracts them, and the polynomial in glibc's split form
// R = z6 R4 + (z4 R3 + (z Lp1 + z2 R2)), R2 = Lp2 + z Lp3, R3 = Lp4 + z Lp5, R4 = Lp6 + z Lp7.
// Domain used by the sampler: x in (-1, 0]; the full case split is kept.
BF_LM_FN double log1p_d(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  double f = 0.0, c = 0.0, u;
  int32_t k = 1, hu = 0;
  const int32_t hx = hi_word(x), ax = hx & 0x7fffffff;
  if (hx < 0x3FDA827A) {  // x < 0.41422
    if (ax >= 0x3ff00000) {  // x <= -1
      if (x == -1.0) return -1.0 / 0.0;
      return (x - x) / (x - x);
    }
    if (ax < 0x3e200000) {  // |x| < 2^-29
      if (ax < 0x3c900000) return x;
      return BF_LM_DFMA(-BF_LM_DMUL(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return BF_LM_DADD(x, x);
  }
  if (k != 0) {
    if (hx < 0x43400000) {
      u = BF_LM_DADD(1.0, x);
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? BF_LM_DSUB(1.0, BF_LM_DSUB(u, x)) : BF_LM_DSUB(x, BF_LM_DSUB(u, 1.0));
      c = BF_LM_DDIV(c, u);
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, hu | 0x3ff00000);  // normalize u
    } else {
      k += 1;
      u = with_hi_word(u, hu | 0x3fe00000);  // normalize u/2
      hu = (0x00100000 - hu) >> 2;
    }
    f = BF_LM_DSUB(u, 1.0);
  }
  const double hfsq = BF_LM_DMUL(BF_LM_DMUL(f, 0.5), f);
  const double dk = (double)k;
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = BF_LM_DFMA(dk, ln2_lo, c);
      return BF_LM_DFMA(dk, ln2_hi, c);
    }
    const double R = BF_LM_DMUL(BF_LM_DFMA(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return BF_LM_DSUB(f, R);
    return BF_LM_DFMA(dk, ln2_hi, -BF_LM_DSUB(BF_LM_DSUB(R, BF_LM_DFMA(dk, ln2_lo, c)), f));
  }
  const double s = BF_LM_DDIV(f, BF_LM_DADD(f, 2.0));
  const double z = BF_LM_DMUL(s, s);
  const double R2 = BF_LM_DFMA(z, Lp3, Lp2), R3 = BF_LM_DFMA(z, Lp5, Lp4), R4 = BF_LM_DFMA(z, Lp7, Lp6);
  const double z2 = BF_LM_DMUL(z, z), z4 = BF_LM_DMUL(z2, z2), z6 = BF_LM_DMUL(z2, z4);
  const double R = BF_LM_DFMA(z6, R4, BF_LM_DFMA(z4, R3, BF_LM_DFMA(z, Lp1, BF_LM_DMUL(z2, R2))));
  const double sr = BF_LM_DMUL(BF_LM_DADD(R, hfsq), s);
  if (k == 0) return BF_LM_DSUB(f, BF_LM_DSUB(hfsq, sr));
  return BF_LM_DFMA(dk, ln2_hi, -BF_LM_DSUB(BF_LM_DSUB(hfsq, BF_LM_DADD(BF_LM_DFMA(dk, ln2_lo, c), sr)), f));
}

// float log1pf (same algorithm in single precision).
BF_LM_FN float log1p_f(float x) {
  const float ln2_hi = 6.9313812256e-01f, ln2_lo = 9.0580006145e-06f;
  const float Lp1 = 6.6666668653e-01f, Lp2 = 4.0000000596e-01f, Lp3 = 2.8571429849e-01f, Lp4 = 2.2222198546e-01f,
              Lp5 = 1.8183572590e-01f, Lp6 = 1.5313838422e-01f, Lp7 = 1.4798198640e-01f;
  float f = 0.0f, c = 0.0f, u;
  int32_t k = 1, hu = 0;
  const int32_t hx = f_word(x), ax = hx & 0x7fffffff;
  if (hx < 0x3ed413d7) {  // x < 0.41422
    if (ax >= 0x3f800000) {
      if (x == -1.0f) return -1.0f / 0.0f;
      return (x - x) / (x - x);
    }
    if (ax < 0x31000000) {  // |x| < 2^-29
      if (ax < 0x24800000) return x;
      return BF_LM_FSUB(x, BF_LM_FMUL(BF_LM_FMUL(x, x), 0.5f));
    }
    if (hx > 0 || hx <= (int32_t)0xbe95f61f) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7f800000) {
    return BF_LM_FADD(x, x);
  }
  if (k != 0) {
    if (hx < 0x5a000000) {
      u = BF_LM_FADD(1.0f, x);
      hu = f_word(u);
      k = (hu >> 23) - 127;
      c = (k > 0) ? BF_LM_FSUB(1.0f, BF_LM_FSUB(u, x)) : BF_LM_FSUB(x, BF_LM_FSUB(u, 1.0f));
      c = BF_LM_FDIV(c, u);
    } else {
      u = x;
      hu = f_word(u);
      k = (hu >> 23) - 127;
      c = 0.0f;
    }
    hu &= 0x007fffff;
    if (hu < 0x3504f7) {
      u = f_from_word(hu | 0x3f800000);
    } else {
      k += 1;
      u = f_from_word(hu | 0x3f000000);
      hu = (0x00800000 - hu) >> 2;
    }
    f = BF_LM_FSUB(u, 1.0f);
  }
  const float hfsq = BF_LM_FMUL(BF_LM_FMUL(0.5f, f), f);
  const float fk = (float)k;
  if (hu == 0) {
    if (f == 0.0f) {
      if (k == 0) return 0.0f;
      c = BF_LM_FADD(c, BF_LM_FMUL(fk, ln2_lo));
      return BF_LM_FADD(BF_LM_FMUL(fk, ln2_hi), c);
    }
    const float R = BF_LM_FMUL(hfsq, BF_LM_FSUB(1.0f, BF_LM_FMUL(0.66666666666666666f, f)));
    if (k == 0) return BF_LM_FSUB(f, R);
    return BF_LM_FSUB(BF_LM_FMUL(fk, ln2_hi),
                      BF_LM_FSUB(BF_LM_FSUB(R, BF_LM_FADD(BF_LM_FMUL(fk, ln2_lo), c)), f));
  }
  const float s = BF_LM_FDIV(f, BF_LM_FADD(2.0f, f));
  const float z = BF_LM_FMUL(s, s);
  // Horner: z (Lp1 + z (Lp2 + z (Lp3 + z (Lp4 + z (Lp5 + z (Lp6 + z Lp7))))))
  float R = BF_LM_FADD(Lp6, BF_LM_FMUL(z, Lp7));
  R = BF_LM_FADD(Lp5, BF_LM_FMUL(z, R));
  R = BF_LM_FADD(Lp4, BF_LM_FMUL(z, R));
  R = BF_LM_FADD(Lp3, BF_LM_FMUL(z, R));
  R = BF_LM_FADD(Lp2, BF_LM_FMUL(z, R));
  R = BF_LM_FADD(Lp1, BF_LM_FMUL(z, R));
  R = BF_LM_FMUL(z, R);
  if (k == 0) return BF_LM_FSUB(f, BF_LM_FSUB(hfsq, BF_LM_FMUL(s, BF_LM_FADD(hfsq, R))));
  return BF_LM_FSUB(BF_LM_FMUL(fk, ln2_hi),
                    BF_LM_FSUB(BF_LM_FSUB(hfsq, BF_LM_FADD(BF_LM_FMUL(s, BF_LM_FADD(hfsq, R)),
                                                           BF_LM_FADD(BF_LM_FMUL(fk, ln2_lo), c))),
                               f));
}

}  // namespace bf_libm
