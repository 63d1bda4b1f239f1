// Compares the restated log1p / log1pf (paper_1707_05141_b200/csrc/libm_log1p.h, the header the
// CUDA sampler uses) with the host C library, which is what numpy's ziggurat tail calls.
// Prints one line per check: "<name> <mismatches> <count>". Built and run by
// tests/test_libm_restatement.py (gcc, -ffp-contract=off: every op IEEE-rounded as on the device).
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "libm_log1p.h"

static uint64_t s_state = 88172645463325252ULL;
static uint64_t xr() {
  s_state ^= s_state << 13;
  s_state ^= s_state >> 7;
  s_state ^= s_state << 17;
  return s_state;
}

int main(int argc, char** argv) {
  long n_double = argc > 1 ? atol(argv[1]) : 2000000;
  long bad = 0, n = 0;
  // every argument the float tail can see: -next_float = -(k / 2^24)
  for (uint32_t k = 0; k < (1u << 24); ++k) {
    float x = -(float)k * (1.0f / 16777216.0f);
    float a = log1pf(x), b = bf_libm::log1p_f(x);
    bad += memcmp(&a, &b, 4) != 0;
    ++n;
  }
  printf("log1pf_tail_grid %ld %ld\n", bad, n);
  bad = n = 0;
  for (uint32_t w = 0; w < 0x7f800000u; w += 997) {  // strided sweep of all finite floats > -1
    for (int sg = 0; sg < 2; ++sg) {
      uint32_t ww = w | (sg ? 0x80000000u : 0u);
      float x;
      memcpy(&x, &ww, 4);
      if (!(x > -1.0f)) continue;
      float a = log1pf(x), b = bf_libm::log1p_f(x);
      bad += memcmp(&a, &b, 4) != 0;
      ++n;
    }
  }
  printf("log1pf_all_strided %ld %ld\n", bad, n);
  bad = n = 0;
  for (long i = 0; i < n_double; ++i) {  // the double tail's arguments: -next_double, 53-bit grid
    double x = -(double)(xr() >> 11) * (1.0 / 9007199254740992.0);
    double a = log1p(x), b = bf_libm::log1p_d(x);
    bad += memcmp(&a, &b, 8) != 0;
    ++n;
  }
  printf("log1p_tail_random %ld %ld\n", bad, n);
  bad = n = 0;
  for (long i = 0; i < n_double; ++i) {  // arbitrary finite doubles > -1 (all fdlibm branches)
    uint64_t r = xr();
    double x;
    memcpy(&x, &r, 8);
    if (!(x > -1.0) || isinf(x)) continue;
    double a = log1p(x), b = bf_libm::log1p_d(x);
    bad += memcmp(&a, &b, 8) != 0;
    ++n;
  }
  printf("log1p_all_random %ld %ld\n", bad, n);
  return 0;
}
