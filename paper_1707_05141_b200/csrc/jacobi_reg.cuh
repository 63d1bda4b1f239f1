// Register-resident one-sided Jacobi sweeps (the paper's register tier, PAPER.md:163-191,
// generalised to n <= 64 and m <= 32*WW through warps of rows).
//
// Layout: lane = row; each thread holds its row of W (NP column slots) in registers.
// Orderings are realised with a FIXED slot structure so every register index is a
// compile-time constant:
//  * round_robin (jacobi.py:102-115): slot k pairs logical positions (k, NP-1-k); after each
//    step positions 1..NP-1 rotate one place -- exactly the reference's
//    `idx = [idx0, idx[-1]] + idx[1:-1]`. NP must equal the working width nw.
//  * serial (jacobi.py:118-155): executed as its p+q wavefront (each step the disjoint pairs
//    (p, s-p); ordering pairs by p+q respects every column dependency of the row-cyclic sweep,
//    so the rotation sequence seen by each column is the serial sweep's). Columns sit on a ring
//    of NP >= n slots; odd steps pair slots (x, NP-1-x), even steps (x+1, NP-1-x); pairs whose
//    columns do not sum to s (or touch padding) are masked; the ring shifts every two steps.
// Steps are unrolled by two with the data lagging one step in the second copy (compile-time
// register remap), so positions physically move every other step.
//
// Per step only g_pq needs a cross-lane reduction: the column norms g_pp, g_qq are carried
// per column (recomputed exactly at every sweep start, updated with the exact 2x2
// eigenvalues d_p - t g_pq, d_q + t g_pq after each rotation, and recomputed whenever an
// update cancels) -- LAPACK dgesvj's scheme. g_pq partials are reduced with a recursive-
// halving shuffle tree (16 pairs per 16 shuffles); each pair's Rutishauser rotation
// (jacobi.py:68-80) is computed by ONE lane (not redundantly per lane) with
// the reference's skip rule (jacobi.py:134/167); (c, s) reach the other lanes through a
// per-warp shared-memory slot, and are appended to a rotation log from which V is rebuilt
// afterwards (so V never occupies registers during the sweeps).
#pragma once
#include "common.cuh"

namespace bf {

template <int NP, int WW>
struct RegCfg {
  static constexpr int np = NP, ww = WW;
  static constexpr int pairs = NP / 2;
  static constexpr int chunks = (pairs + 15) / 16;  // 16 pairs per reduction chunk
  static constexpr int threads = 32 * WW;
  static_assert(chunks <= 2, "at most 32 slot pairs (NP <= 64)");
  static_assert(NP % 2 == 0 && NP >= 4, "even NP");
};

// Named barrier among the WW row-warps of the CTA (id 1).
BF_DEV void named_bar(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }

// Recursive-halving reduce of 16 values per lane: returns on every lane the full-warp sum
// for pair index ((L>>4)&1)*8 + ((L>>3)&1)*4 + ((L>>2)&1)*2 + ((L>>1)&1).
template <typename T>
BF_DEV T halving16(T (&x)[16], int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    T send = b4 ? x[i] : x[i + 8];
    T keep = b4 ? x[i + 8] : x[i];
    x[i] = keep + shfl_xor(send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    T send = b3 ? x[i] : x[i + 4];
    T keep = b3 ? x[i + 4] : x[i];
    x[i] = keep + shfl_xor(send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    T send = b2 ? x[i] : x[i + 2];
    T keep = b2 ? x[i + 2] : x[i];
    x[i] = keep + shfl_xor(send, 4);
  }
  T send = b1 ? x[0] : x[1];
  T keep = b1 ? x[1] : x[0];
  T v = keep + shfl_xor(send, 2);
  return v + shfl_xor(v, 1);
}

BF_DEV int halving16_index(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

// Rutishauser rotation returning t as well (jacobi.py:68-80), g_pq != 0.
BF_DEV void jacobi_rotation_t(double gpp, double gpq, double gqq, double& c, double& s, double& t) {
  double den = 2.0 * gpq;
  double diff = gqq - gpp;
  double aden = fabs(den);
  if (aden > 1e-290 && aden < 1e290 && fabs(diff) < 1e290) {
    double zeta = diff * rcp_fast(den);
    double az = fabs(zeta);
    if (az < 1e150) {
      double x = fma(az, az, 1.0);
      double h = x * rsqrt_fast(x);  // hypot(1, zeta)
      t = copysign(rcp_fast(az + h), zeta);
    } else {
      t = copysign(0.5 / az, zeta);
    }
    c = rsqrt_fast(fma(t, t, 1.0));
    s = c * t;
  } else {
    double zeta = diff / den;
    t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
    c = 1.0 / hypot(1.0, t);
    s = c * t;
  }
}

// Step kinds: 0 round robin, 1 serial odd step, 2 serial even step.
template <class C, int ORD>
struct RegGeom {
  static constexpr int NP = C::np, NPAIR = C::pairs;
  template <int KIND>
  static BF_DEV constexpr int nslots() {
    return KIND == 2 ? NPAIR - 1 : NPAIR;
  }
  template <int KIND>
  static BF_DEV constexpr int la(int k) {
    return KIND == 2 ? k + 1 : k;
  }
  static BF_DEV constexpr int lb(int k) { return NP - 1 - k; }
  // physical register of a logical position when the data lags PH steps (rr) / ring shifts
  template <int KIND, int PH>
  static BF_DEV constexpr int phys(int x) {
    return KIND == 0 ? (x == 0 ? 0 : 1 + ((x - 1 - PH) % (NP - 1) + (NP - 1)) % (NP - 1)) : (x + PH) % NP;
  }
  template <int KIND, int PH>
  static BF_DEV constexpr int pa(int k) {
    return phys<KIND, PH>(la<KIND>(k));
  }
  template <int KIND, int PH>
  static BF_DEV constexpr int pb(int k) {
    return phys<KIND, PH>(lb(k));
  }
  // columns held by slot k at round-robin step t / serial ring offset off (physical (x + PH))
  template <int KIND, int PH>
  static BF_DEV void cols(int k, int t_rr, int off, int& ca, int& cb) {
    const int a = la<KIND>(k), b = lb(k);
    if (KIND == 0) {
      const int L = NP - 1;
      ca = a == 0 ? 0 : 1 + (((a - 1 - t_rr) % L) + L) % L;
      cb = 1 + (((b - 1 - t_rr) % L) + L) % L;
    } else {
      ca = ((a + PH - off) % NP + NP) % NP;
      cb = ((b + PH - off) % NP + NP) % NP;
    }
  }

  // apply the (c, s) of every slot (uniform per slot; s == 0 means identity) to one row
  template <typename T, int KIND, int PH>
  static BF_DEV void apply(T (&w)[NP], const double* cs) {
#pragma unroll
    for (int k = 0; k < nslots<KIND>(); ++k) {
      const double2 p = *reinterpret_cast<const double2*>(cs + 2 * k);
      if (p.y != 0.0) {
        const T c = (T)p.x, sn = (T)p.y;
        T a = w[pa<KIND, PH>(k)], b = w[pb<KIND, PH>(k)];
        w[pa<KIND, PH>(k)] = fma(c, a, -sn * b);
        w[pb<KIND, PH>(k)] = fma(sn, a, c * b);
      }
    }
  }

  // positions 1..NP-1 rotate D places: new[j] = old[1 + (j - 1 - D) mod (NP - 1)]
  template <typename T, int D>
  static BF_DEV void rotate_rr(T (&x)[NP]) {
    T tmp[NP];
#pragma unroll
    for (int j = 1; j < NP; ++j) tmp[j] = x[j];
#pragma unroll
    for (int j = 1; j < NP; ++j) x[j] = tmp[1 + ((j - 1 - D) % (NP - 1) + (NP - 1)) % (NP - 1)];
  }
  // ring shift: new[x] = old[(x + D) mod NP]
  template <typename T, int D>
  static BF_DEV void shift_ring(T (&x)[NP]) {
    T tmp[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) tmp[j] = x[j];
#pragma unroll
    for (int j = 0; j < NP; ++j) x[j] = tmp[(j + D) % NP];
  }
};

// Drives the step sequence (orderings, 2-step unrolling, physical moves, sweep boundaries)
// for any per-step action. Action provides:
//   template <int KIND, int PH> void step(T (&w)[NP], int s, int off, int t_rr);
//   template <int PH> void sweep_start(T (&w)[NP], int off);
//   bool sweep_end();   // true -> stop
template <typename T, class C, int ORD>
struct RegDriver {
  using G = RegGeom<C, ORD>;
  static constexpr int NP = C::np;

  template <class A>
  static BF_DEV void run(T (&w)[NP], int n, A& act) {
    if (ORD == 1) {
      int t = 0, pend = 0;
      act.template sweep_start<0>(w, 0);
      for (;;) {
        act.template step<0, 0>(w, 0, 0, t);
        if (++t == NP - 1) {
          t = 0;
          if (act.sweep_end()) {
            pend = 1;
            break;
          }
          act.template sweep_start<1>(w, 0);
        }
        act.template step<0, 1>(w, 0, 0, t);
        if (++t == NP - 1) {
          t = 0;
          if (act.sweep_end()) {
            pend = 2;
            break;
          }
          G::template rotate_rr<T, 2>(w);
          act.template sweep_start<0>(w, 0);
          continue;
        }
        G::template rotate_rr<T, 2>(w);
      }
      if (pend == 1) G::template rotate_rr<T, 1>(w);
      if (pend == 2) G::template rotate_rr<T, 2>(w);
    } else {
      const int off0 = NP / 2 - 1;
      for (;;) {
        int off = off0, u = 0;
        act.template sweep_start<0>(w, off);
        for (; u + 1 < n - 1; u += 2) {
          act.template step<1, 0>(w, 2 * u + 1, off, 0);
          act.template step<2, 0>(w, 2 * u + 2, off, 0);
          act.template step<1, 1>(w, 2 * u + 3, off, 0);
          act.template step<2, 1>(w, 2 * u + 4, off, 0);
          G::template shift_ring<T, 2>(w);
          off -= 2;
        }
        if (u < n - 1) {
          act.template step<1, 0>(w, 2 * u + 1, off, 0);
          act.template step<2, 0>(w, 2 * u + 2, off, 0);
          G::template shift_ring<T, 1>(w);
          off -= 1;
        }
        // realign: column c back at slot c + off0 ((NP - n + 1) mod NP more shifts)
        for (int k = (NP - n + 1) % NP; k > 0; --k) G::template shift_ring<T, 1>(w);
        if (act.sweep_end()) break;
      }
    }
  }
};

// ---------------------------------------------------------------------------------------------
// W phase: sweeps until a rotation-free sweep (jacobi.py:270-281), logging (c, s) per slot.
// Shared memory per warp: cs[32][2], d[NP] (tracked squared norms by column);
// CTA-wide: red[WW][32] (cross-warp partials), red2[WW][64].
template <typename T, class C, int ORD>
struct WAction {
  using G = RegGeom<C, ORD>;
  static constexpr int NP = C::np, NPAIR = C::pairs, WW = C::ww, CH = C::chunks;

  int lane, warp, n, max_sweeps;
  double tol2;
  double* cs;    // this warp's (c, s) slot area, 32 x 2
  double* d;     // this warp's tracked norms, NP
  double* red;   // WW x 32
  double* red2;  // WW x 64
  double2* log;  // this matrix's log cursor (global)
  int sweeps, conv, rot, recompute;
  long long rots;

  // lane L computes pair k = chunk (L & 1) * 16 + halving16_index(L)
  BF_DEV int my_pair() const { return (lane & 1) * 16 + halving16_index(lane); }

  // exact squared column norms of all NP positions (via the rr / odd-step slot pairing)
  template <int KIND, int PH>
  BF_DEV void norms(T (&w)[NP], int off, int t_rr) {
    T na = T(0), nb = T(0);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      T x[16], y[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = c * 16 + i;
        x[i] = y[i] = T(0);
        if (k < NPAIR) {
          T a = w[G::template pa<KIND, PH>(k)], b = w[G::template pb<KIND, PH>(k)];
          x[i] = a * a;
          y[i] = b * b;
        }
      }
      T sx = halving16(x, lane), sy = halving16(y, lane);
      if ((lane & 1) == c) {
        na = sx;
        nb = sy;
      }
    }
    const int k = my_pair();
    const bool mine = k < NPAIR;
    double da = (double)na, db = (double)nb;
    if (WW > 1) {
      if (mine) {
        red2[warp * 64 + 2 * k] = da;
        red2[warp * 64 + 2 * k + 1] = db;
      }
      named_bar(1, WW * 32);
      if (mine) {
        da = db = 0.0;
#pragma unroll
        for (int q = 0; q < WW; ++q) {
          da += red2[q * 64 + 2 * k];
          db += red2[q * 64 + 2 * k + 1];
        }
      }
    }
    if (mine) {
      int ca, cb;
      G::template cols<KIND, PH>(k, t_rr, off, ca, cb);
      d[ca] = da;
      d[cb] = db;
    }
    __syncwarp();
    if (WW > 1) named_bar(1, WW * 32);  // red2 reuse
    recompute = 0;
  }

  template <int PH>
  BF_DEV void sweep_start(T (&w)[NP], int off) {
    rot = 0;
    if (ORD == 1)
      norms<0, PH>(w, off, 0);
    else
      norms<1, PH>(w, off, 0);
  }

  template <int KIND, int PH>
  BF_DEV void step(T (&w)[NP], int s, int off, int t_rr) {
    if (recompute) {
      // the even serial step's pairing skips two slots: recompute through the odd pairing
      norms<KIND == 0 ? 0 : 1, PH>(w, off, t_rr);
    }
    constexpr int NS = G::template nslots<KIND>();
    T g = T(0);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      T x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = c * 16 + i;
        x[i] = k < NS ? w[G::template pa<KIND, PH>(k)] * w[G::template pb<KIND, PH>(k)] : T(0);
      }
      T sg = halving16(x, lane);
      if ((lane & 1) == c) g = sg;
    }
    const int k = my_pair();
    const bool mine = k < NS;
    double gpq = (double)g;
    if (WW > 1) {
      if (mine) red[warp * 32 + k] = gpq;
      named_bar(1, WW * 32);
      if (mine) {
        gpq = 0.0;
#pragma unroll
        for (int q = 0; q < WW; ++q) gpq += red[q * 32 + k];
      }
    }
    int flag = 0;
    if (mine) {
      int ca, cb;
      G::template cols<KIND, PH>(k, t_rr, off, ca, cb);
      bool active = ORD == 1 || (ca != cb && ca < n && cb < n && ca + cb == s);
      double cc = 1.0, sn = 0.0;
      if (active) {
        const bool rev = ca > cb;  // slot a holds the larger column: rotate with swapped roles
        const int p = rev ? cb : ca, q = rev ? ca : cb;
        const double dpp = d[p], dqq = d[q];
        if (gpq * gpq > tol2 * (dpp * dqq)) {
          double t;
          jacobi_rotation_t(dpp, gpq, dqq, cc, sn, t);
          const double np_ = dpp - t * gpq, nq = dqq + t * gpq;
          d[p] = np_ > 0.0 ? np_ : 0.0;
          d[q] = nq > 0.0 ? nq : 0.0;
          flag = (np_ < 1e-2 * dpp) | (nq < 1e-2 * dqq);  // cancellation -> recompute next step
          if (rev) sn = -sn;
          ++rot;
        }
      }
      cs[2 * k] = cc;
      cs[2 * k + 1] = sn;
    }
    recompute = __any_sync(FULL, flag);
    __syncwarp();
    if (log != nullptr && warp == 0 && mine && (CH == 2 || (lane & 1) == 0)) log[k] = make_double2(cs[2 * k], cs[2 * k + 1]);
    if (log != nullptr) log += NPAIR;
    G::template apply<T, KIND, PH>(w, cs);
    __syncwarp();
  }

  BF_DEV bool sweep_end() {
    // identical in every warp (identical sums and decisions); with one chunk each pair lives
    // on two lanes, count it once
    int r = (CH == 2 || (lane & 1) == 0) ? rot : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(FULL, r, o);
    rots += r;
    ++sweeps;
    if (r == 0) conv = 1;
    return conv || sweeps >= max_sweeps;
  }
};

// V phase: replay the logged rotations on V rows (lane = V row), staging the log through
// shared memory STAGE steps at a time.
template <typename T, class C, int ORD>
struct VAction {
  using G = RegGeom<C, ORD>;
  static constexpr int NP = C::np, NPAIR = C::pairs, WW = C::ww;
  static constexpr int STAGE = 8;
  const double2* log;  // global cursor
  double2* stage;      // STAGE x NPAIR smem (CTA-shared)
  int in_stage, sweeps_left;

  BF_DEV void refill() {
    // all WW warps cooperatively copy the next STAGE steps (log is padded by STAGE steps)
    if (WW > 1) named_bar(1, WW * 32);
    __syncwarp();
    for (int e = threadIdx.x; e < STAGE * NPAIR; e += WW * 32) stage[e] = log[e];
    log += STAGE * NPAIR;
    if (WW > 1) named_bar(1, WW * 32);
    __syncwarp();
    in_stage = 0;
  }
  template <int PH>
  BF_DEV void sweep_start(T (&)[NP], int) {}
  template <int KIND, int PH>
  BF_DEV void step(T (&v)[NP], int, int, int) {
    if (in_stage == STAGE) refill();
    G::template apply<T, KIND, PH>(v, reinterpret_cast<const double*>(stage + in_stage * NPAIR));
    ++in_stage;
  }
  BF_DEV bool sweep_end() { return --sweeps_left <= 0; }
};

}  // namespace bf
