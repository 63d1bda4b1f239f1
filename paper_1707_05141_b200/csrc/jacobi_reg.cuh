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
// Per step only g_pq needs a cross-row reduction: the column norms g_pp, g_qq are carried
// per column (recomputed exactly at every sweep start, updated with the exact 2x2
// eigenvalues d_p - t g_pq, d_q + t g_pq after each rotation, and recomputed whenever an
// update cancels) -- LAPACK dgesvj's scheme. The row products are transposed through a
// shared-memory buffer and summed by a few threads per pair (WAction below); each pair's
// Rutishauser rotation (jacobi.py:68-80) is computed by that pair's threads only (not by
// every lane) with the reference's skip rule (jacobi.py:134/167); (c, s) reach
// the rows through shared memory and are appended to a rotation log from which V is rebuilt
// afterwards (so V never occupies registers during the sweeps).
#pragma once
#include "common.cuh"

namespace bf {

#ifdef BF_PHASE_TIMING
// kernel-experiment instrumentation: per-phase clock totals of warp 0 lane 0 (debug builds only)
__device__ unsigned long long g_phase_clk[8];
#define BF_T(i) long long _t##i = clock64()
#define BF_ACC(slot, a, b) if (threadIdx.x == 0) atomicAdd(&g_phase_clk[slot], (unsigned long long)(_t##b - _t##a))
#else
#define BF_T(i)
#define BF_ACC(slot, a, b)
#endif

constexpr int pow2_floor(int x) { return x >= 32 ? 32 : x >= 16 ? 16 : x >= 8 ? 8 : x >= 4 ? 4 : x >= 2 ? 2 : 1; }

template <int NP, int WW>
struct RegCfg {
  static constexpr int np = NP, ww = WW;
  static constexpr int pairs = NP / 2;
  static constexpr int threads = 32 * WW;
  static constexpr int rows = 32 * WW;
  // slot-sum geometry: tpp threads per slot (power of two, one warp at most) each add rp rows
  static constexpr int tpp = pow2_floor(rows / pairs);
  static constexpr int rp = rows / tpp;
  static constexpr int rs = rows + 2;  // product-buffer row stride (doubles; 16-byte multiple)
  static_assert(pairs <= 32, "at most 32 slot pairs (NP <= 64)");
  static_assert(NP % 2 == 0 && NP >= 4, "even NP");
  static_assert(rp % 4 == 0, "rows per slot part must be a multiple of 4");
};

// Named barrier among the WW row-warps of the CTA (id 1).
BF_DEV void named_bar(int id, int nthreads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory"); }

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
      // round robin applies the identity to skipped pairs like the reference
      // (jacobi.py:177-185); the serial sweep leaves them untouched (jacobi.py:134-136)
      if (ORD == 1 || p.y != 0.0) {
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
// CTA-level synchronisation among the WW row-warps (named barrier 1; a warp sync when WW == 1).
template <int WW>
BF_DEV void rows_sync() {
  if (WW > 1)
    named_bar(1, WW * 32);
  else
    __syncwarp();
}
// Barrier that also ORs a predicate over the WW*32 threads.
template <int WW>
BF_DEV int rows_sync_or(int pred) {
  if (WW > 1) {
    int r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\tbarrier.cta.red.or.pred q, 1, %2, p;\n\t"
        "selp.s32 %0, 1, 0, q;\n\t}"
        : "=r"(r)
        : "r"(pred), "r"(WW * 32)
        : "memory");
    return r;
  }
  __syncwarp();
  return __any_sync(FULL, pred);
}

// Sum of RP consecutive doubles in shared memory (16-byte aligned), four accumulators.
template <int RP>
BF_DEV double sum_rows(const double* p) {
  static_assert(RP % 4 == 0, "RP multiple of 4");
  const double2* q = reinterpret_cast<const double2*>(p);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
  for (int j = 0; j < RP / 4; ++j) {
    const double2 x = q[2 * j], y = q[2 * j + 1];
    a0 += x.x;
    a1 += x.y;
    a2 += y.x;
    a3 += y.y;
  }
  return (a0 + a1) + (a2 + a3);
}

// W phase: sweeps until a rotation-free sweep (jacobi.py:270-281), logging (c, s) per slot.
// Per step: every row-thread writes its NS slot products w_a * w_b to the shared product
// buffer P[slot][row] (one transposing store per slot, conflict-free); after one barrier,
// TPP threads per slot sum RP rows each (vector loads) and combine by an xor butterfly, so
// every one of them holds the same g_pq and computes the same rotation (no broadcast of the
// scalars needed inside the slot group); one of them records (c, s) in cs[slot] and in the
// log; after a second barrier (which also ORs the cancellation flags) every row applies all
// slots. Column norms d[col] are tracked (dgesvj scheme, see header).
template <typename T, class C, int ORD>
struct WAction {
  using G = RegGeom<C, ORD>;
  static constexpr int NP = C::np, NPAIR = C::pairs, WW = C::ww;
  static constexpr int TPP = C::tpp, RP = C::rp, RS = C::rs;

  int tid, n, max_sweeps;
  double tol2;
  double* cs;    // NPAIR x (c, s), CTA-shared
  double* d;     // NP tracked squared norms by column, CTA-shared
  double* P;     // 2 * NPAIR x RS product buffer, CTA-shared
  int* swrot;    // 2 sweep rotation counters (parity), CTA-shared
  double2* log;  // this matrix's log cursor (global)
  int sweeps, conv, rot, recompute;
  long long rots;

  BF_DEV int slot() const { return tid / TPP; }
  BF_DEV int part() const { return tid % TPP; }

  BF_DEV double butterfly(double g) const {
#pragma unroll
    for (int o = TPP / 2; o > 0; o >>= 1) g += shfl_xor(g, o);
    return g;
  }

  // exact squared column norms of all NP positions (via the rr / odd-step slot pairing)
  template <int KIND, int PH>
  BF_DEV void norms(T (&w)[NP], int off, int t_rr) {
#pragma unroll
    for (int k = 0; k < NPAIR; ++k) {
      const T a = w[G::template pa<KIND, PH>(k)], b = w[G::template pb<KIND, PH>(k)];
      P[k * RS + tid] = a * a;
      P[(NPAIR + k) * RS + tid] = b * b;
    }
    rows_sync<WW>();
    const int k = slot(), h = part();
    double da = 0.0, db = 0.0;
    if (k < NPAIR) {
      da = sum_rows<RP>(P + k * RS + h * RP);
      db = sum_rows<RP>(P + (NPAIR + k) * RS + h * RP);
    }
    da = butterfly(da);
    db = butterfly(db);
    if (k < NPAIR && h == 0) {
      int ca, cb;
      G::template cols<KIND, PH>(k, t_rr, off, ca, cb);
      d[ca] = da;
      d[cb] = db;
    }
    rows_sync<WW>();  // d visible, P free
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
    BF_T(0);
#pragma unroll
    for (int k = 0; k < NS; ++k) P[k * RS + tid] = w[G::template pa<KIND, PH>(k)] * w[G::template pb<KIND, PH>(k)];
    BF_T(1);
    rows_sync<WW>();
    BF_T(2);
    const int k = slot(), h = part();
    double gpq = k < NS ? sum_rows<RP>(P + k * RS + h * RP) : 0.0;
    gpq = butterfly(gpq);
    BF_T(3);
    int flag = 0, p = 0, q = 0;
    bool did = false;
    double cc = 1.0, sn = 0.0, np_ = 0.0, nq = 0.0;
    if (k < NS) {
      int ca, cb;
      G::template cols<KIND, PH>(k, t_rr, off, ca, cb);
      const bool active = ORD == 1 || (ca != cb && ca < n && cb < n && ca + cb == s);
      if (active) {
        const bool rev = ca > cb;  // slot a holds the larger column: rotate with swapped roles
        p = rev ? cb : ca;
        q = rev ? ca : cb;
        const double dpp = d[p], dqq = d[q];
        // skip rule (jacobi.py:134 / :167)
        if (gpq * gpq > tol2 * (dpp * dqq)) {
          double t;
          jacobi_rotation_t(dpp, gpq, dqq, cc, sn, t);
          np_ = dpp - t * gpq;
          nq = dqq + t * gpq;
          flag = (np_ < 1e-2 * dpp) | (nq < 1e-2 * dqq);  // cancellation -> recompute next step
          if (rev) sn = -sn;
          did = true;
        }
      }
    }
    __syncwarp();  // every thread of the slot group has read d[p], d[q]
    if (k < NS && h == 0) {
      if (did) {
        d[p] = np_ > 0.0 ? np_ : 0.0;
        d[q] = nq > 0.0 ? nq : 0.0;
        ++rot;
      }
      const double2 v = make_double2(cc, sn);
      *reinterpret_cast<double2*>(cs + 2 * k) = v;
      if (log != nullptr) log[k] = v;
    }
    if (log != nullptr) log += NPAIR;
    BF_T(4);
    recompute = rows_sync_or<WW>(flag);
    BF_T(5);
    G::template apply<T, KIND, PH>(w, cs);
    BF_T(6);
    BF_ACC(0, 0, 1);
    BF_ACC(1, 1, 2);
    BF_ACC(2, 2, 3);
    BF_ACC(3, 3, 4);
    BF_ACC(4, 4, 5);
    BF_ACC(5, 5, 6);
    BF_ACC(6, 0, 6);
  }

  BF_DEV bool sweep_end() {
    int r = rot;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(FULL, r, o);
    if (WW > 1) {
      const int par = sweeps & 1;
      if ((tid & 31) == 0) atomicAdd(swrot + par, r);
      rows_sync<WW>();
      r = swrot[par];
      if (tid == 0) swrot[par ^ 1] = 0;
    }
    rots += r;
    ++sweeps;
    if (r == 0) conv = 1;
    return conv || sweeps >= max_sweeps;
  }
};

// V phase: replay the logged rotations on V rows (lane = V row). The log streams through two
// shared-memory stages of STAGE steps each: while one stage is replayed, cp.async fills the
// other, so the (L2/DRAM-resident) log reads stay off the dependency chain.
BF_DEV void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
BF_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
BF_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T, class C, int ORD, int STAGE>
struct VAction {
  using G = RegGeom<C, ORD>;
  static constexpr int NP = C::np, NPAIR = C::pairs, WW = C::ww;
  const double2* log;  // global cursor: next stage to prefetch
  double2* stage;      // 2 x STAGE x NPAIR smem (CTA-shared)
  int in_stage, cur, sweeps_left;

  BF_DEV void prefetch(int buf) {
    double2* dst = stage + buf * STAGE * NPAIR;
    for (int e = threadIdx.x; e < STAGE * NPAIR; e += WW * 32) cp_async16(dst + e, log + e);
    cp_async_commit();
    log += STAGE * NPAIR;
  }
  // all threads: stage 0 ready, stage 1 in flight (the log is padded by 2 STAGE steps)
  BF_DEV void start() {
    prefetch(0);
    cp_async_wait_all();
    prefetch(1);
    rows_sync<WW>();
    cur = 0;
    in_stage = 0;
  }
  BF_DEV void next_stage() {
    cp_async_wait_all();  // stage cur ^ 1 landed (this thread's part)
    rows_sync<WW>();      // ... everyone's part, and everyone is done with stage cur
    prefetch(cur);
    cur ^= 1;
    in_stage = 0;
  }
  template <int PH>
  BF_DEV void sweep_start(T (&)[NP], int) {}
  template <int KIND, int PH>
  BF_DEV void step(T (&v)[NP], int, int, int) {
    if (in_stage == STAGE) next_stage();
    G::template apply<T, KIND, PH>(v, reinterpret_cast<const double*>(stage + (cur * STAGE + in_stage) * NPAIR));
    ++in_stage;
  }
  BF_DEV bool sweep_end() { return --sweeps_left <= 0; }
};

}  // namespace bf
