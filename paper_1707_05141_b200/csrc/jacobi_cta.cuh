// CTA-cooperative one-sided Jacobi building blocks (shared-memory tier).
//
// One CTA owns one matrix. W (m x nw, column j at W + j*ldw) and V (nw x nw,
// column j at V + j*ldv) live in shared memory (or, for matrices that do not
// fit, in an L2-resident global workspace -- same code, different pointer).
// Each round-robin / wavefront step is a perfect matching of columns, so the
// pairs of a step are spread over the warps (one warp per column pair, rows
// over lanes, dot products by xor-butterfly shuffles) with one CTA barrier per
// step -- exactly the parallel sweep of the reference's _round_robin_sweep
// (jacobi.py:158-186) and, through the p+q wavefront, of _serial_sweep
// (jacobi.py:118-155).
#pragma once
#include "common.cuh"

namespace bf {

struct SweepStats {
  int sweeps;
  int converged;
  long long rotations;
};

// Process up to PB pairs per warp at once so the rotation latency chains overlap.
template <typename T, int PB>
BF_DEV long long jacobi_step(T* W, int ldw, T* V, int ldv, int m, int nw, int ordering, int step, double tol2,
                             int warp, int nwarps, int lane) {
  const int P = ordering == 0 ? wf_count(nw, step) : (nw >> 1);
  long long rot = 0;
  for (int base = warp; base < P; base += nwarps * PB) {
    int pp[PB], qq[PB];
    T gpp[PB], gpq[PB], gqq[PB];
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      int k = base + j * nwarps;
      gpp[j] = gpq[j] = gqq[j] = T(0);
      pp[j] = -1;
      qq[j] = -1;
      if (k < P) {
        if (ordering == 0)
          wf_pair(nw, step, k, pp[j], qq[j]);
        else
          rr_pair(nw, step, k, pp[j], qq[j]);
        const T* wp = W + (size_t)pp[j] * ldw;
        const T* wq = W + (size_t)qq[j] * ldw;
        for (int i = lane; i < m; i += 32) {
          T a = wp[i], b = wq[i];
          gpp[j] = fma(a, a, gpp[j]);
          gpq[j] = fma(a, b, gpq[j]);
          gqq[j] = fma(b, b, gqq[j]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        gpp[j] += shfl_xor(gpp[j], o);
        gpq[j] += shfl_xor(gpq[j], o);
        gqq[j] += shfl_xor(gqq[j], o);
      }
    }
    // the PB rotations are independent: form them all before applying any (their latency
    // chains overlap instead of serialising with the column updates)
    T cj[PB], sj[PB];
    bool doit[PB];
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      double dpp = (double)gpp[j], dpq = (double)gpq[j], dqq = (double)gqq[j];
      // skip rule (jacobi.py:134 / :167): |g_pq|^2 <= tol^2 g_pp g_qq
      doit[j] = pp[j] >= 0 && dpq * dpq > tol2 * (dpp * dqq);
      double cd = 1.0, sd = 0.0, td;
      if (doit[j]) jacobi_rotation_t(dpp, dpq, dqq, cd, sd, td);
      cj[j] = (T)cd;
      sj[j] = (T)sd;
    }
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      if (!doit[j]) continue;
      const T c = cj[j], s = sj[j];
      ++rot;
      T* wp = W + (size_t)pp[j] * ldw;
      T* wq = W + (size_t)qq[j] * ldw;
      for (int i = lane; i < m; i += 32) {
        T a = wp[i], b = wq[i];
        wp[i] = fma(c, a, -s * b);
        wq[i] = fma(s, a, c * b);
      }
      if (V) {
        T* vp = V + (size_t)pp[j] * ldv;
        T* vq = V + (size_t)qq[j] * ldv;
        for (int i = lane; i < nw; i += 32) {
          T a = vp[i], b = vq[i];
          vp[i] = fma(c, a, -s * b);
          vq[i] = fma(s, a, c * b);
        }
      }
    }
  }
  return rot;
}

// Sweeps until one performs no rotation (jacobi.py:270-281). counters: 2 ints of smem.
template <typename T, int PB>
BF_DEV SweepStats jacobi_sweeps(T* W, int ldw, T* V, int ldv, int m, int n, int nw, int ordering, double tol,
                                int max_sweeps, int* counters) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const double tol2 = tol * tol;
  SweepStats st{0, n < 2, 0};
  const int nsteps = ordering == 0 ? (nw >= 2 ? 2 * nw - 3 : 0) : nw - 1;
  if (tid == 0) counters[0] = counters[1] = 0;
  __syncthreads();
  for (int sw = 0; sw < max_sweeps && !st.converged; ++sw) {
    long long rot = 0;
    for (int s = 0; s < nsteps; ++s) {
      rot += jacobi_step<T, PB>(W, ldw, V, ldv, m, nw, ordering, ordering == 0 ? s + 1 : s, tol2, warp, nwarps,
                                lane);
      __syncthreads();
    }
    int* ctr = counters + (sw & 1);
    if (lane == 0 && rot) atomicAdd(ctr, (int)rot);
    __syncthreads();
    int total = *ctr;
    st.rotations += total;
    st.sweeps++;
    if (total == 0) st.converged = 1;
    __syncthreads();
    if (tid == 0) *ctr = 0;
  }
  return st;
}

// off_orthogonality (jacobi.py:83-99) over the nw columns of W; CTA-wide, result broadcast.
template <typename T>
BF_DEV double off_orthogonality_cta(const T* W, int ldw, int m, int nw, T* dsc /* nw smem */, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int j = warp; j < nw; j += nwarps) {
    T acc = 0;
    for (int i = lane; i < m; i += 32) acc = fma(W[(size_t)j * ldw + i], W[(size_t)j * ldw + i], acc);
    acc = warp_allreduce_sum(acc);
    if (lane == 0) dsc[j] = (T)sqrt((double)(acc < 0 ? -acc : acc));
  }
  if (tid == 0) *red = 0.0;
  __syncthreads();
  double best = 0.0;
  const int npairs = nw * (nw - 1) / 2;
  for (int k = warp; k < npairs; k += nwarps) {
    // k -> (i, j), i < j
    int i = 0, rem = k;
    while (rem >= nw - 1 - i) {
      rem -= nw - 1 - i;
      ++i;
    }
    int j = i + 1 + rem;
    T acc = 0;
    for (int r = lane; r < m; r += 32) acc = fma(W[(size_t)i * ldw + r], W[(size_t)j * ldw + r], acc);
    acc = warp_allreduce_sum(acc);
    T den = dsc[i] * dsc[j];
    if (den > T(0)) {
      double rt = (double)((acc < 0 ? -acc : acc) / den);
      best = rt > best ? rt : best;
    }
  }
  if (lane == 0 && best > 0.0) atomicMax((unsigned long long*)red, (unsigned long long)__double_as_longlong(best));
  __syncthreads();
  double r = *red;
  __syncthreads();
  return r;
}

template <typename T>
BF_DEV bool sort_greater(T a, T b) {
  // descending with NaN last (numpy argsort(-x, kind="stable"))
  return (a > b) || (b != b && a == a);
}

// _extract_svd (jacobi.py:212-228): sigma_j = ||w_j||, stable descending order,
// U = W[:, order] / sigma, V = V[:n, order]. Zero columns are completed by
// _complete_zero_rows (jacobi.py:189-209). Returns true if completion ran.
// sig/rank/order: smem scratch of n entries each; cand: 2*m scratch for completion.
// n_out: sorted columns emitted (block_svd drops its padding, blockjacobi.py:156-167);
// v_rows: rows of V emitted.
template <typename T>
BF_DEV void extract_svd_cta(const T* W, int ldw, const T* V, int ldv, int m, int n, int n_out, int v_rows, T* U_out,
                            int ldu, T* S_out, T* V_out, int ldvo, T* sig, int* order, T* cand, int* flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int j = warp; j < n; j += nwarps) {
    T acc = 0;
    for (int i = lane; i < m; i += 32) acc = fma(W[(size_t)j * ldw + i], W[(size_t)j * ldw + i], acc);
    acc = warp_allreduce_sum(acc);
    if (lane == 0) sig[j] = sqrt(acc);
  }
  if (tid == 0) *flag = 0;
  __syncthreads();
  for (int j = tid; j < n; j += blockDim.x) {
    T sj = sig[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) {
      T si = sig[i];
      bool gt = sort_greater(si, sj);
      bool eq = !gt && !sort_greater(sj, si);
      rank += gt || (eq && i < j);
    }
    order[rank] = j;
  }
  __syncthreads();
  for (int r = tid; r < n_out; r += blockDim.x) {
    T sg = sig[order[r]];
    S_out[r] = sg;
    if (!(sg > T(0))) atomicOr(flag, 1);
  }
  for (int r = warp; r < n_out; r += nwarps) {
    int j = order[r];
    T sg = sig[j];
    bool nz = sg > T(0);
    for (int i = lane; i < m; i += 32) {
      T x = W[(size_t)j * ldw + i];
      U_out[(size_t)r * ldu + i] = nz ? x / sg : x;
    }
    if (V_out)
      for (int i = lane; i < v_rows; i += 32) V_out[(size_t)r * ldvo + i] = V[(size_t)j * ldv + i];
  }
  __syncthreads();
  if (*flag == 0) return;
  // ---- rare path: complete zero columns (warp 0), U columns are the reference's ut rows
  if (warp == 0) {
    T* c = cand;
    T* best = cand + m;
    for (int z = 0; z < n_out; ++z) {
      if (sig[order[z]] > T(0)) continue;
      double best_norm = -1.0;
      for (int e = 0; e < m; ++e) {
        for (int i = lane; i < m; i += 32) c[i] = (i == e) ? T(1) : T(0);
        __syncwarp();
        // done = nonzero columns in sorted order, then already-completed zero columns in order
        for (int pass = 0; pass < 2; ++pass) {
          for (int d = 0; d < (pass == 0 ? n_out : z); ++d) {
            bool isz = !(sig[order[d]] > T(0));
            if (pass == 0 ? isz : !isz) continue;
            const T* row = U_out + (size_t)d * ldu;
            T pr = 0;
            for (int i = lane; i < m; i += 32) pr = fma(row[i], c[i], pr);
            pr = warp_allreduce_sum(pr);
            for (int i = lane; i < m; i += 32) c[i] -= row[i] * pr;
            __syncwarp();
          }
        }
        T nn = 0;
        for (int i = lane; i < m; i += 32) nn = fma(c[i], c[i], nn);
        double nrm = sqrt((double)warp_allreduce_sum(nn));
        if (nrm > best_norm) {
          best_norm = nrm;
          for (int i = lane; i < m; i += 32) best[i] = c[i];
        }
        __syncwarp();
      }
      for (int pass = 0; pass < 2; ++pass) {
        for (int d = 0; d < (pass == 0 ? n_out : z); ++d) {
          bool isz = !(sig[order[d]] > T(0));
          if (pass == 0 ? isz : !isz) continue;
          const T* row = U_out + (size_t)d * ldu;
          T pr = 0;
          for (int i = lane; i < m; i += 32) pr = fma(row[i], best[i], pr);
          pr = warp_allreduce_sum(pr);
          for (int i = lane; i < m; i += 32) best[i] -= row[i] * pr;
          __syncwarp();
        }
      }
      T nb = 0;
      for (int i = lane; i < m; i += 32) nb = fma(best[i], best[i], nb);
      nb = sqrt(warp_allreduce_sum(nb));
      for (int i = lane; i < m; i += 32) U_out[(size_t)z * ldu + i] = best[i] / nb;
      __syncwarp();
    }
  }
  __syncthreads();
}

}  // namespace bf
