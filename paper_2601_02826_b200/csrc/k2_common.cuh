// k2_common.cuh — end-of-pass logic shared by the X~^T theta kernels (TC and SIMT):
// CTA reduction of the a2/a6 partials, last-CTA convergence test (a6) and the
// per-RHS lambda-path state machine (a8).
#pragma once
#include "fsqr_dev.cuh"

template <int RMAX>
__device__ void k2_load_ctx(const Dev& D, K2Ctx<RMAX>& C) {
  // clear the forward accumulators of the previous iteration (its finalize has completed: every
  // K2 kernel calls this after griddepcontrol.wait; this iteration's forward product starts after
  // this kernel ends).  Spread over the whole grid instead of a store per row on the finalize's
  // critical path.
  {
    const size_t total = (size_t)D.R * D.n;
    for (size_t o = (size_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (size_t)gridDim.x * blockDim.x)
      D.sacc[o] = 0;
  }
  C.k = *D.iter;
  C.use_w = *D.use_w != 0;
  const int par = (int)(C.k & 1);
  C.beta_in = D.beta[par];
  C.beta_out = D.beta[par ^ 1];
  C.sidx = D.sup_idx[par ^ 1];
  C.scs = D.sup_cs[par ^ 1];
  C.colsum = D.colsum;
  C.sc = D.sup_c[par ^ 1];
  C.sb = D.sup_b[par ^ 1];
  C.scnt = D.sup_cnt + (par ^ 1);
  C.R = D.R;
  __shared__ K2Const<RMAX> k2c;   // every thread of the block calls this (then a block barrier)
  if (threadIdx.x < RMAX) {
    const int r = threadIdx.x;
    k2c.active[r] = r < D.R && D.status[r] == ST_ACTIVE;
    k2c.lam[r] = r < D.R ? D.lam_cur[r] : 0.0;
    k2c.lam2[r] = r < D.R ? D.lam2[r] : 0.0;
    k2c.gscale[r] = r < D.R ? D.delta[r] / (double)D.n : 0.0;
    k2c.Tsum[r] = r < D.R ? D.Tsum[r] : 0;
  }
  __syncthreads();
  C.cs = &k2c;
}

// Block reduction of the per-thread partials (fixed order), publication of the
// CTA partials, and, in the last CTA to finish, the a6 test.  Must be called by
// every thread of the block; `red` needs blockDim/32 * RMAX * (NPART+1) doubles.
// zero the reduction buffer and point a shared-memory-mode K2Part at this warp's slot (all threads,
// before k2_load_ctx, whose block barrier orders the zeroing before any epilogue add)
// In shared-memory mode a kernel whose partials come from a subset of its warps may pass that
// warp's slot and the number of slots (red then needs only nslots * RMAX * (NPART+1) doubles).
template <int RMAX>
__device__ __forceinline__ void k2_part_init(K2Part<RMAX>& P, double* red, int slot = -1, int nslots = -1) {
  P.zero();
  if constexpr (K2Part<RMAX>::SM) {
    const int nw = nslots < 0 ? (int)(blockDim.x >> 5) : nslots;
    for (int q = threadIdx.x; q < nw * RMAX * (FSQR_NPART + 1); q += blockDim.x) red[q] = 0.0;
    P.slot = red + (slot < 0 ? (int)(threadIdx.x >> 5) : slot) * RMAX * (FSQR_NPART + 1);
  }
}

template <int RMAX>
__device__ void k2_finish(const Dev& D, const K2Ctx<RMAX>& C, K2Part<RMAX>& P, double* red, int nslots = -1) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nw = (K2Part<RMAX>::SM && nslots >= 0) ? nslots : (int)(blockDim.x >> 5);
  constexpr int W = FSQR_NPART + 1;
  if constexpr (!K2Part<RMAX>::SM) {   // shared-memory mode: the per-warp slots are already in red
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r >= C.R) break;
#pragma unroll
      for (int q = 0; q < FSQR_NPART; ++q) {
        double v = warp_sum_d(P.v[r][q]);
        if (lane == 0) red[(wid * RMAX + r) * W + q] = v;
      }
      double m = P.cmax[r];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) red[(wid * RMAX + r) * W + FSQR_NPART] = m;
    }
  }
  __syncthreads();
  __shared__ bool s_last;
  if (tid < C.R) {
    const int r = tid;
    double acc[FSQR_NPART] = {0, 0, 0, 0, 0};
    double m = 0.0;
    for (int w = 0; w < nw; ++w) {
      for (int q = 0; q < FSQR_NPART; ++q) acc[q] += red[(w * RMAX + r) * W + q];
      m = fmax(m, red[(w * RMAX + r) * W + FSQR_NPART]);
    }
    for (int q = 0; q < FSQR_NPART; ++q) D.k2part[((size_t)blockIdx.x * D.R + r) * FSQR_NPART + q] = acc[q];
    if (D.update && m > 0.0)
      atomicMax(D.cmax + (size_t)((C.k + 1) & 1) * D.R + r, (unsigned long long)__double_as_longlong(m));
  }
  // ticket as in a cooperative grid sync: bar.sync orders the CTA's partial stores before thread 0's
  // gpu-scope fence and atomic (cumulativity); the last CTA's reads are ordered after its fence
  __syncthreads();
  if (tid == 0) {
    fence_acq_rel_gpu();
    const unsigned t = atomicAdd(D.ticket, 1u);
    s_last = (t == gridDim.x - 1);
    if (s_last) fence_acq_rel_gpu();
  }
  __syncthreads();
  if (!s_last) return;

  // ---------------- last CTA: R(w^k) for every active RHS (deterministic block sum over CTAs)
  __shared__ int s_rec[FSQR_MAXR];
  __shared__ double s_tot[FSQR_MAXR][FSQR_NPART];
  for (int r = 0; r < C.R; ++r) {
    double t5[FSQR_NPART];
    reduce_records<FSQR_NPART>(D.k2part + (size_t)r * FSQR_NPART, (int)gridDim.x, D.R * FSQR_NPART, t5, red);
    if (tid == 0)
      for (int q = 0; q < FSQR_NPART; ++q) s_tot[r][q] = t5[q];
  }
  __syncthreads();
  if (tid < C.R) {
    const int r = tid;
    s_rec[r] = -1;
    if (C.cs->active[r]) {
      double a[FSQR_NPART];
      for (int q = 0; q < FSQR_NPART; ++q) a[q] = s_tot[r][q];
      const double g0 = D.sumth[r], b0 = C.beta_in[r];
      const double rb = a[0] + g0 * g0, bb = a[1] + b0 * b0, gg = a[2] + g0 * g0;
      const double Rb = sqrt(rb) / (1.0 + sqrt(bb) + sqrt(gg));
      const double* sc = D.scal + r * FSQR_NSCAL;
      const double Rp = sc[0], Rz = sc[1];
      const double obj = sc[2] / (double)D.n + a[3];
      double* lr = D.lastR + r * FSQR_TRACE_W;
      lr[0] = Rp;
      lr[1] = Rb;
      lr[2] = Rz;
      lr[3] = obj;
      lr[4] = a[4];
      if (D.update) {
        double* tr = D.trace + ((size_t)(C.k % D.trace_cap) * D.R + r) * FSQR_TRACE_W;
        for (int q = 0; q < FSQR_TRACE_W; ++q) tr[q] = lr[q];
        const double Rm = fmax(Rp, fmax(Rb, Rz));
        const bool fin = isfinite(Rp) && isfinite(Rb) && isfinite(Rz) && isfinite(obj);
        if (!fin) {
          D.status[r] = ST_NUMERIC;
          D.commit_iter[r] = C.k;
        } else if (D.path) {
          const bool conv = Rm <= D.tol;
          const long long it = D.pt_iters[r];
          if (conv || it >= D.max_iter_point) {
            const int t = D.t_idx[r];
            double* pr = D.path_rec + ((size_t)r * D.T + t) * FSQR_PATH_W;
            pr[0] = (double)it;
            pr[1] = Rp;
            pr[2] = Rb;
            pr[3] = Rz;
            pr[4] = obj;
            pr[5] = a[4];
            pr[6] = conv ? 1.0 : 0.0;
            pr[7] = sc[2];   // sum_i rho_tau(y_i - x~_i^T beta^k): HBIC of the point (E18)
            s_rec[r] = t;
            if (t == D.T - 1) {
              D.status[r] = conv ? ST_CONVERGED : ST_MAXITER;
              D.commit_iter[r] = C.k;
            } else {
              // w^k initialises lambda_{t+1} (L412): discard this iteration's update for r
              D.status[r] = ST_SWITCH;
              D.t_idx[r] = t + 1;
              D.lam_cur[r] = D.lam_path[(size_t)r * D.T + t + 1];
              D.pt_iters[r] = 0;
            }
          } else {
            D.pt_iters[r] = it + 1;
          }
        } else if (D.check) {
          if (Rm <= D.tol) {
            D.status[r] = ST_CONVERGED;
            D.commit_iter[r] = C.k;
          } else if (C.k - *D.kbase >= D.max_iter) {
            D.status[r] = ST_MAXITER;
            D.commit_iter[r] = C.k;
          }
        }
      }
    }
  }
  __syncthreads();
  // ---------------- path: the sparse solution beta^k of each recorded RHS, in index order
  // (deterministic: a block-wide ordered compaction of the dense column), capped at path_cap
  // (the true count is stored; fsqr_path_beta reports truncation).  An RHS that switches lambda
  // also gets beta^k copied over the beta^{k+1} this pass wrote (ST_SWITCH).
  if (D.update && D.path) {
    constexpr int E = 4;   // consecutive coefficients per thread and step
    __shared__ int s_wtot[32];
    __shared__ long long s_base;
    for (int r = 0; r < C.R; ++r) {
      const int t = s_rec[r];
      if (t < 0) continue;
      const bool sw = D.status[r] == ST_SWITCH;
      const size_t base = ((size_t)r * D.T + t) * D.path_cap;
      if (tid == 0) s_base = 0;
      __syncthreads();
      for (int64_t j0 = 0; j0 <= D.p; j0 += (int64_t)E * blockDim.x) {
        double v[E];
        int c = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int64_t j = j0 + (int64_t)E * tid + e;
          v[e] = 0.0;
          if (j <= D.p) {
            v[e] = C.beta_in[j * C.R + r];
            if (sw) C.beta_out[j * C.R + r] = v[e];
          }
          c += v[e] != 0.0;
        }
        int incl = c;   // inclusive warp scan of the per-thread counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        if (lane == 31) s_wtot[wid] = incl;
        __syncthreads();
        long long off = s_base + incl - c;
        for (int w = 0; w < wid; ++w) off += s_wtot[w];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (v[e] != 0.0) {
            if (off < D.path_cap) {
              D.path_idx[base + off] = (int32_t)(j0 + (int64_t)E * tid + e);
              D.path_beta[base + off] = v[e];
            }
            ++off;
          }
        }
        __syncthreads();
        if (tid == 0) {
          long long tot = 0;
          for (int w = 0; w < nw; ++w) tot += s_wtot[w];
          s_base += tot;
        }
        __syncthreads();
      }
      if (tid == 0) D.path_cnt[(size_t)r * D.T + t] = s_base;
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (D.update) {
      int any = 0;
      for (int r = 0; r < D.R; ++r) any |= (D.status[r] == ST_ACTIVE || D.status[r] == ST_SWITCH);
      *D.stop = any ? 0 : 1;
    }
    *D.ticket = 0u;
  }
}
