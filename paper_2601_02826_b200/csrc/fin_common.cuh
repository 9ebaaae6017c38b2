// fin_common.cuh — the n-vector half of one FS-QRPPA iteration (a3, a5 and the n-vector parts of
// a6), shared by the stand-alone finalize kernel (kfin.cu, used after the CUDA-core forward
// product) and the finalize fused into the tensor-core forward product (k1_tcp.cu):
//
//   s^{k+1}_i   = 2^-E (n S_i - M)/n + beta_0^{k+1}        (a4 result: exact int64 sums, intercept)
//   z^{k+1}     = E15(z^k, theta^k)
//   r^{k+1}     = s^{k+1} + z^{k+1} - y
//   theta^{k+1} = theta^k - mu/(G+1) (2 r^{k+1} - r^k)     E12, L253-254
//   partial sums of ||r||^2, ||z||^2, ||n theta||^2, ||z - P_tau(z + n theta)||^2, sum rho_tau,
//   sum theta, ||y||^2, max|theta| (reading R1), and the int8 digit planes of theta^{k+1}.
//
// Unit of work: a RECORD = 256 consecutive rows of one RHS, computed by a group of 256 threads
// (one row per thread, named barrier).  Records are reduced in a fixed order (fin_reduce_warp), so
// the result is bitwise the same whichever kernel computed the records.
#pragma once
#include "fsqr_dev.cuh"

constexpr int FG = 256;   // threads per finalize group = rows per record



__device__ __forceinline__ void grp_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(FG) : "memory"); }

// group reductions (t = thread index in the group): fixed butterfly within warps, then warp 0
// combines the 8 warp sums with a second butterfly.  sm: 32 * NV + NV doubles.
template <int NV>
__device__ __forceinline__ void grp_sum(double (&v)[NV], double* sm, int t, int bar) {
  const int lane = t & 31, wid = t >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double x = warp_sum_d(v[q]);
    if (lane == 0) sm[wid * NV + q] = x;
  }
  grp_bar(bar);
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = lane < FG / 32 ? sm[lane * NV + q] : 0.0;
      x = warp_sum_d(x);
      if (lane == 0) sm[32 * NV + q] = x;
    }
  }
  grp_bar(bar);
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = sm[32 * NV + q];
  grp_bar(bar);
}

__device__ __forceinline__ long long grp_sum_ll(long long v, long long* sm, int t, int bar) {
  const int lane = t & 31, wid = t >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sm[wid] = v;
  grp_bar(bar);
  if (wid == 0) {
    long long x = lane < FG / 32 ? sm[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sm[32] = x;
  }
  grp_bar(bar);
  const long long r = sm[32];
  grp_bar(bar);
  return r;
}

// max of finite values; a non-finite value wins (it flags the numeric error downstream)
__device__ __forceinline__ double grp_max(double v, double* sm, int t, int bar) {
  const int lane = t & 31, wid = t >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[wid] = v;
  grp_bar(bar);
  if (wid == 0) {
    double x = lane < FG / 32 ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sm[32] = x;
  }
  grp_bar(bar);
  const double r = sm[32];
  grp_bar(bar);
  return r;
}

__device__ __forceinline__ double rho_tau(double u, double tau) { return (tau - (u < 0.0 ? 1.0 : 0.0)) * u; }

// theta_i -> T = round(theta_i / delta) and its balanced base-256 digits in rows 4r..4r+3 of Bq
__device__ __forceinline__ long long quant_row(const Dev& D, int r, int i, double th, double inv) {
  long long T = isfinite(th) ? __double2ll_rn(th * inv) : 0;
  const long long Tr = T;
  int8_t* b0 = D.Bq + (int64_t)(4 * r) * D.ldk;
  const int d3 = (int)(int8_t)(T & 0xFF);
  T = (T - d3) >> 8;
  const int d2 = (int)(int8_t)(T & 0xFF);
  T = (T - d2) >> 8;
  const int d1 = (int)(int8_t)(T & 0xFF);
  T = (T - d1) >> 8;
  const int ix = bq_index(D, i);
  b0[ix] = (int8_t)T;
  b0[D.ldk + ix] = (int8_t)d1;
  b0[2 * D.ldk + ix] = (int8_t)d2;
  b0[3 * D.ldk + ix] = (int8_t)d3;
  return Tr;
}

__device__ __forceinline__ int theta_exponent(double mx) {
  int ex = 0;
  if (mx > 0.0 && isfinite(mx)) frexp(mx, &ex);
  return ex;
}

// per-RHS constants of one finalize (iteration k, RHS r); mt = the colsum term M of the forward sums
struct FinRHS {
  double b0, tau, tn, un, inv_scale, inv_prev;
  long long mt;
};

__device__ __forceinline__ FinRHS fin_rhs(const Dev& D, int r, long long k, long long mt) {
  const int par = (int)(k & 1), par1 = par ^ 1;
  FinRHS c;
  // intercept: lambda_0 = 0, so E14 gives beta_0 + g_0 / eta_1 with g_0 = sum theta^k
  c.b0 = D.beta[par][r] + D.sumth[r] / D.eta[0];
  c.tau = D.tau[r];
  c.tn = c.tau / ((double)D.n * D.mu);
  c.un = (1.0 - c.tau) / ((double)D.n * D.mu);
  const int cnt = D.sup_cnt[par1];
  const double cm = __longlong_as_double((long long)D.cmax[par1 * D.R + r]);
  c.inv_scale = ldexp(1.0, -fwd_exponent(cm, cnt, D.n));
  c.inv_prev = 1.0 / D.delta[r];   // 1/delta^k, exact (a power of two)
  c.mt = mt;
  return c;
}

// The state rows a record batch reads that do not depend on this iteration's forward product
// (z^k, theta^k, r^k, y): loaded before the forward sums are complete (fin_load), so that after
// them only the accumulators remain on the critical path.
template <int NB>
struct FinRows {
  double zo[NB], th[NB], ro[NB], yi[NB];
};

template <int NB>
__device__ __forceinline__ void fin_load(const Dev& D, int r, int b0, int nb, int t, FinRows<NB>& w) {
  const int n = D.n;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int i = (b0 + q) * FG + t;
    const bool ok = q < nb && i < n;
    const int64_t o = (int64_t)r * n + i;
    w.zo[q] = ok ? D.z[o] : 0.0;
    w.th[q] = ok ? D.theta[o] : 0.0;
    w.ro[q] = ok ? D.rres[o] : 0.0;
    w.yi[q] = ok ? D.y[i] : 0.0;
  }
}

// Records b0 .. b0 + nb - 1 (nb <= NB) of RHS r, thread t taking row 256 (b0 + q) + t of each
// (rows pre-loaded by fin_load).  Each record is reduced the same way wherever it is computed: a
// butterfly within each warp, then the 8 warp sums added in warp order (max and int64 alike).
// Writes fpart[b][r][0..7] and ftsum[b][r].  sm: NB * 8 * 9 doubles.  Group-wide call.
template <int NB>
__device__ __forceinline__ void fin_records(const Dev& D, int r, int b0, int nb, const FinRHS& c, int t, int bar,
                                            double* sm, const FinRows<NB>& w) {
  const int n = D.n, lane = t & 31, wid = t >> 5;
  const double mu = D.mu, sig = D.sigma;
  double sa[NB];
  const double *zo = w.zo, *th = w.th, *ro = w.ro, *yi = w.yi;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int i = (b0 + q) * FG + t;
    const bool ok = q < nb && i < n;
    sa[q] = ok ? (double)((long long)n * __ldcg(D.sacc + (int64_t)r * n + i) - c.mt) : 0.0;
  }
  double acc[NB][8];
  long long ts[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int i = (b0 + q) * FG + t;
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[q][v] = 0.0;
    ts[q] = 0;
    if (q < nb && i < n) {
      const int64_t o = (int64_t)r * n + i;
      const double sv = sa[q] * c.inv_scale / (double)n + c.b0;
      const double zn = pos_part(zo[q] + th[q] / mu - c.tn) - pos_part(-zo[q] - th[q] / mu - c.un);   // E15
      const double rn = sv + zn - yi[q];
      const double thn = th[q] - sig * (2.0 * rn - ro[q]);                                             // E12
      D.z[o] = zn;
      D.theta[o] = thn;
      D.rres[o] = rn;
      D.s[o] = sv;
      const double nt = (double)n * thn;
      const double dz = zn - prox_rho1(zn + nt, c.tau);
      acc[q][0] = rn * rn;
      acc[q][1] = zn * zn;
      acc[q][2] = nt * nt;
      acc[q][3] = dz * dz;
      acc[q][4] = rho_tau(yi[q] - sv, c.tau);
      acc[q][5] = thn;
      acc[q][6] = yi[q] * yi[q];
      acc[q][7] = isfinite(thn) ? fabs(thn) : thn;
      ts[q] = quant_row(D, r, i, thn, c.inv_prev);   // provisional: the exponent of delta^k
    }
  }
  // warp level, all records and values interleaved level by level (the same butterfly per value as
  // warp_sum_d; lane 0 ends with the warp's values)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
#pragma unroll
      for (int v = 0; v < 7; ++v) acc[q][v] += __shfl_xor_sync(0xffffffffu, acc[q][v], o);
      acc[q][7] = fmax(acc[q][7], __shfl_xor_sync(0xffffffffu, acc[q][7], o));
      ts[q] += __shfl_xor_sync(0xffffffffu, ts[q], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      double* w = sm + (q * 8 + wid) * 9;
#pragma unroll
      for (int v = 0; v < 8; ++v) w[v] = acc[q][v];
      w[8] = __longlong_as_double(ts[q]);
    }
  }
  grp_bar(bar);
  // record level: thread (q, v) adds the 8 warp values in warp order
  if (t < nb * 9) {
    const int q = t / 9, v = t % 9;
    const double* w = sm + q * 8 * 9 + v;
    const int b = b0 + q;
    if (v < 7) {
      double a = w[0];
      for (int u = 1; u < 8; ++u) a += w[u * 9];
      D.fpart[((size_t)b * D.R + r) * FSQR_FPART + v] = a;
    } else if (v == 7) {
      double m = w[0];
      for (int u = 1; u < 8; ++u) m = fmax(m, w[u * 9]);
      D.fpart[((size_t)b * D.R + r) * FSQR_FPART + 7] = m;
    } else {
      long long a = __double_as_longlong(w[0]);
      for (int u = 1; u < 8; ++u) a += __double_as_longlong(w[u * 9]);
      D.ftsum[(size_t)b * D.R + r] = a;
    }
  }
  grp_bar(bar);
}

// All nblk records of RHS r are written: reduce them in record order, publish R_p, R_z, the loss
// and sum theta^{k+1}, beta_0^{k+1}, and fix the digit planes if max|theta^{k+1}| left the binade
// of delta^k (then every row is re-quantised with delta^{k+1} = 2^(e-28)).  Group-wide call.
// All nblk records of RHS r are written: ONE WARP reduces them in record order (lane l adds records
// l, l + 32, ..., all nine values of a record in one round of loads; then a level-major butterfly),
// and lane 0 publishes R_p, R_z, the loss and sum theta^{k+1}, beta_0^{k+1} and delta^{k+1}.
// Returns (on every lane) whether max|theta^{k+1}| / delta^k left [2^26, 2^28): then every row must be
// re-quantised with delta^{k+1} = 2^(e-28) (fin_requant).  Several RHS reduce on different warps.
__device__ __forceinline__ bool fin_reduce_warp(const Dev& D, int r, int nblk, double b0, long long k, int lane,
                                                bool commit = true) {
  double a[7] = {0, 0, 0, 0, 0, 0, 0};
  double mx = 0.0;
  long long tsum = 0;
  const double dprev = D.delta[r];   // issued with the record loads (one memory latency in all)
  // records lane, lane + 32, ... in that order; two per lane per round, every load of a round issued
  // before the first add (one memory latency per 64 records)
  for (int bb = 0; bb < nblk; bb += 64) {
    double v[2][8];
    long long ts[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int b = bb + 32 * u + lane;
      const bool ok = b < nblk;
      const double* fp = D.fpart + ((size_t)(ok ? b : 0) * D.R + r) * FSQR_FPART;
#pragma unroll
      for (int q = 0; q < 8; ++q) v[u][q] = ok ? __ldcg(fp + q) : 0.0;
      ts[u] = ok ? __ldcg(D.ftsum + (size_t)b * D.R + r) : 0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (bb + 32 * u + lane >= nblk) break;
#pragma unroll
      for (int q = 0; q < 7; ++q) a[q] += v[u][q];
      mx = (v[u][7] > mx || !isfinite(v[u][7])) ? v[u][7] : mx;
      tsum += ts[u];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < 7; ++q) a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
    const double m = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (m > mx || !isfinite(m)) ? m : mx;
    tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
  }
  // The scale delta^k is kept while max|theta^{k+1}| / delta^k stays in [2^26, 2^28): every T then
  // has 26..28 significant bits and |T| < 2^28 (the int64 bounds of K2's reconstruction).  Leaving
  // that range (one binade of hysteresis downwards, none upwards) re-quantises every row with
  // delta^{k+1} = 2^(e - 28), e the binary exponent of max|theta^{k+1}|.
  const int e_new = theta_exponent(mx);
  const int e_old = theta_exponent(dprev * ldexp(1.0, 28) * 0.75);   // delta^k = 2^(e_old - 28)
  const bool live = mx > 0.0 && isfinite(mx);
  const bool requant = !live || e_new > e_old || e_new < e_old - 1;
  const double rp = sqrt(a[0]) / (1.0 + sqrt(a[6]));
  const double rz = sqrt(a[3]) / (1.0 + sqrt(a[1]) + sqrt(a[2]));
  const double dnew = !requant ? dprev : (live ? ldexp(1.0, e_new - 28) : 1.0);
  if (commit && lane == 0) {
    double* sc = D.scal + r * FSQR_NSCAL;
    sc[0] = rp;
    sc[1] = rz;
    sc[2] = a[4];
    sc[3] = a[6];
    D.beta[(int)(k & 1) ^ 1][r] = b0;
    D.sumth[r] = a[5];
    if (!requant) D.Tsum[r] = tsum;
    D.delta[r] = dnew;
  }
  return requant;
}

// re-quantise every row of RHS r with delta^{k+1} (already published); group-wide call
__device__ __forceinline__ void fin_requant(const Dev& D, int r, int t, int bar, long long* smll) {
  const int n = D.n;
  const double inv = 1.0 / D.delta[r];
  long long t2 = 0;
  for (int ii = t; ii < n; ii += FG) t2 += quant_row(D, r, ii, D.theta[(int64_t)r * n + ii], inv);
  t2 = grp_sum_ll(t2, smll, t, bar);
  if (t == 0) D.Tsum[r] = t2;
  grp_bar(bar);
}

// every active RHS's records: warp w of the group reduces RHS w, w + 8, ...; then the rare
// re-quantisations, group-wide.  b0 per RHS from the state before this call (beta^k, sum theta^k).
// commit = false: the same code path without any store (a dry run that warms the instruction cache
// of a CTA that will reduce once the records are complete).
__device__ __forceinline__ void fin_reduce_all(const Dev& D, int nblk, long long k, int t, int bar, long long* smll,
                                               bool commit = true) {
  __shared__ unsigned s_req;
  const int lane = t & 31, wid = t >> 5;
  if (t == 0) s_req = 0u;
  grp_bar(bar);
  for (int r = wid; r < D.R; r += FG / 32) {
    // status, beta_0, sum theta and the records are loaded together; an RHS that is not active
    // (its records were not written this iteration) publishes nothing
    const int st = D.status[r];
    const double b0 = D.beta[(int)(k & 1)][r] + D.sumth[r] / D.eta[0];   // E14 with lambda_0 = 0, g_0 = sum theta^k
    const bool act = st == ST_ACTIVE;
    if (fin_reduce_warp(D, r, nblk, b0, k, lane, commit && act) && act && lane == 0) atomicOr(&s_req, 1u << r);
  }
  grp_bar(bar);
  const unsigned req = commit ? s_req : 0u;
  for (int r = 0; r < D.R; ++r)
    if (req & (1u << r)) fin_requant(D, r, t, bar, smll);
}

// iteration tail (after every RHS is reduced): clear the forward scale and support count of the
// list just consumed, advance the iteration counter, re-activate RHS that switched lambda
__device__ __forceinline__ void fin_iteration_tail(const Dev& D, long long k, int t) {
  const int par = (int)(k & 1);
  if (t < D.R) {
    D.cmax[par * D.R + t] = 0ull;
    if (D.status[t] == ST_SWITCH) D.status[t] = ST_ACTIVE;   // re-test w^k at lambda_{t+1}
  }
  if (t == 0) {
    D.sup_cnt[par] = 0;
    *D.iter = k + 1;
  }
}
