// kfin.cu — a3 + a5 + a6 (n-vector part) and the setup kernels.
//
// finalize (one CTA, 1024 threads, fixed-order reductions):
//   s^{k+1}_i = 2^-E (n S_i - M)/n + beta_0^{k+1}       (a4 result, intercept added here)
//   z^{k+1}   = E15(z^k, theta^k)
//   r^{k+1}   = s^{k+1} + z^{k+1} - y
//   theta^{k+1} = theta^k - mu/(G+1) (2 r^{k+1} - r^k)   E12, L253-254
//   R_p, R_z (w^{k+1}), loss, sum theta, and the digit planes of theta^{k+1}
//   for the next X~^T theta pass.
// Setup: column statistics (a0), power method pieces (a0'), lambda_max, state init.
#include "fin_common.cuh"

namespace {

constexpr int FT = 1024;

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double x = warp_sum_d(v[q]);
    if (lane == 0) sm[wid * NV + q] = x;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double x = lane < nw ? sm[lane * NV + q] : 0.0;
      x = warp_sum_d(x);
      if (lane == 0) sm[32 * NV + q] = x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = sm[32 * NV + q];
  __syncthreads();
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  if (wid == 0) {
    long long x = lane < nw ? sm[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sm[32] = x;
  }
  __syncthreads();
  const long long r = sm[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double block_max(double v, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sm[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double x = lane < nw ? sm[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sm[32] = x;
  }
  __syncthreads();
  const double r = sm[32];
  __syncthreads();
  return r;
}


// theta -> balanced base-256 digit planes (rows 4r..4r+3 of Bq); returns sum T (exact)
__device__ void quantize_theta(const Dev& D, int r, double mx, long long* smll) {
  const int n = D.n;
  int ex = 0;
  double dlt = 1.0;
  if (mx > 0.0 && isfinite(mx)) {
    frexp(mx, &ex);          // mx < 2^ex
    dlt = ldexp(1.0, ex - 28);
  }
  const double inv = 1.0 / dlt;  // exact (power of two)
  long long ts = 0;
  int8_t* b0 = D.Bq + (int64_t)(4 * r) * D.ldk;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double th = D.theta[(int64_t)r * n + i];
    long long T = isfinite(th) ? __double2ll_rn(th * inv) : 0;
    ts += T;
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
  }
  ts = block_sum_ll(ts, smll);
  if (threadIdx.x == 0) {
    D.Tsum[r] = ts;
    D.delta[r] = dlt;
  }
}

// shared n-vector step: from s (already including beta_0), update z, theta, r and the per-RHS scalars
// mode 0: iteration (a3+a5), mode 1: state init (z, theta given; only r and the scalars)
__device__ void nvec_step(const Dev& D, int r, int mode, double b0, int fwd_par, double* smd, long long* smll) {
  const int n = D.n;
  const double tau = D.tau[r];
  const double mu = D.mu, sig = D.sigma;
  const double tn = tau / ((double)n * mu), un = (1.0 - tau) / ((double)n * mu);
  int E = 0;
  long long mt = 0;
  if (D.storage != 0) {
    const int cnt = D.sup_cnt[fwd_par];
    const double cm = __longlong_as_double((long long)D.cmax[fwd_par * D.R + r]);
    E = fwd_exponent(cm, cnt, n);
    mt = D.mterm[r];
  }
  const double inv_scale = ldexp(1.0, -E);
  double acc[7] = {0, 0, 0, 0, 0, 0, 0};  // rr, zz, tt, rzz, loss, sumth, yy
  double mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t o = (int64_t)r * n + i;
    double sv;
    if (D.storage == 0) {
      sv = D.sdense[o] + b0;
    } else {
      sv = (double)((long long)n * D.sacc[o] - mt) * inv_scale / (double)n + b0;
      D.sacc[o] = 0;
    }
    const double yi = D.y[i];
    double zn, thn;
    if (mode == 0) {
      const double zo = D.z[o], th = D.theta[o], ro = D.rres[o];
      zn = pos_part(zo + th / mu - tn) - pos_part(-zo - th / mu - un);   // E15
      const double rn = sv + zn - yi;
      thn = th - sig * (2.0 * rn - ro);                                   // E12
      D.z[o] = zn;
      D.theta[o] = thn;
      D.rres[o] = rn;
      acc[0] += rn * rn;
    } else {
      zn = D.z[o];
      thn = D.theta[o];
      const double rn = sv + zn - yi;
      D.rres[o] = rn;
      acc[0] += rn * rn;
    }
    D.s[o] = sv;
    const double nt = (double)n * thn;
    const double dz = zn - prox_rho1(zn + nt, tau);
    acc[1] += zn * zn;
    acc[2] += nt * nt;
    acc[3] += dz * dz;
    acc[4] += rho_tau(yi - sv, tau);
    acc[5] += thn;
    acc[6] += yi * yi;
    mx = fmax(mx, fabs(thn));
    if (!isfinite(thn)) mx = thn;
  }
  block_sum<7>(acc, smd);
  mx = block_max(mx, smd);
  if (threadIdx.x == 0) {
    double* sc = D.scal + r * FSQR_NSCAL;
    sc[0] = sqrt(acc[0]) / (1.0 + sqrt(acc[6]));
    sc[1] = sqrt(acc[3]) / (1.0 + sqrt(acc[1]) + sqrt(acc[2]));
    sc[2] = acc[4];
    sc[3] = acc[6];
    D.sumth[r] = acc[5];
    D.mterm[r] = 0;
  }
  if (D.storage != 0) quantize_theta(D, r, mx, smll);
  __syncthreads();
}

__global__ void __launch_bounds__(FT) k_finalize(const Dev D) {
  __shared__ double smd[32 * 8 + 8];
  __shared__ long long smll[33];
  pdl_launch_dependents();
  pdl_wait();
  if (*D.stop) return;
  const long long k = *D.iter;
  const int par = (int)(k & 1), par1 = par ^ 1;
  for (int r = 0; r < D.R; ++r) {
    if (D.status[r] != ST_ACTIVE) continue;
    // intercept: lambda_0 = 0, so E14 gives beta_0 + g_0/eta_1 with g_0 = sum theta^k
    const double b0 = D.beta[par][r] + D.sumth[r] / D.eta[0];
    if (threadIdx.x == 0) D.beta[par1][r] = b0;
    nvec_step(D, r, 0, b0, par1, smd, smll);
  }
  __syncthreads();
  if (threadIdx.x < D.R) {
    D.cmax[par * D.R + threadIdx.x] = 0ull;
    if (D.status[threadIdx.x] == ST_SWITCH) D.status[threadIdx.x] = ST_ACTIVE;   // re-test w^k at lambda_{t+1}
  }
  if (threadIdx.x == 0) {
    D.sup_cnt[par] = 0;
    *D.iter = k + 1;
  }
}

// ---------------------------------------------------------------- multi-CTA finalize
// The n-vector step after the CUDA-core forward product (k1_bulk; the tensor-core forward product
// k1_tcp runs the same records in its own tail, fin_common.cuh).  Grid (ceil(n/256), R): CTA
// (x, r) computes record x of RHS r (rows 256x.., one row per thread), quantising theta^{k+1}
// provisionally with the previous exponent; the last CTA of RHS r (ticket fticket[1 + r]) reduces
// its records in order and re-quantises only on a binade change; the last CTA overall runs the
// iteration tail.

__global__ void __launch_bounds__(FIN_THREADS) k_finalize_mc(const Dev D) {
  static_assert(FIN_THREADS == FG, "one record per CTA");
  __shared__ double smd[32 * 8 + 8];
  __shared__ long long smll[33];
  __shared__ bool s_last;
  pdl_launch_dependents();
  pdl_wait();
  if (*D.stop) return;
  const long long k = *D.iter;
  const int r = blockIdx.y, t = threadIdx.x;
  const int nblk = gridDim.x;
  if (D.status[r] == ST_ACTIVE) {
    const FinRHS c = fin_rhs(D, r, k, D.mterm[r]);
    FinRows<1> w;
    fin_load<1>(D, r, blockIdx.x, 1, t, w);
    fin_records<1>(D, r, blockIdx.x, 1, c, t, 0, smd, w);
    fence_acq_rel_gpu();
    __syncthreads();
    if (t == 0) s_last = atomicAdd(D.fticket + 1 + r, 1u) == (unsigned)nblk - 1;
    __syncthreads();
    if (s_last) {
      fence_acq_rel_gpu();
      __shared__ int s_req;
      if (t < 32) {
        const bool req = fin_reduce_warp(D, r, nblk, c.b0, k, t);
        if (t == 0) s_req = req ? 1 : 0;
      }
      __syncthreads();
      if (s_req) fin_requant(D, r, t, 0, smll);
      if (t == 0) {
        D.mterm[r] = 0;
        D.fticket[1 + r] = 0u;
      }
      if (D.R == 1) {   // one RHS: its last CTA is the last CTA overall, no second ticket round
        fin_iteration_tail(D, k, t);
        return;
      }
    }
    if (D.R == 1) return;
  }
  // ------------------------------------------------ last CTA overall: iteration tail
  fence_acq_rel_gpu();
  __syncthreads();
  if (t == 0) s_last = atomicAdd(D.fticket, 1u) == (unsigned)(nblk * D.R) - 1;
  __syncthreads();
  if (!s_last) return;
  fence_acq_rel_gpu();
  fin_iteration_tail(D, k, t);
  if (t == 0) *D.fticket = 0u;
}

// state init after create / set_state: s from the support list of the current parity (k1 in cur mode)
__global__ void __launch_bounds__(FT) k_init_state(const Dev D) {
  __shared__ double smd[32 * 8 + 8];
  __shared__ long long smll[33];
  const long long k = *D.iter;
  const int par = (int)(k & 1);
  for (int r = 0; r < D.R; ++r) nvec_step(D, r, 1, D.beta[par][r], par, smd, smll);
  __syncthreads();
}

// ---------------------------------------------------------------- setup kernels

// u8 -> PACKED2 repack (fsqr_pack2): one thread per packed 32-bit word = 16 samples of one column.
// Byte b of the word holds samples 16j+4b..16j+4b+3 at bits 2(i%4): for a little-endian word
// a = x0|x1<<8|x2<<16|x3<<24 with every x <= 3, (a | a>>6 | a>>12 | a>>18) & 0xFF.
__global__ void k_pack2(const uint8_t* __restrict__ x8, int64_t ld8, int n, int64_t p, uint32_t* __restrict__ x2,
                        int64_t ld2, int* bad) {
  const int64_t wpc = ld2 / 4;   // packed words per column
  const int64_t total = p * wpc;
  int flag = 0;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = w / wpc;
    const int i0 = (int)(w - c * wpc) * 16;
    uint32_t a[4];
    const uint8_t* src = x8 + c * ld8 + i0;
    if (i0 + 16 <= n) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src));
      a[0] = v.x, a[1] = v.y, a[2] = v.z, a[3] = v.w;
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        uint32_t u = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (i0 + 4 * b + e < n) u |= (uint32_t)src[4 * b + e] << (8 * e);
        a[b] = u;
      }
    }
    uint32_t out = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      flag |= (a[b] & 0xFCFCFCFCu) != 0;
      out |= ((a[b] | (a[b] >> 6) | (a[b] >> 12) | (a[b] >> 18)) & 0xFFu) << (8 * b);
    }
    x2[w] = out;
  }
  if (__syncthreads_or(flag) && threadIdx.x == 0) atomicOr(bad, 1);
}

template <int ST>
__global__ void k_colstats_int(const Dev D, int32_t* colsum, double* mean, double* inv_sd, double* sd, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = gw; c < D.p; c += nw) {
    const uint8_t* col = D.X8 + c * D.ld;
    long long s1 = 0, s2 = 0;
    // 16-byte loads over the stored bytes of the column (the padding past n is zero, so it adds 0):
    // u8 sums by dp4a (sum of bytes, sum of squares); 2-bit codes c = b0 + 2 b1 by popcounts:
    // sum c = |b0| + 2|b1|, sum c^2 = |b0| + 4|b1| + 4|b0 b1|
    const int nb = (int)min(D.ld, (int64_t)(ST == 1 ? (D.n + 15) / 16 * 16 : ((D.n + 3) / 4 + 15) / 16 * 16));
    for (int off = lane * 16; off < nb; off += 512) {
      const uint4 v = __ldcs((const uint4*)(col + off));
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
      // samples past n in the last chunk are masked (the layout's padding is zero, but do not rely on it)
      const int valid = ST == 1 ? D.n - off : D.n - 4 * off;   // samples of this chunk that exist
      if (valid < (ST == 1 ? 16 : 64)) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int k = valid - (ST == 1 ? 4 : 16) * q;   // samples of word q that exist
          const int bits = k <= 0 ? 0 : (ST == 1 ? 8 * k : 2 * k);
          if (bits < 32) w[q] &= bits == 0 ? 0u : (0xFFFFFFFFu >> (32 - bits));
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (ST == 1) {
          s1 += (unsigned)__dp4a(w[q], 0x01010101u, 0u);
          s2 += (unsigned)__dp4a(w[q], w[q], 0u);
        } else {
          const uint32_t lo = w[q] & 0x55555555u, hi = w[q] & 0xAAAAAAAAu;
          const int a = __popc(lo), b = __popc(hi), ab = __popc(lo & (hi >> 1));
          s1 += a + 2 * b;
          s2 += a + 4 * b + 4 * ab;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      const long long n = D.n;
      const long long num = n * s2 - s1 * s1;   // n(n-1) * sample variance, exact
      colsum[c] = (int32_t)s1;
      mean[c] = (double)s1 / (double)n;
      const double v = (double)num / ((double)n * (double)(n - 1));
      const double s = sqrt(v);
      sd[c] = s;
      inv_sd[c] = 1.0 / s;
      if (num <= 0) atomicMin(bad, (int)c);
    }
  }
}

__global__ void k_colstats_f32(const Dev D, double* mean, double* inv_sd, double* sd, int* bad) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = gw; c < D.p; c += nw) {
    const float* col = D.Xf + c * D.ld;
    double s1 = 0.0;
    for (int i = lane; i < D.n; i += 32) s1 += (double)col[i];
    s1 = warp_sum_d(s1);
    const double m = s1 / (double)D.n;
    double s2 = 0.0;
    for (int i = lane; i < D.n; i += 32) {
      const double d = (double)col[i] - m;
      s2 += d * d;
    }
    s2 = warp_sum_d(s2);
    if (lane == 0) {
      const double s = sqrt(s2 / (double)(D.n - 1));
      mean[c] = m;
      sd[c] = s;
      inv_sd[c] = 1.0 / s;
      if (!(s > 0.0)) atomicMin(bad, (int)c);
    }
  }
}

__device__ __forceinline__ double xt_raw(const Dev& D, int64_t c, int i) {
  if (D.storage == 0) return (double)D.Xf[c * D.ld + i];
  if (D.storage == 1) return (double)D.X8[c * D.ld + i];
  return (double)((D.X8[c * D.ld + (i >> 2)] >> (2 * (i & 3))) & 3);
}

// power method start vector: 2U - 1, U from the splitmix64 finaliser keyed by (seed, j)
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void k_power_start(int64_t p1, uint64_t seed, double* v) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p1; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(seed ^ mix64((uint64_t)j));
    v[j] = 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
  }
}

// u[g][i] = sum_{j in block g} x~_ij v_j (ascending j), thread per (i, g)
__global__ void k_power_fwd(const Dev D, const int64_t* bstart, const double* v, const int* frozen, double* u) {
  const int g = blockIdx.y;
  if (frozen[g]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D.n) return;
  const int64_t j0 = bstart[g], j1 = bstart[g + 1];
  double a = 0.0;
  for (int64_t j = j0; j < j1; ++j) {
    const double vj = v[j];
    if (j == 0) {
      a = fma(1.0, vj, a);
      continue;
    }
    const int64_t c = j - 1;
    a = fma((xt_raw(D, c, i) - D.mean[c]) * D.inv_sd[c], vj, a);
  }
  u[(int64_t)g * D.n + i] = a;
}

// w_j = sum_i x~_ij u_{g(j), i}  (warp per model column, fixed butterfly); optional max |w_j| (j >= 1)
__global__ void k_back_f64(const Dev D, const double* u, int per_block, const int* frozen, double* w,
                           unsigned long long* maxbits) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = gw; j <= D.p; j += nw) {
    const int g = per_block ? block_of_col(D, j) : 0;
    if (frozen && frozen[g]) continue;
    const double* ug = u + (int64_t)g * D.n;
    double a = 0.0;
    if (j == 0) {
      for (int i = lane; i < D.n; i += 32) a += ug[i];
    } else {
      const int64_t c = j - 1;
      const double m = D.mean[c], isd = D.inv_sd[c];
      for (int i = lane; i < D.n; i += 32) a = fma((xt_raw(D, c, i) - m) * isd, ug[i], a);
    }
    a = warp_sum_d(a);
    if (lane == 0) {
      if (w) w[j] = a;
      if (maxbits && j >= 1) atomicMax(maxbits, (unsigned long long)__double_as_longlong(fabs(a)));
    }
  }
}

// ---- genotype-storage power / lambda_max products (a0', R3-R4): 16 rows per thread, vector loads

// a small unsigned integer as a double without the quarter-rate I2F.F64: (2^52 + c) - 2^52, exact
__device__ __forceinline__ double code_to_double(uint32_t c) {
  return __hiloint2double(0x43300000, (int)c) - 4503599627370496.0;
}

// codes of rows i0..i0+15 of data column c (u8: one 16-byte load; 2-bit: one 4-byte load)
template <int ST>
__device__ __forceinline__ void codes16(const Dev& D, int64_t c, int i0, double (&x)[16]) {
  if (ST == 1) {
    const uint4 v = __ldcs((const uint4*)(D.X8 + c * D.ld + i0));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = code_to_double((w[q >> 2] >> (8 * (q & 3))) & 0xFFu);
  } else {
    const uint32_t w = __ldcs((const uint32_t*)(D.X8 + c * D.ld + (i0 >> 2)));
#pragma unroll
    for (int q = 0; q < 16; ++q) x[q] = code_to_double((w >> (2 * q)) & 3u);
  }
}

// part[s][g][i] = sum over the s-th of S contiguous slices of block g of x~_ij v_j
//              = sum_j x_ij (v_j/s_j) - sum_j m_j v_j / s_j   (+ v_0 for the intercept)
template <int ST>
__global__ void __launch_bounds__(128) k_power_fwd_int(const Dev D, const int64_t* bstart, const double* v,
                                                       const int* frozen, double* part, int S) {
  const int g = blockIdx.y, s = blockIdx.z;
  if (frozen[g]) return;
  const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 16;
  if (i0 >= D.n) return;
  const int64_t j0 = bstart[g], len = bstart[g + 1] - j0;
  const int64_t a0 = j0 + len * s / S, a1 = j0 + len * (s + 1) / S;
  double acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0.0;
  double cterm = 0.0;
  // four columns per step with every load issued first (the per-column scalars and codes are
  // otherwise one memory latency per column); the sums keep the column order
  constexpr int U = 4;
  for (int64_t jb = a0; jb < a1; jb += U) {
    double vj[U], isd[U], mn[U];
    uint4 cw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = jb + u;
      const bool ok = j < a1 && j >= 1;
      const int64_t c = ok ? j - 1 : 0;
      vj[u] = j < a1 ? v[j] : 0.0;
      isd[u] = ok ? D.inv_sd[c] : 0.0;
      mn[u] = ok ? D.mean[c] : 0.0;
      if (ST == 1) cw[u] = ok ? __ldcs((const uint4*)(D.X8 + c * D.ld + i0)) : make_uint4(0, 0, 0, 0);
      else cw[u].x = ok ? __ldcs((const uint32_t*)(D.X8 + c * D.ld + (i0 >> 2))) : 0u;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = jb + u;
      if (j >= a1) break;
      if (j == 0) {
        cterm -= vj[u];
        continue;
      }
      const double a = isd[u] * vj[u];
      cterm = fma(mn[u], a, cterm);
      if (ST == 1) {
        const uint32_t w[4] = {cw[u].x, cw[u].y, cw[u].z, cw[u].w};
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = fma(code_to_double((w[q >> 2] >> (8 * (q & 3))) & 0xFFu), a, acc[q]);
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = fma(code_to_double((cw[u].x >> (2 * q)) & 3u), a, acc[q]);
      }
    }
  }
  double* out = part + ((int64_t)s * D.G + g) * D.n;
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (i0 + q < D.n) out[i0 + q] = acc[q] - cterm;
}

// u[g][i] = sum_s part[s][g][i] (fixed order); Ug[g] = sum_i u[g][i] (fixed block tree)
__global__ void __launch_bounds__(1024) k_sum_parts(const double* part, int S, int G, int n, const int* frozen,
                                                    double* u, double* Ug) {
  __shared__ double smd[33];
  const int g = blockIdx.x;
  if (frozen && frozen[g]) return;
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double a = 0.0;
    for (int ss = 0; ss < S; ++ss) a += part[((int64_t)ss * G + g) * n + i];
    u[(int64_t)g * n + i] = a;
    t += a;
  }
  double tt[1] = {t};
  block_sum<1>(tt, smd);
  if (threadIdx.x == 0) Ug[g] = tt[0];
}

// w_j = sum_i x~_ij u_{g(j),i} = (sum_i x_ij u_i - m_j Ug) / s_j; lane = model column, 16 rows per step
template <int ST>
__global__ void __launch_bounds__(256) k_back_int(const Dev D, const double* u, const double* Ug, int per_block,
                                                  const int* frozen, double* w, unsigned long long* maxbits) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t jb = gw * 32; jb <= D.p; jb += nw * 32) {
    const int64_t j = jb + lane;
    const bool in = j <= D.p;
    const int g = (per_block && in) ? block_of_col(D, j) : 0;
    const bool live = in && !(frozen && frozen[g]);
    const double* ug = u + (int64_t)g * D.n;
    double acc = 0.0;
    const int64_t c = j >= 1 ? j - 1 : 0;
    if (live && j >= 1) {
      if (ST == 2) {
        // 64 rows per 16-byte load (the column stride and i0 / 4 are multiples of 16 bytes; the
        // bytes past n / 4 are zero padding), rows in order: the same sum as 16 at a time
        for (int i0 = 0; i0 < D.n; i0 += 64) {
          const uint4 v = __ldg((const uint4*)(D.X8 + c * D.ld + (i0 >> 2)));
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
          const int lim = min(64, D.n - i0);
#pragma unroll
          for (int q = 0; q < 64; ++q)
            if (q < lim) acc = fma(code_to_double((w[q >> 4] >> (2 * (q & 15))) & 3u), __ldg(ug + i0 + q), acc);
        }
      } else {
        for (int i0 = 0; i0 < D.n; i0 += 16) {
          double x[16];
          codes16<ST>(D, c, i0, x);
          const int lim = min(16, D.n - i0);
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (q < lim) acc = fma(x[q], __ldg(ug + i0 + q), acc);
        }
      }
    }
    if (live) {
      const double wj = (j == 0) ? Ug[g] : (acc - D.mean[c] * Ug[g]) * D.inv_sd[c];
      if (w) w[j] = wj;
      if (maxbits && j >= 1) atomicMax(maxbits, (unsigned long long)__double_as_longlong(fabs(wj)));
    }
  }
}

// per block g (one CTA each): u_g as 28-bit fixed point T_gi = round(u_gi / delta_g), delta_g =
// 2^(e - 28) with e the binary exponent of max_i |u_gi|, split into four signed base-256 digits in
// rows 4g..4g+3 of Bp (the tensor-core K order of bq_index), Tsum_g = sum_i T_gi, gs_g = delta_g / n;
// and w_0 = sum_i u_0i for the intercept (block 0).  The back pass k2p_kernel reads them.
__global__ void __launch_bounds__(FT) k_power_quant(const Dev D, const double* u, const double* Ug, const int* frozen,
                                                    int8_t* Bp, int ldk, long long* Tsum, double* gs, double* w) {
  __shared__ double smd[33];
  __shared__ long long smll[33];
  const int g = blockIdx.x;
  if (frozen[g]) return;
  const double* ug = u + (int64_t)g * D.n;
  double mx = 0.0;
  for (int i = threadIdx.x; i < D.n; i += blockDim.x) mx = fmax(mx, fabs(ug[i]));
  mx = block_max(mx, smd);
  int e = 0;
  if (mx > 0.0 && isfinite(mx)) frexp(mx, &e);
  const double delta = (mx > 0.0 && isfinite(mx)) ? ldexp(1.0, e - 28) : 1.0, inv = 1.0 / delta;
  int8_t* b0 = Bp + (int64_t)(4 * g) * ldk;
  long long ts = 0;
  for (int i = threadIdx.x; i < D.n; i += blockDim.x) {
    long long T = isfinite(ug[i]) ? __double2ll_rn(ug[i] * inv) : 0;
    ts += T;
    const int d3 = (int)(int8_t)(T & 0xFF);
    T = (T - d3) >> 8;
    const int d2 = (int)(int8_t)(T & 0xFF);
    T = (T - d2) >> 8;
    const int d1 = (int)(int8_t)(T & 0xFF);
    T = (T - d1) >> 8;
    const int ix = bq_index(D, i);
    b0[ix] = (int8_t)T;
    b0[ldk + ix] = (int8_t)d1;
    b0[2 * ldk + ix] = (int8_t)d2;
    b0[3 * ldk + ix] = (int8_t)d3;
  }
  ts = block_sum_ll(ts, smll);
  if (threadIdx.x == 0) {
    Tsum[g] = ts;
    gs[g] = delta / (double)D.n;
    if (g == 0) w[0] = Ug[0];
  }
}

// ---- a0' forward pass on the tensor cores (k1_tcp power mode): coefficients, identity entry list,
// and the per-block n-vectors from the exact int64 sums
__global__ void k_iota(int32_t* ix, int64_t p) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < p; c += (int64_t)gridDim.x * blockDim.x)
    ix[c] = (int32_t)c;
}
// a_c = v_{c+1} / s_c for every data column of a live block (0 in a frozen one); bits of max |a_c|
// into both parity slots of cmax
__global__ void k_power_coef(const Dev D, const double* v, const int* frozen, double* a, unsigned long long* cmax) {
  unsigned long long m = 0;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < D.p; c += (int64_t)gridDim.x * blockDim.x) {
    const double x = frozen[block_of_col(D, c + 1)] ? 0.0 : v[c + 1] * D.inv_sd[c];
    a[c] = x;
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(x));
    m = b > m ? b : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long u = __shfl_xor_sync(0xffffffffu, m, o);
    m = u > m ? u : m;
  }
  if ((threadIdx.x & 31) == 0 && m) {
    atomicMax(cmax, m);
    atomicMax(cmax + 1, m);
  }
}
// per block g (one CTA each): u_gi = 2^-E (n S_gi - M_g) / n (+ v_0 for the intercept in block 0), the
// same reconstruction as the finalize's s; Ug = sum_i u_gi (fixed order); then the accumulators are cleared
__global__ void __launch_bounds__(FT) k_power_fwd_fin(const Dev D, long long* sacc, long long* mterm,
                                                      const unsigned long long* cmax, int maxcnt, const double* v,
                                                      const int* frozen, double* u, double* Ug) {
  __shared__ double smd[33];
  const int g = blockIdx.x;
  if (frozen[g]) return;
  const double inv = ldexp(1.0, -fwd_exponent(__longlong_as_double((long long)cmax[0]), maxcnt, D.n));
  const long long M = mterm[g];
  const double v0 = g == 0 ? v[0] : 0.0;
  long long* sg = sacc + (int64_t)g * D.n;
  double t = 0.0;
  for (int i = threadIdx.x; i < D.n; i += blockDim.x) {
    const double x = (double)((long long)D.n * sg[i] - M) * inv / (double)D.n + v0;
    u[(int64_t)g * D.n + i] = x;
    sg[i] = 0;
    t += x;
  }
  double tt[1] = {t};
  block_sum<1>(tt, smd);
  if (threadIdx.x == 0) {
    Ug[g] = tt[0];
    mterm[g] = 0;
  }
}

// per block g: est = v_g . w_g, nrm = ||w_g||  (one CTA per block, fixed order)
__global__ void k_power_reduce(const int64_t* bstart, const double* v, const double* w, const int* frozen,
                               double* est, double* nrm) {
  __shared__ double sm[32 * 2 + 2];
  const int g = blockIdx.x;
  if (frozen[g]) return;
  double a[2] = {0.0, 0.0};
  for (int64_t j = bstart[g] + threadIdx.x; j < bstart[g + 1]; j += blockDim.x) {
    a[0] += v[j] * w[j];
    a[1] += w[j] * w[j];
  }
  block_sum<2>(a, sm);
  if (threadIdx.x == 0) {
    est[g] = a[0];
    nrm[g] = sqrt(a[1]);
  }
}

// v_j <- w_j / ||w_g||  (or v_g normalised when w == nullptr)
__global__ void k_power_norm(const Dev D, double* v, const double* w, const double* nrm, const int* frozen) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= D.p; j += (int64_t)gridDim.x * blockDim.x) {
    const int g = block_of_col(D, j);
    if (frozen[g]) continue;
    v[j] = (w ? w[j] : v[j]) / nrm[g];
  }
}

// Lanczos step (a0', L259): w_g <- w_g - alpha_g v_g - beta_g vp_g for the live blocks (alpha, beta
// device arrays [G]; beta_g of the previous step, 0 at the first)
__global__ void k_lanczos_orth(const Dev D, const double* v, const double* vp, double* w, const double* alpha,
                               const double* beta, const int* frozen) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= D.p; j += (int64_t)gridDim.x * blockDim.x) {
    const int g = block_of_col(D, j);
    if (frozen[g]) continue;
    w[j] = w[j] - alpha[g] * v[j] - beta[g] * vp[j];
  }
}

// vp_g <- v_g, v_g <- w_g / beta_g for the live blocks
__global__ void k_lanczos_next(const Dev D, double* v, double* vp, const double* w, const double* beta,
                               const int* frozen) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= D.p; j += (int64_t)gridDim.x * blockDim.x) {
    const int g = block_of_col(D, j);
    if (frozen[g]) continue;
    vp[j] = v[j];
    v[j] = w[j] / beta[g];
  }
}

// sample tau-quantile by exact rank selection and the null-model score psi/n (DESIGN reading R4)
// rank_i = #{y_j < y_i} + #{j < i : y_j == y_i} (a permutation of 0..n-1); ord[rank_i] = i.  One thread
// per i, y in shared-memory tiles: n^2 comparisons spread over the whole GPU
__global__ void __launch_bounds__(256) k_ranks(const double* y, int n, int* ord) {
  __shared__ double ys[2048];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const double yi = i < n ? y[i] : 0.0;
  int rank = 0;
  for (int t0 = 0; t0 < n; t0 += 2048) {
    __syncthreads();
    for (int t = threadIdx.x; t < 2048 && t0 + t < n; t += blockDim.x) ys[t] = y[t0 + t];
    __syncthreads();
    const int tn = min(2048, n - t0);
    for (int t = 0; t < tn; ++t) {
      const double yt = ys[t];
      rank += (yt < yi) || (yt == yi && t0 + t < i);
    }
  }
  if (i < n) ord[rank] = i;
}

// per RHS r (one CTA each): q = y_(ceil(n tau)) = y[ord[k - 1]], the null-model score psi (reading R4)
__global__ void k_null_score(const double* y, int n, const double* tau, const int* ord, double* psi /*[R][n]*/) {
  __shared__ int cnt[3];
  const int r = blockIdx.x;
  int k = (int)ceil((double)n * tau[r]);
  if (k < 1) k = 1;
  if (k > n) k = n;
  if (threadIdx.x == 0) cnt[0] = cnt[1] = cnt[2] = 0;
  __syncthreads();
  const double q = y[ord[k - 1]];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double yi = y[i];
    atomicAdd(&cnt[yi < q ? 0 : (yi > q ? 2 : 1)], 1);
  }
  __syncthreads();
  const double t = tau[r];
  const double tie = -((double)cnt[0] * (t - 1.0) + (double)cnt[2] * t) / (double)cnt[1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double yi = y[i];
    psi[(int64_t)r * n + i] = (yi < q ? t - 1.0 : (yi > q ? t : tie)) / (double)n;
  }
}

// support list of the current beta (parity par) — used after set_state
__global__ void k_build_support(const Dev D, int par) {
  const int lane = threadIdx.x & 31;
  const double* beta = D.beta[par];
  const int R = D.R;
  for (int64_t c0 = (int64_t)blockIdx.x * blockDim.x; c0 < D.p; c0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = c0 + threadIdx.x;
    bool nz = false;
    double mx[FSQR_MAXR];
    for (int r = 0; r < R; ++r) {
      mx[r] = 0.0;
      if (c < D.p && beta[(c + 1) * R + r] != 0.0) nz = true;
    }
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (m == 0) continue;
    int base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(D.sup_cnt + par, __popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (nz) {
      const int e = base + __popc(m & ((1u << lane) - 1u));
      D.sup_idx[par][e] = (int32_t)c;
      D.sup_cs[par][e] = D.colsum[c];
      for (int r = 0; r < R; ++r) {
        const double b = beta[(c + 1) * R + r];
        const double cv = b * D.inv_sd[c];
        D.sup_c[par][(int64_t)e * R + r] = cv;
        D.sup_b[par][(int64_t)e * R + r] = b;
        if (cv != 0.0) atomicMax(D.cmax + par * R + r, (unsigned long long)__double_as_longlong(fabs(cv)));
      }
    }
  }
}

// penalty of the committed beta and original-scale conversion (one CTA, fixed order)
__global__ void __launch_bounds__(FT) k_commit_stats(const Dev D, double* pen_out /*[R]*/, double* beta_out /*[R][p+1] or null*/,
                                                     int orig) {
  __shared__ double smd[32 * 3 + 3];
  const long long k = *D.iter;
  const bool use_w = *D.use_w != 0;
  for (int r = 0; r < D.R; ++r) {
    const long long ci = D.status[r] == ST_ACTIVE ? k : D.commit_iter[r];
    const double* beta = D.beta[(int)(ci & 1)];
    double a[3] = {0.0, 0.0, 0.0};
    for (int64_t j = 1 + threadIdx.x; j <= D.p; j += blockDim.x) {
      const double b = beta[j * D.R + r];
      const double lam = use_w ? D.lam_cur[r] * D.lamw[j * D.R + r] : D.lam_cur[r];
      a[0] += lam * fabs(b) + 0.5 * D.lam2[r] * b * b;
      const double bo = b * D.inv_sd[j - 1];
      a[1] += D.mean[j - 1] * bo;
      a[2] += b != 0.0 ? 1.0 : 0.0;
      if (beta_out) beta_out[(int64_t)r * (D.p + 1) + j] = orig ? bo : b;
    }
    block_sum<3>(a, smd);
    if (threadIdx.x == 0) {
      if (pen_out) {
        pen_out[r] = a[0];
        pen_out[D.R + r] = a[2];   // |A|: nonzero penalised coefficients
      }
      if (beta_out) beta_out[(int64_t)r * (D.p + 1)] = orig ? beta[r] - a[1] : beta[r];
    }
    __syncthreads();
  }
}

// Algorithm 2: w_jr = p'_lam_r(|beta~_jr|) / lam_r from the committed beta,
// SCAD (kind 1, E16 L354-361) or MCP (kind 2, E17 L363-369); the intercept is never penalised.
__global__ void k_lla_weights(const Dev D, int kind, double a) {
  const long long k = *D.iter;
  for (int r = 0; r < D.R; ++r) {
    const long long ci = D.status[r] == ST_ACTIVE ? k : D.commit_iter[r];
    const double* beta = D.beta[(int)(ci & 1)];
    const double lam = D.lam_cur[r];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= D.p; j += (int64_t)gridDim.x * blockDim.x) {
      double w = 0.0;
      if (j > 0) {
        const double ab = fabs(beta[j * D.R + r]);
        double d;
        if (kind == 1) d = ab <= lam ? lam : (ab < a * lam ? (a * lam - ab) / (a - 1.0) : 0.0);
        else d = ab <= a * lam ? lam - ab / a : 0.0;
        w = d / lam;
      }
      D.lamw[j * D.R + r] = w;
    }
  }
}

// resume after a stop: the K2 pass that detected convergence at iteration k had already appended
// beta^{k+1} to the support list of parity k+1 (and raised its cmax) before K1/finalize were
// skipped; that list must be empty again before iteration k is re-run.
__global__ void k_resume(const Dev D) {
  const int par1 = (int)((*D.iter + 1) & 1);
  if (threadIdx.x == 0) {
    D.sup_cnt[par1] = 0;
    *D.kbase = *D.iter;
  }
  if (threadIdx.x < D.R) D.cmax[par1 * D.R + threadIdx.x] = 0ull;
}

// resume after a solve froze some RHS: bring their committed beta into the current parity buffer
__global__ void k_unfreeze(const Dev D) {
  const long long k = *D.iter;
  const int par = (int)(k & 1);
  for (int r = 0; r < D.R; ++r) {
    if (D.status[r] == ST_ACTIVE) continue;
    const int cp = (int)(D.commit_iter[r] & 1);
    if (cp == par) continue;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= D.p; j += (int64_t)gridDim.x * blockDim.x)
      D.beta[par][j * D.R + r] = D.beta[cp][j * D.R + r];
  }
}

}  // namespace

void launch_finalize(const Dev& D, cudaStream_t st) {
  if (D.storage == 0)
    launch_pdl(k_finalize, dim3(1), dim3(FT), 0, st, D);
  else
    launch_pdl(k_finalize_mc, dim3((D.n + FIN_THREADS - 1) / FIN_THREADS, D.R), dim3(FIN_THREADS), 0, st, D);
}
// PACKED2 -> u8 (the pivotal statistic streams u8 tiles): one thread per packed word, 16 codes out
static __global__ void k_unpack2(const uint32_t* __restrict__ x2, int64_t ld2, int64_t p, uint8_t* __restrict__ x8,
                          int64_t ld8) {
  const int64_t wpc = ld8 / 16;   // 16-sample output groups per column
  const int64_t total = p * wpc;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = w / wpc, j = w - c * wpc;
    const uint32_t v = x2[(c * ld2) / 4 + j];
    uint32_t o[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t y = (v >> (8 * b)) & 0xFFu;
      o[b] = (y & 3u) | (((y >> 2) & 3u) << 8) | (((y >> 4) & 3u) << 16) | (((y >> 6) & 3u) << 24);
    }
    *reinterpret_cast<uint4*>(x8 + c * ld8 + 16 * j) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

void launch_unpack2(const uint8_t* x2, int64_t ld2, int64_t p, uint8_t* x8, int64_t ld8, cudaStream_t st) {
  k_unpack2<<<148 * 8, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(x2), ld2, p, x8, ld8);
}

void launch_pack2(const uint8_t* x8, int64_t ld8, int n, int64_t p, uint8_t* x2, int64_t ld2, int* bad,
                  cudaStream_t st) {
  k_pack2<<<148 * 8, 256, 0, st>>>(x8, ld8, n, p, reinterpret_cast<uint32_t*>(x2), ld2, bad);
}
void launch_init_state(const Dev& D, cudaStream_t st) { k_init_state<<<1, FT, 0, st>>>(D); }
void launch_colstats(const Dev& D, int32_t* colsum, double* mean, double* inv_sd, double* sd, int* bad,
                     cudaStream_t st) {
  const int grid = 148 * 8;
  if (D.storage == 0) k_colstats_f32<<<grid, 256, 0, st>>>(D, mean, inv_sd, sd, bad);
  else if (D.storage == 1) k_colstats_int<1><<<grid, 256, 0, st>>>(D, colsum, mean, inv_sd, sd, bad);
  else k_colstats_int<2><<<grid, 256, 0, st>>>(D, colsum, mean, inv_sd, sd, bad);
}
void launch_power_start(int64_t p1, uint64_t seed, double* v, cudaStream_t st) {
  k_power_start<<<256, 256, 0, st>>>(p1, seed, v);
}
void launch_power_fwd(const Dev& D, const int64_t* bstart, const double* v, const int* frozen, double* u,
                      cudaStream_t st) {
  dim3 grid((D.n + 127) / 128, D.G);
  k_power_fwd<<<grid, 128, 0, st>>>(D, bstart, v, frozen, u);
}
void launch_back_f64(const Dev& D, const double* u, int per_block, const int* frozen, double* w,
                     unsigned long long* maxbits, cudaStream_t st) {
  k_back_f64<<<148 * 8, 256, 0, st>>>(D, u, per_block, frozen, w, maxbits);
}
void launch_power_reduce(const Dev& D, const int64_t* bstart, const double* v, const double* w, const int* frozen,
                         double* est, double* nrm, cudaStream_t st) {
  k_power_reduce<<<D.G, 1024, 0, st>>>(bstart, v, w, frozen, est, nrm);
}
void launch_power_norm(const Dev& D, double* v, const double* w, const double* nrm, const int* frozen,
                       cudaStream_t st) {
  k_power_norm<<<512, 256, 0, st>>>(D, v, w, nrm, frozen);
}
void launch_lanczos_orth(const Dev& D, const double* v, const double* vp, double* w, const double* alpha,
                         const double* beta, const int* frozen, cudaStream_t st) {
  k_lanczos_orth<<<512, 256, 0, st>>>(D, v, vp, w, alpha, beta, frozen);
}
void launch_lanczos_next(const Dev& D, double* v, double* vp, const double* w, const double* beta, const int* frozen,
                         cudaStream_t st) {
  k_lanczos_next<<<512, 256, 0, st>>>(D, v, vp, w, beta, frozen);
}
void launch_power_fwd_int(const Dev& D, const int64_t* bstart, const double* v, const int* frozen, double* part,
                          int S, double* u, double* Ug, cudaStream_t st) {
  dim3 grid((D.n + 2047) / 2048, D.G, S);
  if (D.storage == 1) k_power_fwd_int<1><<<grid, 128, 0, st>>>(D, bstart, v, frozen, part, S);
  else k_power_fwd_int<2><<<grid, 128, 0, st>>>(D, bstart, v, frozen, part, S);
  k_sum_parts<<<D.G, 1024, 0, st>>>(part, S, D.G, D.n, frozen, u, Ug);
}
void launch_sum_parts(const double* part, int S, int G, int n, double* u, double* Ug, cudaStream_t st) {
  k_sum_parts<<<G, 1024, 0, st>>>(part, S, G, n, nullptr, u, Ug);
}
void launch_back_int(const Dev& D, const double* u, const double* Ug, int per_block, const int* frozen, double* w,
                     unsigned long long* maxbits, cudaStream_t st) {
  if (D.storage == 1) k_back_int<1><<<148 * 8, 256, 0, st>>>(D, u, Ug, per_block, frozen, w, maxbits);
  else k_back_int<2><<<148 * 8, 256, 0, st>>>(D, u, Ug, per_block, frozen, w, maxbits);
}
void launch_null_score(const double* y, int n, const double* tau, int R, int* ord, double* psi, cudaStream_t st) {
  k_ranks<<<(n + 255) / 256, 256, 0, st>>>(y, n, ord);
  k_null_score<<<R, 1024, 0, st>>>(y, n, tau, ord, psi);
}
void launch_build_support(const Dev& D, int par, cudaStream_t st) {
  k_build_support<<<(int)((D.p + 255) / 256 < 4096 ? (D.p + 255) / 256 : 4096), 256, 0, st>>>(D, par);
}
void launch_commit_stats(const Dev& D, double* pen, double* beta_out, int orig, cudaStream_t st) {
  k_commit_stats<<<1, FT, 0, st>>>(D, pen, beta_out, orig);
}
void launch_unfreeze(const Dev& D, cudaStream_t st) {
  k_resume<<<1, 32, 0, st>>>(D);
  k_unfreeze<<<256, 256, 0, st>>>(D);
}
void launch_lla_weights(const Dev& D, int kind, double a, cudaStream_t st) {
  k_lla_weights<<<592, 256, 0, st>>>(D, kind, a);
}
void launch_power_quant(const Dev& D, const double* u, const double* Ug, const int* frozen, int8_t* Bp, int ldk,
                        long long* Tsum, double* gs, double* w, cudaStream_t st) {
  k_power_quant<<<D.G, FT, 0, st>>>(D, u, Ug, frozen, Bp, ldk, Tsum, gs, w);
}
void launch_iota(int32_t* ix, int64_t p, cudaStream_t st) { k_iota<<<1184, 256, 0, st>>>(ix, p); }
void launch_power_coef(const Dev& D, const double* v, const int* frozen, double* a, unsigned long long* cmax,
                       cudaStream_t st) {
  k_power_coef<<<1184, 256, 0, st>>>(D, v, frozen, a, cmax);
}
void launch_power_fwd_fin(const Dev& D, long long* sacc, long long* mterm, const unsigned long long* cmax, int maxcnt,
                          const double* v, const int* frozen, double* u, double* Ug, cudaStream_t st) {
  k_power_fwd_fin<<<D.G, FT, 0, st>>>(D, sacc, mterm, cmax, maxcnt, v, frozen, u, Ug);
}
