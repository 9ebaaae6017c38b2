// k1_fwd.cu — a4: the forward product s^{k+1} = X~ beta^{k+1} (PAPER.md:L287,
// "computation of X beta ... divided into G simultaneous sub-tasks ... followed
// by computing their sum"), restricted to the support of beta^{k+1}: only the
// columns listed by the a2 epilogue are read (n * |S| bytes).
//
// Genotype storage: a CTA owns a slab of 32*RPL rows and a slice of support
// entries; its 8 warps take 32-entry groups of the slice round-robin.  A lane
// stages one entry of the group (column index and the int64 fixed-point
// C_j = round(2^E beta_j / s_j), split into 22-bit low / signed high halves),
// the warp broadcasts them with shuffles and keeps four 128-bit column loads in
// flight while it accumulates x * C_lo and x * C_hi in int32 registers (exact:
// |x C| < 2^23 and at most 256 entries per flush).  Warp partials meet in
// shared memory and leave the CTA as one 64-bit integer atomic per row, so the
// cross-block sum (the paper's barrier aggregation) is exact and independent of
// scheduling.  The centring term sum_j colsum_j C_j is accumulated the same
// way; finalize forms s_i = 2^-E (n S_i - M)/n + beta_0.
// fp32 storage: one thread per row walks the columns in ascending order (fp64),
// deterministic by construction (small designs only).
#include "fsqr_dev.cuh"

namespace {

constexpr int THREADS = 256;
constexpr int NWARP = THREADS / 32;
constexpr int UNR = 4;   // column loads in flight per lane

template <int RPL>
struct Codes {
  uint32_t w[(RPL + 3) / 4];   // u8: RPL bytes; 2-bit: RPL codes packed (RPL/4 bytes)
};

template <int RPL, int ST>
__device__ __forceinline__ void load_codes(const uint8_t* col, int row0, bool inb, Codes<RPL>& c) {
  if (!inb) {
#pragma unroll
    for (int q = 0; q < (RPL + 3) / 4; ++q) c.w[q] = 0;
    return;
  }
  if (ST == 1) {
    if (RPL == 16) {
      const uint4 v = __ldcs((const uint4*)(col + row0));
      c.w[0] = v.x; c.w[1] = v.y; c.w[2] = v.z; c.w[3] = v.w;
    } else if (RPL == 8) {
      const uint2 v = __ldcs((const uint2*)(col + row0));
      c.w[0] = v.x; c.w[1] = v.y;
    } else {
      c.w[0] = __ldcs((const uint32_t*)(col + row0));
    }
  } else {
    uint32_t v;
    if (RPL == 16) v = __ldcs((const uint32_t*)(col + (row0 >> 2)));
    else if (RPL == 8) v = __ldcs((const uint16_t*)(col + (row0 >> 2)));
    else v = __ldcs(col + (row0 >> 2));
    c.w[0] = v;
  }
}

template <int RPL, int ST>
__device__ __forceinline__ uint32_t code_at(const Codes<RPL>& c, int i) {
  if (ST == 1) return (c.w[i >> 2] >> (8 * (i & 3))) & 0xFFu;
  return (c.w[0] >> (2 * i)) & 3u;
}

template <int RMAX, int ST>
__global__ void __launch_bounds__(THREADS) k1_int(const Dev D, int cur) {
  constexpr int RPL = RMAX <= 2 ? 16 : (RMAX <= 4 ? 8 : 4);
  constexpr int RPW = 32 * RPL;   // rows per slab
  __shared__ unsigned long long sacc[RPW * RMAX];
  __shared__ unsigned long long smt[RMAX];
  if (*D.stop) return;
  const long long k = *D.iter;
  const int par = (int)((k + (cur ? 0 : 1)) & 1);
  const int cnt = D.sup_cnt[par];
  if (cnt == 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int R = D.R;
  double scale[RMAX];
  bool act[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    act[r] = r < R && (cur || D.status[r] == ST_ACTIVE);
    const double cm = r < R ? __longlong_as_double((long long)D.cmax[par * R + r]) : 0.0;
    scale[r] = ldexp(1.0, fwd_exponent(cm, cnt, D.n));
  }
  const int nrc = (D.n + RPW - 1) / RPW;
  // entries per CTA slice: balance nrc * nslices ~ gridDim, at least one 32-group per warp
  int64_t es = ((int64_t)cnt * nrc + gridDim.x - 1) / gridDim.x;
  es = ((es + 32 * NWARP - 1) / (32 * NWARP)) * (32 * NWARP);
  const int64_t nsl = (cnt + es - 1) / es;
  const int64_t nwork = nsl * nrc;
  const int32_t* sidx = D.sup_idx[par];
  const double* sc = D.sup_c[par];
  for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    const int rc = (int)(w % nrc);
    const int64_t e0 = (w / nrc) * es, e1 = min((int64_t)cnt, e0 + es);
    for (int q = threadIdx.x; q < RPW * RMAX; q += THREADS) sacc[q] = 0ull;
    if (threadIdx.x < RMAX) smt[threadIdx.x] = 0ull;
    __syncthreads();
    const int row0 = rc * RPW + lane * RPL;
    const bool inb = (ST == 1) ? (row0 < D.ld) : ((row0 >> 2) < D.ld);
    long long acc[RPL][RMAX];
#pragma unroll
    for (int i = 0; i < RPL; ++i)
#pragma unroll
      for (int r = 0; r < RMAX; ++r) acc[i][r] = 0;
    long long mt[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) mt[r] = 0;
    for (int64_t g0 = e0 + 32 * wid; g0 < e1; g0 += 32 * NWARP) {
      // stage one entry per lane
      const int64_t e = g0 + lane;
      const int ng = (int)min((int64_t)32, e1 - g0);
      int32_t myc = 0;
      int32_t clo[RMAX], chi[RMAX];
      if (e < e1) {
        myc = sidx[e];
        const long long cs = (rc == 0) ? (long long)D.colsum[myc] : 0;
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          const long long C = act[r] ? __double2ll_rn(sc[e * R + r] * scale[r]) : 0;
          clo[r] = (int32_t)(C & 0x3FFFFF);
          chi[r] = (int32_t)(C >> 22);
          mt[r] += cs * C;
        }
      } else {
#pragma unroll
        for (int r = 0; r < RMAX; ++r) clo[r] = chi[r] = 0;
      }
      int32_t alo[RPL][RMAX], ahi[RPL][RMAX];
#pragma unroll
      for (int i = 0; i < RPL; ++i)
#pragma unroll
        for (int r = 0; r < RMAX; ++r) alo[i][r] = ahi[i][r] = 0;
      for (int u0 = 0; u0 < ng; u0 += UNR) {
        Codes<RPL> cd[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int cu = __shfl_sync(0xffffffffu, myc, (u0 + u) & 31);
          load_codes<RPL, ST>(D.X8 + (int64_t)cu * D.ld, row0, inb && (u0 + u < ng), cd[u]);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            const int32_t lo = __shfl_sync(0xffffffffu, clo[r], (u0 + u) & 31);
            const int32_t hi = __shfl_sync(0xffffffffu, chi[r], (u0 + u) & 31);
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              const int32_t x = (int32_t)code_at<RPL, ST>(cd[u], i);
              alo[i][r] += x * lo;
              ahi[i][r] += x * hi;
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i)
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          acc[i][r] += (long long)(uint32_t)alo[i][r] + ((long long)ahi[i][r] << 22);
    }
    // warp partials -> shared (exact integer atomics) -> one global atomic per row
#pragma unroll
    for (int i = 0; i < RPL; ++i)
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (act[r] && acc[i][r] != 0) atomicAdd(&sacc[(lane * RPL + i) * RMAX + r], (unsigned long long)acc[i][r]);
    if (rc == 0) {
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        long long v = mt[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && v != 0) atomicAdd(&smt[r], (unsigned long long)v);
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < RPW * RMAX; q += THREADS) {
      const int row = rc * RPW + q / RMAX, r = q % RMAX;
      const unsigned long long v = sacc[q];
      if (row < D.n && r < R && v != 0ull) atomicAdd((unsigned long long*)&D.sacc[(int64_t)r * D.n + row], v);
    }
    if (rc == 0 && threadIdx.x < R && smt[threadIdx.x] != 0ull)
      atomicAdd((unsigned long long*)&D.mterm[threadIdx.x], smt[threadIdx.x]);
    __syncthreads();
  }
}

// fp32 design: s_i = sum_j (x_ij - m_j) beta_j / s_j in ascending j (beta_0 added by finalize)
template <int RMAX>
__global__ void __launch_bounds__(THREADS) k1_f32(const Dev D, int cur) {
  if (*D.stop) return;
  const long long k = *D.iter;
  const double* beta = D.beta[(int)((k + (cur ? 0 : 1)) & 1)];
  const int R = D.R;
  for (int i = blockIdx.x * THREADS + threadIdx.x; i < D.n; i += gridDim.x * THREADS) {
    double a[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) a[r] = 0.0;
    for (int64_t c = 0; c < D.p; ++c) {
      const double* bj = beta + (c + 1) * R;
      bool any = false;
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r < R) any |= bj[r] != 0.0;
      if (!any) continue;
      const double x = (double)D.Xf[c * D.ld + i] - D.mean[c];
      const double isd = D.inv_sd[c];
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r < R) a[r] = fma(x, bj[r] * isd, a[r]);
    }
#pragma unroll
    for (int r = 0; r < RMAX; ++r)
      if (r < R && (cur || D.status[r] == ST_ACTIVE)) D.sdense[(int64_t)r * D.n + i] = a[r];
  }
}

template <int RMAX>
void launch_r(const Dev& D, int grid, cudaStream_t st, int cur) {
  if (D.storage == 0)
    k1_f32<RMAX><<<(D.n + THREADS - 1) / THREADS, THREADS, 0, st>>>(D, cur);
  else if (D.storage == 1)
    k1_int<RMAX, 1><<<grid, THREADS, 0, st>>>(D, cur);
  else
    k1_int<RMAX, 2><<<grid, THREADS, 0, st>>>(D, cur);
}

}  // namespace

void launch_k1_mode(const Dev& D, int grid, cudaStream_t st, int cur) {
  if (D.R <= 1) launch_r<1>(D, grid, st, cur);
  else if (D.R <= 2) launch_r<2>(D, grid, st, cur);
  else if (D.R <= 4) launch_r<4>(D, grid, st, cur);
  else if (D.R <= 8) launch_r<8>(D, grid, st, cur);
  else launch_r<16>(D, grid, st, cur);
}

void launch_k1(const Dev& D, int grid, cudaStream_t st) { launch_k1_mode(D, grid, st, 0); }
