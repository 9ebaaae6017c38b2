// k1_fwd.cu — a4: the forward product s^{k+1} = X~ beta^{k+1} (PAPER.md:L287,
// "computation of X beta ... divided into G simultaneous sub-tasks ... followed
// by computing their sum"), restricted to the support of beta^{k+1}: only the
// columns listed by the a2 epilogue are read (n * |S| bytes).
//
// Genotype storage: each warp owns a 32*RPL-row slab and a slice of support
// entries; per entry it loads RPL codes per lane and accumulates int64
// fixed-point C_j = round(2^E beta_j / s_j).  Slabs are summed across slices
// with 64-bit integer atomics, so the cross-block sum (the paper's barrier
// aggregation) is exact and independent of scheduling.  The centring term
// sum_j colsum_j C_j is accumulated the same way; finalize forms
// s_i = 2^-E (n S_i - M)/n + beta_0.
// fp32 storage: one thread per row walks the columns in ascending order (fp64),
// deterministic by construction (small designs only).
#include "fsqr_dev.cuh"

namespace {

constexpr int THREADS = 256;

template <int RMAX, int ST>
__global__ void __launch_bounds__(THREADS) k1_int(const Dev D, int cur) {
  constexpr int RPL = RMAX <= 2 ? 16 : (RMAX <= 4 ? 8 : 4);
  constexpr int RPW = 32 * RPL;
  if (*D.stop) return;
  const long long k = *D.iter;
  const int par = (int)((k + (cur ? 0 : 1)) & 1);
  const int cnt = D.sup_cnt[par];
  if (cnt == 0) return;
  const int lane = threadIdx.x & 31;
  const int R = D.R;
  double scale[RMAX];
  bool act[RMAX];
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    act[r] = r < R && (cur || D.status[r] == ST_ACTIVE);
    const double cm = r < R ? __longlong_as_double((long long)D.cmax[par * R + r]) : 0.0;
    scale[r] = ldexp(1.0, fwd_exponent(cm, cnt, D.n));
  }
  const int64_t nwarps = (int64_t)gridDim.x * (THREADS / 32);
  const int64_t gw = (int64_t)blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
  const int nrc = (D.n + RPW - 1) / RPW;
  int64_t es = ((int64_t)cnt * nrc + nwarps - 1) / nwarps;
  if (es < 16) es = 16;
  const int64_t nsl = (cnt + es - 1) / es;
  const int64_t nwork = nsl * nrc;
  const int32_t* sidx = D.sup_idx[par];
  const double* sc = D.sup_c[par];
  for (int64_t w = gw; w < nwork; w += nwarps) {
    const int rc = (int)(w % nrc);
    const int64_t e0 = (w / nrc) * es, e1 = min((int64_t)cnt, e0 + es);
    const int row0 = rc * RPW + lane * RPL;
    long long acc[RPL][RMAX];
#pragma unroll
    for (int i = 0; i < RPL; ++i)
#pragma unroll
      for (int r = 0; r < RMAX; ++r) acc[i][r] = 0;
    const bool inb = (ST == 1) ? (row0 < D.ld) : ((row0 >> 2) < D.ld);
    for (int64_t e = e0; e < e1; ++e) {
      const int64_t c = sidx[e];
      long long Cv[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) Cv[r] = act[r] ? __double2ll_rn(sc[e * R + r] * scale[r]) : 0;
      uint8_t code[RPL];
      if (inb) {
        const uint8_t* col = D.X8 + c * D.ld;
        if (ST == 1) {
          if (RPL == 16) {
            const uint4 v = *(const uint4*)(col + row0);
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 16; ++i) code[i] = (wv[i >> 2] >> (8 * (i & 3))) & 0xFF;
          } else if (RPL == 8) {
            const uint2 v = *(const uint2*)(col + row0);
            const uint32_t wv[2] = {v.x, v.y};
#pragma unroll
            for (int i = 0; i < 8; ++i) code[i] = (wv[i >> 2] >> (8 * (i & 3))) & 0xFF;
          } else {
            const uint32_t v = *(const uint32_t*)(col + row0);
#pragma unroll
            for (int i = 0; i < RPL; ++i) code[i] = (v >> (8 * i)) & 0xFF;
          }
        } else {
          // 2-bit: RPL codes = RPL/4 bytes starting at byte row0/4
          uint32_t v;
          if (RPL == 16) v = *(const uint32_t*)(col + (row0 >> 2));
          else if (RPL == 8) v = *(const uint16_t*)(col + (row0 >> 2));
          else v = col[row0 >> 2];
#pragma unroll
          for (int i = 0; i < RPL; ++i) code[i] = (v >> (2 * i)) & 3;
        }
      } else {
#pragma unroll
        for (int i = 0; i < RPL; ++i) code[i] = 0;
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const long long x = code[i];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) acc[i][r] += x * Cv[r];
      }
    }
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int row = row0 + i;
      if (row < D.n) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          if (act[r] && acc[i][r] != 0)
            atomicAdd((unsigned long long*)&D.sacc[(int64_t)r * D.n + row], (unsigned long long)acc[i][r]);
      }
    }
    if (rc == 0) {
      // centring term sum_j colsum_j * C_j over this slice
      long long mt[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) mt[r] = 0;
      for (int64_t e = e0 + lane; e < e1; e += 32) {
        const long long cs = D.colsum[sidx[e]];
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          if (act[r]) mt[r] += cs * __double2ll_rn(sc[e * R + r] * scale[r]);
      }
#pragma unroll
      for (int r = 0; r < RMAX; ++r) {
        long long v = mt[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && act[r] && v != 0) atomicAdd((unsigned long long*)&D.mterm[r], (unsigned long long)v);
      }
    }
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
