// k2_simt.cu — a1+a2 on the CUDA cores (sm_100a): the cross-check and fallback
// for the tensor-core kernel, and the path for the 2-bit and fp32 storages.
//
//  * U8 / PACKED2: exact integer dot products with dp4a on the same theta digit
//    rows the tensor-core kernel consumes, so beta^{k+1} is bitwise identical
//    to the TC path (same epilogue on identical integers).  Each warp owns CPW
//    adjacent columns and walks the samples in 512-row chunks (16 rows / lane,
//    128-bit loads of X, digit rows shared by the CPW columns from L1).
//  * F32_DENSE: warp per column, fp64 accumulation of (x_ij - m_j) theta_i with
//    a fixed butterfly reduction (deterministic).
// PAPER.md:L392 (X^T theta across G blocks), E14 L274-277.
#include "k2_common.cuh"

namespace {

constexpr int THREADS = 256;
#define K2_RED_DOUBLES(RM) ((THREADS / 32) * (RM) * (FSQR_NPART + 1) > 33 * FSQR_NPART ? (THREADS / 32) * (RM) * (FSQR_NPART + 1) : 33 * FSQR_NPART)

__device__ __forceinline__ uint32_t unpack2(uint32_t b) {
  // byte of four 2-bit codes -> four bytes {0,1,2}
  return (b | (b << 6) | (b << 12) | (b << 18)) & 0x03030303u;
}

template <int RMAX, int ST>
__global__ void __launch_bounds__(THREADS) k2_simt_int(const Dev D) {
  constexpr int CPW = RMAX <= 2 ? 4 : (RMAX <= 4 ? 2 : 1);   // columns per warp
  constexpr int ND = 4 * RMAX;                                 // digit rows
  __shared__ double red[K2_RED_DOUBLES(RMAX)];
  pdl_launch_dependents();
  pdl_wait();
  if (*D.stop) return;
  K2Part<RMAX> P;
  k2_part_init(P, red);
  K2Ctx<RMAX> C;
  k2_load_ctx(D, C);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (THREADS / 32);
  const int64_t ngroups = (D.p + CPW - 1) / CPW;
  const int nd = 4 * D.R;
  for (int64_t grp = gw; grp < ngroups; grp += nwarps) {
    int32_t acc[CPW][ND];
#pragma unroll
    for (int a = 0; a < CPW; ++a)
#pragma unroll
      for (int q = 0; q < ND; ++q) acc[a][q] = 0;
    for (int i0 = lane * 16; i0 < D.n; i0 += 512) {
      uint4 xv[CPW];
#pragma unroll
      for (int a = 0; a < CPW; ++a) {
        const int64_t c = grp * CPW + a;
        if (c < D.p) {
          if (ST == 1) {
            xv[a] = __ldcs((const uint4*)(D.X8 + c * D.ld + i0));
          } else {
            const uint32_t w = __ldcs((const uint32_t*)(D.X8 + c * D.ld + (i0 >> 2)));
            xv[a] = make_uint4(unpack2(w & 0xFF), unpack2((w >> 8) & 0xFF), unpack2((w >> 16) & 0xFF),
                               unpack2(w >> 24));
          }
        } else {
          xv[a] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int q = 0; q < ND; ++q) {
        if (q < nd) {
          const uint4 bv = __ldg((const uint4*)(D.Bq + (int64_t)q * D.ldk + i0));
#pragma unroll
          for (int a = 0; a < CPW; ++a) {
            int s = acc[a][q];
            s = __dp4a((int)xv[a].x, (int)bv.x, s);
            s = __dp4a((int)xv[a].y, (int)bv.y, s);
            s = __dp4a((int)xv[a].z, (int)bv.z, s);
            s = __dp4a((int)xv[a].w, (int)bv.w, s);
            acc[a][q] = s;
          }
        }
      }
    }
    // exact integer butterfly: every lane ends with the full sums
#pragma unroll
    for (int a = 0; a < CPW; ++a)
#pragma unroll
      for (int q = 0; q < ND; ++q) {
        int v = acc[a][q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[a][q] = v;
      }
    bool nz = false;
    int64_t cc = -1;
#pragma unroll
    for (int a = 0; a < CPW; ++a) {
      const int64_t c = grp * CPW + a;
      const bool valid = lane == a && c < D.p;
      double g[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) g[r] = 0.0;
      if (valid) {
        cc = c;
        const int32_t cs = D.colsum[c];
        const double isd = D.inv_sd[c];
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          g[r] = r < C.R ? g_from_digits(D.n, cs, C.cs->Tsum[r], C.cs->gscale[r], isd, &acc[a][4 * r]) : 0.0;
      }
      const bool z2 = epi_column<RMAX>(D, C, valid ? c : 0, g, P, valid);
      if (valid) nz = z2;
    }
    if (D.update) support_append<RMAX>(D, C, nz, cc);
  }
  __syncthreads();
  k2_finish<RMAX>(D, C, P, red);
}

template <int RMAX>
__global__ void __launch_bounds__(THREADS) k2_simt_f32(const Dev D) {
  __shared__ double red[K2_RED_DOUBLES(RMAX)];
  pdl_launch_dependents();
  pdl_wait();
  if (*D.stop) return;
  K2Part<RMAX> P;
  k2_part_init(P, red);
  K2Ctx<RMAX> C;
  k2_load_ctx(D, C);
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (THREADS / 32) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (THREADS / 32);
  for (int64_t c = gw; c < D.p; c += nwarps) {
    const float* col = D.Xf + c * D.ld;
    const double m = D.mean[c];
    double a[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) a[r] = 0.0;
    for (int i = lane; i < D.n; i += 32) {
      const double x = (double)col[i] - m;
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        if (r < C.R) a[r] = fma(x, D.theta[(int64_t)r * D.n + i], a[r]);
    }
    double g[RMAX];
    const double isd = D.inv_sd[c];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) g[r] = warp_sum_d(a[r]) * isd;
    const bool nz = epi_column<RMAX>(D, C, c, g, P, lane == 0);
    if (D.update) support_append<RMAX>(D, C, nz, c);
  }
  __syncthreads();
  k2_finish<RMAX>(D, C, P, red);
}

template <int RMAX>
void launch_r(const Dev& D, int grid, cudaStream_t st) {
  if (D.storage == 0)
    launch_pdl(k2_simt_f32<RMAX>, dim3(grid), dim3(THREADS), 0, st, D);
  else if (D.storage == 1)
    launch_pdl(k2_simt_int<RMAX, 1>, dim3(grid), dim3(THREADS), 0, st, D);
  else
    launch_pdl(k2_simt_int<RMAX, 2>, dim3(grid), dim3(THREADS), 0, st, D);
}

}  // namespace

void launch_k2_simt(const Dev& D, int grid, cudaStream_t st) {
  if (D.R <= 1) launch_r<1>(D, grid, st);
  else if (D.R <= 2) launch_r<2>(D, grid, st);
  else if (D.R <= 4) launch_r<4>(D, grid, st);
  else if (D.R <= 8) launch_r<8>(D, grid, st);
  else launch_r<16>(D, grid, st);
}
