// k1_fwd.cu — a4: the forward product s^{k+1} = X~ beta^{k+1} (PAPER.md:L287,
// "computation of X beta ... divided into G simultaneous sub-tasks ... followed
// by computing their sum"), restricted to the support of beta^{k+1}: only the
// columns listed by the a2 epilogue are read (n * |S| bytes).
//
// Genotype storage (k1_bulk): a persistent CTA takes work items = (row slab of
// RPW = 256*RPT rows) x (slice of the support list).  A producer warp turns 32
// support entries at a time into int64 fixed-point coefficients
// C_j = round(2^E beta_j / s_j) (split into 22-bit low / signed high halves,
// written to shared memory with each column's slot) and issues one
// cp.async.bulk copy per entry of the column's slab segment (contiguous bytes)
// into an mbarrier ring, so the copy engine -- not registers -- keeps the bytes
// in flight.  Eight consumer warps each own RPT consecutive rows per thread and
// accumulate x * C_lo and x * C_hi in int32 registers (exact: |x C| < 2^23 and
// at most 256 entries per flush into int64).  Each thread owns its rows, so a
// work item leaves the CTA as one 64-bit integer atomic per row and RHS: the
// cross-block sum (the paper's barrier aggregation, L287) is exact and
// independent of scheduling.  The centring term sum_j colsum_j C_j is summed by
// the producer on slab 0; finalize forms s_i = 2^-E (n S_i - M)/n + beta_0.
#include "fsqr_dev.cuh"

namespace {

#ifndef K1_SMEM_KB
#define K1_SMEM_KB 96   // stage-ring budget per CTA (two CTAs per SM)
#endif
#ifndef K1_RPT1
#define K1_RPT1 8       // rows per consumer thread for one RHS
#endif
#ifndef K1_QC_BIG
#define K1_QC_BIG 8     // columns per stage for 2 KB segments
#endif

constexpr int THREADS = 256;
constexpr int NCW = 8;              // consumer warps
constexpr int KTHREADS = 32 * (NCW + 1);

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// rows per thread: keep 4 * RPT * RMAX int32-equivalent accumulator registers <= 64
// (measured at M: 16 rows per thread / 4 KB copies was slower (58-61 vs 52 us); an fp64
// one-DFMA-per-element variant ran the same 53 us as the two-IMAD one; 2, 3 or 4 CTAs per SM
// (96 / 64 / 48 KB rings) all ran 52 us; 16 columns per stage 65 us)
template <int RMAX, int ST>
struct K1Shape {
  static constexpr int RPT = RMAX == 1 ? K1_RPT1 : (RMAX <= 2 ? 8 : (RMAX <= 4 ? 4 : (RMAX <= 8 ? 2 : 1)));
  static constexpr int RPW = 256 * RPT;
};

// codes of rows t*RPT .. t*RPT+RPT-1 of one slab segment in shared memory
template <int RPT, int ST>
__device__ __forceinline__ void seg_codes(const uint8_t* seg, int t, uint32_t (&x)[RPT]) {
  if (ST == 1) {
    if (RPT == 16) {
      const uint4 v = *(const uint4*)(seg + 16 * t);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int q = 0; q < 16; ++q) x[q] = __byte_perm(w[q >> 2], 0u, 0x4440u + (q & 3));
    } else if (RPT == 8) {
      const uint2 v = *(const uint2*)(seg + 8 * t);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        x[q] = (v.x >> (8 * q)) & 0xFFu;
        x[4 + q] = (v.y >> (8 * q)) & 0xFFu;
      }
    } else if (RPT == 4) {
      const uint32_t v = *(const uint32_t*)(seg + 4 * t);
#pragma unroll
      for (int q = 0; q < RPT; ++q) x[q] = (v >> (8 * q)) & 0xFFu;
    } else if (RPT == 2) {
      const uint32_t v = *(const uint16_t*)(seg + 2 * t);
#pragma unroll
      for (int q = 0; q < RPT; ++q) x[q] = (v >> (8 * q)) & 0xFFu;
    } else {
      x[0] = seg[t];
    }
  } else {
    // 2-bit: row i at bits 2(i%4) of byte i/4
    if (RPT == 32) {
      const uint2 v = *(const uint2*)(seg + 8 * t);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        x[q] = (v.x >> (2 * q)) & 3u;
        x[16 + q] = (v.y >> (2 * q)) & 3u;
      }
    } else if (RPT == 16) {
      const uint32_t v = *(const uint32_t*)(seg + 4 * t);
#pragma unroll
      for (int q = 0; q < 16; ++q) x[q] = (v >> (2 * q)) & 3u;
    } else if (RPT == 8) {
      const uint32_t v = *(const uint16_t*)(seg + 2 * t);
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = (v >> (2 * q)) & 3u;
    } else if (RPT == 4) {
      const uint32_t v = seg[t];
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = (v >> (2 * q)) & 3u;
    } else {
      const int i0 = t * RPT;
      const uint32_t v = seg[i0 >> 2] >> (2 * (i0 & 3));
#pragma unroll
      for (int q = 0; q < RPT; ++q) x[q] = (v >> (2 * q)) & 3u;
    }
  }
}

// one support column of a stage: x * C_lo and x * C_hi into the int32 accumulators of the
// thread's RPT rows (u8 codes zero-extended with one PRMT each)
template <int RPT, int ST, int RMAX>
__device__ __forceinline__ void consume_col(const uint8_t* seg, const int32_t* cf, int tid,
                                            int32_t (&alo)[RPT][RMAX], int32_t (&ahi)[RPT][RMAX]) {
  uint32_t x[RPT];
  if (ST == 1 && RPT == 8) {
    const uint2 v = *(const uint2*)(seg + 8 * tid);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] = __byte_perm(v.x, 0u, 0x4440u + i);
      x[4 + i] = __byte_perm(v.y, 0u, 0x4440u + i);
    }
  } else {
    seg_codes<RPT, ST>(seg, tid, x);
  }
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    const int2 c = *(const int2*)(cf + 2 * r);
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      alo[i][r] += (int32_t)x[i] * c.x;
      ahi[i][r] += (int32_t)x[i] * c.y;
    }
  }
}


template <int RMAX, int ST>
struct K1Smem {
  static constexpr int RPT = K1Shape<RMAX, ST>::RPT;
  static constexpr int SEG = ST == 1 ? 256 * RPT : 64 * RPT;   // bytes of one column's slab segment
  static constexpr int QC = SEG >= 2048 ? K1_QC_BIG : (SEG >= 1024 ? 16 : 32);   // columns per stage (divides 32)
  static constexpr int ST0 = (K1_SMEM_KB * 1024) / (QC * SEG);
  static constexpr int STAGES = ST0 < 4 ? 4 : (ST0 > 12 ? 12 : ST0);
  static constexpr int DATA = STAGES * QC * SEG;
  static constexpr int COEF = STAGES * QC * RMAX * 2 * 4;      // int32 lo/hi per slot and RHS
  static constexpr int BYTES = 128 + DATA + COEF + 2 * STAGES * 8 + 64;
};

template <int RMAX, int ST>
__global__ void __launch_bounds__(KTHREADS) k1_bulk(const Dev D, int cur) {
  using SH = K1Smem<RMAX, ST>;
  constexpr int QC = SH::QC;
  constexpr int STAGES = SH::STAGES;
  constexpr int RPT = SH::RPT;
  constexpr int RPW = 256 * RPT;
  constexpr int SEG = SH::SEG;
  extern __shared__ uint8_t k1_smem_raw[];
  uint8_t* sm = k1_smem_raw + (((127 + 1) - (smem_u32(k1_smem_raw) & 127)) & 127);
  uint8_t* sdata = sm;
  int32_t* scoef = (int32_t*)(sm + SH::DATA);
  uint64_t* full = (uint64_t*)(sm + SH::DATA + SH::COEF);
  uint64_t* empty = full + STAGES;

  pdl_launch_dependents();
  pdl_wait();
  if (*D.stop) return;
  const long long k = *D.iter;
  const int par = (int)((k + (cur ? 0 : 1)) & 1);
  const int cnt = D.sup_cnt[par];
  if (cnt == 0) return;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int R = D.R;

  const int nslab = (D.n + RPW - 1) / RPW;
  // slices per slab so that every CTA gets about one work item; 32-entry granularity
  const int per = max(1, (int)gridDim.x / nslab);
  int64_t es = ((int64_t)cnt + per - 1) / per;
  es = ((es + 31) / 32) * 32;
  const int64_t nsl = ((int64_t)cnt + es - 1) / es;
  const int64_t nwork = nsl * nslab;
  const int32_t* sidx = D.sup_idx[par];
  const double* sc = D.sup_c[par];
  const int64_t seg_stride = (ST == 1) ? RPW : RPW / 4;    // bytes between slabs within a column

  if (tid == 0) {
    for (int q = 0; q < STAGES; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (wid == NCW) {
    // ===================== producer warp
    double scale[RMAX];
    bool act[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      act[r] = r < R && (cur || D.status[r] == ST_ACTIVE);
      const double cm = r < R ? __longlong_as_double((long long)D.cmax[par * R + r]) : 0.0;
      scale[r] = ldexp(1.0, fwd_exponent(cm, cnt, D.n));
    }
    const uint64_t pol = D.k1_policy == 2 ? policy_evict_last()
                         : (D.k1_policy == 1 ? policy_evict_normal() : policy_evict_first());
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const int slab = (int)(w % nslab);
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      const int64_t boff = (int64_t)slab * seg_stride;
      const uint32_t bytes = (uint32_t)min((int64_t)SEG, D.ld - boff);
      long long mt[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) mt[r] = 0;
      // software pipeline: the next group's (column, beta/s) loads are in flight while this group's
      // stages are issued, and its colsum load after them
      int32_t ncol = 0;
      double nsc[RMAX];
      long long ncs = 0;
      {
        const int64_t e = e0 + lane;
#pragma unroll
        for (int r = 0; r < RMAX; ++r) nsc[r] = 0.0;
        if (e < e1) {
          ncol = sidx[e];
#pragma unroll
          for (int r = 0; r < RMAX; ++r) nsc[r] = r < R ? sc[e * R + r] : 0.0;
          ncs = (slab == 0) ? (long long)D.colsum[ncol] : 0;
        }
      }
      for (int64_t g0 = e0; g0 < e1; g0 += 32) {
        const int64_t e = g0 + lane;
        const int32_t col = ncol;
        const long long cs = ncs;
        int32_t clo[RMAX], chi[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) clo[r] = chi[r] = 0;
        if (e < e1) {
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            const long long C = act[r] ? __double2ll_rn(nsc[r] * scale[r]) : 0;
            clo[r] = (int32_t)(C & 0x3FFFFF);
            chi[r] = (int32_t)(C >> 22);
            mt[r] += cs * C;
          }
        }
        {
          const int64_t en = e + 32;
          if (en < e1) {
            ncol = sidx[en];
#pragma unroll
            for (int r = 0; r < RMAX; ++r) nsc[r] = r < R ? sc[en * R + r] : 0.0;
          }
        }
        const int ng = (int)min((int64_t)32, e1 - g0);
        for (int q0 = 0; q0 < ng; q0 += QC) {
          mbar_wait(&empty[stage], phase ^ 1);
          // slot q of this stage <- entry q0 + q of the group (lanes q0 .. q0+QC-1)
          const int q = lane - q0;
          if (q >= 0 && q < QC) {
            int32_t* cf = scoef + (stage * QC + q) * RMAX * 2;
            const bool live = lane < ng;
#pragma unroll
            for (int r = 0; r < RMAX; ++r) {
              cf[2 * r] = live ? clo[r] : 0;
              cf[2 * r + 1] = live ? chi[r] : 0;
            }
          }
          __syncwarp();
          const int nq = min(QC, ng - q0);
          if (lane == 0) mbar_expect_tx(&full[stage], bytes * (uint32_t)nq);
          // every lane holding a column of this stage issues its own copy (lane q0+u)
          if (q >= 0 && q < nq)
            bulk_g2s(sdata + (stage * QC + q) * SEG, D.X8 + (int64_t)col * D.ld + boff, bytes, &full[stage], pol);
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (slab == 0 && e + 32 < e1) ncs = (long long)D.colsum[ncol];
      }
      if (slab == 0) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          long long v = mt[r];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0 && v != 0) atomicAdd((unsigned long long*)&D.mterm[r], (unsigned long long)v);
        }
      }
    }
  } else {
    // ===================== consumer warps: thread t owns rows slab*RPW + t*RPT .. +RPT-1
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const int slab = (int)(w % nslab);
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      long long acc[RPT][RMAX];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int r = 0; r < RMAX; ++r) acc[i][r] = 0;
      int32_t alo[RPT][RMAX], ahi[RPT][RMAX];
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int r = 0; r < RMAX; ++r) alo[i][r] = ahi[i][r] = 0;
      int since = 0;
      for (int64_t g0 = e0; g0 < e1; g0 += 32) {
        const int ng = (int)min((int64_t)32, e1 - g0);
        for (int q0 = 0; q0 < ng; q0 += QC) {
          mbar_wait(&full[stage], phase);
          const int nq = min(QC, ng - q0);
          const uint8_t* sd = sdata + stage * QC * SEG;
          const int32_t* cf = scoef + stage * QC * RMAX * 2;
          if (nq == QC) {
#pragma unroll
            for (int q = 0; q < QC; ++q) consume_col<RPT, ST, RMAX>(sd + q * SEG, cf + q * RMAX * 2, tid, alo, ahi);
          } else {
            for (int q = 0; q < nq; ++q) consume_col<RPT, ST, RMAX>(sd + q * SEG, cf + q * RMAX * 2, tid, alo, ahi);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
          since += nq;
          if (since >= 256 - QC) {
#pragma unroll
            for (int i = 0; i < RPT; ++i)
#pragma unroll
              for (int r = 0; r < RMAX; ++r) {
                acc[i][r] += (long long)(uint32_t)alo[i][r] + ((long long)ahi[i][r] << 22);
                alo[i][r] = ahi[i][r] = 0;
              }
            since = 0;
          }
        }
      }
      const int rowb = slab * RPW + tid * RPT;
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          const long long v = acc[i][r] + (long long)(uint32_t)alo[i][r] + ((long long)ahi[i][r] << 22);
          if (r < R && rowb + i < D.n && v != 0)
            atomicAdd((unsigned long long*)&D.sacc[(int64_t)r * D.n + rowb + i], (unsigned long long)v);
        }
    }
  }
}

// fp32 design: s_i = sum_j (x_ij - m_j) beta_j / s_j (beta_0 added by finalize).  Warp per row:
// lane L takes the columns j = L, L+32, ... in ascending order (coalesced beta reads, X read only
// for nonzero beta_j), then a fixed butterfly: deterministic for any launch.
template <int RMAX>
__global__ void __launch_bounds__(THREADS) k1_f32(const Dev D, int cur) {
  pdl_launch_dependents();
  pdl_wait();
  if (*D.stop) return;
  const long long k = *D.iter;
  const double* beta = D.beta[(int)((k + (cur ? 0 : 1)) & 1)];
  const int R = D.R;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * THREADS) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * THREADS + threadIdx.x) >> 5; i < D.n; i += nw) {
    double a[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) a[r] = 0.0;
    for (int64_t c = lane; c < D.p; c += 32) {
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
    for (int r = 0; r < RMAX; ++r) {
      const double v = warp_sum_d(a[r]);
      if (lane == 0 && r < R && (cur || D.status[r] == ST_ACTIVE)) D.sdense[(int64_t)r * D.n + i] = v;
    }
  }
}

template <int RMAX, int ST>
int bulk_grid(int grid) {
  // persistent: as many CTAs as fit (shared memory bound), grid = 148 x that by default
  const int per_sm = (200 * 1024) / K1Smem<RMAX, ST>::BYTES;
  return grid * (per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm));
}

template <int RMAX>
void launch_r(const Dev& D, int grid, cudaStream_t st, int cur) {
  if (D.storage == 0)
    launch_pdl(k1_f32<RMAX>, dim3((D.n + THREADS / 32 - 1) / (THREADS / 32)), dim3(THREADS), 0, st, D, cur);
  else if (D.storage == 1)
    launch_pdl(k1_bulk<RMAX, 1>, dim3(bulk_grid<RMAX, 1>(grid)), dim3(KTHREADS), K1Smem<RMAX, 1>::BYTES, st, D, cur);
  else
    launch_pdl(k1_bulk<RMAX, 2>, dim3(bulk_grid<RMAX, 2>(grid)), dim3(KTHREADS), K1Smem<RMAX, 2>::BYTES, st, D, cur);
}

template <int RMAX>
cudaError_t init_r() {
  cudaError_t e = cudaFuncSetAttribute(k1_bulk<RMAX, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       K1Smem<RMAX, 1>::BYTES);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k1_bulk<RMAX, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, K1Smem<RMAX, 2>::BYTES);
}

}  // namespace

// grid = number of SMs; the bulk kernel scales it by its resident CTAs per SM
void launch_k1_mode(const Dev& D, int grid, cudaStream_t st, int cur) {
  if ((D.k1_tc == 3 && D.storage == 2) || (D.k1_tc == 4 && D.storage == 1)) {
    launch_k1_tcp(D, grid, st, cur);
    return;
  }
  if (D.R <= 1) launch_r<1>(D, grid, st, cur);
  else if (D.R <= 2) launch_r<2>(D, grid, st, cur);
  else if (D.R <= 4) launch_r<4>(D, grid, st, cur);
  else if (D.R <= 8) launch_r<8>(D, grid, st, cur);
  else launch_r<16>(D, grid, st, cur);
}

void launch_k1(const Dev& D, int grid, cudaStream_t st) { launch_k1_mode(D, grid, st, 0); }

bool k1_fuses_finalize(const Dev& D) { return (D.k1_tc == 3 && D.storage == 2) || (D.k1_tc == 4 && D.storage == 1); }

cudaError_t k1_init() {
  cudaError_t e;
  if ((e = init_r<1>()) != cudaSuccess) return e;
  if ((e = init_r<2>()) != cudaSuccess) return e;
  if ((e = init_r<4>()) != cudaSuccess) return e;
  if ((e = init_r<8>()) != cudaSuccess) return e;
  return init_r<16>();
}
