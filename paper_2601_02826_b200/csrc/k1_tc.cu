// k1_tc.cu — a4 on the tensor cores: s^{k+1} = X~ beta^{k+1} over the support of beta^{k+1}
// ("computation of X beta ... divided into G simultaneous sub-tasks ... followed by
// computing their sum"), exact integer arithmetic.
//
// With C_{j,r} = round(2^E beta_{j,r} / s_j) split into six balanced base-256 digits d_{k}(j, r),
//   S_{i,r} = sum_{j in S} x_ij C_{j,r} = sum_k 256^k D_{i,(r,k)},   D = X_S · Dig,
// a GEMM with M = rows of X (128 per row tile), K = support entries, N = 6 R digit columns
// (padded to 16 / 32 / 48 / 96).  X is SNP-major (each column's rows contiguous), i.e. the
// wrong major-ness for a K-major A, so the transpose happens on chip:
//   producer warp (lane = support entry): digits of C into the K-major B tile in smem (no
//       swizzle), one cp.async.bulk of the column's slab segment (SR contiguous rows, 2 KB for
//       one RHS) into an mbarrier ring; the colsum·C centring term as before;
//   converter warps (TMEM lane = row): one byte per (row, entry) from the staged segments,
//       packed 4 entries per 32-bit cell, tcgen05.st into TMEM A buffers (lane = row, K along
//       the columns -- the layout k2_tc2 already uses);
//   MMA warp: one tcgen05.mma.kind::i8 (A from TMEM) per row tile and 32 entries;
//   epilogue (converter warps): tcgen05.ld the digit sums, S = sum_k 256^k D_k in int64, one
//       64-bit integer atomic per row and RHS, exactly as the CUDA-core k1_bulk.
// The per-element CUDA-core work is one shared-memory byte load and 3/4 of a byte permute,
// independent of R (k1_bulk needs 2 R integer multiply-adds per element).
#include <cuda.h>

#include "fsqr_dev.cuh"

namespace {

constexpr int KC = 32;         // support entries per chunk (one kind::i8 MMA K step)
// warps: 0 producer, 1 MMA, 2 TMEM alloc, 3 idle, 4..4+CW-1 convert + epilogue (CW/4 warps per
// TMEM lane quarter, each taking every (CW/4)-th row tile: the byte-gather loop is latency-bound)

template <int RMAX, int ST>
struct K1T {
  static constexpr int CW = 12;                                            // converter warps
  static constexpr int THREADS = 32 * (4 + CW);
  static constexpr int NDIG = 6 * RMAX;                                    // digit columns in use
  static constexpr int N = NDIG <= 16 ? 16 : (NDIG <= 32 ? 32 : (NDIG <= 48 ? 48 : 96));
  static constexpr int RT = N <= 16 ? 16 : (N <= 32 ? 8 : (N <= 48 ? 4 : 2));   // row tiles per slab
  static constexpr int SR = 128 * RT;                                      // rows per slab
  static constexpr int SEGB = ST == 1 ? SR : SR / 4;                       // bytes per column segment
  static constexpr int BTILE = N * KC;                                     // digit bytes per chunk
  static constexpr int STAGE = KC * SEGB + BTILE;
  static constexpr int ST0 = (192 * 1024) / STAGE;
  static constexpr int STAGES = ST0 < 2 ? 2 : (ST0 > 8 ? 8 : ST0);
  static constexpr int NAB = 2;                                            // TMEM A buffers
  static constexpr int ACOLS = RT * (KC / 4);                              // TMEM columns per A buffer
  static constexpr int A_COL0 = RT * N;                                    // accumulators first
  static constexpr int SMEM = 1024 + STAGES * STAGE + 1024;
  static_assert(A_COL0 + NAB * ACOLS <= 512, "TMEM budget");
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void umma_i8_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// K-major B tile without swizzle: core matrices of 8 digit rows x 16 entries (128 B), the two
// 16-entry halves of K at LBO = 128 B, groups of 8 digit rows at SBO = 256 B
__device__ __forceinline__ int btile_off(int nrow, int k) {
  return (nrow >> 3) * 256 + (nrow & 7) * 16 + (k >> 4) * 128 + (k & 15);
}
__device__ __forceinline__ uint64_t umma_desc_kmajor_noswz(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(128u >> 4) << 16;   // LBO: K direction (the two 16-byte halves)
  d |= (uint64_t)(256u >> 4) << 32;   // SBO: 8-row groups
  d |= (uint64_t)1u << 46;            // version = 1 (sm100)
  return d;                            // layout type 0 = SWIZZLE_NONE
}

template <int RMAX, int ST>
__global__ void __launch_bounds__(K1T<RMAX, ST>::THREADS, 1) k1_tc_kernel(const Dev D, int cur) {
  using T = K1T<RMAX, ST>;
  constexpr int CW = T::CW, CG = CW / 4;
  constexpr int RT = T::RT, SR = T::SR, SEGB = T::SEGB, N = T::N, STAGES = T::STAGES, NAB = T::NAB;
  extern __shared__ uint8_t k1t_raw[];
  uint8_t* sm = k1t_raw + (((1023 + 1) - (smem_u32(k1t_raw) & 1023)) & 1023);
  uint8_t* sdata = sm;                                   // [STAGES][KC][SEGB]
  uint8_t* sB = sm + STAGES * KC * SEGB;                 // [STAGES][BTILE]
  uint64_t* full = (uint64_t*)(sm + STAGES * T::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* afull = empty + STAGES;
  uint64_t* aempty = afull + NAB;
  uint64_t* tfull = aempty + NAB;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (wid == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NAB; ++a) {
      mbar_init(&afull[a], CW);
      mbar_init(&aempty[a], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, CW);
    fence_mbar_init();
  }
  if (wid == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();

  const long long kit = *D.iter;
  const int par = (int)((kit + (cur ? 0 : 1)) & 1);
  const int cnt = D.sup_cnt[par];
  const bool skip = *D.stop || cnt == 0;
  const int R = D.R;
  const int nslab = (D.n + SR - 1) / SR;
  const int per = max(1, (int)gridDim.x / nslab);
  int64_t es = ((int64_t)max(cnt, 1) + per - 1) / per;
  es = ((es + KC - 1) / KC) * KC;
  const int64_t nsl = ((int64_t)cnt + es - 1) / es;
  const int64_t nwork = skip ? 0 : nsl * nslab;

  if (wid == 0) {
    // ===================== producer: lane = support entry of the chunk
    const int32_t* sidx = D.sup_idx[par];
    const double* sc = D.sup_c[par];
    double scale[RMAX];
    bool act[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      act[r] = r < R && (cur || D.status[r] == ST_ACTIVE);
      const double cm = r < R ? __longlong_as_double((long long)D.cmax[par * R + r]) : 0.0;
      scale[r] = ldexp(1.0, fwd_exponent(cm, cnt, D.n));
    }
    const uint64_t pol = policy_evict_first();
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const int slab = (int)(w % nslab);
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      const int64_t boff = (int64_t)slab * SEGB;
      const uint32_t bytes = (uint32_t)min((int64_t)SEGB, D.ld - boff);
      long long mt[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) mt[r] = 0;
      // software pipeline: the entry (column, beta/s) loads of chunk i+1 and the colsum load of
      // chunk i+1 are in flight while chunk i is written out
      int32_t ncol = 0;
      double nsc[RMAX];
      long long ncs = 0;
      {
        const int64_t e = e0 + lane;
        if (e < e1) {
          ncol = sidx[e];
#pragma unroll
          for (int r = 0; r < RMAX; ++r) nsc[r] = r < R ? sc[e * R + r] : 0.0;
          ncs = (slab == 0) ? (long long)D.colsum[ncol] : 0;
        }
      }
      for (int64_t g0 = e0; g0 < e1; g0 += KC) {
        const int64_t e = g0 + lane;
        const bool live = e < e1;
        const int ng = (int)min((int64_t)KC, e1 - g0);
        const int32_t col = ncol;
        const long long cs = ncs;
        long long C[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          C[r] = (live && act[r]) ? __double2ll_rn(nsc[r] * scale[r]) : 0;
          mt[r] += cs * C[r];
        }
        {
          const int64_t en = e + KC;
          if (en < e1) {
            ncol = sidx[en];
#pragma unroll
            for (int r = 0; r < RMAX; ++r) nsc[r] = r < R ? sc[en * R + r] : 0.0;
          }
        }
        mbar_wait(&empty[stage], phase ^ 1);
        // digits of C: six balanced base-256 digits per RHS, d0 least significant; rows >= 6R stay 0
        uint8_t* bt = sB + stage * T::BTILE;
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          long long v = C[r];
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const int d = (int)(int8_t)(v & 0xFF);
            v = (v - d) >> 8;
            bt[btile_off(6 * r + q, lane)] = (uint8_t)(int8_t)d;
          }
        }
        for (int nrow = 6 * RMAX; nrow < N; ++nrow) bt[btile_off(nrow, lane)] = 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_expect_tx(&full[stage], bytes * (uint32_t)ng);
        __syncwarp();
        if (live) bulk_g2s(sdata + (stage * KC + lane) * SEGB, D.X8 + (int64_t)col * D.ld + boff, bytes, &full[stage], pol);
        if (slab == 0 && e + KC < e1) ncs = (long long)D.colsum[ncol];
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
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
  } else if (wid == 1) {
    // ===================== MMA issuer (elected lane)
    constexpr uint32_t idesc = idesc_i8(N);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t sB0 = smem_u32(sB);
    int stage = 0, ab = 0;
    uint32_t phase = 0, aphase = 0, tph = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      mbar_wait(tempty, tph ^ 1);
      tc_fence_after();
      bool first = true;
      for (int64_t g0 = e0; g0 < e1; g0 += KC) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&afull[ab], aphase);
        tc_fence_after();
        const uint64_t bdesc = umma_desc_kmajor_noswz(sB0 + (uint32_t)(stage * T::BTILE));
        if (elect_one()) {
#pragma unroll
          for (int t = 0; t < RT; ++t)
            umma_i8_ta(tbase + (uint32_t)(t * N), tbase + (uint32_t)(T::A_COL0 + ab * T::ACOLS + t * (KC / 4)), bdesc,
                       idesc, first ? 0u : 1u);
          umma_commit(&empty[stage]);
          umma_commit(&aempty[ab]);
        }
        __syncwarp();
        first = false;
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++ab == NAB) {
          ab = 0;
          aphase ^= 1;
        }
      }
      if (elect_one()) umma_commit(tfull);
      __syncwarp();
      tph ^= 1;
    }
  } else if (wid >= 4) {
    // ===================== converters (TMEM lane quarter wid-4 = rows of every row tile) + epilogue
    const int q4 = wid & 3, h = (wid - 4) >> 2;   // lane quarter, row-tile subset
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int stage = 0, ab = 0;
    uint32_t phase = 0, aphase = 0, tph = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const int slab = (int)(w % nslab);
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      for (int64_t g0 = e0; g0 < e1; g0 += KC) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&aempty[ab], aphase ^ 1);
        tc_fence_after();
        const uint8_t* sd = sdata + stage * KC * SEGB;
#pragma unroll 1
        for (int t = h; t < RT; t += CG) {
          const int row = t * 128 + q4 * 32 + lane;   // row within the slab
          uint32_t wv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int k = 4 * j + u;
              if (ST == 1) {
                b[u] = sd[k * SEGB + row];
              } else {
                b[u] = (sd[k * SEGB + (row >> 2)] >> (2 * (row & 3))) & 3u;
              }
            }
            wv[j] = __byte_perm(__byte_perm(b[0], b[1], 0x1140u), __byte_perm(b[2], b[3], 0x1140u), 0x5410u);
          }
          tmem_st8(tmem_base + lane_off + (uint32_t)(T::A_COL0 + ab * T::ACOLS + t * (KC / 4)), wv);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[ab]);
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++ab == NAB) {
          ab = 0;
          aphase ^= 1;
        }
      }
      // ---- epilogue of the work item: S_{i,r} = sum_k 256^k D_k, one int64 atomic per row and RHS
      mbar_wait(tfull, tph);
      tph ^= 1;
      tc_fence_after();
#pragma unroll 1
      for (int t = h; t < RT; t += CG) {
        const int row = slab * SR + t * 128 + q4 * 32 + lane;
        int32_t dv[N];
#pragma unroll
        for (int h = 0; h < N / 16; ++h) {
          uint32_t v[16];
          tmem_ld16(tmem_base + lane_off + (uint32_t)(t * N + h * 16), v);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 16; ++u) dv[h * 16 + u] = (int32_t)v[u];
        }
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          long long S = 0;
#pragma unroll
          for (int q = 5; q >= 0; --q) S = S * 256 + (long long)dv[6 * r + q];
          if (r < R && row < D.n && S != 0)
            atomicAdd((unsigned long long*)&D.sacc[(int64_t)r * D.n + row], (unsigned long long)S);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

template <int RMAX, int ST>
cudaError_t init_one() {
  return cudaFuncSetAttribute(k1_tc_kernel<RMAX, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              K1T<RMAX, ST>::SMEM);
}

template <int RMAX>
void launch_r(const Dev& D, int grid, cudaStream_t st, int cur) {
  if (D.storage == 1)
    launch_pdl(k1_tc_kernel<RMAX, 1>, dim3(grid), dim3(K1T<RMAX, 1>::THREADS), K1T<RMAX, 1>::SMEM, st, D, cur);
  else
    launch_pdl(k1_tc_kernel<RMAX, 2>, dim3(grid), dim3(K1T<RMAX, 2>::THREADS), K1T<RMAX, 2>::SMEM, st, D, cur);
}

}  // namespace

cudaError_t k1_tc_init() {
  cudaError_t e;
#define K1TC_INIT(R)                                              \
  if ((e = init_one<R, 1>()) != cudaSuccess) return e;            \
  if ((e = init_one<R, 2>()) != cudaSuccess) return e;
  K1TC_INIT(1) K1TC_INIT(2) K1TC_INIT(4) K1TC_INIT(8) K1TC_INIT(16)
#undef K1TC_INIT
  return cudaSuccess;
}

// grid = number of SMs (one CTA per SM: the stage ring takes ~192 KB of shared memory)
void launch_k1_tc(const Dev& D, int grid, cudaStream_t st, int cur) {
  if (D.R <= 1) launch_r<1>(D, grid, st, cur);
  else if (D.R <= 2) launch_r<2>(D, grid, st, cur);
  else if (D.R <= 4) launch_r<4>(D, grid, st, cur);
  else if (D.R <= 8) launch_r<8>(D, grid, st, cur);
  else launch_r<16>(D, grid, st, cur);
}
