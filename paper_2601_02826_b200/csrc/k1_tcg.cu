// k1_tcg.cu — a4 on the tensor cores for uint8 genotypes with NO CUDA-core touch of X:
// s^{k+1} = X~ beta^{k+1} over the support, exact integer arithmetic.
//
//   S_{i,r} = sum_{j in S} x_ij C_{j,r} = sum_k 256^k D_{i,(r,k)},   D = X_S · Dig   (see k1_tc.cu)
//
// X is SNP-major, so for the GEMM D[M = rows][N = digits] = A[rows][K = support] · B the A
// operand is MN-major (rows contiguous) -- a major-ness tcgen05 accepts for 8-bit integers.
// The producer gathers it with TMA `tile::gather4`: one instruction brings the same 128-row
// window of four support columns, and the 128B swizzle of the destination rows is exactly the
// canonical MN-major SWIZZLE_128B atom (8 K-rows of 128 MN-bytes).  Eight gathers fill the
// 128-row x 32-entry A tile of one row tile; the MMA reads it straight from shared memory.
// The coefficient digits (B, K-major, no swizzle) are written by the producer lanes; four
// epilogue warps turn the int32 digit sums into one int64 atomic per row and RHS.
#include <cuda.h>

#include "fsqr_dev.cuh"

namespace {

constexpr int KC = 32;         // support entries per chunk (one kind::i8 MMA K step)
constexpr int THREADS = 256;   // w0 producer, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 epilogue

template <int RMAX>
struct K1G {
  static constexpr int NDIG = 6 * RMAX;
  static constexpr int N = NDIG <= 16 ? 16 : (NDIG <= 32 ? 32 : (NDIG <= 48 ? 48 : 96));
  static constexpr int RT0 = 512 / N;
  static constexpr int RT = RT0 >= 16 ? 16 : (RT0 >= 8 ? 8 : (RT0 >= 4 ? 4 : 2));   // row tiles per slab
  static constexpr int SR = 128 * RT;
  static constexpr int ATILE = 128 * KC;                  // one row tile x one chunk: 4 KB
  static constexpr int BTILE = N * KC;
  static constexpr int STAGE = RT * ATILE + BTILE;
  static constexpr int ST0 = (192 * 1024) / STAGE;
  static constexpr int STAGES = ST0 < 2 ? 2 : (ST0 > 8 ? 8 : ST0);
  static constexpr int SMEM = 1024 + STAGES * STAGE + 1024;
  static_assert(RT * N <= 512, "TMEM budget");
};

__device__ __forceinline__ void tma_gather4(void* dst, const void* tmap, uint64_t* bar, int x, int y0, int y1,
                                            int y2, int y3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y0), "r"(y1), "r"(y2), "r"(y3), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ int btile_off(int nrow, int k) {
  return (nrow >> 3) * 256 + (nrow & 7) * 16 + (k >> 4) * 128 + (k & 15);
}
// K-major, no swizzle (B: digits)
__device__ __forceinline__ uint64_t desc_k_noswz(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(128u >> 4) << 16;   // LBO: the two 16-entry halves of K
  d |= (uint64_t)(256u >> 4) << 32;   // SBO: 8-row groups
  d |= (uint64_t)1u << 46;
  return d;
}
// MN-major, SWIZZLE_128B (A: 128 rows x 32 entries = four 1 KB atoms of 8 entries)
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(4096u >> 4) << 16;  // LBO: next 128-row MN atom (unused for M = 128)
  d |= (uint64_t)(1024u >> 4) << 32;  // SBO: next group of 8 entries
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;            // SWIZZLE_128B
  return d;
}
// kind::i8, D s32, A s8 MN-major, B s8 K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_i8_amn(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int RMAX>
__global__ void __launch_bounds__(THREADS, 1)
    k1_tcg_kernel(const Dev D, const __grid_constant__ CUtensorMap tmG, int cur) {
  using T = K1G<RMAX>;
  constexpr int RT = T::RT, SR = T::SR, N = T::N, STAGES = T::STAGES;
  extern __shared__ uint8_t k1g_raw[];
  uint8_t* sm = k1g_raw + (((1023 + 1) - (smem_u32(k1g_raw) & 1023)) & 1023);
  uint8_t* sA = sm;                                    // [STAGES][RT][4 KB]
  uint8_t* sB = sm + STAGES * RT * T::ATILE;           // [STAGES][BTILE]
  uint64_t* full = (uint64_t*)(sm + STAGES * T::STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (wid == 0 && lane == 0) {
    prefetch_tmap(&tmG);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
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
      long long mt[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) mt[r] = 0;
      const int col_first = sidx[e0];   // stands in for the missing entries of a tail chunk (digits 0)
      for (int64_t g0 = e0; g0 < e1; g0 += KC) {
        const int64_t e = g0 + lane;
        const bool live = e < e1;
        int32_t col = col_first;
        long long C[RMAX];
#pragma unroll
        for (int r = 0; r < RMAX; ++r) C[r] = 0;
        if (live) {
          col = sidx[e];
          const long long cs = (slab == 0) ? (long long)D.colsum[col] : 0;
#pragma unroll
          for (int r = 0; r < RMAX; ++r) {
            C[r] = act[r] ? __double2ll_rn(sc[e * R + r] * scale[r]) : 0;
            mt[r] += cs * C[r];
          }
        }
        mbar_wait(&empty[stage], phase ^ 1);
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
        if (lane == 0) mbar_expect_tx(&full[stage], (uint32_t)(RT * T::ATILE));
        __syncwarp();
        // 8 gathers of 4 entries per row tile; lane L issues (row tile, group) pairs L, L + 32, ...
        for (int q = lane; q < RT * 8; q += 32) {
          const int t = q >> 3, gq = q & 7;
          const int c0 = __shfl_sync(__activemask(), col, 4 * gq);
          const int c1 = __shfl_sync(__activemask(), col, 4 * gq + 1);
          const int c2 = __shfl_sync(__activemask(), col, 4 * gq + 2);
          const int c3 = __shfl_sync(__activemask(), col, 4 * gq + 3);
          tma_gather4(sA + (stage * RT + t) * T::ATILE + gq * 512, &tmG, &full[stage], slab * SR + t * 128, c0, c1,
                      c2, c3, pol);
        }
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
    // ===================== MMA issuer (elected lane): A MN-major from smem, B K-major from smem
    constexpr uint32_t idesc = idesc_i8_amn(N);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
    int stage = 0;
    uint32_t phase = 0, tph = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      mbar_wait(tempty, tph ^ 1);
      tc_fence_after();
      bool first = true;
      for (int64_t g0 = e0; g0 < e1; g0 += KC) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t bdesc = desc_k_noswz(sB0 + (uint32_t)(stage * T::BTILE));
        if (elect_one()) {
#pragma unroll
          for (int t = 0; t < RT; ++t)
            umma_i8(tbase + (uint32_t)(t * N), desc_mn_sw128(sA0 + (uint32_t)((stage * RT + t) * T::ATILE)), bdesc,
                    idesc, first ? 0u : 1u);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        first = false;
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) umma_commit(tfull);
      __syncwarp();
      tph ^= 1;
    }
  } else if (wid >= 4) {
    // ===================== epilogue: TMEM lane quarter wid-4 = rows of every row tile
    const int q4 = wid - 4;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    uint32_t tph = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x) {
      const int slab = (int)(w % nslab);
      mbar_wait(tfull, tph);
      tph ^= 1;
      tc_fence_after();
#pragma unroll 1
      for (int t = 0; t < RT; ++t) {
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

template <int RMAX>
void launch_r(const Dev& D, const void* tmG, int grid, cudaStream_t st, int cur) {
  launch_pdl(k1_tcg_kernel<RMAX>, dim3(grid), dim3(THREADS), K1G<RMAX>::SMEM, st, D, *(const CUtensorMap*)tmG, cur);
}

template <int RMAX>
cudaError_t init_one() {
  return cudaFuncSetAttribute(k1_tcg_kernel<RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, K1G<RMAX>::SMEM);
}

}  // namespace

cudaError_t k1_tcg_init() {
  cudaError_t e;
  if ((e = init_one<1>()) != cudaSuccess) return e;
  if ((e = init_one<2>()) != cudaSuccess) return e;
  if ((e = init_one<4>()) != cudaSuccess) return e;
  if ((e = init_one<8>()) != cudaSuccess) return e;
  return init_one<16>();
}

void launch_k1_tcg(const Dev& D, const void* tmG, int grid, cudaStream_t st, int cur) {
  if (D.R <= 1) launch_r<1>(D, tmG, grid, st, cur);
  else if (D.R <= 2) launch_r<2>(D, tmG, grid, st, cur);
  else if (D.R <= 4) launch_r<4>(D, tmG, grid, st, cur);
  else if (D.R <= 8) launch_r<8>(D, tmG, grid, st, cur);
  else launch_r<16>(D, tmG, grid, st, cur);
}
