// k2_tc.cu — a1+a2 on the 5th-generation tensor cores (sm_100a).
//
// One outer FS-QRPPA iteration streams the whole genotype matrix once through
// this kernel: g^k = X~^T theta^k (PAPER.md:L392,
// "matrix-vector products ... X^T theta"), then the weighted soft-threshold prox
// beta^{k+1} = E14(beta^k, g^k) (L274-277), the support list of beta^{k+1}, and
// the R_beta(w^k) / penalty partials of the stopping test.
//
// Mapping: X is stored SNP-major (column c = n contiguous bytes), which is
// exactly the K-major A operand of D[c, q] = sum_i X[i, c] * B[i, q] with
// M = 128 columns per tile, K = n samples and N = npad digit rows of theta.
// Persistent CTAs (one per SM) walk tiles of 128 columns; a TMA producer warp
// streams 128x128-byte A boxes (SWIZZLE_128B) plus the matching B box through
// an mbarrier ring; one elected thread issues tcgen05.mma kind::i8 into a
// double-buffered int32 TMEM accumulator; four epilogue warps (one per TMEM
// lane quarter) read the exact digit sums with tcgen05.ld and run the fp64
// epilogue while the next tile accumulates.  X is read from HBM exactly once
// per iteration with an evict-first L2 policy; B (theta digits, <= 1.3 MB) is
// L2-resident and re-read per stage with evict-last.
#include <cuda.h>

#include "k2_common.cuh"

namespace {

constexpr int TILE_M = 128;   // columns per tile (UMMA M)
constexpr int TILE_K = 128;   // bytes of K per stage (one 128B swizzle row)
constexpr int A_BYTES = TILE_M * TILE_K;
constexpr int THREADS = 256;  // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4..7 epilogue

template <int NPAD, int RM>
struct Cfg {
  static constexpr int B_BYTES = NPAD * TILE_K;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE;
  static constexpr int RMAX = RM;   // RHS slots compiled in (<= NPAD / 4)
  static constexpr int TMEM_COLS = (2 * NPAD <= 32) ? 32 : (2 * NPAD <= 64 ? 64 : (2 * NPAD <= 128 ? 128 : 256));
  static constexpr int RED0 = (THREADS / 32) * RMAX * (FSQR_NPART + 1);
  static constexpr int RED_DOUBLES = RED0 > 33 * FSQR_NPART ? RED0 : 33 * FSQR_NPART;
  static constexpr int SMEM = 1024 /*align slack*/ + STAGES * STAGE + 1024 /*barriers*/ + RED_DOUBLES * 8;
};

template <int NPAD, int RM>
__global__ void __launch_bounds__(THREADS, 1)
    k2_tc_kernel(const Dev D, const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmB) {
  using CF = Cfg<NPAD, RM>;
  constexpr int RMAX = CF::RMAX;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((1023 + 1) - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + CF::STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + CF::STAGES * CF::STAGE);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* tfull = empty + CF::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  double* red = (double*)(smem + CF::STAGES * CF::STAGE + 1024);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (D.p + TILE_M - 1) / TILE_M;
  const int kblocks = (D.n + TILE_K - 1) / TILE_K;

  if (wid == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmB);
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (wid == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(CF::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // digit rows 4R..NPAD-1 of every B stage are never loaded (the TMA box has 4R rows): zero them
  // once, then make the generic-proxy stores visible to the tensor core's async proxy
  {
    constexpr int BROW = 128;   // bytes of one digit row per stage
    const int live = 4 * D.R;
    for (int s = 0; s < CF::STAGES; ++s)
      for (int a = 0; a < 1; ++a) {
        uint8_t* base = sB + s * CF::B_BYTES + a * NPAD * 128;
        for (int q = live * 128 + tid * 16; q < NPAD * 128; q += THREADS * 16) *(uint4*)(base + q) = make_uint4(0, 0, 0, 0);
      }
    (void)BROW;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();
  if (*D.stop) {   // uniform: every thread reads the same flag
    tc_fence_before();
    __syncthreads();
    if (wid == 2) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CF::TMEM_COLS)
                   : "memory");
    }
    return;
  }
  K2Part<RMAX> P;
  k2_part_init(P, red);
  K2Ctx<RMAX> C;
  k2_load_ctx(D, C);

  if (wid == 0) {
    // ===== TMA producer: the whole warp walks the ring, one elected lane issues =====
    {
      const uint64_t pol_x = D.x_policy == 2 ? policy_evict_last()
                             : (D.x_policy == 1 ? policy_evict_normal() : policy_evict_first());
      const uint64_t pol_b = policy_evict_last();
      const uint32_t bytes = (uint32_t)(A_BYTES + 4 * D.R * 128);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&full[stage], bytes);
            tma_load_2d(sA + stage * A_BYTES, &tmX, &full[stage], kb * TILE_K, (int)(t * TILE_M), pol_x);
            tma_load_2d(sB + stage * CF::B_BYTES, &tmB, &full[stage], kb * TILE_K, 0, pol_b);
          }
          __syncwarp();
          if (++stage == CF::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (wid == 1) {
    // ===== MMA issuer: the whole warp walks the pipeline, one elected lane issues =====
    {
      constexpr uint32_t idesc = idesc_i8(NPAD);
      const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
      int stage = 0;
      uint32_t phase = 0;
      int lt = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const int acc = lt & 1;
        const uint32_t aph = (lt >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tbase + (uint32_t)(acc * NPAD);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(sA0 + (uint32_t)(stage * A_BYTES));
          const uint64_t bdesc = umma_desc_sw128(sB0 + (uint32_t)(stage * CF::B_BYTES));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < TILE_K / 32; ++k)   // K = 32 bytes per kind::i8 MMA
              umma_i8(d_tmem, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc, (kb | k) != 0);
            umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == CF::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
      }
    }
  } else if (wid >= 4) {
    // ===== epilogue: TMEM lanes 32*(wid-4) .. +31 = columns of the tile =====
    const int q = wid - 4;
    int lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int acc = lt & 1;
      const uint32_t aph = (lt >> 1) & 1;
      epi_prefetch<RMAX>(D, C, (t + (int64_t)gridDim.x) * TILE_M + q * 32 + lane);
      mbar_wait_park(&tfull[acc], aph);
      tc_fence_after();
      int32_t dv[NPAD];
#pragma unroll
      for (int h = 0; h < NPAD / 16; ++h) {
        uint32_t v[16];
        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * NPAD + h * 16), v);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) dv[h * 16 + u] = (int32_t)v[u];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);

      const int64_t c = t * TILE_M + q * 32 + lane;
      const bool valid = c < D.p;
      double g[RMAX];
      if (valid) {
        const int32_t cs = D.colsum[c];
        const double isd = D.inv_sd[c];
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          g[r] = r < C.R ? g_from_digits(D.n, cs, C.cs->Tsum[r], C.cs->gscale[r], isd, dv + 4 * r) : 0.0;
      } else {
#pragma unroll
        for (int r = 0; r < RMAX; ++r) g[r] = 0.0;
      }
      const bool nz = epi_column<RMAX>(D, C, valid ? c : 0, g, P, valid);
      if (D.update) support_append<RMAX>(D, C, nz, c);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CF::TMEM_COLS)
                 : "memory");
  }
  k2_finish<RMAX>(D, C, P, red);
}

template <int NPAD, int RM>
void launch_np(const Dev& D, const void* tmX, const void* tmB, int grid, cudaStream_t st) {
  launch_pdl(k2_tc_kernel<NPAD, RM>, dim3(grid), dim3(THREADS), Cfg<NPAD, RM>::SMEM, st, D, *(const CUtensorMap*)tmX,
                                                                *(const CUtensorMap*)tmB);
}

template <int NPAD, int RM>
cudaError_t init_np() {
  return cudaFuncSetAttribute(k2_tc_kernel<NPAD, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<NPAD, RM>::SMEM);
}

}  // namespace

cudaError_t k2_tc_init() {
  cudaError_t e;
  if ((e = init_np<16, 1>()) != cudaSuccess) return e;
  if ((e = init_np<16, 4>()) != cudaSuccess) return e;
  if ((e = init_np<32, 8>()) != cudaSuccess) return e;
  if ((e = init_np<48, 12>()) != cudaSuccess) return e;
  return init_np<64, 16>();
}

int k2_tc_supported(int npad) { return npad == 16 || npad == 32 || npad == 48 || npad == 64; }

int k2_tc_smem_bytes(int npad) {
  switch (npad) {
    case 16: return Cfg<16, 4>::SMEM;
    case 32: return Cfg<32, 8>::SMEM;
    case 48: return Cfg<48, 12>::SMEM;
    default: return Cfg<64, 16>::SMEM;
  }
}

void launch_k2_tc(const Dev& D, const void* tmX, const void* tmB, int grid, cudaStream_t st) {
  if (D.R == 1) launch_np<16, 1>(D, tmX, tmB, grid, st);
  else if (D.npad == 16) launch_np<16, 4>(D, tmX, tmB, grid, st);
  else if (D.npad == 32) launch_np<32, 8>(D, tmX, tmB, grid, st);
  else if (D.npad == 48) launch_np<48, 12>(D, tmX, tmB, grid, st);
  else launch_np<64, 16>(D, tmX, tmB, grid, st);
}
