// k_pivotal.cu — the pivotal statistic of the lambda grid ("generated via the
// pivotal quantity approach"; App. F is missing, reading R18) on the tensor cores.
//
//   Lambda_b = max_{j>=1} | sum_i x~_ij (tau - 1{U_ib <= tau}) | / n,   b = 0..B-1.
//
// With b_i = 1{U_ib <= tau} in {0, 1} and sum_i x~_ij = 0 (standardised columns),
//   sum_i x~_ij (tau - b_i) = -(n Sb_j - colsum_j nb) / (n s_j),   Sb_j = sum_i G_ij b_i,
// an exact integer GEMM: D[draw, column] = sum_i b_{draw,i} G_{i,column}.  This is the
// genuinely skinny-GEMM-shaped step of the method: 128 replicates per
// pass over X as the M = 128 rows of tcgen05.mma.kind::i8, 256 genotype columns per tile as N,
// samples as K (both operands K-major: draws are stored sample-contiguous, and X is SNP-major).
// The epilogue keeps, per thread (= replicate = TMEM lane), the running max over columns.
#include <cuda.h>

#include "fsqr_dev.cuh"

namespace {

constexpr int PD = 128;                  // replicates per pass (UMMA M, TMEM lanes)
constexpr int PN = 256;                  // genotype columns per tile (UMMA N)
constexpr int PK = 128;                  // samples per stage (one 128-byte swizzle row)
constexpr int A_BYTES = PD * PK;         // 16 KB of draws
constexpr int B_BYTES = PN * PK;         // 32 KB of X
constexpr int STAGE = A_BYTES + B_BYTES;
constexpr int STAGES = 4;
constexpr int THREADS = 256;             // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-7 epilogue
constexpr int SMEM = 1024 + STAGES * STAGE + 1024;

__device__ __forceinline__ uint64_t pmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// U_bi = top 53 bits of splitmix64(seed ^ splitmix64((b << 32) | i)); draws[q][i] = 1{U <= tau}
__global__ void k_piv_draws(int n, int ldk, double tau, uint64_t seed, long long b0, int8_t* draws, int* nb) {
  __shared__ int red[32];
  const int q = blockIdx.x;
  int cnt = 0;
  for (int i = threadIdx.x; i < ldk; i += blockDim.x) {
    int8_t v = 0;
    if (i < n) {
      const uint64_t h = pmix(seed ^ pmix(((uint64_t)(b0 + q) << 32) | (uint64_t)i));
      v = ((double)(h >> 11) * 0x1.0p-53) <= tau ? 1 : 0;
    }
    draws[(int64_t)q * ldk + i] = v;
    cnt += v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w];
    nb[q] = a;
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    k_piv_kernel(const Dev D, const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                 const int* nb, unsigned long long* lmax) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((1023 + 1) - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (D.p + PN - 1) / PN;
  const int kblocks = (D.n + PK - 1) / PK;

  if (wid == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmX);
    for (int s = 0; s < STAGES; ++s) {
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
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (wid == 0) {
    const uint64_t pol_x = policy_evict_first(), pol_a = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&full[stage], (uint32_t)STAGE);
          tma_load_2d(sA + stage * A_BYTES, &tmA, &full[stage], kb * PK, 0, pol_a);
          tma_load_2d(sB + stage * B_BYTES, &tmX, &full[stage], kb * PK, (int)(t * PN), pol_x);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (wid == 1) {
    constexpr uint32_t idesc = idesc_i8(PN);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
    int stage = 0;
    uint32_t phase = 0;
    int lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int acc = lt & 1;
      mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tbase + (uint32_t)(acc * PN);
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t adesc = umma_desc_sw128(sA0 + (uint32_t)(stage * A_BYTES));
        const uint64_t bdesc = umma_desc_sw128(sB0 + (uint32_t)(stage * B_BYTES));
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < PK / 32; ++k)
            umma_i8(d_tmem, adesc + (uint64_t)(2 * k), bdesc + (uint64_t)(2 * k), idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (wid >= 4) {
    // thread = replicate (TMEM lane 32*(wid-4) + lane); running max over the columns of its tiles
    const int q = wid - 4;
    const int d = q * 32 + lane;
    const long long n = D.n;
    const long long nbd = nb[d];
    double vmax = 0.0;
    int lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < PN / 16; ++h) {
        uint32_t v[16];
        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * PN + h * 16), v);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int64_t c = t * PN + h * 16 + u;
          if (c < D.p) {
            const long long num = n * (long long)(int32_t)v[u] - (long long)D.colsum[c] * nbd;
            vmax = fmax(vmax, fabs((double)num) * D.inv_sd[c]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    const double lam = vmax / ((double)n * (double)n);
    atomicMax(lmax + d, (unsigned long long)__double_as_longlong(lam));
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

}  // namespace

int pivotal_smem_bytes() { return SMEM; }

cudaError_t pivotal_init() {
  return cudaFuncSetAttribute(k_piv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
}

void launch_piv_draws(int n, int ldk, double tau, uint64_t seed, long long b0, int8_t* draws, int* nb,
                      cudaStream_t st) {
  k_piv_draws<<<PD, 256, 0, st>>>(n, ldk, tau, seed, b0, draws, nb);
}

void launch_pivotal(const Dev& D, const void* tmA, const void* tmX256, const int* nb, unsigned long long* lmax,
                    int grid, cudaStream_t st) {
  k_piv_kernel<<<grid, THREADS, SMEM, st>>>(D, *(const CUtensorMap*)tmA, *(const CUtensorMap*)tmX256, nb, lmax);
}
