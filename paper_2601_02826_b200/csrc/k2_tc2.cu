// k2_tc2.cu — a1+a2 for 2-bit packed genotypes on the 5th-generation tensor cores.
//
// The same pass as k2_tc.cu (g^k = X~^T theta^k; beta prox E14,
// L274-277; support list; R_beta / penalty partials), for the PACKED2 storage
// of config C4 (4 samples per byte).  Unpacking 2-bit codes to bytes in shared
// memory would cost 4x the shared-memory bandwidth of the packed stream, so the
// unpacked A operand goes to TENSOR MEMORY instead:
//
//   TMA (warp 0): 128 columns x 128 packed bytes (= 512 samples) per stage,
//       SWIZZLE_128B, plus the matching 512-sample slice of the theta digit
//       planes (four 128-byte swizzle atoms of NPAD rows).
//   convert (warps 4-7, one TMEM lane quarter each): thread = tile column c
//       reads its 128 packed bytes (8 conflict-free 16-byte loads thanks to the
//       swizzle), and for q = 0..3 forms (w >> 2q) & 0x03030303 from each packed
//       word w -- the codes of samples 16u + 4b + q, one per byte -- and stores
//       them with tcgen05.st into a 128-column TMEM A buffer (3 buffers).  The
//       K order inside a 512-sample block is therefore kappa = 128q + 4u + b for
//       sample s = 16u + 4b + q; the digit planes of theta are written in that
//       same order by finalize (D.bperm), so the dot products are unchanged.
//   MMA (warp 1, one thread): 16 x tcgen05.mma.kind::i8 (K = 32) per stage with
//       A read from TMEM and B from shared memory into a double-buffered int32
//       accumulator (exact).
//   epilogue (warps 8-11): identical to k2_tc.cu.
// X is read from HBM exactly once per iteration; the CUDA cores spend about two
// instructions per four samples on unpacking.
// Two kernels: k2_tc2_kernel (1..4 RHS, one tile at a time) and k2_tc2_pair_kernel (5..16 RHS:
// two tiles share each theta-digit stage, see its header below); k2p_kernel is the same pipeline
// for the power / Lanczos back pass of the setup.
#include <cuda.h>

#include "k2_common.cuh"

#ifndef K2TC2_SMEM_KB
#define K2TC2_SMEM_KB 226
#endif
#ifndef K2TC2_CW
#define K2TC2_CW 8   // converter warps (two per SM sub-partition: the unpack loop is latency-bound with one)
#endif
#ifndef K2TC2_CWM
#define K2TC2_CWM 8  // converter warps with several RHS, NPAD 32/48 (a 640-thread block: 96 registers, at most 16 bytes
                     // of stack; C5 K2 0.581 -> 0.572 ms against 4); NPAD = 64 keeps 4 (8 spills 144 bytes there)
#endif


#ifndef K2TC2_PAIR
#define K2TC2_PAIR 1 // several RHS (NPAD > 16): k2_tc2_pair_kernel, two column tiles share each theta-digit stage
#endif
#ifndef K2TC2_BTRIM
#define K2TC2_BTRIM 1  // pair order: a theta-digit stage holds only the 8-row groups with a live row
#endif
#ifndef K2TC2_NB
#define K2TC2_NB 3   // theta-digit stages of the pair order's own ring
#endif

namespace {

constexpr int TILE_M = 128;               // columns per tile (UMMA M)
constexpr int PK = 128;                   // packed bytes per column per stage
constexpr int KS = 4 * PK;                // samples (K) per stage
constexpr int A_BYTES = TILE_M * PK;      // 16 KB packed A per stage
constexpr int A_COLS = KS / 4;            // TMEM columns per A buffer (4 int8 per 32-bit cell)

// warps: 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4..4+CW-1 convert, then EW epilogue warps.  One RHS
// (the C4 workload) keeps few registers per thread, so it affords 8 converter warps (two per SM
// sub-partition: the unpack loop is latency-bound with one); more RHS keep 4.
template <int NPAD, int RM>
struct Cfg2 {
  // up to 4 RHS: 8 converter warps, 4 epilogue warps; more: the per-column epilogue (E14, KKT
  // partials and support entries for every RHS) is the slower side, so 4 converters and two sets
  // of 4 epilogue warps taking alternate tiles (one accumulator buffer each)
  static constexpr int CW = NPAD == 16 ? K2TC2_CW : (NPAD >= 64 ? 4 : K2TC2_CWM);   // (4 converters at NPAD = 16 would spill)
  static constexpr int EW = NPAD == 16 ? 4 : 8;
  // NPAD == 16: one accumulator per code plane q, so the converter can leave the codes in place
  // ((w & (3 << 2q)) = x * 4^q, one LOP per word instead of shift + mask); the epilogue divides
  // each plane's exact sum by 4^q.  Needs 2 x 4 x 16 = 128 TMEM columns.
  // NPAD > 16 (several RHS): four planes would not fit next to the A buffers, so two scale
  // groups: with w4 = w >> 4 (one SHF per word), planes 0 and 2 are w & M and w4 & M (x 1),
  // planes 1 and 3 are w & (M << 2) and w4 & (M << 2) (x 4): 5 instructions per word instead of 8.
  static constexpr bool SPLITQ = NPAD == 16;
  static constexpr int ACC_COLS = SPLITQ ? 4 * NPAD : 2 * NPAD;   // columns of one accumulator buffer
  static constexpr int A_COL0 = 2 * ACC_COLS;                     // A buffers after the accumulators
  static constexpr int NAB = (512 - A_COL0) / A_COLS < 3 ? (512 - A_COL0) / A_COLS : 3;   // TMEM A buffers
  static_assert(NAB >= 2, "TMEM budget");
  static constexpr int THREADS = 32 * (4 + CW + EW);
  static constexpr int B_ATOM = NPAD * 128;
  static constexpr int B_BYTES = 4 * B_ATOM;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int RMAX = RM;   // RHS slots compiled in (<= NPAD / 4)
  static constexpr int RED0 = (THREADS / 32) * RMAX * (FSQR_NPART + 1);
  static constexpr int RED_DOUBLES = RED0 > 33 * FSQR_NPART ? RED0 : 33 * FSQR_NPART;
  // as many stages as fit: several RHS make the theta-digit B tile (4 x NPAD x 128 B) larger than
  // the 16 KB X tile, and the X bytes in flight are what keep HBM busy
  static constexpr int STAGES = (K2TC2_SMEM_KB * 1024 - 2048 - RED_DOUBLES * 8) / STAGE;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 1024 + RED_DOUBLES * 8;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ void umma_i8_tmem_a(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int NPAD, int RM>
__global__ void __launch_bounds__(Cfg2<NPAD, RM>::THREADS, 1)
    k2_tc2_kernel(const Dev D, const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmB) {
  using CF = Cfg2<NPAD, RM>;
  constexpr int RMAX = CF::RMAX;
  constexpr int CW = CF::CW;
  constexpr int THREADS = CF::THREADS;
  constexpr int EPI0 = 4 + CW;   // first epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((1023 + 1) - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + CF::STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + CF::STAGES * CF::STAGE);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* afull = empty + CF::STAGES;
  constexpr int NAB = CF::NAB, A_COL0 = CF::A_COL0;
  uint64_t* aempty = afull + NAB;
  uint64_t* tfull = aempty + NAB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  double* red = (double*)(smem + CF::STAGES * CF::STAGE + 1024);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (D.p + TILE_M - 1) / TILE_M;
  const int kblocks = (int)((D.ld + PK - 1) / PK);

  if (wid == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmB);
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NAB; ++a) {
      mbar_init(&afull[a], CW);
      mbar_init(&aempty[a], 1);
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
  // digit rows 4R..NPAD-1 of every B stage are never loaded (the TMA box has 4R rows): zero them
  // once, then make the generic-proxy stores visible to the tensor core's async proxy
  {
    constexpr int BROW = 512;   // bytes of one digit row per stage
    const int live = 4 * D.R;
    for (int s = 0; s < CF::STAGES; ++s)
      for (int a = 0; a < 4; ++a) {
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
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
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
      const uint32_t bytes = (uint32_t)(A_BYTES + 4 * 4 * D.R * 128);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&full[stage], bytes);
            tma_load_2d(sA + stage * A_BYTES, &tmX, &full[stage], kb * PK, (int)(t * TILE_M), pol_x);
#pragma unroll
            for (int a = 0; a < 4; ++a)
              tma_load_2d(sB + stage * CF::B_BYTES + a * CF::B_ATOM, &tmB, &full[stage], kb * KS + a * 128, 0, pol_b);
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
      constexpr uint32_t idesc = CF::SPLITQ ? idesc_u8s8(NPAD) : idesc_i8(NPAD);   // (codes x 4 <= 12 fit s8)
      const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t sB0 = smem_u32(sB);
      int stage = 0, ab = 0;
      uint32_t phase = 0, aphase = 0;
      int lt = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const int acc = lt & 1;
        const uint32_t tph = (lt >> 1) & 1;
        mbar_wait(&tempty[acc], tph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tbase + (uint32_t)(acc * CF::ACC_COLS);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          mbar_wait(&afull[ab], aphase);
          tc_fence_after();
          const uint32_t a_tmem = tbase + (uint32_t)(A_COL0 + ab * A_COLS);
          const uint64_t bdesc0 = umma_desc_sw128(sB0 + (uint32_t)(stage * CF::B_BYTES));
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < KS / 32; ++kk) {   // K = 32 samples per kind::i8 MMA; plane q = kk / 4
              const uint32_t dq = CF::SPLITQ ? d_tmem + (uint32_t)((kk >> 2) * NPAD)
                                             : d_tmem + (uint32_t)(((kk >> 2) & 1) * NPAD);
              const bool accum = CF::SPLITQ ? (kb != 0 || (kk & 3) != 0) : (kb != 0 || (kk & 11) != 0);   // first of each group: kk = 0, 4
              umma_i8_tmem_a(dq, a_tmem + (uint32_t)(8 * kk),
                             bdesc0 + (uint64_t)((kk >> 2) * (CF::B_ATOM >> 4) + 2 * (kk & 3)), idesc, accum);
            }
            umma_commit(&empty[stage]);
            umma_commit(&aempty[ab]);
          }
          __syncwarp();
          if (++stage == CF::STAGES) {
            stage = 0;
            phase ^= 1;
          }
          if (++ab == NAB) {
            ab = 0;
            aphase ^= 1;
          }
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
      }
    }
  } else if (wid >= 4 && wid < EPI0) {
    // ===== converters: TMEM lane quarter wid % 4 (thread = tile column), column half h of the
    // packed row when CW = 8 =====
    constexpr int CH = 8 / (CW / 4);          // 16-byte chunks per converter thread (8 or 4)
    constexpr int NW = 4 * CH;                // packed words per thread
    const int q4 = wid & 3;
    const int h = (wid - 4) >> 2;             // 0 (CW = 4) or 0/1 (CW = 8)
    const int c = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int stage = 0, ab = 0;
    uint32_t phase = 0, aphase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&aempty[ab], aphase ^ 1);
        tc_fence_after();
        uint32_t w[NW], w4[CF::SPLITQ ? 1 : NW];
        const uint8_t* row = sA + stage * A_BYTES + c * PK;
#pragma unroll
        for (int jj = 0; jj < CH; ++jj) {   // logical 16-byte chunk j sits at chunk j ^ (c & 7) (SWIZZLE_128B)
          const int j = h * CH + jj;
          const uint4 v = *(const uint4*)(row + ((j ^ (c & 7)) << 4));
          w[4 * jj] = v.x;
          w[4 * jj + 1] = v.y;
          w[4 * jj + 2] = v.z;
          w[4 * jj + 3] = v.w;
        }
        const uint32_t abase = tmem_base + lane_off + (uint32_t)(A_COL0 + ab * A_COLS + h * NW);
        if constexpr (!CF::SPLITQ) {
#pragma unroll
          for (int u = 0; u < NW; ++u) w4[u] = w[u] >> 4;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t o[NW];
#pragma unroll
          for (int u = 0; u < NW; ++u)
            o[u] = CF::SPLITQ ? (w[u] & (0x03030303u << (2 * q)))
                              : ((q & 2 ? w4[u] : w[u]) & (0x03030303u << (2 * (q & 1))));
          if constexpr (NW == 32) tmem_st32(abase + (uint32_t)(32 * q), o);
          else tmem_st16(abase + (uint32_t)(32 * q), o);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[ab]);
        if (++stage == CF::STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++ab == NAB) {
          ab = 0;
          aphase ^= 1;
        }
      }
    }
  } else if (wid >= EPI0) {
    // ===== epilogue: TMEM lanes 32*(wid%4) .. +31 = columns of the tile =====
    const int q = wid & 3;
    const int eset = (wid - EPI0) >> 2;   // 0, or 0/1 with two epilogue sets (alternate tiles)
    int lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int acc = lt & 1;
      if (CF::EW == 8 && acc != eset) continue;
      const uint32_t aph = (lt >> 1) & 1;
      epi_prefetch<RMAX>(D, C, (t + (int64_t)gridDim.x * (CF::EW == 8 ? 2 : 1)) * TILE_M + q * 32 + lane);
      mbar_wait_park(&tfull[acc], aph);
      tc_fence_after();
      int32_t dv[NPAD];
      if constexpr (CF::SPLITQ) {
#pragma unroll
        for (int u = 0; u < NPAD; ++u) dv[u] = 0;
#pragma unroll
        for (int pq = 0; pq < 4; ++pq) {   // plane pq holds 4^pq x its exact sum: divide exactly
#pragma unroll
          for (int h = 0; h < NPAD / 16; ++h) {
            uint32_t v[16];
            tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) +
                          (uint32_t)(acc * CF::ACC_COLS + pq * NPAD + h * 16), v);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 16; ++u) dv[h * 16 + u] += ((int32_t)v[u]) >> (2 * pq);
          }
        }
      } else {   // scale group 0 (planes 0, 2) + scale group 1 (planes 1, 3) / 4, exactly
#pragma unroll
        for (int h = 0; h < NPAD / 16; ++h) {
          uint32_t v[16], v1[16];
          tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * CF::ACC_COLS + h * 16), v);
          tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * CF::ACC_COLS + NPAD + h * 16), v1);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 16; ++u) dv[h * 16 + u] = (int32_t)v[u] + ((int32_t)v1[u] >> 2);
        }
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
  k2_finish<RMAX>(D, C, P, red);
}

// ---------------------------------------------------------------- several RHS: tile-pair order
// The same pass for NPAD > 16 (5..16 RHS).  With nine RHS a stage's theta digits (36 rows x 512 B =
// 18 KB, L2-resident) outweigh its 16 KB of X, and re-reading them for every 128-column tile made
// the L2 -> SM traffic 2.7x the X bytes (ncu: 6.9 GB of L2 sectors per pass).  So here a CTA walks
// its tiles two at a time, k-block by k-block: one theta-digit stage (its own ring of NB stages,
// its own producer warp) serves the X stages of both tiles; each tile of the pair has its
// accumulator buffer (two scale groups of NPAD columns, as above) and its set of four epilogue
// warps; the converters free an X stage as soon as its packed words are in registers.
// k2_tc2_kernel above stays the single-tile-order kernel (1..4 RHS): merging the two into one
// rewritten kernel cost 5 % at M and 8 % at C4 (profiles/r02s3_k2_single_vs_merged_ab.txt).
// warps: 0 TMA (X), 1 MMA, 2 TMEM alloc, 3 TMA (theta digits), 4..4+CW-1 convert, then 8 epilogue warps.
template <int NPAD, int RM>
struct Cfg2P {
  static_assert(NPAD > 16 && NPAD % 16 == 0 && 4 * RM <= NPAD, "several RHS");
  static constexpr int CW = NPAD >= 64 ? 4 : K2TC2_CWM;
  static constexpr int EW = 8;
  static constexpr int ACC_COLS = 2 * NPAD;      // columns of one accumulator buffer (scale groups x1, x4)
  static constexpr int A_COL0 = 2 * ACC_COLS;    // A buffers after the two accumulators
  static constexpr int NAB = (512 - A_COL0) / A_COLS < 3 ? (512 - A_COL0) / A_COLS : 3;   // TMEM A buffers
  static_assert(NAB >= 2, "TMEM budget");
  static constexpr int THREADS = 32 * (4 + CW + EW);
  static constexpr int RMAX = RM;   // RHS slots compiled in (<= NPAD / 4)
  // digit rows held per 128-byte K atom of a theta-digit stage: only the 8-row groups with a live
  // row (the MMA's N = NPAD then reads up to NPAD - BROWS rows of whatever follows in shared memory
  // into accumulator columns the epilogue never uses; integer arithmetic, so harmless)
  static constexpr int BROWS = K2TC2_BTRIM ? (4 * RM + 7) / 8 * 8 : NPAD;
  static constexpr int B_ATOM = BROWS * 128;
  static constexpr int B_BYTES = 4 * B_ATOM;
  static constexpr int RED0 = (THREADS / 32) * RMAX * (FSQR_NPART + 1);
  static constexpr int RED_DOUBLES = RED0 > 33 * FSQR_NPART ? RED0 : 33 * FSQR_NPART;
  static constexpr int BUDGET = K2TC2_SMEM_KB * 1024 - 2048 - RED_DOUBLES * 8;
  static constexpr int NBS = K2TC2_NB;                                 // theta-digit stages
  static constexpr int STAGES = (BUDGET - NBS * B_BYTES) / A_BYTES;    // X stages: as many as fit
  static_assert(STAGES >= 3 && 2 * STAGES + 2 * NBS + 2 * NAB + 5 <= 128, "ring sizes");
  static constexpr int RING = STAGES * A_BYTES + NBS * B_BYTES;
  static constexpr int SMEM = 1024 + RING + 1024 + RED_DOUBLES * 8;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

template <int NPAD, int RM>
__global__ void __launch_bounds__(Cfg2P<NPAD, RM>::THREADS, 1)
    k2_tc2_pair_kernel(const Dev D, const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmB) {
  using CF = Cfg2P<NPAD, RM>;
  constexpr int RMAX = CF::RMAX;
  constexpr int CW = CF::CW;
  constexpr int THREADS = CF::THREADS;
  constexpr int EPI0 = 4 + CW;   // first epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((1023 + 1) - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + CF::STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + CF::RING);   // X stage landed
  uint64_t* empty = full + CF::STAGES;             // X stage free: every converter warp has read it
  uint64_t* bfull = empty + CF::STAGES;            // theta-digit stage landed
  uint64_t* bempty = bfull + CF::NBS;              // theta-digit stage consumed by the MMAs of both tiles
  uint64_t* afull = bempty + CF::NBS;
  constexpr int NAB = CF::NAB, A_COL0 = CF::A_COL0;
  uint64_t* aempty = afull + NAB;
  uint64_t* tfull = aempty + NAB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  double* red = (double*)(smem + CF::RING + 1024);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (D.p + TILE_M - 1) / TILE_M;
  const int kblocks = (int)((D.ld + PK - 1) / PK);
  // this CTA's tiles: blockIdx.x, + gridDim.x, ... (local index lt; pair lt >> 1, accumulator lt & 1)
  const int ntl = blockIdx.x < ntiles ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;

  if (wid == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmB);
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    for (int s = 0; s < CF::NBS; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < NAB; ++a) {
      mbar_init(&afull[a], CW);
      mbar_init(&aempty[a], 1);
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
  // digit rows 4R..BROWS-1 of every theta-digit atom are never loaded (the TMA box has 4R rows):
  // zero them once, then make the generic-proxy stores visible to the tensor core's async proxy
  {
    const int live = 4 * D.R;
    for (int s = 0; s < CF::NBS; ++s)
      for (int a = 0; a < 4; ++a) {
        uint8_t* base = sB + s * CF::B_BYTES + a * CF::B_ATOM;
        for (int q = live * 128 + tid * 16; q < CF::B_ATOM; q += THREADS * 16) *(uint4*)(base + q) = make_uint4(0, 0, 0, 0);
      }
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
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
    }
    return;
  }
  K2Part<RMAX> P;
  k2_part_init(P, red);
  K2Ctx<RMAX> C;
  k2_load_ctx(D, C);

  if (wid == 0) {
    // ===== TMA producer of the X ring: stages in (pair, k-block, tile of the pair) order =====
    const uint64_t pol_x = D.x_policy == 2 ? policy_evict_last()
                           : (D.x_policy == 1 ? policy_evict_normal() : policy_evict_first());
    int stage = 0;
    uint32_t phase = 0;
    for (int lt = 0; lt < ntl; lt += 2) {
      const int nh = ntl - lt < 2 ? 1 : 2;
      for (int kb = 0; kb < kblocks; ++kb) {
        for (int h = 0; h < nh; ++h) {
          const int64_t t = blockIdx.x + (int64_t)(lt + h) * gridDim.x;
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            mbar_expect_tx(&full[stage], (uint32_t)A_BYTES);
            tma_load_2d(sA + stage * A_BYTES, &tmX, &full[stage], kb * PK, (int)(t * TILE_M), pol_x);
          }
          __syncwarp();
          if (++stage == CF::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (wid == 3) {
    // ===== TMA producer of the theta-digit ring: one stage per k-block of a tile pair =====
    const uint64_t pol_b = policy_evict_last();
    const uint32_t bbytes = (uint32_t)(4 * 4 * D.R * 128);
    int bs = 0;
    uint32_t bph = 0;
    for (int lt = 0; lt < ntl; lt += 2) {
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&bempty[bs], bph ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&bfull[bs], bbytes);
#pragma unroll
          for (int a = 0; a < 4; ++a)
            tma_load_2d(sB + bs * CF::B_BYTES + a * CF::B_ATOM, &tmB, &bfull[bs], kb * KS + a * 128, 0, pol_b);
        }
        __syncwarp();
        if (++bs == CF::NBS) {
          bs = 0;
          bph ^= 1;
        }
      }
    }
  } else if (wid == 1) {
    // ===== MMA issuer: the whole warp walks the pipeline, one elected lane issues =====
    constexpr uint32_t idesc = idesc_i8(NPAD);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t sB0 = smem_u32(sB);
    int ab = 0, bs = 0;
    uint32_t aphase = 0, bph = 0;
    for (int lt = 0; lt < ntl; lt += 2) {
      const int nh = ntl - lt < 2 ? 1 : 2;
      const uint32_t tph = (lt >> 1) & 1;
      for (int h = 0; h < nh; ++h) mbar_wait(&tempty[h], tph ^ 1);   // the epilogue sets have drained the previous pair
      tc_fence_after();
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&bfull[bs], bph);
        const uint64_t bdesc0 = umma_desc_sw128(sB0 + (uint32_t)(bs * CF::B_BYTES));
        for (int h = 0; h < nh; ++h) {
          mbar_wait(&afull[ab], aphase);
          tc_fence_after();
          const uint32_t a_tmem = tbase + (uint32_t)(A_COL0 + ab * A_COLS);
          const uint32_t d_tmem = tbase + (uint32_t)(h * CF::ACC_COLS);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < KS / 32; ++kk) {   // K = 32 samples per kind::i8 MMA; plane q = kk / 4
              // planes 0, 2 (x1) into scale group 0, planes 1, 3 (x4) into group 1; the first MMA of
              // each group of a tile overwrites (kk = 0, 4)
              umma_i8_tmem_a(d_tmem + (uint32_t)(((kk >> 2) & 1) * NPAD), a_tmem + (uint32_t)(8 * kk),
                             bdesc0 + (uint64_t)((kk >> 2) * (CF::B_ATOM >> 4) + 2 * (kk & 3)), idesc,
                             kb != 0 || (kk & 11) != 0);
            }
            umma_commit(&aempty[ab]);
            if (h == nh - 1) umma_commit(&bempty[bs]);
            if (kb == kblocks - 1) umma_commit(&tfull[h]);
          }
          __syncwarp();
          if (++ab == NAB) {
            ab = 0;
            aphase ^= 1;
          }
        }
        if (++bs == CF::NBS) {
          bs = 0;
          bph ^= 1;
        }
      }
    }
  } else if (wid >= 4 && wid < EPI0) {
    // ===== converters: TMEM lane quarter wid % 4 (thread = tile column), column half h of the
    // packed row when CW = 8.  They take the X stages in ring order, whatever tile each belongs to
    constexpr int CH = 8 / (CW / 4);          // 16-byte chunks per converter thread (8 or 4)
    constexpr int NW = 4 * CH;                // packed words per thread
    const int q4 = wid & 3;
    const int h = (wid - 4) >> 2;             // 0 (CW = 4) or 0/1 (CW = 8)
    const int c = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int stage = 0, ab = 0;
    uint32_t phase = 0, aphase = 0;
    const int64_t nst = (int64_t)ntl * kblocks;
    for (int64_t seq = 0; seq < nst; ++seq) {
      mbar_wait(&full[stage], phase);
      mbar_wait(&aempty[ab], aphase ^ 1);
      tc_fence_after();
      uint32_t w[NW], w4[NW];
      const uint8_t* row = sA + stage * A_BYTES + c * PK;
#pragma unroll
      for (int jj = 0; jj < CH; ++jj) {   // logical 16-byte chunk j sits at chunk j ^ (c & 7) (SWIZZLE_128B)
        const int j = h * CH + jj;
        const uint4 v = *(const uint4*)(row + ((j ^ (c & 7)) << 4));
        w[4 * jj] = v.x;
        w[4 * jj + 1] = v.y;
        w[4 * jj + 2] = v.z;
        w[4 * jj + 3] = v.w;
      }
      const uint32_t abase = tmem_base + lane_off + (uint32_t)(A_COL0 + ab * A_COLS + h * NW);
#pragma unroll
      for (int u = 0; u < NW; ++u) w4[u] = w[u] >> 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t o[NW];
#pragma unroll
        for (int u = 0; u < NW; ++u) o[u] = (q & 2 ? w4[u] : w[u]) & (0x03030303u << (2 * (q & 1)));
        if constexpr (NW == 32) tmem_st32(abase + (uint32_t)(32 * q), o);
        else tmem_st16(abase + (uint32_t)(32 * q), o);
      }
      // the packed words are in registers (the stores above consumed them): free the X stage
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[ab]);
      if (++stage == CF::STAGES) {
        stage = 0;
        phase ^= 1;
      }
      if (++ab == NAB) {
        ab = 0;
        aphase ^= 1;
      }
    }
  } else if (wid >= EPI0) {
    // ===== epilogue: TMEM lanes 32*(wid%4) .. +31 = columns of the tile; set `eset` takes the tiles
    // of accumulator buffer eset =====
    const int q = wid & 3;
    const int eset = (wid - EPI0) >> 2;
    for (int lt = eset; lt < ntl; lt += 2) {
      const int64_t t = blockIdx.x + (int64_t)lt * gridDim.x;
      epi_prefetch<RMAX>(D, C, (t + (int64_t)gridDim.x * 2) * TILE_M + q * 32 + lane);
      mbar_wait_park(&tfull[eset], (lt >> 1) & 1);
      tc_fence_after();
      int32_t dv[NPAD];
#pragma unroll
      for (int hh = 0; hh < NPAD / 16; ++hh) {   // scale group 0 (planes 0, 2) + scale group 1 (planes 1, 3) / 4, exactly
        uint32_t v[16], v1[16];
        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(eset * CF::ACC_COLS + hh * 16), v);
        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(eset * CF::ACC_COLS + NPAD + hh * 16), v1);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) dv[hh * 16 + u] = (int32_t)v[u] + ((int32_t)v1[u] >> 2);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[eset]);

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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
  k2_finish<RMAX>(D, C, P, red);
}

// ---------------------------------------------------------------- power-method back pass (a0')
// w_j = (X~_g^T u_g)_j for every model column j >= 1 of its block g (L259: the power / Lanczos
// products for eta_g), on the same TMA -> TMEM-unpack -> tcgen05 pipeline: the B operand of a tile
// is the int8 digit planes of u_g (28-bit fixed point per block, Bp rows 4g..4g+3, written by
// k_power_quant in the converter's K order).  Blocks hold >= 128 columns (checked by the host), so a
// 128-column tile touches blocks g0 and g0 + 1 at most and each stage loads their 8 digit rows.
struct PowBack {
  const long long* Tsum;   // [G] sum_i T_gi
  const double* gs;        // [G] delta_g / n
  const int* frozen;       // [G]
  double* w;               // [p + 1]
};

__global__ void __launch_bounds__(Cfg2<16, 1>::THREADS, 1)
    k2p_kernel(const Dev D, const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmBp,
               const PowBack PB) {
  using CF = Cfg2<16, 1>;
  constexpr int NPAD = 16;
  constexpr int CW = CF::CW;
  constexpr int EPI0 = 4 + CW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + (((1023 + 1) - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + CF::STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + CF::STAGES * CF::STAGE);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* afull = empty + CF::STAGES;
  constexpr int NAB = CF::NAB, A_COL0 = CF::A_COL0;
  uint64_t* aempty = afull + NAB;
  uint64_t* tfull = aempty + NAB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (D.p + TILE_M - 1) / TILE_M;
  const int kblocks = (int)((D.ld + PK - 1) / PK);
  if (wid == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmBp);
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < NAB; ++a) {
      mbar_init(&afull[a], CW);
      mbar_init(&aempty[a], 1);
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
  // digit rows 8..15 of every B stage are never loaded (the box has 8 rows): zero them once
  for (int s = 0; s < CF::STAGES; ++s)
    for (int a = 0; a < 4; ++a) {
      uint8_t* base = sB + s * CF::B_BYTES + a * NPAD * 128;
      for (int q = 8 * 128 + tid * 16; q < NPAD * 128; q += CF::THREADS * 16) *(uint4*)(base + q) = make_uint4(0, 0, 0, 0);
    }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (wid == 0) {
    const uint64_t pol_x = policy_evict_first(), pol_b = policy_evict_last();
    const uint32_t bytes = (uint32_t)(A_BYTES + 4 * 8 * 128);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int g0 = block_of_col(D, t * TILE_M + 1);
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&full[stage], bytes);
          tma_load_2d(sA + stage * A_BYTES, &tmX, &full[stage], kb * PK, (int)(t * TILE_M), pol_x);
#pragma unroll
          for (int a = 0; a < 4; ++a)
            tma_load_2d(sB + stage * CF::B_BYTES + a * CF::B_ATOM, &tmBp, &full[stage], kb * KS + a * 128, 4 * g0, pol_b);
        }
        __syncwarp();
        if (++stage == CF::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (wid == 1) {
    constexpr uint32_t idesc = idesc_u8s8(NPAD);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t sB0 = smem_u32(sB);
    int stage = 0, ab = 0;
    uint32_t phase = 0, aphase = 0;
    int lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int acc = lt & 1;
      mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tbase + (uint32_t)(acc * CF::ACC_COLS);
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&afull[ab], aphase);
        tc_fence_after();
        const uint32_t a_tmem = tbase + (uint32_t)(A_COL0 + ab * A_COLS);
        const uint64_t bdesc0 = umma_desc_sw128(sB0 + (uint32_t)(stage * CF::B_BYTES));
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < KS / 32; ++kk)
            umma_i8_tmem_a(d_tmem + (uint32_t)((kk >> 2) * NPAD), a_tmem + (uint32_t)(8 * kk),
                           bdesc0 + (uint64_t)((kk >> 2) * (CF::B_ATOM >> 4) + 2 * (kk & 3)), idesc,
                           (kb != 0 || (kk & 3) != 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          umma_commit(&aempty[ab]);
        }
        __syncwarp();
        if (++stage == CF::STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++ab == NAB) {
          ab = 0;
          aphase ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (wid >= 4 && wid < EPI0) {
    // converters: identical to k2_tc2_kernel<16, 1> (codes left in place, one plane per accumulator)
    constexpr int CH = 8 / (CW / 4);
    constexpr int NW = 4 * CH;
    static_assert(NW == 16, "eight converter warps");
    const int q4 = wid & 3;
    const int h = (wid - 4) >> 2;
    const int c = q4 * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    int stage = 0, ab = 0;
    uint32_t phase = 0, aphase = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        mbar_wait(&aempty[ab], aphase ^ 1);
        tc_fence_after();
        uint32_t w[NW];
        const uint8_t* row = sA + stage * A_BYTES + c * PK;
#pragma unroll
        for (int jj = 0; jj < CH; ++jj) {
          const int j = h * CH + jj;
          const uint4 v = *(const uint4*)(row + ((j ^ (c & 7)) << 4));
          w[4 * jj] = v.x;
          w[4 * jj + 1] = v.y;
          w[4 * jj + 2] = v.z;
          w[4 * jj + 3] = v.w;
        }
        const uint32_t abase = tmem_base + lane_off + (uint32_t)(A_COL0 + ab * A_COLS + h * NW);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t o[NW];
#pragma unroll
          for (int u = 0; u < NW; ++u) o[u] = w[u] & (0x03030303u << (2 * q));
          tmem_st16(abase + (uint32_t)(32 * q), o);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[ab]);
        if (++stage == CF::STAGES) {
          stage = 0;
          phase ^= 1;
        }
        if (++ab == NAB) {
          ab = 0;
          aphase ^= 1;
        }
      }
    }
  } else if (wid >= EPI0) {
    const int q = wid & 3;
    int lt = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int acc = lt & 1;
      mbar_wait_park(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      int32_t dv[NPAD];
#pragma unroll
      for (int u = 0; u < NPAD; ++u) dv[u] = 0;
#pragma unroll
      for (int pq = 0; pq < 4; ++pq) {
        uint32_t v[16];
        tmem_ld16(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * CF::ACC_COLS + pq * NPAD), v);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 16; ++u) dv[u] += ((int32_t)v[u]) >> (2 * pq);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      const int64_t c = t * TILE_M + q * 32 + lane;
      if (c < D.p) {
        const int g0 = block_of_col(D, t * TILE_M + 1), g = block_of_col(D, c + 1);
        if (!PB.frozen[g]) {
          const bool sl = g != g0;   // second block of the tile: digit rows 4..7 (selects, not an indexed load)
          const int32_t Dk[4] = {sl ? dv[4] : dv[0], sl ? dv[5] : dv[1], sl ? dv[6] : dv[2], sl ? dv[7] : dv[3]};
          PB.w[c + 1] = g_from_digits(D.n, D.colsum[c], PB.Tsum[g], PB.gs[g], D.inv_sd[c], Dk);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

template <int NPAD, int RM>
void launch_np(const Dev& D, const void* tmX, const void* tmB, int grid, cudaStream_t st) {
  if constexpr (NPAD > 16 && K2TC2_PAIR)
    launch_pdl(k2_tc2_pair_kernel<NPAD, RM>, dim3(grid), dim3(Cfg2P<NPAD, RM>::THREADS), Cfg2P<NPAD, RM>::SMEM, st, D,
               *(const CUtensorMap*)tmX, *(const CUtensorMap*)tmB);
  else
    launch_pdl(k2_tc2_kernel<NPAD, RM>, dim3(grid), dim3(Cfg2<NPAD, RM>::THREADS), Cfg2<NPAD, RM>::SMEM, st, D,
               *(const CUtensorMap*)tmX, *(const CUtensorMap*)tmB);
}

template <int NPAD, int RM>
cudaError_t init_np() {
  if constexpr (NPAD > 16 && K2TC2_PAIR)
    return cudaFuncSetAttribute(k2_tc2_pair_kernel<NPAD, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                Cfg2P<NPAD, RM>::SMEM);
  else
    return cudaFuncSetAttribute(k2_tc2_kernel<NPAD, RM>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2<NPAD, RM>::SMEM);
}

}  // namespace

cudaError_t k2_tc2_init() {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k2p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2<16, 1>::SMEM)) !=
      cudaSuccess)
    return e;
  if ((e = init_np<16, 1>()) != cudaSuccess) return e;
  if ((e = init_np<16, 4>()) != cudaSuccess) return e;
  if ((e = init_np<32, 8>()) != cudaSuccess) return e;
  if ((e = init_np<48, 9>()) != cudaSuccess) return e;
  if ((e = init_np<48, 12>()) != cudaSuccess) return e;
  return init_np<64, 16>();
}

void launch_k2_tc2(const Dev& D, const void* tmX, const void* tmB, int grid, cudaStream_t st) {
  if (D.R == 1) launch_np<16, 1>(D, tmX, tmB, grid, st);
  else if (D.npad == 16) launch_np<16, 4>(D, tmX, tmB, grid, st);
  else if (D.npad == 32) launch_np<32, 8>(D, tmX, tmB, grid, st);
  else if (D.npad == 48 && D.R <= 9) launch_np<48, 9>(D, tmX, tmB, grid, st);   // C5: nine quantile levels
  else if (D.npad == 48) launch_np<48, 12>(D, tmX, tmB, grid, st);
  else launch_np<64, 16>(D, tmX, tmB, grid, st);
}

void launch_power_back_tc2(const Dev& D, const void* tmX, const void* tmBp, const long long* Tsum, const double* gs,
                           const int* frozen, double* w, int grid, cudaStream_t st) {
  const PowBack PB{Tsum, gs, frozen, w};
  k2p_kernel<<<grid, Cfg2<16, 1>::THREADS, Cfg2<16, 1>::SMEM, st>>>(D, *(const CUtensorMap*)tmX, *(const CUtensorMap*)tmBp,
                                                                   PB);
}
