// k1_tcp.cu — a4 on the tensor cores for 2-bit packed genotypes: s^{k+1} = X~ beta^{k+1} over
// the support of beta^{k+1} ("computation of X beta ... divided into G
// simultaneous sub-tasks ... followed by computing their sum"), exact integer arithmetic.
//
//   S_{i,r} = sum_{j in S} x_ij C_{j,r} = sum_k 256^k D_{i,(r,k)},   D = X_S · Dig,
// C_{j,r} = round(2^E beta_{j,r} / s_j) in six balanced base-256 digits (k1_fwd.cu)
//
// GEMM D[M = rows][N = digit columns] = A[rows][K = support] · B, A MN-major (X is SNP-major:
// each column's rows are contiguous).  The CUDA-core kernel k1_bulk spends ~4 instructions per
// 2-bit code (extract, two multiply-adds); here the codes are unpacked on chip into the
// canonical MN-major SWIZZLE_128B A tile and the multiply-adds run on the tensor cores.
//
//   producer warp: balanced base-256 digits of C (beta/s and colsum arrive in bulk-copied
//       metadata blocks, two blocks ahead) into a ring of K-major B tiles; the colsum·C term;
//   converter warps (4 support entries of each 32-entry chunk per warp): every lane fetches its
//       own 16-byte pieces of those columns' packed slab segments with cp.async (LDGSTS: per-lane
//       addresses, no per-copy issue cost -- one cp.async.bulk per column capped the copy rate
//       at ~1 per 95 cycles per SM), SD-1 chunks ahead into a private ring; then each 32-bit
//       word w (16 rows) becomes the 16-byte chunk {w & 0x03030303, w & 0x0C0C0C0C,
//       w & 0x30303030, w & 0xC0C0C0C0}: the codes stay in place, so byte 4q+b of chunk c holds
//       row 16c+4b+q times 4^q (unsigned A, one LOP per 4 codes), stored into row k of the row
//       tile at chunk position c ^ (k & 7) -- the 128-byte swizzle (a per-lane rotation of the
//       four chunks keeps the 8 lanes of each store phase on distinct bank groups);
//   MMA warp: one tcgen05.mma.kind::i8 (A, B from shared memory) per row tile and 32 entries;
//   epilogue (converter warps): TMEM lane m of a row tile is row 16(m>>4) + 4(m&3) + ((m>>2)&3)
//       scaled by 4^((m>>2)&3); each digit sum is shifted back exactly (a multiple of 4^q), then
//       S = sum_k 256^k D_k in int64 and one 64-bit integer atomic per row and RHS, exactly the
//       fixed-point sum k1_bulk forms (bit-identical results);
//   fused finalize (cur = 0): after its last item every CTA arrives at a grid barrier (the grid
//       is one CTA per SM and fully co-resident: the next kernel is only launched once every CTA
//       of this one has started, and nothing here waits on it); then the 256-row records of the
//       n-vector step (fin_common.cuh: E15, residual, E12, theta digits) are spread over the CTAs,
//       and the last CTA to finish them (ticket) reduces the records in fixed order and ends the
//       iteration.  One launch instead of two.  (A first version let the last item of each row
//       slab finalize that slab's 2048 rows: 8 records in one CTA put ~18 us on the tail.)
#include <cuda.h>
__device__ __forceinline__ unsigned __smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

#include "fin_common.cuh"

#ifndef K1P_RTMAX
#define K1P_RTMAX 16   // row tiles per slab cap (measurement knob)
#endif
#ifndef K1P_SMEM_KB
#define K1P_SMEM_KB 220
#endif
#ifndef K1P_NAB2
#define K1P_NAB2 2     // A tile buffers of the 2-bit variant (measurement knob)
#endif
#ifndef K1P_CTAS
#define K1P_CTAS 1     // CTAs per SM the launch grid assumes
#endif
#ifndef K1P_L2PF
#define K1P_L2PF 0     // L2 prefetch of the next X~^T theta pass's first tiles (measurement knob)
#endif
#ifndef K1P_TIMING
#define K1P_TIMING 0   // measurement build: per-CTA globaltimer stamps of iteration K1P_TIMING (fsqr_debug_stamps)
#endif
#ifndef K1P_DBG
#define K1P_DBG 0   // measurement variants: bit 0 skips the MMAs, bit 1 the unpack, bit 2 the loads, bit 3 the atomics
#endif

namespace {

constexpr int KC = 32;          // support entries per chunk (one kind::i8 MMA K step)
constexpr int CW = 8;           // converter / epilogue warps (4..11), 4 entries of each chunk per warp
constexpr int THREADS = 32 * (4 + CW);
constexpr int ATILE = 128 * KC; // one row tile x one chunk: 4 KB (four 1 KB swizzle atoms)
constexpr int SB = 4;           // B tile ring

template <int RMAX, int ST>
struct K1P {
  static constexpr int NDIG = 6 * RMAX;
  static constexpr int N = NDIG <= 16 ? 16 : (NDIG <= 32 ? 32 : (NDIG <= 48 ? 48 : 96));
  static constexpr int RT0 = N <= 32 ? 16 : (N <= 48 ? 8 : 4);  // row tiles per slab (RT * N <= 512)
  static constexpr int RT = RT0 < K1P_RTMAX ? RT0 : K1P_RTMAX;
  static constexpr int SR = 128 * RT;                          // rows per slab
  static constexpr int SEGB = ST == 1 ? SR : SR / 4;           // bytes per column segment
  static constexpr int UPL = ST == 1 ? RT : RT / 4;            // 16-byte units per lane per chunk
  static constexpr int DSTAGE = ST == 1 ? 0 : KC * SEGB;       // one chunk of packed segments (2-bit)
  static constexpr int BTILE = N * KC;
  static constexpr int NAB = ST == 1 ? 3 : K1P_NAB2;           // A tile buffers (u8: the copy ring)
  static constexpr int ABUF = RT * ATILE;
  static constexpr int MB = RMAX <= 4 ? 256 : 128;             // metadata entries per block
  static constexpr int META = 2 * MB * (4 + 8 * RMAX);         // two blocks: colsum, beta/s
  static constexpr int SD0 = ST == 1 ? 0 : (K1P_SMEM_KB * 1024 - NAB * ABUF - SB * BTILE - META) / (DSTAGE ? DSTAGE : 1);
  static constexpr int SD = ST == 1 ? 0 : (SD0 < 2 ? 2 : (SD0 > 6 ? 6 : SD0));   // 2-bit data ring depth (chunks)
  static constexpr int TCOLS = RT * N <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 + NAB * ABUF + SD * DSTAGE + SB * BTILE + META + 1024;
  static_assert(RT * N <= 512, "TMEM budget");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// (the .L2::cache_hint form faulted with "illegal instruction" on the B200: plain cp.async.cg)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ int btile_off(int nrow, int k) {
  return (nrow >> 3) * 256 + (nrow & 7) * 16 + (k >> 4) * 128 + (k & 15);
}
// K-major, no swizzle (B: digits): core matrices of 8 digit rows x 16 entries
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
// kind::i8, D s32, A u8 MN-major, B s8 K-major, M = 128
__host__ __device__ constexpr uint32_t idesc_u8mn_s8(int N) {
  return (2u << 4) | (1u << 10) | (1u << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}


// Fused finalize, record part (warps 4..11 of every CTA): records (r, b) of the active RHS in
// contiguous shares per CTA, batches of <= NB records of one RHS.  The first batch's state rows and
// constants are loaded BEFORE the grid barrier (every CTA's forward sums complete); after it only
// the forward accumulators and the colsum term are on the critical path.  Called by all threads.
template <int NB>
__device__ __forceinline__ void fused_records(const Dev& D, long long kit, int R, int nblk, int q0, int q1, int t,
                                              int wid, int tid, double* smd, unsigned nct) {
  FinRows<NB> pre;
  FinRHS pc;
  if (wid >= 4 && q0 < q1) {
    const int r = q0 / nblk, b = q0 % nblk, nb = min(min(NB, nblk - b), q1 - q0);
    if (D.status[r] == ST_ACTIVE) {
      fin_load<NB>(D, r, b, nb, t, pre);
      pc = fin_rhs(D, r, kit, 0);
    }
  }
  // barrier of the nct product CTAs: the grid is one CTA per SM and fully co-resident.  As in a
  // cooperative grid sync, only thread 0 fences: bar.sync orders the CTA's forward-sum atomics before
  // its gpu-scope release (cumulativity)
  __syncthreads();
  if (tid == 0) {
    fence_acq_rel_gpu();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(D.k1bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(D.k1bar) : "memory");
    } while (v < nct);
  }
  __syncthreads();
  if (wid < 4) return;
#if K1P_TIMING
  const long long rc0 = clock64();
#endif
  for (int q = q0; q < q1;) {
    const int r = q / nblk, b = q % nblk, nb = min(min(NB, nblk - b), q1 - q);
    if (D.status[r] == ST_ACTIVE) {
      if (q == q0) {
        pc.mt = __ldcg(D.mterm + r);
        fin_records<NB>(D, r, b, nb, pc, t, 1, smd, pre);
      } else {
        FinRows<NB> w;
        fin_load<NB>(D, r, b, nb, t, w);
        const FinRHS c = fin_rhs(D, r, kit, __ldcg(D.mterm + r));
        fin_records<NB>(D, r, b, nb, c, t, 1, smd, w);
      }
    }
    q += nb;
  }
#if K1P_TIMING
  grp_bar(1);
  if (t == 0 && kit == K1P_TIMING) D.tstamp[8 * 148 + 200 + blockIdx.x] = (unsigned long long)(clock64() - rc0);
#endif
}

template <int RMAX, int ST>
__global__ void __launch_bounds__(THREADS, K1P_CTAS) k1_tcp_kernel(const Dev D, int cur) {
  using T = K1P<RMAX, ST>;
  constexpr int RT = T::RT, SR = T::SR, SEGB = T::SEGB, N = T::N, SD = T::SD, NAB = T::NAB, MB = T::MB;
  constexpr int UPL = T::UPL;
  extern __shared__ uint8_t k1p_raw[];
  uint8_t* sm = k1p_raw + (((1023 + 1) - (smem_u32(k1p_raw) & 1023)) & 1023);
  uint8_t* sA = sm;                                      // [NAB][RT][ATILE], 1 KB aligned
  uint8_t* sD = sA + NAB * T::ABUF;                      // [SD][KC][SEGB] packed segments
  uint8_t* sB = sD + SD * T::DSTAGE;                     // [SB][BTILE]
  double* msc = (double*)(sB + SB * T::BTILE);           // [2][MB * RMAX] (R per entry used)
  int32_t* mcs = (int32_t*)(msc + 2 * MB * RMAX);        // [2][MB]
  uint64_t* bfull = (uint64_t*)(mcs + 2 * MB);
  uint64_t* bempty = bfull + SB;
  uint64_t* afull = bempty + SB;
  uint64_t* aempty = afull + NAB;
  uint64_t* tfull = aempty + NAB;
  uint64_t* tempty = tfull + 1;
  uint64_t* mfull = tempty + 1;
  uint32_t* tmem_slot = (uint32_t*)(mfull + 2);

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (wid == 0 && lane == 0) {
    for (int s = 0; s < SB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < NAB; ++a) {
      mbar_init(&afull[a], CW);
      mbar_init(&aempty[a], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, CW);
    mbar_init(&mfull[0], 1);
    mbar_init(&mfull[1], 1);
    fence_mbar_init();
  }
  if (wid == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(T::TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_launch_dependents();
  pdl_wait();
#if K1P_L2PF
  // 2-bit, iteration mode: pull the first column tile the next X~^T theta pass will stream on this
  // CTA's index (128 columns, contiguous) into L2 while this kernel runs -- HBM is nearly idle here
  if (ST == 2 && !cur && threadIdx.x == 0 && D.k1_pw == 0) {
    const int64_t c0 = (int64_t)blockIdx.x * 128;
    if (c0 < D.p) {
      const int64_t bytes = (min((int64_t)D.p, c0 + 128) - c0) * D.ld;
      const uint8_t* base = D.X8 + c0 * D.ld;
      for (int64_t o = 0; o < bytes; o += 32768) {
        const uint32_t sz = (uint32_t)min((int64_t)32768, bytes - o);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(sz) : "memory");
      }
    }
  }
#endif
#if K1P_TIMING
  unsigned long long ts0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts0));
#endif

  const long long kit = *D.iter;
  const int par = (int)((kit + (cur ? 0 : 1)) & 1);
  const int cnt = D.sup_cnt[par];
  const bool stopped = *D.stop != 0;
  const bool skip = stopped || cnt == 0 || (K1P_DBG & 16);
  const bool fused = !cur;   // iteration mode: this kernel also runs the finalize (fin_common.cuh)
  // fused: the last CTA is the REDUCER (no product items, no records): it waits for every product
  // CTA's records and reduces them, its code already warm; the other nct CTAs do the product
  const int nct = fused && gridDim.x > 1 ? (int)gridDim.x - 1 : (int)gridDim.x;
  const bool reducer = (int)blockIdx.x >= nct;
  const int R = D.R;
  const int nslab = (D.n + SR - 1) / SR;
  // entries per work item: about one item per CTA, at most 2^16 (int32 digit sums stay exact:
  // |code 4^q| <= 192, |digit| <= 128, 192 * 128 * 2^16 < 2^31)
  const int per = max(1, nct / nslab);
  int64_t es = ((int64_t)max(cnt, 1) + per - 1) / per;
  // (u8 codes up to 255: 255 * 128 * 2^15 < 2^31, so at most 2^15 entries per item there)
  es = min((int64_t)min(D.k1_esmax, ST == 1 ? 32768 : 65536), ((es + KC - 1) / KC) * KC);
  // power mode: an item must not span more than two blocks (the host guarantees >= 128 columns per block)
  const bool pw = RMAX == 2 && D.k1_pw > 0;
  if (pw) es = min(es, (int64_t)(D.gq - 1) / KC * KC);
  const int64_t nsl = ((int64_t)cnt + es - 1) / es;
  const int64_t nwork = (skip || reducer) ? 0 : nsl * nslab;

  if (wid == 0) {
    // ===================== producer: lane = support entry of the chunk
    const int32_t* scs = D.sup_cs[par];
    const double* sc = D.sup_c[par];
    double scale[RMAX];
    bool act[RMAX];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      act[r] = pw || (r < R && (cur || D.status[r] == ST_ACTIVE));
      const double cm = (pw || r < R) ? __longlong_as_double((long long)D.cmax[pw ? par : par * R + r]) : 0.0;
      scale[r] = ldexp(1.0, fwd_exponent(cm, pw ? (long long)D.k1_pw : (long long)cnt, D.n));
    }
    const uint64_t pol_m = policy_evict_normal();
    int bst = 0;
    uint32_t bph = 0;
    long long mbc = 0;   // metadata blocks used so far (buffer mbc & 1, parity (mbc >> 1) & 1)
    for (int64_t w = blockIdx.x; w < nwork; w += nct) {
      const int slab = (int)(w % nslab);
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      const int64_t nb = (e1 - e0 + MB - 1) / MB;
      auto issue_meta = [&](int64_t b) {
        const int buf = (int)((mbc + b) & 1);
        const int64_t bs = e0 + b * MB;
        const uint32_t ne4 = (uint32_t)((min((int64_t)MB, e1 - bs) + 3) & ~3);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mfull[buf], ne4 * 4u + ne4 * 8u * (uint32_t)R);
        bulk_g2s(mcs + buf * MB, scs + bs, ne4 * 4u, &mfull[buf], pol_m);
        bulk_g2s(msc + buf * MB * RMAX, sc + bs * R, ne4 * 8u * (uint32_t)R, &mfull[buf], pol_m);
      };
      if (lane == 0) {
        issue_meta(0);
        if (nb > 1) issue_meta(1);
      }
      long long mt[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) mt[r] = 0;
      const int g0 = pw ? block_of_col(D, e0 + 1) : 0;   // power mode: the item's first block (entry e = column e)
      for (int64_t b = 0; b < nb; ++b) {
        const int buf = (int)((mbc + b) & 1);
        mbar_wait(&mfull[buf], (uint32_t)(((mbc + b) >> 1) & 1));
        const int64_t bs = e0 + b * MB, be = min(e1, bs + MB);
        for (int64_t g0e = bs; g0e < be; g0e += KC) {
          const bool live = g0e + lane < be;
          const int o = (int)(g0e - bs) + lane;
          const long long cs = (live && slab == 0) ? (long long)mcs[buf * MB + o] : 0;
          long long C[RMAX];
          if (pw) {   // one coefficient per column, into the slot of its block
            const long long cv = live ? __double2ll_rn(msc[buf * MB * RMAX + o] * scale[0]) : 0;
            const int sl = live ? block_of_col(D, g0e + lane + 1) - g0 : 0;
#pragma unroll
            for (int r = 0; r < RMAX; ++r) {
              C[r] = sl == r ? cv : 0;
              mt[r] += cs * C[r];
            }
          } else {
#pragma unroll
            for (int r = 0; r < RMAX; ++r) {
              C[r] = (live && act[r]) ? __double2ll_rn(msc[buf * MB * RMAX + o * R + r] * scale[r]) : 0;
              mt[r] += cs * C[r];
            }
          }
          mbar_wait(&bempty[bst], bph ^ 1);
          uint8_t* bt = sB + bst * T::BTILE;
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
          if (lane == 0) mbar_arrive(&bfull[bst]);
          if (++bst == SB) {
            bst = 0;
            bph ^= 1;
          }
        }
        __syncwarp();
        if (lane == 0 && b + 2 < nb) issue_meta(b + 2);   // into the buffer just consumed
      }
      mbc += nb;
      if (slab == 0) {
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          long long v = mt[r];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0 && v != 0) atomicAdd((unsigned long long*)&D.mterm[pw ? g0 + r : r], (unsigned long long)v);
        }
      }
    }
  } else if (wid == 1) {
    // ===================== MMA issuer (elected lane)
    constexpr uint32_t idesc = idesc_u8mn_s8(N);
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t sA0 = smem_u32(sA), sB0 = smem_u32(sB);
    int bst = 0, ab = 0;
    uint32_t bph = 0, aphase = 0, tph = 0;
    for (int64_t w = blockIdx.x; w < nwork; w += nct) {
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      mbar_wait(tempty, tph ^ 1);
      tc_fence_after();
      bool first = true;
      for (int64_t g0 = e0; g0 < e1; g0 += KC) {
        mbar_wait(&bfull[bst], bph);
        mbar_wait(&afull[ab], aphase);
        tc_fence_after();
        const uint64_t bdesc = desc_k_noswz(sB0 + (uint32_t)(bst * T::BTILE));
        if (elect_one()) {
#pragma unroll
          for (int t = 0; t < RT; ++t)
            if (!(K1P_DBG & 1))
              umma_i8(tbase + (uint32_t)(t * N), desc_mn_sw128(sA0 + (uint32_t)((ab * RT + t) * ATILE)), bdesc, idesc,
                      first ? 0u : 1u);
          umma_commit(&bempty[bst]);
          umma_commit(&aempty[ab]);
        }
        __syncwarp();
        first = false;
        if (++bst == SB) {
          bst = 0;
          bph ^= 1;
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
    // ===================== converters (entries 4cw .. 4cw+3 of every chunk) + epilogue
    const int cw = wid - 4;
    const int q4 = wid & 3, hsel = cw >> 2;   // epilogue: TMEM lane quarter, row-tile subset
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t sA0 = smem_u32(sA), sD0 = smem_u32(sD);
    const int32_t* sidx = D.sup_idx[par];
    int ab = 0;
    uint32_t aphase = 0, tph = 0;
    long long ga = 0;   // u8: chunks handed to the MMA so far (A-buffer ring position)
    for (int64_t w = blockIdx.x; w < nwork; w += nct) {
      const int slab = (int)(w % nslab);
      const int64_t e0 = (w / nslab) * es, e1 = min((int64_t)cnt, e0 + es);
      const int64_t nch = (e1 - e0 + KC - 1) / KC;
      const int64_t boff = (int64_t)slab * SEGB;
      // bytes of this slab's segment that hold samples (2-bit: up to the 32-byte sector holding the
      // last one; the column padding beyond it is never fetched)
      const int64_t dw = ST == 1 ? D.ld : min(D.ld, (int64_t)((D.n + 3) / 4 + 31) / 32 * 32);
      const int bytes = (int)min((int64_t)SEGB, dw - boff);
      const uint8_t* xs = D.X8 + boff;
      // my columns of chunk c: entries e0 + 32c + 4cw + kk, kk < 4 (-1 past the end).  Lane l holds
      // them for chunk 32 b + l of batch b (bi: the batch of the chunk being issued, bn: the next),
      // so the column indices are loaded 32 chunks ahead and read with one shuffle each.
      auto load_batch = [&](int64_t b, int (&ix)[4]) {
        const int64_t c = 32 * b + lane;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const int64_t e = e0 + KC * c + 4 * cw + kk;
          ix[kk] = (c < nch && e < e1) ? sidx[e] : -1;
        }
      };
      int bi[4], bn[4];
      load_batch(0, bi);
      load_batch(1, bn);
      auto get_idx = [&](int64_t c, int (&ix)[4]) {
        if (c > 0 && (c & 31) == 0) {   // entering batch c / 32: rotate and fetch the one after
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) bi[kk] = bn[kk];
          load_batch((c >> 5) + 1, bn);
        }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) ix[kk] = __shfl_sync(0xffffffffu, bi[kk], (int)(c & 31));
      };
      if constexpr (ST == 1) {
        // u8: the codes are already bytes, so each lane's cp.async lands straight in the swizzled
        // A tile (16 samples = one 16-byte chunk: row k, chunk c at c ^ (k & 7)); the A buffers
        // are the copy ring, NAB - 1 chunks ahead.  Chunk c of the item is global chunk ga + c
        // (buffer (ga + c) % NAB), the order the MMA warp consumes them in.
        auto issue_u8 = [&](int64_t c, const int (&ix)[4]) {
          const long long G = ga + c;
          const int buf = (int)(G % NAB);
          mbar_wait(&aempty[buf], (uint32_t)(((G / NAB) & 1) ^ 1));   // MMA of chunk G - NAB done
          const uint32_t abuf = sA0 + (uint32_t)(buf * T::ABUF);
#pragma unroll
          for (int i = 0; i < UPL; ++i) {
            const int u = i * 32 + lane, kk = u / (SEGB / 16), off = 16 * (u % (SEGB / 16));
            const int k = 4 * cw + kk, t = off >> 7, c16 = (off >> 4) & 7;
            int col = ix[0];
#pragma unroll
            for (int q = 1; q < 4; ++q)
              if (kk == q) col = ix[q];
            if (!(K1P_DBG & 4) && col >= 0 && off < bytes)
              cp_async16(abuf + (uint32_t)(t * ATILE + k * 128 + ((c16 ^ (k & 7)) << 4)),
                         xs + (int64_t)col * D.ld + off);
          }
          cp_async_commit();
        };
#pragma unroll 1
        for (int c = 0; c < NAB - 1; ++c) {
          if (c < nch) {
            int ix[4];
            get_idx(c, ix);
            issue_u8(c, ix);
          } else {
            cp_async_commit();
          }
        }
        for (int64_t c = 0; c < nch; ++c) {
          if (c + NAB - 1 < nch) {
            int ix[4];
            get_idx(c + NAB - 1, ix);
            issue_u8(c + NAB - 1, ix);
          } else {
            cp_async_commit();
          }
          cp_async_wait<NAB - 1>();   // this lane's pieces of chunk c are in the tile
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&afull[(int)((ga + c) % NAB)]);
        }
        ga += nch;
      } else {
        auto issue = [&](int64_t c, const int (&ix)[4]) {
          const uint32_t slot = sD0 + (uint32_t)((c % SD) * T::DSTAGE + 4 * cw * SEGB);
  #pragma unroll
          for (int i = 0; i < UPL; ++i) {
            const int u = i * 32 + lane, kk = u / (2 * RT), off = 16 * (u % (2 * RT));
            int col = ix[0];   // ix[kk] without a local-memory array for lane-dependent kk
  #pragma unroll
            for (int q = 1; q < 4; ++q)
              if (kk == q) col = ix[q];
            if (!(K1P_DBG & 4) && col >= 0 && off < bytes)
              cp_async16(slot + (uint32_t)(kk * SEGB + off), xs + (int64_t)col * D.ld + off);
          }
          cp_async_commit();
        };
  #pragma unroll 1
        for (int c = 0; c < SD - 1; ++c) {
          int ix[4];
          get_idx(c, ix);
          issue(c, ix);
        }
        for (int64_t c = 0; c < nch; ++c) {
          {
            int ix[4];
            get_idx(c + SD - 1, ix);
            issue(c + SD - 1, ix);
          }
          cp_async_wait<SD - 1>();   // this lane's pieces of chunk c have landed
          mbar_wait(&aempty[ab], aphase ^ 1);
          const uint32_t src = sD0 + (uint32_t)((c % SD) * T::DSTAGE + 4 * cw * SEGB);
          const uint32_t abuf = sA0 + (uint32_t)(ab * T::ABUF);
  #pragma unroll
          for (int i = 0; i < ((K1P_DBG & 2) ? 0 : UPL); ++i) {
            const int u = i * 32 + lane, kk = u / (2 * RT), off = 16 * (u % (2 * RT));
            const int k = 4 * cw + kk, t = off >> 5, h = (off >> 4) & 1;
            uint32_t a, b, cc, d;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(a), "=r"(b), "=r"(cc), "=r"(d)
                         : "r"(src + (uint32_t)(kk * SEGB + off)));
            // rotate by t & 3: step jj stores word (jj + t) & 3
            if (t & 1) {
              const uint32_t x = a;
              a = b, b = cc, cc = d, d = x;
            }
            if (t & 2) {
              uint32_t x = a;
              a = cc, cc = x;
              x = b, b = d, d = x;
            }
            const uint32_t wv[4] = {a, b, cc, d};
            const uint32_t row = abuf + (uint32_t)(t * ATILE + k * 128);
  #pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const uint32_t ch = (uint32_t)(4 * h + ((jj + t) & 3));
              const uint32_t x = wv[jj];
              sts128(row + ((ch ^ (uint32_t)(k & 7)) << 4), x & 0x03030303u, x & 0x0C0C0C0Cu, x & 0x30303030u,
                     x & 0xC0C0C0C0u);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&afull[ab]);
          if (++ab == NAB) {
            ab = 0;
            aphase ^= 1;
          }
        }
      }
      cp_async_wait<0>();
      // ---- epilogue of the work item
      mbar_wait(tfull, tph);
      tph ^= 1;
      tc_fence_after();
      const int gb = pw ? block_of_col(D, e0 + 1) : 0;                // power mode: accumulator of slot r is block gb + r
      const int rlim = pw ? min(RMAX, D.G - gb) : R;
      const int m = q4 * 32 + lane;                                  // TMEM lane of the row tile
      const int qs = ST == 1 ? 0 : (m >> 2) & 3;                     // 2-bit plane: scale 4^qs
      const int rin = ST == 1 ? m : ((m & ~15) | ((m & 3) << 2) | qs);   // row within the tile
#pragma unroll 1
      for (int t = hsel; t < RT; t += CW / 4) {
        const int row = slab * SR + t * 128 + rin;
        int32_t dv[N];
#pragma unroll
        for (int hh = 0; hh < N / 16; ++hh) {
          uint32_t v[16];
          tmem_ld16(tmem_base + lane_off + (uint32_t)(t * N + hh * 16), v);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 16; ++u) dv[hh * 16 + u] = (int32_t)v[u] >> (2 * qs);   // exact
        }
#pragma unroll
        for (int r = 0; r < RMAX; ++r) {
          long long S = 0;
#pragma unroll
          for (int q = 5; q >= 0; --q) S = S * 256 + (long long)dv[6 * r + q];
          if (!(K1P_DBG & 8) && r < rlim && row < D.n && S != 0)
            atomicAdd((unsigned long long*)&D.sacc[(int64_t)(gb + r) * D.n + row], (unsigned long long)S);
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(T::TCOLS) : "memory");
  }
  if (!fused || stopped) return;
#if K1P_TIMING
  unsigned long long ts1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts1));
#endif

  // ===================== fused finalize (fused_records; the A buffers are free scratch now)
  double* smd = (double*)sA;
  long long* smll = (long long*)(smd + 4 * 8 * 9);
  const int nblk = (D.n + FG - 1) / FG;
  const int t = tid - 128;
  if (!reducer) {
    const int tot = R * nblk, rper = (tot + nct - 1) / nct;
    const int q0 = min(tot, (int)blockIdx.x * rper), q1 = min(tot, q0 + rper);
    if (rper == 1) fused_records<1>(D, kit, R, nblk, q0, q1, t, wid, tid, smd, (unsigned)nct);
    else fused_records<4>(D, kit, R, nblk, q0, q1, t, wid, tid, smd, (unsigned)nct);
    // publish this CTA's records to the reducer
#if K1P_TIMING
    __syncthreads();
    unsigned long long ts2b;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts2b));
#endif
    __syncthreads();
    if (tid == 0) {
      fence_acq_rel_gpu();
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(D.fticket) : "memory");
    }
#if K1P_TIMING
    unsigned long long ts3;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts3));
    if (tid == 0 && kit == K1P_TIMING) {
      unsigned long long* st = D.tstamp + 8 * blockIdx.x;
      st[0] = ts0; st[1] = ts1; st[2] = ts1; st[3] = ts2b; st[4] = ts3; st[5] = ts3;
      st[6] = (unsigned long long)__smid();
      st[7] = (unsigned long long)((nwork - blockIdx.x + nct - 1) / nct);
    }
#endif
    return;
  }
  if (wid < 4) return;
  // reducer: a dry run of the reduction (no stores) while the records are being written, so that
  // the committed pass runs from a warm instruction cache; then wait for all nct tickets
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      if (t == 0) {
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(D.fticket) : "memory");
        } while (v < (unsigned)nct);
      }
      grp_bar(1);
      fence_acq_rel_gpu();
#if K1P_TIMING
      if (t == 0 && kit == K1P_TIMING) {
        unsigned long long tq0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tq0));
        D.tstamp[8 * 148 + 70] = tq0;
      }
#endif
    }
    fin_reduce_all(D, nblk, kit, t, 1, smll, pass == 1);
  }
  if (t < R) D.mterm[t] = 0;
  fin_iteration_tail(D, kit, t);
  if (t == 0) {
    *D.fticket = 0u;
    *D.k1bar = 0u;   // every product CTA has left the barrier (each published its records after it)
  }
#if K1P_TIMING
  {
    unsigned long long ts4;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts4));
    if (t == 0 && kit == K1P_TIMING) {
      D.tstamp[8 * 148 + 40] = ts4;
      unsigned long long* st = D.tstamp + 8 * blockIdx.x;
      st[0] = ts0; st[1] = ts1; st[2] = ts1; st[3] = ts1; st[4] = ts1; st[5] = ts1;
      st[6] = (unsigned long long)__smid() | (1ull << 32);
      st[7] = 0;
    }
  }
#endif
}

template <int RMAX, int ST>
cudaError_t init_one() {
  return cudaFuncSetAttribute(k1_tcp_kernel<RMAX, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              K1P<RMAX, ST>::SMEM);
}

template <int RMAX, int ST>
void launch_r(const Dev& D, int grid, cudaStream_t st, int cur) {
  launch_pdl(k1_tcp_kernel<RMAX, ST>, dim3(grid * K1P_CTAS), dim3(THREADS), K1P<RMAX, ST>::SMEM, st, D, cur);
}

template <int ST>
void launch_st(const Dev& D, int grid, cudaStream_t st, int cur) {
  if (D.k1_pw > 0) launch_r<2, ST>(D, grid, st, cur);
  else if (D.R <= 1) launch_r<1, ST>(D, grid, st, cur);
  else if (D.R <= 2) launch_r<2, ST>(D, grid, st, cur);
  else if (D.R <= 4) launch_r<4, ST>(D, grid, st, cur);
  else if (D.R <= 8) launch_r<8, ST>(D, grid, st, cur);
  else launch_r<16, ST>(D, grid, st, cur);
}

}  // namespace

cudaError_t k1_tcp_init() {
  cudaError_t e;
#define K1TCP_INIT(R)                                              \
  if ((e = init_one<R, 1>()) != cudaSuccess) return e;             \
  if ((e = init_one<R, 2>()) != cudaSuccess) return e;
  K1TCP_INIT(1) K1TCP_INIT(2) K1TCP_INIT(4) K1TCP_INIT(8) K1TCP_INIT(16)
#undef K1TCP_INIT
  return cudaSuccess;
}

// grid = number of SMs (one CTA per SM: A buffers + rings take ~210 KB of shared memory)
void launch_k1_tcp(const Dev& D, int grid, cudaStream_t st, int cur) {
  if (D.storage == 1) launch_st<1>(D, grid, st, cur);
  else launch_st<2>(D, grid, st, cur);
}
