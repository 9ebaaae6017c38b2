// fsqr_dev.cuh — device-side state, PTX wrappers and the shared epilogue of the
// FS-QRPPA hot path (sm_100a).  Shared by every kernel translation unit.
//
// Arithmetic design:
//  * a1 (X~^T theta) is computed EXACTLY in integers for genotype storage:
//    theta^k is quantised once per iteration to T_i = round(theta_i / delta),
//    delta = 2^e with |T_i| <= 2^28, and split into four signed base-256 digits
//    d_0..d_3 (T = d0*2^24 + d1*2^16 + d2*2^8 + d3).  Each digit row is an int8
//    B operand; D_jk = sum_i G_ij d_k(i) is an exact int32 (tcgen05 kind::i8
//    accumulator or dp4a), so sum_i (G_ij - m_j) T_i = (n*S_j - colsum_j*sum T)/n
//    is exact and order-independent; g_j = delta * that / s_j in fp64.
//  * a4 (X~ beta) accumulates int64 fixed-point C_j = round(2^E beta_j / s_j)
//    with E chosen from max|C| and |S| so nothing overflows; integer atomics
//    make the result independent of scheduling (bitwise deterministic).
//  * proxes, residuals, dual step and all reductions are fp64.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FSQR_NPART 5          // per-CTA K2 partials per RHS: rb, bb, gg, pen, nnz
#define FSQR_NSCAL 4          // per-RHS scalars of the current iterate: Rp, Rz, loss_sum, (spare)
#define FSQR_MAXR 16
#define FSQR_TRACE_W 5        // trace row: Rp, Rb, Rz, obj, nnz
#define FSQR_FPART 8          // finalize partials per CTA and RHS: 7 sums + max|theta|
#define FIN_THREADS 256
#define FIN_MAXGRID 256       // ceil(65536 / FIN_THREADS)
#define FSQR_TSTAMPS 2048     // per-CTA timing stamps of measurement builds
#define FSQR_PATH_W 8         // path record: iters, Rp, Rb, Rz, obj, nnz, converged, loss sum

// ST_SWITCH: path mode, w^k was just recorded as point t and becomes the start of point t+1
// (reading R10): the update of iteration k (taken with lambda_t) is discarded -- K1 and finalize
// skip the RHS, K2's last CTA restored beta^k into the next parity -- and finalize's tail sets the
// RHS active again, so iteration k+1 re-tests w^k at lambda_{t+1}.
enum { ST_ACTIVE = 0, ST_CONVERGED = 1, ST_MAXITER = 2, ST_NUMERIC = 3, ST_SWITCH = 4 };

struct Dev {
  // sizes / layout
  int n, R, G, storage, npad, ldk;
  int k1_esmax;                     // k1_tcp: support entries per work item cap (<= 65536; FSQR_K1_ESMAX, tests)
  int k1_tc;                        // forward product: 0 k1_bulk (CUDA cores), 3 k1_tcp 2-bit, 4 k1_tcp u8 (tensor cores)
  int k1_pw;                        // > 0: k1_tcp in power mode (a0' forward pass X~_g v_g for every block g): the
                                    // entries are all columns, an item spans <= 2 blocks (slots 0/1 = blocks g0, g0+1),
                                    // accumulator (and colsum term) of block g; the value is the max entries per block
  int x_policy;                     // L2 hint of the X stream in K2: 0 evict_first, 1 normal, 2 evict_last
  int k1_policy;                    // L2 hint of the forward gather: 0 evict_first, 1 normal, 2 evict_last
  int bperm;                        // 1: theta digit rows in the 2-bit tcgen05 K order (k2_tc2.cu)
  int64_t p, ld;
  int64_t gq, grem;                 // block partition of the p+1 model columns: q = (p+1)/G, rem
  // design (borrowed) + statistics
  const uint8_t* X8;
  const float* Xf;
  const int32_t* colsum;            // exact integer column sums (genotype storage)
  const double* mean;
  const double* inv_sd;
  double* lamw;                     // [(p+1)*R] penalty weights w_jr (lam_jr = lam_r w_jr), coefficient-major
  int* use_w;                       // [1] device flag: 0 -> all weights 1 (lamw not read)
  const double* eta;                // [G]
  const double* inv_eta;            // [G] 1/eta_g (host IEEE division; E14 multiplies by it)
  // state
  double* beta[2];                  // [(p+1)*R], coefficient-major
  double* z;                        // [R*n]
  double* theta;                    // [R*n]
  double* rres;                     // [R*n] r^k
  double* s;                        // [R*n] X~beta^k
  const double* y;                  // [n]
  double* sdense;                   // [R*n] forward output of the fp32 path
  int8_t* Bq;                       // [npad][ldk] theta digits
  long long* Tsum;                  // [R]
  double* delta;                    // [R]
  double* sumth;                    // [R] sum theta^k (fp64)
  // support lists, double-buffered by iteration parity
  int32_t* sup_idx[2];              // data column index
  double* sup_c[2];                 // [cap*R] beta_j / s_j
  int32_t* sup_cs[2];               // colsum_j of each entry (forward-product centring term)
  double* sup_b[2];                 // [cap*R] beta_j
  int* sup_cnt;                     // [2]
  unsigned long long* cmax;         // [2][R] bits of max |beta_j/s_j|
  long long* sacc;                  // [R*n] int64 forward accumulators
  long long* mterm;                 // [R] the colsum term of the forward sums
  unsigned int* k1bar;              // [1] grid-barrier counter of k1_tcp's fused finalize
  unsigned long long* tstamp;       // [FSQR_TSTAMPS] globaltimer stamps of instrumented builds (fsqr_debug_stamps)
  // K2 partials + last-CTA ticket
  double* k2part;                   // [grid][R][FSQR_NPART]
  unsigned int* ticket;
  // multi-CTA finalize partials + ticket
  double* fpart;                    // [FIN_MAXGRID][R][FSQR_FPART]
  long long* ftsum;                 // [FIN_MAXGRID][R]
  unsigned int* fticket;            // [1 + MAXR]: overall, then per RHS
  // per-RHS control
  const double* tau;                // [R]
  double* lam_cur;                  // [R]
  double* lam2;                     // [R] elastic-net quadratic weights (0 = LASSO / weighted l1)
  double* scal;                     // [R][FSQR_NSCAL]
  int* status;                      // [R]
  long long* commit_iter;           // [R]
  long long* iter;                  // [1]
  long long* kbase;                 // [1] iteration at which the current solve call started (max_iter is per call)
  int* stop;                        // [1]
  double* lastR;                    // [R][FSQR_TRACE_W]
  double* trace;                    // [trace_cap][R][FSQR_TRACE_W]
  int trace_cap;
  double tol, mu, sigma;            // sigma = mu/(G+1)
  long long max_iter;
  // path
  const double* lam_path;           // [R][T]
  int T;
  int* t_idx;                       // [R]
  long long* pt_iters;              // [R]
  long long max_iter_point;
  double* path_rec;                 // [R][T][FSQR_PATH_W]
  int32_t* path_idx;                // [R][T][path_cap]
  double* path_beta;                // [R][T][path_cap]
  long long* path_cnt;              // [R][T]
  int path_cap;
  // mode (baked per captured graph)
  int check;                        // stop test on
  int path;                         // lambda-path state machine on
  int update;                       // 0: K2 computes R(w^k) only (fsqr_kkt)
};

// ------------------------------------------------------------------ helpers

// column of sample i in the theta digit rows: natural order, or (bperm) the K order of the
// 2-bit tensor-core kernel, kappa = 128q + 4u + b for sample s = 16u + 4b + q of each 512-block
__device__ __forceinline__ int bq_index(const Dev& D, int i) {
  if (!D.bperm) return i;
  const int s = i & 511;
  return (i & ~511) | ((s & 3) << 7) | ((s >> 4) << 2) | ((s >> 2) & 3);
}

__device__ __forceinline__ int block_of_col(const Dev& D, int64_t j) {
  // contiguous near-equal blocks of the p+1 model columns (first `grem` blocks hold q+1)
  // p + 1 <= 2^31, so 32-bit unsigned divisions suffice (a 64-bit one is a long software sequence)
  const uint32_t q1 = (uint32_t)(D.gq + 1), big = (uint32_t)(D.grem * (D.gq + 1)), jj = (uint32_t)j;
  return (int)(jj < big ? jj / q1 : (uint32_t)D.grem + (jj - big) / (uint32_t)D.gq);
}

__device__ __forceinline__ double pos_part(double v) { return v > 0.0 ? v : 0.0; }

// E14
__device__ __forceinline__ double prox_beta(double b, double g, double lam, double eta) {
  double a = eta * b + g;
  return (pos_part(a - lam) - pos_part(-a - lam)) / eta;
}

// E14 with a precomputed 1/eta (the product differs from the quotient by at most one rounding)
__device__ __forceinline__ double prox_beta_inv(double b, double g, double lam, double eta, double inv_eta) {
  double a = eta * b + g;
  return (pos_part(a - lam) - pos_part(-a - lam)) * inv_eta;
}

// soft-threshold S_c(v) for the KKT residual
__device__ __forceinline__ double soft_thr(double v, double c) {
  return v > c ? v - c : (v < -c ? v + c : 0.0);
}

// prox of rho_tau with unit weight (KKT residual R_z)
__device__ __forceinline__ double prox_rho1(double v, double tau) {
  return v > tau ? v - tau : (v < tau - 1.0 ? v + 1.0 - tau : 0.0);
}

// fixed-point exponent for the forward product: 2 n cnt max|c| 2^E < 2^61 (no int64 overflow in
// n*S - M) and max|c| 2^E < 2^43 (22-bit split of C in the int32 inner loop of k1)
__device__ __forceinline__ int fwd_exponent(double cmax, long long cnt, int n) {
  if (!(cmax > 0.0) || cnt <= 0) return 0;
  int e1, e2;
  frexp(2.0 * (double)n * (double)cnt * cmax, &e1);
  frexp(cmax, &e2);
  return min(61 - e1, 43 - e2);
}

// release/acquire fence at GPU scope for the ticket pattern (writer: stores, fence, ticket atomic;
// last CTA: ticket atomic, fence, loads).  __threadfence() is a sequentially consistent fence
// (fence.sc.gpu), which measured up to 8 us on some SMs of the B200 in k1_tcp's tail; the
// ticket pattern only needs acquire-release ordering.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic sum of NV values over `count` per-CTA partial records (record b at
// base + b*stride) by a whole block: thread t adds records t, t+blockDim, ... in order,
// then a fixed-shape butterfly within warps and a fixed-order sum across warps.  The
// result depends only on (count, blockDim), never on scheduling.  `sm` needs
// 32*NV + NV doubles.  Every thread of the block must call it; all receive the sums.
template <int NV>
__device__ __forceinline__ void reduce_records(const double* base, int count, int stride, double (&out)[NV],
                                               double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double v[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = 0.0;
  for (int b = threadIdx.x; b < count; b += blockDim.x)
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] += base[(size_t)b * stride + q];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const double x = warp_sum_d(v[q]);
    if (lane == 0) sm[wid * NV + q] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double a = 0.0;
    for (int w = 0; w < nw; ++w) a += sm[w * NV + threadIdx.x];
    sm[32 * NV + threadIdx.x] = a;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) out[q] = sm[32 * NV + q];
  __syncthreads();
}

// ------------------------------------------------------------------ PTX: mbarrier / TMA / tcgen05

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// the same wait for a warp with nothing else to do (an epilogue waiting for its next accumulator):
// the suspend-time hint lets the hardware park the warp until the phase completes instead of
// re-issuing try_wait, so the spin does not take issue slots from the converter warps
__device__ __forceinline__ void mbar_wait_park(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity), "r"(0x100000u)
      : "memory");
}
// one non-blocking probe of a phase (for waits that back off with __nanosleep)
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int x, int y,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
// L2 prefetch of one TMA box (no shared-memory destination, no completion to wait for)
__device__ __forceinline__ void tma_prefetch_l2(const void* tmap, int x, int y, uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile.L2::cache_hint [%0, {%1, %2}], %3;" ::"l"(tmap),
               "r"(x), "r"(y), "l"(policy)
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// Programmatic dependent launch: every hot-path kernel lets the next one be scheduled at once
// (its prologue -- barrier init, TMEM allocation, tensor-map prefetch -- overlaps this kernel's
// tail) and waits for the previous grid's completion (memory visible) before touching state.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// one lane of a converged warp (the tcgen05.mma issuer); operands computed before the branch stay
// warp-uniform, so ptxas keeps them in uniform registers (no per-MMA waterfall)
__device__ __forceinline__ bool elect_one() {
  uint32_t p = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n}"
      : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SM100 shared-memory matrix descriptor, K-major, 128B swizzle: SBO = 1024 B (8 rows x 128 B), LBO = 16 B
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;               // LBO (unused for swizzled K-major) = 16 B
  d |= (uint64_t)(1024u >> 4) << 32;     // SBO
  d |= (uint64_t)1u << 46;               // version = 1 (sm100)
  d |= (uint64_t)2u << 61;               // SWIZZLE_128B
  return d;
}

// instruction descriptor: kind::i8, D = s32, A = s8, B = s8, both K-major, M = 128, N = npad
// same with an UNSIGNED 8-bit A operand (k2_tc2's plane-split codes reach 2 * 64 = 128)
__host__ __device__ constexpr uint32_t idesc_u8s8(int N) {
  return (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__host__ __device__ constexpr uint32_t idesc_i8(int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ per-launch K2 context

// per-RHS constants of one K2 launch, in shared memory (read once per column; keeping them in
// registers costs ~9 registers per RHS and spilled the 9-RHS epilogue)
template <int RMAX>
struct K2Const {
  double lam[RMAX];
  double lam2[RMAX];        // elastic-net quadratic weight (reading R19)
  double gscale[RMAX];      // delta_r / n (genotype storage)
  long long Tsum[RMAX];
  int active[RMAX];
};

template <int RMAX>
struct K2Ctx {
  long long k;
  bool use_w;
  const double* beta_in;
  double* beta_out;
  int32_t* sidx;
  int32_t* scs;
  const int32_t* colsum;
  double* sc;
  double* sb;
  int* scnt;
  int R;
  const K2Const<RMAX>* cs;  // shared memory
};

// fp64 partials of the stopping test: per thread in registers for up to 4 RHS; for 5+ RHS the
// registers would spill the epilogue, so every column's contributions are warp-reduced at once
// and added by lane 0 to this warp's slot [RMAX][NPART+1] of the CTA reduction buffer (fixed
// order: deterministic).  In that mode epi_column must be called by all 32 lanes.
template <int RMAX>
struct K2Part {
  static constexpr bool SM = RMAX > 4;
  double v[SM ? 1 : RMAX][FSQR_NPART];
  double cmax[SM ? 1 : RMAX];
  double* slot;   // SM mode: red + wid * RMAX * (NPART + 1)
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int r = 0; r < (SM ? 1 : RMAX); ++r) {
      cmax[r] = 0.0;
#pragma unroll
      for (int q = 0; q < FSQR_NPART; ++q) v[r][q] = 0.0;
    }
  }
  __device__ __forceinline__ void add(int r, const double (&x)[FSQR_NPART], double cm) {
    if constexpr (SM) {
      constexpr int W = FSQR_NPART + 1;
      static_assert(FSQR_NPART == 5, "partials: four sums and a 0/1 count");
      // warp reduction of one column group's partials, fixed order: the 0/1 count (x[4]) exactly as
      // the popcount of a ballot; the max of the non-negative cm as the max of its bit pattern (two
      // 32-bit redux); the four sums by a reduce-scatter butterfly -- at xor 16 a lane keeps one pair
      // and sends the other, at xor 8 one value, then three full levels -- so lane group (lane >> 3)
      // ends with sum number (lane >> 3): 12 shuffles instead of 40 for the same four totals
      const int lane = threadIdx.x & 31;
      const unsigned bal = __ballot_sync(0xffffffffu, x[4] != 0.0);
      const unsigned long long mb = (unsigned long long)__double_as_longlong(cm);
      const unsigned mhi = __reduce_max_sync(0xffffffffu, (unsigned)(mb >> 32));
      const unsigned mlo = __reduce_max_sync(0xffffffffu, (unsigned)(mb >> 32) == mhi ? (unsigned)mb : 0u);
      const bool h16 = (lane & 16) != 0, h8 = (lane & 8) != 0;
      double k0 = h16 ? x[2] : x[0], k1 = h16 ? x[3] : x[1];
      const double s0 = h16 ? x[0] : x[2], s1 = h16 ? x[1] : x[3];
      k0 += __shfl_xor_sync(0xffffffffu, s0, 16);
      k1 += __shfl_xor_sync(0xffffffffu, s1, 16);
      double k = (h8 ? k1 : k0) + __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
      if ((lane & 7) == 0) slot[r * W + (lane >> 3)] += k;
      if (lane == 0) {
        slot[r * W + 4] += (double)__popc(bal);
        slot[r * W + FSQR_NPART] =
            fmax(slot[r * W + FSQR_NPART], __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo)));
      }
    } else {
#pragma unroll
      for (int q = 0; q < FSQR_NPART; ++q) v[r][q] += x[q];
      cmax[r] = fmax(cmax[r], cm);
    }
  }
};

// a2 epilogue for one data column c with g_r = (X~^T theta^k)_j, j = c + 1 (valid lanes only;
// invalid lanes contribute zeros -- all lanes must call it when K2Part is in shared-memory mode).
// Writes beta^{k+1}, accumulates R_beta(w^k) partials and the penalty of beta^k,
// returns whether beta^{k+1}_j != 0 for some active RHS (support membership) and
// fills cval/bval for the support entry.
// bsrc / bdst: this column's R values of beta^k / beta^{k+1} ([j][R] rows of the state, or a
// shared-memory staging copy of them; nullptr = the state rows C.beta_in / C.beta_out + j R)
template <int RMAX>
__device__ __forceinline__ bool epi_column(const Dev& D, const K2Ctx<RMAX>& C, int64_t c, const double* g,
                                           K2Part<RMAX>& P, bool valid = true, const double* bsrc = nullptr,
                                           double* bdst = nullptr) {
  const int64_t j = c + 1;
  const double isd = valid ? D.inv_sd[c] : 0.0;
  const int gb = valid ? block_of_col(D, j) : 0;
  const double eta = valid ? D.eta[gb] : 1.0;
  const double inv_eta = valid ? D.inv_eta[gb] : 1.0;   // E14 multiplies by 1/eta_g
  // every RHS's beta^k_j is loaded before any store of this column: with several RHS
  // the partial sums below write shared memory, which would otherwise keep the compiler from
  // hoisting the next RHS's global load over them (one memory latency per RHS per column)
  double bin[RMAX];
#pragma unroll
  if (!bsrc) bsrc = C.beta_in + j * C.R;
  if (!bdst) bdst = C.beta_out + j * C.R;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) bin[r] = (valid && r < C.R) ? bsrc[r] : 0.0;
  bool nz = false;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    if (r >= C.R || !C.cs->active[r]) continue;   // warp-uniform
    double x[FSQR_NPART] = {0.0, 0.0, 0.0, 0.0, 0.0};
    double cm = 0.0;
    if (valid) {
      const double b = bin[r];
      const double lam = C.use_w ? C.cs->lam[r] * D.lamw[j * C.R + r] : C.cs->lam[r];
      // KKT residual part of w^k and penalty at beta^k
      const double l2 = C.cs->lam2[r];
      const double d = b - soft_thr(b + (g[r] - l2 * b), lam);   // KKT: g - lam2 b in lam d|b|
      x[0] = d * d;
      x[1] = b * b;
      x[2] = g[r] * g[r];
      x[3] = lam * fabs(b) + 0.5 * l2 * b * b;
      x[4] = (b != 0.0) ? 1.0 : 0.0;
      if (D.update) {
        // E14, or the elastic-net block prox (Remark 3, L347-349; reading R19) when lam2 > 0
        const double bn = l2 == 0.0 ? prox_beta_inv(b, g[r], lam, eta, inv_eta)
                                    : (pos_part(eta * b + g[r] - lam) - pos_part(-eta * b - g[r] - lam)) / (eta + l2);
        bdst[r] = bn;
        if (bn != 0.0) {
          nz = true;
          cm = fabs(bn * isd);
        }
      }
    }
    P.add(r, x, cm);
  }
  return nz;
}

// warp-aggregated append of support entries (lanes with nz); the entry's beta^{k+1}_j and
// beta^{k+1}_j / s_j of every RHS are re-read from beta_out (this thread wrote them in epi_column),
// so the epilogue keeps no per-RHS copies in registers; an inactive RHS gets zeros
template <int RMAX>
__device__ __forceinline__ void support_append(const Dev& D, const K2Ctx<RMAX>& C, bool nz, int64_t c,
                                               const double* bout = nullptr) {
  const unsigned m = __ballot_sync(0xffffffffu, nz);
  if (m == 0) return;
  const int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(C.scnt, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (nz) {
    const int e = base + __popc(m & ((1u << lane) - 1u));
    const double isd = D.inv_sd[c];
    C.sidx[e] = (int32_t)c;
    C.scs[e] = C.colsum[c];
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r < C.R) {
        const double bn = C.cs->active[r] ? (bout ? bout[r] : C.beta_out[(c + 1) * C.R + r]) : 0.0;
        C.sc[(int64_t)e * C.R + r] = bn != 0.0 ? bn * isd : 0.0;
        C.sb[(int64_t)e * C.R + r] = bn;
      }
    }
  }
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// L1 prefetch of the per-column state the a2 epilogue reads for data column c (beta^k of every RHS,
// colsum, 1/s_j), issued one tile ahead: the epilogue's loads then hit L1 instead of waiting on HBM
template <int RMAX>
__device__ __forceinline__ void epi_prefetch(const Dev& D, const K2Ctx<RMAX>& C, int64_t c, bool beta = true) {
  if (c >= D.p) return;
  if (beta) {
    const double* b = C.beta_in + (c + 1) * C.R;
    prefetch_l1(b);
    if (C.R > 1) prefetch_l1(b + C.R - 1);
  }
  prefetch_l1(D.colsum + c);
  prefetch_l1(D.inv_sd + c);
}

// exact integer reconstruction of g_r from the four digit accumulators of RHS r
__device__ __forceinline__ double g_from_digits(int n, int32_t colsum, long long Tsum, double gscale, double isd,
                                                const int32_t* Dk) {
  long long S = ((long long)Dk[0] << 24) + ((long long)Dk[1] << 16) + ((long long)Dk[2] << 8) + (long long)Dk[3];
  long long num = (long long)n * S - (long long)colsum * Tsum;
  return (double)num * gscale * isd;
}

// ------------------------------------------------------------------ host launchers (one per TU)

extern int g_fsqr_pdl;   // 1: hot-path kernels are launched with programmatic stream serialization

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_fsqr_pdl;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

struct LaunchCfg {
  int grid;
  cudaStream_t st;
};

void launch_k2_tc(const Dev& D, const void* tmX, const void* tmB, int grid, cudaStream_t st);
void launch_k2_tc2(const Dev& D, const void* tmX, const void* tmB, int grid, cudaStream_t st);
cudaError_t k2_tc2_init();
void launch_k2_simt(const Dev& D, int grid, cudaStream_t st);
void launch_k1(const Dev& D, int grid, cudaStream_t st);
bool k1_fuses_finalize(const Dev& D);   // the forward-product kernel also runs the finalize
void launch_finalize(const Dev& D, cudaStream_t st);
void launch_pack2(const uint8_t* x8, int64_t ld8, int n, int64_t p, uint8_t* x2, int64_t ld2, int* bad,
                  cudaStream_t st);
void launch_unpack2(const uint8_t* x2, int64_t ld2, int64_t p, uint8_t* x8, int64_t ld8, cudaStream_t st);
int k2_tc_smem_bytes(int npad);
cudaError_t k2_tc_init();
cudaError_t k1_init();
void launch_k1_tcp(const Dev& D, int grid, cudaStream_t st, int cur);
cudaError_t k1_tcp_init();
int k2_tc_supported(int npad);
