// fsqr_api.cu — host runtime and C ABI (include/fsqr.h) of the FS-QRPPA hot path.
//
// Owns the device state, runs the setup passes (a0 column statistics, a0'
// power method, lambda_max), builds the TMA descriptors, and drives the
// iteration as CUDA-graph chunks of {K2: X~^T theta + beta prox + support,
// K1: support-gather X~ beta, finalize: z prox + dual step + theta digits}.
// Convergence is decided on the device (last CTA of K2); the host only polls a
// flag between chunks.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fsqr.h"
#include "fsqr_dev.cuh"

void launch_init_state(const Dev& D, cudaStream_t st);
void launch_colstats(const Dev& D, int32_t* colsum, double* mean, double* inv_sd, double* sd, int* bad,
                     cudaStream_t st);
void launch_power_start(int64_t p1, uint64_t seed, double* v, cudaStream_t st);
void launch_power_fwd(const Dev& D, const int64_t* bstart, const double* v, const int* frozen, double* u,
                      cudaStream_t st);
void launch_back_f64(const Dev& D, const double* u, int per_block, const int* frozen, double* w,
                     unsigned long long* maxbits, cudaStream_t st);
void launch_power_reduce(const Dev& D, const int64_t* bstart, const double* v, const double* w, const int* frozen,
                         double* est, double* nrm, cudaStream_t st);
void launch_power_norm(const Dev& D, double* v, const double* w, const double* nrm, const int* frozen,
                       cudaStream_t st);
void launch_lanczos_orth(const Dev& D, const double* v, const double* vp, double* w, const double* alpha,
                         const double* beta, const int* frozen, cudaStream_t st);
void launch_lanczos_next(const Dev& D, double* v, double* vp, const double* w, const double* beta, const int* frozen,
                         cudaStream_t st);
void launch_null_score(const double* y, int n, const double* tau, int R, int* ord, double* psi, cudaStream_t st);
void launch_iota(int32_t* ix, int64_t p, cudaStream_t st);
void launch_power_coef(const Dev& D, const double* v, const int* frozen, double* a, unsigned long long* cmax,
                       cudaStream_t st);
void launch_power_fwd_fin(const Dev& D, long long* sacc, long long* mterm, const unsigned long long* cmax, int maxcnt,
                          const double* v, const int* frozen, double* u, double* Ug, cudaStream_t st);
void launch_power_quant(const Dev& D, const double* u, const double* Ug, const int* frozen, int8_t* Bp, int ldk,
                        long long* Tsum, double* gs, double* w, cudaStream_t st);
void launch_power_back_tc2(const Dev& D, const void* tmX, const void* tmBp, const long long* Tsum, const double* gs,
                           const int* frozen, double* w, int grid, cudaStream_t st);
void launch_power_fwd_int(const Dev& D, const int64_t* bstart, const double* v, const int* frozen, double* part,
                          int S, double* u, double* Ug, cudaStream_t st);
void launch_sum_parts(const double* part, int S, int G, int n, double* u, double* Ug, cudaStream_t st);
void launch_back_int(const Dev& D, const double* u, const double* Ug, int per_block, const int* frozen, double* w,
                     unsigned long long* maxbits, cudaStream_t st);
void launch_build_support(const Dev& D, int par, cudaStream_t st);
void launch_commit_stats(const Dev& D, double* pen, double* beta_out, int orig, cudaStream_t st);
void launch_unfreeze(const Dev& D, cudaStream_t st);
void launch_lla_weights(const Dev& D, int kind, double a, cudaStream_t st);
cudaError_t pivotal_init();
void launch_piv_draws(int n, int ldk, double tau, uint64_t seed, long long b0, int8_t* draws, int* nb,
                      cudaStream_t st);
void launch_pivotal(const Dev& D, const void* tmA, const void* tmX256, const int* nb, unsigned long long* lmax,
                    int grid, cudaStream_t st);
void launch_k1_mode(const Dev& D, int grid, cudaStream_t st, int cur);

int g_fsqr_pdl = 1;   // FSQR_PDL=0 launches the hot path without programmatic dependent launch

namespace {

thread_local std::string g_err;

struct Graph {
  cudaGraphExec_t exec = nullptr;
  int iters = 0;
};

enum Mode { M_ITER = 0, M_SOLVE = 1, M_PATH = 2, M_KKT = 3, M_COUNT = 4 };

}  // namespace

struct fsqr_ctx {
  Dev D{};
  Dev mode_dev[M_COUNT];
  Graph graph[M_COUNT];
  int backend = FSQR_BACKEND_SIMT;
  int sms = 148;
  int k2_grid = 148, k1_grid = 148;
  int chunk = 16;
  CUtensorMap tmX{}, tmB{};
  cudaStream_t cap_stream = nullptr;
  cudaStream_t alloc_st = nullptr;   // stream of the API call that is allocating (zero-fill is ordered on it)
  std::vector<void*> allocs;
  std::string err;
  fsqr_options opt{};
  std::vector<double> tau, lambda, lambda_max, eta, inv_eta;
  int R = 1, T = 0;
  int64_t n = 0, p = 0;
  double* h_pin = nullptr;  // small pinned scratch
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  bool owns_stats = true;
  int64_t path_cap = 0;
  // pivotal statistic (lazily allocated)
  int8_t* piv_draws = nullptr;
  int* piv_nb = nullptr;
  unsigned long long* piv_lmax = nullptr;
  CUtensorMap tmPivA{}, tmPivX{};
  void* piv_enc = nullptr;      // cuTensorMapEncodeTiled
  bool piv_x_ready = false;     // tmPivX describes the borrowed u8 X (not rebuilt per call)
};

namespace {

fsqr_status set_err(fsqr_ctx* c, fsqr_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  g_err = buf;
  return s;
}

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return set_err(ctx, e_ == cudaErrorMemoryAllocation ? FSQR_ERR_OOM : FSQR_ERR_CUDA, "%s: %s (%s:%d)", \
                     #call, cudaGetErrorString(e_), __FILE__, __LINE__);                           \
  } while (0)

template <class T>
fsqr_status dalloc(fsqr_ctx* ctx, T** p, size_t count) {
  void* q = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(&q, count * sizeof(T));
  if (e != cudaSuccess) return set_err(ctx, FSQR_ERR_OOM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
  // zero-fill on the calling API's stream: a legacy-stream cudaMemset is not ordered against the
  // caller's (typically non-blocking) stream and could land after work enqueued there
  e = cudaMemsetAsync(q, 0, count * sizeof(T), ctx->alloc_st);
  if (e != cudaSuccess) return set_err(ctx, FSQR_ERR_CUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  ctx->allocs.push_back(q);
  *p = (T*)q;
  return FSQR_OK;
}

// calls without a stream argument read or write state that queued work may still be using: they
// first wait for the device (a legacy-stream cudaMemcpy is not ordered against non-blocking streams)
#define SYNC_DEVICE() CK(cudaDeviceSynchronize())

#define AL(ptr, cnt)                                        \
  do {                                                      \
    fsqr_status s_ = dalloc(ctx, &(ptr), (size_t)(cnt));    \
    if (s_ != FSQR_OK) return s_;                           \
  } while (0)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// column stride of an owned 2-bit copy (FSQR_DESIGN_PACK2): ceil(n/4) bytes rounded up to 128
int64_t pack2_ld(int64_t n) { return ((n + 3) / 4 + 127) / 128 * 128; }

fsqr_status make_tmaps(fsqr_ctx* ctx) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return set_err(ctx, FSQR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  EncodeTiledFn enc = (EncodeTiledFn)fn;
  const Dev& D = ctx->D;
  {
    // u8: inner extent n samples; 2-bit: the packed column (ld bytes, zero padding beyond n/4)
    cuuint64_t dims[2] = {(cuuint64_t)(D.storage == 2 ? std::min<int64_t>(D.ld, ((D.n + 3) / 4 + 15) / 16 * 16) : D.n),
                          (cuuint64_t)D.p};
    cuuint64_t strides[1] = {(cuuint64_t)D.ld};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t es[2] = {1, 1};
    // L2 promotion for the streamed design: 256-byte promotion re-fetches the boundary line of
    // each column when ld % 256 != 0 (+1.6% DRAM bytes at n = 10k, ncu), but its larger DRAM
    // requests still finish the pass 3.5% sooner than no promotion (1.55 vs 1.61 ms, B200).
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (const char* ev = getenv("FSQR_L2PROMO")) promo = (CUtensorMapL2promotion)atoi(ev);
    CUresult r = enc(&ctx->tmX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)D.X8, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(ctx, FSQR_ERR_CUDA, "tensor map for X failed (%d)", (int)r);
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)D.ldk, (cuuint64_t)D.npad};
    cuuint64_t strides[1] = {(cuuint64_t)D.ldk};
    cuuint32_t box[2] = {128, (cuuint32_t)(4 * D.R)};   // only the 4R live digit rows (rows up to npad stay 0 in smem)
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&ctx->tmB, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)D.Bq, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(ctx, FSQR_ERR_CUDA, "tensor map for theta digits failed (%d)", (int)r);
  }
  return FSQR_OK;
}

void launch_k2(fsqr_ctx* ctx, const Dev& D, cudaStream_t st) {
  if (ctx->backend == FSQR_BACKEND_TC && D.storage == FSQR_PACKED2)
    launch_k2_tc2(D, &ctx->tmX, &ctx->tmB, ctx->k2_grid, st);
  else if (ctx->backend == FSQR_BACKEND_TC)
    launch_k2_tc(D, &ctx->tmX, &ctx->tmB, ctx->k2_grid, st);
  else
    launch_k2_simt(D, ctx->k2_grid, st);
}

void enqueue_iteration(fsqr_ctx* ctx, const Dev& D, cudaStream_t st) {
  launch_k2(ctx, D, st);
  launch_k1(D, ctx->k1_grid, st);
  if (!k1_fuses_finalize(D)) launch_finalize(D, st);
}

fsqr_status get_graph(fsqr_ctx* ctx, int mode, Graph** out) {
  Graph& g = ctx->graph[mode];
  if (!g.exec) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < ctx->chunk; ++i) enqueue_iteration(ctx, ctx->mode_dev[mode], ctx->cap_stream);
    CK(cudaStreamEndCapture(ctx->cap_stream, &graph));
    CK(cudaGraphInstantiate(&g.exec, graph, 0));
    cudaGraphDestroy(graph);
    g.iters = ctx->chunk;
  }
  *out = &g;
  return FSQR_OK;
}

fsqr_status run_chunk(fsqr_ctx* ctx, int mode, cudaStream_t st) {
  Graph* g;
  fsqr_status s = get_graph(ctx, mode, &g);
  if (s != FSQR_OK) return s;
  CK(cudaGraphLaunch(g->exec, st));
  return FSQR_OK;
}

fsqr_status reset_control(fsqr_ctx* ctx, cudaStream_t st) {
  // unfreeze committed betas into the current parity, then mark every RHS active
  launch_unfreeze(ctx->D, st);
  CK(cudaGetLastError());
  CK(cudaMemsetAsync(ctx->D.status, 0, sizeof(int) * ctx->R, st));
  CK(cudaMemsetAsync(ctx->D.stop, 0, sizeof(int), st));
  return FSQR_OK;
}

fsqr_status init_state(fsqr_ctx* ctx, cudaStream_t st) {
  // support list of the current beta (parity of iter), forward product, n-vector state
  Dev& D = ctx->D;
  long long k = 0;
  CK(cudaMemcpyAsync(&k, D.iter, sizeof k, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int par = (int)(k & 1);
  CK(cudaMemsetAsync(D.sup_cnt, 0, 2 * sizeof(int), st));
  CK(cudaMemsetAsync(D.cmax, 0, 2 * ctx->R * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(D.sacc, 0, (size_t)ctx->R * ctx->n * sizeof(long long), st));
  CK(cudaMemsetAsync(D.mterm, 0, ctx->R * sizeof(long long), st));
  CK(cudaMemsetAsync(D.k1bar, 0, sizeof(unsigned), st));
  CK(cudaMemsetAsync(D.fticket, 0, (1 + FSQR_MAXR) * sizeof(unsigned), st));
  CK(cudaMemsetAsync(D.stop, 0, sizeof(int), st));
  if (D.storage != 0) launch_build_support(D, par, st);
  launch_k1_mode(D, ctx->k1_grid, st, 1);
  launch_init_state(D, st);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(st));
  return FSQR_OK;
}

// largest eigenvalue of the symmetric tridiagonal Lanczos matrix (diagonal a, off-diagonal b,
// b.size() == a.size() - 1): bisection on Sturm counts inside the Gershgorin interval
double tridiag_top(const std::vector<double>& a, const std::vector<double>& b) {
  const int k = (int)a.size();
  double lo = a[0], hi = a[0];
  for (int i = 0; i < k; ++i) {
    const double rad = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < k ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - rad);
    hi = std::max(hi, a[i] + rad);
  }
  auto below = [&](double x) {   // eigenvalues < x
    int cnt = 0;
    double q = a[0] - x;
    cnt += q < 0.0;
    for (int i = 1; i < k; ++i) {
      if (q == 0.0) q = 1e-300;
      q = (a[i] - x) - b[i - 1] * b[i - 1] / q;
      cnt += q < 0.0;
    }
    return cnt;
  };
  for (int it = 0; it < 200 && hi > lo; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (below(mid) == k) hi = mid; else lo = mid;
  }
  return hi;
}

fsqr_status power_method(fsqr_ctx* ctx, cudaStream_t st) {
  Dev& D = ctx->D;
  const int G = D.G;
  const int64_t p1 = D.p + 1;
  // block boundaries (same rule as block_of_col)
  std::vector<int64_t> bs(G + 1);
  bs[0] = 0;
  for (int g = 0; g < G; ++g) bs[g + 1] = bs[g] + D.gq + (g < D.grem ? 1 : 0);
  int64_t* d_bs;
  int* d_frozen;
  double *v, *w, *u, *est, *nrm;
  AL(d_bs, G + 1);
  AL(d_frozen, G);
  AL(v, p1);
  AL(w, p1);
  AL(u, (size_t)G * D.n);
  AL(est, G);
  AL(nrm, G);
  const bool geno = D.storage != 0;
  constexpr int S = 8;   // column slices per block in the genotype forward (partials summed in fixed order)
  double *part = nullptr, *Ug = nullptr;
  if (geno) {
    AL(part, (size_t)S * G * D.n);
    AL(Ug, G);
  }
  // back pass X~_g^T u_g on the tensor cores for 2-bit storage (k2p_kernel): u_g as int8 digit planes
  // (rows 4g..4g+3 of Bp, plus 4 zero rows for the last block's pair); blocks of >= 128 columns keep
  // every 128-column tile within two blocks.  Otherwise the CUDA-core k_back_int.
  const bool tcback = ctx->backend == FSQR_BACKEND_TC && D.storage == FSQR_PACKED2 && D.gq >= 128;
  int8_t* Bp = nullptr;
  long long* Tsum = nullptr;
  double* gsc = nullptr;
  CUtensorMap tmBp{};
  if (tcback) {
    AL(Bp, (size_t)4 * (G + 1) * D.ldk);
    AL(Tsum, G);
    AL(gsc, G);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return set_err(ctx, FSQR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)D.ldk, (cuuint64_t)(4 * (G + 1))};
    cuuint64_t strides[1] = {(cuuint64_t)D.ldk};
    cuuint32_t box[2] = {128, 8};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeTiledFn)fn)(&tmBp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)Bp, dims, strides, box, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(ctx, FSQR_ERR_CUDA, "tensor map for the power digits failed (%d)", (int)r);
  }
  // forward pass X~_g v_g on the tensor cores as well (k1_tcp in power mode: every column an entry,
  // items spanning <= 2 blocks, one int64 accumulator row per block) when the forward product runs
  // on k1_tcp for this storage
  const bool tcfwd = tcback && D.k1_tc == 3;
  Dev Dp = D;
  double* acoef = nullptr;
  if (tcfwd) {
    int32_t* ident;
    int *cntp, *stop0;
    unsigned long long* cmx;
    long long *sacc_pw, *mterm_pw;
    AL(ident, (size_t)D.p);
    AL(acoef, (size_t)D.p);
    AL(cntp, 2);
    AL(stop0, 1);
    AL(cmx, 2);
    AL(sacc_pw, (size_t)G * D.n);
    AL(mterm_pw, G);
    launch_iota(ident, D.p, st);
    const int cnt2[2] = {(int)D.p, (int)D.p};
    CK(cudaMemcpyAsync(cntp, cnt2, sizeof(cnt2), cudaMemcpyHostToDevice, st));
    Dp.R = 1;
    Dp.k1_pw = (int)D.gq + 1;
    Dp.stop = stop0;
    Dp.sup_cnt = cntp;
    Dp.cmax = cmx;
    Dp.sacc = sacc_pw;
    Dp.mterm = mterm_pw;
    for (int q = 0; q < 2; ++q) {
      Dp.sup_idx[q] = ident;
      Dp.sup_cs[q] = const_cast<int32_t*>(D.colsum);   // read only in k1_tcp
      Dp.sup_c[q] = acoef;
    }
  }
  auto fwd = [&](const double* vv, double* uu, double* ug) {
    if (tcfwd) {
      CK(cudaMemsetAsync(Dp.cmax, 0, 2 * sizeof(unsigned long long), st));
      launch_power_coef(D, vv, d_frozen, acoef, Dp.cmax, st);
      launch_k1_mode(Dp, ctx->k1_grid, st, 1);
      launch_power_fwd_fin(D, Dp.sacc, Dp.mterm, Dp.cmax, Dp.k1_pw, vv, d_frozen, uu, ug, st);
    } else if (geno) {
      launch_power_fwd_int(D, d_bs, vv, d_frozen, part, S, uu, ug, st);
    } else {
      launch_power_fwd(D, d_bs, vv, d_frozen, uu, st);
    }
    return FSQR_OK;
  };
  auto back = [&](const double* uu, const double* ug, double* ww) {
    if (tcback) {
      launch_power_quant(D, uu, ug, d_frozen, Bp, D.ldk, Tsum, gsc, ww, st);
      launch_power_back_tc2(D, &ctx->tmX, &tmBp, Tsum, gsc, d_frozen, ww, ctx->k2_grid, st);
    } else {
      launch_back_int(D, uu, ug, 1, d_frozen, ww, nullptr, st);
    }
  };
  CK(cudaMemcpyAsync(d_bs, bs.data(), sizeof(int64_t) * (G + 1), cudaMemcpyHostToDevice, st));
  launch_power_start(p1, ctx->opt.seed, v, st);
  launch_power_reduce(D, d_bs, v, v, d_frozen, est, nrm, st);
  launch_power_norm(D, v, nullptr, nrm, d_frozen, st);
  CK(cudaGetLastError());
  std::vector<double> h_est(G), prev(G, 0.0), lam(G, 0.0), h_nrm(G);
  std::vector<int> frozen(G, 0);
  int live = G;
  if (ctx->opt.eta_method == FSQR_ETA_LANCZOS) {
    // Lanczos (L259): alpha_k = v^T X~_g^T X~_g v, w -= alpha v + beta_{k-1} v_{k-1}, beta_k = ||w||;
    // the estimate is the largest eigenvalue of the tridiagonal T_k (Ritz value <= Lambda_max)
    double *vp, *alpha, *beta, *junk;
    AL(vp, p1);
    AL(alpha, G);
    AL(beta, G);
    AL(junk, G);
    std::vector<std::vector<double>> ta(G), tb(G);
    std::vector<double> h_alpha(G), h_beta(G);
    for (int it = 1; it <= ctx->opt.power_max_iter && live > 0; ++it) {
      if (geno) {
        fwd(v, u, Ug);
        back(u, Ug, w);
      } else {
        launch_power_fwd(D, d_bs, v, d_frozen, u, st);
        launch_back_f64(D, u, 1, d_frozen, w, nullptr, st);
      }
      launch_power_reduce(D, d_bs, v, w, d_frozen, alpha, junk, st);
      launch_lanczos_orth(D, v, vp, w, alpha, beta, d_frozen, st);
      launch_power_reduce(D, d_bs, w, w, d_frozen, junk, beta, st);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h_alpha.data(), alpha, sizeof(double) * G, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_beta.data(), beta, sizeof(double) * G, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int g = 0; g < G; ++g) {
        if (frozen[g]) continue;
        ta[g].push_back(h_alpha[g]);
        lam[g] = tridiag_top(ta[g], tb[g]);
        if ((it > 1 && std::fabs(lam[g] - prev[g]) <= ctx->opt.power_tol * lam[g]) ||
            !(h_beta[g] > 1e-12 * std::fabs(h_alpha[g]))) {
          frozen[g] = 1;
          --live;
        } else {
          tb[g].push_back(h_beta[g]);
        }
        prev[g] = lam[g];
      }
      CK(cudaMemcpyAsync(d_frozen, frozen.data(), sizeof(int) * G, cudaMemcpyHostToDevice, st));
      launch_lanczos_next(D, v, vp, w, beta, d_frozen, st);
    }
    CK(cudaStreamSynchronize(st));
    ctx->eta.resize(G);
    for (int g = 0; g < G; ++g) ctx->eta[g] = ctx->opt.eta_safety * ctx->opt.mu * lam[g];
    return FSQR_OK;
  }
  for (int it = 1; it <= ctx->opt.power_max_iter && live > 0; ++it) {
    if (geno) {
      fwd(v, u, Ug);
      back(u, Ug, w);
    } else {
      launch_power_fwd(D, d_bs, v, d_frozen, u, st);
      launch_back_f64(D, u, 1, d_frozen, w, nullptr, st);
    }
    launch_power_reduce(D, d_bs, v, w, d_frozen, est, nrm, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_est.data(), est, sizeof(double) * G, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_nrm.data(), nrm, sizeof(double) * G, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int g = 0; g < G; ++g) {
      if (frozen[g]) continue;
      lam[g] = h_est[g];
      if ((it > 1 && std::fabs(h_est[g] - prev[g]) <= ctx->opt.power_tol * h_est[g]) || !(h_nrm[g] > 0.0)) {
        frozen[g] = 1;
        --live;
      }
      prev[g] = h_est[g];
    }
    CK(cudaMemcpyAsync(d_frozen, frozen.data(), sizeof(int) * G, cudaMemcpyHostToDevice, st));
    launch_power_norm(D, v, w, nrm, d_frozen, st);
  }
  CK(cudaStreamSynchronize(st));
  ctx->eta.resize(G);
  for (int g = 0; g < G; ++g) ctx->eta[g] = ctx->opt.eta_safety * ctx->opt.mu * lam[g];
  return FSQR_OK;
}

fsqr_status lambda_max(fsqr_ctx* ctx, cudaStream_t st) {
  Dev& D = ctx->D;
  double* psi;
  unsigned long long* mb;
  AL(psi, (size_t)ctx->R * D.n);
  AL(mb, ctx->R);
  int* ord;
  AL(ord, D.n);
  launch_null_score(D.y, D.n, D.tau, ctx->R, ord, psi, st);
  if (D.storage != 0) {
    double *tmp, *Us;
    AL(tmp, D.n);
    AL(Us, ctx->R);
    for (int r = 0; r < ctx->R; ++r) {
      launch_sum_parts(psi + (size_t)r * D.n, 1, 1, D.n, tmp, Us + r, st);
      launch_back_int(D, psi + (size_t)r * D.n, Us + r, 0, nullptr, nullptr, mb + r, st);
    }
  } else {
    for (int r = 0; r < ctx->R; ++r) launch_back_f64(D, psi + (size_t)r * D.n, 0, nullptr, nullptr, mb + r, st);
  }
  CK(cudaGetLastError());
  std::vector<unsigned long long> h(ctx->R);
  CK(cudaMemcpyAsync(h.data(), mb, sizeof(unsigned long long) * ctx->R, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  ctx->lambda_max.resize(ctx->R);
  for (int r = 0; r < ctx->R; ++r) {
    double v;
    memcpy(&v, &h[r], sizeof v);
    ctx->lambda_max[r] = v;
  }
  return FSQR_OK;
}

}  // namespace

// =====================================================================================================

extern "C" {

void fsqr_default_options(fsqr_options* o) {
  memset(o, 0, sizeof *o);
  o->G = 5;
  o->backend = FSQR_BACKEND_AUTO;
  o->mu = 0.0;
  o->eta_safety = 1.05;
  o->eta_host = nullptr;
  o->tol = 1e-6;
  o->max_iter = 100000;
  o->power_max_iter = 1000;
  o->trace_cap = 4096;
  o->power_tol = 1e-4;
  o->seed = 0x5EED;
  o->max_iter_point = 10000;
  o->eta_method = FSQR_ETA_LANCZOS;
}

const char* fsqr_status_str(fsqr_status s) {
  switch (s) {
    case FSQR_OK: return "FSQR_OK";
    case FSQR_NOT_CONVERGED: return "FSQR_NOT_CONVERGED";
    case FSQR_ERR_CONFIG: return "FSQR_ERR_CONFIG";
    case FSQR_ERR_DATA: return "FSQR_ERR_DATA";
    case FSQR_ERR_NUMERIC: return "FSQR_ERR_NUMERIC";
    case FSQR_ERR_CUDA: return "FSQR_ERR_CUDA";
    case FSQR_ERR_OOM: return "FSQR_ERR_OOM";
    case FSQR_ERR_STATE: return "FSQR_ERR_STATE";
  }
  return "FSQR_UNKNOWN";
}

const char* fsqr_last_error(const fsqr_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }
const char* fsqr_global_error(void) { return g_err.c_str(); }
const char* fsqr_backend_name(const fsqr_ctx* c) { return c && c->backend == FSQR_BACKEND_TC ? "tc" : "simt"; }

void fsqr_destroy(fsqr_ctx* ctx) {
  if (!ctx) return;
  cudaDeviceSynchronize();
  for (auto& g : ctx->graph)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  delete ctx;
}

static fsqr_status create_impl(fsqr_ctx* ctx, const fsqr_design* X, const double* y_dev, int32_t R,
                               const double* tau, const double* lambda, const double* lamw_dev,
                               const fsqr_options* opt, cudaStream_t st) {
  // ---------------- validation
  ctx->alloc_st = st;
  if (!X || !y_dev || !tau || !lambda) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  if (R < 1 || R > FSQR_MAXR) return set_err(ctx, FSQR_ERR_CONFIG, "n_rhs=%d not in [1,%d]", R, FSQR_MAXR);
  if (X->storage < 0 || X->storage > 2) return set_err(ctx, FSQR_ERR_CONFIG, "bad storage %d", X->storage);
  if (X->n < 2 || X->n > 65536) return set_err(ctx, FSQR_ERR_CONFIG, "n=%lld not in [2,65536]", (long long)X->n);
  if (X->p < 1 || X->p > 2147483647LL) return set_err(ctx, FSQR_ERR_CONFIG, "p=%lld out of range", (long long)X->p);
  if (!X->data_dev) return set_err(ctx, FSQR_ERR_CONFIG, "data_dev is NULL");
  if ((X->mean_dev == nullptr) != (X->scale_dev == nullptr))
    return set_err(ctx, FSQR_ERR_CONFIG, "mean_dev and scale_dev must be given together");
  const int64_t minld = X->storage == 2 ? (X->n + 3) / 4 : X->n;
  const int align = X->storage == 0 ? 4 : 16;
  if (X->ld < minld || X->ld % align) return set_err(ctx, FSQR_ERR_CONFIG, "ld=%lld invalid (min %lld, multiple of %d)",
                                                     (long long)X->ld, (long long)minld, align);
  if (((uintptr_t)X->data_dev) % 16) return set_err(ctx, FSQR_ERR_CONFIG, "data_dev must be 16-byte aligned");
  if (X->flags & ~FSQR_DESIGN_PACK2) return set_err(ctx, FSQR_ERR_CONFIG, "unknown design flags 0x%x", X->flags);
  fsqr_design Xpk;
  if (X->flags & FSQR_DESIGN_PACK2) {
    // owned 2-bit copy of the u8 codes; everything below sees PACKED2 storage
    if (X->storage != FSQR_U8) return set_err(ctx, FSQR_ERR_CONFIG, "FSQR_DESIGN_PACK2 needs U8 storage");
    // column stride a multiple of 128 bytes: every TMA box row of K2 and every 512-byte row-slab
    // segment of the forward product is then one aligned line run (no straddled sectors); K2's
    // tensor map still ends at round_up(n/4, 16), so the padding is never streamed
    const int64_t ld2 = pack2_ld(X->n);
    uint8_t* x2;
    int* bad2;
    AL(x2, ld2 * X->p);
    AL(bad2, 1);
    launch_pack2((const uint8_t*)X->data_dev, X->ld, (int)X->n, X->p, x2, ld2, bad2, st);
    CK(cudaGetLastError());
    int h_bad = 0;
    CK(cudaMemcpyAsync(&h_bad, bad2, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h_bad) return set_err(ctx, FSQR_ERR_DATA, "FSQR_DESIGN_PACK2: a genotype code exceeds 3");
    Xpk = *X;
    Xpk.storage = FSQR_PACKED2;
    Xpk.flags = 0;
    Xpk.data_dev = x2;
    Xpk.ld = ld2;
    X = &Xpk;
  }
  fsqr_options o;
  if (opt) o = *opt; else fsqr_default_options(&o);
  if (o.mu == 0.0) o.mu = 2.0 / (double)X->n;   // DESIGN.md reading R2
  if (!(o.mu > 0.0)) return set_err(ctx, FSQR_ERR_CONFIG, "mu must be > 0");
  if (o.G < 1 || (int64_t)o.G > X->p + 1) return set_err(ctx, FSQR_ERR_CONFIG, "G=%d not in [1, p+1]", o.G);
  if (!(o.eta_safety > 1.0) && !o.eta_host) return set_err(ctx, FSQR_ERR_CONFIG, "eta_safety must be > 1");
  if (o.max_iter < 0 || o.power_max_iter < 1 || o.trace_cap < 1) return set_err(ctx, FSQR_ERR_CONFIG, "bad iteration caps");
  if (o.eta_method != FSQR_ETA_LANCZOS && o.eta_method != FSQR_ETA_POWER)
    return set_err(ctx, FSQR_ERR_CONFIG, "eta_method %d unknown", o.eta_method);
  for (int r = 0; r < R; ++r) {
    if (!(tau[r] > 0.0 && tau[r] < 1.0)) return set_err(ctx, FSQR_ERR_CONFIG, "tau[%d]=%g not in (0,1)", r, tau[r]);
    if (!(lambda[r] >= 0.0) || !std::isfinite(lambda[r])) return set_err(ctx, FSQR_ERR_CONFIG, "lambda[%d]=%g invalid", r, lambda[r]);
  }
  if (o.eta_host)
    for (int g = 0; g < o.G; ++g)
      if (!(o.eta_host[g] > 0.0)) return set_err(ctx, FSQR_ERR_CONFIG, "eta[%d] must be > 0", g);
  int dev;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return set_err(ctx, FSQR_ERR_CUDA, "device %s is sm_%d%d; this library targets sm_100a",
                                       prop.name, prop.major, prop.minor);
  ctx->sms = prop.multiProcessorCount;
  ctx->opt = o;
  ctx->R = R;
  ctx->n = X->n;
  ctx->p = X->p;
  ctx->tau.assign(tau, tau + R);
  ctx->lambda.assign(lambda, lambda + R);
  CK(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
  CK(cudaEventCreate(&ctx->ev0));
  CK(cudaEventCreate(&ctx->ev1));
  CK(cudaMallocHost(&ctx->h_pin, 4096));

  Dev& D = ctx->D;
  D.n = (int)X->n;
  D.p = X->p;
  D.ld = X->ld;
  D.R = R;
  D.G = o.G;
  D.storage = X->storage;
  D.gq = (X->p + 1) / o.G;
  D.grem = (X->p + 1) % o.G;
  D.npad = ((4 * R + 15) / 16) * 16;
  if (const char* ev = getenv("FSQR_PDL")) g_fsqr_pdl = atoi(ev) != 0;
  D.k1_policy = 0;
  D.x_policy = 0;
  if (const char* ev = getenv("FSQR_X_POLICY")) D.x_policy = atoi(ev);
  if (const char* ev = getenv("FSQR_K1_POLICY")) D.k1_policy = atoi(ev);
  D.k1_esmax = 65536;
  if (const char* ev = getenv("FSQR_K1_ESMAX")) D.k1_esmax = std::max(32, std::min(65536, atoi(ev) / 32 * 32));
  D.ldk = (int)(((X->n + 127) / 128) * 128);
  D.X8 = X->storage != 0 ? (const uint8_t*)X->data_dev : nullptr;
  D.Xf = X->storage == 0 ? (const float*)X->data_dev : nullptr;
  D.mu = o.mu;
  D.sigma = o.mu / (double)(o.G + 1);
  D.tol = o.tol;
  D.max_iter = o.max_iter;
  D.trace_cap = o.trace_cap;
  D.max_iter_point = o.max_iter_point;
  const int64_t p1 = X->p + 1;
  const size_t nR = (size_t)R * X->n;

  // backend
  ctx->backend = FSQR_BACKEND_SIMT;
  if (X->storage != FSQR_F32_DENSE && k2_tc_supported(D.npad) && o.backend != FSQR_BACKEND_SIMT)
    ctx->backend = FSQR_BACKEND_TC;
  if (o.backend == FSQR_BACKEND_TC && ctx->backend != FSQR_BACKEND_TC)
    return set_err(ctx, FSQR_ERR_CONFIG, "tcgen05 backend needs U8 or PACKED2 storage and n_rhs <= 16");
  if (ctx->backend == FSQR_BACKEND_TC && X->storage == FSQR_PACKED2) {
    // 2-bit tensor-core kernel: 512-sample K blocks, theta digits in its K order
    D.ldk = (int)(((X->n + 511) / 512) * 512);
    D.bperm = 1;
  }
  if (ctx->backend == FSQR_BACKEND_TC) {
    CK(k2_tc_init());
    CK(k2_tc2_init());
    ctx->k2_grid = (int)std::min<int64_t>((X->p + 127) / 128, ctx->sms);
  } else {
    ctx->k2_grid = ctx->sms * 8;
  }
  ctx->k1_grid = ctx->sms;   // k1_bulk scales by its resident CTAs per SM; k1_tcp runs one CTA per SM
  CK(k1_init());
  // forward-product kernel: k1_tcp (tensor cores, A tile built on chip from per-lane cp.async) for
  // genotype storage -- 2-bit M 53 -> 29 us and C4 210 -> 104 us against the CUDA-core k1_bulk,
  // u8 C2 3 RHS 31 -> 14 us and C5 9 RHS 18.5 -> 14.4 us against a TMA gather4 kernel (round 1,
  // since removed).  FSQR_K1=bulk selects k1_bulk (the bitwise cross-check of the tests).
  D.k1_tc = 0;
  if (ctx->backend == FSQR_BACKEND_TC && X->storage == FSQR_U8) D.k1_tc = 4;
  if (ctx->backend == FSQR_BACKEND_TC && X->storage == FSQR_PACKED2) D.k1_tc = 3;
  if (const char* ev = getenv("FSQR_K1"))
    if (!strcmp(ev, "bulk")) D.k1_tc = 0;
  if (D.k1_tc == 3 || D.k1_tc == 4) CK(k1_tcp_init());

  // ---------------- allocations
  // Everything the n-vector step and the per-iteration control touch (n-vectors, theta digits,
  // finalize records, scalars, tickets) lives in ONE arena: measured on the B200, the first
  // accesses of the tail to a dozen separate small allocations right after the 2.5 GB X stream
  // stalled up to 8 us (address-translation misses); one contiguous block needs few translations.
  int32_t* colsum;
  double *mean, *inv_sd, *sd, *eta_d, *inv_eta_d, *y, *tau_d, *lam_cur;
  AL(colsum, X->p);
  AL(mean, X->p);
  AL(inv_sd, X->p);
  AL(sd, X->p);
  {
    std::vector<std::pair<void**, size_t>> req;
    auto add = [&](auto** ptr, size_t count) { req.push_back({(void**)ptr, count * sizeof(**ptr)}); };
    add(&y, X->n);
    add(&D.z, nR);
    add(&D.theta, nR);
    add(&D.rres, nR);
    add(&D.s, nR);
    add(&D.sdense, nR);
    add(&D.sacc, nR);
    add(&D.Bq, (size_t)D.npad * D.ldk);
    add(&D.fpart, (size_t)FIN_MAXGRID * R * FSQR_FPART);
    add(&D.ftsum, (size_t)FIN_MAXGRID * R);
    add(&D.k2part, (size_t)std::max(ctx->k2_grid, ctx->sms * 8) * R * FSQR_NPART);
    add(&eta_d, o.G);
    add(&inv_eta_d, o.G);
    add(&tau_d, R);
    add(&lam_cur, R);
    add(&D.lam2, R);
    add(&D.use_w, 1);
    add(&D.Tsum, R);
    add(&D.delta, R);
    add(&D.sumth, R);
    add(&D.sup_cnt, 2);
    add(&D.cmax, 2 * R);
    add(&D.mterm, R);
    add(&D.k1bar, 1);
    add(&D.ticket, 1);
    add(&D.kbase, 1);
    add(&D.fticket, 1 + FSQR_MAXR);
    add(&D.scal, R * FSQR_NSCAL);
    add(&D.status, R);
    add(&D.commit_iter, R);
    add(&D.iter, 1);
    add(&D.stop, 1);
    add(&D.lastR, R * FSQR_TRACE_W);
    add(&D.t_idx, R);
    add(&D.pt_iters, R);
    size_t total = 0;
    for (auto& q : req) total += (q.second + 255) / 256 * 256;
    uint8_t* arena;
    AL(arena, total);
    for (auto& q : req) {
      *q.first = arena;
      arena += (q.second + 255) / 256 * 256;
    }
  }
  D.colsum = colsum;
  D.mean = mean;
  D.inv_sd = inv_sd;
  D.eta = eta_d;
  D.inv_eta = inv_eta_d;
  D.y = y;
  D.tau = tau_d;
  D.lam_cur = lam_cur;
  // penalty weights: ctx-owned [(p+1)][R]; the caller's [p+1] vector (if any) is broadcast to every RHS
  AL(D.lamw, p1 * R);
  if (lamw_dev) {
    for (int r = 0; r < R; ++r)
      CK(cudaMemcpy2DAsync(D.lamw + r, sizeof(double) * R, lamw_dev, sizeof(double), sizeof(double), p1,
                           cudaMemcpyDeviceToDevice, st));
    const int one = 1;
    CK(cudaMemcpyAsync(D.use_w, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  CK(cudaMemcpyAsync(y, y_dev, sizeof(double) * X->n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(tau_d, tau, sizeof(double) * R, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(lam_cur, lambda, sizeof(double) * R, cudaMemcpyHostToDevice, st));
  AL(D.beta[0], p1 * R);
  AL(D.beta[1], p1 * R);
  for (int b = 0; b < 2; ++b) {
    // padded by 16 entries: the forward kernels copy metadata blocks in 16-byte units
    AL(D.sup_idx[b], X->p + 16);
    AL(D.sup_cs[b], X->p + 16);
    AL(D.sup_c[b], (size_t)(X->p + 16) * R);
    AL(D.sup_b[b], (size_t)X->p * R);
  }
  AL(D.tstamp, FSQR_TSTAMPS);
  AL(D.trace, (size_t)o.trace_cap * R * FSQR_TRACE_W);

  // ---------------- a0: column statistics
  int* bad;
  AL(bad, 1);
  if (X->mean_dev) {
    CK(cudaMemcpyAsync(mean, X->mean_dev, sizeof(double) * X->p, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(sd, X->scale_dev, sizeof(double) * X->p, cudaMemcpyDeviceToDevice, st));
  }
  {
    const int big = 0x7fffffff;
    CK(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    int32_t* cs_tmp = colsum;
    double *m_tmp = mean, *sd_tmp = sd, *isd_tmp = inv_sd;
    if (X->mean_dev) {  // still need exact colsum for genotype storage; recompute into scratch
      AL(m_tmp, X->p);
      AL(sd_tmp, X->p);
      AL(isd_tmp, X->p);
    }
    launch_colstats(D, cs_tmp, m_tmp, isd_tmp, sd_tmp, bad, st);
    CK(cudaGetLastError());
    int h_bad = 0;
    CK(cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!X->mean_dev && h_bad != big)
      return set_err(ctx, FSQR_ERR_DATA, "zero-variance column %d (stored column index)", h_bad);
    if (X->mean_dev) {
      // caller-supplied scale: inv_sd = 1/scale
      std::vector<double> hs(X->p);
      CK(cudaMemcpy(hs.data(), sd, sizeof(double) * X->p, cudaMemcpyDeviceToHost));
      for (int64_t c = 0; c < X->p; ++c) {
        if (!(hs[c] > 0.0)) return set_err(ctx, FSQR_ERR_DATA, "scale[%lld] must be > 0", (long long)c);
        hs[c] = 1.0 / hs[c];
      }
      CK(cudaMemcpy(inv_sd, hs.data(), sizeof(double) * X->p, cudaMemcpyHostToDevice));
    }
  }
  // y must be finite
  {
    std::vector<double> hy(X->n);
    CK(cudaMemcpy(hy.data(), y, sizeof(double) * X->n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < X->n; ++i)
      if (!std::isfinite(hy[i])) return set_err(ctx, FSQR_ERR_DATA, "y[%lld] is not finite", (long long)i);
  }

  if (ctx->backend == FSQR_BACKEND_TC) {   // (the power method's tensor-core back pass streams X through tmX)
    fsqr_status s = make_tmaps(ctx);
    if (s != FSQR_OK) return s;
  }
  // ---------------- a0': eta_g
  if (o.eta_host) {
    ctx->eta.assign(o.eta_host, o.eta_host + o.G);
  } else {
    fsqr_status s = power_method(ctx, st);
    if (s != FSQR_OK) return s;
  }
  CK(cudaMemcpyAsync(eta_d, ctx->eta.data(), sizeof(double) * o.G, cudaMemcpyHostToDevice, st));
  ctx->inv_eta.resize(o.G);
  for (int g = 0; g < o.G; ++g) ctx->inv_eta[g] = 1.0 / ctx->eta[g];
  CK(cudaMemcpyAsync(inv_eta_d, ctx->inv_eta.data(), sizeof(double) * o.G, cudaMemcpyHostToDevice, st));

  // ---------------- lambda_max per tau
  {
    fsqr_status s = lambda_max(ctx, st);
    if (s != FSQR_OK) return s;
  }

  // ---------------- cold start: beta = 0, z = y, theta = 0
  for (int r = 0; r < R; ++r) CK(cudaMemcpyAsync(D.z + (size_t)r * X->n, y, sizeof(double) * X->n, cudaMemcpyDeviceToDevice, st));
  {
    std::vector<double> one(R, 1.0);
    CK(cudaMemcpyAsync(D.delta, one.data(), sizeof(double) * R, cudaMemcpyHostToDevice, st));
  }
  {
    fsqr_status s = init_state(ctx, st);
    if (s != FSQR_OK) return s;
  }

  // ---------------- per-mode kernel parameter blocks and graph chunk size
  for (int m = 0; m < M_COUNT; ++m) {
    ctx->mode_dev[m] = D;
    ctx->mode_dev[m].update = m == M_KKT ? 0 : 1;
    ctx->mode_dev[m].check = m == M_SOLVE ? 1 : 0;
    ctx->mode_dev[m].path = m == M_PATH ? 1 : 0;
  }
  const double xbytes = (double)X->ld * (double)X->p * (X->storage == 0 ? 4.0 : 1.0);
  const double est = xbytes / 5.0e12 + 25e-6;
  ctx->chunk = (int)std::max(1.0, std::min(128.0, std::floor(0.02 / est)));
  return FSQR_OK;
}

fsqr_status fsqr_create(const fsqr_design* X, const double* y_dev, int32_t n_rhs, const double* tau_host,
                        const double* lambda_host, const double* lambda_w_dev, const fsqr_options* opt, void* stream,
                        fsqr_ctx** out) {
  if (!out) return set_err(nullptr, FSQR_ERR_CONFIG, "out is NULL");
  *out = nullptr;
  fsqr_ctx* ctx = new fsqr_ctx();
  fsqr_status s = create_impl(ctx, X, y_dev, n_rhs, tau_host, lambda_host, lambda_w_dev, opt, (cudaStream_t)stream);
  if (s != FSQR_OK) {
    g_err = ctx->err;
    fsqr_destroy(ctx);
    return s;
  }
  *out = ctx;
  return FSQR_OK;
}

fsqr_status fsqr_iterate(fsqr_ctx* ctx, int64_t k, void* stream) {
  if (!ctx) return set_err(nullptr, FSQR_ERR_CONFIG, "ctx is NULL");
  if (k < 0) return set_err(ctx, FSQR_ERR_CONFIG, "k < 0");
  cudaStream_t st = (cudaStream_t)stream;
  {
    fsqr_status s = reset_control(ctx, st);
    if (s != FSQR_OK) return s;
  }
  int64_t done = 0;
  while (k - done >= ctx->chunk) {
    fsqr_status s = run_chunk(ctx, M_ITER, st);
    if (s != FSQR_OK) return s;
    done += ctx->chunk;
  }
  for (; done < k; ++done) enqueue_iteration(ctx, ctx->mode_dev[M_ITER], st);
  CK(cudaGetLastError());
  return FSQR_OK;
}

static fsqr_status collect(fsqr_ctx* ctx, fsqr_result* out, int64_t it0, cudaStream_t st, float ms) {
  std::vector<int> status(ctx->R);
  std::vector<double> lr((size_t)ctx->R * FSQR_TRACE_W);
  long long it = 0;
  CK(cudaMemcpyAsync(status.data(), ctx->D.status, sizeof(int) * ctx->R, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(lr.data(), ctx->D.lastR, sizeof(double) * lr.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&it, ctx->D.iter, sizeof it, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  fsqr_status ret = FSQR_OK;
  if (out) {
    memset(out, 0, sizeof *out);
    out->iterations = it - it0;
    out->total_iterations = it;
    out->n_rhs = ctx->R;
    out->wall_ms = ms;
  }
  for (int r = 0; r < ctx->R; ++r) {
    int s = status[r] == ST_CONVERGED ? 0 : (status[r] == ST_NUMERIC ? -3 : 2);
    if (s == -3) ret = FSQR_ERR_NUMERIC;
    else if (s == 2 && ret == FSQR_OK) ret = FSQR_NOT_CONVERGED;
    if (out) {
      out->status[r] = s;
      for (int q = 0; q < 3; ++q) out->R[r][q] = lr[r * FSQR_TRACE_W + q];
      out->objective[r] = lr[r * FSQR_TRACE_W + 3];
    }
  }
  if (ret == FSQR_ERR_NUMERIC) set_err(ctx, ret, "non-finite value in the iteration state");
  return ret;
}

static fsqr_status drive(fsqr_ctx* ctx, int mode, cudaStream_t st, int64_t* it0_out, float* ms_out) {
  long long it0 = 0;
  CK(cudaMemcpyAsync(&it0, ctx->D.iter, sizeof it0, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *it0_out = it0;
  CK(cudaEventRecord(ctx->ev0, st));
  int* hstop = (int*)ctx->h_pin;
  const int64_t guard = (mode == M_PATH ? (int64_t)1 << 40 : ctx->opt.max_iter) + 2LL * ctx->chunk + 2;
  int64_t launched = 0;
  for (;;) {
    fsqr_status s = run_chunk(ctx, mode, st);
    if (s != FSQR_OK) return s;
    launched += ctx->chunk;
    CK(cudaMemcpyAsync(hstop, ctx->D.stop, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*hstop) break;
    if (launched > guard) break;
  }
  CK(cudaEventRecord(ctx->ev1, st));
  CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  *ms_out = ms;
  return FSQR_OK;
}

fsqr_status fsqr_solve(fsqr_ctx* ctx, fsqr_result* out, void* stream) {
  if (!ctx) return set_err(nullptr, FSQR_ERR_CONFIG, "ctx is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  fsqr_status s = reset_control(ctx, st);
  if (s != FSQR_OK) return s;
  int64_t it0;
  float ms;
  s = drive(ctx, M_SOLVE, st, &it0, &ms);
  if (s != FSQR_OK) return s;
  return collect(ctx, out, it0, st, ms);
}

fsqr_status fsqr_objective(fsqr_ctx* ctx, double* obj_host, void* stream) {
  if (!ctx || !obj_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  double* pen = nullptr;
  CK(cudaMallocAsync(&pen, sizeof(double) * 2 * ctx->R, st));
  launch_commit_stats(ctx->D, pen, nullptr, 0, st);
  CK(cudaGetLastError());
  std::vector<double> hp(ctx->R), sc((size_t)ctx->R * FSQR_NSCAL);
  CK(cudaMemcpyAsync(hp.data(), pen, sizeof(double) * ctx->R, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(sc.data(), ctx->D.scal, sizeof(double) * sc.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(pen, st));
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r < ctx->R; ++r) obj_host[r] = sc[r * FSQR_NSCAL + 2] / (double)ctx->n + hp[r];
  return FSQR_OK;
}

fsqr_status fsqr_hbic(fsqr_ctx* ctx, double* hbic_host, void* stream) {
  if (!ctx || !hbic_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  double* pen = nullptr;
  CK(cudaMallocAsync(&pen, sizeof(double) * 2 * ctx->R, st));
  launch_commit_stats(ctx->D, pen, nullptr, 0, st);
  CK(cudaGetLastError());
  std::vector<double> hp(2 * ctx->R), sc((size_t)ctx->R * FSQR_NSCAL);
  CK(cudaMemcpyAsync(hp.data(), pen, sizeof(double) * 2 * ctx->R, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(sc.data(), ctx->D.scal, sizeof(double) * sc.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(pen, st));
  CK(cudaStreamSynchronize(st));
  const double n = (double)ctx->n, p = (double)ctx->p;
  for (int r = 0; r < ctx->R; ++r)
    hbic_host[r] = std::log(sc[r * FSQR_NSCAL + 2]) + hp[ctx->R + r] * (std::log(std::log(n)) / n) * std::log(p);
  return FSQR_OK;
}

fsqr_status fsqr_set_lambda_weights(fsqr_ctx* ctx, const double* w_host, void* stream) {
  if (!ctx) return set_err(nullptr, FSQR_ERR_CONFIG, "ctx is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const int R = ctx->R;
  const int64_t p1 = ctx->p + 1;
  int flag = 0;
  if (w_host) {
    std::vector<double> t((size_t)p1 * R);
    for (int r = 0; r < R; ++r)
      for (int64_t j = 0; j < p1; ++j) {
        const double w = w_host[(size_t)r * p1 + j];
        if (!(w >= 0.0) || !std::isfinite(w))
          return set_err(ctx, FSQR_ERR_CONFIG, "weight[%d][%lld]=%g invalid", r, (long long)j, w);
        t[(size_t)j * R + r] = w;
      }
    CK(cudaMemcpyAsync(ctx->D.lamw, t.data(), sizeof(double) * t.size(), cudaMemcpyHostToDevice, st));
    flag = 1;
  }
  CK(cudaMemcpyAsync(ctx->D.use_w, &flag, sizeof(int), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return FSQR_OK;
}

fsqr_status fsqr_set_lambda2(fsqr_ctx* ctx, const double* lam2_host) {
  if (!ctx || !lam2_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  SYNC_DEVICE();
  for (int r = 0; r < ctx->R; ++r)
    if (!(lam2_host[r] >= 0.0) || !std::isfinite(lam2_host[r]))
      return set_err(ctx, FSQR_ERR_CONFIG, "lambda2[%d]=%g invalid", r, lam2_host[r]);
  CK(cudaMemcpy(ctx->D.lam2, lam2_host, sizeof(double) * ctx->R, cudaMemcpyHostToDevice));
  return FSQR_OK;
}

fsqr_status fsqr_lla(fsqr_ctx* ctx, int32_t penalty, double a, int32_t L, int64_t* stage_iters_host,
                     fsqr_result* out, void* stream) {
  if (!ctx) return set_err(nullptr, FSQR_ERR_CONFIG, "ctx is NULL");
  if (penalty != FSQR_SCAD && penalty != FSQR_MCP) return set_err(ctx, FSQR_ERR_CONFIG, "penalty %d unknown", penalty);
  if (penalty == FSQR_SCAD && !(a > 2.0)) return set_err(ctx, FSQR_ERR_CONFIG, "SCAD needs a > 2 (E16)");
  if (penalty == FSQR_MCP && !(a > 1.0)) return set_err(ctx, FSQR_ERR_CONFIG, "MCP needs a > 1 (E17)");
  if (L < 0) return set_err(ctx, FSQR_ERR_CONFIG, "L must be >= 0");
  for (int r = 0; r < ctx->R; ++r)
    if (!(ctx->lambda[r] > 0.0)) return set_err(ctx, FSQR_ERR_CONFIG, "LLA needs lambda > 0 (rhs %d)", r);
  cudaStream_t st = (cudaStream_t)stream;
  fsqr_result res{};
  fsqr_status last = FSQR_OK;
  for (int l = 0; l <= L; ++l) {
    if (l > 0) {
      // lambda~_j = p'_lambda(|beta~_j^{l-1}|) from the committed stage-(l-1) solution
      launch_lla_weights(ctx->D, penalty, a, st);
      CK(cudaGetLastError());
      const int one = 1;
      CK(cudaMemcpyAsync(ctx->D.use_w, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    }
    last = fsqr_solve(ctx, &res, stream);
    if (last < 0) return last;
    if (stage_iters_host) stage_iters_host[l] = res.iterations;
  }
  if (out) *out = res;
  return last;
}

fsqr_status fsqr_pivotal(fsqr_ctx* ctx, int32_t rhs, int64_t B, uint64_t seed, double* Lambda_host, void* stream) {
  if (!ctx || !Lambda_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  if (rhs < 0 || rhs >= ctx->R) return set_err(ctx, FSQR_ERR_CONFIG, "rhs %d out of range", rhs);
  if (B < 1) return set_err(ctx, FSQR_ERR_CONFIG, "B must be >= 1");
  if (ctx->D.storage != FSQR_U8 && ctx->D.storage != FSQR_PACKED2)
    return set_err(ctx, FSQR_ERR_CONFIG, "the pivotal statistic needs genotype storage");
  cudaStream_t st = (cudaStream_t)stream;
  const int ldk = (int)(((ctx->n + 127) / 128) * 128);
  const bool packed = ctx->D.storage == FSQR_PACKED2;
  ctx->alloc_st = st;
  if (!ctx->piv_draws) {
    AL(ctx->piv_draws, (size_t)128 * ldk);
    AL(ctx->piv_nb, 128);
    AL(ctx->piv_lmax, 128);
    CK(pivotal_init());
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return set_err(ctx, FSQR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    EncodeTiledFn enc = (EncodeTiledFn)fn;
    cuuint32_t es[2] = {1, 1};
    {
      cuuint64_t dims[2] = {(cuuint64_t)ldk, 128};
      cuuint64_t strides[1] = {(cuuint64_t)ldk};
      cuuint32_t box[2] = {128, 128};
      CUresult r = enc(&ctx->tmPivA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)ctx->piv_draws, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return set_err(ctx, FSQR_ERR_CUDA, "tensor map for the draws failed (%d)", (int)r);
    }
    ctx->piv_enc = fn;
  }
  // X as u8 tiles of 256 columns x 128 samples.  A 2-bit design is unpacked into a temporary u8
  // copy for the duration of the call (the statistic is a one-off tuning step, not the hot loop).
  const uint8_t* x8 = ctx->D.X8;
  int64_t ld8 = ctx->D.ld;
  uint8_t* tmp = nullptr;
  struct TmpFree {   // the temporary copy goes on every exit path
    uint8_t** p;
    cudaStream_t s;
    ~TmpFree() {
      if (*p) {
        cudaFreeAsync(*p, s);
        cudaStreamSynchronize(s);
      }
    }
  } tmp_guard{&tmp, st};
  if (packed) {
    ld8 = (ctx->n + 15) / 16 * 16;
    CK(cudaMallocAsync((void**)&tmp, (size_t)ld8 * ctx->p, st));
    launch_unpack2(ctx->D.X8, ctx->D.ld, ctx->p, tmp, ld8, st);
    CK(cudaGetLastError());
    x8 = tmp;
  }
  if (packed || !ctx->piv_x_ready) {
    cuuint32_t es[2] = {1, 1};
    cuuint64_t dims[2] = {(cuuint64_t)ctx->n, (cuuint64_t)ctx->p};
    cuuint64_t strides[1] = {(cuuint64_t)ld8};
    cuuint32_t box[2] = {128, 256};
    CUresult r = ((EncodeTiledFn)ctx->piv_enc)(&ctx->tmPivX, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)x8, dims, strides,
                                               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(ctx, FSQR_ERR_CUDA, "tensor map for X (256 rows) failed (%d)", (int)r);
    ctx->piv_x_ready = !packed;
  }
  const int grid = (int)std::min<int64_t>((ctx->p + 255) / 256, ctx->sms);
  std::vector<unsigned long long> h(128);
  for (int64_t b0 = 0; b0 < B; b0 += 128) {
    launch_piv_draws((int)ctx->n, ldk, ctx->tau[rhs], seed, (long long)b0, ctx->piv_draws, ctx->piv_nb, st);
    CK(cudaMemsetAsync(ctx->piv_lmax, 0, sizeof(unsigned long long) * 128, st));
    launch_pivotal(ctx->D, &ctx->tmPivA, &ctx->tmPivX, ctx->piv_nb, ctx->piv_lmax, grid, st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h.data(), ctx->piv_lmax, sizeof(unsigned long long) * 128, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int64_t q = 0; q < 128 && b0 + q < B; ++q) {
      double v;
      memcpy(&v, &h[q], sizeof v);
      Lambda_host[b0 + q] = v;
    }
  }
  return FSQR_OK;
}

fsqr_status fsqr_kkt(fsqr_ctx* ctx, double* R_host, void* stream) {
  if (!ctx || !R_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  launch_unfreeze(ctx->D, st);
  // K2 in diagnostic mode: every RHS at its committed state, no state change
  Dev D = ctx->mode_dev[M_KKT];
  std::vector<int> status(ctx->R);
  CK(cudaMemcpyAsync(status.data(), ctx->D.status, sizeof(int) * ctx->R, cudaMemcpyDeviceToHost, st));
  CK(cudaMemsetAsync(ctx->D.status, 0, sizeof(int) * ctx->R, st));
  CK(cudaMemsetAsync(ctx->D.stop, 0, sizeof(int), st));
  launch_k2(ctx, D, st);
  CK(cudaGetLastError());
  std::vector<double> lr((size_t)ctx->R * FSQR_TRACE_W);
  CK(cudaMemcpyAsync(lr.data(), ctx->D.lastR, sizeof(double) * lr.size(), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(ctx->D.status, status.data(), sizeof(int) * ctx->R, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r < ctx->R; ++r)
    for (int q = 0; q < 3; ++q) R_host[r * 3 + q] = lr[r * FSQR_TRACE_W + q];
  return FSQR_OK;
}

fsqr_status fsqr_get_beta(fsqr_ctx* ctx, double* beta_host, int32_t scale, void* stream) {
  if (!ctx || !beta_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  double* tmp = nullptr;
  const size_t cnt = (size_t)ctx->R * (ctx->p + 1);
  CK(cudaMallocAsync(&tmp, sizeof(double) * cnt, st));
  launch_commit_stats(ctx->D, nullptr, tmp, scale ? 1 : 0, st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(beta_host, tmp, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(tmp, st));
  CK(cudaStreamSynchronize(st));
  return FSQR_OK;
}

fsqr_status fsqr_get_state(fsqr_ctx* ctx, double* beta_host, double* z_host, double* theta_host, void* stream) {
  if (!ctx) return set_err(nullptr, FSQR_ERR_CONFIG, "ctx is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  if (beta_host) {
    fsqr_status s = fsqr_get_beta(ctx, beta_host, 0, stream);
    if (s != FSQR_OK) return s;
  }
  const size_t nR = (size_t)ctx->R * ctx->n;
  if (z_host) CK(cudaMemcpyAsync(z_host, ctx->D.z, sizeof(double) * nR, cudaMemcpyDeviceToHost, st));
  if (theta_host) CK(cudaMemcpyAsync(theta_host, ctx->D.theta, sizeof(double) * nR, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return FSQR_OK;
}

fsqr_status fsqr_set_state(fsqr_ctx* ctx, const double* beta_host, const double* z_host, const double* theta_host,
                           void* stream) {
  if (!ctx || !beta_host || !z_host || !theta_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int R = ctx->R;
  const int64_t p1 = ctx->p + 1;
  std::vector<double> bt((size_t)p1 * R);
  for (int r = 0; r < R; ++r)
    for (int64_t j = 0; j < p1; ++j) {
      const double b = beta_host[(size_t)r * p1 + j];
      if (!std::isfinite(b)) return set_err(ctx, FSQR_ERR_DATA, "beta not finite");
      bt[(size_t)j * R + r] = b;
    }
  const size_t nR0 = (size_t)R * ctx->n;
  for (size_t i = 0; i < nR0; ++i)
    if (!std::isfinite(z_host[i]) || !std::isfinite(theta_host[i]))
      return set_err(ctx, FSQR_ERR_DATA, "z or theta not finite at %zu", i);
  // everything on the caller's stream, in order after any work still queued there
  CK(cudaMemcpyAsync(ctx->D.beta[0], bt.data(), sizeof(double) * bt.size(), cudaMemcpyHostToDevice, st));
  const size_t nR = (size_t)R * ctx->n;
  CK(cudaMemcpyAsync(ctx->D.z, z_host, sizeof(double) * nR, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(ctx->D.theta, theta_host, sizeof(double) * nR, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(ctx->D.iter, 0, sizeof(long long), st));
  CK(cudaMemsetAsync(ctx->D.status, 0, sizeof(int) * R, st));
  CK(cudaMemsetAsync(ctx->D.commit_iter, 0, sizeof(long long) * R, st));
  return init_state(ctx, st);   // synchronises st before bt goes out of scope
}

fsqr_status fsqr_set_lambda(fsqr_ctx* ctx, const double* lambda_host) {
  if (!ctx || !lambda_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  SYNC_DEVICE();
  for (int r = 0; r < ctx->R; ++r)
    if (!(lambda_host[r] >= 0.0) || !std::isfinite(lambda_host[r]))
      return set_err(ctx, FSQR_ERR_CONFIG, "lambda[%d] invalid", r);
  ctx->lambda.assign(lambda_host, lambda_host + ctx->R);
  CK(cudaMemcpy(ctx->D.lam_cur, lambda_host, sizeof(double) * ctx->R, cudaMemcpyHostToDevice));
  return FSQR_OK;
}

fsqr_status fsqr_set_tolerance(fsqr_ctx* ctx, double tol, int64_t max_iter) {
  if (!ctx) return set_err(nullptr, FSQR_ERR_CONFIG, "ctx is NULL");
  if (!(tol > 0.0) || !std::isfinite(tol) || max_iter < 0)
    return set_err(ctx, FSQR_ERR_CONFIG, "need tol > 0 and max_iter >= 0");
  SYNC_DEVICE();
  ctx->opt.tol = tol;
  ctx->opt.max_iter = max_iter;
  ctx->D.tol = tol;
  ctx->D.max_iter = max_iter;
  for (int m = 0; m < M_COUNT; ++m) {   // the captured graphs bake the kernel parameters
    ctx->mode_dev[m].tol = tol;
    ctx->mode_dev[m].max_iter = max_iter;
    if (ctx->graph[m].exec) {
      cudaGraphExecDestroy(ctx->graph[m].exec);
      ctx->graph[m].exec = nullptr;
    }
  }
  return FSQR_OK;
}

fsqr_status fsqr_debug_stamps(fsqr_ctx* ctx, uint64_t* out_host, int64_t n) {
  if (!ctx || !out_host || n < 0) return set_err(ctx, FSQR_ERR_CONFIG, "bad arguments");
  SYNC_DEVICE();
  CK(cudaMemcpy(out_host, ctx->D.tstamp, sizeof(uint64_t) * (size_t)std::min<int64_t>(n, FSQR_TSTAMPS),
                cudaMemcpyDeviceToHost));
  return FSQR_OK;
}

int32_t fsqr_launches_per_iteration(const fsqr_ctx* ctx) {
  if (!ctx) return -1;
  return k1_fuses_finalize(ctx->mode_dev[M_ITER]) ? 2 : 3;
}

fsqr_status fsqr_lambda_max(const fsqr_ctx* ctx, double* out_host) {
  if (!ctx || !out_host) return set_err(nullptr, FSQR_ERR_CONFIG, "null argument");
  for (int r = 0; r < ctx->R; ++r) out_host[r] = ctx->lambda_max[r];
  return FSQR_OK;
}

fsqr_status fsqr_get_eta(const fsqr_ctx* ctx, double* eta_host) {
  if (!ctx || !eta_host) return set_err(nullptr, FSQR_ERR_CONFIG, "null argument");
  for (size_t g = 0; g < ctx->eta.size(); ++g) eta_host[g] = ctx->eta[g];
  return FSQR_OK;
}

fsqr_status fsqr_get_colstats(fsqr_ctx* ctx, double* mean_host, double* sd_host) {
  if (!ctx) return set_err(nullptr, FSQR_ERR_CONFIG, "ctx is NULL");
  SYNC_DEVICE();
  if (mean_host) CK(cudaMemcpy(mean_host, ctx->D.mean, sizeof(double) * ctx->p, cudaMemcpyDeviceToHost));
  if (sd_host) {
    std::vector<double> isd(ctx->p);
    CK(cudaMemcpy(isd.data(), ctx->D.inv_sd, sizeof(double) * ctx->p, cudaMemcpyDeviceToHost));
    for (int64_t c = 0; c < ctx->p; ++c) sd_host[c] = 1.0 / isd[c];
  }
  return FSQR_OK;
}

fsqr_status fsqr_path(fsqr_ctx* ctx, const double* lam_path_host, int32_t T, int64_t* total, int64_t* iters_host,
                      double* obj_host, double* R_host, int64_t* nnz_host, int32_t* converged_host, void* stream) {
  if (!ctx || !lam_path_host || T < 1) return set_err(ctx, FSQR_ERR_CONFIG, "bad path arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int R = ctx->R;
  for (int64_t q = 0; q < (int64_t)R * T; ++q)
    if (!(lam_path_host[q] >= 0.0)) return set_err(ctx, FSQR_ERR_CONFIG, "lam_path[%lld] invalid", (long long)q);
  Dev& D = ctx->D;
  ctx->alloc_st = st;
  if (T != ctx->T || !D.path_rec) {
    ctx->T = T;
    ctx->path_cap = std::min<int64_t>(ctx->p + 1, 4 * ctx->n + 64);
    double* lp;
    AL(lp, (size_t)R * T);
    D.lam_path = lp;
    AL(D.path_rec, (size_t)R * T * FSQR_PATH_W);
    AL(D.path_idx, (size_t)R * T * ctx->path_cap);
    AL(D.path_beta, (size_t)R * T * ctx->path_cap);
    AL(D.path_cnt, (size_t)R * T);
    D.T = T;
    D.path_cap = (int)ctx->path_cap;
    for (int m = 0; m < M_COUNT; ++m) {
      ctx->mode_dev[m].lam_path = D.lam_path;
      ctx->mode_dev[m].path_rec = D.path_rec;
      ctx->mode_dev[m].path_idx = D.path_idx;
      ctx->mode_dev[m].path_beta = D.path_beta;
      ctx->mode_dev[m].path_cnt = D.path_cnt;
      ctx->mode_dev[m].T = T;
      ctx->mode_dev[m].path_cap = D.path_cap;
    }
    if (ctx->graph[M_PATH].exec) {
      cudaGraphExecDestroy(ctx->graph[M_PATH].exec);
      ctx->graph[M_PATH].exec = nullptr;
    }
  }
  CK(cudaMemcpyAsync((void*)D.lam_path, lam_path_host, sizeof(double) * R * T, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(D.path_rec, 0, sizeof(double) * R * T * FSQR_PATH_W, st));
  CK(cudaMemsetAsync(D.path_cnt, 0, sizeof(long long) * R * T, st));
  CK(cudaMemsetAsync(D.t_idx, 0, sizeof(int) * R, st));
  CK(cudaMemsetAsync(D.pt_iters, 0, sizeof(long long) * R, st));
  std::vector<double> l0(R);
  for (int r = 0; r < R; ++r) l0[r] = lam_path_host[(size_t)r * T];
  CK(cudaMemcpyAsync(D.lam_cur, l0.data(), sizeof(double) * R, cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  fsqr_status s = reset_control(ctx, st);
  if (s != FSQR_OK) return s;
  int64_t it0;
  float ms;
  s = drive(ctx, M_PATH, st, &it0, &ms);
  if (s != FSQR_OK) return s;
  std::vector<double> rec((size_t)R * T * FSQR_PATH_W);
  long long it = 0;
  CK(cudaMemcpy(rec.data(), D.path_rec, sizeof(double) * rec.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&it, D.iter, sizeof it, cudaMemcpyDeviceToHost));
  if (total) *total = it - it0;
  for (int64_t q = 0; q < (int64_t)R * T; ++q) {
    const double* pr = &rec[q * FSQR_PATH_W];
    if (iters_host) iters_host[q] = (int64_t)pr[0];
    if (R_host)
      for (int a = 0; a < 3; ++a) R_host[q * 3 + a] = pr[1 + a];
    if (obj_host) obj_host[q] = pr[4];
    if (nnz_host) nnz_host[q] = (int64_t)pr[5];
    if (converged_host) converged_host[q] = pr[6] > 0.5 ? 1 : 0;
  }
  return FSQR_OK;
}

fsqr_status fsqr_path_hbic(fsqr_ctx* ctx, double* hbic_host) {
  if (!ctx || !hbic_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  SYNC_DEVICE();
  if (!ctx->D.path_rec) return set_err(ctx, FSQR_ERR_STATE, "fsqr_path has not run");
  const int R = ctx->R, T = ctx->T;
  std::vector<double> rec((size_t)R * T * FSQR_PATH_W);
  CK(cudaMemcpy(rec.data(), ctx->D.path_rec, sizeof(double) * rec.size(), cudaMemcpyDeviceToHost));
  const double n = (double)ctx->n, p = (double)ctx->p;
  for (int64_t q = 0; q < (int64_t)R * T; ++q) {
    const double* pr = &rec[q * FSQR_PATH_W];
    hbic_host[q] = std::log(pr[7]) + pr[5] * (std::log(std::log(n)) / n) * std::log(p);
  }
  return FSQR_OK;
}

fsqr_status fsqr_tune(fsqr_ctx* ctx, const fsqr_tune_options* o, double* grid_host, double* hbic_host,
                      int32_t* best_host, double* lam_piv_host, int64_t* total, void* stream) {
  if (!ctx || !o || !best_host) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  if (o->T < 2 || !(o->lam_min_frac > 0.0 && o->lam_min_frac < 1.0) || o->B < 0 ||
      (o->B > 0 && (!(o->alpha > 0.0 && o->alpha < 1.0) || !(o->c > 0.0))))
    return set_err(ctx, FSQR_ERR_CONFIG, "fsqr_tune: need T >= 2, lam_min_frac in (0,1), B >= 0, alpha in (0,1), c > 0");
  const int R = ctx->R, T = o->T;
  std::vector<double> grid((size_t)R * T), piv(R, 0.0);
  for (int r = 0; r < R; ++r) {
    const double lmax = ctx->lambda_max[r];
    double hi = lmax, lo = o->lam_min_frac * lmax;
    if (o->B > 0) {
      // pivotal lambda (reading R18): c times the ceil((1-alpha) B)-th order statistic of Lambda_b
      std::vector<double> L((size_t)o->B);
      fsqr_status s = fsqr_pivotal(ctx, r, o->B, o->seed, L.data(), stream);
      if (s != FSQR_OK) return s;
      std::sort(L.begin(), L.end());
      const int64_t k = std::max<int64_t>(1, (int64_t)std::ceil((1.0 - o->alpha) * (double)o->B));
      piv[r] = o->c * L[(size_t)(k - 1)];
      hi = std::max(lmax, piv[r]);
      lo = o->lam_min_frac * std::min(lmax, piv[r]);
    }
    // geometric grid hi -> lo (reading R20)
    for (int t = 0; t < T; ++t) grid[(size_t)r * T + t] = hi * std::pow(lo / hi, (double)t / (double)(T - 1));
  }
  fsqr_status s = fsqr_path(ctx, grid.data(), T, total, nullptr, nullptr, nullptr, nullptr, nullptr, stream);
  if (s != FSQR_OK) return s;
  std::vector<double> h((size_t)R * T);
  s = fsqr_path_hbic(ctx, h.data());
  if (s != FSQR_OK) return s;
  for (int r = 0; r < R; ++r) {
    int b = 0;
    for (int t = 1; t < T; ++t)
      if (h[(size_t)r * T + t] < h[(size_t)r * T + b]) b = t;   // first minimal point
    best_host[r] = b;
  }
  if (grid_host) memcpy(grid_host, grid.data(), sizeof(double) * grid.size());
  if (hbic_host) memcpy(hbic_host, h.data(), sizeof(double) * h.size());
  if (lam_piv_host) memcpy(lam_piv_host, piv.data(), sizeof(double) * R);
  return FSQR_OK;
}

fsqr_status fsqr_path_beta(fsqr_ctx* ctx, int32_t r, int32_t t, int64_t cap, int64_t* idx_host, double* beta_host,
                           int64_t* count) {
  if (!ctx || !count) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  SYNC_DEVICE();
  if (!ctx->D.path_rec) return set_err(ctx, FSQR_ERR_STATE, "fsqr_path has not run");
  if (r < 0 || r >= ctx->R || t < 0 || t >= ctx->T) return set_err(ctx, FSQR_ERR_CONFIG, "bad (r, t)");
  const size_t q = (size_t)r * ctx->T + t;
  long long cnt = 0;
  CK(cudaMemcpy(&cnt, ctx->D.path_cnt + q, sizeof cnt, cudaMemcpyDeviceToHost));
  *count = cnt;
  const int64_t m = std::min<int64_t>(std::min<int64_t>(cnt, cap), ctx->path_cap);
  if (m > 0 && idx_host && beta_host) {
    std::vector<int32_t> ii(m);
    CK(cudaMemcpy(ii.data(), ctx->D.path_idx + q * ctx->path_cap, sizeof(int32_t) * m, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(beta_host, ctx->D.path_beta + q * ctx->path_cap, sizeof(double) * m, cudaMemcpyDeviceToHost));
    for (int64_t a = 0; a < m; ++a) idx_host[a] = ii[a];
  }
  if (cnt > ctx->path_cap)
    return set_err(ctx, FSQR_ERR_STATE,
                   "path point (rhs %d, t %d) has %lld nonzero coefficients, more than the path store holds "
                   "(%lld = min(p+1, 4n+64)); the first %lld in index order were returned",
                   r, t, cnt, (long long)ctx->path_cap, (long long)m);
  return FSQR_OK;
}

fsqr_status fsqr_trace(fsqr_ctx* ctx, double* out_host, int64_t cap_rows, int64_t* rows) {
  if (!ctx || !out_host || !rows) return set_err(ctx, FSQR_ERR_CONFIG, "null argument");
  SYNC_DEVICE();
  long long it = 0;
  int stopped = 0;
  CK(cudaMemcpy(&it, ctx->D.iter, sizeof it, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&stopped, ctx->D.stop, sizeof stopped, cudaMemcpyDeviceToHost));
  if (stopped) ++it;   // the pass that found R(w^k) <= tol wrote row k before the iteration stopped
  const int W = ctx->R * FSQR_TRACE_W;
  std::vector<double> tr((size_t)ctx->opt.trace_cap * W);
  CK(cudaMemcpy(tr.data(), ctx->D.trace, sizeof(double) * tr.size(), cudaMemcpyDeviceToHost));
  const int64_t avail = std::min<int64_t>(it, ctx->opt.trace_cap);
  const int64_t m = std::min<int64_t>(avail, cap_rows);
  for (int64_t a = 0; a < m; ++a) {
    const int64_t k = it - m + a;
    memcpy(out_host + a * W, &tr[(size_t)(k % ctx->opt.trace_cap) * W], sizeof(double) * W);
  }
  *rows = m;
  return FSQR_OK;
}

fsqr_status fsqr_profile_iterate(fsqr_ctx* ctx, int64_t k, double* stage_ms_host, double* total_ms_host,
                                 void* stream) {
  if (!ctx || k < 1) return set_err(ctx, FSQR_ERR_CONFIG, "bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  fsqr_status s = reset_control(ctx, st);
  if (s != FSQR_OK) return s;
  std::vector<cudaEvent_t> ev((size_t)3 * k + 1);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  const Dev& D = ctx->mode_dev[M_ITER];
  CK(cudaEventRecord(ev[0], st));
  for (int64_t i = 0; i < k; ++i) {
    launch_k2(ctx, D, st);
    CK(cudaEventRecord(ev[3 * i + 1], st));
    launch_k1(D, ctx->k1_grid, st);
    CK(cudaEventRecord(ev[3 * i + 2], st));
    if (!k1_fuses_finalize(D)) launch_finalize(D, st);   // else stage 3 is empty (fused into K1)
    CK(cudaEventRecord(ev[3 * i + 3], st));
  }
  CK(cudaGetLastError());
  CK(cudaEventSynchronize(ev.back()));
  double acc[3] = {0, 0, 0};
  for (int64_t i = 0; i < k; ++i)
    for (int q = 0; q < 3; ++q) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev[3 * i + q], ev[3 * i + q + 1]));
      acc[q] += ms;
    }
  float tot = 0.f;
  CK(cudaEventElapsedTime(&tot, ev[0], ev.back()));
  for (auto& e : ev) cudaEventDestroy(e);
  if (stage_ms_host)
    for (int q = 0; q < 3; ++q) stage_ms_host[q] = acc[q];
  if (total_ms_host) *total_ms_host = tot;
  return FSQR_OK;
}

int64_t fsqr_iterations(fsqr_ctx* ctx) {
  if (!ctx) return -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  long long it = 0;
  if (cudaMemcpy(&it, ctx->D.iter, sizeof it, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return it;
}

fsqr_status fsqr_pack2(const uint8_t* x8, int64_t ld8, int64_t n, int64_t p, uint8_t* x2, int64_t ld2, void* stream) {
  fsqr_ctx* ctx = nullptr;
  if (!x8 || !x2) return set_err(nullptr, FSQR_ERR_CONFIG, "null argument");
  if (n < 1 || n > 65536 || p < 1 || ld8 < n || ld8 % 16 || ld2 < (n + 3) / 4 || ld2 % 16 ||
      ((uintptr_t)x8) % 16 || ((uintptr_t)x2) % 16)
    return set_err(nullptr, FSQR_ERR_CONFIG, "fsqr_pack2: bad sizes or alignment");
  cudaStream_t st = (cudaStream_t)stream;
  int* bad = nullptr;
  CK(cudaMallocAsync((void**)&bad, sizeof(int), st));
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), st);
  if (e == cudaSuccess) {
    launch_pack2(x8, ld8, (int)n, p, x2, ld2, bad, st);
    e = cudaGetLastError();
  }
  int h_bad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(bad, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  CK(e);
  if (h_bad) return set_err(nullptr, FSQR_ERR_DATA, "fsqr_pack2: a genotype code exceeds 3");
  return FSQR_OK;
}

fsqr_status fsqr_fit_host(const fsqr_design* Xh, const double* y_host, int32_t n_rhs, const double* tau_host,
                          const double* lambda_host, const fsqr_options* opt, int64_t iters, double* beta_host,
                          fsqr_result* out, void* stream) {
  fsqr_ctx* ctx = nullptr;
  if (!Xh || !y_host || !beta_host) return set_err(nullptr, FSQR_ERR_CONFIG, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t esz = Xh->storage == 0 ? 4 : 1;
  const size_t xb = (size_t)Xh->ld * (size_t)Xh->p * esz;
  void* dX = nullptr;
  double* dy = nullptr;
  auto fail = [&](const char* what, cudaError_t e) {
    if (dX) cudaFreeAsync(dX, st);
    if (dy) cudaFreeAsync(dy, st);
    return set_err(nullptr, e == cudaErrorMemoryAllocation ? FSQR_ERR_OOM : FSQR_ERR_CUDA, "%s: %s", what,
                   cudaGetErrorString(e));
  };
  fsqr_design Xd = *Xh;
  Xd.mean_dev = nullptr;
  Xd.scale_dev = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dy, sizeof(double) * Xh->n, st);
  if (e != cudaSuccess) return fail("device copy of y", e);
  e = cudaMemcpyAsync(dy, y_host, sizeof(double) * Xh->n, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return fail("host-to-device copy", e);
  if ((Xh->flags & FSQR_DESIGN_PACK2) && Xh->storage == FSQR_U8 && Xh->data_dev && Xh->n >= 2 && Xh->n <= 65536 &&
      Xh->p >= 1 && Xh->ld >= Xh->n && Xh->ld % 16 == 0) {
    // u8 codes repacked on the way in: 256 MB column chunks are copied into a staging buffer and
    // packed straight into the 2-bit design, so only n*p/4 bytes of X are ever resident
    const int64_t ld2 = pack2_ld(Xh->n);
    const int64_t cc = std::max<int64_t>(1, std::min<int64_t>(Xh->p, ((int64_t)256 << 20) / Xh->ld));
    uint8_t* stg = nullptr;
    int* bad = nullptr;
    e = cudaMallocAsync(&dX, (size_t)ld2 * Xh->p, st);
    if (e != cudaSuccess) return fail("device copy of X", e);
    e = cudaMallocAsync((void**)&stg, (size_t)cc * Xh->ld, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&bad, sizeof(int), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, sizeof(int), st);
    for (int64_t c0 = 0; e == cudaSuccess && c0 < Xh->p; c0 += cc) {
      const int64_t nc = std::min(cc, Xh->p - c0);
      e = cudaMemcpyAsync(stg, (const uint8_t*)Xh->data_dev + c0 * Xh->ld, (size_t)nc * Xh->ld, cudaMemcpyHostToDevice, st);
      if (e == cudaSuccess) {
        launch_pack2(stg, Xh->ld, (int)Xh->n, nc, (uint8_t*)dX + c0 * ld2, ld2, bad, st);
        e = cudaGetLastError();
      }
    }
    int h_bad = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (stg) cudaFreeAsync(stg, st);
    if (bad) cudaFreeAsync(bad, st);
    if (e != cudaSuccess) return fail("host-to-device copy / repack", e);
    if (h_bad) {
      cudaFreeAsync(dX, st);
      cudaFreeAsync(dy, st);
      cudaStreamSynchronize(st);
      return set_err(nullptr, FSQR_ERR_DATA, "FSQR_DESIGN_PACK2: a genotype code exceeds 3");
    }
    Xd.storage = FSQR_PACKED2;
    Xd.flags = 0;
    Xd.ld = ld2;
  } else {
    e = cudaMallocAsync(&dX, xb, st);
    if (e != cudaSuccess) return fail("device copy of X", e);
    e = cudaMemcpyAsync(dX, Xh->data_dev, xb, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail("host-to-device copy", e);
  }
  Xd.data_dev = dX;
  fsqr_status s = fsqr_create(&Xd, dy, n_rhs, tau_host, lambda_host, nullptr, opt, stream, &ctx);
  if (s == FSQR_OK && (Xd.flags & FSQR_DESIGN_PACK2)) {   // the ctx owns its packed copy
    cudaFreeAsync(dX, st);
    dX = nullptr;
  }
  if (s == FSQR_OK) {
    if (iters >= 0) {
      s = fsqr_iterate(ctx, iters, stream);
      if (s == FSQR_OK && out) s = collect(ctx, out, 0, st, 0.f);
    } else {
      s = fsqr_solve(ctx, out, stream);
    }
    if (s == FSQR_OK || s == FSQR_NOT_CONVERGED) {
      fsqr_status s2 = fsqr_get_beta(ctx, beta_host, 0, stream);
      if (s2 != FSQR_OK) s = s2;
    }
    fsqr_destroy(ctx);
  }
  if (dX) cudaFreeAsync(dX, st);
  cudaFreeAsync(dy, st);
  cudaStreamSynchronize(st);
  return s;
}

}  // extern "C"
