/*
 * fsqr.h — C ABI of the B200-native FS-QRPPA hot path (libfsqr.so).
 *
 * FS-QRPPA (§4, Algorithm 1) solves the l1-penalised
 * quantile regression (PQR)
 *
 *     min_beta  (1/n) sum_i rho_tau(y_i - x~_i^T beta) + sum_{j>=1} lam_j |beta_j|      (E1, L61-66)
 *
 * on a column-split design X~ = [X~_1 | ... | X~_G] (E7, L177-180) with the
 * Jacobi prox step on every beta_g (E14, L274-277) and on z (E15, L279-285)
 * followed by the extrapolated dual step (E12, L247-257):
 *
 *     beta_g^{k+1} = (1/eta_g)[(eta_g beta_g^k + X~_g^T theta^k - lam_g)_+ - (-eta_g beta_g^k - X~_g^T theta^k - lam_g)_+]
 *     z^{k+1}      = (z^k + theta^k/mu - tau/(n mu))_+ - (-z^k - theta^k/mu - (1-tau)/(n mu))_+
 *     theta^{k+1}  = theta^k - mu/(G+1) [2 r^{k+1} - r^k],   r = X~ beta + z - y
 *
 * X~ is the standardised design: column 0 is a virtual
 * all-ones intercept (lam_0 = 0, L155); model column j >= 1 is stored data
 * column c = j-1 and standardised on the fly, x~_ij = (x_ij - m_j)/s_j with the
 * sample mean m_j and sample sd s_j (n-1 divisor).
 *
 * Conventions
 *  - Every pointer named *_dev is a device pointer; *_host is host memory.
 *  - n-vectors for RHS r are stored contiguously: v[r*n + i].
 *  - beta is stored coefficient-major: beta[j*n_rhs + r], j = 0..p.
 *  - Streams: `stream` is a cudaStream_t (CUstream) handle passed as void*;
 *    NULL means the legacy default stream.  All work is enqueued on it.
 *    Calls that take no stream (fsqr_set_lambda, fsqr_set_lambda2, fsqr_get_colstats,
 *    fsqr_path_hbic, fsqr_path_beta, fsqr_trace, fsqr_iterations) first wait for the whole
 *    device, so they never race with iterations still queued on a caller's stream.
 *  - No call aborts or prints.  Failures return a status < 0 and the message
 *    is available from fsqr_last_error(ctx) (or fsqr_global_error() when no
 *    context exists).  FSQR_NOT_CONVERGED is a flag, not an error: the state
 *    is valid and readable.
 *  - A context is single-writer and not thread-safe; distinct contexts are
 *    independent.  Identical inputs give bitwise-identical outputs run to run.
 *  - There is no CPU fallback: every step of the iteration runs in CUDA
 *    kernels compiled for sm_100a.  A missing or non-sm_100 device is
 *    FSQR_ERR_CUDA.
 */
#ifndef FSQR_H_
#define FSQR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FSQR_OK = 0,
  FSQR_NOT_CONVERGED = 2,   /* max_iter reached; state valid */
  FSQR_ERR_CONFIG = -1,     /* G < 1 or G > p+1, tau not in (0,1), mu <= 0, lambda < 0, bad storage/ld/sizes */
  FSQR_ERR_DATA = -2,       /* zero-variance column (message names it), non-finite y */
  FSQR_ERR_NUMERIC = -3,    /* NaN/Inf appeared in the state */
  FSQR_ERR_CUDA = -4,       /* CUDA runtime/driver failure (message has the CUDA error string) */
  FSQR_ERR_OOM = -5,        /* device allocation failed */
  FSQR_ERR_STATE = -6       /* call not valid in the current state (e.g. path not run) */
} fsqr_status;

typedef enum {
  FSQR_F32_DENSE = 0,   /* fp32, column-major, ld >= n floats, ld % 4 == 0 */
  FSQR_U8 = 1,          /* genotype codes {0,1,2} one byte each, ld >= n bytes, ld % 16 == 0 */
  FSQR_PACKED2 = 2      /* 2-bit codes, sample i at bits 2*(i%4) of byte i/4, ld >= ceil(n/4), ld % 16 == 0 */
} fsqr_storage;

typedef enum {
  FSQR_BACKEND_AUTO = 0,    /* tcgen05 for U8 and PACKED2 (n_rhs <= 16), else SIMT */
  FSQR_BACKEND_TC = 1,      /* tcgen05.mma kind::i8, TMA-staged tiles; PACKED2 unpacks into a TMEM A operand */
  FSQR_BACKEND_SIMT = 2     /* CUDA-core path (dp4a exact integer for U8/PACKED2, fp64 for F32) */
} fsqr_backend;

/* folded-concave penalties for the LLA driver (Section 5, Algorithm 2) */
typedef enum {
  FSQR_SCAD = 1,            /* p'_lambda of E16 (L354-361), a > 2 (a = 3.7 in the paper's studies, L404) */
  FSQR_MCP = 2              /* p'_lambda of E17 (L363-369), a > 1 (a = 3 in the paper's studies, L404) */
} fsqr_penalty;

/* fsqr_design.flags */
enum {
  /* U8 storage only: at create, repack the codes into an OWNED 2-bit copy (fsqr_pack2) and run the
   * PACKED2 kernels on it, so every iteration streams n*p/4 instead of n*p bytes (DESIGN.md §5,
   * "storage").  Codes must be in {0..3} (else FSQR_ERR_DATA); data_dev is read only during
   * create and may be freed afterwards.  Results are those of PACKED2 storage on the same codes.
   * The owned copy's column stride is ceil(n/4) rounded up to 128 bytes (aligned TMA rows). */
  FSQR_DESIGN_PACK2 = 1
};

typedef struct {
  int32_t storage;          /* fsqr_storage */
  int32_t flags;            /* FSQR_DESIGN_* bits, 0 = none */
  int64_t n;                /* observations, 2 <= n <= 65536 */
  int64_t p;                /* stored columns (the intercept is virtual and not stored) */
  const void* data_dev;     /* BORROWED: [p][ld] column-major; must stay alive and unmodified for the ctx lifetime
                               (with FSQR_DESIGN_PACK2: only during fsqr_create) */
  int64_t ld;               /* column stride in elements (F32) or bytes (U8, PACKED2); padding must be zero */
  const double* mean_dev;   /* optional [p] m_j (NULL: computed, a0) */
  const double* scale_dev;  /* optional [p] s_j (NULL: computed, a0); both or neither */
} fsqr_design;

typedef struct {
  int32_t G;                /* number of column blocks (Remark 1, L307-310) */
  int32_t backend;          /* fsqr_backend */
  double mu;                /* augmented parameter mu > 0 (L259) */
  double eta_safety;        /* eta_g = eta_safety * mu * Lambda_hat_g, default 1.05 */
  const double* eta_host;   /* optional [G]: use these eta_g instead of the power method */
  double tol;               /* stop when R(w^k) = max(R_p, R_beta, R_z) <= tol (reading R1) */
  int64_t max_iter;         /* iteration cap per fsqr_solve call (each LLA stage is one call) */
  int32_t power_max_iter;   /* power method cap (default 1000) */
  int32_t trace_cap;        /* rows of the per-iteration trace ring buffer (default 4096) */
  double power_tol;         /* power method relative tolerance (default 1e-4) */
  uint64_t seed;            /* power-method / Lanczos start vector seed */
  int64_t max_iter_point;   /* per-lambda-point cap in fsqr_path (default 10000) */
  int32_t eta_method;       /* Lambda_hat_g by FSQR_ETA_LANCZOS (default) or FSQR_ETA_POWER (L259 names both);
                               power_max_iter / power_tol are the step cap and relative tolerance of either */
  int32_t pad_;
} fsqr_options;

enum { FSQR_ETA_LANCZOS = 0, FSQR_ETA_POWER = 1 };

typedef struct {
  int64_t iterations;       /* outer iterations performed by this call */
  int64_t total_iterations; /* iterations since create / set_state */
  int32_t n_rhs;
  int32_t status[16];       /* per RHS: 0 converged, 2 not converged, -3 numeric */
  double R[16][3];          /* per RHS: R_p, R_beta, R_z at the committed iterate */
  double objective[16];     /* per RHS: E1 at the committed iterate (standardised scale) */
  double wall_ms;           /* device time of the call (CUDA events) */
} fsqr_result;

typedef struct fsqr_ctx fsqr_ctx;

/* Fills defaults: G=5, backend AUTO, mu=0 (=> 2/n, reading R2), eta_safety 1.05, tol 1e-6,
 * max_iter 100000, power 1000 / 1e-4, trace 4096, seed 0x5EED, max_iter_point 10000, eta by Lanczos. */
void fsqr_default_options(fsqr_options* opt);

/*
 * Create a solver for n_rhs (1..16) independent quantile levels sharing X.
 * y_dev: [n] response (copied).  tau_host, lambda_host: [n_rhs] (copied);
 * lambda_w_dev: optional [p+1] non-negative penalty weights w_j (lam_j = lambda * w_j, the weighted
 * l1 of E4, L150-155; copied and applied to every RHS; w_0 is ignored: the intercept is never
 * penalised), NULL = all ones.
 * Performs a0 (column statistics, exact integer sums for genotype storage),
 * a0' (eta_g = eta_safety mu Lambda_hat_g by Lanczos or the power method, L259, unless
 * opt->eta_host) and lambda_max (per tau);
 * cold start beta = 0, z = y, theta = 0.  Synchronises `stream`.
 */
fsqr_status fsqr_create(const fsqr_design* X, const double* y_dev, int32_t n_rhs, const double* tau_host,
                        const double* lambda_host, const double* lambda_w_dev, const fsqr_options* opt,
                        void* stream, fsqr_ctx** out);

/* Enqueue exactly k outer iterations (a1-a5), ignoring the stopping test.  Asynchronous. */
fsqr_status fsqr_iterate(fsqr_ctx* ctx, int64_t k, void* stream);

/* Iterate until every RHS satisfies R(w^k) <= tol or max_iter iterations of this call (blocking).
 * The committed iterate is the first w^k that passed (or the last one).  out may be NULL. */
fsqr_status fsqr_solve(fsqr_ctx* ctx, fsqr_result* out, void* stream);

/* E1 at the committed beta per RHS: (1/n) sum rho_tau(y - X~beta) + sum_{j>=1} lam_j |beta_j|
 * (standardised scale).  Uses the cached s = X~beta (no pass over X).  Blocking. */
fsqr_status fsqr_objective(fsqr_ctx* ctx, double* obj_host, void* stream);

/* Relative KKT residuals [n_rhs][3] = (R_p, R_beta, R_z) at the committed iterate; one pass over X. Blocking. */
fsqr_status fsqr_kkt(fsqr_ctx* ctx, double* R_host, void* stream);

/* HBIC (E18) per RHS at the committed iterate:
 * log(sum_i rho_tau(y_i - x~_i^T beta)) + |A| (log log n / n) log p, |A| = #{j >= 1: beta_j != 0}.
 * Uses the cached s = X~beta (no pass over X).  Blocking. */
fsqr_status fsqr_hbic(fsqr_ctx* ctx, double* hbic_host, void* stream);

/* Elastic-net quadratic weight per RHS (Remark 3; App. B missing, DESIGN.md
 * reading R19): the objective gains (lambda2_r / 2) sum_{j>=1} beta_j^2 and the block prox becomes
 *     beta+ = [(eta beta + g - lam)_+ - (-eta beta - g - lam)_+] / (eta + lambda2)   (E14 at 0).
 * lam2_host [n_rhs], >= 0 and finite (else FSQR_ERR_CONFIG); 0 (the default) is the LASSO. */
fsqr_status fsqr_set_lambda2(fsqr_ctx* ctx, const double* lam2_host);

/* Per-RHS penalty weights (weighted l1, E4 L150-155): w_host [n_rhs][p+1], lam_jr = lambda_r * w_jr,
 * w >= 0 and finite (else FSQR_ERR_CONFIG), w_0 ignored; NULL restores unit weights.  The state is
 * kept (warm start).  Blocking. */
fsqr_status fsqr_set_lambda_weights(fsqr_ctx* ctx, const double* w_host, void* stream);

/*
 * L-step LLA for SCAD or MCP (Algorithm 2): solve with the current weights
 * (unit weights = the LASSO stage), then L times set lam_j = p'_lambda(|beta~_j|) from the committed
 * solution (device kernel, E16/E17) and solve again warm-started from (beta~, z~, theta~).  Each
 * stage runs to tol / max_iter as fsqr_solve.  stage_iters_host [L+1] (may be NULL) receives the
 * iterations of each stage; out (may be NULL) the result of the last stage.  Blocking.
 * Errors: FSQR_ERR_CONFIG for an unknown penalty, a out of range, L < 0 or lambda = 0.
 */
fsqr_status fsqr_lla(fsqr_ctx* ctx, int32_t penalty, double a, int32_t L, int64_t* stage_iters_host,
                     fsqr_result* out, void* stream);

/*
 * Pivotal statistic for the lambda grid ("the pivotal quantity approach"; App. F is
 * missing, reading R18): for Monte-Carlo replicates b = 0..B-1 with uniforms
 * U_bi = top 53 bits of splitmix64(seed ^ splitmix64((b << 32) | i)),
 *     Lambda_host[b] = max_{j>=1} | sum_i x~_ij (tau_rhs - 1{U_bi <= tau_rhs}) | / n.
 * 128 replicates per pass over X on the tensor cores (exact integer sums).  The conventional
 * choice is lambda = 1.1 x the 0.9 empirical quantile of Lambda (Belloni-Chernozhukov).
 * Genotype storage (U8 or PACKED2; a 2-bit design is unpacked into a temporary u8 copy of n*p
 * bytes for the duration of the call, since the tiles are streamed as bytes).  Blocking.
 */
fsqr_status fsqr_pivotal(fsqr_ctx* ctx, int32_t rhs, int64_t B, uint64_t seed, double* Lambda_host, void* stream);

/* beta of the committed iterate, [n_rhs][p+1] row per RHS.
 * scale 0: standardised; scale 1: original scale, beta_j/s_j and beta_0 - sum m_j beta_j/s_j (L404). */
fsqr_status fsqr_get_beta(fsqr_ctx* ctx, double* beta_host, int32_t scale, void* stream);

/* committed state: beta [n_rhs][p+1] (standardised), z [n_rhs][n], theta [n_rhs][n]; any may be NULL. */
fsqr_status fsqr_get_state(fsqr_ctx* ctx, double* beta_host, double* z_host, double* theta_host, void* stream);

/* warm start (Algorithm 1 inputs beta^0, z^0, theta^0, L290-292); layouts as fsqr_get_state; resets iteration counters. */
fsqr_status fsqr_set_state(fsqr_ctx* ctx, const double* beta_host, const double* z_host, const double* theta_host,
                           void* stream);

/* change the penalty level per RHS (lambda_host [n_rhs]); the state is kept (warm start). */
fsqr_status fsqr_set_lambda(fsqr_ctx* ctx, const double* lambda_host);

/* change the stopping tolerance (tol > 0) and the per-call iteration cap (max_iter >= 0) of
 * fsqr_solve / fsqr_lla / fsqr_path's stopping test; the state is kept.  Waits for the device. */
fsqr_status fsqr_set_tolerance(fsqr_ctx* ctx, double tol, int64_t max_iter);

/* kernel launches per outer iteration on the hot path (2: X~^T theta pass + forward product with
 * the fused finalize; 3 when the finalize runs as its own kernel, e.g. fp32 storage). */
int32_t fsqr_launches_per_iteration(const fsqr_ctx* ctx);

/* lambda_max(tau) per RHS (null-model threshold, reading R4), computed on the GPU at create. */
fsqr_status fsqr_lambda_max(const fsqr_ctx* ctx, double* out_host);

/* eta_g [G] in use; column statistics m_j, s_j [p] (either may be NULL). */
fsqr_status fsqr_get_eta(const fsqr_ctx* ctx, double* eta_host);
fsqr_status fsqr_get_colstats(fsqr_ctx* ctx, double* mean_host, double* sd_host);

/*
 * Warm-started lambda path: RHS r walks lam_path_host[r*T + t],
 * t = 0..T-1, all RHS in lockstep through one pass over X per iteration.  When R(w^k) <= tol at
 * point t (or max_iter_point updates were taken there) w^k is recorded as point t and is itself the
 * initialisation of point t+1 ("the solution from the preceding lambda serves as the
 * initialization", L412; reading R10): the update that pass computed with lam_t is
 * discarded and the next pass re-tests w^k at lam_{t+1}.  After its last point the RHS is frozen.
 * Blocking.  iters_host [n_rhs][T] (updates taken at each point), obj_host [n_rhs][T],
 * R_host [n_rhs][T][3], nnz_host [n_rhs][T], converged_host [n_rhs][T] (any may be NULL).
 * *total = lockstep passes over X (updates plus the T-1 re-tests per RHS that share them).
 */
fsqr_status fsqr_path(fsqr_ctx* ctx, const double* lam_path_host, int32_t T, int64_t* total, int64_t* iters_host,
                      double* obj_host, double* R_host, int64_t* nnz_host, int32_t* converged_host, void* stream);

/* HBIC (E18, L408-411) of every recorded path point, hbic_host [n_rhs][T]: log(sum_i rho_tau) +
 * |A| (log log n / n) log p at the recorded iterate (the paper's lambda selection in sparse
 * settings, L406-411).  FSQR_ERR_STATE before fsqr_path. */
fsqr_status fsqr_path_hbic(fsqr_ctx* ctx, double* hbic_host);

/*
 * The paper's tuning protocol for sparse settings, one call: per RHS r
 *   1. the grid top: lambda_max(tau_r) (reading R4); with B > 0 also the pivotal lambda
 *      lambda_piv = c * q_{1-alpha}(Lambda_1..Lambda_B) of fsqr_pivotal (reading R18; the order
 *      statistic ceil((1-alpha) B) of the sorted Lambda_b; c = 1.1, alpha = 0.1 in B-C);
 *   2. a geometric grid of T points from lam_hi = max(lambda_max, lambda_piv) down to
 *      lam_lo = lam_min_frac * min(lambda_max, lambda_piv) (reading R20; B = 0: lambda_max to
 *      lam_min_frac * lambda_max), written to grid_host [n_rhs][T];
 *   3. the warm-started path over that grid (fsqr_path, "the solution from the preceding lambda
 *      serves as the initialization", L412) from the context's current state;
 *   4. HBIC (E18, L408-411) of every point into hbic_host [n_rhs][T] and its argmin (the first
 *      minimal point) into best_host [n_rhs]; the selected solution is fsqr_path_beta(r, best).
 * lam_piv_host [n_rhs] receives lambda_piv (0 when B = 0); total the lockstep passes over X.
 * Any output pointer may be NULL except best_host.  Blocking.  Errors: FSQR_ERR_CONFIG for
 * T < 2, lam_min_frac not in (0, 1), B < 0, alpha not in (0, 1) or c <= 0.
 */
typedef struct {
  int32_t T;             /* grid points per RHS (the paper: 50) */
  int32_t pad_;
  double lam_min_frac;   /* bottom of the grid (see 2.) */
  int64_t B;             /* pivotal replicates (0: no pivotal statistic) */
  uint64_t seed;         /* pivotal draws */
  double alpha, c;       /* lambda_piv = c * q_{1-alpha}(Lambda) */
} fsqr_tune_options;

fsqr_status fsqr_tune(fsqr_ctx* ctx, const fsqr_tune_options* o, double* grid_host, double* hbic_host,
                      int32_t* best_host, double* lam_piv_host, int64_t* total, void* stream);

/* Sparse solution of path point t for RHS r: writes up to cap (index j, beta_j standardised) pairs
 * in ascending j (deterministic), returns the count of nonzeros in *count (which may exceed cap:
 * then only cap were written).  The store keeps min(p+1, 4n+64) entries per point: a point with
 * more nonzeros returns FSQR_ERR_STATE (after writing the first ones) instead of truncating silently. */
fsqr_status fsqr_path_beta(fsqr_ctx* ctx, int32_t r, int32_t t, int64_t cap, int64_t* idx_host, double* beta_host,
                           int64_t* count);

/* Per-iteration trace [rows][n_rhs][5] = (R_p, R_beta, R_z, objective, |support|) of w^k for the
 * last min(k_last + 1, trace_cap, cap_rows) iterates k, oldest first (after a stop, the last row is
 * the iterate that passed the test); returns rows written in *rows. */
fsqr_status fsqr_trace(fsqr_ctx* ctx, double* out_host, int64_t cap_rows, int64_t* rows);

/* Measurement entry: run exactly k iterations like fsqr_iterate but as individual launches with
 * CUDA events around each stage on `stream`; returns the summed device time per stage
 * stage_ms_host[3] = {X~^T theta + beta prox (a1,a2,a6), X~ beta (a4), finalize (a3,a5)} and
 * the total (first to last event).  Blocking. */
fsqr_status fsqr_profile_iterate(fsqr_ctx* ctx, int64_t k, double* stage_ms_host, double* total_ms_host, void* stream);

/* Measurement builds only (compile-time instrumentation, tools/k1_timing.py): copies up to n of the
 * per-CTA %globaltimer stamps the instrumented kernels wrote for one iteration; all zero in the
 * shipped build.  Waits for the device. */
fsqr_status fsqr_debug_stamps(fsqr_ctx* ctx, uint64_t* out_host, int64_t n);

/* total outer iterations since create/set_state (device counter; synchronises). */
int64_t fsqr_iterations(fsqr_ctx* ctx);

/* which X^T theta kernel is in use: "tc" or "simt" */
const char* fsqr_backend_name(const fsqr_ctx* ctx);

/*
 * End-to-end convenience entry with HOST buffers (for users without device memory):
 * copies X and y to the device on `stream`, creates a context, runs `iters` iterations
 * (iters < 0: fsqr_solve), copies beta (standardised, [n_rhs][p+1]) back, destroys the
 * context and frees the copies.  X->data_dev here points to HOST memory (pinned for speed).
 * With U8 storage and FSQR_DESIGN_PACK2 the codes travel in 256 MB column chunks through a
 * staging buffer and are repacked on the device as they arrive: only the 2-bit design (n*p/4
 * bytes) is ever resident; a code > 3 is FSQR_ERR_DATA.
 */
fsqr_status fsqr_fit_host(const fsqr_design* X_host, const double* y_host, int32_t n_rhs, const double* tau_host,
                          const double* lambda_host, const fsqr_options* opt, int64_t iters, double* beta_host,
                          fsqr_result* out, void* stream);

/*
 * Repack uint8 genotype codes into the PACKED2 layout (north_star subsystem (1): "uint8 or 2-bit
 * packed {0,1,2}").  x8_dev: [p][ld8] bytes (ld8 >= n, ld8 % 16 == 0, 16-byte aligned); x2_dev:
 * [p][ld2] bytes (ld2 >= ceil(n/4), ld2 % 16 == 0, 16-byte aligned), caller-owned, fully written
 * (sample i of column c at bits 2*(i%4) of byte c*ld2 + i/4, padding zero).  Returns
 * FSQR_ERR_DATA if any code of the first n rows exceeds 3 (x2_dev contents then unspecified),
 * FSQR_ERR_CONFIG for bad sizes.  Synchronises `stream`.
 */
fsqr_status fsqr_pack2(const uint8_t* x8_dev, int64_t ld8, int64_t n, int64_t p, uint8_t* x2_dev, int64_t ld2,
                       void* stream);

const char* fsqr_last_error(const fsqr_ctx* ctx);
const char* fsqr_global_error(void);
const char* fsqr_status_str(fsqr_status s);

/* frees everything the ctx owns (never the borrowed X). NULL is a no-op. */
void fsqr_destroy(fsqr_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* FSQR_H_ */
