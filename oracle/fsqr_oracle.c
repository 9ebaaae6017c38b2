/*
 * fsqr_oracle.c — plain, slow, obviously-correct fp64 CPU FS-QRPPA.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code with the CUDA path (paper_2601_02826_b200/): no headers,
 * no helpers, no constants.  Every loop is written from the paper:
 *
 *   E1  PQR objective            PAPER.md:L61-66  (x_i includes the intercept; lambda_0 = 0)
 *   E4  weighted l1
 *   E7  column split             PAPER.md:L177-180 (contiguous near-equal blocks)
 *   E12 FS-QRPPA update
 *   L259 eta_g > mu*Lambda_max(X_g^T X_g), power method
 *   E14 beta prox
 *   E15 z prox
 *   L287 aggregation X beta = sum_g X_g beta_g
 *   Alg. 1
 *   Prop. 1 saddle point / KKT
 *   L404 standardised design     (x~_ij = (x_ij - m_j)/s_j, sample sd with n-1)
 *
 * Readings where the paper is silent (DESIGN.md §2 lists them all): the
 * stopping rule is the relative KKT residual R = max(R_p, R_beta, R_z)
 * (SURVEY §8(c) #3); initialisation beta=0, z=y, theta=0; lambda_max is the
 * exact null-model threshold with a balanced subgradient at the tie.
 *
 * Determinism: every output element is computed by exactly one thread with a
 * fixed summation order, so results do not depend on OMP_NUM_THREADS.
 * Scalars that combine many elements (norms, objective) are summed serially.
 *
 * Parity pins (tests/test_oracle_*.py): prox closed forms vs brute-force 1-D
 * minimisation, SPEC worked values, products vs numpy on small slabs, power
 * method vs numpy.linalg.eigvalsh, brute-force LP vertex enumeration and
 * HiGHS on tiny inputs, the lambda_max textbook case, partition invariance,
 * Prop. 1 certificate, geometric decay (Corollary 1).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t storage;      /* 0 = fp32 dense, 1 = uint8 {0,1,2}, 2 = 2-bit packed */
  int32_t pad_;
  int64_t n, p, ld;     /* ld: floats (fp32) or bytes (u8 / 2-bit) per stored column */
  const void* data;     /* data column c holds model column j = c + 1 */
  const double* mean;   /* [p] m_j, or NULL until orc_colstats ran */
  const double* sd;     /* [p] s_j */
} orc_design;

typedef struct {
  double tau, mu;
  int32_t G, check;     /* check = 0: run exactly max_iter iterations, ignore the stop test */
  const double* eta;    /* [G] */
  const double* lam;    /* [p+1], lam[0] = 0 (intercept unpenalised) */
  int64_t max_iter;
  double tol;
  double lam2;          /* elastic-net quadratic weight (Remark 3, L347-349; reading R19); 0 = E14 */
} orc_opts;

/* ---------------------------------------------------------------- design */

static double raw(const orc_design* X, int64_t c, int64_t i) {
  if (X->storage == 0) return (double)((const float*)X->data)[c * X->ld + i];
  const uint8_t* b = (const uint8_t*)X->data;
  if (X->storage == 1) return (double)b[c * X->ld + i];
  return (double)((b[c * X->ld + i / 4] >> (2 * (i % 4))) & 3);
}

/* x~_ij: standardised design entry, column 0 is the all-ones intercept (L404) */
double orc_xt(const orc_design* X, int64_t j, int64_t i) {
  if (j == 0) return 1.0;
  return (raw(X, j - 1, i) - X->mean[j - 1]) / X->sd[j - 1];
}

/* sample mean and sample sd (n-1 divisor), two-pass; returns 0 or -(1+c) for a zero-variance column */
int64_t orc_colstats(const orc_design* X, double* mean, double* sd) {
  int64_t bad = -1;
#pragma omp parallel for schedule(dynamic, 256) if (X->n * X->p > 200000)
  for (int64_t c = 0; c < X->p; ++c) {
    double s = 0.0;
    for (int64_t i = 0; i < X->n; ++i) s += raw(X, c, i);
    double m = s / (double)X->n;
    double v = 0.0;
    for (int64_t i = 0; i < X->n; ++i) { double d = raw(X, c, i) - m; v += d * d; }
    mean[c] = m;
    sd[c] = sqrt(v / (double)(X->n - 1));
    if (!(sd[c] > 0.0)) {
#pragma omp critical
      if (bad < 0 || c < bad) bad = c;
    }
  }
  return bad < 0 ? 0 : -(1 + bad);
}

/* contiguous near-equal partition of ncols columns into G blocks */
void orc_blocks(int64_t ncols, int32_t G, int64_t* start) {
  int64_t q = ncols / G, rem = ncols % G;
  start[0] = 0;
  for (int32_t g = 0; g < G; ++g) start[g + 1] = start[g] + q + (g < rem ? 1 : 0);
}

static int32_t block_of(int64_t j, const int64_t* start, int32_t G) {
  int32_t g = 0;
  while (g + 1 < G && j >= start[g + 1]) ++g;
  return g;
}

/* ------------------------------------------------------------- products */

/* g_j = sum_i x~_ij theta_i for model columns j in [j0, j1)  (X_g^T theta, E14 input) */
void orc_backprod_range(const orc_design* X, const double* theta, int64_t j0, int64_t j1, double* g) {
#pragma omp parallel for schedule(dynamic, 64) if (X->n * (j1 - j0) > 200000)
  for (int64_t j = j0; j < j1; ++j) {
    double acc = 0.0;
    for (int64_t i = 0; i < X->n; ++i) acc += orc_xt(X, j, i) * theta[i];
    g[j - j0] = acc;
  }
}

void orc_backprod(const orc_design* X, const double* theta, double* g) {
  orc_backprod_range(X, theta, 0, X->p + 1, g);
}

/* s_i = sum_j x~_ij b_j over model columns j in [j0, j1), in ascending j for every i.
 * Terms with b_j == 0 are exactly +0 and are skipped.  Threads own row ranges. */
void orc_fwdprod_range(const orc_design* X, const double* b, int64_t j0, int64_t j1, double* s) {
  const int64_t n = X->n;
#pragma omp parallel if (n * (j1 - j0) > 200000)
  {
#ifdef _OPENMP
    extern int omp_get_thread_num(void);
    extern int omp_get_num_threads(void);
    int64_t nt = omp_get_num_threads(), t = omp_get_thread_num();
#else
    int64_t nt = 1, t = 0;
#endif
    int64_t i0 = n * t / nt, i1 = n * (t + 1) / nt;
    for (int64_t i = i0; i < i1; ++i) s[i] = 0.0;
    for (int64_t j = j0; j < j1; ++j) {
      double bj = b[j - j0];
      if (bj == 0.0) continue;
      for (int64_t i = i0; i < i1; ++i) s[i] += orc_xt(X, j, i) * bj;
    }
  }
}

void orc_fwdprod(const orc_design* X, const double* beta, double* s) {
  orc_fwdprod_range(X, beta, 0, X->p + 1, s);
}

/* --------------------------------------------------------------- proxes */

static double pos(double v) { return v > 0.0 ? v : 0.0; }

/* E14: beta+ = (1/eta)[(eta*beta + g - lam)_+ - (-eta*beta - g - lam)_+] */
double orc_prox_beta(double beta, double g, double lam, double eta) {
  return (pos(eta * beta + g - lam) - pos(-eta * beta - g - lam)) / eta;
}

/* Elastic-net block prox (Remark 3, L347-349; App. B missing, reading R19):
 *   argmin_b lam1 |b| + (lam2/2) b^2 - g b + (eta/2)(b - beta)^2
 *   = [(eta*beta + g - lam1)_+ - (-eta*beta - g - lam1)_+] / (eta + lam2)   (E14 when lam2 = 0) */
double orc_prox_en(double beta, double g, double lam1, double lam2, double eta) {
  return (pos(eta * beta + g - lam1) - pos(-eta * beta - g - lam1)) / (eta + lam2);
}

/* E15: z+ = (z + theta/mu - tau/(n mu))_+ - (-z - theta/mu - (1-tau)/(n mu))_+ */
double orc_prox_z(double z, double theta, double mu, double tau, int64_t n) {
  return pos(z + theta / mu - tau / ((double)n * mu)) - pos(-z - theta / mu - (1.0 - tau) / ((double)n * mu));
}

/* E12 dual step: theta+ = theta - mu/(G+1) * (2 r+ - r) */
double orc_dual(double theta, double r_new, double r_old, double mu, int32_t G) {
  return theta - mu / (double)(G + 1) * (2.0 * r_new - r_old);
}

/* soft-threshold S_c(v) = sign(v) max(|v| - c, 0) (KKT residual) */
static double soft(double v, double c) {
  return v > c ? v - c : (v < -c ? v + c : 0.0);
}

/* prox of rho_tau with unit weight: P_tau(v) (KKT residual) */
static double prox_rho(double v, double tau) {
  return v > tau ? v - tau : (v < tau - 1.0 ? v + 1.0 - tau : 0.0);
}

/* pinball loss rho_tau(u) = (tau - 1{u<0}) u (L66) */
double orc_rho(double u, double tau) { return (tau - (u < 0.0 ? 1.0 : 0.0)) * u; }

/* --------------------------------------------------------- diagnostics */

/* relative KKT residuals R_p, R_beta, R_z at w = (beta, z, theta) given g = X~^T theta and s = X~ beta */
static void kkt_parts(int64_t n, int64_t p1, const double* y, double tau, const double* lam, double lam2,
                      const double* beta, const double* z, const double* theta, const double* g, const double* s,
                      double* R) {
  double rp = 0, yy = 0, rb = 0, bb = 0, gg = 0, rz = 0, zz = 0, tt = 0;
  for (int64_t i = 0; i < n; ++i) {
    double r = s[i] + z[i] - y[i];
    rp += r * r;
    yy += y[i] * y[i];
    double nt = (double)n * theta[i];
    double d = z[i] - prox_rho(z[i] + nt, tau);
    rz += d * d;
    zz += z[i] * z[i];
    tt += nt * nt;
  }
  for (int64_t j = 0; j < p1; ++j) {
    /* g_j - lam2 beta_j in lam_j d|beta_j| (lam2 = 0: the LASSO condition; intercept lam2 = 0) */
    double d = beta[j] - soft(beta[j] + (g[j] - (j > 0 ? lam2 : 0.0) * beta[j]), lam[j]);
    rb += d * d;
    bb += beta[j] * beta[j];
    gg += g[j] * g[j];
  }
  R[0] = sqrt(rp) / (1.0 + sqrt(yy));
  R[1] = sqrt(rb) / (1.0 + sqrt(bb) + sqrt(gg));
  R[2] = sqrt(rz) / (1.0 + sqrt(zz) + sqrt(tt));
}

void orc_kkt_rel(const orc_design* X, const double* y, double tau, const double* lam, const double* beta,
                 const double* z, const double* theta, double* R) {
  int64_t n = X->n, p1 = X->p + 1;
  double* g = (double*)malloc(sizeof(double) * p1);
  double* s = (double*)malloc(sizeof(double) * n);
  orc_backprod(X, theta, g);
  orc_fwdprod(X, beta, s);
  kkt_parts(n, p1, y, tau, lam, 0.0, beta, z, theta, g, s, R);
  free(g);
  free(s);
}

/* elastic-net objective: E1 + (lam2/2) sum_{j>=1} beta_j^2 (Remark 3, reading R19) */
double orc_objective_en(const orc_design* X, const double* y, double tau, const double* lam, double lam2,
                        const double* beta) {
  int64_t n = X->n, p1 = X->p + 1;
  double* s = (double*)malloc(sizeof(double) * n);
  orc_fwdprod(X, beta, s);
  double loss = 0.0, pen = 0.0;
  for (int64_t i = 0; i < n; ++i) loss += orc_rho(y[i] - s[i], tau);
  for (int64_t j = 1; j < p1; ++j) pen += lam[j] * fabs(beta[j]) + 0.5 * lam2 * beta[j] * beta[j];
  free(s);
  return loss / (double)n + pen;
}

/* E1 objective: (1/n) sum rho_tau(y - X~ beta) + sum_{j>=1} lam_j |beta_j| */
double orc_objective(const orc_design* X, const double* y, double tau, const double* lam, const double* beta) {
  int64_t n = X->n, p1 = X->p + 1;
  double* s = (double*)malloc(sizeof(double) * n);
  orc_fwdprod(X, beta, s);
  double loss = 0.0, pen = 0.0;
  for (int64_t i = 0; i < n; ++i) loss += orc_rho(y[i] - s[i], tau);
  for (int64_t j = 1; j < p1; ++j) pen += lam[j] * fabs(beta[j]);
  free(s);
  return loss / (double)n + pen;
}

/* Prop. 1 certificate: max violations of
 *   (a) z = y - X~ beta,  (b) g_j in lam_j d|beta_j|,  (c) n theta_i in d rho_tau(z_i).  out[0..2] */
void orc_kkt_cert(const orc_design* X, const double* y, double tau, const double* lam, const double* beta,
                  const double* z, const double* theta, double* out) {
  int64_t n = X->n, p1 = X->p + 1;
  double* g = (double*)malloc(sizeof(double) * p1);
  double* s = (double*)malloc(sizeof(double) * n);
  orc_backprod(X, theta, g);
  orc_fwdprod(X, beta, s);
  double va = 0, vb = 0, vc = 0;
  for (int64_t i = 0; i < n; ++i) {
    double a = fabs(y[i] - s[i] - z[i]);
    if (a > va) va = a;
    double t = (double)n * theta[i], v;
    if (z[i] > 0) v = fabs(t - tau);
    else if (z[i] < 0) v = fabs(t - (tau - 1.0));
    else v = t > tau ? t - tau : (t < tau - 1.0 ? tau - 1.0 - t : 0.0);
    if (v > vc) vc = v;
  }
  for (int64_t j = 0; j < p1; ++j) {
    double v;
    if (beta[j] > 0) v = fabs(g[j] - lam[j]);
    else if (beta[j] < 0) v = fabs(g[j] + lam[j]);
    else v = pos(fabs(g[j]) - lam[j]);
    if (v > vb) vb = v;
  }
  out[0] = va;
  out[1] = vb;
  out[2] = vc;
  free(g);
  free(s);
}

/* ------------------------------------------------------------ power method */

static uint64_t orc_mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* start vector entry for model column j: 2*U - 1, U = top 53 bits of mix(seed ^ mix(j)) */
double orc_power_start(uint64_t seed, int64_t j) {
  uint64_t h = orc_mix(seed ^ orc_mix((uint64_t)j));
  return 2.0 * ((double)(h >> 11) * 0x1.0p-53) - 1.0;
}

/* Lambda_max(X~_g^T X~_g) for model columns [j0, j1) by the power method (L259):
 * v <- w/||w||, w = X~_g^T (X~_g v); estimate = v^T w (Rayleigh quotient);
 * stop when |est_k - est_{k-1}| <= tol * est_k or after maxit steps. */
double orc_power(const orc_design* X, int64_t j0, int64_t j1, double tol, int64_t maxit, uint64_t seed,
                 int64_t* iters) {
  int64_t m = j1 - j0, n = X->n;
  double* v = (double*)malloc(sizeof(double) * m);
  double* w = (double*)malloc(sizeof(double) * m);
  double* u = (double*)malloc(sizeof(double) * n);
  double nv = 0.0;
  for (int64_t a = 0; a < m; ++a) { v[a] = orc_power_start(seed, j0 + a); nv += v[a] * v[a]; }
  nv = sqrt(nv);
  for (int64_t a = 0; a < m; ++a) v[a] /= nv;
  double est = 0.0, prev = 0.0;
  int64_t k;
  for (k = 1; k <= maxit; ++k) {
    orc_fwdprod_range(X, v, j0, j1, u);
    orc_backprod_range(X, u, j0, j1, w);
    est = 0.0;
    double nw = 0.0;
    for (int64_t a = 0; a < m; ++a) { est += v[a] * w[a]; nw += w[a] * w[a]; }
    nw = sqrt(nw);
    if (k > 1 && fabs(est - prev) <= tol * est) break;
    prev = est;
    if (!(nw > 0.0)) break;
    for (int64_t a = 0; a < m; ++a) v[a] = w[a] / nw;
  }
  if (iters) *iters = k > maxit ? maxit : k;
  free(v);
  free(w);
  free(u);
  return est;
}

/* Largest eigenvalue of the symmetric tridiagonal matrix with diagonal a[0..k-1] and off-diagonal
 * b[0..k-2], by bisection on Sturm-sequence counts inside the Gershgorin bracket (textbook; 200
 * halvings reach the fp64 resolution of any bracket). */
static int sturm_below(const double* a, const double* b, int k, double x) {
  int cnt = 0;
  double q = a[0] - x;
  if (q < 0.0) ++cnt;
  for (int i = 1; i < k; ++i) {
    if (q == 0.0) q = 1e-300;
    q = (a[i] - x) - b[i - 1] * b[i - 1] / q;
    if (q < 0.0) ++cnt;
  }
  return cnt;   /* number of eigenvalues < x */
}

double orc_tridiag_max_eig(const double* a, const double* b, int k) {
  double lo = a[0], hi = a[0];
  for (int i = 0; i < k; ++i) {
    double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i + 1 < k ? fabs(b[i]) : 0.0);
    if (a[i] - r < lo) lo = a[i] - r;
    if (a[i] + r > hi) hi = a[i] + r;
  }
  for (int it = 0; it < 200 && hi > lo; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_below(a, b, k, mid) == k) hi = mid; else lo = mid;
  }
  return hi;
}

/* Lambda_max(X~_g^T X~_g) for model columns [j0, j1) by the Lanczos method (L259: "the power method
 * ... or Lanczos"), from the same seeded start vector as orc_power:
 *   v_1 = start/||start||, beta_0 = 0;  for k = 1, 2, ...:
 *     w = X~_g^T (X~_g v_k);  alpha_k = v_k^T w;  w -= alpha_k v_k + beta_{k-1} v_{k-1};  beta_k = ||w||
 *     est_k = largest eigenvalue of tridiag(alpha_1..k; beta_1..k-1)  (Ritz value, <= Lambda_max)
 *     stop when |est_k - est_{k-1}| <= tol * est_k, beta_k = 0 (invariant subspace: exact), or k = maxit
 *     v_{k+1} = w / beta_k
 * (no reorthogonalisation: the largest Ritz value converges regardless). */
double orc_lanczos(const orc_design* X, int64_t j0, int64_t j1, double tol, int64_t maxit, uint64_t seed,
                   int64_t* iters) {
  int64_t m = j1 - j0, n = X->n;
  double* v = (double*)malloc(sizeof(double) * m);
  double* vp = (double*)calloc((size_t)m, sizeof(double));
  double* w = (double*)malloc(sizeof(double) * m);
  double* u = (double*)malloc(sizeof(double) * n);
  double* al = (double*)malloc(sizeof(double) * (maxit + 1));
  double* be = (double*)malloc(sizeof(double) * (maxit + 1));
  double nv = 0.0;
  for (int64_t a = 0; a < m; ++a) { v[a] = orc_power_start(seed, j0 + a); nv += v[a] * v[a]; }
  nv = sqrt(nv);
  for (int64_t a = 0; a < m; ++a) v[a] /= nv;
  double est = 0.0, prev = 0.0, bprev = 0.0;
  int64_t k;
  for (k = 1; k <= maxit; ++k) {
    orc_fwdprod_range(X, v, j0, j1, u);
    orc_backprod_range(X, u, j0, j1, w);
    double alpha = 0.0;
    for (int64_t a = 0; a < m; ++a) alpha += v[a] * w[a];
    double nw = 0.0;
    for (int64_t a = 0; a < m; ++a) {
      w[a] = w[a] - alpha * v[a] - bprev * vp[a];
      nw += w[a] * w[a];
    }
    double beta = sqrt(nw);
    al[k - 1] = alpha;
    est = orc_tridiag_max_eig(al, be, (int)k);
    if (k > 1 && fabs(est - prev) <= tol * est) break;
    if (!(beta > 1e-12 * fabs(alpha))) break;
    prev = est;
    be[k - 1] = beta;
    for (int64_t a = 0; a < m; ++a) {
      vp[a] = v[a];
      v[a] = w[a] / beta;
    }
    bprev = beta;
  }
  if (iters) *iters = k > maxit ? maxit : k;
  free(v);
  free(vp);
  free(w);
  free(u);
  free(al);
  free(be);
  return est;
}

/* ----------------------------------------------------------- lambda_max */

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* lambda_max(tau) = max_{j>=1} |sum_i x~_ij psi_i| / n, psi the null-model score with the
 * intercept at the sample tau-quantile q = y_(ceil(n tau)); ties at q share the value that
 * makes sum psi = 0, so psi is a valid subgradient and lambda >= lambda_max gives beta_{1..p} = 0. */
double orc_lambda_max(const orc_design* X, const double* y, double tau, double* q_out) {
  int64_t n = X->n, p1 = X->p + 1;
  double* ys = (double*)malloc(sizeof(double) * n);
  memcpy(ys, y, sizeof(double) * n);
  qsort(ys, (size_t)n, sizeof(double), cmp_double);
  int64_t k = (int64_t)ceil((double)n * tau);
  if (k < 1) k = 1;
  if (k > n) k = n;
  double q = ys[k - 1];
  free(ys);
  int64_t nb = 0, ne = 0, na = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (y[i] < q) ++nb; else if (y[i] > q) ++na; else ++ne;
  }
  double tie = -((double)nb * (tau - 1.0) + (double)na * tau) / (double)ne;
  double* psi = (double*)malloc(sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) psi[i] = (y[i] < q ? tau - 1.0 : (y[i] > q ? tau : tie)) / (double)n;
  double* g = (double*)malloc(sizeof(double) * p1);
  orc_backprod(X, psi, g);
  double lm = 0.0;
  for (int64_t j = 1; j < p1; ++j) if (fabs(g[j]) > lm) lm = fabs(g[j]);
  if (q_out) *q_out = q;
  free(psi);
  free(g);
  return lm;
}

/* --------------------------------------------------------------- solver */

/*
 * Algorithm 1 from the state (beta, z, theta) given in-place.
 * Iteration k:
 *   g = X~^T theta^k;  R(w^k) from (beta^k, z^k, theta^k, g, s^k);
 *   stop if check && R <= tol (status 0), or k == max_iter (status 2);
 *   beta^{k+1}_j = E14(beta^k_j, g_j, lam_j, eta_{G(j)})     ParFor over blocks
 *   z^{k+1}      = E15(z^k, theta^k)
 *   s^{k+1}      = X~ beta^{k+1}                             (sum over blocks, L287)
 *   r^{k+1}      = s^{k+1} + z^{k+1} - y
 *   theta^{k+1}  = theta^k - mu/(G+1) (2 r^{k+1} - r^k)      E12
 * trace (optional, [max_iter+1][5]): R_p, R_beta, R_z, objective(w^k), |support(beta^k)|.
 * Returns 0 converged, 2 max_iter reached, -3 non-finite state.
 */
int orc_solve(const orc_design* X, const double* y, const orc_opts* o, double* beta, double* z, double* theta,
              int64_t* iters, double* R, double* obj, double* trace) {
  const int64_t n = X->n, p1 = X->p + 1;
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (o->G + 1));
  orc_blocks(p1, o->G, start);
  int32_t* blk = (int32_t*)malloc(sizeof(int32_t) * p1);
  for (int64_t j = 0; j < p1; ++j) blk[j] = block_of(j, start, o->G);
  double* g = (double*)malloc(sizeof(double) * p1);
  double* s = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * n);
  orc_fwdprod(X, beta, s);
  for (int64_t i = 0; i < n; ++i) r[i] = s[i] + z[i] - y[i];
  const double sigma = o->mu / (double)(o->G + 1);
  int status = 2;
  int64_t k = 0;
  for (;; ++k) {
    /* fixed-count mode: the state after max_iter updates is the output; its R is not needed */
    if (!o->check && k == o->max_iter && k > 0 && !trace) { status = 2; break; }
    orc_backprod(X, theta, g);
    double Rk[3];
    kkt_parts(n, p1, y, o->tau, o->lam, o->lam2, beta, z, theta, g, s, Rk);
    double loss = 0.0, pen = 0.0;
    int64_t nnz = 0;
    for (int64_t i = 0; i < n; ++i) loss += orc_rho(y[i] - s[i], o->tau);
    for (int64_t j = 1; j < p1; ++j) {
      pen += o->lam[j] * fabs(beta[j]) + 0.5 * o->lam2 * beta[j] * beta[j];
      nnz += beta[j] != 0.0;
    }
    double ob = loss / (double)n + pen;
    if (trace) {
      trace[5 * k + 0] = Rk[0];
      trace[5 * k + 1] = Rk[1];
      trace[5 * k + 2] = Rk[2];
      trace[5 * k + 3] = ob;
      trace[5 * k + 4] = (double)nnz;
    }
    if (R) { R[0] = Rk[0]; R[1] = Rk[1]; R[2] = Rk[2]; }
    if (obj) *obj = ob;
    if (!isfinite(Rk[0]) || !isfinite(Rk[1]) || !isfinite(Rk[2])) { status = -3; break; }
    double Rmax = fmax(Rk[0], fmax(Rk[1], Rk[2]));
    if (o->check && Rmax <= o->tol) { status = 0; break; }
    if (k == o->max_iter) { status = 2; break; }
    /* ParFor g: beta_g^{k+1} by E14 */
    for (int64_t j = 0; j < p1; ++j)
      beta[j] = o->lam2 == 0.0 || j == 0 ? orc_prox_beta(beta[j], g[j], o->lam[j], o->eta[blk[j]])
                                         : orc_prox_en(beta[j], g[j], o->lam[j], o->lam2, o->eta[blk[j]]);
    /* z^{k+1} by E15 (uses z^k, theta^k) */
    for (int64_t i = 0; i < n; ++i) z[i] = orc_prox_z(z[i], theta[i], o->mu, o->tau, n);
    /* theta^{k+1} by E12 */
    orc_fwdprod(X, beta, s);
    for (int64_t i = 0; i < n; ++i) {
      double rn = s[i] + z[i] - y[i];
      theta[i] = orc_dual(theta[i], rn, r[i], o->mu, o->G);
      r[i] = rn;
    }
  }
  (void)sigma;
  if (iters) *iters = k;
  free(start);
  free(blk);
  free(g);
  free(s);
  free(r);
  return status;
}

/*
 * Warm-started lambda path for one tau ("the solution from the preceding lambda
 * serves as the initialization").  For t = 0..T-1 with
 * lam_t = lam_path[t] * w_j (w_0 = 0), Algorithm 1 runs from the current (beta, z, theta):
 *   g = X~^T theta^k, R(w^k) at lam_t;
 *   if R(w^k) <= tol, or max_iter_point updates were taken at this point: w^k is point t, and
 *     the same w^k is the initialisation of point t+1 (tested again there, at lam_{t+1});
 *   else one update with lam_t (E14, E15, L287, E12).
 * Outputs per point: iters[t] (updates taken at the point), R_out[3t..], obj[t],
 * beta_path[t*(p+1)..] (dense, optional), converged[t].  Returns the total number of updates.
 */
int64_t orc_path(const orc_design* X, const double* y, double tau, double mu, int32_t G, const double* eta,
                 const double* w, const double* lam_path, int32_t T, double tol, int64_t max_iter_point,
                 double* beta, double* z, double* theta, int64_t* iters, double* R_out, double* obj,
                 double* beta_path, int32_t* converged) {
  const int64_t n = X->n, p1 = X->p + 1;
  int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (G + 1));
  orc_blocks(p1, G, start);
  int32_t* blk = (int32_t*)malloc(sizeof(int32_t) * p1);
  for (int64_t j = 0; j < p1; ++j) blk[j] = block_of(j, start, G);
  double* lam = (double*)malloc(sizeof(double) * p1);
  double* g = (double*)malloc(sizeof(double) * p1);
  double* s = (double*)malloc(sizeof(double) * n);
  double* r = (double*)malloc(sizeof(double) * n);
  orc_fwdprod(X, beta, s);
  for (int64_t i = 0; i < n; ++i) r[i] = s[i] + z[i] - y[i];
  int64_t total = 0;
  for (int32_t t = 0; t < T; ++t) {
    for (int64_t j = 0; j < p1; ++j) lam[j] = lam_path[t] * w[j];
    for (int64_t kpt = 0;; ++kpt) {
      orc_backprod(X, theta, g);
      double Rk[3];
      kkt_parts(n, p1, y, tau, lam, 0.0, beta, z, theta, g, s, Rk);
      double Rmax = fmax(Rk[0], fmax(Rk[1], Rk[2]));
      if (Rmax <= tol || kpt == max_iter_point) {
        double loss = 0.0, pen = 0.0;
        for (int64_t i = 0; i < n; ++i) loss += orc_rho(y[i] - s[i], tau);
        for (int64_t j = 1; j < p1; ++j) pen += lam[j] * fabs(beta[j]);
        iters[t] = kpt;
        R_out[3 * t] = Rk[0];
        R_out[3 * t + 1] = Rk[1];
        R_out[3 * t + 2] = Rk[2];
        obj[t] = loss / (double)n + pen;
        converged[t] = Rmax <= tol;
        if (beta_path) memcpy(beta_path + (int64_t)t * p1, beta, sizeof(double) * p1);
        break;
      }
      for (int64_t j = 0; j < p1; ++j) beta[j] = orc_prox_beta(beta[j], g[j], lam[j], eta[blk[j]]);
      for (int64_t i = 0; i < n; ++i) z[i] = orc_prox_z(z[i], theta[i], mu, tau, n);
      orc_fwdprod(X, beta, s);
      for (int64_t i = 0; i < n; ++i) {
        double rn = s[i] + z[i] - y[i];
        theta[i] = orc_dual(theta[i], rn, r[i], mu, G);
        r[i] = rn;
      }
      ++total;
    }
  }
  free(start);
  free(blk);
  free(lam);
  free(g);
  free(s);
  free(r);
  return total;
}

/* ------------------------------------------------ folded-concave penalties (Section 5) */

/*
 * p'_lambda(|b|) for SCAD (kind 1, a > 2; E16) and MCP
 * (kind 2, a > 1; E17), written exactly as displayed.
 */
double orc_penalty_deriv(int32_t kind, double a, double lam, double b) {
  const double ab = fabs(b);
  if (kind == 1) {
    if (ab <= lam) return lam;
    if (ab < a * lam) return (a * lam - ab) / (a - 1.0);
    return 0.0;
  }
  if (ab <= a * lam) return lam - ab / a;
  return 0.0;
}

/*
 * LLA weights of Algorithm 2: lambda~_j = p'_lambda(|beta~_j|) for the
 * penalised coefficients j >= 1, written as the weight w_j = p'_lambda(|beta~_j|) / lambda so
 * that lambda_j = lambda * w_j (the weighted l1 of E4, L150-155); w_0 = 0 (intercept, L155).
 */
void orc_lla_weights(int32_t kind, double a, double lam, const double* beta, int64_t p1, double* w) {
  w[0] = 0.0;
  for (int64_t j = 1; j < p1; ++j) w[j] = orc_penalty_deriv(kind, a, lam, beta[j]) / lam;
}

/*
 * HBIC (E18): log(sum_i rho_tau(y_i - x~_i^T beta)) + |A| (log log n / n) C_n
 * with C_n = log p (L411).  |A| counts the nonzero penalised coefficients.
 */
double orc_hbic_value(double loss, int64_t active, int64_t n, int64_t p) {
  return log(loss) + (double)active * (log(log((double)n)) / (double)n) * log((double)p);
}

double orc_hbic(const orc_design* X, const double* y, double tau, const double* beta) {
  const int64_t n = X->n, p1 = X->p + 1;
  double* s = (double*)malloc(sizeof(double) * n);
  orc_fwdprod(X, beta, s);
  double loss = 0.0;
  for (int64_t i = 0; i < n; ++i) loss += orc_rho(y[i] - s[i], tau);
  int64_t act = 0;
  for (int64_t j = 1; j < p1; ++j) act += beta[j] != 0.0;
  free(s);
  return orc_hbic_value(loss, act, n, X->p);
}

/* ------------------------------------------------ pivotal lambda (Section 6) */

/*
 * Uniform draw U_ib in [0, 1) of Monte-Carlo replicate b for observation i: the top 53 bits of
 * splitmix64(seed ^ splitmix64((b << 32) | i)).  The CUDA path implements the same
 * counter-based generator independently (shared definition, no shared code).
 */
double orc_piv_uniform(uint64_t seed, int64_t b, int64_t i) {
  uint64_t h = orc_mix(seed ^ orc_mix(((uint64_t)b << 32) | (uint64_t)i));
  return (double)(h >> 11) * 0x1.0p-53;
}

uint64_t orc_splitmix(uint64_t x) { return orc_mix(x); }

/*
 * Pivotal statistic of Belloni and Chernozhukov (the "pivotal quantity approach", L412; App. F
 * missing, reading R18): for replicates b = 0..B-1,
 *   Lambda_b = max_{j >= 1} | sum_i x~_ij (tau - 1{U_ib <= tau}) | / n.
 * Written out directly: psi, then one X~^T psi per replicate.
 */
void orc_pivotal(const orc_design* X, double tau, int64_t B, uint64_t seed, double* Lambda) {
  const int64_t n = X->n, p1 = X->p + 1;
  double* psi = (double*)malloc(sizeof(double) * n);
  double* g = (double*)malloc(sizeof(double) * p1);
  for (int64_t b = 0; b < B; ++b) {
    for (int64_t i = 0; i < n; ++i) psi[i] = tau - (orc_piv_uniform(seed, b, i) <= tau ? 1.0 : 0.0);
    orc_backprod(X, psi, g);
    double m = 0.0;
    for (int64_t j = 1; j < p1; ++j) m = fmax(m, fabs(g[j]));
    Lambda[b] = m / (double)n;
  }
  free(psi);
  free(g);
}
