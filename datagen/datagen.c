/*
 * datagen.c — seeded synthetic inputs for the FS-QRPPA hot path.
 *
 * This module is SHARED INPUT INFRASTRUCTURE: the oracle (oracle/) and the
 * CUDA path (paper_2601_02826_b200/) both consume the bytes it writes, and it
 * holds none of the method's arithmetic (no standardisation from sample
 * statistics, no products X^T theta / X beta, no proxes).  The response is
 * built with the *population* standardisation of each causal SNP,
 * (G - 2f)/sqrt(2f(1-f)), which is a property of the data-generating process,
 * not the solver's sample standardisation.
 *
 * Randomness is counter-based (splitmix64 finaliser keyed by
 * (seed, stream, index)), so every byte is a pure function of its
 * coordinates and the output does not depend on the OpenMP thread count.
 *
 * Workload recipes follow BASELINE.json `configs` and SURVEY.md §8(d):
 *   - genotype u8 / 2-bit: G_ij = 1{u1 < f_j} + 1{u2 < f_j}, f_j ~ U(fa, fb)
 *   - LD-structured 2-bit: latent AR(1) (rho) across blocks of SNPs,
 *     thresholded at the HWE quantiles Phi^-1((1-f)^2), Phi^-1(1-f^2)
 *   - dense Gaussian fp32 design
 * Layouts (column-major, "SNP-major"):
 *   u8:   X[c * ld + i], ld = round_up(n, 16) bytes, pad = 0
 *   2bit: X[c * ld + i/4] bits 2*(i%4)..2*(i%4)+1, ld = round_up(ceil(n/4), 16)
 *   f32:  X[c * ld + i], ld = round_up(n, 4) floats, pad = 0
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define STREAM_MAF 1u
#define STREAM_GENO 2u
#define STREAM_CAUSAL 3u
#define STREAM_EFFECT 4u
#define STREAM_NOISE 5u
#define STREAM_GAMMA 6u
#define STREAM_LATENT 7u
#define STREAM_GAUSS 8u
#define STREAM_SIGN 9u

static inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t dg_u64(uint64_t seed, uint64_t stream, uint64_t idx) {
  return mix64(mix64(mix64(seed) ^ (stream * 0xD1B54A32D192ED03ull)) ^ idx);
}

/* uniform on the open interval (0, 1) */
double dg_unif(uint64_t seed, uint64_t stream, uint64_t idx) {
  return ((double)(dg_u64(seed, stream, idx) >> 11) + 0.5) * 0x1.0p-53;
}

/* standard normal by Box-Muller (cosine branch) on counters 2k, 2k+1 */
double dg_normal(uint64_t seed, uint64_t stream, uint64_t k) {
  double u1 = dg_unif(seed, stream, 2 * k), u2 = dg_unif(seed, stream, 2 * k + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2);
}

static double phi_cdf(double x) { return 0.5 * erfc(-x / 1.4142135623730950488); }

/* Phi^{-1}(q) by bisection + Newton on erfc; deterministic, ~1e-15 accurate */
double dg_probit(double q) {
  double lo = -40.0, hi = 40.0, x = 0.0;
  for (int it = 0; it < 200; ++it) {
    x = 0.5 * (lo + hi);
    if (phi_cdf(x) < q) lo = x; else hi = x;
    if (hi - lo < 1e-13) break;
  }
  for (int it = 0; it < 3; ++it) {
    double pdf = exp(-0.5 * x * x) * 0.39894228040143267794;
    if (pdf <= 0) break;
    x -= (phi_cdf(x) - q) / pdf;
  }
  return x;
}

/* causal positions: k distinct data-column indices in [0, p), by rejection */
void dg_causal(uint64_t seed, int64_t p, int64_t k, int64_t* out) {
  uint64_t ctr = 0;
  for (int64_t a = 0; a < k; ++a) {
    for (;;) {
      int64_t c = (int64_t)(dg_unif(seed, STREAM_CAUSAL, ctr++) * (double)p);
      if (c >= p) c = p - 1;
      int dup = 0;
      for (int64_t b = 0; b < a; ++b) dup |= (out[b] == c);
      if (!dup) { out[a] = c; break; }
    }
  }
}

/* MAF per data column */
void dg_maf(uint64_t seed, int64_t p, double fa, double fb, double* f) {
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < p; ++c) f[c] = fa + (fb - fa) * dg_unif(seed, STREAM_MAF, (uint64_t)c);
}

/*
 * Binomial(2, f_j) genotypes.  A column that comes out constant (possible only
 * at toy sizes) is redrawn with the next "attempt" counter block, so every
 * column has nonzero variance (the solver rejects zero-variance columns,
 * SPEC.md:L56).  packed = 0 -> u8 layout, 1 -> 2-bit layout.
 */
void dg_genotypes(uint64_t seed, int64_t n, int64_t p, const double* f, int packed, int64_t ld,
                  uint8_t* X) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t c = 0; c < p; ++c) {
    uint8_t* col = X + c * ld;
    for (uint64_t attempt = 0;; ++attempt) {
      memset(col, 0, (size_t)ld);
      int first = -1, varies = 0;
      for (int64_t i = 0; i < n; ++i) {
        uint64_t base = (((uint64_t)c * 64u + attempt) * (uint64_t)n + (uint64_t)i) * 2u;
        int g = (dg_unif(seed, STREAM_GENO, base) < f[c]) + (dg_unif(seed, STREAM_GENO, base + 1) < f[c]);
        if (first < 0) first = g; else if (g != first) varies = 1;
        if (packed) col[i >> 2] |= (uint8_t)(g << (2 * (i & 3)));
        else col[i] = (uint8_t)g;
      }
      if (varies || n < 2 || attempt >= 63) break;
    }
  }
}

/*
 * LD-structured genotypes (config 4): per individual, within blocks of `blk`
 * SNPs, a latent AR(1) L_j = rho L_{j-1} + sqrt(1-rho^2) xi_j (L_first ~ N(0,1))
 * thresholded at HWE quantiles so that P(G>=1) = 1-(1-f)^2, P(G=2) = f^2.
 *
 * Throughput matters here (C4 is 4e10 latent draws): individuals are taken in
 * groups of four (one packed byte); for each SNP c the group's four innovations
 * xi come from two 64-bit counter draws keyed by (c, group), each split into
 * two 32-bit uniforms and turned into a pair of normals by both branches of
 * Box-Muller in single precision (a DGP needs no more).  Both layouts use the
 * same draws, so the u8 and 2-bit designs hold identical codes.
 */
static inline void ld_normals4(uint64_t key, uint64_t ctr, float* xi) {
  for (int h = 0; h < 2; ++h) {
    uint64_t u = mix64(key ^ (2u * ctr + (uint64_t)h));
    float u1 = ((float)(uint32_t)(u >> 40) + 0.5f) * 0x1.0p-24f;    /* (0,1), 24-bit */
    float u2 = ((float)(uint32_t)(u & 0xFFFFFFu) + 0.5f) * 0x1.0p-24f;
    float r = sqrtf(-2.0f * logf(u1));
    float s, c;
    sincosf(6.28318530717958647692f * u2, &s, &c);
    xi[2 * h] = r * c;
    xi[2 * h + 1] = r * s;
  }
}

void dg_genotypes_ld(uint64_t seed, int64_t n, int64_t p, const double* f, double rho, int64_t blk,
                     int packed, int64_t ld, uint8_t* X) {
  float* t1 = (float*)malloc(sizeof(float) * (size_t)p);
  float* t2 = (float*)malloc(sizeof(float) * (size_t)p);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < p; ++c) {
    t1[c] = (float)dg_probit((1.0 - f[c]) * (1.0 - f[c]));
    t2[c] = (float)dg_probit(1.0 - f[c] * f[c]);
  }
  const float rf = (float)rho, sr = (float)sqrt(1.0 - rho * rho);
  const uint64_t key = mix64(mix64(seed) ^ (STREAM_LATENT * 0xD1B54A32D192ED03ull));
  const int64_t nblk = (p + blk - 1) / blk, nb = (n + 3) / 4;
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < p; ++c) memset(X + c * ld, 0, (size_t)ld);
  /* work item = (SNP block b, run of 64 groups of four individuals) */
  const int64_t RUN = 64, nrun = (nb + RUN - 1) / RUN;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nblk * nrun; ++q) {
    const int64_t b = q / nrun, g0 = (q % nrun) * RUN, g1 = g0 + RUN < nb ? g0 + RUN : nb;
    const int64_t c0 = b * blk, c1 = c0 + blk < p ? c0 + blk : p;
    for (int64_t gi = g0; gi < g1; ++gi) {
      float L[4] = {0, 0, 0, 0}, xi[4];
      const int nv = (int)(n - 4 * gi < 4 ? n - 4 * gi : 4);
      for (int64_t c = c0; c < c1; ++c) {
        ld_normals4(key, (uint64_t)c * (uint64_t)nb + (uint64_t)gi, xi);
        uint32_t byte = 0;
        for (int s = 0; s < 4; ++s) {
          L[s] = (c == c0) ? xi[s] : rf * L[s] + sr * xi[s];
          uint32_t g = (uint32_t)(L[s] > t1[c]) + (uint32_t)(L[s] > t2[c]);
          if (s >= nv) g = 0;
          if (packed) byte |= g << (2 * s);
          else X[c * ld + 4 * gi + s] = (uint8_t)g;
        }
        if (packed) X[c * ld + gi] = (uint8_t)byte;
      }
    }
  }
  free(t1);
  free(t2);
}

/* dense Gaussian design stored as fp32 (config 1) */
void dg_gauss_f32(uint64_t seed, int64_t n, int64_t p, int64_t ld, float* X) {
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < p; ++c) {
    for (int64_t i = 0; i < ld; ++i)
      X[c * ld + i] = i < n ? (float)dg_normal(seed, STREAM_GAUSS, (uint64_t)c * (uint64_t)n + (uint64_t)i) : 0.0f;
  }
}

/* read genotype code (0/1/2) of individual i in data column c */
static inline int geno(const uint8_t* X, int packed, int64_t ld, int64_t c, int64_t i) {
  return packed ? (X[c * ld + (i >> 2)] >> (2 * (i & 3))) & 3 : X[c * ld + i];
}

/*
 * Linear predictor of the DGP, eta_i = sum_a w_a * xpop_{i, c_a}, with the
 * population standardisation xpop = (G - 2f)/sqrt(2f(1-f)) for genotypes, or
 * the raw value for the Gaussian fp32 design (population mean 0, sd 1).
 */
void dg_linpred(int storage, int64_t n, const void* X, int64_t ld, const double* f, int64_t k,
                const int64_t* cols, const double* w, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t a = 0; a < k; ++a) {
      int64_t c = cols[a];
      double x;
      if (storage == 0) x = ((const float*)X)[c * ld + i];
      else {
        int g = geno((const uint8_t*)X, storage == 2, ld, c, i);
        x = (g - 2.0 * f[c]) / sqrt(2.0 * f[c] * (1.0 - f[c]));
      }
      acc += w[a] * x;
    }
    out[i] = acc;
  }
}

/* effect sizes: kind 0 -> N(0, sd^2); kind 1 -> U(+-[a, b]) (magnitude U(a,b), random sign) */
void dg_effects(uint64_t seed, uint64_t stream, int64_t k, int kind, double a, double b, double* w) {
  for (int64_t t = 0; t < k; ++t) {
    if (kind == 0) w[t] = a * dg_normal(seed, stream, (uint64_t)t);
    else {
      double mag = a + (b - a) * dg_unif(seed, stream, (uint64_t)t);
      w[t] = dg_unif(seed, STREAM_SIGN + stream * 16u, (uint64_t)t) < 0.5 ? -mag : mag;
    }
  }
}

/* noise: 0 N(0,1); 1 Student-t(3); 2 Laplace(0,1); 3 skew-normal(0,1,alpha=4) */
void dg_noise(uint64_t seed, int64_t n, int kind, double* e) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t b = (uint64_t)i * 8u;
    double v;
    if (kind == 0) v = dg_normal(seed, STREAM_NOISE, b);
    else if (kind == 1) {
      double z = dg_normal(seed, STREAM_NOISE, b);
      double c = 0.0;
      for (int q = 1; q <= 3; ++q) { double t = dg_normal(seed, STREAM_NOISE, b + q); c += t * t; }
      v = z / sqrt(c / 3.0);
    } else if (kind == 2) {
      double u = dg_unif(seed, STREAM_NOISE, b) - 0.5;
      v = (u < 0 ? 1.0 : -1.0) * log(1.0 - 2.0 * fabs(u));
    } else {
      const double alpha = 4.0, d = alpha / sqrt(1.0 + alpha * alpha);
      double u0 = dg_normal(seed, STREAM_NOISE, b), u1 = dg_normal(seed, STREAM_NOISE, b + 1);
      v = d * fabs(u0) + sqrt(1.0 - d * d) * u1;
    }
    e[i] = v;
  }
}
