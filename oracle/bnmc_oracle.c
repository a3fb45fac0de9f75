/* oracle/bnmc_oracle.c -- TEST INFRASTRUCTURE ONLY (see bnmc_oracle.h).
 *
 * A sequential restatement of the reference's hot path.  Every function cites
 * the reference code it follows.  Arithmetic is written expression-for-expression
 * in the reference's evaluation order, compiled without FMA contraction, so on the
 * same glibc libm the results are bit-identical to the compiled reference
 * (tests/test_oracle.py asserts exactly that).
 */
#include "bnmc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

const char* bo_last_error(void) { return g_err; }

/* ---------------------------------------------------------------------------
 * RNG -- proj/include/bnmc/rng.hpp:12-51
 * ------------------------------------------------------------------------- */
#define BO_GOLDEN 0x9E3779B97F4A7C15ull

uint64_t bo_mix(uint64_t z) { /* rng.hpp:19-23 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t bo_fold(uint64_t k, uint64_t v) { /* rng.hpp:27-29 */
  return bo_mix(k * BO_GOLDEN + v + 0x632BE59BD9B4E019ull);
}

uint64_t bo_keyed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) { /* :31-34 */
  return bo_fold(bo_fold(bo_fold(bo_fold(bo_fold(1, seed), a), b), c), d);
}

uint64_t bo_derive(uint64_t key, uint64_t a, uint64_t b) { /* rng.hpp:36-38 */
  return bo_fold(bo_fold(key, a), b);
}

uint64_t bo_next_u64(bo_rng* r) { return bo_mix(r->key + BO_GOLDEN * ++r->counter); } /* :40 */

double bo_next_unit(bo_rng* r) { /* rng.hpp:43 */
  return ((double)(bo_next_u64(r) >> 11) + 0.5) * 0x1p-53;
}

double bo_next_gaussian(bo_rng* r) { /* rng.hpp:46-50 (Box-Muller, cos branch) */
  const double u1 = bo_next_unit(r);
  const double u2 = bo_next_unit(r);
  return sqrt(-2.0 * log(u1)) * cos(6.28318530717958647692529 * u2);
}

static bo_rng stream(uint64_t key) {
  bo_rng r = {key, 0};
  return r;
}

/* ---------------------------------------------------------------------------
 * Distributions -- proj/src/dist.cpp
 * ------------------------------------------------------------------------- */
double bo_draw_gamma(bo_rng* r, double shape) { /* dist.cpp:136-155, Marsaglia-Tsang */
  if (!(shape > 0.0)) return NAN;
  if (shape < 1.0) {
    const double g = bo_draw_gamma(r, shape + 1.0);
    return g * pow(bo_next_unit(r), 1.0 / shape);
  }
  const double d = shape - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      x = bo_next_gaussian(r);
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = bo_next_unit(r);
    if (u < 1.0 - 0.0331 * (x * x) * (x * x)) return d * v;
    if (log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) return d * v;
  }
}

int64_t bo_draw_categorical(bo_rng* r, const double* p, int64_t n) { /* dist.cpp:183-191 */
  const double u = bo_next_unit(r);
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    acc += p[i];
    if (u < acc) return i;
  }
  return n - 1;
}

void bo_draw_dirichlet(bo_rng* r, const double* alpha, int64_t n, double* out) { /* :193-200 */
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    out[i] = bo_draw_gamma(r, alpha[i]);
    sum += out[i];
  }
  for (int64_t i = 0; i < n; ++i) out[i] /= sum;
}

int64_t bo_draw_from_log_weights(bo_rng* r, const double* logw, int64_t n) { /* :202-215 */
  double mx = -INFINITY;
  for (int64_t i = 0; i < n; ++i) {
    if (mx < logw[i]) mx = logw[i]; /* std::max(mx, w) */
  }
  if (!isfinite(mx)) {
    fail("all candidate log-weights are -inf");
    return -1;
  }
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += exp(logw[i] - mx);
  const double u = bo_next_unit(r) * total;
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    acc += exp(logw[i] - mx);
    if (u < acc) return i;
  }
  return n - 1;
}

#define BO_LOG2PI 1.8378770664093454835606594728112

double bo_log_pdf_gaussian(double x, double mean, double var) { /* dist.cpp:61-68 */
  if (!(var > 0.0)) return -INFINITY;
  const double d = x - mean;
  return -0.5 * (d * d / var + log(var) + BO_LOG2PI);
}

double bo_log_pdf_uniform(double x, double lo, double hi) { /* dist.cpp:70-75 */
  if (!(hi > lo)) return -INFINITY;
  if (x < lo || x > hi) return -INFINITY;
  return -log(hi - lo);
}

double bo_log_pdf_inverse_gamma(double x, double shape, double scale) { /* dist.cpp:92-97 */
  if (!(shape > 0.0) || !(scale > 0.0)) return -INFINITY;
  if (!(x > 0.0)) return -INFINITY;
  return shape * log(scale) - lgamma(shape) - (shape + 1.0) * log(x) - scale / x;
}

double bo_log_pmf_categorical(int64_t x, const double* p, int64_t n) { /* dist.cpp:107-113 */
  if (x < 0 || x >= n) return -INFINITY;
  if (!(p[x] > 0.0)) return -INFINITY;
  return log(p[x]);
}

double bo_log_pdf_dirichlet(const double* x, const double* alpha, int64_t n) { /* :115-130 */
  if (n <= 0) return -INFINITY;
  double sum = 0.0, lp = 0.0, norm = 0.0, asum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(alpha[i] > 0.0)) return -INFINITY;
    if (!(x[i] > 0.0)) return -INFINITY;
    sum += x[i];
    lp += (alpha[i] - 1.0) * log(x[i]);
    norm += lgamma(alpha[i]);
    asum += alpha[i];
  }
  if (fabs(sum - 1.0) > 1e-9) return -INFINITY;
  return lp - norm + lgamma(asum);
}

/* Symmetric-concentration Dirichlet log-pdf: alpha[i] == a for all i.  The
 * reference still sums lgamma(a) and a sequentially, reproduced here. */
static double log_pdf_dirichlet_sym(const double* x, double a, int64_t n) {
  if (n <= 0 || !(a > 0.0)) return -INFINITY;
  double sum = 0.0, lp = 0.0, norm = 0.0, asum = 0.0;
  const double la = lgamma(a);
  for (int64_t i = 0; i < n; ++i) {
    if (!(x[i] > 0.0)) return -INFINITY;
    sum += x[i];
    lp += (a - 1.0) * log(x[i]);
    norm += la;
    asum += a;
  }
  if (fabs(sum - 1.0) > 1e-9) return -INFINITY;
  return lp - norm + lgamma(asum);
}

/* sample_dirichlet_batch, RowParallel order (batch.cpp:38-63; ColumnParallel is
 * bit-identical by construction, batch.cpp:66-82). */
int bo_dirichlet_batch(int64_t rows, int64_t cols, const double* alpha, uint64_t key,
                       double* out) {
  if (rows < 1 || cols < 1) return fail("batch needs rows, cols >= 1");
  for (int64_t i = 0; i < rows * cols; ++i)
    if (!(alpha[i] > 0.0)) return fail("Dirichlet concentrations must be positive");
  for (int64_t r = 0; r < rows; ++r) {
    double* row = out + r * cols;
    double sum = 0.0;
    for (int64_t c = 0; c < cols; ++c) {
      bo_rng g = stream(bo_derive(key, (uint64_t)r, (uint64_t)c));
      row[c] = bo_draw_gamma(&g, alpha[r * cols + c]);
      sum += row[c];
    }
    for (int64_t c = 0; c < cols; ++c) row[c] /= sum;
  }
  return 0;
}

/* ParallelExecutor::chunk_size (executor.hpp:27-31): <= 64 chunks, size depends on n only. */
static int64_t chunk_size(int64_t n) { return n <= 64 ? 1 : (n + 63) / 64; }

/* Purposes (sampler.cpp:12-17, 545). */
enum { P_PROPOSAL = 1, P_ACCEPT = 2, P_DISCRETE = 3, P_CONJUGATE = 4, P_INIT = 5 };

/* ---------------------------------------------------------------------------
 * LDA
 * ------------------------------------------------------------------------- */
int bo_lda_count_phi(const bo_lda* m, const int64_t* z, int64_t d0, int64_t d1, int64_t* nkw) {
  /* run_conjugate counting phase for phi (sampler.cpp:61-136): bin = z[i,j], child w[i,j]. */
  for (int64_t t = m->offsets[d0]; t < m->offsets[d1]; ++t) {
    const int64_t k = z[t], v = m->w[t];
    if (k < 0 || k >= m->K) return fail("conjugate update bin out of range for 'phi'");
    if (v >= 0 && v < m->V) nkw[k * m->V + v] += 1;
  }
  return 0;
}

int bo_lda_draw_phi(const bo_lda* m, const int64_t* nkw, uint64_t seed, int64_t iter,
                    double* phi) {
  /* alpha = beta + count (sampler.cpp:161-170), then sample_dirichlet_batch (:173-179). */
  const int64_t n = m->K * m->V;
  double* alpha = (double*)malloc(sizeof(double) * (size_t)n);
  if (!alpha) return fail("out of memory");
  for (int64_t i = 0; i < n; ++i) alpha[i] = m->beta + (double)nkw[i];
  const uint64_t key = bo_keyed(seed, P_CONJUGATE, (uint64_t)m->var_phi, (uint64_t)iter, 0);
  const int rc = bo_dirichlet_batch(m->K, m->V, alpha, key, phi);
  free(alpha);
  return rc;
}

int bo_lda_phi_gammas(const bo_lda* m, const int64_t* nkw, uint64_t seed, int64_t iter, int64_t v0,
                      int64_t v1, double* g) {
  /* The unnormalised cells g[k][v], v in [v0,v1), of the phi block's Dirichlet batch:
   * the per-cell streams keyed(seed,4,var_phi,iter).derive(k,v) and Gamma(beta + count)
   * draws of bo_dirichlet_batch (batch.cpp:38-41, 45-83) -- the vocabulary slice a rank
   * of the sharded sweep draws before the all-gather and the row normalisation. */
  const uint64_t key = bo_keyed(seed, P_CONJUGATE, (uint64_t)m->var_phi, (uint64_t)iter, 0);
  for (int64_t k = 0; k < m->K; ++k)
    for (int64_t v = v0; v < v1; ++v) {
      bo_rng r = stream(bo_derive(key, (uint64_t)k, (uint64_t)v));
      g[k * m->V + v] = bo_draw_gamma(&r, m->beta + (double)nkw[k * m->V + v]);
    }
  return 0;
}

int bo_lda_theta_z(const bo_lda* m, int64_t* z, const double* phi, double* theta, uint64_t seed,
                   int64_t iter, int64_t d0, int64_t d1) {
  const int64_t K = m->K, V = m->V;
  double* alpha = (double*)malloc(sizeof(double) * (size_t)K);
  double* logw = (double*)malloc(sizeof(double) * (size_t)K);
  if (!alpha || !logw) {
    free(alpha);
    free(logw);
    return fail("out of memory");
  }
  /* theta block: counts c[d][z] (bin = document), alpha + c, per-cell gamma draws
   * with stream keyed(seed,4,var_theta,iter).derive(d,k), left-to-right row sum. */
  const uint64_t tkey = bo_keyed(seed, P_CONJUGATE, (uint64_t)m->var_theta, (uint64_t)iter, 0);
  for (int64_t d = d0; d < d1; ++d) {
    for (int64_t k = 0; k < K; ++k) alpha[k] = 0.0;
    for (int64_t t = m->offsets[d]; t < m->offsets[d + 1]; ++t) {
      const int64_t k = z[t];
      if (k >= 0 && k < K) alpha[k] += 1.0;
    }
    double* row = theta + d * K;
    double sum = 0.0;
    for (int64_t k = 0; k < K; ++k) {
      bo_rng g = stream(bo_derive(tkey, (uint64_t)d, (uint64_t)k));
      row[k] = bo_draw_gamma(&g, m->alpha + alpha[k]);
      sum += row[k];
    }
    for (int64_t k = 0; k < K; ++k) row[k] /= sum;
  }
  /* z block: logw[v] = (0 + log theta[d,v]) + log phi[v, w] (sampler.cpp:230-245),
   * drawn with keyed(seed,3,var_z,t,iter) (sampler.cpp:246-249). */
  for (int64_t d = d0; d < d1; ++d) {
    const double* th = theta + d * K;
    for (int64_t t = m->offsets[d]; t < m->offsets[d + 1]; ++t) {
      const int64_t w = m->w[t];
      for (int64_t v = 0; v < K; ++v) {
        double lp = 0.0;
        lp += bo_log_pmf_categorical(v, th, K);
        lp += bo_log_pmf_categorical(w, phi + v * V, V);
        logw[v] = lp;
      }
      bo_rng g = stream(bo_keyed(seed, P_DISCRETE, (uint64_t)m->var_z, (uint64_t)t, (uint64_t)iter));
      const int64_t k = bo_draw_from_log_weights(&g, logw, K);
      if (k < 0) {
        free(alpha);
        free(logw);
        return 1;
      }
      z[t] = k;
    }
  }
  free(alpha);
  free(logw);
  return 0;
}

double bo_lda_log_joint(const bo_lda* m, const int64_t* z, const double* phi,
                        const double* theta) {
  /* Joint = prod_k p(phi[k]) prod_m p(theta[m]) prod_i prod_j p(z|theta) prod_i prod_j
   * p(w|phi[z]) (tests/golden/describe_lda.txt); each top-level indexed product is a
   * reduce_sum over <= 64 chunks of its outer index (eval.cpp:393-422, executor.cpp:84-97). */
  const int64_t K = m->K, V = m->V, M = m->M;
  double total = 0.0;
  double f;
  int64_t ch;

  /* phi factor (n = K; n <= 1 evaluates sequentially, identical value) */
  f = 0.0;
  ch = chunk_size(K);
  for (int64_t c0 = 0; c0 < K; c0 += ch) {
    double acc = 0.0;
    for (int64_t k = c0; k < c0 + ch && k < K; ++k) acc += log_pdf_dirichlet_sym(phi + k * V, m->beta, V);
    f += acc;
  }
  total += f;

  f = 0.0;
  ch = chunk_size(M);
  for (int64_t c0 = 0; c0 < M; c0 += ch) {
    double acc = 0.0;
    for (int64_t d = c0; d < c0 + ch && d < M; ++d) acc += log_pdf_dirichlet_sym(theta + d * K, m->alpha, K);
    f += acc;
  }
  total += f;

  f = 0.0;
  for (int64_t c0 = 0; c0 < M; c0 += ch) {
    double acc = 0.0;
    for (int64_t d = c0; d < c0 + ch && d < M; ++d) {
      double in = 0.0;
      for (int64_t t = m->offsets[d]; t < m->offsets[d + 1]; ++t)
        in += bo_log_pmf_categorical(z[t], theta + d * K, K);
      acc += in;
    }
    f += acc;
  }
  total += f;

  f = 0.0;
  for (int64_t c0 = 0; c0 < M; c0 += ch) {
    double acc = 0.0;
    for (int64_t d = c0; d < c0 + ch && d < M; ++d) {
      double in = 0.0;
      for (int64_t t = m->offsets[d]; t < m->offsets[d + 1]; ++t) {
        const int64_t k = z[t];
        in += (k >= 0 && k < K) ? bo_log_pmf_categorical(m->w[t], phi + k * V, V) : -INFINITY;
      }
      acc += in;
    }
    f += acc;
  }
  total += f;
  return total;
}

int bo_lda_sweep(const bo_lda* m, int64_t* z, double* phi, double* theta, uint64_t seed,
                 int64_t iter, int observe_phi, double* log_joint) {
  /* Engine::sweep (sampler.cpp:390-405): blocks in plan order phi, theta, z. */
  if (!observe_phi) {
    int64_t* nkw = (int64_t*)calloc((size_t)(m->K * m->V), sizeof(int64_t));
    if (!nkw) return fail("out of memory");
    int rc = bo_lda_count_phi(m, z, 0, m->M, nkw);
    if (!rc) rc = bo_lda_draw_phi(m, nkw, seed, iter, phi);
    free(nkw);
    if (rc) return rc;
  }
  const int rc = bo_lda_theta_z(m, z, phi, theta, seed, iter, 0, m->M);
  if (rc) return rc;
  if (log_joint) *log_joint = bo_lda_log_joint(m, z, phi, theta);
  return 0;
}

int bo_lda_prior_init(const bo_lda* m, uint64_t seed, double* phi, double* theta, int64_t* z) {
  /* prior_init: one stream keyed(seed,5,var,elem) per element, declaration order
   * (sampler.cpp:542-555); Dirichlet rows draw all gammas from that one stream
   * (draw_dirichlet, dist.cpp:193-200); z by linear-scan draw_categorical. */
  const int64_t K = m->K, V = m->V, M = m->M;
  double* a = (double*)malloc(sizeof(double) * (size_t)(V > K ? V : K));
  if (!a) return fail("out of memory");
  for (int64_t i = 0; i < V; ++i) a[i] = m->beta;
  for (int64_t k = 0; k < K; ++k) {
    bo_rng g = stream(bo_keyed(seed, P_INIT, (uint64_t)m->var_phi, (uint64_t)k, 0));
    bo_draw_dirichlet(&g, a, V, phi + k * V);
  }
  for (int64_t i = 0; i < K; ++i) a[i] = m->alpha;
  for (int64_t d = 0; d < M; ++d) {
    bo_rng g = stream(bo_keyed(seed, P_INIT, (uint64_t)m->var_theta, (uint64_t)d, 0));
    bo_draw_dirichlet(&g, a, K, theta + d * K);
  }
  for (int64_t d = 0; d < M; ++d) {
    for (int64_t t = m->offsets[d]; t < m->offsets[d + 1]; ++t) {
      bo_rng g = stream(bo_keyed(seed, P_INIT, (uint64_t)m->var_z, (uint64_t)t, 0));
      z[t] = bo_draw_categorical(&g, theta + d * K, K);
    }
  }
  free(a);
  return 0;
}

double bo_lda_lpp(const double* phi, const double* theta, int64_t K, int64_t V,
                  const int64_t* w, const int64_t* offsets, int64_t docs) {
  /* log_predictive_probability (metrics.cpp:9-34): sum log10 sum_k theta[d,k] phi[k,w]. */
  double total = 0.0;
  for (int64_t d = 0; d < docs; ++d) {
    const double* th = theta + d * K;
    for (int64_t t = offsets[d]; t < offsets[d + 1]; ++t) {
      double p = 0.0;
      for (int64_t k = 0; k < K; ++k) p += th[k] * phi[k * V + w[t]];
      total += log10(p);
    }
  }
  return total;
}

/* ---------------------------------------------------------------------------
 * GMM
 * ------------------------------------------------------------------------- */
/* reduce_accumulate (executor.cpp:99-114): per-chunk zeroed partials folded in chunk
 * order into the zeroed stats buffer. */
static void gmm_stats(const bo_gmm* m, const int64_t* z, const double* mu, const double* sigma2,
                      int which, double* stats /* K*2 */) {
  const int64_t N = m->N, K = m->K, ch = chunk_size(N);
  double* part = (double*)malloc(sizeof(double) * (size_t)(2 * K));
  for (int64_t j = 0; j < 2 * K; ++j) stats[j] = 0.0;
  for (int64_t c0 = 0; c0 < N; c0 += ch) {
    for (int64_t j = 0; j < 2 * K; ++j) part[j] = 0.0;
    for (int64_t i = c0; i < c0 + ch && i < N; ++i) {
      const int64_t k = z[i];
      double* a = part + k * 2;
      const double x = m->x[i];
      if (which == 0) { /* GaussianMean (sampler.cpp:114-121) */
        const double v = sigma2[k];
        a[0] += 1.0 / v;
        a[1] += x / v;
      } else { /* InverseGammaVariance (sampler.cpp:122-130) */
        const double mean = mu[k];
        a[0] += 1.0;
        a[1] += (x - mean) * (x - mean);
      }
    }
    for (int64_t j = 0; j < 2 * K; ++j) stats[j] += part[j];
  }
  free(part);
}

int bo_gmm_sweep(const bo_gmm* m, int64_t* z, double* pi, double* mu, double* sigma2,
                 uint64_t seed, int64_t iter, double* log_joint) {
  const int64_t N = m->N, K = m->K;
  for (int64_t i = 0; i < N; ++i)
    if (z[i] < 0 || z[i] >= K) return fail("conjugate update bin out of range");
  double* buf = (double*)malloc(sizeof(double) * (size_t)(4 * K));
  double* stats = buf;      /* 2K */
  double* alpha = buf + 2 * K;
  double* logw = buf + 3 * K;

  /* pi block: Dirichlet-Categorical over the single row (rows = 1, cols = K). */
  for (int64_t k = 0; k < K; ++k) alpha[k] = 0.0;
  for (int64_t i = 0; i < N; ++i) alpha[z[i]] += 1.0;
  for (int64_t k = 0; k < K; ++k) alpha[k] = m->alpha + alpha[k];
  bo_dirichlet_batch(1, K, alpha, bo_keyed(seed, P_CONJUGATE, (uint64_t)m->var_pi, (uint64_t)iter, 0), pi);

  /* mu block: stats with the current sigma2, draw_gaussian (sampler.cpp:199-204). */
  gmm_stats(m, z, mu, sigma2, 0, stats);
  {
    const uint64_t key = bo_keyed(seed, P_CONJUGATE, (uint64_t)m->var_mu, (uint64_t)iter, 0);
    for (int64_t t = 0; t < K; ++t) {
      bo_rng g = stream(bo_derive(key, (uint64_t)t, 0));
      const double s0 = m->mu0, s1 = m->v0;
      const double n = stats[t * 2], s = stats[t * 2 + 1];
      const double prec = 1.0 / s1 + n;
      const double wsum = s0 / s1 + s;
      const double post_var = 1.0 / prec;
      mu[t] = post_var * wsum + sqrt(post_var) * bo_next_gaussian(&g); /* draw_gaussian */
    }
  }
  /* sigma2 block: stats with the new mu, draw_inverse_gamma (sampler.cpp:206-208). */
  gmm_stats(m, z, mu, sigma2, 1, stats);
  {
    const uint64_t key = bo_keyed(seed, P_CONJUGATE, (uint64_t)m->var_sigma2, (uint64_t)iter, 0);
    for (int64_t t = 0; t < K; ++t) {
      bo_rng g = stream(bo_derive(key, (uint64_t)t, 0));
      const double n = stats[t * 2], s = stats[t * 2 + 1];
      const double scale = m->b0 + 0.5 * s;
      sigma2[t] = scale / bo_draw_gamma(&g, m->a0 + 0.5 * n);
    }
  }
  /* z block: logw[v] = (0 + log pi[v]) + log N(x | mu_v, sigma2_v). */
  for (int64_t i = 0; i < N; ++i) {
    for (int64_t v = 0; v < K; ++v) {
      double lp = 0.0;
      lp += bo_log_pmf_categorical(v, pi, K);
      lp += bo_log_pdf_gaussian(m->x[i], mu[v], sigma2[v]);
      logw[v] = lp;
    }
    bo_rng g = stream(bo_keyed(seed, P_DISCRETE, (uint64_t)m->var_z, (uint64_t)i, (uint64_t)iter));
    const int64_t k = bo_draw_from_log_weights(&g, logw, K);
    if (k < 0) {
      free(buf);
      return 1;
    }
    z[i] = k;
  }
  free(buf);
  if (log_joint) *log_joint = bo_gmm_log_joint(m, z, pi, mu, sigma2);
  return 0;
}

double bo_gmm_log_joint(const bo_gmm* m, const int64_t* z, const double* pi, const double* mu,
                        const double* sigma2) {
  /* p(pi) prod_k p(mu[k]) prod_m p(sigma2[m]) prod_i p(z|pi) prod_i p(x|mu,sigma2)
   * (tests/golden/describe_gmm.txt), chunked as in eval.cpp:393-422. */
  const int64_t N = m->N, K = m->K;
  double total = 0.0, f;
  int64_t ch;
  total += log_pdf_dirichlet_sym(pi, m->alpha, K);
  ch = chunk_size(K);
  f = 0.0;
  for (int64_t c0 = 0; c0 < K; c0 += ch) {
    double acc = 0.0;
    for (int64_t k = c0; k < c0 + ch && k < K; ++k) acc += bo_log_pdf_gaussian(mu[k], m->mu0, m->v0);
    f += acc;
  }
  total += (K > 1) ? f : bo_log_pdf_gaussian(mu[0], m->mu0, m->v0);
  f = 0.0;
  for (int64_t c0 = 0; c0 < K; c0 += ch) {
    double acc = 0.0;
    for (int64_t k = c0; k < c0 + ch && k < K; ++k) acc += bo_log_pdf_inverse_gamma(sigma2[k], m->a0, m->b0);
    f += acc;
  }
  total += f;
  ch = chunk_size(N);
  f = 0.0;
  for (int64_t c0 = 0; c0 < N; c0 += ch) {
    double acc = 0.0;
    for (int64_t i = c0; i < c0 + ch && i < N; ++i) acc += bo_log_pmf_categorical(z[i], pi, K);
    f += acc;
  }
  total += f;
  f = 0.0;
  for (int64_t c0 = 0; c0 < N; c0 += ch) {
    double acc = 0.0;
    for (int64_t i = c0; i < c0 + ch && i < N; ++i) {
      const int64_t k = z[i];
      acc += (k >= 0 && k < K) ? bo_log_pdf_gaussian(m->x[i], mu[k], sigma2[k]) : -INFINITY;
    }
    f += acc;
  }
  total += f;
  return total;
}

int bo_gmm_prior_init(const bo_gmm* m, uint64_t seed, double* pi, double* mu, double* sigma2,
                      int64_t* z) {
  const int64_t K = m->K;
  double* a = (double*)malloc(sizeof(double) * (size_t)K);
  for (int64_t k = 0; k < K; ++k) a[k] = m->alpha;
  bo_rng g = stream(bo_keyed(seed, P_INIT, (uint64_t)m->var_pi, 0, 0));
  bo_draw_dirichlet(&g, a, K, pi);
  free(a);
  for (int64_t k = 0; k < K; ++k) {
    g = stream(bo_keyed(seed, P_INIT, (uint64_t)m->var_mu, (uint64_t)k, 0));
    mu[k] = m->mu0 + sqrt(m->v0) * bo_next_gaussian(&g);
  }
  for (int64_t k = 0; k < K; ++k) {
    g = stream(bo_keyed(seed, P_INIT, (uint64_t)m->var_sigma2, (uint64_t)k, 0));
    sigma2[k] = m->b0 / bo_draw_gamma(&g, m->a0);
  }
  for (int64_t i = 0; i < m->N; ++i) {
    g = stream(bo_keyed(seed, P_INIT, (uint64_t)m->var_z, (uint64_t)i, 0));
    z[i] = bo_draw_categorical(&g, pi, K);
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * MH over i.i.d. rows -- run_mh_block (sampler.cpp:284-340)
 * ------------------------------------------------------------------------- */
static double softplus(double s) { return s > 0.0 ? s + log1p(exp(-s)) : log1p(exp(s)); }

/* Row likelihood factor reduced over rows in <= 64 chunks. */
static double mh_lik(const bo_mh* m, const double* w, double b, double tau) {
  const int64_t N = m->N, K = m->K, ch = chunk_size(N);
  double f = 0.0;
  for (int64_t c0 = 0; c0 < N; c0 += ch) {
    double acc = 0.0;
    for (int64_t i = c0; i < c0 + ch && i < N; ++i) {
      const double* xi = m->x + i * K;
      double s = 0.0; /* SumLoop (eval.cpp:255-264) */
      for (int64_t j = 0; j < K; ++j) s += w[j] * xi[j];
      s = s + b;
      if (m->logistic) {
        acc += m->y[i] * s - softplus(s);
      } else {
        acc += bo_log_pdf_gaussian(m->y[i], s, tau);
      }
    }
    f += acc;
  }
  return N > 1 ? f : f; /* n <= 1 evaluates sequentially: same value */
}

static double mh_prior_w(const bo_mh* m, const double* w) {
  const int64_t K = m->K, ch = chunk_size(K);
  double f = 0.0;
  for (int64_t c0 = 0; c0 < K; c0 += ch) {
    double acc = 0.0;
    for (int64_t j = c0; j < c0 + ch && j < K; ++j) acc += bo_log_pdf_gaussian(w[j], 0.0, m->w_var);
    f += acc;
  }
  return f;
}

double bo_mh_blanket(const bo_mh* m, const double* w, double b, double tau) {
  /* plan.cpp:121-137: blanket = var factors mentioning w, b or tau, declaration order. */
  double s = 0.0;
  s += mh_prior_w(m, w);
  s += bo_log_pdf_gaussian(b, 0.0, m->b_var);
  if (!m->logistic) s += bo_log_pdf_inverse_gamma(tau, m->tau_a, m->tau_b);
  s += mh_lik(m, w, b, tau);
  return s;
}

double bo_mh_log_joint(const bo_mh* m, const double* w, double b, double tau) {
  const int64_t N = m->N, K = m->K, ch = chunk_size(N);
  double total = 0.0;
  total += mh_prior_w(m, w);
  total += bo_log_pdf_gaussian(b, 0.0, m->b_var);
  if (!m->logistic) total += bo_log_pdf_inverse_gamma(tau, m->tau_a, m->tau_b);
  double f = 0.0; /* prod_i prod_j p(x[i,j]) -- Uniform(lo, hi) */
  for (int64_t c0 = 0; c0 < N; c0 += ch) {
    double acc = 0.0;
    for (int64_t i = c0; i < c0 + ch && i < N; ++i) {
      double in = 0.0;
      for (int64_t j = 0; j < K; ++j) in += bo_log_pdf_uniform(m->x[i * K + j], m->lo, m->hi);
      acc += in;
    }
    f += acc;
  }
  total += f;
  total += mh_lik(m, w, b, tau);
  return total;
}

int bo_mh_step(const bo_mh* m, double* w, double* b, double* tau, uint64_t seed, int64_t iter,
               double* log_joint, int* accepted) {
  const int64_t K = m->K;
  const double before = bo_mh_blanket(m, w, *b, *tau);
  double* old_w = (double*)malloc(sizeof(double) * (size_t)K);
  memcpy(old_w, w, sizeof(double) * (size_t)K);
  const double old_b = *b, old_tau = *tau;
  /* Proposals: keyed(seed,1,var,t,iter), arr[t] += mh_scale * N(0,1) (sampler.cpp:311-318). */
  for (int64_t t = 0; t < K; ++t) {
    bo_rng g = stream(bo_keyed(seed, P_PROPOSAL, (uint64_t)m->var_w, (uint64_t)t, (uint64_t)iter));
    w[t] += m->mh_scale * bo_next_gaussian(&g);
  }
  {
    bo_rng g = stream(bo_keyed(seed, P_PROPOSAL, (uint64_t)m->var_b, 0, (uint64_t)iter));
    *b += m->mh_scale * bo_next_gaussian(&g);
  }
  if (!m->logistic) {
    bo_rng g = stream(bo_keyed(seed, P_PROPOSAL, (uint64_t)m->var_tau, 0, (uint64_t)iter));
    *tau += m->mh_scale * bo_next_gaussian(&g);
  }
  const double after = bo_mh_blanket(m, w, *b, *tau);
  const double delta = after - before;
  bo_rng acc = stream(bo_keyed(seed, P_ACCEPT, (uint64_t)m->var_w, (uint64_t)iter, 0));
  const int take = isfinite(after) && log(bo_next_unit(&acc)) < delta; /* :325-328 */
  if (!take) {
    memcpy(w, old_w, sizeof(double) * (size_t)K);
    *b = old_b;
    *tau = old_tau;
  }
  free(old_w);
  if (accepted) *accepted = take;
  if (log_joint) *log_joint = bo_mh_log_joint(m, w, *b, *tau);
  return 0;
}
