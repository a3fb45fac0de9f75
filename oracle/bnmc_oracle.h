/* oracle/bnmc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's data-parallel MCMC sweep
 * used as the CPU checker for the CUDA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Pinning: every routine here is checked bit-for-bit against the compiled reference
 * (oracle/_ref/libbnmc_ref.so, built from /root/reference/proj/src by oracle/Makefile)
 * and against the committed golden vectors in tests/golden/ (tests/test_oracle.py).
 * The logistic-regression likelihood has no reference implementation (the DSL has
 * no exp/log: proj/src/parser.cpp:471-474) -- that one routine is "parity unpinned"
 * and is anchored only on the MH machinery it shares with bo_linreg_mh_step.
 *
 * Conventions mirror the reference store (proj/include/bnmc/store.hpp:44-83):
 * int64 assignments, fp64 row-major parameters, ragged documents as prefix sums.
 * Functions return 0 on success, non-zero on the errors the reference throws
 * (RuntimeError / std::domain_error / std::invalid_argument); bo_last_error()
 * names the problem.
 */
#ifndef BNMC_ORACLE_H
#define BNMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* bo_last_error(void);

/* ---- counter RNG: proj/include/bnmc/rng.hpp:12-51 ---- */
typedef struct {
  uint64_t key;
  uint64_t counter;
} bo_rng;

uint64_t bo_mix(uint64_t z);
uint64_t bo_fold(uint64_t k, uint64_t v);
uint64_t bo_keyed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d);
uint64_t bo_derive(uint64_t key, uint64_t a, uint64_t b);
uint64_t bo_next_u64(bo_rng* r);
double bo_next_unit(bo_rng* r);
double bo_next_gaussian(bo_rng* r);

/* ---- distributions: proj/src/dist.cpp ---- */
double bo_draw_gamma(bo_rng* r, double shape);                 /* dist.cpp:136-155 */
int64_t bo_draw_categorical(bo_rng* r, const double* p, int64_t n); /* dist.cpp:183-191 */
void bo_draw_dirichlet(bo_rng* r, const double* alpha, int64_t n, double* out); /* dist.cpp:193-200 */
/* dist.cpp:202-215; returns -1 (error set) when every weight is -inf/NaN. */
int64_t bo_draw_from_log_weights(bo_rng* r, const double* logw, int64_t n);
double bo_log_pdf_gaussian(double x, double mean, double var);      /* dist.cpp:61-68 */
double bo_log_pdf_uniform(double x, double lo, double hi);          /* dist.cpp:70-75 */
double bo_log_pdf_inverse_gamma(double x, double shape, double scale); /* dist.cpp:92-97 */
double bo_log_pmf_categorical(int64_t x, const double* p, int64_t n);  /* dist.cpp:107-113 */
double bo_log_pdf_dirichlet(const double* x, const double* alpha, int64_t n); /* dist.cpp:115-130 */

/* sample_dirichlet_batch, per-row concentrations (proj/src/batch.cpp:38-63):
 * cell (r,c) uses stream derive(key, r, c); rows normalised left to right. */
int bo_dirichlet_batch(int64_t rows, int64_t cols, const double* alpha, uint64_t key,
                       double* out);

/* ---- LDA (proj/models/lda.bn): var ids phi=0, theta=1, z=2, w=3 ---- */
typedef struct {
  int64_t K, V, M;
  const int64_t* offsets; /* M+1 prefix sums of document lengths (eval.cpp:117-127) */
  const int64_t* w;       /* offsets[M] observed word ids */
  double alpha;           /* theta prior concentration (lda.bn alpha = vector(K, 0.1)) */
  double beta;            /* phi prior concentration (lda.bn beta = vector(V, 0.1)) */
  int32_t var_phi, var_theta, var_z;
} bo_lda;

/* Topic-word counts over documents [d0,d1): nkw[k*V+v] += 1 (sampler.cpp:61-136). */
int bo_lda_count_phi(const bo_lda* m, const int64_t* z, int64_t d0, int64_t d1, int64_t* nkw);
/* phi block draw from counts (sampler.cpp:138-181 + batch.cpp). */
int bo_lda_draw_phi(const bo_lda* m, const int64_t* nkw, uint64_t seed, int64_t iter,
                    double* phi);
/* The phi block's unnormalised gamma cells g[k*V+v] for v in [v0,v1) (batch.cpp:38-41). */
int bo_lda_phi_gammas(const bo_lda* m, const int64_t* nkw, uint64_t seed, int64_t iter, int64_t v0,
                      int64_t v1, double* g);
/* theta block (counts + draw) then z block for documents [d0,d1) (sampler.cpp:222-265). */
int bo_lda_theta_z(const bo_lda* m, int64_t* z, const double* phi, double* theta, uint64_t seed,
                   int64_t iter, int64_t d0, int64_t d1);
/* Engine::sweep for LDA: blocks phi, theta, z then the log-joint (sampler.cpp:390-405).
 * observe_phi != 0 drops the phi block (the lpp_curve protocol, bench.cpp:30-77). */
int bo_lda_sweep(const bo_lda* m, int64_t* z, double* phi, double* theta, uint64_t seed,
                 int64_t iter, int observe_phi, double* log_joint);
/* eval_log_joint with the reference's 64-chunk reduction order (eval.cpp:393-422). */
double bo_lda_log_joint(const bo_lda* m, const int64_t* z, const double* phi,
                        const double* theta);
/* prior_init for phi, theta, z (sampler.cpp:542-555, 457-540). */
int bo_lda_prior_init(const bo_lda* m, uint64_t seed, double* phi, double* theta, int64_t* z);
/* log_predictive_probability (proj/src/metrics.cpp:9-34), uniform or ragged held-out docs. */
double bo_lda_lpp(const double* phi, const double* theta, int64_t K, int64_t V,
                  const int64_t* w, const int64_t* offsets, int64_t docs);

/* ---- GMM (proj/models/gmm.bn): pi=0, mu=1, sigma2=2, z=3, x=4 ---- */
typedef struct {
  int64_t N, K;
  const double* x;
  double alpha;           /* pi prior concentration (0.1) */
  double mu0, v0;         /* mu prior Gaussian(0, 10) */
  double a0, b0;          /* sigma2 prior InverseGamma(1, 1) */
  int32_t var_pi, var_mu, var_sigma2, var_z;
} bo_gmm;

int bo_gmm_sweep(const bo_gmm* m, int64_t* z, double* pi, double* mu, double* sigma2,
                 uint64_t seed, int64_t iter, double* log_joint);
double bo_gmm_log_joint(const bo_gmm* m, const int64_t* z, const double* pi, const double* mu,
                        const double* sigma2);
int bo_gmm_prior_init(const bo_gmm* m, uint64_t seed, double* pi, double* mu, double* sigma2,
                      int64_t* z);

/* ---- MH over i.i.d. rows (run_mh_block, sampler.cpp:284-340) ----
 * linreg  = proj/models/regression.bn: w=0 (K), b=1, tau=2, x=3 (observed), y=4 (observed)
 * logreg  = same priors on w,b with y ~ Bernoulli(sigmoid(w.x+b)); vars w=0, b=1, x=2, y=3.
 *           (no reference model: parity unpinned for the likelihood itself) */
typedef struct {
  int64_t N, K;
  const double* x;  /* N*K row-major */
  const double* y;  /* N */
  double lo, hi;    /* x ~ Uniform(lo, hi) */
  double w_var, b_var;      /* Gaussian(0, 10) priors */
  double tau_a, tau_b;      /* InverseGamma(3, 1) (linreg only) */
  double mh_scale;          /* RunConfig::mh_scale (0.5) */
  int32_t var_w, var_b, var_tau;
  int32_t logistic;         /* 0 = linreg (regression.bn), 1 = logreg */
} bo_mh;

/* One MH step + the log-joint (Engine::sweep semantics).  tau ignored for logreg. */
int bo_mh_step(const bo_mh* m, double* w, double* b, double* tau, uint64_t seed, int64_t iter,
               double* log_joint, int* accepted);
double bo_mh_log_joint(const bo_mh* m, const double* w, double b, double tau);
/* Sum over blanket factors (the MH "before"/"after" score). */
double bo_mh_blanket(const bo_mh* m, const double* w, double b, double tau);

#ifdef __cplusplus
}
#endif
#endif
