// csrc/mh.cu -- random-walk Metropolis-Hastings over i.i.d. rows
// (Engine::run_mh_block, proj/src/sampler.cpp:284-340).
//
// Models: proj/models/regression.bn (y ~ N(w.x + b, tau), method MH; with
// BNMC_GPU_TAU_PRECISION the precision variant y ~ N(w.x + b, pow(tau, -1)), tau ~ Gamma,
// oracle/models/regprec.bn -- the GammaPrecision conjugate kind) and its
// logistic twin (y ~ Bernoulli(sigmoid(w.x + b)); no reference model exists, the
// MH machinery is shared).  The reference evaluates the blanket before, the
// blanket after, and the full log-joint: three passes over the N x K data.  Here
// the current state's blanket is cached on the device, so one step is ONE pass:
//
//   propose_kernel   w' = w + s*N(0,1) from keyed(seed,1,var,t,iter) (:311-318)
//   lik_kernel       per-row log-likelihood of the proposal, warp per row,
//                    fixed-grid partial sums (the data-parallel reduction)
//   [allreduce]      NCCL double sum of the partial (row-sharded, world > 1)
//   accept_kernel    after = priors(w') + lik; accept iff isfinite(after) &&
//                    log(u) < after - before, u from keyed(seed,2,vars[0],iter)
//                    (:321-328); commit or keep; log-joint
//                    = Fw + Fb + Ftau + Fx + Fy in the reference's order.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "dist.cuh"

namespace bnmc_gpu {
namespace {

constexpr int kThreads = 256;
constexpr int kBlocks = 148 * 8;

struct MhArgs {
  std::int64_t N;  // local rows
  int K;
  const double* x;
  const double* y;
  double* w;      // [K+2]: w..., b, tau (current)
  double* wp;     // [K+2]: proposal
  double* part;   // [kBlocks]
  double* state;  // [8]: cur_lik, cur_fw, cur_fb, cur_ftau, fx, lik_prop, -, -
  double lo, hi, w_var, b_var, tau_a, tau_b, mh_scale;
  std::uint64_t seed;
  int var_w, var_b, var_tau;
  int logistic;
  int notau;        // logistic or polyreg: no tau variable (polyreg: y ~ N(mean, 1.0))
  int prec;         // tau is a precision: y ~ N(mean, pow(tau, -1)), tau ~ Gamma(tau_a, tau_b)
  const double* xr; // fx factor input: raw x (polyreg: N scalars) or the feature matrix
  std::int64_t nfx; // its length
};

__device__ __forceinline__ double softplus(double s) {
  return s > 0.0 ? s + log1p(exp(-s)) : log1p(exp(s));
}

__global__ void propose_kernel(MhArgs a, const std::int64_t* iter_p) {
  const std::int64_t iter = *iter_p;
  for (int t = threadIdx.x; t < a.K + 2; t += blockDim.x) {
    double v = a.w[t];
    if (t < a.K) {
      Stream r(keyed(a.seed, kProposal, static_cast<std::uint64_t>(a.var_w), static_cast<std::uint64_t>(t),
                     static_cast<std::uint64_t>(iter)));
      v += a.mh_scale * r.next_gaussian();
    } else if (t == a.K) {
      Stream r(keyed(a.seed, kProposal, static_cast<std::uint64_t>(a.var_b), 0, static_cast<std::uint64_t>(iter)));
      v += a.mh_scale * r.next_gaussian();
    } else if (!a.notau) {
      Stream r(keyed(a.seed, kProposal, static_cast<std::uint64_t>(a.var_tau), 0, static_cast<std::uint64_t>(iter)));
      v += a.mh_scale * r.next_gaussian();
    }
    a.wp[t] = v;
  }
}

// Sum over local rows of the row log-likelihood at parameters p (K + 2 values).
// A group of 8 lanes per row: lane gl reads the row's 4-feature chunks gl, gl+8, ...
// with one 256-bit load each (8 lanes = 256 contiguous bytes per request), keeps its
// slice of w in registers, and the dot product is a fixed 3-step butterfly; a group
// takes 4 consecutive rows per iteration and lane r evaluates row r's log-likelihood.
constexpr int kRowGroup = 8;
constexpr int kMaxChunks = 8;  // K <= 4 * 8 * kMaxChunks = 256 on the vector path

__device__ __forceinline__ void ldg256(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// y's variance from the tau variable: tau itself (regression.bn), or pow(tau, -1) for a
// precision (the reference evaluates std::pow(tau, -1.0), correctly rounded like 1 / tau)
__device__ __forceinline__ double tau_variance(const MhArgs& a, double tau) { return a.prec ? 1.0 / tau : tau; }

__device__ __forceinline__ double row_loglik(const MhArgs& a, double s, double yi, double var) {
  return a.logistic ? yi * s - softplus(s) : log_pdf_gaussian(yi, s, var);
}

// log p(tau): InverseGamma(shape, scale) variance or Gamma(shape, scale) precision
__device__ __forceinline__ double tau_prior(const MhArgs& a, double tau) {
  return a.prec ? log_pdf_gamma(tau, a.tau_a, a.tau_b) : log_pdf_inverse_gamma(tau, a.tau_a, a.tau_b);
}

template <bool VEC, int CPL = 1>  // CPL: 4-feature chunks per lane (vector path)
__global__ void __launch_bounds__(kThreads) lik_kernel(MhArgs a, const double* p, double* part) {
  extern __shared__ double wsh[];
  __shared__ double scratch[32];
  for (int j = threadIdx.x; j < a.K + 2; j += blockDim.x) wsh[j] = p[j];
  __syncthreads();
  const double b = wsh[a.K], tau = tau_variance(a, wsh[a.K + 1]);
  double acc = 0.0;
  if constexpr (VEC) {
    const int gl = threadIdx.x & (kRowGroup - 1);
    const unsigned gm = 0xffu << ((threadIdx.x & 31) & ~(kRowGroup - 1));
    const int chunks = a.K / 4;
    double wr[CPL][4];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = 4 * (gl + kRowGroup * c);
#pragma unroll
      for (int e = 0; e < 4; ++e) wr[c][e] = j < a.K ? wsh[j + e] : 0.0;
    }
    const std::int64_t g = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) / kRowGroup;
    const std::int64_t ng = static_cast<std::int64_t>(gridDim.x) * blockDim.x / kRowGroup;
    // kRows consecutive rows per group iteration: all their loads are issued before
    // any reduction (kRows * CPL 256-bit loads in flight per lane), and the rows'
    // log-likelihoods (exp/log1p chains) run on kRows different lanes of the group
    // instead of serially on lane 0.
    constexpr int kRows = 4;
    for (std::int64_t i0 = g * kRows; i0 < a.N; i0 += ng * kRows) {
      double xv[kRows][CPL][4];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const double* xi = a.x + (i0 + r) * a.K;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int ch = gl + kRowGroup * c;
          if (ch < chunks && i0 + r < a.N) {
            ldg256(xi + 4 * ch, xv[r][c][0], xv[r][c][1], xv[r][c][2], xv[r][c][3]);
          } else {
            xv[r][c][0] = xv[r][c][1] = xv[r][c][2] = xv[r][c][3] = 0.0;
          }
        }
      }
      double mine = 0.0;
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          s += wr[c][0] * xv[r][c][0];
          s += wr[c][1] * xv[r][c][1];
          s += wr[c][2] * xv[r][c][2];
          s += wr[c][3] * xv[r][c][3];
        }
#pragma unroll
        for (int o = kRowGroup / 2; o > 0; o >>= 1) s += __shfl_xor_sync(gm, s, o, kRowGroup);
        if (gl == r) mine = s;
      }
      if (gl < kRows && i0 + gl < a.N) acc += row_loglik(a, mine + b, __ldg(a.y + i0 + gl), tau);
    }
  } else {
    // any K: warp per row, lanes stride the features
    const int lane = threadIdx.x & 31;
    const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (std::int64_t i = warp; i < a.N; i += nwarps) {
      const double* xi = a.x + i * a.K;
      double s = 0.0;
      for (int j = lane; j < a.K; j += 32) s += wsh[j] * __ldg(xi + j);
      s = warp_sum(s) + b;
      if (lane == 0) acc += row_loglik(a, s, __ldg(a.y + i), tau);
    }
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// log prod_{i,j} Uniform(x_ij | lo, hi): -log(hi - lo) each, -inf outside [lo, hi].
__global__ void fx_kernel(MhArgs a, double* part) {
  __shared__ double scratch[32];
  double acc = 0.0;
  const double c = -log(a.hi - a.lo);
  const std::int64_t n = a.nfx;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const double v = a.xr[i];
    acc += (!(a.hi > a.lo) || v < a.lo || v > a.hi) ? -INFINITY : c;
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__device__ double priors(const MhArgs& a, const double* p, double* fw, double* fb, double* ftau) {
  double s = 0.0;
  for (int j = 0; j < a.K; ++j) s += log_pdf_gaussian(p[j], 0.0, a.w_var);
  *fw = s;
  *fb = log_pdf_gaussian(p[a.K], 0.0, a.b_var);
  *ftau = a.notau ? 0.0 : tau_prior(a, p[a.K + 1]);
  return a.notau ? (*fw + *fb) : ((*fw + *fb) + *ftau);
}

// priors() with the K weight terms evaluated by the block's threads (each term bitwise the
// sequential one) and summed by thread 0 in j order, as priors() does: same value, no
// K-long chain of log-pdf evaluations on one thread.  Call with every thread; the result
// is valid in thread 0.  K > kPriorTerms falls back to priors().
constexpr int kPriorTerms = 1024;

__device__ double priors_block(const MhArgs& a, const double* p, double* fw, double* fb, double* ftau, double* terms) {
  if (a.K > kPriorTerms) {
    double r = 0.0;
    if (threadIdx.x == 0) r = priors(a, p, fw, fb, ftau);
    return r;
  }
  for (int j = threadIdx.x; j < a.K; j += blockDim.x) terms[j] = log_pdf_gaussian(p[j], 0.0, a.w_var);
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int j = 0; j < a.K; ++j) s += terms[j];
    *fw = s;
    *fb = log_pdf_gaussian(p[a.K], 0.0, a.b_var);
    *ftau = a.notau ? 0.0 : tau_prior(a, p[a.K + 1]);
    r = a.notau ? (*fw + *fb) : ((*fw + *fb) + *ftau);
  }
  return r;
}

__device__ double sum_parts(const double* part, int n, double* scratch) {
  double s = 0.0;
  for (int b = threadIdx.x; b < n; b += blockDim.x) s += part[b];
  return block_sum(s, scratch);
}

// mode 0: initialise the cache from the current state (no step);
// mode 1: MH step; mode 2: log-joint of the current state only;
// mode 3: as 0, and advance the iteration (end of a Gibbs / MWG sweep).
__global__ void accept_kernel(MhArgs a, Outputs o, int mode, const double* lik_total) {
  __shared__ double scratch[32];
  __shared__ double terms[kPriorTerms];
  __shared__ int take_s;
  const double lik = sum_parts(a.part, kBlocks, scratch);
  const double fx = a.state[4];
  double fw = 0.0, fb = 0.0, ft = 0.0, pr = 0.0;
  if (mode == 0 || mode == 3) pr = priors_block(a, a.w, &fw, &fb, &ft, terms);
  else if (mode == 1) pr = priors_block(a, a.wp, &fw, &fb, &ft, terms);
  if (threadIdx.x == 0) {
    const std::int64_t it = *o.iter;
    const double lik_all = lik_total ? *lik_total : lik;
    int take = 0;
    if (mode == 0 || mode == 3) {
      a.state[0] = lik_all;
      a.state[1] = fw;
      a.state[2] = fb;
      a.state[3] = ft;
    } else if (mode == 1) {
      const double after = pr + lik_all;
      const double before = a.notau ? ((a.state[1] + a.state[2]) + a.state[0])
                                       : (((a.state[1] + a.state[2]) + a.state[3]) + a.state[0]);
      const double delta = after - before;
      Stream acc(keyed(a.seed, kAccept, static_cast<std::uint64_t>(a.var_w), static_cast<std::uint64_t>(it)));
      take = isfinite(after) && log(acc.next_unit()) < delta;
      if (take) {
        a.state[0] = lik_all;
        a.state[1] = fw;
        a.state[2] = fb;
        a.state[3] = ft;
      }
    }
    take_s = take;
    const double lj = a.notau ? (((a.state[1] + a.state[2]) + fx) + a.state[0])
                                 : ((((a.state[1] + a.state[2]) + a.state[3]) + fx) + a.state[0]);
    o.lj[it & (kRing - 1)] = lj;
    o.acc[it & (kRing - 1)] = mode == 3 ? static_cast<int>(a.state[5]) : take;
    if (mode == 1 || mode == 3) *o.iter = it + 1;
  }
  __syncthreads();
  if (mode == 1 && take_s)
    for (int t = threadIdx.x; t < a.K + 2; t += blockDim.x) a.w[t] = a.wp[t];
}

__global__ void fx_finalize_kernel(MhArgs a, const double* fx_total) {
  __shared__ double scratch[32];
  const double s = sum_parts(a.part, kBlocks, scratch);
  if (threadIdx.x == 0) a.state[4] = fx_total ? *fx_total : s;
}

// prior_init: w_t ~ N(0, w_var), b ~ N(0, b_var), tau ~ IG(tau_a, tau_b), one stream
// keyed(seed,5,var,t) per element (sampler.cpp:542-555, draw_gaussian dist.cpp:161-163).
__global__ void prior_kernel(MhArgs a, std::uint64_t seed) {
  for (int t = threadIdx.x; t < a.K + 2; t += blockDim.x) {
    if (t < a.K) {
      Stream r(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_w), static_cast<std::uint64_t>(t)));
      a.w[t] = 0.0 + sqrt(a.w_var) * r.next_gaussian();
    } else if (t == a.K) {
      Stream r(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_b), 0));
      a.w[t] = 0.0 + sqrt(a.b_var) * r.next_gaussian();
    } else {
      if (a.notau) {
        a.w[t] = a.logistic ? 0.0 : 1.0;  // polyreg: the fixed unit variance of y
      } else {
        Stream r(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_tau), 0));
        // InverseGamma: scale / gamma (dist.cpp:175-177); Gamma: scale * gamma (:157-159)
        a.w[t] = a.prec ? a.tau_b * draw_gamma(r, a.tau_a) : a.tau_b / draw_gamma(r, a.tau_a);
      }
    }
  }
}

__global__ void sum_to_kernel(const double* part, int n, double* out) {
  __shared__ double scratch[32];
  const double s = sum_parts(part, n, scratch);
  if (threadIdx.x == 0) *out = s;
}

// ---------------------------------------------------------------------------------
// MWG plan of regression.bn / polyreg.bn (RunConfig::method = mwg): w[t] and b are
// single-site random-walk blocks (run_mwg_block, sampler.cpp:342-388), in declaration
// order, each element against its own conditional numerator 0 + log p(elem) +
// sum_i log p(y_i | ...); regression.bn's tau is conjugate (InverseGammaVariance,
// sampler.cpp:122-130, 206-208).  Element e's proposal cur + mh_scale * N(0,1) and its
// accept uniform come from ONE stream keyed(seed,1,var,t,iter) (gaussian, then unit).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void mwg_element(const MhArgs& a, int e, int& var, std::uint64_t& t, double& pvar) {
  if (e < a.K) {
    var = a.var_w;
    t = static_cast<std::uint64_t>(e);
    pvar = a.w_var;
  } else {
    var = a.var_b;
    t = 0;
    pvar = a.b_var;
  }
}

__device__ __forceinline__ double mwg_proposal(const MhArgs& a, int e, std::int64_t iter, Stream& r) {
  int var;
  std::uint64_t t;
  double pvar;
  mwg_element(a, e, var, t, pvar);
  r = Stream(keyed(a.seed, kProposal, static_cast<std::uint64_t>(var), t, static_cast<std::uint64_t>(iter)));
  return a.w[e] + a.mh_scale * r.next_gaussian();
}

// Per block: sum_i ll(y_i | mean_i) at the current state (part[2b]) and with element e
// moved to its proposal (part[2b+1]); RSS: sum_i (y_i - mean_i)^2 instead (tau block).
template <bool RSS>
__global__ void __launch_bounds__(kThreads) mwg_lik_kernel(MhArgs a, const std::int64_t* iter_p, int e, double* part) {
  __shared__ double scratch[32];
  __shared__ double dlt;
  if (threadIdx.x == 0) {
    Stream r(0);
    dlt = RSS ? 0.0 : mwg_proposal(a, e, *iter_p, r) - a.w[e];
  }
  __syncthreads();
  const double b = a.w[a.K], tau = tau_variance(a, a.w[a.K + 1]), d = dlt;
  const int lane = threadIdx.x & 31;
  double acc0 = 0.0, acc1 = 0.0;
  const std::int64_t warp = (blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const std::int64_t nwarps = (static_cast<std::int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (std::int64_t i = warp; i < a.N; i += nwarps) {
    const double* xi = a.x + i * a.K;
    double sdot = 0.0;
    for (int j = lane; j < a.K; j += 32) sdot += a.w[j] * __ldg(xi + j);
    sdot = warp_sum(sdot);
    if (lane == 0) {
      const double m0 = sdot + b, yi = __ldg(a.y + i);
      if (RSS) {
        acc0 += (yi - m0) * (yi - m0);
      } else {
        const double m1 = e < a.K ? (sdot + d * __ldg(xi + e)) + b : sdot + (b + d);
        acc0 += row_loglik(a, m0, yi, tau);
        acc1 += row_loglik(a, m1, yi, tau);
      }
    }
  }
  acc0 = block_sum(acc0, scratch);
  acc1 = block_sum(acc1, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = acc0;
    part[2 * blockIdx.x + 1] = acc1;
  }
}

__global__ void mwg_accept_kernel(MhArgs a, const std::int64_t* iter_p, int e, const double* part) {
  __shared__ double scratch[32];
  double s0 = 0.0, s1 = 0.0;
  for (int b = threadIdx.x; b < kBlocks; b += blockDim.x) {
    s0 += part[2 * b];
    s1 += part[2 * b + 1];
  }
  s0 = block_sum(s0, scratch);
  s1 = block_sum(s1, scratch);
  if (threadIdx.x == 0) {
    int var;
    std::uint64_t t;
    double pvar;
    mwg_element(a, e, var, t, pvar);
    Stream r(0);
    const double cur = a.w[e];
    const double prop = mwg_proposal(a, e, *iter_p, r);
    const double before = (0.0 + log_pdf_gaussian(cur, 0.0, pvar)) + s0;
    const double after = (0.0 + log_pdf_gaussian(prop, 0.0, pvar)) + s1;
    if (isfinite(after) && log(r.next_unit()) < after - before) a.w[e] = prop;
  }
}

// tau ~ InverseGamma(tau_a + n/2, tau_b + rss/2) (InverseGammaVariance), or for a precision
// tau ~ Gamma(tau_a + n/2, scale 1 / (1/tau_b + rss/2)) (GammaPrecision, sampler.cpp:205-207);
// stream keyed(seed,4,var_tau,iter).derive(0)
__global__ void mwg_tau_kernel(MhArgs a, const std::int64_t* iter_p, const double* part) {
  __shared__ double scratch[32];
  double rss = 0.0;
  for (int b = threadIdx.x; b < kBlocks; b += blockDim.x) rss += part[2 * b];
  rss = block_sum(rss, scratch);
  if (threadIdx.x == 0) {
    const std::uint64_t key = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_tau),
                                    static_cast<std::uint64_t>(*iter_p));
    Stream r(derive(key, 0));
    const double n = static_cast<double>(a.N);
    a.w[a.K + 1] = a.prec ? (1.0 / (1.0 / a.tau_b + 0.5 * rss)) * draw_gamma(r, a.tau_a + 0.5 * n)
                          : (a.tau_b + 0.5 * rss) / draw_gamma(r, a.tau_a + 0.5 * n);
  }
}

// Gibbs plan (Method::Gibbs, plan.cpp:139-164): a non-conjugate real variable is ONE
// random-walk MH block (run_mh_block, sampler.cpp:284-340) over its elements
// [e0, e1) of the parameter vector: proposals keyed(seed,1,var,t,iter), blanket = the
// variable's prior factor + the y factor, accept keyed(seed,2,var,iter).
__global__ void blk_propose_kernel(MhArgs a, const std::int64_t* iter_p, int e0, int e1, int var) {
  const std::int64_t iter = *iter_p;
  for (int e = threadIdx.x; e < a.K + 2; e += blockDim.x) {
    double v = a.w[e];
    if (e >= e0 && e < e1) {
      Stream r(keyed(a.seed, kProposal, static_cast<std::uint64_t>(var), static_cast<std::uint64_t>(e - e0),
                     static_cast<std::uint64_t>(iter)));
      v += a.mh_scale * r.next_gaussian();
    }
    a.wp[e] = v;
  }
}

// before = prior(cur) + lik(cur), after = prior(prop) + lik(prop); the prior factor's
// elements are summed in order (eval_density of the var's factor)
__global__ void blk_accept_kernel(MhArgs a, const std::int64_t* iter_p, int e0, int e1, int var, double pvar,
                                  const double* part_cur, const double* part_prop) {
  __shared__ double scratch[32];
  __shared__ int take_s;
  const double l0 = sum_parts(part_cur, kBlocks, scratch);
  const double l1 = sum_parts(part_prop, kBlocks, scratch);
  if (threadIdx.x == 0) {
    double p0 = 0.0, p1 = 0.0;
    for (int e = e0; e < e1; ++e) {
      p0 += log_pdf_gaussian(a.w[e], 0.0, pvar);
      p1 += log_pdf_gaussian(a.wp[e], 0.0, pvar);
    }
    const double before = p0 + l0, after = p1 + l1;
    Stream acc(keyed(a.seed, kAccept, static_cast<std::uint64_t>(var), static_cast<std::uint64_t>(*iter_p)));
    const int take = isfinite(after) && log(acc.next_unit()) < after - before;
    take_s = take;
    a.state[5] = take;  // Engine::sweep reports the last MH block's decision
  }
  __syncthreads();
  if (take_s)
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) a.w[e] = a.wp[e];
}

// polyreg.bn's design matrix: X[i][j] = pow(x_i, j + 1), the terms of the mean
// sum(j in 1..M, w(j) * pow(x(i), j + 1)) (models/polyreg.bn).
__global__ void poly_features_kernel(const double* x, double* X, std::int64_t n, int K) {
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < n * K;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = e / K;
    const int j = static_cast<int>(e - i * K);
    X[e] = pow(x[i], static_cast<double>(j + 1));
  }
}

class Mh final : public Model {
 public:
  Mh(const bnmc_gpu_desc& d, const Comm& c, Outputs o) : comm_(c) {
    if (const char* e = std::getenv("BNMC_SPECULATE")) skip_unchanged_ = std::string(e) != "0";
    out = o;
    logistic_ = d.kind == BNMC_GPU_MH_LOGREG;
    poly_ = d.kind == BNMC_GPU_MH_POLYREG;
    gibbs_ = (d.flags & BNMC_GPU_GIBBS) != 0;
    mwg_ = (d.flags & BNMC_GPU_MWG) != 0;
    prec_ = (d.flags & BNMC_GPU_TAU_PRECISION) != 0;
    require(!prec_ || d.kind == BNMC_GPU_MH_LINREG, BNMC_GPU_ERR_ARG,
            "BNMC_GPU_TAU_PRECISION applies to the linear-regression kind only");
    require(!(gibbs_ || mwg_) || (!logistic_ && c.world == 1), BNMC_GPU_ERR_ARG,
            "the Gibbs / MWG plans serve regression.bn / polyreg.bn on one GPU");
    require(d.K >= 1 && d.N >= 0, BNMC_GPU_ERR_ARG, "MH needs K >= 1 features");
    K_ = static_cast<int>(d.K);
    N_ = d.N;
    r0_ = N_ * c.rank / c.world;
    r1_ = N_ * (c.rank + 1) / c.world;
    Nl_ = r1_ - r0_;
    const double* h = d.hyper;
    lo_ = h[0];
    hi_ = h[1];
    w_var_ = h[2] > 0 ? h[2] : (poly_ ? 1.0 : 10.0);
    b_var_ = h[3] > 0 ? h[3] : (poly_ ? 1.0 : 10.0);
    if (poly_ && !(hi_ > lo_)) {
      lo_ = 0.0;  // x ~ Uniform(0.0, 2.0) (models/polyreg.bn)
      hi_ = 2.0;
    }
    tau_a_ = h[4] > 0 ? h[4] : 3.0;
    tau_b_ = h[5] > 0 ? h[5] : 1.0;
    mh_scale_ = d.mh_scale;
    seed_ = d.seed;
    for (int i = 0; i < 5; ++i) var_[i] = d.var_ids[i];
    x_.alloc(std::max<std::int64_t>(Nl_ * K_, 1));
    if (poly_) xraw_.alloc(std::max<std::int64_t>(Nl_, 1));
    if (gibbs_ || mwg_) mwg_part_.alloc(2 * kBlocks);
    y_.alloc(std::max<std::int64_t>(Nl_, 1));
    w_.alloc(K_ + 2);
    wp_.alloc(K_ + 2);
    part_.alloc(kBlocks);
    state_.alloc(8);
    tot_.alloc(2);
    w_.zero(nullptr);
    wp_.zero(nullptr);
    part_.zero(nullptr);
    state_.zero(nullptr);
    tot_.zero(nullptr);
    BNMC_CUDA(cudaDeviceSynchronize());
  }

  void upload(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, true); }
  void upload_state(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, !data_); }

  void upload_impl(const bnmc_gpu_store& s, cudaStream_t st, bool with_data) {
    const int vw = var_[0], vb = var_[1];
    const bool notau = logistic_ || poly_;
    const int vtau = notau ? -1 : var_[2];
    const int vx = notau ? var_[2] : var_[3], vy = notau ? var_[3] : var_[4];
    require(s.len[vw] == K_ && s.len[vb] == 1 && s.len[vx] == N_ * (poly_ ? 1 : K_) && s.len[vy] == N_ &&
                (vtau < 0 || s.len[vtau] == 1),
            BNMC_GPU_ERR_RUNTIME, "MH store arrays have the wrong flat lengths");
    const std::vector<double> p = store_params(s);
    BNMC_CUDA(cudaMemcpyAsync(w_.p, p.data(), sizeof(double) * (K_ + 2), cudaMemcpyHostToDevice, st));
    h2d_bytes += static_cast<std::int64_t>(sizeof(double)) * (K_ + 2);
    last_valid_ = false;
    if (Nl_ > 0 && with_data) {
      if (poly_) {
        BNMC_CUDA(cudaMemcpyAsync(xraw_.p, s.real[vx] + r0_, sizeof(double) * Nl_, cudaMemcpyHostToDevice, st));
        poly_features_kernel<<<kBlocks, kThreads, 0, st>>>(xraw_.p, x_.p, Nl_, K_);
      } else {
        BNMC_CUDA(cudaMemcpyAsync(x_.p, s.real[vx] + r0_ * K_, sizeof(double) * Nl_ * K_, cudaMemcpyHostToDevice, st));
      }
      BNMC_CUDA(cudaMemcpyAsync(y_.p, s.real[vy] + r0_, sizeof(double) * Nl_, cudaMemcpyHostToDevice, st));
    }
    data_ = true;
    BNMC_CUDA(cudaStreamSynchronize(st));
    refresh(st);
  }

  // (w, b, tau) as the store holds them (tau: 0 / 1 placeholders without it)
  std::vector<double> store_params(const bnmc_gpu_store& s) const {
    const int vw = var_[0], vb = var_[1];
    const int vtau = (logistic_ || poly_) ? -1 : var_[2];
    std::vector<double> p(K_ + 2, 0.0);
    for (int j = 0; j < K_; ++j) p[j] = s.real[vw][j];
    p[K_] = s.real[vb][0];
    p[K_ + 1] = vtau >= 0 ? s.real[vtau][0] : (poly_ ? 1.0 : 0.0);
    return p;
  }

  // Engine::sweep on a bound store: the parameters are uploaded every call; when they
  // are bit for bit the state this context last wrote back and nothing ran since
  // (Model::quiet), the cached log-likelihood of the device state is current and the
  // refresh pass over the data (as long as the sweep's own likelihood pass) is skipped.
  void upload_sweep_inputs(const bnmc_gpu_store& s, cudaStream_t st) override {
    const std::vector<double> p = store_params(s);
    // (single rank: the refresh's all-reduce must not become a per-rank decision)
    if (!(quiet && skip_unchanged_ && last_valid_ && !comm_.active() &&
          std::memcmp(p.data(), last_.data(), sizeof(double) * p.size()) == 0)) {
      upload_state(s, st);
      return;
    }
    BNMC_CUDA(cudaMemcpyAsync(w_.p, p.data(), sizeof(double) * (K_ + 2), cudaMemcpyHostToDevice, st));
    BNMC_CUDA(cudaStreamSynchronize(st));  // p is a host temporary
    h2d_bytes += static_cast<std::int64_t>(sizeof(double)) * (K_ + 2);
  }

  void download(const bnmc_gpu_store& s, cudaStream_t st) override {
    std::vector<double> p(K_ + 2);
    BNMC_CUDA(cudaMemcpyAsync(p.data(), w_.p, sizeof(double) * (K_ + 2), cudaMemcpyDeviceToHost, st));
    BNMC_CUDA(cudaStreamSynchronize(st));
    d2h_bytes += static_cast<std::int64_t>(sizeof(double)) * (K_ + 2);
    const char* obs = s.observed;
    const int vw = var_[0], vb = var_[1];
    if (!(obs && obs[vw]))
      for (int j = 0; j < K_; ++j) s.real[vw][j] = p[j];
    if (!(obs && obs[vb])) s.real[vb][0] = p[K_];
    if (!logistic_ && !poly_ && !(obs && obs[var_[2]])) s.real[var_[2]][0] = p[K_ + 1];
    last_ = store_params(s);  // what the store holds now (observed entries: the caller's)
    last_valid_ = std::memcmp(last_.data(), p.data(), sizeof(double) * p.size()) == 0;
  }

  void on_state_restored(cudaStream_t st) override { refresh(st); }

  std::vector<StateBuf> state_buffers() override {
    return {{reinterpret_cast<void**>(&w_.p), sizeof(double) * static_cast<std::size_t>(K_ + 2)}};
  }

  void enqueue_sweep(cudaStream_t st) override {
    MhArgs a = args();
    mark(st, "begin");
    if (gibbs_ || mwg_) {
      if (mwg_) {
        // Method::MWG: single-site blocks w[0..K-1], b in declaration order
        for (int e = 0; e <= K_; ++e) {
          mwg_lik_kernel<false><<<kBlocks, kThreads, 0, st>>>(a, out.iter, e, mwg_part_.p);
          mwg_accept_kernel<<<1, 256, 0, st>>>(a, out.iter, e, mwg_part_.p);
        }
        mark(st, "mwg_w_b");
      } else {
        // Method::Gibbs: one random-walk MH block per variable, w then b
        const int ranges[2][3] = {{0, K_, var_[0]}, {K_, K_ + 1, var_[1]}};
        const double pv[2] = {w_var_, b_var_};
        for (int bi = 0; bi < 2; ++bi) {
          blk_propose_kernel<<<1, 128, 0, st>>>(a, out.iter, ranges[bi][0], ranges[bi][1], ranges[bi][2]);
          launch_lik(a, w_.p, st, mwg_part_.p);
          launch_lik(a, wp_.p, st, part_.p);
          blk_accept_kernel<<<1, 256, 0, st>>>(a, out.iter, ranges[bi][0], ranges[bi][1], ranges[bi][2], pv[bi],
                                               mwg_part_.p, part_.p);
        }
        mark(st, "mh_w_b");
      }
      if (!poly_) {
        mwg_lik_kernel<true><<<kBlocks, kThreads, 0, st>>>(a, out.iter, 0, mwg_part_.p);
        mwg_tau_kernel<<<1, 256, 0, st>>>(a, out.iter, mwg_part_.p);
        mark(st, "tau");
      }
      launch_lik(a, w_.p, st);
      accept_kernel<<<1, 256, 0, st>>>(a, out, 3, nullptr);
      mark(st, "log_joint");
      BNMC_CUDA(cudaGetLastError());
      return;
    }
    propose_kernel<<<1, 128, 0, st>>>(a, out.iter);
    mark(st, "propose");
    launch_lik(a, wp_.p, st);
    mark(st, "lik");
    const double* tot = nullptr;
    if (comm_.active()) {
      sum_to_kernel<<<1, 256, 0, st>>>(part_.p, kBlocks, tot_.p);
      comm_.all_reduce(tot_.p, 1, RedType::F64, RedOp::Sum, st);
      tot = tot_.p;
      mark(st, "allreduce_lik");
    }
    accept_kernel<<<1, 256, 0, st>>>(a, out, 1, tot);
    mark(st, "accept");
    BNMC_CUDA(cudaGetLastError());
  }

  void enqueue_log_joint(cudaStream_t st) override {
    MhArgs a = args();
    // The cached state already holds the current blanket; report it.
    accept_kernel_cached(a, st);
  }

  void prior_init(std::uint64_t seed, cudaStream_t st) override {
    prior_kernel<<<1, 128, 0, st>>>(args(), seed);
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
    refresh(st);
  }

 private:

  void launch_lik(const MhArgs& a, const double* p, cudaStream_t st, double* dst = nullptr) {
    const std::size_t sm = sizeof(double) * (K_ + 2);
    const int cpl = (K_ / 4 + kRowGroup - 1) / kRowGroup;
    double* o = dst ? dst : part_.p;
    if (K_ % 4 == 0 && cpl <= 1)
      lik_kernel<true, 1><<<kBlocks, kThreads, sm, st>>>(a, p, o);
    else if (K_ % 4 == 0 && cpl <= 2)
      lik_kernel<true, 2><<<kBlocks, kThreads, sm, st>>>(a, p, o);
    else if (K_ % 4 == 0 && cpl <= 4)
      lik_kernel<true, 4><<<kBlocks, kThreads, sm, st>>>(a, p, o);
    else if (K_ % 4 == 0 && cpl <= kMaxChunks)
      lik_kernel<true, 8><<<kBlocks, kThreads, sm, st>>>(a, p, o);
    else
      lik_kernel<false><<<kBlocks, kThreads, sizeof(double) * (K_ + 2), st>>>(a, p, o);
  }

  void accept_kernel_cached(const MhArgs& a, cudaStream_t st) {
    launch_lik(a, w_.p, st);
    const double* tot = nullptr;
    if (comm_.active()) {
      sum_to_kernel<<<1, 256, 0, st>>>(part_.p, kBlocks, tot_.p);
      comm_.all_reduce(tot_.p, 1, RedType::F64, RedOp::Sum, st);
      tot = tot_.p;
    }
    accept_kernel<<<1, 256, 0, st>>>(a, out, 0, tot);
    BNMC_CUDA(cudaGetLastError());
  }

  // Recompute the constant data factor and the cached blanket of the current state.
  void refresh(cudaStream_t st) {
    MhArgs a = args();
    fx_kernel<<<kBlocks, kThreads, 0, st>>>(a, part_.p);
    const double* tot = nullptr;
    if (comm_.active()) {
      sum_to_kernel<<<1, 256, 0, st>>>(part_.p, kBlocks, tot_.p + 1);
      comm_.all_reduce(tot_.p + 1, 1, RedType::F64, RedOp::Sum, st);
      tot = tot_.p + 1;
    }
    fx_finalize_kernel<<<1, 256, 0, st>>>(a, tot);
    accept_kernel_cached(a, st);
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  MhArgs args() const {
    MhArgs a{};
    a.N = Nl_;
    a.K = K_;
    a.x = x_.p;
    a.y = y_.p;
    a.w = w_.p;
    a.wp = wp_.p;
    a.part = part_.p;
    a.state = state_.p;
    a.lo = lo_;
    a.hi = hi_;
    a.w_var = w_var_;
    a.b_var = b_var_;
    a.tau_a = tau_a_;
    a.tau_b = tau_b_;
    a.mh_scale = mh_scale_;
    a.seed = seed_;
    a.var_w = var_[0];
    a.var_b = var_[1];
    a.var_tau = (logistic_ || poly_) ? -1 : var_[2];
    a.logistic = logistic_ ? 1 : 0;
    a.notau = (logistic_ || poly_) ? 1 : 0;
    a.prec = prec_ ? 1 : 0;
    a.xr = poly_ ? xraw_.p : x_.p;
    a.nfx = poly_ ? Nl_ : Nl_ * K_;
    return a;
  }

  Comm comm_;
  bool data_ = false;
  bool logistic_ = false, poly_ = false, gibbs_ = false, mwg_ = false, prec_ = false;
  int K_ = 0;
  std::int64_t N_ = 0, r0_ = 0, r1_ = 0, Nl_ = 0;
  double lo_, hi_, w_var_, b_var_, tau_a_, tau_b_, mh_scale_;
  std::uint64_t seed_ = 0;
  int var_[5] = {0, 1, 2, 3, 4};
  std::vector<double> last_;  // the store's (w, b, tau) after the last write-back
  bool last_valid_ = false;   // ... and they equal the device state
  bool skip_unchanged_ = true;  // BNMC_SPECULATE=0: always refresh on a bound-store upload
  DevBuf<double> x_, y_, w_, wp_, part_, state_, tot_, xraw_, mwg_part_;
};

}  // namespace

std::unique_ptr<Model> make_mh(const bnmc_gpu_desc& d, const Comm& c, Outputs o) {
  return std::make_unique<Mh>(d, c, o);
}

}  // namespace bnmc_gpu
