// csrc/gmm.cu -- univariate Gaussian-mixture Gibbs sweep (proj/models/gmm.bn).
//
// Plan order pi, mu, sigma2, z (tests/golden/describe_gmm.txt).  Per sweep:
//   stats_kernel(MU)   counts + sum 1/sigma2[z] + sum x/sigma2[z] with the current
//                      z and sigma2 (sampler.cpp:114-121), per-block partials
//   draw_pi_mu_kernel  pi ~ Dir(alpha + c) (rows = 1, batch.cpp:51-63);
//                      mu_k ~ N(v*(mu0/v0 + W), v*), v* = 1/(1/v0 + P)
//                      (sampler.cpp:199-204), stream keyed(seed,4,var,iter).derive(k)
//   stats_kernel(RSS)  n, sum (x - mu[z])^2 with the NEW mu (sampler.cpp:122-130)
//   draw_s2_kernel     sigma2_k = (b0 + rss/2) / Gamma(a0 + n/2) (dist.cpp:175-177)
//   z_kernel           log pi_v + log N(x | mu_v, sigma2_v), draw_from_log_weights
//                      with keyed(seed,3,var_z,i,iter) (sampler.cpp:222-265);
//                      accumulates the log-joint pieces of z and x
//   finalize_kernel    log-joint in the reference's factor order.
// K <= 8 (default): three kernels -- draw_params_kernel (pi, mu, sigma2 from the
// sufficient statistics the previous z kernel left, centred on the mu it used), the z
// kernel (draws z, accumulates the log-joint pieces and the statistics of the new z),
// finalize -- instead of two extra passes over the data per sweep.
// Every reduction runs over a fixed grid with a fixed tree: results are
// reproducible run to run.  Replicas only across GPUs.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "dist.cuh"

namespace bnmc_gpu {
namespace {

constexpr int kThreads = 256;
constexpr int kBlocks = 148 * 2;     // grid of the six-kernel path's data passes
constexpr int kMaxBlocks = 148 * 4;  // partial slots (the fused z kernel sizes its grid to N)
constexpr int kMaxK = 64;

struct GmmArgs {
  std::int64_t N;
  int K;
  const double* x;
  int* z;
  double* pi;
  double* mu;
  double* s2;
  int nb;        // blocks that wrote part / lpart (the grid of the kernels producing them)
  double* part;  // [nb][K][3]
  double* mu_at_stats;  // [K] (fused path) the mu the z kernel's shifted sums are centred on
  double* lpart; // [nb][2]
  double alpha, mu0, v0, a0, b0;
  std::uint64_t seed;
  int var_pi, var_mu, var_s2, var_z;
};

enum { kStatsMu = 0, kStatsRss = 1 };

template <int WHICH>
__global__ void __launch_bounds__(kThreads) stats_kernel(GmmArgs a, int* err) {
  __shared__ double scratch[32];
  for (int k = 0; k < a.K; ++k) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    const double m = a.mu[k], v = a.s2[k];
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < a.N;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
      const int zi = a.z[i];
      if (k == 0 && (zi < 0 || zi >= a.K)) atomicOr(err, kErrBin);
      if (zi != k) continue;
      const double xi = a.x[i];
      if (WHICH == kStatsMu) {
        s0 += 1.0;
        s1 += 1.0 / v;
        s2 += xi / v;
      } else {
        s0 += 1.0;
        s1 += (xi - m) * (xi - m);
      }
    }
    s0 = block_sum(s0, scratch);
    s1 = block_sum(s1, scratch);
    s2 = block_sum(s2, scratch);
    if (threadIdx.x == 0) {
      double* p = a.part + (static_cast<std::size_t>(blockIdx.x) * a.K + k) * 3;
      p[0] = s0;
      p[1] = s1;
      p[2] = s2;
    }
  }
}

// All K x J sums over the kBlocks partials at once (J <= 3; K * J <= blockDim): thread t
// sums (k, j) = t mod (K J) over every groups-th partial, then threads t < K J add the
// groups' sums in group order -- fixed order, one barrier pair instead of one block
// reduction per (k, j) (the per-(k, j) reductions were ~1 us each, serialised).
__device__ void reduce_parts(const GmmArgs& a, int J, double* out, double* tmp) {
  const int n = a.K * J, t = threadIdx.x;
  const int groups = static_cast<int>(blockDim.x) / n, grp = t / n, q = t - grp * n;
  double s = 0.0;
  if (grp < groups) {
    const int k = q / J, j = q - (q / J) * J;
    int b = grp;
    for (; b + 7 * groups < a.nb; b += 8 * groups) {  // 8 loads in flight
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a.part[(static_cast<std::size_t>(b + u * groups) * a.K + k) * 3 + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; b < a.nb; b += groups) s += a.part[(static_cast<std::size_t>(b) * a.K + k) * 3 + j];
  }
  tmp[t] = s;
  __syncthreads();
  if (t < n) {
    double r = 0.0;
    for (int g = 0; g < groups; ++g) r += tmp[g * n + t];
    out[t] = r;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) draw_pi_mu_kernel(GmmArgs a, const std::int64_t* iter_p) {
  __shared__ double sums[3 * kMaxK], tmp[kThreads];
  const std::int64_t iter = *iter_p;
  reduce_parts(a, 3, sums, tmp);
  const double* cnt = sums;  // [k * 3 + 0]: count, 1: precision sum, 2: weighted x sum
  // Independent per-component streams: thread k draws the pi cell's gamma and mu_k (the
  // draws were serial on one thread: ~2 gamma chains of latency per component).
  __shared__ double g[kMaxK];
  const std::uint64_t kp = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_pi),
                                 static_cast<std::uint64_t>(iter));
  const std::uint64_t km = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_mu),
                                 static_cast<std::uint64_t>(iter));
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    // pi block: Dirichlet over a single row, cells derive(0, c)
    Stream r(derive(kp, 0, static_cast<std::uint64_t>(k)));
    g[k] = draw_gamma(r, a.alpha + cnt[3 * k]);
    // mu block
    Stream q(derive(km, static_cast<std::uint64_t>(k)));
    const double prec = 1.0 / a.v0 + cnt[3 * k + 1];
    const double wsum = a.mu0 / a.v0 + cnt[3 * k + 2];
    const double post_var = 1.0 / prec;
    a.mu[k] = post_var * wsum + sqrt(post_var) * q.next_gaussian();
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // left-to-right row sum (batch.cpp:55-58)
    double sum = 0.0;
    for (int k = 0; k < a.K; ++k) sum += g[k];
    for (int k = 0; k < a.K; ++k) a.pi[k] = g[k] / sum;
  }
}

__global__ void __launch_bounds__(kThreads) draw_s2_kernel(GmmArgs a, const std::int64_t* iter_p) {
  __shared__ double sums[2 * kMaxK], tmp[kThreads];
  const std::int64_t iter = *iter_p;
  reduce_parts(a, 2, sums, tmp);
  const std::uint64_t ks = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_s2),
                                 static_cast<std::uint64_t>(iter));
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    Stream r(derive(ks, static_cast<std::uint64_t>(k)));
    const double scale = a.b0 + 0.5 * sums[2 * k + 1];
    a.s2[k] = scale / draw_gamma(r, a.a0 + 0.5 * sums[2 * k]);
  }
}

// FUSE (K <= kFuseK): the z kernel also leaves, per block and component, the sufficient
// statistics of the NEW z centred on the current mu -- n, S1 = sum (x - c), S2 = sum
// (x - c)^2, c = mu[k] -- so the next sweep's pi / mu / sigma2 draws need no data pass:
// P = n / sigma2, W = (S1 + n c) / sigma2 and rss = S2 - 2 d S1 + n d^2 with
// d = mu_new - c (the shift keeps the cancellation to the size of d, a posterior sd).
constexpr int kFuseK = 8;

template <bool SAMPLE, bool FUSE = false, int FK = kFuseK>
__global__ void __launch_bounds__(kThreads) z_kernel(GmmArgs a, const std::int64_t* iter_p, int* err) {
  __shared__ double scratch[32];
  __shared__ double lpi[kMaxK], mu[kMaxK], var[kMaxK], lvar[kMaxK];
  const std::int64_t iter = *iter_p;
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    lpi[k] = a.pi[k] > 0.0 ? log(a.pi[k]) : -INFINITY;
    mu[k] = a.mu[k];
    var[k] = a.s2[k];
    lvar[k] = log(a.s2[k]);
  }
  __syncthreads();
  const std::uint64_t zp = fold(fold(fold(1, a.seed), kDiscrete), static_cast<std::uint64_t>(a.var_z));
  double lz = 0.0, lx = 0.0;
  double fn[FUSE ? FK : 1], f1[FUSE ? FK : 1], f2[FUSE ? FK : 1];
#pragma unroll
  for (int v = 0; v < (FUSE ? FK : 1); ++v) fn[v] = f1[v] = f2[v] = 0.0;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < a.N;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const double xi = a.x[i];
    // logw[v] = (0 + log pi_v) + log N(x | mu_v, sigma2_v); log_pdf_gaussian (dist.cpp:61-68)
    auto logw = [&](int v) {
      const double d = xi - mu[v];
      const double g = var[v] > 0.0 ? -0.5 * (d * d / var[v] + lvar[v] + kLog2Pi) : -INFINITY;
      return lpi[v] + g;
    };
    int k;
    if (SAMPLE) {
      double mx = -INFINITY;
      for (int v = 0; v < a.K; ++v) mx = fmax(mx, logw(v));
      if (!isfinite(mx)) {
        atomicOr(err, kErrDomain);
        continue;
      }
      double total = 0.0;
      for (int v = 0; v < a.K; ++v) total += exp(logw(v) - mx);
      Stream r(fold(fold(zp, static_cast<std::uint64_t>(i)), static_cast<std::uint64_t>(iter)));
      const double u = r.next_unit() * total;
      double acc = 0.0;
      k = a.K - 1;
      for (int v = 0; v < a.K; ++v) {
        acc += exp(logw(v) - mx);
        if (u < acc) {
          k = v;
          break;
        }
      }
      a.z[i] = k;
    } else {
      k = a.z[i];
      if (k < 0 || k >= a.K) {
        lz += -INFINITY;
        lx += -INFINITY;
        continue;
      }
    }
    lz += lpi[k];
    const double d = xi - mu[k];
    lx += var[k] > 0.0 ? -0.5 * (d * d / var[k] + lvar[k] + kLog2Pi) : -INFINITY;
    if constexpr (FUSE) {
#pragma unroll
      for (int v = 0; v < FK; ++v)
        if (v == k) {
          fn[v] += 1.0;
          f1[v] += d;
          f2[v] += d * d;
        }
    }
  }
  lz = block_sum(lz, scratch);
  lx = block_sum(lx, scratch);
  if (threadIdx.x == 0) {
    a.lpart[blockIdx.x * 2 + 0] = lz;
    a.lpart[blockIdx.x * 2 + 1] = lx;
  }
  if constexpr (FUSE) {
    __shared__ double sc3[3 * 32];
#pragma unroll
    for (int v = 0; v < FK; ++v) {
      if (v >= a.K) break;
      double t[3] = {fn[v], f1[v], f2[v]};
      block_sum_n<3>(t, sc3);
      if (threadIdx.x == 0) {
        double* p = a.part + (static_cast<std::size_t>(blockIdx.x) * a.K + v) * 3;
        p[0] = t[0];
        p[1] = t[1];
        p[2] = t[2];
      }
    }
    if (blockIdx.x == 0)
      for (int v = threadIdx.x; v < a.K; v += blockDim.x) a.mu_at_stats[v] = mu[v];
  }
}

// Fused path: pi, mu and sigma2 in one block from the z kernel's shifted sums.
constexpr int kDrawThreads = 1024;  // draw_params_kernel: 1024 threads reduce the partials in ~one round

__global__ void __launch_bounds__(kDrawThreads) draw_params_kernel(GmmArgs a, const std::int64_t* iter_p) {
  __shared__ double sums[3 * kMaxK], tmp[kDrawThreads], g[kMaxK];
  const std::int64_t iter = *iter_p;
  reduce_parts(a, 3, sums, tmp);
  const std::uint64_t kp = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_pi),
                                 static_cast<std::uint64_t>(iter));
  const std::uint64_t km = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_mu),
                                 static_cast<std::uint64_t>(iter));
  const std::uint64_t ks = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_s2),
                                 static_cast<std::uint64_t>(iter));
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    const double n = sums[3 * k], S1 = sums[3 * k + 1], S2 = sums[3 * k + 2];
    const double c = a.mu_at_stats[k], v = a.s2[k];
    // pi block: Dirichlet over a single row, cells derive(0, k)
    Stream r(derive(kp, 0, static_cast<std::uint64_t>(k)));
    g[k] = draw_gamma(r, a.alpha + n);
    // mu block (sampler.cpp:199-204): P = sum 1/sigma2, W = sum x/sigma2 over the cluster
    Stream q(derive(km, static_cast<std::uint64_t>(k)));
    const double prec = 1.0 / a.v0 + n * (1.0 / v);
    const double wsum = a.mu0 / a.v0 + (S1 + n * c) / v;
    const double post_var = 1.0 / prec;
    const double mu_new = post_var * wsum + sqrt(post_var) * q.next_gaussian();
    a.mu[k] = mu_new;
    // sigma2 block with the new mu: rss = sum (x - mu_new)^2 from the shifted sums
    const double dd = mu_new - c;
    const double rss = fmax(0.0, S2 - 2.0 * dd * S1 + n * dd * dd);
    Stream t(derive(ks, static_cast<std::uint64_t>(k)));
    a.s2[k] = (a.b0 + 0.5 * rss) / draw_gamma(t, a.a0 + 0.5 * n);
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // left-to-right row sum (batch.cpp:55-58)
    double sum = 0.0;
    for (int k = 0; k < a.K; ++k) sum += g[k];
    for (int k = 0; k < a.K; ++k) a.pi[k] = g[k] / sum;
  }
}

__global__ void finalize_kernel(GmmArgs a, Outputs o, int advance) {
  __shared__ double scratch[32];
  double lz = 0.0, lx = 0.0;
  for (int b = threadIdx.x; b < a.nb; b += blockDim.x) {
    lz += a.lpart[b * 2 + 0];
    lx += a.lpart[b * 2 + 1];
  }
  lz = block_sum(lz, scratch);
  lx = block_sum(lx, scratch);
  // the per-component prior terms (transcendentals) in parallel, one thread per k; the
  // sums below run in k order as the reference's sequential loops
  __shared__ double tpi[kMaxK], tmu[kMaxK], ts2[kMaxK], lga[2];
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    tpi[k] = (a.alpha - 1.0) * log(a.pi[k]);
    tmu[k] = log_pdf_gaussian(a.mu[k], a.mu0, a.v0);
    ts2[k] = log_pdf_inverse_gamma(a.s2[k], a.a0, a.b0);
  }
  if (threadIdx.x == 32) lga[0] = lgamma(a.alpha);
  if (threadIdx.x == 64) {
    double asum = 0.0;
    for (int k = 0; k < a.K; ++k) asum += a.alpha;
    lga[1] = lgamma(asum);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // p(pi): Dirichlet(alpha,...,alpha) log-pdf (dist.cpp:115-130)
    double sum = 0.0, lp = 0.0, norm = 0.0;
    bool bad = false;
    for (int k = 0; k < a.K; ++k) {
      const double x = a.pi[k];
      bad |= !(x > 0.0);
      sum += x;
      lp += tpi[k];
      norm += lga[0];
    }
    const double fpi = (bad || fabs(sum - 1.0) > 1e-9) ? -INFINITY : lp - norm + lga[1];
    double fmu = 0.0, fs2 = 0.0;
    for (int k = 0; k < a.K; ++k) fmu += tmu[k];
    for (int k = 0; k < a.K; ++k) fs2 += ts2[k];
    const double lj = (((fpi + fmu) + fs2) + lz) + lx;
    const std::int64_t it = *o.iter;
    o.lj[it & (kRing - 1)] = lj;
    o.acc[it & (kRing - 1)] = 0;
    if (advance) *o.iter = it + 1;
  }
}

__global__ void prior_kernel(GmmArgs a, std::uint64_t seed) {
  // prior_init (sampler.cpp:542-555): one stream keyed(seed,5,var,elem) per element.
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Stream s(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_pi), 0));
    double sum = 0.0;
    for (int k = 0; k < a.K; ++k) {
      a.pi[k] = draw_gamma(s, a.alpha);
      sum += a.pi[k];
    }
    for (int k = 0; k < a.K; ++k) a.pi[k] /= sum;
    for (int k = 0; k < a.K; ++k) {
      Stream m(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_mu), static_cast<std::uint64_t>(k)));
      a.mu[k] = a.mu0 + sqrt(a.v0) * m.next_gaussian();
      Stream v(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_s2), static_cast<std::uint64_t>(k)));
      a.s2[k] = a.b0 / draw_gamma(v, a.a0);
    }
  }
}

__global__ void prior_z_kernel(GmmArgs a, std::uint64_t seed) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < a.N;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    Stream s(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_z), static_cast<std::uint64_t>(i)));
    const double u = s.next_unit();
    double acc = 0.0;
    int pick = a.K - 1;
    for (int k = 0; k < a.K; ++k) {
      acc += a.pi[k];
      if (u < acc) {
        pick = k;
        break;
      }
    }
    a.z[i] = pick;
  }
}

__global__ void z_from_i64(const std::int64_t* in, int* out, std::int64_t n, int K, int* err) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t v = in[i];
    if (v < 0 || v >= K) atomicOr(err, kErrBin);
    out[i] = static_cast<int>(v);
  }
}

__global__ void z_to_i64(const int* in, std::int64_t* out, std::int64_t n) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

class Gmm final : public Model {
 public:
  Gmm(const bnmc_gpu_desc& d, const Comm& c, Outputs o) {
    out = o;
    require(d.K >= 1 && d.K <= kMaxK, BNMC_GPU_ERR_ARG, "GMM supports 1 <= K <= 64");
    require(d.N >= 0, BNMC_GPU_ERR_ARG, "GMM needs N >= 0");
    require(c.world == 1, BNMC_GPU_ERR_ARG, "GMM runs as replicas only (world_size must be 1)");
    K_ = static_cast<int>(d.K);
    N_ = d.N;
    const double* h = d.hyper;
    alpha_ = h[0] > 0 ? h[0] : 0.1;
    mu0_ = h[1];
    v0_ = h[2] > 0 ? h[2] : 10.0;
    a0_ = h[3] > 0 ? h[3] : 1.0;
    b0_ = h[4] > 0 ? h[4] : 1.0;
    seed_ = d.seed;
    for (int i = 0; i < 5; ++i) var_[i] = d.var_ids[i];
    x_.alloc(std::max<std::int64_t>(N_, 1));
    z_.alloc(std::max<std::int64_t>(N_, 1));
    pi_.alloc(K_);
    mu_.alloc(K_);
    s2_.alloc(K_);
    part_.alloc(static_cast<std::size_t>(kMaxBlocks) * K_ * 3);
    mu_at_stats_.alloc(K_);
    fuse_ = K_ <= kFuseK;
    // fused path: one point per thread where the grid fits one wave (N = 1e5: 391 blocks)
    nbz_ = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(kMaxBlocks, (N_ + kThreads - 1) / kThreads)));
    if (const char* e = std::getenv("BNMC_GMM_FUSED")) fuse_ = fuse_ && std::string(e) != "0";
    lpart_.alloc(kMaxBlocks * 2);
    part_.zero(nullptr);
    lpart_.zero(nullptr);
    z_.zero(nullptr);
    BNMC_CUDA(cudaDeviceSynchronize());
  }

  void upload(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, true); }
  void upload_state(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, !data_); }

  void upload_impl(const bnmc_gpu_store& s, cudaStream_t st, bool with_data) {
    require(s.n_vars > 4, BNMC_GPU_ERR_RUNTIME, "store has the wrong number of variables");
    const int vpi = var_[0], vmu = var_[1], vs2 = var_[2], vz = var_[3], vx = var_[4];
    require(s.len[vpi] == K_ && s.len[vmu] == K_ && s.len[vs2] == K_ && s.len[vz] == N_ &&
                s.len[vx] == N_,
            BNMC_GPU_ERR_RUNTIME, "GMM store arrays have the wrong flat lengths");
    if (with_data) BNMC_CUDA(cudaMemcpyAsync(x_.p, s.real[vx], sizeof(double) * N_, cudaMemcpyHostToDevice, st));
    data_ = true;
    BNMC_CUDA(cudaMemcpyAsync(pi_.p, s.real[vpi], sizeof(double) * K_, cudaMemcpyHostToDevice, st));
    BNMC_CUDA(cudaMemcpyAsync(mu_.p, s.real[vmu], sizeof(double) * K_, cudaMemcpyHostToDevice, st));
    BNMC_CUDA(cudaMemcpyAsync(s2_.p, s.real[vs2], sizeof(double) * K_, cudaMemcpyHostToDevice, st));
    if (N_ > 0) {
      if (stage64_.n < static_cast<std::size_t>(N_)) stage64_.alloc(N_);  // kept: no per-call cudaMalloc/cudaFree
      BNMC_CUDA(cudaMemcpyAsync(stage64_.p, s.ival[vz], sizeof(std::int64_t) * N_, cudaMemcpyHostToDevice, st));
      z_from_i64<<<kBlocks, kThreads, 0, st>>>(stage64_.p, z_.p, N_, K_, out.err);
    }
    h2d_bytes += static_cast<std::int64_t>(sizeof(double)) * 3 * K_ + static_cast<std::int64_t>(sizeof(std::int64_t)) * N_;
    refresh_stats(st);
    // stream-ordered: the sweep (or the caller's next synchronous call) sees the upload
  }

  void download(const bnmc_gpu_store& s, cudaStream_t st) override {
    const int vpi = var_[0], vmu = var_[1], vs2 = var_[2], vz = var_[3];
    const char* obs = s.observed;
    auto want = [&](int v) { return !(obs && obs[v]); };
    if (want(vpi)) BNMC_CUDA(cudaMemcpyAsync(s.real[vpi], pi_.p, sizeof(double) * K_, cudaMemcpyDeviceToHost, st));
    if (want(vmu)) BNMC_CUDA(cudaMemcpyAsync(s.real[vmu], mu_.p, sizeof(double) * K_, cudaMemcpyDeviceToHost, st));
    if (want(vs2)) BNMC_CUDA(cudaMemcpyAsync(s.real[vs2], s2_.p, sizeof(double) * K_, cudaMemcpyDeviceToHost, st));
    if (want(vz) && N_ > 0) {
      if (stage64_.n < static_cast<std::size_t>(N_)) stage64_.alloc(N_);
      z_to_i64<<<kBlocks, kThreads, 0, st>>>(z_.p, stage64_.p, N_);
      BNMC_CUDA(cudaMemcpyAsync(s.ival[vz], stage64_.p, sizeof(std::int64_t) * N_, cudaMemcpyDeviceToHost, st));
      d2h_bytes += static_cast<std::int64_t>(sizeof(std::int64_t)) * N_;
    }
    for (int v : {vpi, vmu, vs2})
      if (want(v)) d2h_bytes += static_cast<std::int64_t>(sizeof(double)) * K_;
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  std::vector<StateBuf> state_buffers() override {
    return {{reinterpret_cast<void**>(&z_.p), sizeof(int) * static_cast<std::size_t>(N_)},
            {reinterpret_cast<void**>(&pi_.p), sizeof(double) * static_cast<std::size_t>(K_)},
            {reinterpret_cast<void**>(&mu_.p), sizeof(double) * static_cast<std::size_t>(K_)},
            {reinterpret_cast<void**>(&s2_.p), sizeof(double) * static_cast<std::size_t>(K_)}};
  }

  void enqueue_sweep(cudaStream_t st) override {
    GmmArgs a = args();
    mark(st, "begin");
    if (fuse_) {
      // the statistics of the current z were left by the last z kernel (or refresh_stats)
      draw_params_kernel<<<1, kDrawThreads, 0, st>>>(a, out.iter);
      mark(st, "draw_pi_mu_sigma2");
      launch_fused_z<true>(a, st);
      mark(st, "z_stats");
      finalize_kernel<<<1, kThreads, 0, st>>>(a, out, 1);
      mark(st, "finalize");
      BNMC_CUDA(cudaGetLastError());
      return;
    }
    stats_kernel<kStatsMu><<<kBlocks, kThreads, 0, st>>>(a, out.err);
    mark(st, "stats_mu");
    draw_pi_mu_kernel<<<1, kThreads, 0, st>>>(a, out.iter);
    mark(st, "draw_pi_mu");
    stats_kernel<kStatsRss><<<kBlocks, kThreads, 0, st>>>(a, out.err);
    mark(st, "stats_rss");
    draw_s2_kernel<<<1, kThreads, 0, st>>>(a, out.iter);
    mark(st, "draw_sigma2");
    z_kernel<true><<<kBlocks, kThreads, 0, st>>>(a, out.iter, out.err);
    mark(st, "z");
    finalize_kernel<<<1, kThreads, 0, st>>>(a, out, 1);
    mark(st, "finalize");
    BNMC_CUDA(cudaGetLastError());
  }

  template <bool SAMPLE>
  void launch_fused_z(const GmmArgs& a, cudaStream_t st) {
    if (K_ <= 4) z_kernel<SAMPLE, true, 4><<<static_cast<unsigned>(nbz_), kThreads, 0, st>>>(a, out.iter, out.err);
    else z_kernel<SAMPLE, true, kFuseK><<<static_cast<unsigned>(nbz_), kThreads, 0, st>>>(a, out.iter, out.err);
  }

  // Fused path: the statistics of the current state (after any state change).
  void refresh_stats(cudaStream_t st) {
    if (!fuse_ || N_ == 0) return;
    GmmArgs a = args();
    launch_fused_z<false>(a, st);
    BNMC_CUDA(cudaGetLastError());
  }

  void on_state_restored(cudaStream_t st) override {
    refresh_stats(st);
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  void enqueue_log_joint(cudaStream_t st) override {
    GmmArgs a = args();
    z_kernel<false, false><<<static_cast<unsigned>(a.nb), kThreads, 0, st>>>(a, out.iter, out.err);
    finalize_kernel<<<1, kThreads, 0, st>>>(a, out, 0);
    BNMC_CUDA(cudaGetLastError());
  }

  void prior_init(std::uint64_t seed, cudaStream_t st) override {
    GmmArgs a = args();
    prior_kernel<<<1, 32, 0, st>>>(a, seed);
    prior_z_kernel<<<kBlocks, kThreads, 0, st>>>(a, seed);
    refresh_stats(st);
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

 private:
  GmmArgs args() const {
    GmmArgs a{};
    a.N = N_;
    a.K = K_;
    a.x = x_.p;
    a.z = z_.p;
    a.pi = pi_.p;
    a.mu = mu_.p;
    a.s2 = s2_.p;
    a.nb = fuse_ ? nbz_ : kBlocks;
    a.part = part_.p;
    a.lpart = lpart_.p;
    a.mu_at_stats = mu_at_stats_.p;
    a.alpha = alpha_;
    a.mu0 = mu0_;
    a.v0 = v0_;
    a.a0 = a0_;
    a.b0 = b0_;
    a.seed = seed_;
    a.var_pi = var_[0];
    a.var_mu = var_[1];
    a.var_s2 = var_[2];
    a.var_z = var_[3];
    return a;
  }

  bool data_ = false;
  int K_ = 0;
  std::int64_t N_ = 0;
  double alpha_, mu0_, v0_, a0_, b0_;
  std::uint64_t seed_ = 0;
  int var_[5] = {0, 1, 2, 3, 4};
  DevBuf<double> x_, pi_, mu_, s2_, part_, lpart_, mu_at_stats_;
  bool fuse_ = true;
  int nbz_ = kBlocks;  // fused z kernel grid  // draw_params_kernel + z_kernel<.., true> (K <= kFuseK; BNMC_GMM_FUSED=0: 6-kernel sweep)
  DevBuf<int> z_;
  DevBuf<std::int64_t> stage64_;  // z upload / write-back staging (int64 store layout)
};

}  // namespace

std::unique_ptr<Model> make_gmm(const bnmc_gpu_desc& d, const Comm& c, Outputs o) {
  return std::make_unique<Gmm>(d, c, o);
}

}  // namespace bnmc_gpu
