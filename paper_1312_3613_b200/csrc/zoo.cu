// csrc/zoo.cu -- the rest of the reference's Gibbs model zoo on the device
// (the remaining conjugate kinds and the sequential scan).
//
//   catmix.bn      theta[k] ~ Dirichlet(alpha + c) rows, phi ~ Dirichlet(beta + c),
//                  z exact discrete (parallel)        plan: theta, phi, z
//   naivebayes.bn  pC, pF[m] Beta-Bernoulli draws (c, f observed)   plan: pC, pF
//   hmm.bn         T[k] Dirichlet rows from transition counts, bias[m] Beta-Bernoulli,
//                  s exact discrete as a SEQUENTIAL scan (each site sees the fresh
//                  s[t-1] and the old s[t+1]; sampler.cpp:259-264)   plan: T, bias, s
//
// Every draw uses the reference's streams: conjugate Dirichlet cells
// keyed(seed,4,var,iter).derive(row, col) (batch.cpp:38-41), scalar conjugate draws
// keyed(seed,4,var,iter).derive(t) (sampler.cpp:183-217; draw_beta = X/(X+Y) from one
// stream, dist.cpp:166-170), exact-discrete sites keyed(seed,3,var,t,iter) with
// draw_from_log_weights (dist.cpp:202-215), and the log-weight pieces summed in the
// conditional's order (0 + piece 1 + piece 2 ...; a guarded piece whose guard fails
// adds 0, eval.cpp:360-391).  The log-joint adds the joint's factors in declaration
// order (eval.cpp:393-422); within a factor, sums run in fixed order.  These models are
// small (not the hot path): simple kernels, one block where a reduction is needed.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"
#include "dist.cuh"

namespace bnmc_gpu {
namespace {

constexpr int kT = 256;

struct ZooArgs {
  int kind;
  std::int64_t N;
  int K, V, S;
  double* A;       // catmix theta [K*V] | naivebayes pC [1] | hmm T [S*S]
  double* B;       // catmix phi [K]     | naivebayes pF [2K] | hmm bias [S]
  int* z;          // catmix z [N]       | -                  | hmm s [N]
  const int* x;    // catmix x [N]       | naivebayes c [N]   | hmm flips [N]
  const int* f;    // naivebayes f [N*K]
  int* cnt;        // histograms (see Zoo::cnt_size)
  double* red;     // [8] log-joint factor sums
  std::uint64_t seed;
  int var[4];      // reference variable ids (declaration order)
  double conc_a, conc_b;  // catmix alpha, beta (0.5); hmm v (0.1)
};

__device__ __forceinline__ double draw_beta(Stream& r, double a, double b) {
  const double x = draw_gamma(r, a);
  const double y = draw_gamma(r, b);
  return x / (x + y);
}

// log_pdf_beta (dist.cpp:78-83)
__device__ __forceinline__ double log_pdf_beta(double x, double a, double b) {
  if (!(a > 0.0) || !(b > 0.0)) return -INFINITY;
  if (!(x > 0.0) || !(x < 1.0)) return -INFINITY;
  return (a - 1.0) * log(x) + (b - 1.0) * log1p(-x) - (lgamma(a) + lgamma(b) - lgamma(a + b));
}

// log_pmf_bernoulli (dist.cpp:99-105)
__device__ __forceinline__ double log_pmf_bernoulli(long long x, double p) {
  if (p < 0.0 || p > 1.0) return -INFINITY;
  if (x == 1) return p > 0.0 ? log(p) : -INFINITY;
  if (x == 0) return p < 1.0 ? log1p(-p) : -INFINITY;
  return -INFINITY;
}

// log_pdf_dirichlet with a constant concentration (dist.cpp:115-130), sequential
__device__ double log_pdf_dirichlet_const(const double* x, int n, double alpha) {
  double sum = 0.0, lp = 0.0, norm = 0.0, asum = 0.0;
  if (!(alpha > 0.0)) return -INFINITY;
  const double lga = lgamma(alpha);  // the reference's per-element lgamma(alpha), once
  for (int i = 0; i < n; ++i) {
    if (!(x[i] > 0.0)) return -INFINITY;
    sum += x[i];
    lp += (alpha - 1.0) * log(x[i]);
    norm += lga;
    asum += alpha;
  }
  if (fabs(sum - 1.0) > 1e-9) return -INFINITY;
  return lp - norm + lgamma(asum);
}

// draw_from_log_weights (dist.cpp:202-215) over n <= 64 weights; -1 when all are -inf
__device__ int draw_log_weights(Stream& r, const double* lw, int n) {
  double mx = -INFINITY;
  for (int i = 0; i < n; ++i) mx = fmax(mx, lw[i]);
  if (!isfinite(mx)) return -1;
  double total = 0.0;
  for (int i = 0; i < n; ++i) total += exp(lw[i] - mx);
  const double u = r.next_unit() * total;
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += exp(lw[i] - mx);
    if (u < acc) return i;
  }
  return n - 1;
}

// Dirichlet rows (sample_dirichlet_batch, per_row, batch.cpp:45-83): block per row,
// cell (r, c) from keyed(seed,4,var,iter).derive(r, c); alpha = conc + counts.
__global__ void dirichlet_rows_kernel(double* out, const int* counts, int rows, int cols, double conc,
                                      std::uint64_t seed, int var, const std::int64_t* iter_p) {
  __shared__ double scratch[32];
  const std::uint64_t key = keyed(seed, kConjugate, static_cast<std::uint64_t>(var),
                                  static_cast<std::uint64_t>(*iter_p));
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    double part = 0.0;
    for (int c = threadIdx.x; c < cols; c += blockDim.x) {
      Stream s(derive(key, static_cast<std::uint64_t>(r), static_cast<std::uint64_t>(c)));
      const double g = draw_gamma(s, conc + static_cast<double>(counts[r * cols + c]));
      out[static_cast<std::size_t>(r) * cols + c] = g;
      part += g;
    }
    const double S = block_sum(part, scratch);
    for (int c = threadIdx.x; c < cols; c += blockDim.x) out[static_cast<std::size_t>(r) * cols + c] /= S;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------
// catmix
// ---------------------------------------------------------------------------------
// counts of the current z: cnt[k*V + v] (theta block), cnt[K*V + k] (phi block)
__global__ void catmix_count_kernel(ZooArgs a, int* err) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < a.N;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int k = a.z[i], v = a.x[i];
    if (k < 0 || k >= a.K) {
      atomicOr(err, kErrBin);
      continue;
    }
    if (v >= 0 && v < a.V) atomicAdd(&a.cnt[k * a.V + v], 1);
    atomicAdd(&a.cnt[a.K * a.V + k], 1);
  }
}

// z[i] | rest: logw[v] = (0 + log phi[v]) + log theta[v][x_i]
__global__ void catmix_z_kernel(ZooArgs a, const std::int64_t* iter_p, int* err) {
  const std::int64_t iter = *iter_p;
  const std::uint64_t zp = fold(fold(fold(1, a.seed), kDiscrete), static_cast<std::uint64_t>(a.var[2]));
  double lw[64];
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < a.N;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int xi = a.x[i];
    for (int v = 0; v < a.K; ++v) {
      double lp = 0.0;
      lp += log_prob(a.B[v]);
      lp += (xi >= 0 && xi < a.V) ? log_prob(a.A[static_cast<std::size_t>(v) * a.V + xi]) : -INFINITY;
      lw[v] = lp;
    }
    Stream r(fold(fold(zp, static_cast<std::uint64_t>(i)), static_cast<std::uint64_t>(iter)));
    const int k = draw_log_weights(r, lw, a.K);
    if (k < 0) atomicOr(err, kErrDomain);
    else a.z[i] = k;
  }
}

// log-joint factors [theta, phi, z, x] (single block)
constexpr int kZooLjBlocks = 148 * 2;

// per-block partials of the z and x factors (fixed-order block sums)
__global__ void catmix_lj_part_kernel(ZooArgs a, double* part) {
  __shared__ double scratch[64];
  double v[2] = {0.0, 0.0};
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < a.N;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int k = a.z[i], xi = a.x[i];
    if (k < 0 || k >= a.K) {
      v[0] += -INFINITY;
      v[1] += -INFINITY;
      continue;
    }
    v[0] += log_prob(a.B[k]);
    v[1] += (xi >= 0 && xi < a.V) ? log_prob(a.A[static_cast<std::size_t>(k) * a.V + xi]) : -INFINITY;
  }
  block_sum_n<2>(v, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = v[0];
    part[2 * blockIdx.x + 1] = v[1];
  }
}

// log-joint factors [theta, phi, z, x] (single block; the partials in block order)
__global__ void catmix_lj_kernel(ZooArgs a, const double* part) {
  __shared__ double scratch[32];
  double ft = 0.0;
  for (int k = threadIdx.x; k < a.K; k += blockDim.x)
    ft += log_pdf_dirichlet_const(a.A + static_cast<std::size_t>(k) * a.V, a.V, a.conc_a);
  ft = block_sum(ft, scratch);
  if (threadIdx.x == 0) {
    double fz = 0.0, fx = 0.0;
    for (int b = 0; b < kZooLjBlocks; ++b) {
      fz += part[2 * b];
      fx += part[2 * b + 1];
    }
    a.red[0] = ft;
    a.red[1] = log_pdf_dirichlet_const(a.B, a.K, a.conc_b);
    a.red[2] = fz;
    a.red[3] = fx;
    a.red[4] = 0.0;
  }
}

// ---------------------------------------------------------------------------------
// naivebayes (counts of the observed data, computed once at upload)
// ---------------------------------------------------------------------------------
// cnt[1] = sum c; cnt[2 + 2m] = n_m, cnt[3 + 2m] = s_m over f[i,j] with 2j + c_i = m
__global__ void nb_count_kernel(ZooArgs a) {
  for (std::int64_t e = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; e < a.N * a.K;
       e += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t i = e / a.K;
    const int j = static_cast<int>(e - i * a.K);
    const int m = j * 2 + a.x[i];
    if (m >= 0 && m < 2 * a.K) {
      atomicAdd(&a.cnt[2 + 2 * m], 1);
      atomicAdd(&a.cnt[3 + 2 * m], a.f[e]);
    }
    if (j == 0) atomicAdd(&a.cnt[1], a.x[i]);
  }
}

// pC ~ Beta(0.5 + s, 0.5 + n - s), pF[m] ~ Beta(0.5 + s_m, 0.5 + n_m - s_m)
__global__ void nb_draw_kernel(ZooArgs a, const std::int64_t* iter_p) {
  const std::int64_t iter = *iter_p;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {
    const std::uint64_t key = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var[0]),
                                    static_cast<std::uint64_t>(iter));
    Stream r(derive(key, 0));
    const double n = static_cast<double>(a.N), s = static_cast<double>(a.cnt[1]);
    a.A[0] = draw_beta(r, 0.5 + s, 0.5 + (n - s));
  }
  if (t < 2 * a.K) {
    const std::uint64_t key = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var[2]),
                                    static_cast<std::uint64_t>(iter));
    Stream r(derive(key, static_cast<std::uint64_t>(t)));
    const double n = static_cast<double>(a.cnt[2 + 2 * t]), s = static_cast<double>(a.cnt[3 + 2 * t]);
    a.B[t] = draw_beta(r, 0.5 + s, 0.5 + (n - s));
  }
}

// s * log p + (n - s) * log(1 - p): the sum of n Bernoulli log-pmfs with s ones
__device__ __forceinline__ double bern_sum(double n, double s, double p) {
  double out = 0.0;
  if (s > 0.0) out += s * log_pmf_bernoulli(1, p);
  if (n - s > 0.0) out += (n - s) * log_pmf_bernoulli(0, p);
  return out;
}

// log-joint factors [pC, c, pF, f] from the counts (single block)
__global__ void nb_lj_kernel(ZooArgs a) {
  __shared__ double scratch[32];
  double fpf = 0.0, ff = 0.0;
  for (int m = threadIdx.x; m < 2 * a.K; m += blockDim.x) {
    fpf += log_pdf_beta(a.B[m], 0.5, 0.5);
    ff += bern_sum(a.cnt[2 + 2 * m], a.cnt[3 + 2 * m], a.B[m]);
  }
  fpf = block_sum(fpf, scratch);
  ff = block_sum(ff, scratch);
  if (threadIdx.x == 0) {
    a.red[0] = log_pdf_beta(a.A[0], 0.5, 0.5);
    a.red[1] = bern_sum(static_cast<double>(a.N), a.cnt[1], a.A[0]);
    a.red[2] = fpf;
    a.red[3] = ff;
    a.red[4] = 0.0;
  }
}

// ---------------------------------------------------------------------------------
// hmm
// ---------------------------------------------------------------------------------
// cnt[k*S + v]: transitions (s[0] counted in row 0, sampler plan describe_hmm.txt);
// cnt[S*S + m] = n_m, cnt[S*S + S + m] = sum of flips with s = m
__global__ void hmm_count_kernel(ZooArgs a, int* err) {
  extern __shared__ int hist[];  // S*S + 2S block-local counts, added to cnt at the end
  const int S = a.S, nh = S * S + 2 * S;
  for (int i = threadIdx.x; i < nh; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < a.N;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int st = a.z[t];
    if (st < 0 || st >= S) {
      atomicOr(err, kErrBin);
      continue;
    }
    const int prev = t == 0 ? 0 : a.z[t - 1];
    if (prev >= 0 && prev < S) atomicAdd(&hist[prev * S + st], 1);
    atomicAdd(&hist[S * S + st], 1);
    atomicAdd(&hist[S * S + S + st], a.x[t]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nh; i += blockDim.x)
    if (hist[i]) atomicAdd(&a.cnt[i], hist[i]);
}

__global__ void hmm_bias_kernel(ZooArgs a, const std::int64_t* iter_p) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= a.S) return;
  const std::uint64_t key = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var[1]),
                                  static_cast<std::uint64_t>(*iter_p));
  Stream r(derive(key, static_cast<std::uint64_t>(m)));
  const double n = a.cnt[a.S * a.S + m], s = a.cnt[a.S * a.S + a.S + m];
  a.B[m] = draw_beta(r, 1.0 + s, 1.0 + (n - s));
}

// s[t] | rest, t = 0 .. N-1 in order: site t sees the NEW s[t-1] (`prev`) and the OLD
// s[t+1] (read from `zold`):
// logw[v] = 0 + {log T[0][v]}_{t==0} + {log T[s[t-1]][v]}_{t>=1} + {log T[v][s[t+1]]}_{t+1<N}
//             + log Bernoulli(flips[t] | bias[v])
// -1 when every weight is -inf.
__device__ __forceinline__ int hmm_site(const ZooArgs& a, const int* zold, std::uint64_t zp, std::int64_t iter,
                                        std::int64_t t, int prev, double* lw) {
  const int S = a.S;
  const int next = t + 1 < a.N ? zold[t + 1] : 0;
  for (int v = 0; v < S; ++v) {
    double lp = 0.0;
    if (t == 0) lp += log_prob(a.A[v]);
    if (t >= 1) lp += (prev >= 0 && prev < S) ? log_prob(a.A[prev * S + v]) : -INFINITY;
    if (t + 1 < a.N) lp += (next >= 0 && next < S) ? log_prob(a.A[v * S + next]) : -INFINITY;
    lp += log_pmf_bernoulli(a.x[t], a.B[v]);
    lw[v] = lp;
  }
  Stream r(fold(fold(zp, static_cast<std::uint64_t>(t)), static_cast<std::uint64_t>(iter)));
  return draw_log_weights(r, lw, S);
}

__device__ __forceinline__ std::uint64_t hmm_zkey(const ZooArgs& a) {
  return fold(fold(fold(1, a.seed), kDiscrete), static_cast<std::uint64_t>(a.var[2]));
}

// The scan site by site on one thread (BNMC_HMM_SERIAL=1; the parity check of the
// chunked scan below).
__global__ void hmm_scan_kernel(ZooArgs a, const std::int64_t* iter_p, int* err) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const std::int64_t iter = *iter_p;
  const std::uint64_t zp = hmm_zkey(a);
  double lw[64];
  for (std::int64_t t = 0; t < a.N; ++t) {
    const int k = hmm_site(a, a.z, zp, iter, t, t >= 1 ? a.z[t - 1] : 0, lw);
    if (k < 0) {
      atomicOr(err, kErrDomain);
      return;
    }
    a.z[t] = k;
  }
}

// The same scan in parallel. A site's stream does not depend on the state, so site t is
// a map prev -> s[t] over the S states, and a chunk of sites is the composition of its
// sites' maps: (1) every chunk runs from each start state (distinct predecessors drawn
// once per site; -1 marks a chain that hit an all -inf site); (2) one block composes the
// chunk maps by a Hillis-Steele scan and reads each chunk's true start (the chain from
// s[-1] = 0); (3) every chunk redraws its sites from its true start and writes them. The
// old successors come from the sweep-start snapshot `zold`.
__global__ void hmm_scan_ends_kernel(ZooArgs a, const int* zold, const std::int64_t* iter_p, std::int64_t chunk,
                                     std::int64_t nchunks, int* maps) {
  const std::int64_t c = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nchunks) return;
  const int S = a.S;
  const std::int64_t iter = *iter_p;
  const std::uint64_t zp = hmm_zkey(a);
  int st[64], memo[64];
  double lw[64];
  for (int j = 0; j < S; ++j) st[j] = j;
  const std::int64_t t1 = min(a.N, (c + 1) * chunk);
  for (std::int64_t t = c * chunk; t < t1; ++t) {
    for (int j = 0; j < S; ++j) memo[j] = -2;
    for (int j = 0; j < S; ++j) {
      const int p = st[j];
      if (p < 0) continue;
      if (memo[p] == -2) memo[p] = hmm_site(a, zold, zp, iter, t, p, lw);
      st[j] = memo[p];
    }
  }
  for (int j = 0; j < S; ++j) maps[c * S + j] = st[j];
}

constexpr int kHmmLinkMax = 24576;  // map entries: two buffers of 96 KB in shared memory

__global__ void __launch_bounds__(1024) hmm_scan_link_kernel(int S, std::int64_t nchunks, const int* maps,
                                                             int* starts) {
  extern __shared__ int m[];
  int* cur = m;
  int* nxt = m + kHmmLinkMax;
  const int n = static_cast<int>(nchunks) * S;
  for (int i = threadIdx.x; i < n; i += blockDim.x) cur[i] = maps[i];
  __syncthreads();
  for (int off = 1; off < nchunks; off <<= 1) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int c = i / S;
      if (c < off) {
        nxt[i] = cur[i];
      } else {
        const int p = cur[i - off * S];  // chunks (c-off .. ] composed, then chunk c's map
        nxt[i] = p < 0 ? -1 : cur[c * S + p];
      }
    }
    __syncthreads();
    int* t = cur;
    cur = nxt;
    nxt = t;
  }
  for (int c = threadIdx.x; c < nchunks; c += blockDim.x) starts[c] = c == 0 ? 0 : cur[(c - 1) * S];
}

__global__ void hmm_scan_chain_kernel(ZooArgs a, const int* zold, const std::int64_t* iter_p, std::int64_t chunk,
                                      std::int64_t nchunks, const int* starts, int* err) {
  const std::int64_t c = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nchunks) return;
  int st = starts[c];
  if (st < 0) return;  // an earlier site ended the scan
  const std::int64_t iter = *iter_p;
  const std::uint64_t zp = hmm_zkey(a);
  double lw[64];
  const std::int64_t t1 = min(a.N, (c + 1) * chunk);
  for (std::int64_t t = c * chunk; t < t1; ++t) {
    st = hmm_site(a, zold, zp, iter, t, st, lw);
    if (st < 0) {
      atomicOr(err, kErrDomain);
      return;
    }
    a.z[t] = st;
  }
}

// log-joint factors [T, bias, s[0], s[t>=1], flips] (single block)
// per-block partials of the site factors s[t>=1] and flips (fixed-order block sums)
__global__ void hmm_lj_part_kernel(ZooArgs a, double* part) {
  __shared__ double scratch[64];
  const int S = a.S;
  double v[2] = {0.0, 0.0};
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < a.N;
       t += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const int st = a.z[t];
    const bool ok = st >= 0 && st < S;
    if (t >= 1) {
      const int pv = a.z[t - 1];
      v[0] += (ok && pv >= 0 && pv < S) ? log_prob(a.A[pv * S + st]) : -INFINITY;
    }
    v[1] += ok ? log_pmf_bernoulli(a.x[t], a.B[st]) : -INFINITY;
  }
  block_sum_n<2>(v, scratch);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = v[0];
    part[2 * blockIdx.x + 1] = v[1];
  }
}

// log-joint factors [T, bias, s[0], s[t>=1], flips] (single block; the partials in block order)
__global__ void hmm_lj_kernel(ZooArgs a, const double* part) {
  __shared__ double scratch[32];
  const int S = a.S;
  double fT = 0.0, fb = 0.0;
  for (int k = threadIdx.x; k < S; k += blockDim.x) {
    fT += log_pdf_dirichlet_const(a.A + static_cast<std::size_t>(k) * S, S, a.conc_a);
    fb += log_pdf_beta(a.B[k], 1.0, 1.0);
  }
  fT = block_sum(fT, scratch);
  fb = block_sum(fb, scratch);
  if (threadIdx.x == 0) {
    double fs = 0.0, ff = 0.0;
    for (int b = 0; b < kZooLjBlocks; ++b) {
      fs += part[2 * b];
      ff += part[2 * b + 1];
    }
    const int s0 = a.N > 0 ? a.z[0] : 0;
    a.red[0] = fT;
    a.red[1] = fb;
    a.red[2] = a.N > 0 ? ((s0 >= 0 && s0 < S) ? log_prob(a.A[s0]) : -INFINITY) : 0.0;
    a.red[3] = fs;
    a.red[4] = ff;
  }
}

// ((((red0 + red1) + red2) + red3) + red4): the joint's factors in declaration order
__global__ void zoo_finalize_kernel(ZooArgs a, Outputs o, int advance, int nf) {
  double lj = 0.0;
  for (int i = 0; i < nf; ++i) lj += a.red[i];
  const std::int64_t it = *o.iter;
  o.lj[it & (kRing - 1)] = lj;
  o.acc[it & (kRing - 1)] = 0;
  if (advance) *o.iter = it + 1;
}

// prior_init (sampler.cpp:542-555): declaration order, one stream keyed(seed,5,var,elem)
// per element; Dirichlet rows draw their gammas sequentially from that one stream
// (draw_dirichlet, dist.cpp:193-200); categorical by linear scan (dist.cpp:183-191).
__device__ void prior_dirichlet_row(Stream& s, double* row, int n, double conc) {
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    row[i] = draw_gamma(s, conc);
    sum += row[i];
  }
  for (int i = 0; i < n; ++i) row[i] /= sum;
}

__device__ int prior_categorical(Stream& s, const double* p, int n) {
  const double u = s.next_unit();
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += p[i];
    if (u < acc) return i;
  }
  return n - 1;
}

__device__ __forceinline__ Stream prior_stream(std::uint64_t seed, int var, std::int64_t elem) {
  return Stream(keyed(seed, kInit, static_cast<std::uint64_t>(var), static_cast<std::uint64_t>(elem)));
}

// Each element has its own stream, so the elements are drawn in parallel: Dirichlet rows
// thread per row, Beta draws and categorical picks thread per element.
__global__ void zoo_prior_rows_kernel(double* out, int rows, int cols, double conc, std::uint64_t seed, int var) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= rows) return;
  Stream s = prior_stream(seed, var, k);
  prior_dirichlet_row(s, out + static_cast<std::size_t>(k) * cols, cols, conc);
}

__global__ void zoo_prior_beta_kernel(double* out, int n, double a, double b, std::uint64_t seed, int var) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  Stream s = prior_stream(seed, var, m);
  out[m] = draw_beta(s, a, b);
}

__global__ void zoo_prior_cat_kernel(int* z, std::int64_t N, const double* p, int n, std::uint64_t seed, int var) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    Stream r = prior_stream(seed, var, i);
    z[i] = prior_categorical(r, p, n);
  }
}

// HMM prior chain s[t] ~ Cat(T[s[t-1]]), s[-1] = 0, step t with its own stream: step t is
// the map prev -> pick(u_t, T[prev]) over S states, so chunks of steps compose in
// parallel: every chunk runs from each start state (ends), one thread links the chunks
// (starts), every chunk re-runs from its true start and writes the states.
constexpr int kHmmPriorMaxS = 16;

__device__ __forceinline__ int pick_row(double u, const double* row, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += row[i];
    if (u < acc) return i;
  }
  return n - 1;
}

__global__ void hmm_prior_ends_kernel(ZooArgs a, std::uint64_t seed, std::int64_t chunk, std::int64_t nchunks,
                                      int* ends) {
  const std::int64_t c = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nchunks) return;
  int st[kHmmPriorMaxS];
  for (int j = 0; j < a.S; ++j) st[j] = j;
  const std::int64_t t1 = min(a.N, (c + 1) * chunk);
  for (std::int64_t t = c * chunk; t < t1; ++t) {
    const double u = prior_stream(seed, a.var[2], t).next_unit();
    for (int j = 0; j < a.S; ++j) st[j] = pick_row(u, a.A + static_cast<std::size_t>(st[j]) * a.S, a.S);
  }
  for (int j = 0; j < a.S; ++j) ends[c * a.S + j] = st[j];
}

__global__ void hmm_prior_link_kernel(int S, std::int64_t nchunks, const int* ends, int* starts) {
  int st = 0;
  for (std::int64_t c = 0; c < nchunks; ++c) {
    starts[c] = st;
    st = ends[c * S + st];
  }
}

__global__ void hmm_prior_chain_kernel(ZooArgs a, std::uint64_t seed, std::int64_t chunk, std::int64_t nchunks,
                                       const int* starts) {
  const std::int64_t c = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (c >= nchunks) return;
  int st = starts[c];
  const std::int64_t t1 = min(a.N, (c + 1) * chunk);
  for (std::int64_t t = c * chunk; t < t1; ++t) {
    const double u = prior_stream(seed, a.var[2], t).next_unit();
    st = pick_row(u, a.A + static_cast<std::size_t>(st) * a.S, a.S);
    a.z[t] = st;
  }
}

// S > kHmmPriorMaxS (or BNMC_PRIOR_SERIAL=1): the chain step by step
__global__ void hmm_prior_serial_kernel(ZooArgs a, std::uint64_t seed) {
  for (std::int64_t t = 0; t < a.N; ++t) {
    Stream r = prior_stream(seed, a.var[2], t);
    const int prev = t == 0 ? 0 : a.z[t - 1];
    a.z[t] = prior_categorical(r, a.A + static_cast<std::size_t>(prev) * a.S, a.S);
  }
}

__global__ void i64_to_i32(const std::int64_t* in, int* out, std::int64_t n, std::int64_t lo, std::int64_t hi,
                           int* err) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t v = in[i];
    if (v < lo || v >= hi) atomicOr(err, kErrBin);
    out[i] = static_cast<int>(v);
  }
}

__global__ void i32_to_i64(const int* in, std::int64_t* out, std::int64_t n) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

unsigned grid_for(std::int64_t n) {
  return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((n + kT - 1) / kT, 148 * 8)));
}

class Zoo final : public Model {
 public:
  Zoo(const bnmc_gpu_desc& d, const Comm& c, Outputs o) : kind_(d.kind) {
    out = o;
    require(c.world == 1, BNMC_GPU_ERR_ARG, "catmix / naivebayes / hmm run as replicas only (world_size 1)");
    require(d.N >= 0, BNMC_GPU_ERR_ARG, "N must be >= 0");
    N_ = d.N;
    seed_ = d.seed;
    for (int i = 0; i < 4; ++i) var_[i] = d.var_ids[i];
    if (kind_ == BNMC_GPU_CATMIX) {
      require(d.K >= 1 && d.K <= 64 && d.V >= 1, BNMC_GPU_ERR_ARG, "catmix needs 1 <= K <= 64, V >= 1");
      K_ = static_cast<int>(d.K);
      V_ = static_cast<int>(d.V);
      na_ = static_cast<std::int64_t>(K_) * V_;
      nb_ = K_;
      ncnt_ = na_ + K_;
      conc_a_ = d.hyper[0] > 0 ? d.hyper[0] : 0.5;
      conc_b_ = d.hyper[1] > 0 ? d.hyper[1] : 0.5;
    } else if (kind_ == BNMC_GPU_NAIVEBAYES) {
      require(d.K >= 1, BNMC_GPU_ERR_ARG, "naivebayes needs K >= 1 features");
      K_ = static_cast<int>(d.K);
      na_ = 1;
      nb_ = 2 * K_;
      ncnt_ = 2 + 4 * K_;
    } else {
      require(d.K >= 1 && d.K <= 64, BNMC_GPU_ERR_ARG, "hmm needs 1 <= S <= 64 states (desc.K)");
      S_ = static_cast<int>(d.K);
      na_ = static_cast<std::int64_t>(S_) * S_;
      nb_ = S_;
      ncnt_ = na_ + 2 * S_;
      conc_a_ = d.hyper[0] > 0 ? d.hyper[0] : 0.1;
      // chunked s-scan: chunks x S map entries fit the link block's shared memory
      const char* e = std::getenv("BNMC_HMM_SERIAL");
      if (N_ > 1 && !(e && std::string(e) != "0")) {
        hmm_chunks_ = std::min<std::int64_t>(N_, kHmmLinkMax / S_);
        hmm_chunk_ = (N_ + hmm_chunks_ - 1) / hmm_chunks_;
        hmm_chunks_ = (N_ + hmm_chunk_ - 1) / hmm_chunk_;
        zold_.alloc(N_);
        maps_.alloc(hmm_chunks_ * S_);
        BNMC_CUDA(cudaFuncSetAttribute(hmm_scan_link_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sizeof(int) * 2 * kHmmLinkMax)));
        starts_.alloc(hmm_chunks_);
      }
    }
    A_.alloc(na_);
    B_.alloc(nb_);
    ljpart_.alloc(2 * kZooLjBlocks);
    z_.alloc(std::max<std::int64_t>(N_, 1));
    x_.alloc(std::max<std::int64_t>(N_, 1));
    if (kind_ == BNMC_GPU_NAIVEBAYES) f_.alloc(std::max<std::int64_t>(N_ * K_, 1));
    cnt_.alloc(ncnt_);
    red_.alloc(8);
    A_.zero(nullptr);
    B_.zero(nullptr);
    z_.zero(nullptr);
    x_.zero(nullptr);
    cnt_.zero(nullptr);
    red_.zero(nullptr);
    BNMC_CUDA(cudaDeviceSynchronize());
  }

  void upload(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, true); }
  void upload_state(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, !data_); }

  void download(const bnmc_gpu_store& s, cudaStream_t st) override {
    const char* obs = s.observed;
    auto want = [&](int v) { return !(obs && obs[v]); };
    if (want(var_[0]) && s.real[var_[0]])
      BNMC_CUDA(cudaMemcpyAsync(s.real[var_[0]], A_.p, A_.bytes(), cudaMemcpyDeviceToHost, st));
    const int vb = kind_ == BNMC_GPU_CATMIX ? var_[1] : (kind_ == BNMC_GPU_NAIVEBAYES ? var_[2] : var_[1]);
    if (want(vb) && s.real[vb]) BNMC_CUDA(cudaMemcpyAsync(s.real[vb], B_.p, B_.bytes(), cudaMemcpyDeviceToHost, st));
    if (kind_ != BNMC_GPU_NAIVEBAYES && want(var_[2]) && s.ival[var_[2]] && N_ > 0) {
      if (stage_.n < static_cast<std::size_t>(N_)) stage_.alloc(N_);
      i32_to_i64<<<grid_for(N_), kT, 0, st>>>(z_.p, stage_.p, N_);
      BNMC_CUDA(cudaMemcpyAsync(s.ival[var_[2]], stage_.p, stage_.bytes(), cudaMemcpyDeviceToHost, st));
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  void enqueue_sweep(cudaStream_t st) override {
    ZooArgs a = args();
    mark(st, "begin");
    if (kind_ == BNMC_GPU_CATMIX) {
      cnt_.zero(st);
      catmix_count_kernel<<<grid_for(N_), kT, 0, st>>>(a, out.err);
      dirichlet_rows_kernel<<<K_, 128, 0, st>>>(A_.p, cnt_.p, K_, V_, conc_a_, seed_, var_[0], out.iter);
      dirichlet_rows_kernel<<<1, 64, 0, st>>>(B_.p, cnt_.p + na_, 1, K_, conc_b_, seed_, var_[1], out.iter);
      mark(st, "theta_phi");
      catmix_z_kernel<<<grid_for(N_), kT, 0, st>>>(a, out.iter, out.err);
      mark(st, "z");
      catmix_lj_part_kernel<<<kZooLjBlocks, 256, 0, st>>>(a, ljpart_.p);
      catmix_lj_kernel<<<1, 64, 0, st>>>(a, ljpart_.p);
      zoo_finalize_kernel<<<1, 1, 0, st>>>(a, out, 1, 4);
    } else if (kind_ == BNMC_GPU_NAIVEBAYES) {
      nb_draw_kernel<<<static_cast<unsigned>((2 * K_ + kT) / kT), kT, 0, st>>>(a, out.iter);
      mark(st, "pC_pF");
      nb_lj_kernel<<<1, 1024, 0, st>>>(a);
      zoo_finalize_kernel<<<1, 1, 0, st>>>(a, out, 1, 4);
    } else {
      cnt_.zero(st);
      hmm_count_kernel<<<std::min(grid_for(N_), 148u * 2), kT, sizeof(int) * (S_ * S_ + 2 * S_), st>>>(a, out.err);
      dirichlet_rows_kernel<<<S_, 64, 0, st>>>(A_.p, cnt_.p, S_, S_, conc_a_, seed_, var_[0], out.iter);
      hmm_bias_kernel<<<1, 64, 0, st>>>(a, out.iter);
      mark(st, "T_bias");
      if (hmm_chunks_ > 0) {
        BNMC_CUDA(cudaMemcpyAsync(zold_.p, z_.p, sizeof(int) * N_, cudaMemcpyDeviceToDevice, st));
        const unsigned g = static_cast<unsigned>((hmm_chunks_ + 127) / 128);
        hmm_scan_ends_kernel<<<g, 128, 0, st>>>(a, zold_.p, out.iter, hmm_chunk_, hmm_chunks_, maps_.p);
        hmm_scan_link_kernel<<<1, 1024, sizeof(int) * 2 * kHmmLinkMax, st>>>(S_, hmm_chunks_, maps_.p, starts_.p);
        hmm_scan_chain_kernel<<<g, 128, 0, st>>>(a, zold_.p, out.iter, hmm_chunk_, hmm_chunks_, starts_.p, out.err);
      } else {
        hmm_scan_kernel<<<1, 32, 0, st>>>(a, out.iter, out.err);
      }
      mark(st, "s_scan");
      hmm_lj_part_kernel<<<kZooLjBlocks, 256, 0, st>>>(a, ljpart_.p);
      hmm_lj_kernel<<<1, 64, 0, st>>>(a, ljpart_.p);
      zoo_finalize_kernel<<<1, 1, 0, st>>>(a, out, 1, 5);
    }
    mark(st, "log_joint");
    BNMC_CUDA(cudaGetLastError());
  }

  void enqueue_log_joint(cudaStream_t st) override {
    ZooArgs a = args();
    if (kind_ == BNMC_GPU_CATMIX) {
      catmix_lj_part_kernel<<<kZooLjBlocks, 256, 0, st>>>(a, ljpart_.p);
      catmix_lj_kernel<<<1, 64, 0, st>>>(a, ljpart_.p);
      zoo_finalize_kernel<<<1, 1, 0, st>>>(a, out, 0, 4);
    } else if (kind_ == BNMC_GPU_NAIVEBAYES) {
      nb_lj_kernel<<<1, 1024, 0, st>>>(a);
      zoo_finalize_kernel<<<1, 1, 0, st>>>(a, out, 0, 4);
    } else {
      hmm_lj_part_kernel<<<kZooLjBlocks, 256, 0, st>>>(a, ljpart_.p);
      hmm_lj_kernel<<<1, 64, 0, st>>>(a, ljpart_.p);
      zoo_finalize_kernel<<<1, 1, 0, st>>>(a, out, 0, 5);
    }
    BNMC_CUDA(cudaGetLastError());
  }

  void prior_init(std::uint64_t seed, cudaStream_t st) override {
    const ZooArgs a = args();
    if (kind_ == BNMC_GPU_CATMIX) {
      zoo_prior_rows_kernel<<<(K_ + 63) / 64, 64, 0, st>>>(A_.p, K_, V_, a.conc_a, seed, a.var[0]);
      zoo_prior_rows_kernel<<<1, 1, 0, st>>>(B_.p, 1, K_, a.conc_b, seed, a.var[1]);
      zoo_prior_cat_kernel<<<grid_for(N_), kT, 0, st>>>(z_.p, N_, B_.p, K_, seed, a.var[2]);
    } else if (kind_ == BNMC_GPU_NAIVEBAYES) {
      zoo_prior_beta_kernel<<<1, 1, 0, st>>>(A_.p, 1, 0.5, 0.5, seed, a.var[0]);
      zoo_prior_beta_kernel<<<(2 * K_ + 63) / 64, 64, 0, st>>>(B_.p, 2 * K_, 0.5, 0.5, seed, a.var[2]);
    } else {  // hmm
      zoo_prior_rows_kernel<<<(S_ + 63) / 64, 64, 0, st>>>(A_.p, S_, S_, a.conc_a, seed, a.var[0]);
      zoo_prior_beta_kernel<<<(S_ + 63) / 64, 64, 0, st>>>(B_.p, S_, 1.0, 1.0, seed, a.var[1]);
      const char* e = std::getenv("BNMC_PRIOR_SERIAL");
      if (N_ > 0 && S_ <= kHmmPriorMaxS && !(e && std::string(e) != "0")) {
        const std::int64_t nchunks = std::min<std::int64_t>(N_, 148 * 128);
        const std::int64_t chunk = (N_ + nchunks - 1) / nchunks;
        DevBuf<int> ends, starts;
        ends.alloc(nchunks * S_);
        starts.alloc(nchunks);
        hmm_prior_ends_kernel<<<static_cast<unsigned>((nchunks + 127) / 128), 128, 0, st>>>(a, seed, chunk, nchunks,
                                                                                           ends.p);
        hmm_prior_link_kernel<<<1, 1, 0, st>>>(S_, nchunks, ends.p, starts.p);
        hmm_prior_chain_kernel<<<static_cast<unsigned>((nchunks + 127) / 128), 128, 0, st>>>(a, seed, chunk, nchunks,
                                                                                            starts.p);
        BNMC_CUDA(cudaGetLastError());
        BNMC_CUDA(cudaStreamSynchronize(st));
      } else if (N_ > 0) {
        hmm_prior_serial_kernel<<<1, 1, 0, st>>>(a, seed);
      }
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  std::vector<StateBuf> state_buffers() override {
    std::vector<StateBuf> b{{reinterpret_cast<void**>(&A_.p), A_.bytes()}, {reinterpret_cast<void**>(&B_.p), B_.bytes()}};
    if (kind_ != BNMC_GPU_NAIVEBAYES) b.push_back({reinterpret_cast<void**>(&z_.p), sizeof(int) * static_cast<std::size_t>(N_)});
    return b;
  }

 private:
  static void check_len(const bnmc_gpu_store& s, int var, std::int64_t want, const char* name) {
    require(var >= 0 && var < s.n_vars && s.len && s.len[var] == want, BNMC_GPU_ERR_RUNTIME,
            std::string("variable '") + name + "' has flat length " +
                std::to_string(var >= 0 && var < s.n_vars && s.len ? s.len[var] : -1) + ", expected " +
                std::to_string(want));
  }

  void ints_to_device(const std::int64_t* h, int* d, std::int64_t n, std::int64_t hi, cudaStream_t st) {
    if (n <= 0) return;
    if (stage_.n < static_cast<std::size_t>(n)) stage_.alloc(n);
    BNMC_CUDA(cudaMemcpyAsync(stage_.p, h, sizeof(std::int64_t) * n, cudaMemcpyHostToDevice, st));
    i64_to_i32<<<grid_for(n), kT, 0, st>>>(stage_.p, d, n, 0, hi, out.err);
  }

  void upload_impl(const bnmc_gpu_store& s, cudaStream_t st, bool with_data) {
    if (kind_ == BNMC_GPU_CATMIX) {
      check_len(s, var_[0], na_, "theta");
      check_len(s, var_[1], K_, "phi");
      check_len(s, var_[2], N_, "z");
      check_len(s, var_[3], N_, "x");
      BNMC_CUDA(cudaMemcpyAsync(A_.p, s.real[var_[0]], A_.bytes(), cudaMemcpyHostToDevice, st));
      BNMC_CUDA(cudaMemcpyAsync(B_.p, s.real[var_[1]], B_.bytes(), cudaMemcpyHostToDevice, st));
      ints_to_device(s.ival[var_[2]], z_.p, N_, K_, st);
      if (with_data) ints_to_device(s.ival[var_[3]], x_.p, N_, V_, st);
    } else if (kind_ == BNMC_GPU_NAIVEBAYES) {
      check_len(s, var_[0], 1, "pC");
      check_len(s, var_[1], N_, "c");
      check_len(s, var_[2], 2 * K_, "pF");
      check_len(s, var_[3], N_ * K_, "f");
      BNMC_CUDA(cudaMemcpyAsync(A_.p, s.real[var_[0]], A_.bytes(), cudaMemcpyHostToDevice, st));
      BNMC_CUDA(cudaMemcpyAsync(B_.p, s.real[var_[2]], B_.bytes(), cudaMemcpyHostToDevice, st));
      if (with_data) {
        ints_to_device(s.ival[var_[1]], x_.p, N_, 2, st);
        ints_to_device(s.ival[var_[3]], f_.p, N_ * K_, 2, st);
        // the Beta-Bernoulli statistics depend on the observed data only: count once
        cnt_.zero(st);
        ZooArgs a = args();
        nb_count_kernel<<<grid_for(N_ * K_), kT, 0, st>>>(a);
      }
    } else {
      check_len(s, var_[0], na_, "T");
      check_len(s, var_[1], S_, "bias");
      check_len(s, var_[2], N_, "s");
      check_len(s, var_[3], N_, "flips");
      BNMC_CUDA(cudaMemcpyAsync(A_.p, s.real[var_[0]], A_.bytes(), cudaMemcpyHostToDevice, st));
      BNMC_CUDA(cudaMemcpyAsync(B_.p, s.real[var_[1]], B_.bytes(), cudaMemcpyHostToDevice, st));
      ints_to_device(s.ival[var_[2]], z_.p, N_, S_, st);
      if (with_data) ints_to_device(s.ival[var_[3]], x_.p, N_, 2, st);
    }
    data_ = true;
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  ZooArgs args() const {
    ZooArgs a{};
    a.kind = kind_;
    a.N = N_;
    a.K = K_;
    a.V = V_;
    a.S = S_;
    a.A = A_.p;
    a.B = B_.p;
    a.z = z_.p;
    a.x = x_.p;
    a.f = f_.p;
    a.cnt = cnt_.p;
    a.red = red_.p;
    a.seed = seed_;
    for (int i = 0; i < 4; ++i) a.var[i] = var_[i];
    a.conc_a = conc_a_;
    a.conc_b = conc_b_;
    return a;
  }

  int kind_;
  std::int64_t N_ = 0, na_ = 0, nb_ = 0, ncnt_ = 0;
  int K_ = 0, V_ = 0, S_ = 0;
  std::uint64_t seed_ = 0;
  int var_[4] = {0, 1, 2, 3};
  double conc_a_ = 0.5, conc_b_ = 0.5;
  bool data_ = false;
  DevBuf<double> A_, B_, red_, ljpart_;
  DevBuf<int> z_, x_, f_, cnt_, zold_, maps_, starts_;
  std::int64_t hmm_chunks_ = 0, hmm_chunk_ = 0;
  DevBuf<std::int64_t> stage_;
};

}  // namespace

std::unique_ptr<Model> make_zoo(const bnmc_gpu_desc& d, const Comm& c, Outputs o) {
  return std::make_unique<Zoo>(d, c, o);
}

}  // namespace bnmc_gpu
