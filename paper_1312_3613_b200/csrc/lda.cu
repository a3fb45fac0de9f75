// csrc/lda.cu -- LDA uncollapsed Gibbs sweep on sm_100a (proj/models/lda.bn).
//
// One reference sweep (Engine::sweep, proj/src/sampler.cpp:390-405; plan order
// phi, theta, z per tests/golden/describe_lda.txt) becomes, per GPU:
//
//   [allreduce nkw]      NCCL int32 sum of the topic-word counts (world > 1 only)
//   phi_gamma_kernel     phi block draw: per cell Gamma(beta + n[k,v]) from stream
//                        keyed(seed,4,var_phi,iter).derive(k,v) (batch.cpp:38-41);
//                        consumes the counts and zeroes them for this sweep's z-step
//   colsum_kernel        row sums of the gamma matrix (fixed-order, deterministic)
//   phi_norm_kernel      phi = g / sum (batch.cpp:58-61) + Dirichlet log-pdf pieces
//   phi_terms_kernel     per-topic Dirichlet log-pdf (dist.cpp:115-130)
//   doc_kernel           per document: theta-block counts + Dirichlet draw
//                        (sampler.cpp:61-181), then the z block for every token
//                        (sampler.cpp:222-265, draw_from_log_weights dist.cpp:202-215),
//                        next sweep's topic-word counts (atomics) and the document's
//                        log-joint pieces
//   reduce_docs_kernel   fixed-order sum of the per-document log-joint pieces
//   [allreduce 3 doubles]
//   finalize_kernel      log-joint = ((F_phi + F_theta) + F_z) + F_w (eval.cpp:393-422)
//
// Device layout (HBM): w, z int32 [N_local]; phiT fp64 [V][Kp] (word-major, so
// the K weights of a token are one contiguous row; Kp = K rounded up to the
// z-step tile, padding is zero); nkw int32 [V][Kp]; theta fp64 [M_local][K]
// (the reference's row-major layout); per-sweep scratch is O(K * blocks + M).
#include <cmath>
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "dist.cuh"

namespace bnmc_gpu {
namespace {

constexpr int kDocThreads = 256;
constexpr int kPhiThreadsMax = 256;

struct LdaArgs {
  int K, Kp, V;
  std::int64_t Ml, Nl;
  const int* w;
  int* z;
  const std::int64_t* off;  // local offsets, off[0] = 0
  std::int64_t tok_base, doc_base;
  double* phiT;
  double* logphiT;  // exact mode only
  double* theta;
  int* nkw;
  double* colpart;   // [nb_phi][K]
  double* colpart2;  // [nb_phi][K][2]
  double* S;         // [K]
  double* phi_term;  // [K]
  double* doc_part;  // [Ml][3]
  double* red;       // [4]: F_theta, F_z, F_w (local) ; F_phi
  double alpha, beta;
  double phi_norm, phi_lgasum, theta_norm, theta_lgasum;
  std::uint64_t seed;
  std::uint64_t zkey_prefix;  // fold(fold(fold(1, seed), kDiscrete), var_z)
  int var_phi, var_theta, var_z;
  int rows_per_block, nb_phi;
  int count_next;  // accumulate next sweep's topic-word counts (phi block active)
};

// ---------------------------------------------------------------------------------
// phi block
// ---------------------------------------------------------------------------------
__global__ void phi_gamma_kernel(LdaArgs a, const std::int64_t* iter_p) {
  const std::int64_t iter = *iter_p;
  const std::uint64_t key = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_phi),
                                  static_cast<std::uint64_t>(iter));
  const int b = blockIdx.x;
  const int v0 = b * a.rows_per_block;
  const int v1 = min(a.V, v0 + a.rows_per_block);
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    double s = 0.0;
    for (int v = v0; v < v1; ++v) {
      const std::size_t c = static_cast<std::size_t>(v) * a.Kp + k;
      const int n = a.nkw[c];
      a.nkw[c] = 0;
      Stream r(derive(key, static_cast<std::uint64_t>(k), static_cast<std::uint64_t>(v)));
      const double g = draw_gamma(r, a.beta + static_cast<double>(n));
      a.phiT[c] = g;
      s += g;
    }
    a.colpart[static_cast<std::size_t>(b) * a.K + k] = s;
  }
}

// out[k] = sum_b part[b*stride + k*width + which], fixed order.
__global__ void colsum_kernel(const double* part, int nb, int stride, int width, int which,
                              double* out) {
  __shared__ double scratch[32];
  const int k = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    s += part[static_cast<std::size_t>(b) * stride + static_cast<std::size_t>(k) * width + which];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) out[k] = s;
}

// phi = g / S[k]; accumulates (beta-1)*log(phi) and phi per topic for the log-joint.
template <bool NORMALISE>
__global__ void phi_norm_kernel(LdaArgs a) {
  const int b = blockIdx.x;
  const int v0 = b * a.rows_per_block;
  const int v1 = min(a.V, v0 + a.rows_per_block);
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    const double S = NORMALISE ? a.S[k] : 1.0;
    double lp = 0.0, sx = 0.0;
    for (int v = v0; v < v1; ++v) {
      const std::size_t c = static_cast<std::size_t>(v) * a.Kp + k;
      double x = a.phiT[c];
      if (NORMALISE) {
        x = x / S;
        a.phiT[c] = x;
      }
      const double lx = x > 0.0 ? log(x) : -INFINITY;
      if (a.logphiT) a.logphiT[c] = lx;
      lp += (a.beta - 1.0) * lx;
      sx += x;
    }
    double* o = a.colpart2 + (static_cast<std::size_t>(b) * a.K + k) * 2;
    o[0] = lp;
    o[1] = sx;
  }
}

// Dirichlet log-pdf per topic row: lp - sum lgamma(beta) + lgamma(sum beta), -inf
// when |sum x - 1| > 1e-9 (dist.cpp:115-130).
__global__ void phi_terms_kernel(LdaArgs a) {
  __shared__ double scratch[32];
  const int k = blockIdx.x;
  double lp = 0.0, sx = 0.0;
  for (int b = threadIdx.x; b < a.nb_phi; b += blockDim.x) {
    const double* o = a.colpart2 + (static_cast<std::size_t>(b) * a.K + k) * 2;
    lp += o[0];
    sx += o[1];
  }
  lp = block_sum(lp, scratch);
  sx = block_sum(sx, scratch);
  if (threadIdx.x == 0) {
    a.phi_term[k] = (fabs(sx - 1.0) > 1e-9 || !(a.beta > 0.0)) ? -INFINITY
                                                                : lp - a.phi_norm + a.phi_lgasum;
  }
}

// ---------------------------------------------------------------------------------
// z block: grouped inverse-CDF categorical draw
// ---------------------------------------------------------------------------------
// A token's K candidate weights are handled by a group of G lanes; lane gl owns
// candidates 4*(r*G + gl) .. +3 for rounds r < R = Kp/(4G), so each round is one
// coalesced 32*G-byte segment of the token's phiT row.  Weights are either the
// product theta*phi (default) or exp(log theta + log phi - max) exactly as the
// reference (EXACT).  The inverse CDF keeps the reference's candidate order:
// cstart[r] = running sum of every earlier candidate, and the draw is the first k
// with u < acc_k, u = next_unit * total (dist.cpp:209-214).
template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) {
    return 0xffffffffu;
  } else {
    const int lane = threadIdx.x & 31;
    return ((1u << G) - 1u) << (lane & ~(G - 1));
  }
}

template <int G>
__device__ __forceinline__ double g_max(double v, unsigned m) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(m, v, o, G));
  return v;
}

template <int G>
__device__ __forceinline__ int g_max_i(int v, unsigned m) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(m, v, o, G));
  return v;
}

struct Quad {
  double v0, v1, v2, v3;
};

template <bool EXACT>
__device__ __forceinline__ Quad weights(const double* th, const double* lth, const double* row,
                                        const double* lrow, int k, double mx) {
  Quad q;
  if (!EXACT) {
    const double2 a0 = __ldg(reinterpret_cast<const double2*>(row + k));
    const double2 a1 = __ldg(reinterpret_cast<const double2*>(row + k + 2));
    const double2 t0 = *reinterpret_cast<const double2*>(th + k);
    const double2 t1 = *reinterpret_cast<const double2*>(th + k + 2);
    q.v0 = t0.x * a0.x;
    q.v1 = t0.y * a0.y;
    q.v2 = t1.x * a1.x;
    q.v3 = t1.y * a1.y;
  } else {
    const double2 a0 = __ldg(reinterpret_cast<const double2*>(lrow + k));
    const double2 a1 = __ldg(reinterpret_cast<const double2*>(lrow + k + 2));
    const double2 t0 = *reinterpret_cast<const double2*>(lth + k);
    const double2 t1 = *reinterpret_cast<const double2*>(lth + k + 2);
    q.v0 = exp((t0.x + a0.x) - mx);
    q.v1 = exp((t0.y + a0.y) - mx);
    q.v2 = exp((t1.x + a1.x) - mx);
    q.v3 = exp((t1.y + a1.y) - mx);
  }
  return q;
}

// Returns the drawn topic in every lane of the group, or -1 when every weight
// is zero/-inf (the reference throws std::domain_error).
template <int G, int RMAX, bool EXACT>
__device__ int draw_topic(const double* th, const double* lth, const double* row,
                          const double* lrow, int K, int R, double u01) {
  const unsigned m = group_mask<G>();
  const int gl = threadIdx.x & (G - 1);
  double mx = 0.0;
  if (EXACT) {
    double lm = -INFINITY;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
      if (r < R) {
        const int k = 4 * (r * G + gl);
        const double2 a0 = __ldg(reinterpret_cast<const double2*>(lrow + k));
        const double2 a1 = __ldg(reinterpret_cast<const double2*>(lrow + k + 2));
        const double2 t0 = *reinterpret_cast<const double2*>(lth + k);
        const double2 t1 = *reinterpret_cast<const double2*>(lth + k + 2);
        lm = fmax(lm, fmax(fmax(t0.x + a0.x, t0.y + a0.y), fmax(t1.x + a1.x, t1.y + a1.y)));
      }
    }
    mx = g_max<G>(lm, m);
    if (!isfinite(mx)) return -1;
  }
  double cstart[RMAX];
  double B = 0.0;
#pragma unroll
  for (int r = 0; r < RMAX; ++r) {
    cstart[r] = 0.0;
    if (r < R) {
      const Quad q = weights<EXACT>(th, lth, row, lrow, 4 * (r * G + gl), mx);
      const double s = ((q.v0 + q.v1) + q.v2) + q.v3;
      double inc = s;
#pragma unroll
      for (int d = 1; d < G; d <<= 1) {
        const double t = __shfl_up_sync(m, inc, d, G);
        if (gl >= d) inc += t;
      }
      double ex = __shfl_up_sync(m, inc, 1, G);
      if (gl == 0) ex = 0.0;
      const double tot = __shfl_sync(m, inc, G - 1, G);
      cstart[r] = B + ex;
      B = B + tot;
    }
  }
  const double total = B;
  if (!(total > 0.0) || !isfinite(total)) return -1;
  const double u = u01 * total;
  // Last chunk (k-order) whose running start is <= u.
  int q_l = -1;
#pragma unroll
  for (int r = 0; r < RMAX; ++r)
    if (r < R && cstart[r] <= u) q_l = r * G + gl;
  const int qs = g_max_i<G>(q_l, m);
  int kk = 0;
  if (qs >= 0 && (qs & (G - 1)) == gl) {
    const int rs = qs / G;
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < RMAX; ++r)
      if (r == rs) acc = cstart[r];
    const int k0 = 4 * qs;
    const Quad q = weights<EXACT>(th, lth, row, lrow, k0, mx);
    kk = k0 + 3;
    acc += q.v0;
    if (u < acc) {
      kk = k0;
    } else {
      acc += q.v1;
      if (u < acc) {
        kk = k0 + 1;
      } else {
        acc += q.v2;
        if (u < acc) kk = k0 + 2;
      }
    }
    kk = min(kk, K - 1);  // past-the-end fallback (dist.cpp:214)
  }
  return __shfl_sync(m, kk, qs < 0 ? 0 : (qs & (G - 1)), G);
}

// ---------------------------------------------------------------------------------
// theta block + z block, one CTA per document
// ---------------------------------------------------------------------------------
template <int G, int RMAX, bool EXACT>
__global__ void __launch_bounds__(kDocThreads) doc_kernel(LdaArgs a, const std::int64_t* iter_p,
                                                          int* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* th = reinterpret_cast<double*>(smem_raw);  // [Kp]
  double* lth = th + a.Kp;                            // [Kp]
  int* cnt = reinterpret_cast<int*>(lth + a.Kp);      // [Kp]
  __shared__ double scratch[32];

  const std::int64_t iter = *iter_p;
  const std::uint64_t tkey = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_theta),
                                   static_cast<std::uint64_t>(iter));
  const int R = a.Kp / (4 * G);
  const int gid = threadIdx.x / G;
  constexpr int kGroups = kDocThreads / G;

  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const std::int64_t t0 = a.off[m], t1 = a.off[m + 1];
    for (int k = threadIdx.x; k < a.Kp; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    // theta-block counting phase: c[val] += [z[i,j] == val] (sampler.cpp:61-136).
    for (std::int64_t t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
      const int k = a.z[t];
      if (k < 0 || k >= a.K)
        atomicOr(err, kErrBin);
      else
        atomicAdd(&cnt[k], 1);
    }
    __syncthreads();
    // Dirichlet(alpha + c) draw, cell stream keyed(seed,4,var_theta,iter).derive(m,k).
    const std::uint64_t mg = static_cast<std::uint64_t>(a.doc_base + m);
    double part = 0.0;
    for (int k = threadIdx.x; k < a.Kp; k += blockDim.x) {
      double g = 0.0;
      if (k < a.K) {
        Stream r(derive(tkey, mg, static_cast<std::uint64_t>(k)));
        g = draw_gamma(r, a.alpha + static_cast<double>(cnt[k]));
      }
      th[k] = g;
      part += g;
    }
    const double S = block_sum(part, scratch);
    double lp = 0.0, sx = 0.0;
    for (int k = threadIdx.x; k < a.Kp; k += blockDim.x) {
      if (k < a.K) {
        const double x = th[k] / S;
        const double lx = x > 0.0 ? log(x) : -INFINITY;
        th[k] = x;
        lth[k] = lx;
        a.theta[m * a.K + k] = x;
        lp += (a.alpha - 1.0) * lx;
        sx += x;
      } else {
        th[k] = 0.0;
        lth[k] = -INFINITY;
      }
    }
    lp = block_sum(lp, scratch);
    sx = block_sum(sx, scratch);
    const double theta_term =
        fabs(sx - 1.0) > 1e-9 ? -INFINITY : lp - a.theta_norm + a.theta_lgasum;
    __syncthreads();

    // z block: every token of the document, G lanes per token.
    double zs = 0.0, ws = 0.0;
    for (std::int64_t base = t0; base < t1; base += kGroups) {
      const std::int64_t t = base + gid;
      const bool valid = t < t1;
      const int wv = valid ? a.w[t] : 0;
      const double* row = a.phiT + static_cast<std::size_t>(wv) * a.Kp;
      const double* lrow = EXACT ? a.logphiT + static_cast<std::size_t>(wv) * a.Kp : nullptr;
      // keyed(seed, 3, var_z, t, iter) with the first three folds hoisted.
      Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + t)),
                      static_cast<std::uint64_t>(iter)));
      const double u01 = rng.next_unit();
      int k = draw_topic<G, RMAX, EXACT>(th, lth, row, lrow, a.K, R, u01);
      if (!EXACT && k < 0) {
        // Product weights underflowed: redo this token in log space (needs no table:
        // log phi is taken on the fly from the row).
        k = -2;
      }
      if (k == -2) {
        // log-space fallback without a log table: the group recomputes weights.
        const unsigned msk = group_mask<G>();
        const int gl = threadIdx.x & (G - 1);
        double lm = -INFINITY;
        for (int kk = gl; kk < a.K; kk += G) lm = fmax(lm, lth[kk] + (row[kk] > 0.0 ? log(row[kk]) : -INFINITY));
        lm = g_max<G>(lm, msk);
        int pick = -1;
        if (isfinite(lm)) {
          // sequential scan by lane 0, reference order and arithmetic
          if (gl == 0) {
            double total = 0.0;
            for (int kk = 0; kk < a.K; ++kk)
              total += exp((lth[kk] + (row[kk] > 0.0 ? log(row[kk]) : -INFINITY)) - lm);
            const double u = u01 * total;
            double acc = 0.0;
            pick = a.K - 1;
            for (int kk = 0; kk < a.K; ++kk) {
              acc += exp((lth[kk] + (row[kk] > 0.0 ? log(row[kk]) : -INFINITY)) - lm);
              if (u < acc) {
                pick = kk;
                break;
              }
            }
          }
          pick = __shfl_sync(msk, pick, 0, G);
        }
        k = pick;
      }
      if (valid) {
        const int gl = threadIdx.x & (G - 1);
        if (k < 0) {
          if (gl == 0) atomicOr(err, kErrDomain);
        } else if (gl == 0) {
          a.z[t] = k;
          if (a.count_next) atomicAdd(&a.nkw[static_cast<std::size_t>(wv) * a.Kp + k], 1);
          zs += lth[k];
          const double p = row[k];
          ws += p > 0.0 ? log(p) : -INFINITY;
        }
      }
    }
    zs = block_sum(zs, scratch);
    ws = block_sum(ws, scratch);
    if (threadIdx.x == 0) {
      a.doc_part[m * 3 + 0] = theta_term;
      a.doc_part[m * 3 + 1] = zs;
      a.doc_part[m * 3 + 2] = ws;
    }
    __syncthreads();
  }
}

// Log-joint pieces of the current state without sampling (Engine::eval_log_joint).
__global__ void __launch_bounds__(kDocThreads) doc_eval_kernel(LdaArgs a, int* err) {
  __shared__ double scratch[32];
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const double* th = a.theta + m * a.K;
    double lp = 0.0, sx = 0.0;
    bool bad = false;
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
      const double x = th[k];
      lp += (a.alpha - 1.0) * (x > 0.0 ? log(x) : -INFINITY);
      sx += x;
      bad |= !(x > 0.0);
    }
    lp = block_sum(lp, scratch);
    sx = block_sum(sx, scratch);
    const double theta_term = fabs(sx - 1.0) > 1e-9 ? -INFINITY : lp - a.theta_norm + a.theta_lgasum;
    double zs = 0.0, ws = 0.0;
    for (std::int64_t t = a.off[m] + threadIdx.x; t < a.off[m + 1]; t += blockDim.x) {
      const int k = a.z[t];
      if (k < 0 || k >= a.K) {
        zs += -INFINITY;
        ws += -INFINITY;
        continue;
      }
      const double pt = th[k];
      zs += pt > 0.0 ? log(pt) : -INFINITY;
      const double pp = a.phiT[static_cast<std::size_t>(a.w[t]) * a.Kp + k];
      ws += pp > 0.0 ? log(pp) : -INFINITY;
    }
    zs = block_sum(zs, scratch);
    ws = block_sum(ws, scratch);
    if (threadIdx.x == 0) {
      a.doc_part[m * 3 + 0] = bad ? -INFINITY : theta_term;
      a.doc_part[m * 3 + 1] = zs;
      a.doc_part[m * 3 + 2] = ws;
    }
    __syncthreads();
  }
}

// red[0..2] = sum over local documents of the three pieces (fixed order).
__global__ void reduce_docs_kernel(LdaArgs a) {
  __shared__ double scratch[32];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (std::int64_t m = threadIdx.x; m < a.Ml; m += blockDim.x) {
    s0 += a.doc_part[m * 3 + 0];
    s1 += a.doc_part[m * 3 + 1];
    s2 += a.doc_part[m * 3 + 2];
  }
  s0 = block_sum(s0, scratch);
  s1 = block_sum(s1, scratch);
  s2 = block_sum(s2, scratch);
  if (threadIdx.x == 0) {
    a.red[0] = s0;
    a.red[1] = s1;
    a.red[2] = s2;
  }
}

__global__ void finalize_kernel(LdaArgs a, Outputs o, int advance) {
  __shared__ double scratch[32];
  double f = 0.0;
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) f += a.phi_term[k];
  f = block_sum(f, scratch);
  if (threadIdx.x == 0) {
    const double lj = ((f + a.red[0]) + a.red[1]) + a.red[2];
    const std::int64_t it = *o.iter;
    o.lj[it & (kRing - 1)] = lj;
    o.acc[it & (kRing - 1)] = 0;
    if (advance) *o.iter = it + 1;
  }
}

// ---------------------------------------------------------------------------------
// counts, conversions, prior_init, generator
// ---------------------------------------------------------------------------------
__global__ void count_kernel(LdaArgs a, int* err) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t t = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; t < a.Nl;
       t += stride) {
    const int k = a.z[t];
    const int v = a.w[t];
    if (k < 0 || k >= a.K) {
      atomicOr(err, kErrBin);
      continue;
    }
    if (v >= 0 && v < a.V) atomicAdd(&a.nkw[static_cast<std::size_t>(v) * a.Kp + k], 1);
  }
}

__global__ void doc_counts_kernel(LdaArgs a, int* nmk) {
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x)
    for (std::int64_t t = a.off[m] + threadIdx.x; t < a.off[m + 1]; t += blockDim.x) {
      const int k = a.z[t];
      if (k >= 0 && k < a.K) atomicAdd(&nmk[m * a.K + k], 1);
    }
}

__global__ void i64_to_i32_kernel(const std::int64_t* in, int* out, std::int64_t n, std::int64_t lo,
                                  std::int64_t hi, int* err) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    const std::int64_t v = in[i];
    if (v < lo || v >= hi) atomicOr(err, kErrBin);
    out[i] = static_cast<int>(v);
  }
}

__global__ void i32_to_i64_kernel(const int* in, std::int64_t* out, std::int64_t n) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    out[i] = in[i];
}

// phiT [V][Kp] <-> phi [K][V] (reference layout), tiled through shared memory.
__global__ void transpose_kernel(const double* in, double* out, int rows, int cols, int ld_in,
                                 int ld_out) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[static_cast<std::size_t>(r) * ld_in + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[static_cast<std::size_t>(c) * ld_out + r] = tile[threadIdx.x][i];
  }
}

// prior_init (sampler.cpp:542-555): Dirichlet rows drawn sequentially from ONE
// stream keyed(seed,5,var,row) (draw_dirichlet, dist.cpp:193-200), thread per row.
__global__ void prior_rows_kernel(double* out, std::int64_t rows, int cols, std::int64_t ld_row,
                                  std::int64_t ld_col, double conc, std::uint64_t seed, int var,
                                  std::int64_t row_base) {
  const std::int64_t r = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  Stream s(keyed(seed, kInit, static_cast<std::uint64_t>(var),
                 static_cast<std::uint64_t>(row_base + r)));
  double sum = 0.0;
  for (int c = 0; c < cols; ++c) {
    const double g = draw_gamma(s, conc);
    out[r * ld_row + c * ld_col] = g;
    sum += g;
  }
  for (int c = 0; c < cols; ++c) out[r * ld_row + c * ld_col] /= sum;
}

// z ~ Categorical(theta[d]) by linear scan (draw_categorical, dist.cpp:183-191).
__global__ void prior_z_kernel(LdaArgs a, std::uint64_t seed) {
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const double* th = a.theta + m * a.K;
    for (std::int64_t t = a.off[m] + threadIdx.x; t < a.off[m + 1]; t += blockDim.x) {
      Stream s(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_z),
                     static_cast<std::uint64_t>(a.tok_base + t)));
      const double u = s.next_unit();
      double acc = 0.0;
      int pick = a.K - 1;
      for (int k = 0; k < a.K; ++k) {
        acc += th[k];
        if (u < acc) {
          pick = k;
          break;
        }
      }
      a.z[t] = pick;
    }
  }
}

// Device corpus generator following gen_lda's process (gen.cpp:21-60): true phi
// rows ~ Dir(phi_conc), theta_d ~ Dir(theta_conc), z ~ Cat(theta_d), w ~ Cat(phi_z).
// Word draws use a per-topic cumulative table + binary search (not the reference's
// O(V) scan) and counter streams per token (not one serial stream).
__global__ void gen_tokens_kernel(LdaArgs a, const double* cum_phi /*[K][V]*/, const double* theta_true,
                                  std::uint64_t seed) {
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const double* th = theta_true + m * a.K;
    for (std::int64_t t = a.off[m] + threadIdx.x; t < a.off[m + 1]; t += blockDim.x) {
      Stream s(keyed(seed, 0xDA7A, 1, static_cast<std::uint64_t>(a.tok_base + t)));
      const double u = s.next_unit();
      double acc = 0.0;
      int k = a.K - 1;
      for (int j = 0; j < a.K; ++j) {
        acc += th[j];
        if (u < acc) {
          k = j;
          break;
        }
      }
      const double* cp = cum_phi + static_cast<std::size_t>(k) * a.V;
      const double uw = s.next_unit() * cp[a.V - 1];
      int lo = 0, hi = a.V - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (uw < cp[mid])
          hi = mid;
        else
          lo = mid + 1;
      }
      const_cast<int*>(a.w)[t] = lo;
    }
  }
}

__global__ void row_cumsum_kernel(double* x, std::int64_t rows, int cols) {
  const std::int64_t r = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  double acc = 0.0;
  for (int c = 0; c < cols; ++c) {
    acc += x[r * cols + c];
    x[r * cols + c] = acc;
  }
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
double seq_sum_const(double x, std::int64_t n) {  // sum of n copies, left to right
  double s = 0.0;
  for (std::int64_t i = 0; i < n; ++i) s += x;
  return s;
}

class Lda final : public Model {
 public:
  Lda(const bnmc_gpu_desc& d, const Comm& c, Outputs o) : comm_(c) {
    out = o;
    require(d.K >= 1 && d.V >= 1 && d.M >= 0 && d.N >= 0, BNMC_GPU_ERR_ARG, "LDA needs K, V >= 1");
    require(d.K <= 2048, BNMC_GPU_ERR_ARG, "LDA z-step supports K <= 2048");
    require(d.V < (1ll << 31) && d.N < (1ll << 40), BNMC_GPU_ERR_ARG, "LDA sizes out of range");
    require(d.doc_offsets != nullptr, BNMC_GPU_ERR_ARG, "LDA needs doc_offsets");
    K_ = static_cast<int>(d.K);
    V_ = static_cast<int>(d.V);
    M_ = d.M;
    N_ = d.N;
    require(d.doc_offsets[0] == 0 && d.doc_offsets[M_] == N_, BNMC_GPU_ERR_RUNTIME,
            "doc_offsets must run from 0 to N");
    exact_ = (d.flags & BNMC_GPU_EXACT_WEIGHTS) != 0;
    observe_phi_ = (d.flags & BNMC_GPU_OBSERVE_PHI) != 0;
    G_ = K_ <= 256 ? 4 : (K_ <= 512 ? 8 : 32);
    Kp_ = static_cast<int>((d.K + 4 * G_ - 1) / (4 * G_) * (4 * G_));
    partition_docs(d.doc_offsets, M_, c.world, c.rank, &d0_, &d1_);
    Ml_ = d1_ - d0_;
    tok0_ = d.doc_offsets[d0_];
    Nl_ = d.doc_offsets[d1_] - tok0_;
    off_host_.resize(static_cast<std::size_t>(Ml_) + 1);
    for (std::int64_t m = 0; m <= Ml_; ++m) off_host_[m] = d.doc_offsets[d0_ + m] - tok0_;

    alpha_ = d.hyper[0] > 0 ? d.hyper[0] : 0.1;
    beta_ = d.hyper[1] > 0 ? d.hyper[1] : 0.1;
    seed_ = d.seed;
    var_phi_ = d.var_ids[0];
    var_theta_ = d.var_ids[1];
    var_z_ = d.var_ids[2];
    var_w_ = d.var_ids[3];

    const int pt = std::min(kPhiThreadsMax, ((K_ + 31) / 32) * 32);
    phi_threads_ = pt;
    const std::int64_t target_blocks = 148 * 8;
    rows_per_block_ = static_cast<int>(std::max<std::int64_t>(1, (V_ + target_blocks - 1) / target_blocks));
    nb_phi_ = (V_ + rows_per_block_ - 1) / rows_per_block_;

    w_.alloc(std::max<std::int64_t>(Nl_, 1));
    z_.alloc(std::max<std::int64_t>(Nl_, 1));
    off_.alloc(Ml_ + 1);
    phiT_.alloc(static_cast<std::size_t>(V_) * Kp_);
    if (exact_) logphiT_.alloc(static_cast<std::size_t>(V_) * Kp_);
    theta_.alloc(std::max<std::int64_t>(Ml_ * K_, 1));
    nkw_.alloc(static_cast<std::size_t>(V_) * Kp_);
    colpart_.alloc(static_cast<std::size_t>(nb_phi_) * K_);
    colpart2_.alloc(static_cast<std::size_t>(nb_phi_) * K_ * 2);
    S_.alloc(K_);
    phi_term_.alloc(K_);
    doc_part_.alloc(std::max<std::int64_t>(Ml_ * 3, 3));
    red_.alloc(4);
    cudaStream_t s0 = nullptr;
    BNMC_CUDA(cudaMemcpy(off_.p, off_host_.data(), sizeof(std::int64_t) * (Ml_ + 1), cudaMemcpyHostToDevice));
    phiT_.zero(s0);
    nkw_.zero(s0);
    w_.zero(s0);
    z_.zero(s0);
    theta_.zero(s0);
    doc_part_.zero(s0);
    red_.zero(s0);
    phi_term_.zero(s0);
    if (exact_) {
      std::vector<double> ninf(static_cast<std::size_t>(V_) * Kp_, -INFINITY);
      BNMC_CUDA(cudaMemcpy(logphiT_.p, ninf.data(), logphiT_.bytes(), cudaMemcpyHostToDevice));
    }
    BNMC_CUDA(cudaDeviceSynchronize());

    // Dirichlet normalisers, summed left to right as the reference does (dist.cpp:121-126).
    phi_norm_ = seq_sum_const(std::lgamma(beta_), V_);
    phi_lgasum_ = std::lgamma(seq_sum_const(beta_, V_));
    theta_norm_ = seq_sum_const(std::lgamma(alpha_), K_);
    theta_lgasum_ = std::lgamma(seq_sum_const(alpha_, K_));

    configure_doc_kernel();
  }

  void upload(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, true); }

  void upload_state(const bnmc_gpu_store& s, cudaStream_t st) override {
    upload_impl(s, st, !data_on_device_);
  }

  void upload_impl(const bnmc_gpu_store& s, cudaStream_t st, bool with_data) {
    require(s.n_vars > std::max(std::max(var_phi_, var_theta_), std::max(var_z_, var_w_)),
            BNMC_GPU_ERR_RUNTIME, "store has the wrong number of variables");
    check_len(s, var_phi_, static_cast<std::int64_t>(K_) * V_, "phi");
    check_len(s, var_theta_, M_ * K_, "theta");
    check_len(s, var_z_, N_, "z");
    check_len(s, var_w_, N_, "w");
    require(s.ival[var_w_] && s.ival[var_z_] && s.real[var_phi_] && s.real[var_theta_],
            BNMC_GPU_ERR_RUNTIME, "store arrays missing");
    // w (observed data) and z: int64 -> int32 on the device, with range checks.
    if (stage64_.n < static_cast<std::size_t>(std::max<std::int64_t>(Nl_, 1))) stage64_.alloc(std::max<std::int64_t>(Nl_, 1));
    if (Nl_ > 0) {
      if (with_data) {
        BNMC_CUDA(cudaMemcpyAsync(stage64_.p, s.ival[var_w_] + tok0_, sizeof(std::int64_t) * Nl_,
                                  cudaMemcpyHostToDevice, st));
        i64_to_i32_kernel<<<blocks_for(Nl_, 256), 256, 0, st>>>(stage64_.p, w_.p, Nl_, 0, V_, out.err);
      }
      BNMC_CUDA(cudaMemcpyAsync(stage64_.p, s.ival[var_z_] + tok0_, sizeof(std::int64_t) * Nl_,
                                cudaMemcpyHostToDevice, st));
      i64_to_i32_kernel<<<blocks_for(Nl_, 256), 256, 0, st>>>(stage64_.p, z_.p, Nl_, 0, K_, out.err);
    }
    // theta rows of this shard, phi (K x V) -> phiT (V x Kp).
    if (Ml_ > 0)
      BNMC_CUDA(cudaMemcpyAsync(theta_.p, s.real[var_theta_] + d0_ * K_, sizeof(double) * Ml_ * K_,
                                cudaMemcpyHostToDevice, st));
    if (stage_phi_.n == 0) stage_phi_.alloc(static_cast<std::size_t>(K_) * V_);
    BNMC_CUDA(cudaMemcpyAsync(stage_phi_.p, s.real[var_phi_], stage_phi_.bytes(), cudaMemcpyHostToDevice, st));
    transpose_kernel<<<dim3((V_ + 31) / 32, (K_ + 31) / 32), dim3(32, 8), 0, st>>>(stage_phi_.p, phiT_.p, K_, V_, V_, Kp_);
    BNMC_CUDA(cudaGetLastError());
    data_on_device_ = true;
    after_state_change(st);
  }

  void download(const bnmc_gpu_store& s, cudaStream_t st) override {
    const char* obs = s.observed;
    if (!(obs && obs[var_z_]) && s.ival[var_z_] && Nl_ > 0) {
      if (stage64_.n < static_cast<std::size_t>(Nl_)) stage64_.alloc(Nl_);
      i32_to_i64_kernel<<<blocks_for(Nl_, 256), 256, 0, st>>>(z_.p, stage64_.p, Nl_);
      BNMC_CUDA(cudaMemcpyAsync(s.ival[var_z_] + tok0_, stage64_.p, sizeof(std::int64_t) * Nl_,
                                cudaMemcpyDeviceToHost, st));
    }
    if (!(obs && obs[var_theta_]) && s.real[var_theta_] && Ml_ > 0)
      BNMC_CUDA(cudaMemcpyAsync(s.real[var_theta_] + d0_ * K_, theta_.p, sizeof(double) * Ml_ * K_,
                                cudaMemcpyDeviceToHost, st));
    if (!(obs && obs[var_phi_]) && !observe_phi_ && s.real[var_phi_]) {
      if (stage_phi_.n == 0) stage_phi_.alloc(static_cast<std::size_t>(K_) * V_);
      transpose_kernel<<<dim3((K_ + 31) / 32, (V_ + 31) / 32), dim3(32, 8), 0, st>>>(phiT_.p, stage_phi_.p, V_, K_, Kp_, V_);
      BNMC_CUDA(cudaMemcpyAsync(s.real[var_phi_], stage_phi_.p, stage_phi_.bytes(), cudaMemcpyDeviceToHost, st));
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  void enqueue_sweep(cudaStream_t st) override {
    LdaArgs a = args();
    mark(st, "begin");
    if (!observe_phi_) {
      if (comm_.world > 1) {
        BNMC_NCCL(ncclAllReduce(nkw_.p, nkw_.p, nkw_.n, ncclInt32, ncclSum, comm_.comm, st));
        mark(st, "allreduce_counts");
      }
      phi_gamma_kernel<<<nb_phi_, phi_threads_, 0, st>>>(a, out.iter);
      mark(st, "phi_gamma");
      colsum_kernel<<<K_, 128, 0, st>>>(colpart_.p, nb_phi_, K_, 1, 0, S_.p);
      mark(st, "phi_colsum");
      phi_norm_kernel<true><<<nb_phi_, phi_threads_, 0, st>>>(a);
      mark(st, "phi_norm");
      phi_terms_kernel<<<K_, 128, 0, st>>>(a);
      mark(st, "phi_terms");
    }
    launch_doc(a, st);
    mark(st, "doc_theta_z");
    reduce_docs_kernel<<<1, 1024, 0, st>>>(a);
    mark(st, "reduce_docs");
    if (comm_.world > 1) {
      BNMC_NCCL(ncclAllReduce(red_.p, red_.p, 3, ncclFloat64, ncclSum, comm_.comm, st));
      mark(st, "allreduce_lj");
    }
    finalize_kernel<<<1, 256, 0, st>>>(a, out, 1);
    mark(st, "finalize");
    BNMC_CUDA(cudaGetLastError());
  }

  void enqueue_log_joint(cudaStream_t st) override {
    LdaArgs a = args();
    phi_norm_kernel<false><<<nb_phi_, phi_threads_, 0, st>>>(a);
    phi_terms_kernel<<<K_, 128, 0, st>>>(a);
    doc_eval_kernel<<<grid_docs(), kDocThreads, 0, st>>>(a, out.err);
    reduce_docs_kernel<<<1, 1024, 0, st>>>(a);
    if (comm_.world > 1)
      BNMC_NCCL(ncclAllReduce(red_.p, red_.p, 3, ncclFloat64, ncclSum, comm_.comm, st));
    finalize_kernel<<<1, 256, 0, st>>>(a, out, 0);
    BNMC_CUDA(cudaGetLastError());
  }

  void prior_init(std::uint64_t seed, cudaStream_t st) override {
    LdaArgs a = args();
    if (!observe_phi_)
      prior_rows_kernel<<<blocks_for(K_, 32), 32, 0, st>>>(phiT_.p, K_, V_, 1, Kp_, beta_, seed, var_phi_, 0);
    if (Ml_ > 0) {
      prior_rows_kernel<<<blocks_for(Ml_, 64), 64, 0, st>>>(theta_.p, Ml_, K_, K_, 1, alpha_, seed,
                                                           var_theta_, d0_);
      prior_z_kernel<<<grid_docs(), 256, 0, st>>>(a, seed);
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
    after_state_change(st);
  }

  void lda_counts(std::int32_t* nkw_host, std::int32_t* nmk_host, cudaStream_t st) override {
    if (nkw_host) {
      // Topic-word counts of the current z, recomputed (then summed over ranks).
      DevBuf<int> tmp;
      tmp.alloc(static_cast<std::size_t>(V_) * Kp_);
      tmp.zero(st);
      LdaArgs a = args();
      a.nkw = tmp.p;
      if (Nl_ > 0) count_kernel<<<std::min<unsigned>(blocks_for(Nl_, 256), 148 * 16), 256, 0, st>>>(a, out.err);
      if (comm_.world > 1)
        BNMC_NCCL(ncclAllReduce(tmp.p, tmp.p, tmp.n, ncclInt32, ncclSum, comm_.comm, st));
      std::vector<int> h(tmp.n);
      BNMC_CUDA(cudaMemcpyAsync(h.data(), tmp.p, tmp.bytes(), cudaMemcpyDeviceToHost, st));
      BNMC_CUDA(cudaStreamSynchronize(st));
      for (int v = 0; v < V_; ++v)
        for (int k = 0; k < K_; ++k)
          nkw_host[static_cast<std::size_t>(k) * V_ + v] = h[static_cast<std::size_t>(v) * Kp_ + k];
    }
    if (nmk_host && Ml_ > 0) {
      DevBuf<int> nmk;
      nmk.alloc(Ml_ * K_);
      nmk.zero(st);
      LdaArgs a = args();
      doc_counts_kernel<<<grid_docs(), 256, 0, st>>>(a, nmk.p);
      BNMC_CUDA(cudaMemcpyAsync(nmk_host, nmk.p, nmk.bytes(), cudaMemcpyDeviceToHost, st));
      BNMC_CUDA(cudaStreamSynchronize(st));
    }
  }

  void lda_generate(std::uint64_t seed, double phi_conc, double theta_conc, cudaStream_t st) override {
    // True phi (K x V, one stream per topic row as prior_init does) -> cumulative rows.
    DevBuf<double> cum, th;
    cum.alloc(static_cast<std::size_t>(K_) * V_);
    th.alloc(std::max<std::int64_t>(Ml_ * K_, 1));
    prior_rows_kernel<<<blocks_for(K_, 32), 32, 0, st>>>(cum.p, K_, V_, V_, 1, phi_conc, seed ^ 0xDA7Aull, 0, 0);
    row_cumsum_kernel<<<blocks_for(K_, 32), 32, 0, st>>>(cum.p, K_, V_);
    if (Ml_ > 0) {
      prior_rows_kernel<<<blocks_for(Ml_, 64), 64, 0, st>>>(th.p, Ml_, K_, K_, 1, theta_conc,
                                                           seed ^ 0xDA7Aull, 1, d0_);
      LdaArgs a = args();
      gen_tokens_kernel<<<grid_docs(), 256, 0, st>>>(a, cum.p, th.p, seed);
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
    prior_init(seed, st);
  }

 private:
  static void check_len(const bnmc_gpu_store& s, int var, std::int64_t want, const char* name) {
    require(s.len && s.len[var] == want, BNMC_GPU_ERR_RUNTIME,
            std::string("variable '") + name + "' has flat length " +
                std::to_string(s.len ? s.len[var] : -1) + ", expected " + std::to_string(want));
  }

  // After an upload / prior_init: counts of the current z for the next phi block.
  void after_state_change(cudaStream_t st) {
    LdaArgs a = args();
    nkw_.zero(st);
    if (Nl_ > 0) count_kernel<<<std::min<unsigned>(blocks_for(Nl_, 256), 148 * 16), 256, 0, st>>>(a, out.err);
    // phi terms (and the exact-mode log table) of the uploaded phi: used as-is by
    // clamped-phi runs, recomputed by the phi block otherwise.
    phi_norm_kernel<false><<<nb_phi_, phi_threads_, 0, st>>>(a);
    phi_terms_kernel<<<K_, 128, 0, st>>>(a);
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  unsigned grid_docs() const { return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>(Ml_, 1 << 20))); }

  std::size_t doc_smem() const { return sizeof(double) * 2 * Kp_ + sizeof(int) * Kp_; }

  template <int G, int RMAX, bool E>
  void set_attr() {
    BNMC_CUDA(cudaFuncSetAttribute(doc_kernel<G, RMAX, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(doc_smem())));
  }

  void configure_doc_kernel() {
    if (doc_smem() <= 48 * 1024) return;
    if (G_ == 4) exact_ ? set_attr<4, 16, true>() : set_attr<4, 16, false>();
    if (G_ == 8) exact_ ? set_attr<8, 16, true>() : set_attr<8, 16, false>();
    if (G_ == 32) exact_ ? set_attr<32, 16, true>() : set_attr<32, 16, false>();
  }

  void launch_doc(const LdaArgs& a, cudaStream_t st) {
    if (Ml_ == 0) return;
    const unsigned g = grid_docs();
    const std::size_t sm = doc_smem();
#define BNMC_DOC(GG, E) doc_kernel<GG, 16, E><<<g, kDocThreads, sm, st>>>(a, out.iter, out.err)
    if (G_ == 4) {
      if (exact_) BNMC_DOC(4, true); else BNMC_DOC(4, false);
    } else if (G_ == 8) {
      if (exact_) BNMC_DOC(8, true); else BNMC_DOC(8, false);
    } else {
      if (exact_) BNMC_DOC(32, true); else BNMC_DOC(32, false);
    }
#undef BNMC_DOC
  }

  LdaArgs args() const {
    LdaArgs a{};
    a.K = K_;
    a.Kp = Kp_;
    a.V = V_;
    a.Ml = Ml_;
    a.Nl = Nl_;
    a.w = w_.p;
    a.z = z_.p;
    a.off = off_.p;
    a.tok_base = tok0_;
    a.doc_base = d0_;
    a.phiT = phiT_.p;
    a.logphiT = exact_ ? logphiT_.p : nullptr;
    a.theta = theta_.p;
    a.nkw = nkw_.p;
    a.colpart = colpart_.p;
    a.colpart2 = colpart2_.p;
    a.S = S_.p;
    a.phi_term = phi_term_.p;
    a.doc_part = doc_part_.p;
    a.red = red_.p;
    a.alpha = alpha_;
    a.beta = beta_;
    a.phi_norm = phi_norm_;
    a.phi_lgasum = phi_lgasum_;
    a.theta_norm = theta_norm_;
    a.theta_lgasum = theta_lgasum_;
    a.seed = seed_;
    a.zkey_prefix = fold(fold(fold(1, seed_), kDiscrete), static_cast<std::uint64_t>(var_z_));
    a.var_phi = var_phi_;
    a.var_theta = var_theta_;
    a.var_z = var_z_;
    a.rows_per_block = rows_per_block_;
    a.nb_phi = nb_phi_;
    a.count_next = observe_phi_ ? 0 : 1;
    return a;
  }

  Comm comm_;
  int K_ = 0, Kp_ = 0, V_ = 0, G_ = 4;
  std::int64_t M_ = 0, N_ = 0, d0_ = 0, d1_ = 0, Ml_ = 0, Nl_ = 0, tok0_ = 0;
  std::vector<std::int64_t> off_host_;
  bool exact_ = false, observe_phi_ = false;
  double alpha_ = 0.1, beta_ = 0.1, phi_norm_ = 0, phi_lgasum_ = 0, theta_norm_ = 0, theta_lgasum_ = 0;
  std::uint64_t seed_ = 0;
  int var_phi_ = 0, var_theta_ = 1, var_z_ = 2, var_w_ = 3;
  int phi_threads_ = 128, rows_per_block_ = 1, nb_phi_ = 1;
  bool data_on_device_ = false;
  DevBuf<std::int64_t> stage64_;  // int64 <-> int32 staging for z / w
  DevBuf<double> stage_phi_;      // K x V staging for the phi transpose
  DevBuf<int> w_, z_, nkw_;
  DevBuf<std::int64_t> off_;
  DevBuf<double> phiT_, logphiT_, theta_, colpart_, colpart2_, S_, phi_term_, doc_part_, red_;
};

}  // namespace

std::unique_ptr<Model> make_lda(const bnmc_gpu_desc& d, const Comm& c, Outputs o) {
  return std::make_unique<Lda>(d, c, o);
}

}  // namespace bnmc_gpu
