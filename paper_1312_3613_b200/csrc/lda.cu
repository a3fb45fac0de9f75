// csrc/lda.cu -- LDA uncollapsed Gibbs sweep on sm_100a (proj/models/lda.bn).
//
// One reference sweep (Engine::sweep, proj/src/sampler.cpp:390-405; plan order
// phi, theta, z per tests/golden/describe_lda.txt) becomes, per GPU, one CUDA graph:
//
//   [reduce-scatter nkw] the topic-word counts by vocabulary slices (world > 1 only)
//   phi_pool_kernel      phi AND theta blocks: every cell's Gamma(prior + count) draw
//                        (batch.cpp:38-41 streams, dist.cpp:136-155 Marsaglia-Tsang) by
//                        a persistent warp pool; consumes the counts (zeroes them for
//                        this sweep's z-step); sharded: this rank's phi rows, then
//                        [all-gather] of the drawn rows
//   phi_colsum2_kernel   phi column sums S[k] and the phi factor of the log-joint;
//                        theta rows: normalise, theta factor (extra y-blocks)
//   zscreen_t_kernel     z block (sampler.cpp:222-265, draw_from_log_weights
//   / zscreen_kernel     dist.cpp:202-215): fp32 screen of the product-form draw, new z,
//                        the NEXT sweep's counts (integer atomics); ambiguous tokens
//                        queued for; K > 128 with > 32 MB of rows: the word-major
//                        order (th32_kernel + zscreen_kernel<.., WM>, build_word_major)
//   zfallback_kernel     the fp64 product-form draw (one warp per queued token;
//   / zfallback_log_k.   the log-space draw in the exact-weights mode)
//   wterm_kernel<FINAL>  w- and z-factors of the log-joint from the counts, the fixed-
//                        order final sum (eval.cpp:393-422); sharded: this rank's
//                        pieces -> [allreduce 3 doubles] -> finalize_kernel
//
// Device layout (HBM): w, z int32 [N_local]; phiT fp64 [V][Kp] (word-major, so
// the K weights of a token are one contiguous row; Kp = K rounded up to the
// z-step tile, padding is zero); nkw int32 [V][Kp]; nmk int32 [M_local][K];
// theta fp64 [M_local][K] (the reference's row-major layout).
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>

#include "common.cuh"
#include "dist.cuh"

namespace bnmc_gpu {

// wordmajor.cu (CUB): stable pair sort on key bits [0, end_bit) -> which buffer holds
// the result; runs of equal keys of a sorted array -> their count
int sort_pairs_u32(std::uint32_t* keys, std::uint32_t* keys_alt, int* vals, int* vals_alt, std::int64_t n,
                   int end_bit, cudaStream_t st);
std::int64_t run_length_u32(const std::uint32_t* keys, std::int64_t n, std::uint32_t* uniq, int* counts,
                            cudaStream_t st);

namespace {

constexpr int kZThreads = 256;
constexpr int kChunk = 2048;  // max tokens per z-step work unit

// Column of logical candidate k in a phiT32 row (see zscreen_kernel): lane gl of a
// G-lane group owns candidates [CW*R*gl, CW*R*(gl+1)); its round-r chunk of CW is
// stored at CW*(r*G + gl), so each round of a group is one contiguous G*CW*4 bytes.
__host__ __device__ __forceinline__ int phys32(int k, int R, int G, int CW) {
  const int c = k / CW, j = k - c * CW, gl = c / R, r = c - gl * R;
  return (r * G + gl) * CW + j;
}

// Programmatic dependent launch: kernels launched with launch_pdl may start while
// their stream predecessor drains; they wait here before touching its results
// (a no-op for a normal launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets the stream successor's blocks be scheduled once every block of this grid has
// passed this point (they still wait for this grid's completion in pdl_wait).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct LdaArgs {
  int K, Kp, V;
  std::int64_t Ml, Nl;
  const int* w;
  int* z;
  const std::int64_t* off;   // local offsets, off[0] = 0
  const std::int64_t* units; // z-step work units: [n_units][3] = doc, t0, t1
  std::int64_t n_units;
  const std::int64_t* wunits; // warp-level units (<= 256 tokens of one document)
  std::int64_t n_wunits;
  std::int64_t tok_base, doc_base;
  double* phiT;
  float* phiT32;     // fp32 copy of phiT [V][Kp32], columns permuted by phys32 (screen only)
  int Kp32, G32, R32, CW32; // screen layout: Kp32 = CW32 * G32 * R32
  int col_stripes;           // phi_colsum2 column-stripe blocks
  double* logphiT;   // exact mode only
  double* theta;
  int* nkw;          // [V][Kp]
  int* nmk;          // [Ml][K]
  double* colpart2;  // [nb_phi][K][2] (phi_norm_kernel: eval / exact-mode normalisation)
  double* S;         // [K]
  double* phi_term;  // [K]
  double* tpart;     // [Ml] theta-factor pieces
  double* zpart;     // [nbw] z-factor pieces (sum n[d,k] log theta[d,k]) per wterm block
  double* logS;      // [K] log of the gamma row sums
  int logg_valid;    // phiT holds this sweep's gamma draws g and logS their log row sums
                     // (inside a sweep): the w-factor is n (log g - log S)
  float screen_margin;  // kScreenMargin (BNMC_SCREEN_MARGIN overrides: tests force the fallback)
  int2* fq;          // screen fallback queue: (local token, local document) [Nl]
  int* fq_len;
  double* wpart;     // [nbw] w-factor pieces per wterm block
  double* ttpart;    // [nbw] per wterm block: its slice of tpart (single-rank path)
  int nbw;           // wterm_kernel blocks
  double* doc_part;  // [Ml][3] (eval path)
  double* red;       // [4]
  double alpha, beta;
  int pow_alpha, pow_beta;  // 1/alpha, 1/beta when exactly an integer in [2, 64] (boost by squaring), else 0
  int trow_blocks;          // phi_colsum2: y-blocks finishing the pool's theta rows
  int pool_phi;             // phi_pool: the pool draws the phi cells too (0: phi clamped)
  int pool_v0, pool_v1;     // phi_pool: the phi rows it draws (sharded: this rank's row slice)
  double phi_norm, phi_lgasum, theta_norm, theta_lgasum;
  std::uint64_t seed;
  std::uint64_t zkey_prefix;  // fold(fold(fold(1, seed), kDiscrete), var_z)
  int var_phi, var_theta, var_z;
  int rows_per_block, nb_phi;
  double* spart;     // [kColStripes][K][2]
  int* ticket;       // [ceil(K/32)] last-block tickets of phi_colsum2
  int* ticket2;      // last-block ticket of wterm_kernel<true>
  int red_only;      // sharded: the last wterm block writes red[0..2] (this rank's theta, z, w
                     // pieces) for the all-reduce instead of the log-joint
  std::int64_t docs_per_block, nb_doc;
  // word-major z-step order (build_word_major): units [n][3] = word, i0, i1 over the
  // sorted token list; tok / doc of sorted position i; th32 = fp32 theta/S rows
  // [Ml][Kp32] in the phiT32 column order
  const int* wm_tok;
  const int* wm_doc;
  float* th32;
  double* thS;                    // word-major: theta/S in fp64 [Ml][K] (the fallback's operand)
  unsigned long long* wm_ticket;  // next unit to claim (zeroed before each word-major launch)
};

// ---------------------------------------------------------------------------------
// phi block
// ---------------------------------------------------------------------------------
// The shape < 1 boost g * u^(1/shape) (dist.cpp:139-140) when 1/shape is exactly an
// integer e (lda.bn's alpha = beta = 0.1: e = 10): u^e by binary powering (4 multiplies
// for e = 10, <= ~4 ulp from the correctly rounded power -- pow's own error is <= 1 ulp,
// the exp(log) form below ~40 ulp) instead of a log and an exp per zero-count cell.
__device__ __forceinline__ double boost_factor(double u, int e, double inv) {
  if (e == 0) return exp(inv * log(u));
  if (e == 10) {  // lda.bn's alpha = beta = 0.1: the loop below unrolled (same products)
    const double u2 = u * u, u4 = u2 * u2;
    return u2 * (u4 * u4);
  }
  double r = 1.0, b = u;
  for (; e; e >>= 1) {
    if (e & 1) r *= b;
    b *= b;
  }
  return r;
}

constexpr int kGammaTab = 64;

// phi + theta block ("warp pool"): a persistent grid (one resident wave) in which warp w
// owns the contiguous range [w C / W, (w+1) C / W) of the C cells of the sweep's conjugate
// draws -- the phi cells (v, k) of rows [pool_v0, pool_v1) in phiT row order (all V rows
// on one GPU, the rank's row slice when sharded), then the theta cells (m, k) of the
// rank's documents -- so every warp has the same number of cells.  The 32 lanes draw the
// range as one pool, <= kPoolCells cells (one shared-memory chunk of counts) at a time:
// every iteration each lane makes one Marsaglia-Tsang attempt on its current cell, and the
// lanes whose attempt was accepted take the next undrawn cells (ballot + prefix rank).  A
// warp iterates ~(cells x 1.06) / 32 times with all lanes busy until the chunk's last
// attempts -- the r01 kernels' lanes each ran their own cells' rejection sequences and
// waited for the slowest lane of the warp (ncu: ~930 thread instructions per cell, 20.7 of
// 32 lanes active per instruction), the phi grid left a 1.64-wave tail and theta ran on a
// side stream.
// * No column partials and no per-cell log here: phi_colsum2_kernel sums the columns of
//   phiT directly (sum g, and sum log g as the log of a frexp-renormalised product) and
//   finishes the theta rows; the log-joint's w-factor takes log g of the counted cells
//   (wterm_kernel).
// * Streams keyed(seed, 4, var, iter).derive(k, v) (phi) / .derive(doc, k) (theta),
//   consumed in the reference's order (gaussian until 1 + c x > 0, uniform, [boost
//   uniform]; dist.cpp:136-155): the draws are the reference's whichever lane draws a cell.
constexpr int kPoolCells = 512;
constexpr int kPoolWarps = 8;

// cell c of the flat [V][K] order -> (v, k); double reciprocal + one correction step
__device__ __forceinline__ void cell_vk(std::int64_t c, int K, double invK, int& v, int& k) {
  std::int64_t q = static_cast<std::int64_t>(static_cast<double>(c) * invK);
  std::int64_t r = c - q * K;
  if (r < 0) {
    --q;
    r += K;
  } else if (r >= K) {
    ++q;
    r -= K;
  }
  v = static_cast<int>(q);
  k = static_cast<int>(r);
}

// Marsaglia-Tsang's second acceptance test, log(u) < 0.5 x^2 + d (1 - v + log(v))
// (dist.cpp:146-149), with the two logs first taken in fp32 (MUFU.LG2): when the fp32
// sides are further apart than a bound 40x the fp32 log error (1e-5 (1 + |log|) per log,
// lg2.approx is within 2^-21 (1 + |log2|)), that decides the comparison exactly as the
// double expression would; otherwise (~1e-4 of the calls) the double logs decide.  The
// squeeze fails for ~3 % of the attempts, so the double path used to run in most warp
// iterations for one or two lanes (ncu r02: ~19 % of the pool's instructions).
__device__ __forceinline__ bool mt_log_test(double u, double x, double v, double d) {
  if (v > 1e-30 && v < 1e30) {
    const double lu = static_cast<double>(__log2f(static_cast<float>(u))) * 0.69314718055994530942;
    const double lv = static_cast<double>(__log2f(static_cast<float>(v))) * 0.69314718055994530942;
    const double rhs = 0.5 * x * x + d * (1.0 - v + lv);
    const double err = 1e-5 * (1.0 + fabs(lu)) + d * 1e-5 * (1.0 + fabs(lv)) + 1e-12 * (1.0 + fabs(rhs));
    if (lu + err < rhs) return true;
    if (lu - err > rhs) return false;
  }
  return log(u) < 0.5 * x * x + d * (1.0 - v + log(v));
}

template <bool KTAB>
__global__ void __launch_bounds__(256) phi_pool_kernel(LdaArgs a, const std::int64_t* iter_p) {
  __shared__ double tab_d[2][kGammaTab], tab_c[2][kGammaTab], tab_inv[2][kGammaTab];
  __shared__ std::uint64_t kkey_s[KTAB ? kPoolCells : 1];
  __shared__ int col32_s[KTAB ? kPoolCells : 1];
  __shared__ int cnt_s[kPoolWarps][kPoolCells];
  const std::int64_t iter = *iter_p;
  for (int i = threadIdx.x; i < 2 * kGammaTab; i += blockDim.x) {
    const int kind = i / kGammaTab, n = i - kind * kGammaTab;  // 0: phi (beta), 1: theta (alpha)
    const double shape = (kind ? a.alpha : a.beta) + static_cast<double>(n);
    const bool boost = shape < 1.0;
    const double aa = boost ? shape + 1.0 : shape;
    const double d = aa - 1.0 / 3.0;
    tab_d[kind][n] = d;
    tab_c[kind][n] = 1.0 / sqrt(9.0 * d);
    tab_inv[kind][n] = boost ? 1.0 / shape : 0.0;
  }
  const std::uint64_t base = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_phi),
                                   static_cast<std::uint64_t>(iter));
  const std::uint64_t tbase = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_theta),
                                    static_cast<std::uint64_t>(iter));
  if constexpr (KTAB) {
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
      kkey_s[k] = fold(base, static_cast<std::uint64_t>(k));
      col32_s[k] = a.phiT32 ? phys32(k, a.R32, a.G32, a.CW32) : 0;
    }
  }
  __syncthreads();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  int* cnt = cnt_s[threadIdx.x >> 5];
  const unsigned lt = (1u << lane) - 1u;
  const double invK = 1.0 / static_cast<double>(a.K);
  // cells [0, cphi): phi (v, k) of rows [pool_v0, pool_v1) in phiT row order;
  // [cphi, cphi + Ml K): theta (m, k)
  const std::int64_t cphi = a.pool_phi ? static_cast<std::int64_t>(a.pool_v1 - a.pool_v0) * a.K : 0;
  const std::int64_t ncells = cphi + a.Ml * a.K;
  const std::int64_t nw = static_cast<std::int64_t>(gridDim.x) * (blockDim.x >> 5);
  const std::int64_t gw = static_cast<std::int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const std::int64_t c_end = ncells * (gw + 1) / nw;
  const float invKf = 1.0f / static_cast<float>(a.K);
  for (std::int64_t c0 = ncells * gw / nw; c0 < c_end; c0 += kPoolCells) {
    const int n = static_cast<int>(c_end - c0 < kPoolCells ? c_end - c0 : kPoolCells);
    // chunk bases: cells j < jt are phi cells (v, k) = (pv0, pk0) + j, cells j >= jt theta
    // cells (m, k) = (tm0, tk0) + (j - jt) in row-major order; within the chunk, row and
    // column come from a 32-bit offset r < K + 1024 by one float reciprocal (exact: the
    // quotient's fractional part stays >= 0.5 / K away from an integer)
    const int jt = static_cast<int>(cphi - c0 <= 0 ? 0 : (cphi - c0 >= n ? n : cphi - c0));
    int pv0 = 0, pk0 = 0, tm0 = 0, tk0 = 0;
    if (jt > 0) {
      cell_vk(c0, a.K, invK, pv0, pk0);
      pv0 += a.pool_v0;
    }
    if (jt < n) cell_vk(c0 + jt - cphi, a.K, invK, tm0, tk0);
    auto vk_of = [&](int j, int& v, int& k) {  // (v or m, k) of chunk cell j
      const int r = j < jt ? pk0 + j : tk0 + (j - jt);
      const int q = __float2int_rz((static_cast<float>(r) + 0.5f) * invKf);
      v = (j < jt ? pv0 : tm0) + q;
      k = r - q * a.K;
    };
    auto count_at = [&](int j) -> int* {
      int v, k;
      vk_of(j, v, k);
      return j < jt ? a.nkw + static_cast<std::size_t>(v) * a.Kp + k
                    : a.nmk + static_cast<std::size_t>(v) * a.K + k;
    };
    // the chunk's counts into shared memory (consumed: the z-step accumulates the next
    // sweep's counts here), 8 loads in flight per lane before the zeroing stores (the
    // stores may alias the next loads: a load-store loop would serialise one HBM round
    // trip per 32 cells)
    for (int j0 = 0; j0 < n; j0 += 8 * 32) {
      int val[8];
      int* at[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = j0 + 32 * i + lane;
        val[i] = 0;
        at[i] = nullptr;
        if (j < n) {
          at[i] = count_at(j);
          val[i] = __ldcg(at[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (at[i]) {
          cnt[j0 + 32 * i + lane] = val[i];
          *at[i] = 0;
        }
      }
    }
    // the next chunk's counts into L2 meanwhile (one line per 32 cells)
    {
      const std::int64_t cn = c0 + kPoolCells + 32 * lane;
      if (cn < c_end) {
        int v, k;
        cell_vk(cn < cphi ? cn : cn - cphi, a.K, invK, v, k);
        if (cn < cphi) v += a.pool_v0;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(cn < cphi ? a.nkw + static_cast<std::size_t>(v) * a.Kp + k
                                                                : a.nmk + static_cast<std::size_t>(v) * a.K + k));
      }
    }
    __syncwarp();
    int j = lane, next = 32;
    bool fresh = true;
    std::uint64_t pos = 0;
    double d = 1.0, c = 1.0, inv = 0.0;
    double* outp = nullptr;
    float* out32 = nullptr;
    int pw = 0;
    while (__any_sync(0xffffffffu, j < n)) {
      bool accepted = false;
      if (j < n) {
        if (fresh) {
          const int cn = cnt[j];
          const int kind = j >= jt;
          int v, k;
          vk_of(j, v, k);
          if (!kind) {  // phi cell (v, k): Stream(derive(base, k, v))
            pos = fold(KTAB ? kkey_s[k] : fold(base, static_cast<std::uint64_t>(k)), static_cast<std::uint64_t>(v));
            outp = a.phiT + static_cast<std::size_t>(v) * a.Kp + k;
            out32 = a.phiT32 ? a.phiT32 + static_cast<std::size_t>(v) * a.Kp32 +
                                   (KTAB ? col32_s[k] : phys32(k, a.R32, a.G32, a.CW32))
                             : nullptr;
            pw = a.pow_beta;
          } else {  // theta cell (m, k): Stream(derive(tbase, doc_base + m, k)), g unnormalised
            pos = fold(fold(tbase, static_cast<std::uint64_t>(a.doc_base + v)), static_cast<std::uint64_t>(k));
            outp = a.theta + static_cast<std::size_t>(v) * a.K + k;
            out32 = nullptr;
            pw = a.pow_alpha;
          }
          if (cn < kGammaTab) {
            d = tab_d[kind][cn];
            c = tab_c[kind][cn];
            inv = tab_inv[kind][cn];
          } else {
            const double shape = (kind ? a.alpha : a.beta) + static_cast<double>(cn);  // >= 64: no boost
            d = shape - 1.0 / 3.0;
            c = 1.0 / sqrt(9.0 * d);
            inv = 0.0;
          }
          fresh = false;
        }
        pos += kGolden;
        const double u1 = (static_cast<double>(mix(pos) >> 11) + 0.5) * 0x1p-53;
        pos += kGolden;
        const double u2 = (static_cast<double>(mix(pos) >> 11) + 0.5) * 0x1p-53;
        const double x = sqrt(-2.0 * log(u1)) * cos(6.28318530717958647692529 * u2);
        double vv = 1.0 + c * x;
        if (vv > 0.0) {
          vv = vv * vv * vv;
          pos += kGolden;
          const double u = (static_cast<double>(mix(pos) >> 11) + 0.5) * 0x1p-53;
          bool acc = u < 1.0 - 0.0331 * (x * x) * (x * x);
          if (!acc) acc = mt_log_test(u, x, vv, d);
          if (acc) {
            double g = d * vv;
            if (inv != 0.0) {
              pos += kGolden;
              g = g * boost_factor((static_cast<double>(mix(pos) >> 11) + 0.5) * 0x1p-53, pw, inv);
            }
            *outp = g;
            if (out32) *out32 = static_cast<float>(g);
            accepted = true;
          }
        }
      }
      const unsigned am = __ballot_sync(0xffffffffu, accepted);
      if (accepted) {
        j = next + __popc(am & lt);
        fresh = true;
      }
      next += __popc(am);
    }
    __syncwarp();
  }
}

constexpr int kColStripes = 128;

// Per topic k: S[k] = sum_v g[v][k] (the Dirichlet row sum, batch.cpp:55-58) and the phi
// factor (beta-1)(sum log g - V log S) - sum lgamma(beta) + lgamma(sum beta)
// (dist.cpp:115-130; sum phi = sum g / S = 1 by construction), from phiT itself.
// Grid (ceil(K/32), col_stripes + trow_blocks): block (kb, s < col_stripes) sums stripe s
// of the rows for 32 topics (threads 32 x 8: sum g, and sum log g as log(mantissa
// product) + exponent sum, frexp-renormalised after every factor -- one log per thread
// and column instead of one per cell; fixed-order smem reduction) into spart[s][k]; the
// last stripe block of kb to finish (atomic ticket) adds the stripes in stripe order.
// The ticket decides who adds, never the order: deterministic.  Blocks with
// blockIdx.y >= col_stripes finish the pool's theta rows (theta_row_finish).
struct LogProd {
  double mant = 1.0;
  int ex = 0;
  bool zero = false;
  // frexp by bit operations for normal positive doubles (the gamma draws here are
  // >= ~1e-175: normal); frexp's own special-case branches for the rest
  static __device__ __forceinline__ double split(double x, int& e) {
    const long long b = __double_as_longlong(x);
    const int be = static_cast<int>((b >> 52) & 0x7ff);
    if (be == 0 || be == 0x7ff) return frexp(x, &e);
    e = be - 1022;
    return __longlong_as_double((b & 0x000fffffffffffffll) | 0x3fe0000000000000ll);
  }
  __device__ __forceinline__ void mul(double g) {
    if (g > 0.0) {
      int e1, e2;
      mant = split(mant * split(g, e1), e2);
      ex += e1 + e2;
    } else {
      zero = true;
    }
  }
  __device__ __forceinline__ double log_value() const {
    return zero ? -INFINITY : log(mant) + static_cast<double>(ex) * 0.69314718055994530942;
  }
};

// Theta row m of the warp-pool block (one warp): the pool left the gamma draws g in
// theta; S = sum g, sum log g (log of the frexp product), theta = g / S and the
// row's Dirichlet log-pdf piece (dist.cpp:115-130: (alpha-1)(sum log g - K log S)
// - sum lgamma(alpha) + lgamma(sum alpha); sum theta = 1 by construction).  Lane sums
// in k order, lanes combined by a fixed shfl_down tree: deterministic.
__device__ __forceinline__ void theta_row_finish(const LdaArgs& a, std::int64_t m) {
  const int lane = threadIdx.x & 31;
  double* row = a.theta + m * a.K;
  double s = 0.0;
  LogProd lp;
  for (int k = lane; k < a.K; k += 32) {
    const double g = row[k];
    s += g;
    lp.mul(g);
  }
  double l = lp.log_value();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_down_sync(0xffffffffu, s, o);
    l += __shfl_down_sync(0xffffffffu, l, o);
  }
  const double S = __shfl_sync(0xffffffffu, s, 0);
  for (int k = lane; k < a.K; k += 32) row[k] = row[k] / S;
  if (lane == 0) {
    const double lpdf = (a.alpha - 1.0) * (l - static_cast<double>(a.K) * log(S));
    a.tpart[m] = (!(S > 0.0) || !isfinite(S)) ? -INFINITY : lpdf - a.theta_norm + a.theta_lgasum;
  }
}

__global__ void __launch_bounds__(256) phi_colsum2_kernel(LdaArgs a) {
  __shared__ double sg_s[8][33], sl_s[8][33];
  __shared__ bool last;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {  // this sweep's redraw queues
    if (a.fq_len) *a.fq_len = 0;
  }
  const int stripes = a.col_stripes;
  if (static_cast<int>(blockIdx.y) >= stripes) {  // theta rows of the warp-pool block
    const std::int64_t w0 = (static_cast<std::int64_t>(blockIdx.y - stripes) * gridDim.x + blockIdx.x) * 8 + (threadIdx.x >> 5);
    const std::int64_t nwr = static_cast<std::int64_t>(a.trow_blocks) * gridDim.x * 8;
    for (std::int64_t m = w0; m < a.Ml; m += nwr) theta_row_finish(a, m);
    return;
  }
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + tx;
  const std::int64_t rows = a.V;
  const std::int64_t chunk = (rows + stripes - 1) / stripes;
  const std::int64_t b0 = blockIdx.y * chunk, b1 = min(rows, b0 + chunk);
  double sg = 0.0, sl = 0.0;
  if (k < a.K) {
    LogProd lp;
    for (std::int64_t b = b0 + ty; b < b1; b += 64) {  // 8 loads in flight
      double g8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const std::int64_t bj = b + 8 * j;
        g8[j] = bj < b1 ? a.phiT[bj * a.Kp + k] : 1.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (b + 8 * j < b1) {
          sg += g8[j];
          lp.mul(g8[j]);
        }
      }
    }
    sl = lp.log_value();
  }
  sg_s[ty][tx] = sg;
  sl_s[ty][tx] = sl;
  __syncthreads();
  if (ty == 0 && k < a.K) {
    double g = 0.0, l = 0.0;
    for (int j = 0; j < 8; ++j) {
      g += sg_s[j][tx];
      l += sl_s[j][tx];
    }
    a.spart[(static_cast<std::size_t>(blockIdx.y) * a.K + k) * 2] = g;
    a.spart[(static_cast<std::size_t>(blockIdx.y) * a.K + k) * 2 + 1] = l;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int t = atomicAdd(&a.ticket[blockIdx.x], 1);
    last = t == stripes - 1;
    if (last) a.ticket[blockIdx.x] = 0;  // every stripe has arrived: reset for the next sweep
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // stripes s = ty, ty + 8, ... per warp (8 loads in flight: one L2 round trip per 64
  // stripes), then the 8 warp sums in order: fixed order
  sg = sl = 0.0;
  if (k < a.K) {
    for (int s0 = 0; s0 < stripes; s0 += 64) {
      double g8[8], l8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int st = s0 + ty + 8 * j;
        g8[j] = st < stripes ? __ldcg(&a.spart[(static_cast<std::size_t>(st) * a.K + k) * 2]) : 0.0;
        l8[j] = st < stripes ? __ldcg(&a.spart[(static_cast<std::size_t>(st) * a.K + k) * 2 + 1]) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sg += g8[j];
        sl += l8[j];
      }
    }
  }
  __syncthreads();
  sg_s[ty][tx] = sg;
  sl_s[ty][tx] = sl;
  __syncthreads();
  if (ty != 0 || k >= a.K) return;
  double g = 0.0, l = 0.0;
  for (int j = 0; j < 8; ++j) {
    g += sg_s[j][tx];
    l += sl_s[j][tx];
  }
  a.S[k] = g;
  const double lS = log(g);
  a.logS[k] = lS;
  const double lp = (a.beta - 1.0) * (l - static_cast<double>(a.V) * lS);
  a.phi_term[k] = (!(g > 0.0) || !(a.beta > 0.0)) ? -INFINITY : lp - a.phi_norm + a.phi_lgasum;
}

// fp32 screen copy of phi's numerator: phiT32 = (float)(phiT / S) (S = 1 outside a sweep).
__global__ void phi_f32_kernel(LdaArgs a) {
  const std::int64_t n = static_cast<std::int64_t>(a.V) * a.K;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t v = i / a.K, k = i % a.K;
    a.phiT32[v * a.Kp32 + phys32(static_cast<int>(k), a.R32, a.G32, a.CW32)] = static_cast<float>(a.phiT[v * a.Kp + k] / a.S[k]);
  }
}

__global__ void fill_kernel(double* p, int n, double v) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) p[i] = v;
}

// phi = g / S[k]; accumulates (beta-1)*log(phi) and phi per topic for the log-joint.
// NORMALISE (the exact-mode sweep, a checkpoint restore): phi written back in place; its
// colpart2 pieces are not read afterwards (the sweep's phi prior term comes from
// phi_colsum2, a restore recomputes them), so only the log phi table takes logs.
template <bool NORMALISE>
__global__ void phi_norm_kernel(LdaArgs a) {
  const int b = blockIdx.x;
  const int v0 = b * a.rows_per_block;
  const int v1 = min(a.V, v0 + a.rows_per_block);
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    const double S = a.S[k];
    double lp = 0.0, sx = 0.0;
    for (int v = v0; v < v1; ++v) {
      const std::size_t c = static_cast<std::size_t>(v) * a.Kp + k;
      const double x = a.phiT[c] / S;
      if (NORMALISE) {
        a.phiT[c] = x;
        // (exact mode: the fp32 screen then reads phi itself, with S = 1)
        if (a.phiT32) a.phiT32[static_cast<std::size_t>(v) * a.Kp32 + phys32(k, a.R32, a.G32, a.CW32)] = static_cast<float>(x);
      }
      if (NORMALISE && !a.logphiT) continue;
      const double lx = x > 0.0 ? log(x) : -INFINITY;
      if (a.logphiT) a.logphiT[c] = lx;
      lp += (a.beta - 1.0) * lx;
      sx += x;
    }
    if (NORMALISE) continue;
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
// A token's candidate weights are handled by a group of G lanes; lane gl owns
// candidates 4*(r*G + gl) .. +3 for rounds r < Rr = Kp/(4G), so every round is one
// coalesced 32*G-byte segment of the token's phiT row.  All rounds' loads are
// issued before any cross-lane work (memory-level parallelism), then the R
// per-round group scans run interleaved.  Weights are the product theta*phi
// (default) or exp(log theta + log phi - max) exactly as the reference (EXACT).
// The inverse CDF keeps the reference's candidate order: the draw is the first k
// whose running sum exceeds u = next_unit * total (dist.cpp:209-214).
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
__device__ __forceinline__ double g_sum(double v, unsigned m) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(m, v, o, G);
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

// 256-bit read-only global load (LDG.E.ENL2.256 on sm_100a): a lane's 4 candidates
// in one request, so a G=4 group reads one full 128-byte line per round.
__device__ __forceinline__ Quad ldg256(const double* p) {
  Quad q;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(q.v0), "=d"(q.v1), "=d"(q.v2), "=d"(q.v3)
      : "l"(p));
  return q;
}

// Where a lane's theta values come from: registers loaded once per work unit (TR)
// or the CTA's shared-memory row (fewer registers, more LSU traffic).
template <int R, bool TR>
struct ThetaSrc;

template <int R>
struct ThetaSrc<R, true> {
  Quad q[R];
  __device__ __forceinline__ Quad at(int r, int) const { return q[r]; }
  __device__ __forceinline__ Quad dyn(int rr, int) const {
    Quad t = q[0];
#pragma unroll
    for (int r = 1; r < R; ++r)
      if (r == rr) t = q[r];
    return t;
  }
};

template <int R>
struct ThetaSrc<R, false> {
  const double* p;
  __device__ __forceinline__ Quad at(int, int k) const {
    const double2 t0 = *reinterpret_cast<const double2*>(p + k);
    const double2 t1 = *reinterpret_cast<const double2*>(p + k + 2);
    return Quad{t0.x, t0.y, t1.x, t1.y};
  }
  __device__ __forceinline__ Quad dyn(int, int k) const { return at(0, k); }
};

// The lane's 4 candidate weights at column k: theta*phi (tq = the lane's theta
// values, kept in registers for the whole work unit) or, EXACT, exp(log theta +
// log phi - max) with tq = log theta.
template <bool EXACT>
__device__ __forceinline__ Quad weights(const Quad& tq, const double* row, const double* lrow, int k,
                                        double mx) {
  Quad q;
  if constexpr (!EXACT) {
    const Quad a = ldg256(row + k);
    q.v0 = tq.v0 * a.v0;
    q.v1 = tq.v1 * a.v1;
    q.v2 = tq.v2 * a.v2;
    q.v3 = tq.v3 * a.v3;
  } else {
    const Quad a = ldg256(lrow + k);
    q.v0 = exp((tq.v0 + a.v0) - mx);
    q.v1 = exp((tq.v1 + a.v1) - mx);
    q.v2 = exp((tq.v2 + a.v2) - mx);
    q.v3 = exp((tq.v3 + a.v3) - mx);
  }
  return q;
}

// Returns the drawn topic in every lane of the group, or -1 when every weight is
// zero/-inf (the reference throws std::domain_error; the product form retries in
// log space).
template <int G, int R, bool EXACT, class TS>
__device__ __forceinline__ int draw_topic(const TS& tq, const double* row, const double* lrow, int K,
                                          int Rr, double u01) {
  const unsigned m = group_mask<G>();
  const int gl = threadIdx.x & (G - 1);
  double mx = 0.0;
  if constexpr (EXACT) {
    double lm = -INFINITY;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < Rr) {
        const Quad a = ldg256(lrow + 4 * (r * G + gl));
        const Quad t = tq.at(r, 4 * (r * G + gl));
        lm = fmax(lm, fmax(fmax(t.v0 + a.v0, t.v1 + a.v1), fmax(t.v2 + a.v2, t.v3 + a.v3)));
      }
    }
    mx = g_max<G>(lm, m);
    if (!isfinite(mx)) return -1;
  }
  // phase A: every round's weights (independent loads), lane-chunk sums s[r] and the
  // lane's running prefix over rounds Q[r] (registers only, no cross-lane traffic)
  double s[R], Q[R];
  double run = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    s[r] = 0.0;
    if (r < Rr) {
      const Quad q = weights<EXACT>(tq.at(r, 4 * (r * G + gl)), row, lrow, 4 * (r * G + gl), mx);
      s[r] = ((q.v0 + q.v1) + q.v2) + q.v3;
    }
    run += s[r];
    Q[r] = run;
  }
  // Candidate order is round-major, so the running sum at the end of round r is
  // f(r) = sum over the group of Q[r].  total = f(R-1); the crossing round is found
  // by a branch-free binary search over r (log2 R group sums instead of R scans).
  const double total = g_sum<G>(Q[R - 1], m);
  if (!(total > 0x1p-1000) || !isfinite(total)) return -1;
  const double u = u01 * total;
  int pos = 0;
  double base = 0.0;
  constexpr int P = R <= 1 ? 1 : (R <= 2 ? 2 : (R <= 4 ? 4 : (R <= 8 ? 8 : 16)));  // pow2 >= R
#pragma unroll
  for (int step = P / 2; step >= 1; step >>= 1) {
    const int c = pos + step - 1;
    double qc = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (r == c) qc = Q[r];
    const double f = g_sum<G>(qc, m);
    if (c < Rr && !(u < f)) {
      pos += step;
      base = f;
    }
  }
  if (R == 1 || pos >= Rr) pos = Rr - 1;  // u >= total by rounding: last round
  // Within round `pos`: exclusive scan of the lane-chunk sums -> each chunk's start.
  double sc = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (r == pos) sc = s[r];
  double inc = sc;
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    const double t = __shfl_up_sync(m, inc, d, G);
    if (gl >= d) inc += t;
  }
  double ex = __shfl_up_sync(m, inc, 1, G);
  if (gl == 0) ex = 0.0;
  const double start = base + ex;
  const int owner = g_max_i<G>(start <= u ? gl : 0, m);
  int kk = 0;
  if (gl == owner) {
    const int k0 = 4 * (pos * G + gl);
    const Quad q = weights<EXACT>(tq.dyn(pos, k0), row, lrow, k0, mx);
    double acc = start;
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
  return __shfl_sync(m, kk, owner, G);
}


// ---------------------------------------------------------------------------------
// z block, fp32 screen + fp64 verification
// ---------------------------------------------------------------------------------
// The inverse-CDF draw is first evaluated on fp32 copies of theta/S and g (half the
// bytes: one 256-bit load carries 8 candidates).  The fp32 running sums differ from
// the exact cumulative weights by a small multiple of 2^-24 * total (bound below, at
// zscreen_kernel), and the draw is decided by the two running sums adjacent to u.
// When u is farther than kScreenMargin * total from both (and the total is far from
// fp32 underflow), the fp64 draw must pick the same candidate; otherwise the token is
// redrawn with the fp64 path.  The margin (2^-16) makes ~2 * K * 2^-16 of the tokens
// take the fp64 path (0.3 % at K = 100); the result is the fp64 product-form draw
// either way.
constexpr float kScreenMargin = 1.52587890625e-05f;  // 2^-16

struct Oct {
  float v[8];
};

__device__ __forceinline__ Oct ldg256f(const float* p) {
  Oct o;
#ifdef BNMC_LDG_NOALLOC
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
#else
  asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
#endif
      : "=f"(o.v[0]), "=f"(o.v[1]), "=f"(o.v[2]), "=f"(o.v[3]), "=f"(o.v[4]), "=f"(o.v[5]), "=f"(o.v[6]),
        "=f"(o.v[7])
      : "l"(p));
  return o;
}

// Sequential log-space draw exactly as draw_from_log_weights, for the rare token
// whose product weights underflow (lane 0 of the group; result broadcast).
template <int G>
__device__ int draw_topic_logspace(const double* lth, const double* row, int K, double u01) {
  const unsigned m = group_mask<G>();
  const int gl = threadIdx.x & (G - 1);
  int pick = -1;
  if (gl == 0) {
    double mx = -INFINITY;
    for (int k = 0; k < K; ++k) mx = fmax(mx, lth[k] + (row[k] > 0.0 ? log(row[k]) : -INFINITY));
    if (isfinite(mx)) {
      double total = 0.0;
      for (int k = 0; k < K; ++k) total += exp((lth[k] + (row[k] > 0.0 ? log(row[k]) : -INFINITY)) - mx);
      const double u = u01 * total;
      double acc = 0.0;
      pick = K - 1;
      for (int k = 0; k < K; ++k) {
        acc += exp((lth[k] + (row[k] > 0.0 ? log(row[k]) : -INFINITY)) - mx);
        if (u < acc) {
          pick = k;
          break;
        }
      }
    }
  }
  return __shfl_sync(m, pick, 0, G);
}

// Word-major z-step operand: theta/S of every local document in fp32, in the phiT32
// column order (the value the document-major z-step forms per unit in shared memory).
// Padding columns stay 0 (zeroed at allocation).
// Also theta/S in fp64 for the fallback draw (one division per cell per sweep instead of
// one per cell per queued token: the divisions were half the fallback's instructions).
__global__ void th32_kernel(LdaArgs a) {
  const std::int64_t n = a.Ml * a.K;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    const std::int64_t m = i / a.K;
    const int k = static_cast<int>(i - m * a.K);
    const double q = a.theta[i] / a.S[k];
    a.th32[m * a.Kp32 + phys32(k, a.R32, a.G32, a.CW32)] = static_cast<float>(q);
    a.thS[i] = q;  // the same quotient the fallback would form per token
  }
}

// Word-major order keys: (document block, word) per local token, with its index and
// document (the sort carries the index; the document is gathered after it).
__global__ void wm_keys_kernel(LdaArgs a, std::int64_t block_docs, std::uint32_t* keys, int* tok, int* docof) {
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const std::uint32_t hi = static_cast<std::uint32_t>((m / block_docs) * a.V);
    for (std::int64_t t = a.off[m] + threadIdx.x; t < a.off[m + 1]; t += blockDim.x) {
      keys[t] = hi + static_cast<std::uint32_t>(a.w[t]);
      tok[t] = static_cast<int>(t);
      docof[t] = static_cast<int>(m);
    }
  }
}

__global__ void wm_gather_kernel(const int* tok, const int* docof, int* doc, std::int64_t n) {
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x)
    doc[i] = docof[tok[i]];
}

// ---------------------------------------------------------------------------------
// z block, lean fp32 screen (default): lane-contiguous candidates
// ---------------------------------------------------------------------------------
// The screened draw, structured to keep the per-token instruction count low
// (vs. a round-major grouped screen; ncu r01 v6: that kernel issued ~60 warp
// instructions per token, 22 % of them IMAD from RNG evaluated by every lane):
//  * lane gl of a G-lane group owns the CONTIGUOUS candidates [8R*gl, 8R*(gl+1)).
//    phiT32 rows are stored permuted (phys32) so that round r of the group is still
//    one contiguous 32G-byte segment (G = 4: one 128-byte line per round);
//  * the lane's own running prefix over its rounds stays in registers; one group
//    scan of the lane totals gives every lane its [start, end) interval, the owner
//    of u is found with one ballot, and only the owner searches (no per-round
//    group sums, no binary search over rounds);
//  * the RNG (3 splitmix finalizers) and the w load run once per token: lane j of a
//    warp handles token j of the warp's 32-token batch, then the values are
//    shuffled to the group that draws that token;
//  * FMA in the screen (explicit __fmaf_rn: --fmad=false only governs contraction).
// Error budget (u = 2^-24, T = the exact total; non-negative terms, so every rounding
// is bounded relative to T): each fp32 product carries 2u from its rounded operands;
// a compared running sum (prev / acc) passes through CW (the lane's round), R (its
// run), log2 G (the group scan), 1 (lo) and CW (the owner's re-scan) roundings:
// <= (2 CW + R + log2 G + 3) u T; uf = u01 * total: <= (CW + R + log2 G + 4) u T. The
// decision equals the fp64 one when the margin exceeds their sum, (3 CW + 2 R +
// 2 log2 G + 7) u: 49 u for G = 32, CW = 8, R = 4 and at most 57 u (R = 8). The
// grouped kernel uses 2^-17 = 128 u (>= 2.2x that), the transposed one 2^-16.

template <int CW>
struct FChunk {
  float v[CW];
};

template <int CW>
__device__ __forceinline__ FChunk<CW> ldg_chunk(const float* p) {
  FChunk<CW> c;
  if constexpr (CW == 8) {
    const Oct o = ldg256f(p);
#pragma unroll
    for (int j = 0; j < 8; ++j) c.v[j] = o.v[j];
  } else {
    static_assert(CW == 4, "chunk width 4 or 8");
    asm("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
        : "=f"(c.v[0]), "=f"(c.v[1]), "=f"(c.v[2]), "=f"(c.v[3])
        : "l"(p));
  }
  return c;
}

// G lanes per token, CW candidates per lane per round (G * CW = 32: one 128-byte
// line per round), R rounds; TFR keeps the lane's theta operands in registers
// across the work unit (else they are re-read from shared memory every token).
// WM (word-major order, build_word_major): a unit is one word's tokens of a block of
// documents; the word's g row is the resident operand (shared memory / registers) and
// each token streams its document's theta/S row (th32, L2-resident per document block).
// The products, running sums and decisions are the document-major ones operand for
// operand (x * y in fp32 commutes), so z is bitwise the same.
template <int G, int CW, int R, bool TFR, bool WM = false>
__global__ void __launch_bounds__(kZThreads) zscreen_kernel(LdaArgs a, const std::int64_t* iter_p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // theta/S in fp32: lane gl's KL candidates at thf[gl * KLP ..], the +4 pad keeps the
  // G lanes' 16-byte reads of one round in distinct banks
  float* thf = reinterpret_cast<float*>(smem_raw);
  const std::int64_t iter = *iter_p;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), gid = lane / G;
  const int warp = threadIdx.x >> 5;
  constexpr int kWarps = kZThreads / 32;
  constexpr int KL = CW * R;  // candidates per lane
  constexpr int KLP = KL + 4;
  const unsigned gmask = group_mask<G>();
  const unsigned gshift = static_cast<unsigned>(lane & ~(G - 1));
  constexpr unsigned gbits = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  // rounds of this lane that hold real candidates (the rest is padding, not fetched)
  const int rl = min(R, max(0, (a.K - gl * KL + CW - 1) / CW));

  // document-major: a CTA per unit (a document's tokens, warps on alternate batches);
  // word-major: a warp per unit (one word's ~60 tokens of a document block), its own
  // resident row in shared memory
  // word-major units are claimed in order from a ticket, so the units in flight stay
  // within one document block (static striding let warps drift over several blocks)
  if constexpr (WM) thf += warp * (G * KLP);
  auto next_unit = [&](std::int64_t cur) -> std::int64_t {
    if constexpr (WM) {
      unsigned long long u = 0;
      if (lane == 0) u = atomicAdd(a.wm_ticket, 1ull);
      return static_cast<std::int64_t>(__shfl_sync(0xffffffffu, u, 0));
    } else {
      return cur < 0 ? blockIdx.x : cur + gridDim.x;
    }
  };
  for (std::int64_t unit = next_unit(-1); unit < a.n_units; unit = next_unit(unit)) {
    // document-major: m = document, [t0, t1) tokens; word-major: m = word, [t0, t1)
    // positions in the sorted token list
    const std::int64_t m = a.units[unit * 3], t0 = a.units[unit * 3 + 1], t1 = a.units[unit * 3 + 2];
    if constexpr (WM) {
      const float* gv = a.phiT32 + m * a.Kp32;
      for (int k = lane; k < G * KL; k += 32)
        thf[(k / KL) * KLP + k % KL] = k < a.K ? gv[phys32(k, R, G, CW)] : 0.0f;
      __syncwarp();
    } else {
      const double* thg = a.theta + m * a.K;
      for (int k = threadIdx.x; k < G * KL; k += blockDim.x)
        thf[(k / KL) * KLP + k % KL] = k < a.K ? static_cast<float>(thg[k] / a.S[k]) : 0.0f;
      __syncthreads();
    }
    float tf[TFR ? KL : 1];
    if constexpr (TFR) {
#pragma unroll
      for (int i = 0; i < KL; i += 4) {
        const float4 t = *reinterpret_cast<const float4*>(thf + gl * KLP + i);
        tf[i] = t.x;
        tf[i + 1] = t.y;
        tf[i + 2] = t.z;
        tf[i + 3] = t.w;
      }
    }
    for (std::int64_t b0 = t0 + (WM ? 0 : warp * 32); b0 < t1; b0 += (WM ? 32 : kWarps * 32)) {
      // token b0 + lane: its word (word-major: its token index and document) and its
      // uniform, keyed(seed, 3, var_z, t, iter)
      const std::int64_t il = b0 + lane;
      const bool lvalid = il < t1;
      std::int64_t tl = il;
      int wl = 0;
      if constexpr (WM) {
        tl = lvalid ? __ldg(a.wm_tok + il) : 0;
        wl = lvalid ? __ldg(a.wm_doc + il) : 0;
      } else {
        wl = lvalid ? __ldg(a.w + tl) : 0;
      }
      float ul = 0.5f;
      if (lvalid) {
        Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + tl)),
                        static_cast<std::uint64_t>(iter)));
        ul = static_cast<float>(rng.next_unit());
      }
      const int tl32 = static_cast<int>(tl);
#pragma unroll 1
      for (int s = 0; s < G; ++s) {
        if (b0 + s * (32 / G) >= t1) break;  // warp-uniform: no token left in this sub-batch
        const int src = s * (32 / G) + gid;  // lane holding this group's token
        const bool valid = b0 + src < t1;
        // document-major: wv = word, t = token; word-major: wv = document, t shuffled
        const std::int64_t t = WM ? static_cast<std::int64_t>(__shfl_sync(0xffffffffu, tl32, src)) : b0 + src;
        const int wv = __shfl_sync(0xffffffffu, wl, src);
        const float u01 = __shfl_sync(0xffffffffu, ul, src);
        const float* row = WM ? a.th32 + static_cast<std::size_t>(wv) * a.Kp32
                              : a.phiT32 + static_cast<std::size_t>(wv) * a.Kp32;
        // all rounds' loads first (memory-level parallelism), then the fma chains
        FChunk<CW> ph[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r < rl) ph[r] = ldg_chunk<CW>(row + CW * (r * G + gl));
          else ph[r] = FChunk<CW>{};
        }
        float Q[R];
        float run = 0.0f;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float x[CW];
          if constexpr (TFR) {
#pragma unroll
            for (int j = 0; j < CW; ++j) x[j] = tf[CW * r + j];
          } else {
#pragma unroll
            for (int j = 0; j < CW; j += 4) {
              const float4 y = *reinterpret_cast<const float4*>(thf + gl * KLP + CW * r + j);
              x[j] = y.x, x[j + 1] = y.y, x[j + 2] = y.z, x[j + 3] = y.w;
            }
          }
          float sr = x[0] * ph[r].v[0];
#pragma unroll
          for (int j = 1; j < CW; ++j) sr = __fmaf_rn(x[j], ph[r].v[j], sr);
          run += sr;
          Q[r] = run;
        }
        // group inclusive scan of the lane totals -> [start, end) per lane
        float inc = run;
#pragma unroll
        for (int d = 1; d < G; d <<= 1) {
          const float y = __shfl_up_sync(gmask, inc, d, G);
          if (gl >= d) inc += y;
        }
        float start = __shfl_up_sync(gmask, inc, 1, G);
        if (gl == 0) start = 0.0f;
        const float total = __shfl_sync(gmask, inc, G - 1, G);
        const float uf = u01 * total;
        const float mg = a.screen_margin * total;
        int k = -1;
        if (start <= uf && uf < inc && total > 0x1p-90f && total < 0x1p100f) {
          // owner lane: the crossing round (registers), then the crossing candidate
          float lo = start;
          int rr = R - 1;
#pragma unroll
          for (int r = R - 1; r >= 0; --r)
            if (uf < start + Q[r]) rr = r;
#pragma unroll
          for (int r = 0; r < R - 1; ++r)
            if (r < rr) lo = start + Q[r];
          const int kl0 = gl * KL + CW * rr;  // logical index of the chunk's first candidate
          const FChunk<CW> p = ldg_chunk<CW>(row + CW * (rr * G + gl));
          float tv[CW];
#pragma unroll
          for (int j = 0; j < CW; j += 4) {
            const float4 y = *reinterpret_cast<const float4*>(thf + gl * KLP + CW * rr + j);
            tv[j] = y.x, tv[j + 1] = y.y, tv[j + 2] = y.z, tv[j + 3] = y.w;
          }
          // the chunk's running sums (the same fma chain), then the crossing candidate by
          // counting the sums <= uf (they never decrease) and an unrolled select
          float nx[CW];
          float run_c = lo;
#pragma unroll
          for (int jj = 0; jj < CW; ++jj) {
            run_c = __fmaf_rn(tv[jj], p.v[jj], run_c);
            nx[jj] = run_c;
          }
          int j = 0;
#pragma unroll
          for (int jj = 0; jj < CW; ++jj) j += uf >= nx[jj] ? 1 : 0;
          if (j < CW) {
            float acc = nx[0], prev = lo;
#pragma unroll
            for (int jj = 1; jj < CW; ++jj)
              if (j == jj) acc = nx[jj], prev = nx[jj - 1];
            if (kl0 + j < a.K && uf - prev >= mg && acc - uf >= mg) k = kl0 + j;
          }
        }
        const bool decided = ((__ballot_sync(0xffffffffu, k >= 0) >> gshift) & gbits) != 0;
        if (valid) {
          const std::int64_t word = WM ? m : wv, doc = WM ? wv : m;
          if (k >= 0) {
            a.z[t] = k;
            atomicAdd(&a.nkw[static_cast<std::size_t>(word) * a.Kp + k], 1);
            atomicAdd(&a.nmk[doc * a.K + k], 1);
          } else if (!decided && gl == 0) {
            // ambiguous for the screen: queued for the fp64 draw (zfallback_kernel)
            const int slot = atomicAdd(a.fq_len, 1);
            a.fq[slot] = make_int2(static_cast<int>(t), static_cast<int>(doc));
          }
        }
      }
    }
    if constexpr (WM) __syncwarp();
    else __syncthreads();
  }
}

// Transposed-search screen for K <= 128 (default there).  Two phases per warp batch
// of 32 tokens:
//  (1) products: G = 4 lanes per token (CW = 8, R rounds, lane-contiguous chunks as
//      in zscreen_kernel, coalesced 128-byte lines); each lane writes its R chunk
//      sums (8 candidates each) to the warp's shared-memory table csum[token][chunk];
//  (2) search: lane j takes token j -- prefix over the C = 4R chunk sums in
//      registers, u * total, the crossing chunk, one reload of that chunk and the
//      in-chunk scan, the margin check, z and the count atomics.
// Every lane does useful work in (2), instead of 1 lane in 4 for the in-group
// search, and no cross-lane scans are needed (ncu r01 v10: the grouped search was
// ~2/3 of the z-step's ~31 warp instructions per token).
// csum row layout: 16 floats per token row, 16-byte group q of row r stored at group
// q ^ ((r >> 1) & 3): the products phase's float4 writes (2 rows x 4 lanes per
// quarter warp) and the search phase's float4 reads (8 rows, one group) both touch
// 8 distinct bank groups -- no conflicts (ncu r01 v15: 1.05 M conflicting store
// wavefronts with a padded row layout).
__device__ __forceinline__ int cs_idx(int row, int c) {
  return row * 16 + ((((c >> 2) ^ (row >> 1)) & 3) << 2) + (c & 3);
}

// WU: warp-level work units (chunks of <= 256 tokens of one document, `wunits`): every
// warp owns its theta operands, chunk-sum table and doc-topic counts in shared memory
// and never waits on a CTA barrier; short documents (KOS: 136 tokens) no longer leave
// warps of a document-wide CTA idle, and long ones are split into warp-sized chunks.
template <int R, bool TFR, bool WU = false>
__global__ void __launch_bounds__(kZThreads, TFR ? 3 : 1) zscreen_t_kernel(LdaArgs a, const std::int64_t* iter_p) {
  constexpr int G = 4, CW = 8, KL = CW * R, KLP = KL + 4, C = G * R;
  static_assert(C <= 16, "csum rows hold 16 chunk sums");
  const int kWarps = blockDim.x >> 5;  // sized to the work units (zscreen_t_launch)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), gid = lane / G;
  const int warp = threadIdx.x >> 5;
  // CTA units: [thf G*KLP][csum kWarps*32*16][cnt K];  warp units: per warp the same
  const int kpad = (a.K + 3) & ~3;
  float* base = reinterpret_cast<float*>(smem_raw) + (WU ? warp * (G * KLP + 32 * 16 + kpad) : 0);
  float* thf = base;                                  // [G][KLP] theta/S, fp32
  float* csum = thf + G * KLP + (WU ? 0 : warp * 32 * 16);  // [32][16] chunk sums of the batch (cs_idx)
  int* cnt_s = reinterpret_cast<int*>(thf + G * KLP + (WU ? 32 * 16 : kWarps * 32 * 16));  // [K] doc-topic counts
  pdl_wait();
  pdl_trigger();
  const std::int64_t iter = *iter_p;
  const int rl = min(R, max(0, (a.K - gl * KL + CW - 1) / CW));
  const int tid_u = WU ? lane : static_cast<int>(threadIdx.x);      // thread index within the unit's team
  const int nthr_u = WU ? 32 : static_cast<int>(blockDim.x);
  const std::int64_t nunits = WU ? a.n_wunits : a.n_units;
  const std::int64_t* units = WU ? a.wunits : a.units;
  const std::int64_t ustart = WU ? static_cast<std::int64_t>(blockIdx.x) * kWarps + warp : blockIdx.x;
  const std::int64_t ustride = WU ? static_cast<std::int64_t>(gridDim.x) * kWarps : gridDim.x;

  for (std::int64_t unit = ustart; unit < nunits; unit += ustride) {
    const std::int64_t m = units[unit * 3], t0 = units[unit * 3 + 1], t1 = units[unit * 3 + 2];
    const double* thg = a.theta + m * a.K;
    for (int k = tid_u; k < G * KL; k += nthr_u) {
      thf[(k / KL) * KLP + k % KL] = k < a.K ? static_cast<float>(thg[k] / a.S[k]) : 0.0f;
      if (k < a.K) cnt_s[k] = 0;
    }
    if constexpr (WU) __syncwarp();
    else __syncthreads();
    float tf[TFR ? KL : 1];
    if constexpr (TFR) {
#pragma unroll
      for (int i = 0; i < KL; i += 4) {
        const float4 t = *reinterpret_cast<const float4*>(thf + gl * KLP + i);
        tf[i] = t.x, tf[i + 1] = t.y, tf[i + 2] = t.z, tf[i + 3] = t.w;
      }
    }
    for (std::int64_t b0 = t0 + (WU ? 0 : warp * 32); b0 < t1; b0 += (WU ? 32 : kWarps * 32)) {
      const std::int64_t t = b0 + lane;
      const bool valid = t < t1;
      const int wl = valid ? __ldg(a.w + t) : 0;
      // (1) products
#pragma unroll 1
      for (int s = 0; s < 32 / (32 / G); ++s) {
        if (b0 + s * (32 / G) >= t1) break;  // warp-uniform
        const int src = s * (32 / G) + gid;
        const int wv = __shfl_sync(0xffffffffu, wl, src);
        const float* row = a.phiT32 + static_cast<std::size_t>(wv) * a.Kp32;
        Oct ph[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (r < rl) ph[r] = ldg256f(row + CW * (r * G + gl));
          else ph[r] = Oct{};
        }
        float cs[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float x[CW];
          if constexpr (TFR) {
#pragma unroll
            for (int j = 0; j < CW; ++j) x[j] = tf[CW * r + j];
          } else {
            const float4 y0 = *reinterpret_cast<const float4*>(thf + gl * KLP + CW * r);
            const float4 y1 = *reinterpret_cast<const float4*>(thf + gl * KLP + CW * r + 4);
            x[0] = y0.x, x[1] = y0.y, x[2] = y0.z, x[3] = y0.w, x[4] = y1.x, x[5] = y1.y, x[6] = y1.z, x[7] = y1.w;
          }
          float sr = x[0] * ph[r].v[0];
#pragma unroll
          for (int j = 1; j < CW; ++j) sr = __fmaf_rn(x[j], ph[r].v[j], sr);
          cs[r] = sr;
        }
        if constexpr (R == 4) {
          *reinterpret_cast<float4*>(csum + cs_idx(src, gl * R)) = make_float4(cs[0], cs[1], cs[2], cs[3]);
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) csum[cs_idx(src, gl * R + r)] = cs[r];
        }
      }
      __syncwarp();
      // (2) search: lane = token
      if (valid) {
        Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + t)),
                        static_cast<std::uint64_t>(iter)));
        const float u01 = static_cast<float>(rng.next_unit());
        float P[C];
        float run = 0.0f;
#pragma unroll
        for (int c = 0; c < C; c += 4) {
          const float4 y = *reinterpret_cast<const float4*>(csum + cs_idx(lane, c));
          run += y.x;
          P[c] = run;
          run += y.y;
          P[c + 1] = run;
          run += y.z;
          P[c + 2] = run;
          run += y.w;
          P[c + 3] = run;
        }
        const float total = run;
        const float uf = u01 * total;
        const float mg = a.screen_margin * total;
        int k = -1;
        if (uf < total && total > 0x1p-90f && total < 0x1p100f) {
          int cs = C - 1;
          float lo = 0.0f;
#pragma unroll
          for (int c = C - 1; c >= 0; --c)
            if (uf < P[c]) cs = c;
#pragma unroll
          for (int c = 0; c < C - 1; ++c)
            if (c < cs) lo = P[c];
          // chunk cs = lane cs / R's round cs % R (phys32 layout)
          const int og = cs / R, orr = cs - og * R;
          const Oct p = ldg256f(a.phiT32 + static_cast<std::size_t>(wl) * a.Kp32 + CW * (orr * G + og));
          const float4 y0 = *reinterpret_cast<const float4*>(thf + og * KLP + CW * orr);
          const float4 y1 = *reinterpret_cast<const float4*>(thf + og * KLP + CW * orr + 4);
          const float tv[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
          float acc = lo, prev = lo;
          int j = -1;
#pragma unroll
          for (int jj = 0; jj < CW; ++jj) {
            const float nx = __fmaf_rn(tv[jj], p.v[jj], acc);
            if (j < 0) {
              if (uf < nx) {
                j = jj;
                prev = acc;
              }
              acc = nx;
            }
          }
          const int kk = CW * cs + j;
          if (j >= 0 && kk < a.K && uf - prev >= mg && acc - uf >= mg) k = kk;
        }
        if (k >= 0) {
          a.z[t] = k;
          atomicAdd(&a.nkw[static_cast<std::size_t>(wl) * a.Kp + k], 1);
          atomicAdd(&cnt_s[k], 1);  // shared: flushed to nmk once per unit
        } else {
          const int slot = atomicAdd(a.fq_len, 1);  // fp64 redraw (zfallback_kernel)
          a.fq[slot] = make_int2(static_cast<int>(t), static_cast<int>(m));
        }
      }
      __syncwarp();
    }
    if constexpr (WU) __syncwarp();
    else __syncthreads();
    for (int k = tid_u; k < a.K; k += nthr_u) {
      const int n = cnt_s[k];
      if (n) atomicAdd(&a.nmk[m * a.K + k], n);
    }
  }
}

// fp64 product-form draw for the tokens the screen could not decide (~2K * 2^-16
// of them): one warp per queued token.  Lane l owns the contiguous candidates
// [l*c, (l+1)*c), c = ceil(K/32); warp scan of the lane sums, the owner rescans
// its chunk (the reference's candidate order and u = next_unit * total rule,
// dist.cpp:202-215).  Tokens whose product weights underflow take the sequential
// log-space draw.  The products (theta/S) * g are formed in candidate order by the
// whole warp (coalesced row loads) into the warp's shared-memory slice, one pad
// double per 32 (lane-contiguous reads then hit distinct banks); the sums read them
// in the lane-contiguous order (the same additions as reading the rows directly,
// which cost 32 L1 wavefronts per load: ncu, 1B, L1TEX 98 %, 166 ms).
constexpr int kFallbackThreads = 128;

__host__ __device__ constexpr int fallback_stride(int K) { return K + (K >> 5) + 1; }

// kStage = false (K <= 128: <= 4 candidates per lane): the lanes read the rows directly.
template <bool kStage>
__global__ void __launch_bounds__(kFallbackThreads) zfallback_kernel(LdaArgs a, const std::int64_t* iter_p, int* err) {
  extern __shared__ double fprod[];
  pdl_wait();
  pdl_trigger();
  const std::int64_t iter = *iter_p;
  const int lane = threadIdx.x & 31;
  double* prod = fprod + (threadIdx.x >> 5) * fallback_stride(a.K);
  const int n = *a.fq_len;
  const int c = (a.K + 31) / 32;
  const int k0 = min(a.K, lane * c), k1 = min(a.K, k0 + c);
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    const int2 q = a.fq[i];
    const std::int64_t t = q.x, m = q.y;
    const int wv = a.w[t];
    const double* thg = a.theta + m * a.K;
    const double* row = a.phiT + static_cast<std::size_t>(wv) * a.Kp;
    Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + t)),
                    static_cast<std::uint64_t>(iter)));
    const double u01 = rng.next_unit();
    auto term = [&](int k) { return kStage ? prod[k + (k >> 5)] : (thg[k] / a.S[k]) * row[k]; };
    if constexpr (kStage) {
      __syncwarp();  // the previous token's reads of prod are done
      // 8 candidates per lane in flight (24 loads) before the divisions and stores: the
      // loop one load round trip at a time took ~60 us per token at 1B
      for (int kb = lane; kb < a.K; kb += 32 * 8) {
        double th[8], sv[8], rw[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = kb + 32 * j;
          if (k < a.K) {
            th[j] = __ldg((a.thS ? a.thS + m * a.K : thg) + k);
            sv[j] = a.thS ? 1.0 : __ldg(a.S + k);
            rw[j] = __ldg(row + k);
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = kb + 32 * j;
          if (k < a.K) prod[k + (k >> 5)] = (a.thS ? th[j] : th[j] / sv[j]) * rw[j];
        }
      }
      __syncwarp();
    }
    double own = 0.0;
    for (int k = k0; k < k1; ++k) own += term(k);
    double inc = own;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    double start = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) start = 0.0;
    const double total = __shfl_sync(0xffffffffu, inc, 31);
    int pick = -1;
    if (total > 0x1p-1000 && isfinite(total)) {
      const double u = u01 * total;
      int cand = (lane == 31 && !(u < inc)) ? a.K - 1 : -1;  // past-the-end: K - 1
      if (start <= u && u < inc && k0 < k1) {
        double acc = start;
        cand = k1 - 1;
        for (int k = k0; k < k1; ++k) {
          acc += term(k);
          if (u < acc) {
            cand = k;
            break;
          }
        }
      }
      pick = __reduce_max_sync(0xffffffffu, cand);
    } else if (lane == 0) {
      // log-space, sequential (draw_from_log_weights)
      double mx = -INFINITY;
      for (int k = 0; k < a.K; ++k) {
        const double x = thg[k], g = row[k] / a.S[k];
        mx = fmax(mx, (x > 0.0 ? log(x) : -INFINITY) + (g > 0.0 ? log(g) : -INFINITY));
      }
      if (isfinite(mx)) {
        double tot = 0.0;
        for (int k = 0; k < a.K; ++k) {
          const double x = thg[k], g = row[k] / a.S[k];
          tot += exp(((x > 0.0 ? log(x) : -INFINITY) + (g > 0.0 ? log(g) : -INFINITY)) - mx);
        }
        const double u = u01 * tot;
        double acc = 0.0;
        pick = a.K - 1;
        for (int k = 0; k < a.K; ++k) {
          const double x = thg[k], g = row[k] / a.S[k];
          acc += exp(((x > 0.0 ? log(x) : -INFINITY) + (g > 0.0 ? log(g) : -INFINITY)) - mx);
          if (u < acc) {
            pick = k;
            break;
          }
        }
      }
    }
    pick = __shfl_sync(0xffffffffu, pick, 0);
    if (lane == 0) {
      if (pick < 0) {
        atomicOr(err, kErrDomain);
      } else {
        a.z[t] = pick;
        atomicAdd(&a.nkw[static_cast<std::size_t>(wv) * a.Kp + pick], 1);
        atomicAdd(&a.nmk[m * a.K + pick], 1);
      }
    }
  }
}

// The log-space draw (draw_from_log_weights, dist.cpp:202-215) for the tokens the fp32
// screen could not decide in the exact-weights mode: w_k = log theta_k + log phi_k (the
// values the logphiT table would hold), mx = max, exp(w_k - mx) summed in the lane-contiguous order of
// zfallback_kernel, u = next_unit * total, the owner rescans. The screen's decisions are
// the real-number ones (margin >> the ~1e-14 relative error of the fp64 log-space sums),
// so screened tokens get the log-space draw's topic too.
__global__ void __launch_bounds__(kFallbackThreads) zfallback_log_kernel(LdaArgs a, const std::int64_t* iter_p, int* err) {
  extern __shared__ double fw_s[];
  pdl_wait();
  pdl_trigger();
  const std::int64_t iter = *iter_p;
  const int lane = threadIdx.x & 31;
  double* fw = fw_s + (threadIdx.x >> 5) * fallback_stride(a.K);
  const int n = *a.fq_len;
  const int c = (a.K + 31) / 32;
  const int k0 = min(a.K, lane * c), k1 = min(a.K, k0 + c);
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    const int2 q = a.fq[i];
    const std::int64_t t = q.x, m = q.y;
    const int wv = a.w[t];
    const double* thg = a.theta + m * a.K;
    const double* prow = a.phiT + static_cast<std::size_t>(wv) * a.Kp;  // g (phi = g / S)
    Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + t)),
                    static_cast<std::uint64_t>(iter)));
    const double u01 = rng.next_unit();
    __syncwarp();
    double lmx = -INFINITY;
    for (int k = lane; k < a.K; k += 32) {
      const double x = thg[k], p = prow[k] / a.S[k];  // phi exactly as phi_norm_kernel forms it
      const double w = (x > 0.0 ? log(x) : -INFINITY) + (p > 0.0 ? log(p) : -INFINITY);  // = log theta + logphiT
      fw[k + (k >> 5)] = w;
      lmx = fmax(lmx, w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmx = fmax(lmx, __shfl_xor_sync(0xffffffffu, lmx, o));
    __syncwarp();
    int pick = -1;
    if (isfinite(lmx)) {
      double own = 0.0;
      for (int k = k0; k < k1; ++k) own += exp(fw[k + (k >> 5)] - lmx);
      double inc = own;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
      }
      double start = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) start = 0.0;
      const double total = __shfl_sync(0xffffffffu, inc, 31);
      const double u = u01 * total;
      int cand = (lane == 31 && !(u < inc)) ? a.K - 1 : -1;  // past-the-end: K - 1
      if (start <= u && u < inc && k0 < k1) {
        double acc = start;
        cand = k1 - 1;
        for (int k = k0; k < k1; ++k) {
          acc += exp(fw[k + (k >> 5)] - lmx);
          if (u < acc) {
            cand = k;
            break;
          }
        }
      }
      pick = __reduce_max_sync(0xffffffffu, cand);
    }
    if (lane == 0) {
      if (pick < 0) {
        atomicOr(err, kErrDomain);
      } else {
        a.z[t] = pick;
        atomicAdd(&a.nkw[static_cast<std::size_t>(wv) * a.Kp + pick], 1);
        atomicAdd(&a.nmk[m * a.K + pick], 1);
      }
    }
  }
}

// One CTA per work unit (a chunk of <= kChunk tokens of one document).
template <int G, int R, bool EXACT, bool TR>
__global__ void __launch_bounds__(kZThreads) zstep_kernel(LdaArgs a, const std::int64_t* iter_p, int* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* th = reinterpret_cast<double*>(smem_raw);  // [Kp]
  double* lth = th + a.Kp;                            // [Kp]
  const std::int64_t iter = *iter_p;
  const int Rr = a.Kp / (4 * G);
  const int gid = threadIdx.x / G, gl = threadIdx.x & (G - 1);
  constexpr int kGroups = kZThreads / G;

  for (std::int64_t u = blockIdx.x; u < a.n_units; u += gridDim.x) {
    const std::int64_t m = a.units[u * 3], t0 = a.units[u * 3 + 1], t1 = a.units[u * 3 + 2];
    const double* thg = a.theta + m * a.K;
    for (int k = threadIdx.x; k < a.Kp; k += blockDim.x) {
      const double x = k < a.K ? thg[k] : 0.0;
      // phiT holds the unnormalised gamma row g (phi = g / S[k]); fold 1/S into the
      // theta operand: weight = (theta / S) * g.
      th[k] = k < a.K ? x / a.S[k] : 0.0;
      lth[k] = x > 0.0 ? log(x) : -INFINITY;
    }
    __syncthreads();
    // The lane's theta (log theta when EXACT) for its candidates, held in registers
    // across the unit's tokens.
    ThetaSrc<R, TR> tq;
    if constexpr (TR) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = 4 * (r * G + gl);
        const double* src = EXACT ? lth : th;
        if (r < Rr) {
          const double2 t0 = *reinterpret_cast<const double2*>(src + k);
          const double2 t1 = *reinterpret_cast<const double2*>(src + k + 2);
          tq.q[r] = Quad{t0.x, t0.y, t1.x, t1.y};
        } else {
          tq.q[r] = Quad{0.0, 0.0, 0.0, 0.0};
        }
      }
    } else {
      tq.p = EXACT ? lth : th;
    }
    int* cnt = a.nmk + m * a.K;
    int wv_next = t0 + gid < t1 ? __ldg(a.w + t0 + gid) : 0;
    for (std::int64_t base = t0; base < t1; base += kGroups) {
      const std::int64_t t = base + gid;
      const bool valid = t < t1;
      const int wv = wv_next;
      wv_next = t + kGroups < t1 ? __ldg(a.w + t + kGroups) : 0;
      const double* row = a.phiT + static_cast<std::size_t>(wv) * a.Kp;
      const double* lrow = EXACT ? a.logphiT + static_cast<std::size_t>(wv) * a.Kp : nullptr;
      // keyed(seed, 3, var_z, t, iter) with the first three folds hoisted.
      Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + t)),
                      static_cast<std::uint64_t>(iter)));
      const double u01 = rng.next_unit();
      int k = draw_topic<G, R, EXACT>(tq, row, lrow, a.K, Rr, u01);
      if (!EXACT && k < 0) k = draw_topic_logspace<G>(lth, row, a.K, u01);
      if (valid && gl == 0) {
        if (k < 0) {
          atomicOr(err, kErrDomain);
        } else {
          a.z[t] = k;
          atomicAdd(&a.nkw[static_cast<std::size_t>(wv) * a.Kp + k], 1);
          atomicAdd(&cnt[k], 1);
        }
      }
    }
    __syncthreads();
  }
}

// w- and z-factors of the log-joint from the counts the z-step just produced:
// sum_t log phi[z_t, w_t] = sum_{v,k} n[v,k] log phi[k,v]  (blocks < nb_phi) and
// sum_t log theta[d_t, z_t] = sum_{d,k} n[d,k] log theta[d,k]  (the other blocks),
// over this rank's tokens; fixed-order partials.  FINAL (single GPU): the last
// block to finish (atomic ticket) also forms the log-joint from all partials in
// fixed order, as reduce_kernel<false, true> does -- one launch less per sweep.
template <bool FINAL>
__device__ __forceinline__ void loglik_finish(const LdaArgs& a, const Outputs& o, int advance, double* scratch) {
  if constexpr (FINAL) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int t = atomicAdd(a.ticket2, 1);
      last = t == static_cast<int>(gridDim.x) - 1;
      if (last) *a.ticket2 = 0;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // every block's partials, up to 4 per thread and operand in flight (one L2
    // round trip for nbw <= 1024), then one combined block reduction
    double s[4] = {0.0, 0.0, 0.0, 0.0};  // theta, z, w pieces; phi factor
    for (int b0 = threadIdx.x; b0 < a.nbw; b0 += 4 * blockDim.x) {
      double t4[4], z4[4], w4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int b = b0 + j * blockDim.x;
        t4[j] = b < a.nbw ? __ldcg(&a.ttpart[b]) : 0.0;
        z4[j] = b < a.nbw ? __ldcg(&a.zpart[b]) : 0.0;
        w4[j] = b < a.nbw ? __ldcg(&a.wpart[b]) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s[0] += t4[j];
        s[1] += z4[j];
        s[2] += w4[j];
      }
    }
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) s[3] += __ldcg(&a.phi_term[k]);
    block_sum_n<4>(s, scratch);
    const double s0 = s[0], s1 = s[1], s2 = s[2], f = s[3];
    if (a.red_only) {
      if (threadIdx.x == 0) {
        a.red[0] = s0;
        a.red[1] = s1;
        a.red[2] = s2;
      }
      return;
    }
    if (threadIdx.x == 0) {
      const double lj = ((f + s0) + s1) + s2;
      const std::int64_t it = *o.iter;
      o.lj[it & (kRing - 1)] = lj;
      o.acc[it & (kRing - 1)] = 0;
      if (advance) *o.iter = it + 1;
    }
  }
}

// wterm_kernel: 4-cell vectors per thread in flight (1..4 measured equal, r01 v52: the
// kernel is bound by its launch and last-block tail, not its loads)
constexpr int kWU = 2;

// Counted-cell terms n (log x - s) of one warp iteration: each lane holds S slots
// (n = 0: nothing to add); the nonzero slots are compacted through a per-warp shared
// buffer (warp prefix scan of the lanes' counts) and the logs then run at full warp
// width -- ~40 % of the NIPS cells are counted, and per-slot `if (n) log(...)` blocks
// ran every log pass for ~10 of 32 lanes (ncu r02: 60 % of wterm's instructions).
// Item order depends only on the data: the sum is deterministic.
template <int S>
__device__ __forceinline__ double counted_log_terms(const int (&nn)[S], const double (&xx)[S], const double (&ss)[S],
                                                    int* bn, double* bx, double* bs) {
  const int lane = threadIdx.x & 31;
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < S; ++i) cnt += nn[i] != 0;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int p = incl - cnt;
#pragma unroll
  for (int i = 0; i < S; ++i) {
    if (nn[i]) {
      bn[p] = nn[i];
      bx[p] = xx[i];
      bs[p] = ss[i];
      ++p;
    }
  }
  __syncwarp();
  double acc = 0.0;
  for (int i = lane; i < total; i += 32) acc += static_cast<double>(bn[i]) * (log(bx[i]) - bs[i]);  // log(0) = -inf
  __syncwarp();
  return acc;
}

template <bool FINAL>
__global__ void __launch_bounds__(256, 4) wterm_kernel(LdaArgs a, Outputs o, int advance) {
  __shared__ double scratch[4 * 32];
  __shared__ int cb_n[8][32 * 4 * kWU];
  __shared__ double cb_x[8][32 * 4 * kWU], cb_s[8][32 * 4 * kWU];
  pdl_wait();
  const int wib = threadIdx.x >> 5;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  const std::int64_t g0 = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // w-factor over the topic-word cells, static cell -> thread assignment (deterministic).
  // The padded [V][Kp] arrays are read as 4-cell vectors (Kp % 4 == 0: a vector never
  // crosses a row; padding cells have n = 0 and logS is zero-padded to Kp), two vectors
  // per thread in flight; the counted cells' logs compacted per warp.
  double accw = 0.0;
  if (a.logg_valid) {
    const std::int64_t nvec = static_cast<std::int64_t>(a.V) * a.Kp / 4;
    const bool narrow = nvec < (std::int64_t{1} << 29);  // 4 * nvec fits 31 bits
    const int4* n4 = reinterpret_cast<const int4*>(a.nkw);
    const double2* l2 = reinterpret_cast<const double2*>(a.phiT);  // g (the pool stores g, not log g)
    for (std::int64_t c0 = g0; __any_sync(0xffffffffu, c0 < nvec); c0 += kWU * stride) {
      int nn[4 * kWU];
      double xx[4 * kWU], ss[4 * kWU];
#pragma unroll
      for (int j = 0; j < kWU; ++j) {
        const std::int64_t c = c0 + j * stride;
        int4 n = make_int4(0, 0, 0, 0);
        double2 la = make_double2(1.0, 1.0), lb = make_double2(1.0, 1.0);
        if (c < nvec) {
          n = n4[c];
          la = l2[2 * c];
          lb = l2[2 * c + 1];
        }
        const int k0 = c >= nvec ? 0
                       : narrow ? static_cast<int>(static_cast<unsigned>(4 * c) % static_cast<unsigned>(a.Kp))
                                : static_cast<int>((4 * c) % a.Kp);
        nn[4 * j] = n.x, nn[4 * j + 1] = n.y, nn[4 * j + 2] = n.z, nn[4 * j + 3] = n.w;
        xx[4 * j] = la.x, xx[4 * j + 1] = la.y, xx[4 * j + 2] = lb.x, xx[4 * j + 3] = lb.y;
        // (logS loaded unconditionally -- padded to Kp -- so its load issues with n's
        // instead of after it)
#pragma unroll
        for (int q = 0; q < 4; ++q) ss[4 * j + q] = __ldg(&a.logS[k0 + q]);
      }
      accw += counted_log_terms<4 * kWU>(nn, xx, ss, cb_n[wib], cb_x[wib], cb_s[wib]);  // log phi = log g - log S
    }
  } else {
    for (std::int64_t c = g0; c < static_cast<std::int64_t>(a.V) * a.K; c += stride) {
      const std::int64_t v = c / a.K;
      const int k = static_cast<int>(c - v * a.K);
      const std::size_t i = static_cast<std::size_t>(v) * a.Kp + k;
      const int n = a.nkw[i];
      if (n) {
        const double p = a.phiT[i] / a.S[k];  // phi = g / S (S = 1 once normalised)
        accw += static_cast<double>(n) * (p > 0.0 ? log(p) : -INFINITY);
      }
    }
  }
  // z-factor over the doc-topic cells: the flat [Ml][K] arrays as 4-cell vectors
  // (cudaMalloc bases are 256-byte aligned), counted cells compacted as above, the
  // ragged tail scalar
  double accz = 0.0;
  const std::int64_t ncz = a.Ml * a.K, nvz = ncz / 4;
  const int4* m4 = reinterpret_cast<const int4*>(a.nmk);
  const double2* t2 = reinterpret_cast<const double2*>(a.theta);
  for (std::int64_t c = g0; __any_sync(0xffffffffu, c < nvz); c += stride) {
    int nn[4] = {0, 0, 0, 0};
    double xx[4] = {1.0, 1.0, 1.0, 1.0}, ss[4] = {0.0, 0.0, 0.0, 0.0};
    if (c < nvz) {
      const int4 n = m4[c];
      const double2 x = t2[2 * c], y = t2[2 * c + 1];
      nn[0] = n.x, nn[1] = n.y, nn[2] = n.z, nn[3] = n.w;
      xx[0] = x.x, xx[1] = x.y, xx[2] = y.x, xx[3] = y.y;
    }
    accz += counted_log_terms<4>(nn, xx, ss, cb_n[wib], cb_x[wib], cb_s[wib]);
  }
  if (g0 < ncz - 4 * nvz) {
    const int n = a.nmk[4 * nvz + g0];
    const double x = a.theta[4 * nvz + g0];
    if (n) accz += static_cast<double>(n) * (x > 0.0 ? log(x) : -INFINITY);
  }
  // the theta factor's per-document pieces, spread over the grid (single-rank path:
  // the last block then reads nbw partials instead of Ml)
  double acct = 0.0;
  if constexpr (FINAL)
    for (std::int64_t m = g0; m < a.Ml; m += stride) acct += a.tpart[m];
  double v[3] = {accw, accz, acct};
  block_sum_n<3>(v, scratch);
  if (threadIdx.x == 0) {
    a.wpart[blockIdx.x] = v[0];
    a.zpart[blockIdx.x] = v[1];
    if (FINAL) a.ttpart[blockIdx.x] = v[2];
  }
  loglik_finish<FINAL>(a, o, advance, scratch);
}

// Log-joint pieces of the current state without sampling (Engine::eval_log_joint).
__global__ void __launch_bounds__(256) doc_eval_kernel(LdaArgs a, int* err) {
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
      const double pp = a.phiT[static_cast<std::size_t>(a.w[t]) * a.Kp + k] / a.S[k];
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

// red[0..2] = F_theta, F_z, F_w of this rank (fixed order).  FINAL (single GPU):
// also the log-joint, as finalize_kernel.
template <bool EVAL, bool FINAL = false>
__global__ void reduce_kernel(LdaArgs a, Outputs o = Outputs{}, int advance = 0) {
  __shared__ double scratch[32];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  if (EVAL) {
    for (std::int64_t m = threadIdx.x; m < a.Ml; m += blockDim.x) {
      s0 += a.doc_part[m * 3 + 0];
      s1 += a.doc_part[m * 3 + 1];
      s2 += a.doc_part[m * 3 + 2];
    }
  } else {
    for (std::int64_t m = threadIdx.x; m < a.Ml; m += blockDim.x) s0 += a.tpart[m];
    for (int b = threadIdx.x; b < a.nbw; b += blockDim.x) s1 += a.zpart[b];
    for (int b = threadIdx.x; b < a.nbw; b += blockDim.x) s2 += a.wpart[b];
  }
  s0 = block_sum(s0, scratch);
  s1 = block_sum(s1, scratch);
  s2 = block_sum(s2, scratch);
  if (threadIdx.x == 0) {
    a.red[0] = s0;
    a.red[1] = s1;
    a.red[2] = s2;
  }
  if constexpr (FINAL) {
    double f = 0.0;
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) f += a.phi_term[k];
    f = block_sum(f, scratch);
    if (threadIdx.x == 0) {
      const double lj = ((f + s0) + s1) + s2;
      const std::int64_t it = *o.iter;
      o.lj[it & (kRing - 1)] = lj;
      o.acc[it & (kRing - 1)] = 0;
      if (advance) *o.iter = it + 1;
    }
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

// Doc-topic counts of the current z (the theta block's sufficient statistics).
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

__global__ void i32_check_kernel(const int* v, std::int64_t n, int hi, int* err) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    if (v[i] < 0 || v[i] >= hi) atomicOr(err, kErrBin);
}

// z write-back: int64 staging for the store and the copy the next speculative
// sweep_store compares the store with (zprev)
__global__ void z_writeback_kernel(const int* in, std::int64_t* out, int* keep, std::int64_t n) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    const int v = in[i];
    out[i] = v;
    keep[i] = v;
  }
}

// Speculative sweep_store: did the caller's store (uploaded to `up`) differ from the
// state the sweep started from (`prev`)?
__global__ void spec_check_kernel(const std::int64_t* up, const int* prev, std::int64_t n, int* flag) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  bool diff = false;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    diff |= up[i] != static_cast<std::int64_t>(prev[i]);
  if (__any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) *flag = 1;
}

__global__ void i32_to_i64_kernel(const int* in, std::int64_t* out, std::int64_t n) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    out[i] = in[i];
}

// phiT [V][Kp] <-> phi [K][V] (reference layout), tiled through shared memory;
// with `colscale` (download), out = in / colscale[column of in] = g / S.
__global__ void transpose_kernel(const double* in, double* out, int rows, int cols, int ld_in,
                                 int ld_out, const double* colscale = nullptr) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols)
      tile[i][threadIdx.x] = colscale ? in[static_cast<std::size_t>(r) * ld_in + c] / colscale[c]
                                      : in[static_cast<std::size_t>(r) * ld_in + c];
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

// Long Dirichlet rows (phi's V columns per topic) drawn in parallel, same values.
// A row's gammas come from ONE stream whose counters each gamma consumes in a
// data-dependent number (Marsaglia-Tsang rejections), so the start of gamma j is
// known only after gamma j-1. The stream is counter-based (any position can be
// entered directly), so the row's counter range is cut into segments of kPriorSeg:
//   walk:  from each of kPriorCand candidate entries s, s+1, .. of every segment,
//          count the gammas that start inside it and the first start beyond it;
//   link:  per row, left to right: the true entry of segment i is segment i-1's exit;
//          it is a candidate (or the second start of one) except after a rare long
//          rejection run, where this thread walks the segment itself;
//   draw:  every segment redraws its gammas from its true entry into their columns;
//   sum:   per row, the left-to-right sum (draw_dirichlet's order), then normalise.
constexpr int kPriorSeg = 512, kPriorCand = 4;

__global__ void prior_seg_walk_kernel(std::int64_t rows, int nseg, double conc, std::uint64_t seed, int var,
                                      std::int64_t row_base, int* cnt, std::int64_t* exit_pos,
                                      std::int64_t* second) {
  const std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (i >= rows * nseg * kPriorCand) return;
  const int cand = static_cast<int>(i % kPriorCand);
  const std::int64_t rs = i / kPriorCand, r = rs / nseg;
  const std::int64_t seg = rs % nseg, end = (seg + 1) * kPriorSeg;
  Stream s(keyed(seed, kInit, static_cast<std::uint64_t>(var), static_cast<std::uint64_t>(row_base + r)),
           static_cast<std::uint64_t>(seg * kPriorSeg + cand));
  int c = 0;
  std::int64_t sec = -1;
  while (static_cast<std::int64_t>(s.counter) < end) {
    skip_gamma(s, conc);
    if (++c == 1) sec = static_cast<std::int64_t>(s.counter);
  }
  cnt[i] = c;
  exit_pos[i] = static_cast<std::int64_t>(s.counter);
  second[i] = sec;
}

__global__ void prior_seg_link_kernel(std::int64_t rows, int cols, int nseg, double conc, std::uint64_t seed,
                                      int var, std::int64_t row_base, const int* cnt, const std::int64_t* exit_pos,
                                      const std::int64_t* second, std::int64_t* entry, int* first_col) {
  const std::int64_t r = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  const std::uint64_t key = keyed(seed, kInit, static_cast<std::uint64_t>(var), static_cast<std::uint64_t>(row_base + r));
  std::int64_t t = 0;
  int col = 0;
  for (int seg = 0; seg < nseg; ++seg) {
    const std::int64_t rs = r * nseg + seg;
    entry[rs] = t;
    first_col[rs] = col;
    if (col >= cols || seg == nseg - 1) continue;  // the last segment runs open-ended
    const std::int64_t s0 = static_cast<std::int64_t>(seg) * kPriorSeg, d = t - s0;
    const std::int64_t* ex = exit_pos + rs * kPriorCand;
    const int* cn = cnt + rs * kPriorCand;
    int hit = -1, skip = 0;
    if (d < kPriorCand) {
      hit = static_cast<int>(d);
    } else {
      for (int j = 0; j < kPriorCand; ++j)
        if (second[rs * kPriorCand + j] == t) hit = j, skip = 1;
    }
    if (hit >= 0 && cn[hit] > skip) {
      col += cn[hit] - skip;
      t = ex[hit];
    } else {
      Stream s(key, static_cast<std::uint64_t>(t));
      while (static_cast<std::int64_t>(s.counter) < s0 + kPriorSeg) {
        skip_gamma(s, conc);
        ++col;
      }
      t = static_cast<std::int64_t>(s.counter);
    }
  }
}

__global__ void prior_seg_draw_kernel(double* out, std::int64_t rows, int cols, int nseg, std::int64_t ld_row,
                                      std::int64_t ld_col, double conc, std::uint64_t seed, int var,
                                      std::int64_t row_base, const std::int64_t* entry, const int* first_col) {
  const std::int64_t rs = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x;
  if (rs >= rows * nseg) return;
  const std::int64_t r = rs / nseg;
  const int seg = static_cast<int>(rs % nseg);
  int col = first_col[rs];
  if (col >= cols) return;
  const std::int64_t end = seg == nseg - 1 ? INT64_MAX : static_cast<std::int64_t>(seg + 1) * kPriorSeg;
  Stream s(keyed(seed, kInit, static_cast<std::uint64_t>(var), static_cast<std::uint64_t>(row_base + r)),
           static_cast<std::uint64_t>(entry[rs]));
  while (col < cols && static_cast<std::int64_t>(s.counter) < end)
    out[r * ld_row + static_cast<std::int64_t>(col++) * ld_col] = draw_gamma(s, conc);
}

// Left-to-right row sums (draw_dirichlet's order) or running sums (kCum, in place), one
// warp per row: the warp stages 256-column tiles through shared memory, lane 0 adds them
// in order (the roundings of a sequential loop), the warp writes running sums back.
constexpr int kScanTile = 256, kScanWarps = 4;

template <bool kCum>
__global__ void __launch_bounds__(32 * kScanWarps) row_scan_kernel(double* x, std::int64_t rows, int cols,
                                                                     std::int64_t ld_row, std::int64_t ld_col,
                                                                     double* sums) {
  __shared__ double tile[kScanWarps][kScanTile];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const std::int64_t r = blockIdx.x * static_cast<std::int64_t>(kScanWarps) + wi;
  if (r >= rows) return;
  double* row = x + r * ld_row;
  double* tl = tile[wi];
  double acc = 0.0;
  for (int c0 = 0; c0 < cols; c0 += kScanTile) {
    const int n = min(kScanTile, cols - c0);
    for (int j = lane; j < n; j += 32) tl[j] = row[static_cast<std::int64_t>(c0 + j) * ld_col];
    __syncwarp();
    if (lane == 0) {
#pragma unroll 8
      for (int j = 0; j < n; ++j) {
        acc += tl[j];
        if (kCum) tl[j] = acc;
      }
    }
    __syncwarp();
    if (kCum)
      for (int j = lane; j < n; j += 32) row[static_cast<std::int64_t>(c0 + j) * ld_col] = tl[j];
    __syncwarp();
  }
  if (!kCum && lane == 0) sums[r] = acc;
}

__global__ void prior_row_norm_kernel(double* out, std::int64_t rows, int cols, std::int64_t ld_row,
                                      std::int64_t ld_col, const double* sums) {
  const std::int64_t n = rows * cols;
  for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
    // consecutive threads on consecutive rows when the rows are the inner dimension
    const std::int64_t r = ld_row == 1 ? i % rows : i / cols, c = ld_row == 1 ? i / rows : i % cols;
    out[r * ld_row + c * ld_col] /= sums[r];
  }
}

// z ~ Categorical(theta[d]) (draw_categorical, dist.cpp:183-191): the reference scans
// acc += theta[k] until u < acc. The running sums are formed once per document, left to
// right by one thread (the same roundings), in shared memory; each token then binary-
// searches the first k with u < acc[k] (acc is non-decreasing: the same pick as the scan,
// K-1 when u is beyond the last sum). kSmem = false: K too large for shared memory, scan.
__device__ __forceinline__ void doc_cumsum_smem(const double* th, int K, double* cum) {
  for (int k = threadIdx.x; k < K; k += blockDim.x) cum[k] = th[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
#pragma unroll 8
    for (int k = 0; k < K; ++k) {
      acc += cum[k];
      cum[k] = acc;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int first_above(const double* cum, int n, double u) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (u < cum[mid])
      hi = mid;
    else
      lo = mid + 1;
  }
  return lo;
}

__device__ __forceinline__ int scan_pick(const double* th, int K, double u) {
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    acc += th[k];
    if (u < acc) return k;
  }
  return K - 1;
}

constexpr int kDocCumMax = 2048;  // doubles of running sums in shared memory (the z-step's K limit)

template <bool kSmem>
__global__ void prior_z_kernel(LdaArgs a, std::uint64_t seed) {
  extern __shared__ double cum[];
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const double* th = a.theta + m * a.K;
    if (kSmem) doc_cumsum_smem(th, a.K, cum);
    for (std::int64_t t = a.off[m] + threadIdx.x; t < a.off[m + 1]; t += blockDim.x) {
      Stream s(keyed(seed, kInit, static_cast<std::uint64_t>(a.var_z),
                     static_cast<std::uint64_t>(a.tok_base + t)));
      const double u = s.next_unit();
      a.z[t] = kSmem ? first_above(cum, a.K, u) : scan_pick(th, a.K, u);
    }
    if (kSmem) __syncthreads();
  }
}

// Device corpus generator following gen_lda's process (gen.cpp:21-60): true phi
// rows ~ Dir(phi_conc), theta_d ~ Dir(theta_conc), z ~ Cat(theta_d), w ~ Cat(phi_z).
// Word draws use a per-topic cumulative table + binary search (not the reference's
// O(V) scan) and counter streams per token (not one serial stream).
template <bool kSmem>
__global__ void gen_tokens_kernel(LdaArgs a, const double* cum_phi /*[K][V]*/, const double* theta_true,
                                  std::uint64_t seed) {
  extern __shared__ double cum[];
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const double* th = theta_true + m * a.K;
    if (kSmem) doc_cumsum_smem(th, a.K, cum);
    for (std::int64_t t = a.off[m] + threadIdx.x; t < a.off[m + 1]; t += blockDim.x) {
      Stream s(keyed(seed, 0xDA7A, 1, static_cast<std::uint64_t>(a.tok_base + t)));
      const double u = s.next_unit();
      const int k = kSmem ? first_above(cum, a.K, u) : scan_pick(th, a.K, u);
      const double* cp = cum_phi + static_cast<std::size_t>(k) * a.V;
      const_cast<int*>(a.w)[t] = first_above(cp, a.V, s.next_unit() * cp[a.V - 1]);
    }
    if (kSmem) __syncthreads();
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

// prior_init's Dirichlet rows: thread per row for short rows (theta), the segmented
// walk above for long ones (phi's V columns); BNMC_PRIOR_SERIAL=1 forces thread per row.
// Returns after the rows are written (the walk's scratch is freed here).
void dirichlet_rows(double* out, std::int64_t rows, int cols, std::int64_t ld_row, std::int64_t ld_col, double conc,
                    std::uint64_t seed, int var, std::int64_t row_base, cudaStream_t st) {
  const char* e = std::getenv("BNMC_PRIOR_SERIAL");
  const bool serial = (e && std::string(e) != "0") || cols < 4 * kPriorSeg || rows > 148 * 64 || !(conc > 0.0);
  if (serial) {
    prior_rows_kernel<<<blocks_for(rows, 64), 64, 0, st>>>(out, rows, cols, ld_row, ld_col, conc, seed, var, row_base);
    BNMC_CUDA(cudaGetLastError());
    return;
  }
  // counters per gamma: 3 per attempt (+2 per v <= 0 retry), +1 for the shape < 1 boost;
  // over-estimated (a short estimate only lengthens the open-ended last segment)
  const double per = conc < 1.0 ? 4.4 : 3.4;
  const int nseg = static_cast<int>((per * cols + 256) / kPriorSeg) + 1;
  const std::int64_t ns = rows * nseg;
  DevBuf<int> cnt, first_col;
  DevBuf<std::int64_t> exit_pos, second, entry;
  DevBuf<double> sums;
  cnt.alloc(ns * kPriorCand);
  exit_pos.alloc(ns * kPriorCand);
  second.alloc(ns * kPriorCand);
  entry.alloc(ns);
  first_col.alloc(ns);
  sums.alloc(rows);
  prior_seg_walk_kernel<<<blocks_for(ns * kPriorCand, 128), 128, 0, st>>>(rows, nseg, conc, seed, var, row_base,
                                                                          cnt.p, exit_pos.p, second.p);
  prior_seg_link_kernel<<<blocks_for(rows, 32), 32, 0, st>>>(rows, cols, nseg, conc, seed, var, row_base, cnt.p,
                                                              exit_pos.p, second.p, entry.p, first_col.p);
  prior_seg_draw_kernel<<<blocks_for(ns, 128), 128, 0, st>>>(out, rows, cols, nseg, ld_row, ld_col, conc, seed, var,
                                                              row_base, entry.p, first_col.p);
  row_scan_kernel<false><<<blocks_for(rows, kScanWarps), 32 * kScanWarps, 0, st>>>(out, rows, cols, ld_row, ld_col,
                                                                                    sums.p);
  prior_row_norm_kernel<<<148 * 8, 256, 0, st>>>(out, rows, cols, ld_row, ld_col, sums.p);
  BNMC_CUDA(cudaGetLastError());
  BNMC_CUDA(cudaStreamSynchronize(st));
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
    // z-step tile: the smallest group width G whose rounds fit R <= 8 registers.
    G_ = 32;
    for (int g : {4, 8, 16, 32}) {
      if ((K_ + 4 * g - 1) / (4 * g) <= 8) {
        G_ = g;
        break;
      }
    }
    Kp_ = (K_ + 4 * G_ - 1) / (4 * G_) * (4 * G_);
    const int rounds = Kp_ / (4 * G_);
    // G = 4 kernels are instantiated for every round count 1..8 (no dead rounds held
    // in registers); wider groups use 8 or 16.
    R_ = G_ == 4 ? rounds : (rounds <= 8 ? 8 : 16);
    partition_docs(d.doc_offsets, M_, c.world, c.rank, &d0_, &d1_);
    Ml_ = d1_ - d0_;
    tok0_ = d.doc_offsets[d0_];
    Nl_ = d.doc_offsets[d1_] - tok0_;
    // per-GPU token and document indices are 32-bit in the fallback queue and the
    // z-step's work units: shard larger corpora across more GPUs
    require(Nl_ < (1ll << 31) && Ml_ < (1ll << 31), BNMC_GPU_ERR_ARG,
            "LDA shard too large: < 2^31 tokens and documents per GPU");
    off_host_.resize(static_cast<std::size_t>(Ml_) + 1);
    for (std::int64_t m = 0; m <= Ml_; ++m) off_host_[m] = d.doc_offsets[d0_ + m] - tok0_;

    alpha_ = d.hyper[0] > 0 ? d.hyper[0] : 0.1;
    beta_ = d.hyper[1] > 0 ? d.hyper[1] : 0.1;
    seed_ = d.seed;
    var_phi_ = d.var_ids[0];
    var_theta_ = d.var_ids[1];
    var_z_ = d.var_ids[2];
    var_w_ = d.var_ids[3];

    phi_threads_ = std::min(256, ((K_ + 31) / 32) * 32);
    // ~16 resident blocks' worth of gamma cells per SM: rows per phi block.
    const std::int64_t target_blocks = 148 * 16;
    rows_per_block_ = static_cast<int>(std::max<std::int64_t>(1, (V_ + target_blocks - 1) / target_blocks));
    nb_phi_ = (V_ + rows_per_block_ - 1) / rows_per_block_;

    // z-step work units: chunks of <= kChunk tokens of one document (whole documents
    // up to kChunk: one theta setup per document).  The transposed z-step's CTA has
    // one warp per 32-token batch of a mean unit (<= 8), so short documents (KOS: 136
    // tokens) do not leave most warps of a 256-thread CTA idle.
    for (std::int64_t m = 0; m < Ml_; ++m)
      for (std::int64_t t = off_host_[m]; t < off_host_[m + 1]; t += kChunk) {
        units_host_.push_back(m);
        units_host_.push_back(t);
        units_host_.push_back(std::min(t + kChunk, off_host_[m + 1]));
      }
    n_units_ = static_cast<std::int64_t>(units_host_.size() / 3);
    std::vector<std::int64_t> wu;
    for (std::int64_t m = 0; m < Ml_; ++m)
      for (std::int64_t t = off_host_[m]; t < off_host_[m + 1]; t += 256) {
        wu.push_back(m);
        wu.push_back(t);
        wu.push_back(std::min<std::int64_t>(t + 256, off_host_[m + 1]));
      }
    n_wunits_ = static_cast<std::int64_t>(wu.size() / 3);
    wunits_.alloc(std::max<std::size_t>(wu.size(), 3));
    if (!wu.empty())
      BNMC_CUDA(cudaMemcpy(wunits_.p, wu.data(), sizeof(std::int64_t) * wu.size(), cudaMemcpyHostToDevice));
    // warp-level units for short documents (r01 v42: KOS, 136 tokens/doc, z-step 32 -> 27 us;
    // NIPS, 1267 tokens/doc, is faster with document-wide CTA units: 93 vs 110 us)
    zt_wu_ = Ml_ > 0 && Nl_ / Ml_ < 256;
    if (const char* e = std::getenv("BNMC_ZT_WU")) zt_wu_ = std::string(e) != "0";
    {
      const double mean = n_units_ > 0 ? static_cast<double>(Nl_) / static_cast<double>(n_units_) : 32.0;
      // at most 4 warps per document CTA (r01, NIPS z-step: 4 warps 91.5 us, 8 warps 93.5,
      // 5-6 warps 95; smaller CTAs, same warps per SM)
      zt_warps_ = std::min(4, std::max(1, static_cast<int>(std::ceil(mean / 32.0))));
      if (const char* e = std::getenv("BNMC_ZT_WARPS")) zt_warps_ = std::min(8, std::max(1, std::atoi(e)));
    }

    w_.alloc(std::max<std::int64_t>(Nl_, 1));
    z_.alloc(std::max<std::int64_t>(Nl_, 1));
    off_.alloc(Ml_ + 1);
    // phi row slices of the sharded phi block: ceil(V / world) rows per rank (arrays padded
    // to world slices: the collectives move equal chunks)
    {
      const int world = comm_.active() ? comm_.world : 1, rank = comm_.active() ? comm_.rank : 0;
      slice_ = (V_ + world - 1) / world;
      Vpad_ = static_cast<std::int64_t>(slice_) * world;
      pv0_ = std::min(V_, rank * slice_);
      pv1_ = std::min(V_, pv0_ + slice_);
    }
    phiT_.alloc(static_cast<std::size_t>(Vpad_) * Kp_);
    if (exact_) logphiT_.alloc(static_cast<std::size_t>(V_) * Kp_);
    // K <= 128 (transposed screen, a few thousand queued tokens): the r01 grid, 9472 warps
    fb_blocks_ = K_ <= 128 ? 148 * 16 : 148 * 12;
    if (const char* e = std::getenv("BNMC_FB_BLOCKS")) fb_blocks_ = std::max(1, std::atoi(e));
    if (fallback_smem() > 48 * 1024)
    {
      BNMC_CUDA(cudaFuncSetAttribute(zfallback_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(fallback_smem())));
      BNMC_CUDA(cudaFuncSetAttribute(zfallback_log_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(fallback_smem())));
    }
    // fp32-screened z-step; BNMC_ZSTEP_SCREEN=0 disables it.
    const char* sc = std::getenv("BNMC_ZSTEP_SCREEN");
    // (exact-weights mode too: the screen decides the real-number topic; its undecided
    // tokens take the log-space fallback, zfallback_log_kernel)
    screen_ = !(sc && std::string(sc) == "0");
    choose_screen();
    Kp32_ = CW32_ * G32_ * RS_;
    if (screen_) phiT32_.alloc(static_cast<std::size_t>(Vpad_) * Kp32_);
    {
      // word-major z-step order when the fp32 rows exceed a quarter of the L2 (measured,
      // scripts/wm_probe.py: faster at 37 MB of rows and above (K = 300 / V = 3e4: 6.1 ->
      // 4.8 ms; 1B: 410 MB), slower at <= 20 MB (K = 1000 / V = 5000: 2.2 -> 3.0 ms));
      // BNMC_ZSTEP_WM=0/1 forces it off / on (on: the default layouts only)
      const std::size_t rows32 = sizeof(float) * static_cast<std::size_t>(V_) * Kp32_;
      const bool can = screen_ && !transposed_ && Ml_ > 0 && wm_layout(screen_key());
      wm_ = can && rows32 > (32ull << 20);
      if (const char* e = std::getenv("BNMC_ZSTEP_WM")) wm_ = can && std::string(e) != "0";
      // theta/S rows of a document block: ~24 MB of fp32
      wm_block_docs_ = std::max<std::int64_t>(1, (24ll << 20) / (4ll * Kp32_));
      if (const char* e = std::getenv("BNMC_WM_BLOCK_DOCS")) wm_block_docs_ = std::max<std::int64_t>(1, std::atoll(e));
    }
    theta_.alloc(std::max<std::int64_t>(Ml_ * K_, 1));
    nkw_.alloc(static_cast<std::size_t>(Vpad_) * Kp_);
    nmk_.alloc(std::max<std::int64_t>(Ml_ * K_, 1));
    units_.alloc(std::max<std::size_t>(units_host_.size(), 3));
    tpart_.alloc(std::max<std::int64_t>(Ml_, 1));
    docs_per_block_ = std::max<std::int64_t>(1, 4096 / K_);
    nb_doc_ = (Ml_ + docs_per_block_ - 1) / docs_per_block_;
    // grid sizes of the small reductions, scaled to the work (r01 v47 tuning)
    nbw_ = 148 * 4;
    if (const char* e = std::getenv("BNMC_WTERM_BLOCKS")) nbw_ = std::max(1, std::atoi(e));
    zpart_.alloc(nbw_);
    fq_.alloc(std::max<std::int64_t>(Nl_, 1));
    fq_len_.alloc(1);
    wpart_.alloc(nbw_);
    ttpart_.alloc(nbw_);
    {
      // warp-pool conjugate block: a persistent grid (one resident wave), equal cell
      // ranges per warp
      int dev = 0, sms = 148, per_sm = 1;
      BNMC_CUDA(cudaGetDevice(&dev));
      BNMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      if (K_ <= kPoolCells) {
        BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_pool_kernel<true>, 256, 0));
        // 3 resident blocks/SM measured ~2 us faster than 4 on NIPS/KOS (more L1 left
        // beside the tables); 3.5 and 2 are both slower
        per_sm = std::min(per_sm, 3);
      } else
        BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_pool_kernel<false>, 256, 0));
      pool_blocks_ = sms * std::max(per_sm, 1);
      if (const char* e = std::getenv("BNMC_POOL_BLOCKS")) pool_blocks_ = std::max(1, std::atoi(e));
    }
    // column-sum stripes of ~48 rows (<= 128), theta-row blocks of 8 warps (one row each)
    col_stripes_ = static_cast<int>(std::min<std::int64_t>(kColStripes, std::max<std::int64_t>(4, V_ / 48)));
    {
      const std::int64_t gx = (K_ + 31) / 32, wblocks = (Ml_ + 7) / 8;
      trow_blocks_ = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((wblocks + gx - 1) / gx, 16384)));
    }
    if (const char* e = std::getenv("BNMC_COL_STRIPES")) col_stripes_ = std::min(kColStripes, std::max(1, std::atoi(e)));
    spart_.alloc(static_cast<std::size_t>(kColStripes) * K_ * 2);
    ticket_.alloc((K_ + 31) / 32 + 1);
    ticket_.zero(nullptr);
    logS_.alloc(Kp_);
    logS_.zero(nullptr);  // padding columns stay 0 (wterm_kernel reads 4-cell vectors)
    colpart2_.alloc(static_cast<std::size_t>(nb_phi_) * K_ * 2);
    S_.alloc(K_);
    phi_term_.alloc(K_);
    doc_part_.alloc(std::max<std::int64_t>(Ml_ * 3, 3));
    red_.alloc(4);
    cudaStream_t s0 = nullptr;
    BNMC_CUDA(cudaMemcpy(off_.p, off_host_.data(), sizeof(std::int64_t) * (Ml_ + 1), cudaMemcpyHostToDevice));
    if (!units_host_.empty())
      BNMC_CUDA(cudaMemcpy(units_.p, units_host_.data(), sizeof(std::int64_t) * units_host_.size(),
                           cudaMemcpyHostToDevice));
    nmk_.zero(s0);
    tpart_.zero(s0);
    zpart_.zero(s0);
    wpart_.zero(s0);
    phiT_.zero(s0);
    phiT32_.zero(s0);
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

    // theta operands of the z-step: shared memory (default: 60 registers, 4 CTAs/SM)
    // or registers (BNMC_ZSTEP_THETA=regs: 128 registers; measured 20 % slower on NIPS).
    const char* tr = std::getenv("BNMC_ZSTEP_THETA");
    theta_regs_ = tr && std::string(tr) == "regs";
    // grouped screen (K > 128): 2^-17, >= 2.2x its error budget (above zscreen_kernel);
    // 1B: the fp64 queue 1.2 % -> 0.6 % of the tokens, sweep 424 -> 390 ms
    if (!transposed_) screen_margin_ = kScreenMargin * 0.5f;
    if (const char* e = std::getenv("BNMC_SCREEN_MARGIN")) screen_margin_ = static_cast<float>(std::atof(e));
    if (const char* e = std::getenv("BNMC_PDL")) pdl_ = std::string(e) != "0";
    configure_kernels();
    BNMC_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_phi_ready_, cudaEventDisableTiming));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_theta_ready_, cudaEventDisableTiming));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_copy_done_, cudaEventDisableTiming));
    BNMC_CUDA(cudaStreamCreateWithFlags(&up_, cudaStreamNonBlocking));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_up_, cudaEventDisableTiming));
    BNMC_CUDA(cudaMallocHost(reinterpret_cast<void**>(&spec_flag_host_), sizeof(int)));
    spec_flag_.alloc(1);
    if (const char* e = std::getenv("BNMC_SPECULATE")) speculate_ = std::string(e) != "0";
  }

  ~Lda() override {
    if (copy_) cudaStreamDestroy(copy_);
    if (ev_phi_ready_) cudaEventDestroy(ev_phi_ready_);
    if (ev_theta_ready_) cudaEventDestroy(ev_theta_ready_);
    if (ev_copy_done_) cudaEventDestroy(ev_copy_done_);
    if (up_) cudaStreamDestroy(up_);
    if (ev_up_) cudaEventDestroy(ev_up_);
    if (spec_flag_host_) cudaFreeHost(spec_flag_host_);
  }

  void upload(const bnmc_gpu_store& s, cudaStream_t st) override { upload_impl(s, st, true); }

  void upload_state(const bnmc_gpu_store& s, cudaStream_t st) override {
    upload_impl(s, st, !data_on_device_);
  }

  // The LDA sweep reads only z of the latent state: its phi and theta blocks redraw
  // phi and theta from the counts of z before anything reads them (plan order phi,
  // theta, z; sampler.cpp:52-218).  So a bound store's sweep uploads z alone and
  // rebuilds the counts; phiT / S keep the last sweep's values (download-consistent).
  void upload_sweep_inputs(const bnmc_gpu_store& s, cudaStream_t st) override {
    if (!data_on_device_) {
      upload_impl(s, st, true);
      return;
    }
    check_len(s, var_z_, N_, "z");
    require(s.ival[var_z_] != nullptr, BNMC_GPU_ERR_RUNTIME, "store arrays missing");
    if (Nl_ > 0) {
      if (stage64_.n < static_cast<std::size_t>(Nl_)) stage64_.alloc(Nl_);
      BNMC_CUDA(cudaMemcpyAsync(stage64_.p, s.ival[var_z_] + tok0_, sizeof(std::int64_t) * Nl_,
                                cudaMemcpyHostToDevice, st));
      h2d_bytes += static_cast<std::int64_t>(sizeof(std::int64_t)) * Nl_;
    }
    adopt_z(stage64_.p, st);
  }

  // z := the uploaded int64 assignments (range-checked), counts rebuilt from them
  void adopt_z(const std::int64_t* dev64, cudaStream_t st) {
    if (Nl_ > 0) i64_to_i32_kernel<<<blocks_for(Nl_, 256), 256, 0, st>>>(dev64, z_.p, Nl_, 0, K_, out.err);
    LdaArgs a = args();
    nkw_.zero(st);
    nmk_.zero(st);
    if (Nl_ > 0) {
      count_kernel<<<std::min<unsigned>(blocks_for(Nl_, 256), 148 * 16), 256, 0, st>>>(a, out.err);
      doc_counts_kernel<<<grid_docs(), 256, 0, st>>>(a, nmk_.p);
    }
    BNMC_CUDA(cudaGetLastError());
  }

  // Speculative bound-store sweep (Model::spec_begin): the sweep starts from the device
  // state -- the z this context last wrote back to the caller (zprev_), with its counts
  // -- while the caller's z crosses PCIe on up_; spec_verify compares the two after
  // the sweep, and a difference makes sweep_store adopt the upload and redo the sweep.
  // Sharded: whether to speculate and whether to redo are collective decisions (an int
  // all-reduce each), so every rank runs the same sweeps and NCCL calls.
  // BNMC_SPECULATE=0 disables it.
  bool spec_begin(const bnmc_gpu_store& s, cudaStream_t st) override {
    bool ok = quiet && speculate_ && Nl_ > 0 && zprev_valid_ && !(s.observed && s.observed[var_z_]) &&
              s.ival[var_z_] != nullptr;
    if (comm_.active()) {
      *spec_flag_host_ = ok ? 1 : 0;
      BNMC_CUDA(cudaMemcpyAsync(spec_flag_.p, spec_flag_host_, sizeof(int), cudaMemcpyHostToDevice, st));
      comm_.all_reduce(spec_flag_.p, 1, RedType::I32, RedOp::Min, st);
      BNMC_CUDA(cudaMemcpyAsync(spec_flag_host_, spec_flag_.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      BNMC_CUDA(cudaStreamSynchronize(st));
      ok = *spec_flag_host_ == 1;
    }
    if (!ok) return false;
    check_len(s, var_z_, N_, "z");
    if (up64_.n < static_cast<std::size_t>(Nl_)) up64_.alloc(Nl_);
    BNMC_CUDA(cudaMemsetAsync(spec_flag_.p, 0, sizeof(int), st));
    BNMC_CUDA(cudaMemcpyAsync(up64_.p, s.ival[var_z_] + tok0_, sizeof(std::int64_t) * Nl_, cudaMemcpyHostToDevice, up_));
    BNMC_CUDA(cudaEventRecord(ev_up_, up_));
    h2d_bytes += static_cast<std::int64_t>(sizeof(std::int64_t)) * Nl_;
    return true;
  }

  void spec_verify(cudaStream_t st) override {
    BNMC_CUDA(cudaStreamWaitEvent(st, ev_up_, 0));
    spec_check_kernel<<<std::min<unsigned>(blocks_for(Nl_, 256), 148 * 8), 256, 0, st>>>(up64_.p, zprev_.p, Nl_, spec_flag_.p);
    if (comm_.active()) comm_.all_reduce(spec_flag_.p, 1, RedType::I32, RedOp::Max, st);
    BNMC_CUDA(cudaMemcpyAsync(spec_flag_host_, spec_flag_.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  }

  bool spec_failed() override { return *spec_flag_host_ != 0; }

  void spec_adopt(cudaStream_t st) override { adopt_z(up64_.p, st); }

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
    if (with_data) build_word_major(st);
  }

  // An event other streams can wait on: inside a stream capture it must be an external
  // event node (cudaEventRecordExternal), outside a plain record (direct launches).
  static void record_external(cudaEvent_t ev, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    BNMC_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs == cudaStreamCaptureStatusActive) BNMC_CUDA(cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal));
    else BNMC_CUDA(cudaEventRecord(ev, st));
  }

  // phi and theta are final early in the sweep (after the phi block / the theta block):
  // their transpose + device-to-host copies run on a copy stream while the z-step and
  // the log-joint run; z follows the sweep on the main stream.
  // Writes z back into the int64 store slice `dst` (enqueued on st).
  void download_z(std::int64_t* dst, cudaStream_t st) {
    if (stage64_.n < static_cast<std::size_t>(Nl_)) stage64_.alloc(Nl_);
    if (zprev_.n < static_cast<std::size_t>(Nl_)) zprev_.alloc(Nl_);
    z_writeback_kernel<<<std::min<unsigned>(blocks_for(Nl_, 256), 148 * 16), 256, 0, st>>>(z_.p, stage64_.p, zprev_.p, Nl_);
    zprev_valid_ = true;
    BNMC_CUDA(cudaMemcpyAsync(dst, stage64_.p, sizeof(std::int64_t) * Nl_, cudaMemcpyDeviceToHost, st));
    d2h_bytes += static_cast<std::int64_t>(sizeof(std::int64_t)) * Nl_;
  }

  bool download_overlapped(const bnmc_gpu_store& s, cudaStream_t st) override {
    if (marks || observe_phi_ || Ml_ == 0) return false;
    const char* obs = s.observed;
    if (!(obs && obs[var_phi_]) && s.real[var_phi_]) {
      if (stage_phi_.n == 0) stage_phi_.alloc(static_cast<std::size_t>(K_) * V_);
      BNMC_CUDA(cudaStreamWaitEvent(copy_, ev_phi_ready_, 0));
      transpose_kernel<<<dim3((K_ + 31) / 32, (V_ + 31) / 32), dim3(32, 8), 0, copy_>>>(phiT_.p, stage_phi_.p, V_, K_, Kp_, V_, S_.p);
      BNMC_CUDA(cudaMemcpyAsync(s.real[var_phi_], stage_phi_.p, stage_phi_.bytes(), cudaMemcpyDeviceToHost, copy_));
      d2h_bytes += static_cast<std::int64_t>(stage_phi_.bytes());
    }
    if (!(obs && obs[var_theta_]) && s.real[var_theta_]) {
      BNMC_CUDA(cudaStreamWaitEvent(copy_, ev_theta_ready_, 0));
      BNMC_CUDA(cudaMemcpyAsync(s.real[var_theta_] + d0_ * K_, theta_.p, sizeof(double) * Ml_ * K_,
                                cudaMemcpyDeviceToHost, copy_));
      d2h_bytes += static_cast<std::int64_t>(sizeof(double)) * Ml_ * K_;
    }
    BNMC_CUDA(cudaEventRecord(ev_copy_done_, copy_));
    if (!(obs && obs[var_z_]) && s.ival[var_z_] && Nl_ > 0) download_z(s.ival[var_z_] + tok0_, st);
    BNMC_CUDA(cudaStreamWaitEvent(st, ev_copy_done_, 0));  // the sweep call completes with both
    BNMC_CUDA(cudaGetLastError());
    return true;
  }

  void download(const bnmc_gpu_store& s, cudaStream_t st) override {
    const char* obs = s.observed;
    if (!(obs && obs[var_z_]) && s.ival[var_z_] && Nl_ > 0) download_z(s.ival[var_z_] + tok0_, st);
    if (!(obs && obs[var_theta_]) && s.real[var_theta_] && Ml_ > 0)
      BNMC_CUDA(cudaMemcpyAsync(s.real[var_theta_] + d0_ * K_, theta_.p, sizeof(double) * Ml_ * K_,
                                cudaMemcpyDeviceToHost, st));
    if (!(obs && obs[var_phi_]) && !observe_phi_ && s.real[var_phi_]) {
      if (stage_phi_.n == 0) stage_phi_.alloc(static_cast<std::size_t>(K_) * V_);
      transpose_kernel<<<dim3((K_ + 31) / 32, (V_ + 31) / 32), dim3(32, 8), 0, st>>>(phiT_.p, stage_phi_.p, V_, K_, Kp_, V_, S_.p);
      BNMC_CUDA(cudaMemcpyAsync(s.real[var_phi_], stage_phi_.p, stage_phi_.bytes(), cudaMemcpyDeviceToHost, st));
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  void enqueue_sweep(cudaStream_t st) override {
    LdaArgs a = args();
    // this sweep's phi block leaves g (unnormalised) + logS: the w-factor takes
    // log g - log S (the exact mode normalises phiT in place, S = 1: the phi/S path)
    // (exact mode: phiT is normalised in place below and log S zeroed, so the w-factor
    // takes the same compacted n log phi path)
    a.logg_valid = !observe_phi_ ? 1 : 0;
    const bool timed = marks != nullptr;  // phase timing: everything on one stream
    mark(st, "begin");
    // warp-pool conjugate block: phi and theta cells in one balanced kernel, then the
    // phi column sums (phi_colsum2 stripes) and the theta rows (extra y-blocks)
    // Sharded: each rank draws the phi rows of its slice only -- a reduce-scatter gives it
    // the global counts of those rows (the other rows' local counts are then zeroed for
    // this sweep's z-step), and an all-gather of the drawn rows follows the pool.  The
    // draws are keyed by (k, v), so phi is bitwise the unsharded one for every world size.
    const bool sliced = !observe_phi_ && comm_.active();
    if (sliced) {
      comm_.reduce_scatter(nkw_.p, static_cast<std::size_t>(slice_) * Kp_, RedType::I32, st);
      const std::size_t row = static_cast<std::size_t>(Kp_) * sizeof(int);
      if (pv0_ > 0) BNMC_CUDA(cudaMemsetAsync(nkw_.p, 0, row * pv0_, st));
      const std::int64_t after = static_cast<std::int64_t>(pv0_) + slice_;
      if (Vpad_ > after)
        BNMC_CUDA(cudaMemsetAsync(nkw_.p + after * Kp_, 0, row * static_cast<std::size_t>(Vpad_ - after), st));
      mark(st, "reduce_scatter_counts");
    }
    if (observe_phi_) nkw_.zero(st);  // phi clamped: the z-step's counts feed only the w-factor
    a.pool_phi = observe_phi_ ? 0 : 1;
    a.pool_v0 = pv0_;
    a.pool_v1 = pv1_;
    a.trow_blocks = Ml_ > 0 ? trow_blocks_ : 0;
    a.col_stripes = observe_phi_ ? 0 : col_stripes_;
    if (a.pool_phi || Ml_ > 0) {
      if (K_ <= kPoolCells)
        phi_pool_kernel<true><<<pool_blocks_, 256, 0, st>>>(a, out.iter);
      else
        phi_pool_kernel<false><<<pool_blocks_, 256, 0, st>>>(a, out.iter);
      mark(st, "conj_pool");
      if (sliced) {  // the drawn rows: fp64 g, and their fp32 screen copy (4-byte words)
        comm_.all_gather(phiT_.p, static_cast<std::size_t>(slice_) * Kp_, RedType::F64, st);
        if (screen_) comm_.all_gather(phiT32_.p, static_cast<std::size_t>(slice_) * Kp32_, RedType::I32, st);
        mark(st, "all_gather_phi");
      }
      launch_pdl(phi_colsum2_kernel, dim3((K_ + 31) / 32, a.col_stripes + a.trow_blocks), dim3(256), 0, st, a);
      fq_reset_ = true;
      mark(st, "colsum_rows");
    }
    if (!observe_phi_ && exact_ && !screen_) {
      // the unscreened log-space z-step reads log phi: normalise in place, then phi =
      // phiT (S = 1). (Screened, phiT keeps g as in the product mode: the screen reads
      // g and theta/S, the log-space fallback forms phi = g / S itself.)
      phi_norm_kernel<true><<<nb_phi_, phi_threads_, 0, st>>>(a);
      fill_kernel<<<1, 256, 0, st>>>(S_.p, K_, 1.0);
      fill_kernel<<<1, 256, 0, st>>>(logS_.p, K_, 0.0);
      mark(st, "phi_norm");
    }
    if (!timed) {  // phi, theta final: overlapped downloads may start (external event nodes)
      if (!observe_phi_) record_external(ev_phi_ready_, st);
      if (Ml_ > 0) record_external(ev_theta_ready_, st);
    }
    if (Ml_ > 0) {
      launch_zstep(a, st);
      mark(st, "zstep");
      if (timed && std::getenv("BNMC_SCREEN_STATS")) {  // diagnostics: queue lengths of this sweep
        int n3 = -1;
        BNMC_CUDA(cudaStreamSynchronize(st));
        BNMC_CUDA(cudaMemcpy(&n3, fq_len_.p, sizeof(int), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[bnmc] z-step fp64 queue: %d of %lld tokens\n", n3, static_cast<long long>(Nl_));
      }
    }
    const unsigned nbw = static_cast<unsigned>(nbw_);
    if (comm_.active()) {
      // this rank's pieces by the last wterm block, then the all-reduce and the finish
      LdaArgs ar = a;
      ar.red_only = 1;
      launch_pdl(wterm_kernel<true>, dim3(nbw), dim3(256), 0, st, ar, out, 0);
      mark(st, "wterm");
      comm_.all_reduce(red_.p, 3, RedType::F64, RedOp::Sum, st);
      finalize_kernel<<<1, 256, 0, st>>>(a, out, 1);
      mark(st, "reduce_finalize");
    } else {
      launch_pdl(wterm_kernel<true>, dim3(nbw), dim3(256), 0, st, a, out, 1);
      mark(st, "wterm_finalize");
    }
    BNMC_CUDA(cudaGetLastError());
  }

  void enqueue_log_joint(cudaStream_t st) override {
    LdaArgs a = args();
    phi_norm_kernel<false><<<nb_phi_, phi_threads_, 0, st>>>(a);
    phi_terms_kernel<<<K_, 128, 0, st>>>(a);
    if (Ml_ > 0) doc_eval_kernel<<<grid_docs(), 256, 0, st>>>(a, out.err);
    reduce_kernel<true><<<1, 1024, 0, st>>>(a);
    if (comm_.active())
      comm_.all_reduce(red_.p, 3, RedType::F64, RedOp::Sum, st);
    finalize_kernel<<<1, 256, 0, st>>>(a, out, 0);
    BNMC_CUDA(cudaGetLastError());
  }

  void prior_init(std::uint64_t seed, cudaStream_t st) override {
    LdaArgs a = args();
    if (!observe_phi_)
      dirichlet_rows(phiT_.p, K_, V_, 1, Kp_, beta_, seed, var_phi_, 0, st);
    if (Ml_ > 0) {
      dirichlet_rows(theta_.p, Ml_, K_, K_, 1, alpha_, seed, var_theta_, d0_, st);
      if (doc_cum_smem())
        prior_z_kernel<true><<<grid_docs(), 256, sizeof(double) * K_, st>>>(a, seed);
      else
        prior_z_kernel<false><<<grid_docs(), 256, 0, st>>>(a, seed);
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
    after_state_change(st);
  }

  // Checkpoint restore: phiT holds this sweep's gamma draws g with their row sums S;
  // normalise in place (phi = g / S, the value download() reports) and rebuild the
  // counts and phi terms as after an upload.
  void on_state_restored(cudaStream_t st) override {
    LdaArgs a = args();
    phi_norm_kernel<true><<<nb_phi_, phi_threads_, 0, st>>>(a);
    after_state_change(st);
  }

  // Binary corpus (.bnc, see include/bnmc_gpu.h): this shard's token range of w is
  // streamed through a pinned buffer into the device (int32, range-checked); the
  // document offsets must equal the ones the context was created with.
  void lda_load_corpus(const char* path, cudaStream_t st) override {
    std::FILE* f = std::fopen(path, "rb");
    require(f != nullptr, BNMC_GPU_ERR_RUNTIME, std::string("cannot open corpus ") + path);
    struct Closer {
      std::FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[8];
    std::uint32_t ver = 0, pad = 0;
    std::int64_t M = 0, N = 0, V = 0;
    require(std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, "BNMCCORP", 8) == 0, BNMC_GPU_ERR_RUNTIME,
            "not a bnmc corpus file");
    require(std::fread(&ver, 4, 1, f) == 1 && std::fread(&pad, 4, 1, f) == 1 && ver == 1, BNMC_GPU_ERR_RUNTIME,
            "unsupported corpus version");
    require(std::fread(&M, 8, 1, f) == 1 && std::fread(&N, 8, 1, f) == 1 && std::fread(&V, 8, 1, f) == 1,
            BNMC_GPU_ERR_RUNTIME, "truncated corpus header");
    require(M == M_ && N == N_ && V == V_, BNMC_GPU_ERR_RUNTIME, "corpus sizes differ from the model's (M, N, V)");
    std::vector<std::int64_t> off(static_cast<std::size_t>(M) + 1);
    require(std::fread(off.data(), 8, off.size(), f) == off.size(), BNMC_GPU_ERR_RUNTIME, "truncated corpus offsets");
    for (std::int64_t m = 0; m <= Ml_; ++m)
      require(off[d0_ + m] - tok0_ == off_host_[m], BNMC_GPU_ERR_RUNTIME, "corpus document offsets differ");
    const long base = static_cast<long>(8 + 8 + 24 + 8 * (M + 1));
    require(std::fseek(f, base + static_cast<long>(4 * tok0_), SEEK_SET) == 0, BNMC_GPU_ERR_RUNTIME, "corpus seek failed");
    const std::int64_t chunk = 16 << 20;  // tokens per staged copy
    int* pinned = nullptr;
    BNMC_CUDA(cudaMallocHost(&pinned, sizeof(int) * static_cast<std::size_t>(std::min(chunk, std::max<std::int64_t>(Nl_, 1)))));
    struct Pin {
      int* p;
      ~Pin() { cudaFreeHost(p); }
    } pin{pinned};
    if (stage64_.n < static_cast<std::size_t>(std::max<std::int64_t>(Nl_, 1))) stage64_.alloc(std::max<std::int64_t>(Nl_, 1));
    for (std::int64_t t = 0; t < Nl_; t += chunk) {
      const std::int64_t n = std::min(chunk, Nl_ - t);
      require(std::fread(pinned, 4, static_cast<std::size_t>(n), f) == static_cast<std::size_t>(n), BNMC_GPU_ERR_RUNTIME,
              "truncated corpus tokens");
      BNMC_CUDA(cudaMemcpyAsync(w_.p + t, pinned, sizeof(int) * n, cudaMemcpyHostToDevice, st));
      BNMC_CUDA(cudaStreamSynchronize(st));  // the pinned buffer is reused
    }
    i32_check_kernel<<<std::max(1u, std::min<unsigned>(blocks_for(Nl_, 256), 148 * 16)), 256, 0, st>>>(w_.p, Nl_, V_, out.err);
    data_on_device_ = true;
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
    build_word_major(st);
  }

  std::vector<StateBuf> state_buffers() override {
    return {{reinterpret_cast<void**>(&z_.p), sizeof(int) * static_cast<std::size_t>(Nl_)},
            {reinterpret_cast<void**>(&theta_.p), sizeof(double) * static_cast<std::size_t>(Ml_ * K_)},
            {reinterpret_cast<void**>(&phiT_.p), phiT_.bytes()},
            {reinterpret_cast<void**>(&S_.p), S_.bytes()}};
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
      if (comm_.active())
        comm_.all_reduce(tmp.p, tmp.n, RedType::I32, RedOp::Sum, st);
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
    dirichlet_rows(cum.p, K_, V_, V_, 1, phi_conc, seed ^ 0xDA7Aull, 0, 0, st);
    row_scan_kernel<true><<<blocks_for(K_, kScanWarps), 32 * kScanWarps, 0, st>>>(cum.p, K_, V_, V_, 1, nullptr);
    if (Ml_ > 0) {
      dirichlet_rows(th.p, Ml_, K_, K_, 1, theta_conc, seed ^ 0xDA7Aull, 1, d0_, st);
      LdaArgs a = args();
      if (doc_cum_smem())
        gen_tokens_kernel<true><<<grid_docs(), 256, sizeof(double) * K_, st>>>(a, cum.p, th.p, seed);
      else
        gen_tokens_kernel<false><<<grid_docs(), 256, 0, st>>>(a, cum.p, th.p, seed);
    }
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
    build_word_major(st);
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
    fill_kernel<<<1, 256, 0, st>>>(S_.p, K_, 1.0);  // phiT holds phi itself
    LdaArgs a = args();
    nkw_.zero(st);
    nmk_.zero(st);
    if (Nl_ > 0) {
      count_kernel<<<std::min<unsigned>(blocks_for(Nl_, 256), 148 * 16), 256, 0, st>>>(a, out.err);
      doc_counts_kernel<<<grid_docs(), 256, 0, st>>>(a, nmk_.p);
    }
    // phi terms (and the exact-mode log table) of the uploaded phi: used as-is by
    // clamped-phi runs, recomputed by the phi block otherwise.
    phi_norm_kernel<false><<<nb_phi_, phi_threads_, 0, st>>>(a);
    phi_terms_kernel<<<K_, 128, 0, st>>>(a);
    if (screen_) phi_f32_kernel<<<148 * 8, 256, 0, st>>>(a);
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  // running sums per document in shared memory (BNMC_DOC_SCAN=1: the reference's linear scan)
  bool doc_cum_smem() const {
    const char* e = std::getenv("BNMC_DOC_SCAN");
    return K_ <= kDocCumMax && !(e && std::string(e) != "0");
  }

  unsigned grid_docs() const { return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>(Ml_, 1 << 20))); }

  std::size_t zstep_smem() const { return sizeof(double) * 2 * Kp_; }

  std::size_t fallback_smem() const { return sizeof(double) * (kFallbackThreads / 32) * fallback_stride(K_); }

  // The fp64 redraw of the screen's undecided tokens: the log-space draw in the exact-
  // weights mode, else the product form (staged through shared memory for K > 128).
  void launch_fallback(const LdaArgs& a, cudaStream_t st) {
    const std::int64_t* it = out.iter;
    if (exact_)
      launch_pdl(zfallback_log_kernel, dim3(fb_blocks_), dim3(kFallbackThreads), fallback_smem(), st, a, it, out.err);
    else if (K_ <= 128)
      launch_pdl(zfallback_kernel<false>, dim3(fb_blocks_), dim3(kFallbackThreads), 0, st, a, it, out.err);
    else
      launch_pdl(zfallback_kernel<true>, dim3(fb_blocks_), dim3(kFallbackThreads), fallback_smem(), st, a, it, out.err);
  }

  template <int G, int R, bool E>
  void zstep_attr() {
    const int sm = static_cast<int>(zstep_smem());
    BNMC_CUDA(cudaFuncSetAttribute(zstep_kernel<G, R, E, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    BNMC_CUDA(cudaFuncSetAttribute(zstep_kernel<G, R, E, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));

  }

  void configure_kernels() {
    if (zstep_smem() <= 48 * 1024) return;
    dispatch_zstep([&](auto g, auto r, auto e) { zstep_attr<decltype(g)::value, decltype(r)::value, decltype(e)::value>(); });
  }

  template <class F>
  void dispatch_zstep(F&& f) {
    using std::integral_constant;
    auto with_e = [&](auto g, auto r) {
      if (exact_) f(g, r, integral_constant<bool, true>{});
      else f(g, r, integral_constant<bool, false>{});
    };
    if (G_ == 4) {
      switch (R_) {
        case 1: with_e(integral_constant<int, 4>{}, integral_constant<int, 1>{}); break;
        case 2: with_e(integral_constant<int, 4>{}, integral_constant<int, 2>{}); break;
        case 3: with_e(integral_constant<int, 4>{}, integral_constant<int, 3>{}); break;
        case 4: with_e(integral_constant<int, 4>{}, integral_constant<int, 4>{}); break;
        case 5: with_e(integral_constant<int, 4>{}, integral_constant<int, 5>{}); break;
        case 6: with_e(integral_constant<int, 4>{}, integral_constant<int, 6>{}); break;
        case 7: with_e(integral_constant<int, 4>{}, integral_constant<int, 7>{}); break;
        default: with_e(integral_constant<int, 4>{}, integral_constant<int, 8>{}); break;
      }
    }
    else if (G_ == 8) with_e(integral_constant<int, 8>{}, integral_constant<int, 8>{});
    else if (G_ == 16) with_e(integral_constant<int, 16>{}, integral_constant<int, 8>{});
    else if (R_ <= 8) with_e(integral_constant<int, 32>{}, integral_constant<int, 8>{});
    else with_e(integral_constant<int, 32>{}, integral_constant<int, 16>{});
  }

  // Screen layout: G lanes x CW candidates per round (G*CW = 32 floats, one 128-byte
  // line), R rounds.  Default: CW = 4 and the smallest G with R <= 4, theta operands
  // in registers (ncu r01 v8: with G = 4 x CW = 8 the per-token theta re-reads from
  // shared memory doubled the L1 register-writeback traffic, the limiter); K > 512:
  // G = 32 x CW = 8, theta in shared memory.  BNMC_ZSCREEN=g<G>w<CW>[s|r] overrides.
  void choose_screen() {
    transposed_ = K_ <= 128;
    G32_ = 32;
    CW32_ = 8;
    tfr_ = false;
    for (int g : {8, 16, 32}) {
      if ((K_ + 4 * g - 1) / (4 * g) <= 4) {
        G32_ = g;
        CW32_ = 4;
        tfr_ = true;
        break;
      }
    }
    if (const char* e = std::getenv("BNMC_ZSCREEN")) {
      int g = 0, w = 0;
      char mode = 'r';
      if (std::sscanf(e, "g%dw%d%c", &g, &w, &mode) >= 2 && g * w >= 32 && (w == 4 || w == 8) &&
          (g == 4 || g == 8 || g == 16 || g == 32)) {
        G32_ = g;
        CW32_ = w;
        tfr_ = mode != 's';
        transposed_ = false;
      }
    }
    if (const char* e = std::getenv("BNMC_ZSCREEN_T")) transposed_ = std::string(e) != "0" && K_ <= 128;
    if (transposed_) {
      G32_ = 4;
      CW32_ = 8;
      // theta operands in registers (ncu r01 v11: 108 us vs 131 us from shared memory)
      tfr_ = true;
      if (const char* e = std::getenv("BNMC_ZSTEP_THETA")) tfr_ = std::string(e) != "smem";
    }
    RS_ = (K_ + CW32_ * G32_ - 1) / (CW32_ * G32_);
    if (G32_ < 32 || CW32_ == 4) RS_ = RS_ <= 4 ? RS_ : -1;
    require(RS_ >= 1 && RS_ <= 8, BNMC_GPU_ERR_ARG, "z-step screen layout does not fit K");
    if (G32_ == 32 && CW32_ == 8) RS_ = RS_ <= 4 ? 4 : 8;
    else if (G32_ != 8 && G32_ != 4) RS_ = 4;
  }

  template <int G, int CW, int R, bool TFR, bool WM>
  void zscreen_launch(const LdaArgs& a, cudaStream_t st) {
    const unsigned g = static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>(a.n_units, 1 << 24)));
    const std::size_t sm = sizeof(float) * G * (CW * R + 4) * (WM ? kZThreads / 32 : 1);
    if (WM && sm > 48 * 1024)
      BNMC_CUDA(cudaFuncSetAttribute(zscreen_kernel<G, CW, R, TFR, WM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sm)));
    // word-major: one resident wave (warps stride over the units in order, so the units
    // in flight stay within one document block and its theta/S rows stay in L2)
    unsigned gw = g;
    if constexpr (WM) {
      int per_sm = 1, sms = 148, dev = 0;
      BNMC_CUDA(cudaGetDevice(&dev));
      BNMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, zscreen_kernel<G, CW, R, TFR, WM>, kZThreads, sm));
      gw = static_cast<unsigned>(std::max<std::int64_t>(
          1, std::min<std::int64_t>((a.n_units + kZThreads / 32 - 1) / (kZThreads / 32),
                                    static_cast<std::int64_t>(sms) * std::max(per_sm, 1))));
    }
    zscreen_kernel<G, CW, R, TFR, WM><<<gw, kZThreads, sm, st>>>(a, out.iter);
  }

  template <int G, int CW, bool TFR, bool WM = false>
  void zscreen_rounds(const LdaArgs& a, cudaStream_t st) {
    if constexpr (G <= 8) {
      switch (RS_) {
        case 1: zscreen_launch<G, CW, 1, TFR, WM>(a, st); return;
        case 2: zscreen_launch<G, CW, 2, TFR, WM>(a, st); return;
        case 3: zscreen_launch<G, CW, 3, TFR, WM>(a, st); return;
        default: zscreen_launch<G, CW, 4, TFR, WM>(a, st); return;
      }
    } else if constexpr (G == 32 && CW == 8 && !TFR) {
      if (RS_ > 4) zscreen_launch<G, CW, 8, TFR, WM>(a, st);
      else zscreen_launch<G, CW, 4, TFR, WM>(a, st);
    } else {
      zscreen_launch<G, CW, 4, TFR, WM>(a, st);
    }
  }

  // the screen layouts choose_screen picks by default (the word-major order exists for them)
  int screen_key() const { return G32_ * 100 + CW32_ * 10 + (tfr_ ? 1 : 0); }
  static bool wm_layout(int key) { return key == 3280 || key == 3241 || key == 1641 || key == 841; }

  // Word-major z-step order for corpora whose fp32 rows (V x Kp32) do not stay in L2:
  // the local tokens sorted by (block of documents, word); a work unit is one word's
  // tokens within a block (<= kChunk), so the word's row is read from HBM once per block
  // and the block's theta/S rows (wm_block_docs_ x Kp32 fp32, ~24 MB) stay in L2.
  void build_word_major(cudaStream_t st) {
    n_wm_units_ = 0;
    if (!wm_ || Nl_ == 0) return;
    const std::int64_t nblocks = (Ml_ + wm_block_docs_ - 1) / wm_block_docs_;
    const std::uint64_t maxkey = static_cast<std::uint64_t>(nblocks) * static_cast<std::uint64_t>(V_);
    if (maxkey >= (1ull << 32)) {  // keys must fit 32 bits: stay document-major
      wm_ = false;
      return;
    }
    int end_bit = 1;
    while ((1ull << end_bit) < maxkey) ++end_bit;
    DevBuf<std::uint32_t> keys, keys_alt;
    DevBuf<int> tok_a, tok_b, docof;
    keys.alloc(Nl_);
    keys_alt.alloc(Nl_);
    tok_a.alloc(Nl_);
    tok_b.alloc(Nl_);
    docof.alloc(Nl_);
    const LdaArgs a = args();
    wm_keys_kernel<<<grid_docs(), 256, 0, st>>>(a, wm_block_docs_, keys.p, tok_a.p, docof.p);
    BNMC_CUDA(cudaGetLastError());
    const int which = sort_pairs_u32(keys.p, keys_alt.p, tok_a.p, tok_b.p, Nl_, end_bit, st);
    std::uint32_t* skeys = which ? keys_alt.p : keys.p;
    DevBuf<int>& stok = which ? tok_b : tok_a;
    std::swap(wm_tok_.p, stok.p);
    std::swap(wm_tok_.n, stok.n);
    wm_doc_.alloc(Nl_);
    wm_gather_kernel<<<148 * 8, 256, 0, st>>>(wm_tok_.p, docof.p, wm_doc_.p, Nl_);
    // runs of (block, word) -> work units (word, i0, i1), <= kChunk tokens each
    std::uint32_t* uniq = which ? keys.p : keys_alt.p;  // the free buffer of the pair
    int* counts = docof.p;  // free after the gather (same stream)
    const std::int64_t nruns = run_length_u32(skeys, Nl_, uniq, counts, st);
    std::vector<std::uint32_t> hk(static_cast<std::size_t>(nruns));
    std::vector<int> hc(static_cast<std::size_t>(nruns));
    BNMC_CUDA(cudaMemcpyAsync(hk.data(), uniq, sizeof(std::uint32_t) * nruns, cudaMemcpyDeviceToHost, st));
    BNMC_CUDA(cudaMemcpyAsync(hc.data(), counts, sizeof(int) * nruns, cudaMemcpyDeviceToHost, st));
    BNMC_CUDA(cudaStreamSynchronize(st));
    std::vector<std::int64_t> u;
    u.reserve(static_cast<std::size_t>(nruns) * 3);
    std::int64_t pos = 0;
    for (std::int64_t r = 0; r < nruns; ++r) {
      const std::int64_t word = hk[r] % static_cast<std::uint32_t>(V_), end = pos + hc[r];
      for (std::int64_t i = pos; i < end; i += kChunk) {
        u.push_back(word);
        u.push_back(i);
        u.push_back(std::min<std::int64_t>(i + kChunk, end));
      }
      pos = end;
    }
    require(pos == Nl_, BNMC_GPU_ERR_RUNTIME, "word-major order: token count mismatch");
    n_wm_units_ = static_cast<std::int64_t>(u.size() / 3);
    wm_units_.alloc(std::max<std::size_t>(u.size(), 3));
    BNMC_CUDA(cudaMemcpyAsync(wm_units_.p, u.data(), sizeof(std::int64_t) * u.size(), cudaMemcpyHostToDevice, st));
    if (th32_.n == 0) {
      th32_.alloc(static_cast<std::size_t>(Ml_) * Kp32_);
      th32_.zero(st);
      thS_.alloc(static_cast<std::size_t>(Ml_) * K_);
      wm_ticket_.alloc(1);
    }
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  template <int R, bool TFR>
  void zscreen_t_launch(const LdaArgs& a, cudaStream_t st) {
    const unsigned g = static_cast<unsigned>(std::min<std::int64_t>(n_units_, 1 << 24));
    if (zt_wu_) {
      const int kpad = (K_ + 3) & ~3;
      const std::size_t smw = sizeof(float) * 8 * (4 * (8 * R + 4) + 32 * 16 + kpad);
      const unsigned gw = static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((n_wunits_ + 7) / 8, 148 * 3)));
      launch_pdl(zscreen_t_kernel<R, TFR, true>, dim3(gw), dim3(256), smw, st, a,
                 static_cast<const std::int64_t*>(out.iter));
      return;
    }
    const std::size_t sm = sizeof(float) * (4 * (8 * R + 4) + zt_warps_ * 32 * 16) + sizeof(int) * K_;
    launch_pdl(zscreen_t_kernel<R, TFR>, dim3(g), dim3(32 * zt_warps_), sm, st, a, static_cast<const std::int64_t*>(out.iter));
  }

  template <bool TFR>
  void zscreen_t_rounds(const LdaArgs& a, cudaStream_t st) {
    switch (RS_) {
      case 1: zscreen_t_launch<1, TFR>(a, st); break;
      case 2: zscreen_t_launch<2, TFR>(a, st); break;
      case 3: zscreen_t_launch<3, TFR>(a, st); break;
      default: zscreen_t_launch<4, TFR>(a, st); break;
    }
  }

  void launch_zscreen(const LdaArgs& a, cudaStream_t st) {
    if (!fq_reset_) BNMC_CUDA(cudaMemsetAsync(fq_len_.p, 0, sizeof(int), st));
    fq_reset_ = false;
    if (transposed_) {
      if (tfr_) zscreen_t_rounds<true>(a, st);
      else zscreen_t_rounds<false>(a, st);
      launch_fallback(a, st);
      return;
    }
    const int key = screen_key();
    if (wm_ && n_wm_units_ > 0) {
      LdaArgs aw = a;
      aw.units = wm_units_.p;
      aw.n_units = n_wm_units_;
      aw.wm_ticket = wm_ticket_.p;
      th32_kernel<<<148 * 16, 256, 0, st>>>(aw);
      BNMC_CUDA(cudaMemsetAsync(wm_ticket_.p, 0, sizeof(unsigned long long), st));
      switch (key) {
        case 841: zscreen_rounds<8, 4, true, true>(aw, st); break;
        case 1641: zscreen_rounds<16, 4, true, true>(aw, st); break;
        case 3241: zscreen_rounds<32, 4, true, true>(aw, st); break;
        default:
          if (wm_tfr_) zscreen_rounds<32, 8, true, true>(aw, st);
          else zscreen_rounds<32, 8, false, true>(aw, st);
          break;
      }
      launch_fallback(a, st);
      return;
    }
    switch (key) {
      case 441: zscreen_rounds<4, 4, true>(a, st); break;   // (G*CW < 32: experiments only)
      case 481: zscreen_rounds<4, 8, true>(a, st); break;
      case 480: zscreen_rounds<4, 8, false>(a, st); break;
      case 841: zscreen_rounds<8, 4, true>(a, st); break;
      case 840: zscreen_rounds<8, 4, false>(a, st); break;
      case 1641: zscreen_rounds<16, 4, true>(a, st); break;
      case 1640: zscreen_rounds<16, 4, false>(a, st); break;
      case 3241: zscreen_rounds<32, 4, true>(a, st); break;
      case 3240: zscreen_rounds<32, 4, false>(a, st); break;
      default: zscreen_rounds<32, 8, false>(a, st); break;
    }
    launch_fallback(a, st);
  }

  void launch_zstep(const LdaArgs& a, cudaStream_t st) {
    const unsigned g = static_cast<unsigned>(std::min<std::int64_t>(n_units_, 1 << 24));
    const std::size_t sm = zstep_smem();
    const int* err = out.err;
    const std::int64_t* it = out.iter;
    dispatch_zstep([&](auto gg, auto r, auto e) {
      constexpr int GG = decltype(gg)::value, RR = decltype(r)::value;
      constexpr bool EE = decltype(e)::value;
      if (screen_) {
        launch_zscreen(a, st);
        return;
      }
      if (theta_regs_)
        zstep_kernel<GG, RR, EE, true><<<g, kZThreads, sm, st>>>(a, it, const_cast<int*>(err));
      else
        zstep_kernel<GG, RR, EE, false><<<g, kZThreads, sm, st>>>(a, it, const_cast<int*>(err));
    });
  }

  // 1/x when it is exactly an integer in [2, 64] (the boost exponent), else 0
  static int exact_int_inverse(double x) {
    if (!(x > 0.0)) return 0;
    const double inv = 1.0 / x;
    return (inv == std::floor(inv) && inv >= 2.0 && inv <= 64.0) ? static_cast<int>(inv) : 0;
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
    a.phiT32 = screen_ ? phiT32_.p : nullptr;
    a.Kp32 = Kp32_;
    a.G32 = G32_;
    a.R32 = RS_;
    a.CW32 = CW32_;
    a.col_stripes = col_stripes_;
    // the log phi table feeds the unscreened log-space z-step only (the screened mode's
    // fallback takes the logs of its few tokens' rows itself)
    a.logphiT = exact_ && !screen_ ? logphiT_.p : nullptr;
    a.theta = theta_.p;
    a.nkw = nkw_.p;
    a.colpart2 = colpart2_.p;
    a.S = S_.p;
    a.phi_term = phi_term_.p;
    a.doc_part = doc_part_.p;
    a.red = red_.p;
    a.nmk = nmk_.p;
    a.units = units_.p;
    a.n_units = n_units_;
    a.wunits = wunits_.p;
    a.n_wunits = n_wunits_;
    a.tpart = tpart_.p;
    a.zpart = zpart_.p;
    a.wpart = wpart_.p;
    a.ttpart = ttpart_.p;
    a.alpha = alpha_;
    a.beta = beta_;
    a.pow_alpha = boost_pow_ ? exact_int_inverse(alpha_) : 0;
    a.pow_beta = boost_pow_ ? exact_int_inverse(beta_) : 0;
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
    a.logS = logS_.p;
    a.logg_valid = 0;
    a.spart = spart_.p;
    a.ticket = ticket_.p;
    a.ticket2 = ticket_.p + (K_ + 31) / 32;
    a.nb_phi = nb_phi_;
    a.docs_per_block = docs_per_block_;
    a.nb_doc = nb_doc_;
    a.nbw = nbw_;
    a.screen_margin = screen_margin_;
    a.fq = fq_.p;
    a.fq_len = fq_len_.p;
    a.wm_tok = wm_tok_.p;
    a.wm_doc = wm_doc_.p;
    a.th32 = th32_.p;
    a.thS = wm_ && n_wm_units_ > 0 ? thS_.p : nullptr;
    return a;
  }

  Comm comm_;
  int K_ = 0, Kp_ = 0, V_ = 0, G_ = 4, R_ = 8;
  std::int64_t M_ = 0, N_ = 0, d0_ = 0, d1_ = 0, Ml_ = 0, Nl_ = 0, tok0_ = 0;
  std::vector<std::int64_t> off_host_;
  bool exact_ = false, observe_phi_ = false, theta_regs_ = false, screen_ = false;
  int Kp32_ = 0, RS_ = 1, G32_ = 8, CW32_ = 4;
  bool tfr_ = true, transposed_ = false;
  DevBuf<float> phiT32_;
  cudaStream_t copy_ = nullptr;
  // speculative sweep_store
  cudaStream_t up_ = nullptr;
  cudaEvent_t ev_up_ = nullptr;
  DevBuf<std::int64_t> up64_;
  DevBuf<int> zprev_, spec_flag_;
  int* spec_flag_host_ = nullptr;
  bool zprev_valid_ = false, speculate_ = true;
  cudaEvent_t ev_phi_ready_ = nullptr, ev_theta_ready_ = nullptr, ev_copy_done_ = nullptr;
  double alpha_ = 0.1, beta_ = 0.1, phi_norm_ = 0, phi_lgasum_ = 0, theta_norm_ = 0, theta_lgasum_ = 0;
  std::uint64_t seed_ = 0;
  int var_phi_ = 0, var_theta_ = 1, var_z_ = 2, var_w_ = 3;
  int phi_threads_ = 128, rows_per_block_ = 1, nb_phi_ = 1;
  std::vector<std::int64_t> units_host_;
  std::int64_t n_units_ = 0, docs_per_block_ = 1, nb_doc_ = 0, n_wunits_ = 0;
  DevBuf<std::int64_t> wunits_;
  bool zt_wu_ = true;
  int nbw_ = 1, col_stripes_ = kColStripes;
  float screen_margin_ = kScreenMargin;
  bool fq_reset_ = false;  // phi_colsum2 of this sweep zeroes the fallback queue
  int fb_blocks_ = 148 * 12;  // zfallback_kernel grid
  // word-major z-step order (build_word_major)
  bool wm_ = false, wm_tfr_ = !(std::getenv("BNMC_WM_TFR") && std::string(std::getenv("BNMC_WM_TFR")) == "0");
  std::int64_t wm_block_docs_ = 1, n_wm_units_ = 0;
  DevBuf<int> wm_tok_, wm_doc_;
  DevBuf<std::int64_t> wm_units_;
  DevBuf<float> th32_;
  DevBuf<double> thS_;
  DevBuf<unsigned long long> wm_ticket_;

  // cudaLaunchKernelEx with programmatic stream serialization (PDL): the kernel's
  // launch overlaps the predecessor's tail; it calls pdl_wait() before its inputs.
  template <class... KArgs, class... Args>
  void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_ ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    BNMC_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
  }
  bool pdl_ = true;
  int zt_warps_ = 8;
  DevBuf<int2> fq_;
  DevBuf<int> fq_len_;
  bool data_on_device_ = false;
  DevBuf<std::int64_t> stage64_;  // int64 <-> int32 staging for z / w
  DevBuf<double> stage_phi_;      // K x V staging for the phi transpose
  DevBuf<int> w_, z_, nkw_, nmk_;
  DevBuf<std::int64_t> units_;
  DevBuf<std::int64_t> off_;
  bool boost_pow_ = std::getenv("BNMC_BOOST_POW") == nullptr || std::string(std::getenv("BNMC_BOOST_POW")) != "0";
  int pool_blocks_ = 148;
  int slice_ = 1, pv0_ = 0, pv1_ = 1;  // phi rows per rank, this rank's rows [pv0_, pv1_)
  std::int64_t Vpad_ = 1;
  int trow_blocks_ = 1;   // phi_colsum2 y-blocks for the pool's theta rows
  DevBuf<double> spart_, logS_, ttpart_;
  DevBuf<int> ticket_;
  DevBuf<double> phiT_, logphiT_, theta_, colpart2_, S_, phi_term_, doc_part_, red_, tpart_,
      zpart_, wpart_;
};

}  // namespace

std::unique_ptr<Model> make_lda(const bnmc_gpu_desc& d, const Comm& c, Outputs o) {
  return std::make_unique<Lda>(d, c, o);
}

}  // namespace bnmc_gpu
