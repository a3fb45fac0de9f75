// csrc/lda.cu -- LDA uncollapsed Gibbs sweep on sm_100a (proj/models/lda.bn).
//
// One reference sweep (Engine::sweep, proj/src/sampler.cpp:390-405; plan order
// phi, theta, z per tests/golden/describe_lda.txt) becomes, per GPU:
//
//   [allreduce nkw]      NCCL int32 sum of the topic-word counts (world > 1 only)
//   phi_gamma_kernel     phi block draw: per cell Gamma(beta + n[k,v]) from stream
//                        keyed(seed,4,var_phi,iter).derive(k,v) (batch.cpp:38-41);
//                        consumes the counts (zeroes them for this sweep's z-step)
//   colsum_kernel        row sums of the gamma matrix (fixed-order, deterministic)
//   phi_norm_kernel      phi = g / sum (batch.cpp:58-61) + Dirichlet log-pdf pieces
//   phi_terms_kernel     per-topic Dirichlet log-pdf (dist.cpp:115-130)
//   theta_kernel         theta block: per document Dirichlet(alpha + n[d,.]) from the
//                        doc-topic counts the previous z-step left (sampler.cpp:61-181),
//                        stream keyed(seed,4,var_theta,iter).derive(d,k); theta log-pdf
//   zstep_kernel         z block (sampler.cpp:222-265, draw_from_log_weights
//                        dist.cpp:202-215) over token chunks: new z, the NEXT sweep's
//                        topic-word and doc-topic counts (integer atomics), and the
//                        z-factor of the log-joint (sum log theta[d, z])
//   wterm_kernel         w-factor of the log-joint from the counts:
//                        sum_t log phi[z_t, w_t] = sum_{k,v} n[k,v] log phi[k,v]
//   reduce_kernel        fixed-order sums of the theta / z / w pieces
//   [allreduce 3 doubles]
//   finalize_kernel      log-joint = ((F_phi + F_theta) + F_z) + F_w (eval.cpp:393-422)
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
  unsigned short* phiT16;    // fp16 row-scaled copy [V][Kp16], columns permuted by phys16 (level-1 screen)
  int Kp16, RH;              // Kp16 = 64 RH
  float* thS32;              // [Ml][K8] theta/S in fp32 (level-1 units -> level 2)
  int2* q2;                  // level-2 queue (t, m)
  int* q2_len;
  int col_stripes;           // phi_colsum2 stripe blocks (extra y-blocks convert phiT16 rows)
  double* logphiT;   // exact mode only
  double* theta;
  int* nkw;          // [V][Kp]
  int* nmk;          // [Ml][K]
  double* colpart;   // [nb_phi][K]
  double* colpart2;  // [nb_phi][K][2]
  double* S;         // [K]
  double* phi_term;  // [K]
  double* tpart;     // [Ml] theta-factor pieces
  double* zpart;     // [nbw] z-factor pieces (sum n[d,k] log theta[d,k]) per wterm block
  double* logg;      // [V][Kp] log of this sweep's gamma draws (phi block v2)
  double* logS;      // [K] log of the gamma row sums
  int logg_valid;    // logg/logS belong to the current phi (set inside a v2 sweep)
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
  int phi_pf;               // phi_gamma2: count prefetch distance in blocks; phi_pool: in grid-widths of groups (0: off)
  double phi_norm, phi_lgasum, theta_norm, theta_lgasum;
  std::uint64_t seed;
  std::uint64_t zkey_prefix;  // fold(fold(fold(1, seed), kDiscrete), var_z)
  int var_phi, var_theta, var_z;
  int rows_per_block, nb_phi;
  double* gpart;     // [nvb][K] phi block v2 partials: sum g, sum log g
  double* lpart;
  std::int64_t nvb;
  double* spart;     // [kColStripes][K][2]
  int* ticket;       // [ceil(K/32)] last-block tickets of phi_colsum2
  int* ticket2;      // last-block ticket of wterm_kernel<true>
  int red_only;      // sharded: the last wterm block writes red[0..2] (this rank's theta, z, w
                     // pieces) for the all-reduce instead of the log-joint
  std::int64_t docs_per_block, nb_doc;
};

// ---------------------------------------------------------------------------------
// phi block
// ---------------------------------------------------------------------------------
// Block b owns vocabulary rows [b*R, b*R + R); its threads sweep the R x K cells
// (k fastest: coalesced phiT rows), then threads k < K sum their column over the
// block's rows in fixed order -> colpart[b][k].
__global__ void __launch_bounds__(256) phi_gamma_kernel(LdaArgs a, const std::int64_t* iter_p) {
  const std::int64_t iter = *iter_p;
  const std::uint64_t key = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_phi),
                                  static_cast<std::uint64_t>(iter));
  const int b = blockIdx.x;
  const int v0 = b * a.rows_per_block;
  const int v1 = min(a.V, v0 + a.rows_per_block);
  const int cells = (v1 - v0) * a.K;
  // The counts come from HBM at the start of a sweep: issue the thread's count loads
  // up front (<= 4 cells per thread at the configured rows per block) before the
  // latency-bound gamma draws.
  int n[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = threadIdx.x + j * blockDim.x;
    n[j] = 0;
    if (c < cells) {
      const std::size_t i = static_cast<std::size_t>(v0 + c / a.K) * a.Kp + c % a.K;
      n[j] = a.nkw[i];
      a.nkw[i] = 0;
    }
  }
  for (int c = threadIdx.x, j = 0; c < cells; c += blockDim.x, ++j) {
    const int v = v0 + c / a.K, k = c % a.K;
    const std::size_t i = static_cast<std::size_t>(v) * a.Kp + k;
    int cnt;
    if (j < 4) {
      cnt = n[0];
      if (j == 1) cnt = n[1];
      if (j == 2) cnt = n[2];
      if (j == 3) cnt = n[3];
    } else {
      cnt = a.nkw[i];
      a.nkw[i] = 0;
    }
    Stream r(derive(key, static_cast<std::uint64_t>(k), static_cast<std::uint64_t>(v)));
    const double g = draw_gamma(r, a.beta + static_cast<double>(cnt));
    a.phiT[i] = g;
    if (a.phiT32) a.phiT32[static_cast<std::size_t>(v) * a.Kp32 + phys32(k, a.R32, a.G32, a.CW32)] = static_cast<float>(g);
  }
  __syncthreads();
  // Column partials of the block's rows, fixed order: sum g (the Dirichlet row sum,
  // batch.cpp:55-58) and sum log g (the phi factor of the log-joint without a
  // normalisation pass: sum log(g/S) = sum log g - V log S).
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    double sg = 0.0, sl = 0.0;
    for (int v = v0; v < v1; ++v) {
      const double g = a.phiT[static_cast<std::size_t>(v) * a.Kp + k];
      sg += g;
      sl += g > 0.0 ? log(g) : -INFINITY;
    }
    a.colpart[static_cast<std::size_t>(b) * a.K + k] = sg;
    a.colpart2[(static_cast<std::size_t>(b) * a.K + k) * 2] = sl;
  }
}

// phi block, v2: thread (k, vb) draws the cells (v, k), v in [vb*L, vb*L + L), of one
// topic column in order and keeps fixed-order partials of sum g and sum log g.
// * Rejection sampling without warp-level waste: the Marsaglia-Tsang loop runs one
//   attempt per iteration and a thread whose attempt is accepted moves straight on
//   to its next cell, so a warp iterates ~(1 + reject rate) * L times instead of
//   L * (max attempts over the warp) (ncu r01 v6: the per-cell loop executed
//   ~1290 thread instructions per cell, ~2.5x the straight-line count).
// * Per-count constants d = a - 1/3, c = 1/sqrt(9d), 1/shape for counts < 64 come
//   from a shared table computed with the reference's expressions (dist.cpp:136-155;
//   bit-identical), saving a sqrt and two divisions per cell.
// * log g is stored per cell (logg): the w-factor of the log-joint then needs no
//   transcendental after the z-step.
// The stream of every cell is keyed(seed, 4, var_phi, iter).derive(k, v) and is
// consumed in the reference's order (gaussian until 1 + c x > 0, uniform, [boost
// uniform]), so the draws are the reference's.
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
constexpr int kPhiRowsMax = 8;  // L: cells per thread (8, or fewer for small K x V)

template <int kPhiRows>
__global__ void __launch_bounds__(256) phi_gamma2_kernel(LdaArgs a, const std::int64_t* iter_p) {
  __shared__ double tab_d[kGammaTab], tab_c[kGammaTab], tab_inv[kGammaTab];
  __shared__ int cnt_s[kPhiRows][256];  // the thread's counts, loaded up front
  const std::int64_t iter = *iter_p;
  for (int i = threadIdx.x; i < kGammaTab; i += blockDim.x) {
    const double shape = a.beta + static_cast<double>(i);
    const bool boost = shape < 1.0;
    const double aa = boost ? shape + 1.0 : shape;
    const double d = aa - 1.0 / 3.0;
    tab_d[i] = d;
    tab_c[i] = 1.0 / sqrt(9.0 * d);
    tab_inv[i] = boost ? 1.0 / shape : 0.0;
  }
  __syncthreads();
  const std::int64_t idx = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int k = static_cast<int>(idx % a.K);
  const std::int64_t vb = idx / a.K;
  if (vb >= a.nvb) return;
  const int v0 = static_cast<int>(vb * kPhiRows), v1 = min(a.V, v0 + kPhiRows);
#pragma unroll
  for (int j = 0; j < kPhiRows; ++j) {
    if (v0 + j < v1) {
      const std::size_t i = static_cast<std::size_t>(v0 + j) * a.Kp + k;
      cnt_s[j][threadIdx.x] = a.nkw[i];
      a.nkw[i] = 0;  // consumed: the z-step accumulates the next sweep's counts here
    }
  }
  // The counts of the block ~0.7 resident waves later (a.phi_pf blocks on), into L2 while
  // this block draws: the next wave then starts from L2 instead of HBM (the bench flushes
  // L2 before every sweep; r01: phi 73 -> 66 us on NIPS).
  if (a.phi_pf > 0) {
    const std::int64_t idx2 = idx + static_cast<std::int64_t>(a.phi_pf) * blockDim.x;
    const std::int64_t vb2 = idx2 / a.K;
    if (vb2 < a.nvb) {
      const int k2 = static_cast<int>(idx2 % a.K);
#pragma unroll
      for (int j = 0; j < kPhiRows; ++j) {
        const std::int64_t v2 = vb2 * kPhiRows + j;
        if (v2 < a.V) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.nkw + static_cast<std::size_t>(v2) * a.Kp + k2));
      }
    }
  }
  const int col32 = a.phiT32 ? phys32(k, a.R32, a.G32, a.CW32) : 0;
  pdl_trigger();
  const std::uint64_t kkey = fold(keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_phi),
                                        static_cast<std::uint64_t>(iter)),
                                  static_cast<std::uint64_t>(k));
  double sg = 0.0, sl = 0.0;
  int v = v0;
  bool fresh = true;
  Stream r(0);
  double d = 1.0, c = 1.0, inv = 0.0;
  while (v < v1) {
    if (fresh) {
      const int n = cnt_s[v - v0][threadIdx.x];
      r = Stream(fold(kkey, static_cast<std::uint64_t>(v)));
      if (n < kGammaTab) {
        d = tab_d[n];
        c = tab_c[n];
        inv = tab_inv[n];
      } else {
        const double shape = a.beta + static_cast<double>(n);  // >= 64: no boost
        d = shape - 1.0 / 3.0;
        c = 1.0 / sqrt(9.0 * d);
        inv = 0.0;
      }
      fresh = false;
    }
    const double x = r.next_gaussian();
    double vv = 1.0 + c * x;
    if (vv > 0.0) {
      vv = vv * vv * vv;
      const double u = r.next_unit();
      bool acc = u < 1.0 - 0.0331 * (x * x) * (x * x);
      if (!acc) acc = log(u) < 0.5 * x * x + d * (1.0 - vv + log(vv));
      if (acc) {
        double g = d * vv;
        // the reference's boost g * pow(u, 1/shape) (dist.cpp:139-140) as exp(log(u) / shape):
        // |log u / shape| <= 37 / shape, so the relative difference from a correctly
        // rounded pow is <= ~2^-53 * 37 / shape (4e-14 at shape 0.1), far inside the 1e-12
        // contract, and exp + log cost half of pow's double-double path (r01 v33: phi
        // block 83 -> 77 us on NIPS)
        if (inv != 0.0) g = g * boost_factor(r.next_unit(), a.pow_beta, inv);
        const std::size_t i = static_cast<std::size_t>(v) * a.Kp + k;
        a.phiT[i] = g;
        if (a.phiT32) a.phiT32[static_cast<std::size_t>(v) * a.Kp32 + col32] = static_cast<float>(g);
        sg += g;
        // log g: the phi prior term here, the w-factor after the z-step (wterm_kernel)
        const double lg = g > 0.0 ? log(g) : -INFINITY;
        a.logg[i] = lg;
        sl += lg;
        ++v;
        fresh = true;
      }
    }
  }
  a.gpart[vb * a.K + k] = sg;
  a.lpart[vb * a.K + k] = sl;
}

// phi block, v3 ("warp pool"): a persistent grid (one resident wave) in which warp w
// owns the contiguous cell range [w C / W, (w+1) C / W) of the C = V K cells (k
// fastest, the phiT row order), so every warp has the same number of cells.  The 32
// lanes draw the range as one pool, <= kPoolCells cells (one shared-memory chunk of
// counts) at a time: every iteration each lane makes one Marsaglia-Tsang attempt on
// its current cell, and the lanes whose attempt was accepted take the next undrawn
// cells (ballot + prefix rank).  A warp iterates ~(cells x 1.06) / 32 times with all
// lanes busy until the chunk's last attempts -- the v2 kernel's lanes each ran their
// own cells' rejection sequences and waited for the slowest lane of the warp (ncu
// r01: ~930 thread instructions per cell, 20.7 of 32 lanes active per instruction)
// and its 1.64-wave grid left a tail.
// * No column partials and no per-cell log here: phi_colsum2<true> sums the columns of
//   phiT directly (sum g, and sum log g as the log of a frexp-renormalised product),
//   and the log-joint's w-factor takes log g of the counted cells (wterm_kernel).
// * Streams keyed(seed, 4, var_phi, iter).derive(k, v), consumed in the reference's
//   order (gaussian until 1 + c x > 0, uniform, [boost uniform]; dist.cpp:136-155):
//   the draws are the reference's whichever lane draws a cell.
constexpr int kPoolCells = 1024;
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
  // cells [0, cphi): phi (v, k) in phiT row order; [cphi, cphi + Ml K): theta (m, k)
  const std::int64_t cphi = a.pool_phi ? static_cast<std::int64_t>(a.V) * a.K : 0;
  const std::int64_t ncells = cphi + a.Ml * a.K;
  const std::int64_t nw = static_cast<std::int64_t>(gridDim.x) * (blockDim.x >> 5);
  const std::int64_t gw = static_cast<std::int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const std::int64_t c_end = ncells * (gw + 1) / nw;
  auto count_at = [&](std::int64_t c) -> int* {
    if (c >= cphi) return a.nmk + (c - cphi);
    int v, k;
    cell_vk(c, a.K, invK, v, k);
    return a.nkw + static_cast<std::size_t>(v) * a.Kp + k;
  };
  for (std::int64_t c0 = ncells * gw / nw; c0 < c_end; c0 += kPoolCells) {
    const int n = static_cast<int>(c_end - c0 < kPoolCells ? c_end - c0 : kPoolCells);
    // the chunk's counts into shared memory (consumed: the z-step accumulates the next
    // sweep's counts here), 8 loads in flight per lane before the zeroing stores (the
    // stores may alias the next loads: a load-store loop would serialise one HBM round
    // trip per 32 cells); the next chunk's counts into L2 meanwhile
    for (int j0 = 0; j0 < n; j0 += 8 * 32) {
      int val[8];
      int* at[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = j0 + 32 * i + lane;
        val[i] = 0;
        at[i] = nullptr;
        if (j < n) {
          at[i] = count_at(c0 + j);
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
    if (c0 + kPoolCells + 32 * lane < c_end)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(count_at(c0 + kPoolCells + 32 * lane)));
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
          const std::int64_t cell = c0 + j;
          const int cn = cnt[j];
          const int kind = cell >= cphi;
          int v, k;
          if (!kind) {  // phi cell (v, k): Stream(derive(base, k, v))
            cell_vk(cell, a.K, invK, v, k);
            pos = fold(KTAB ? kkey_s[k] : fold(base, static_cast<std::uint64_t>(k)), static_cast<std::uint64_t>(v));
            outp = a.phiT + static_cast<std::size_t>(v) * a.Kp + k;
            out32 = a.phiT32 ? a.phiT32 + static_cast<std::size_t>(v) * a.Kp32 +
                                   (KTAB ? col32_s[k] : phys32(k, a.R32, a.G32, a.CW32))
                             : nullptr;
            pw = a.pow_beta;
          } else {  // theta cell (m, k): Stream(derive(tbase, doc_base + m, k)), g unnormalised
            cell_vk(cell - cphi, a.K, invK, v, k);
            pos = fold(fold(tbase, static_cast<std::uint64_t>(a.doc_base + v)), static_cast<std::uint64_t>(k));
            outp = a.theta + (cell - cphi);
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
          if (!acc) acc = log(u) < 0.5 * x * x + d * (1.0 - vv + log(vv));
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

// Per topic: S[k] = sum over vb of gpart and the phi factor
// (beta-1) (sum log g - V log S) - sum lgamma(beta) + lgamma(sum beta)
// (dist.cpp:115-130).  Grid (ceil(K/32), kColStripes): block (kb, s) sums stripe s of
// the row blocks for 32 topics (threads 32 x 8, fixed-order smem reduction) into
// spart[s][k]; the last stripe block of kb to finish (atomic ticket) adds the
// stripes in stripe order.  The ticket decides who adds, never the order, so the
// result is deterministic.
constexpr int kColStripes = 128;

__device__ void h16_rows(const LdaArgs& a, std::int64_t w0, std::int64_t nw);

// Blocks with blockIdx.y >= col_stripes convert the new phi rows to fp16 for the
// level-1 screen (h16_rows) -- the conversion needs the rows, not S, so it runs beside
// the column sums instead of after them.
// FROM_G (warp-pool phi block): the stripes sum the columns of phiT itself (rows v,
// stride Kp): sum g, and sum log g as log(mantissa product) + exponent sum
// (frexp-renormalised after every factor: one log per thread and column instead of one
// per cell).  Otherwise the v2 kernel's row-block partials gpart / lpart.
struct LogProd {
  double mant = 1.0;
  int ex = 0;
  bool zero = false;
  __device__ __forceinline__ void mul(double g) {
    if (g > 0.0) {
      int e1, e2;
      mant = frexp(mant * frexp(g, &e1), &e2);
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

template <bool FROM_G>
__global__ void __launch_bounds__(256) phi_colsum2_kernel(LdaArgs a) {
  __shared__ double sg_s[8][33], sl_s[8][33];
  __shared__ bool last;
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {  // this sweep's redraw queues
    if (a.fq_len) *a.fq_len = 0;
    if (a.q2_len) *a.q2_len = 0;
  }
  const int stripes = a.col_stripes;
  if (static_cast<int>(blockIdx.y) >= stripes + a.trow_blocks) {
    const std::int64_t hb = static_cast<std::int64_t>(blockIdx.y - stripes - a.trow_blocks) * gridDim.x + blockIdx.x;
    const std::int64_t nhb = static_cast<std::int64_t>(gridDim.y - stripes - a.trow_blocks) * gridDim.x;
    h16_rows(a, hb * 8 + (threadIdx.x >> 5), nhb * 8);
    return;
  }
  if (static_cast<int>(blockIdx.y) >= stripes) {  // theta rows of the warp-pool block
    const std::int64_t w0 = (static_cast<std::int64_t>(blockIdx.y - stripes) * gridDim.x + blockIdx.x) * 8 + (threadIdx.x >> 5);
    const std::int64_t nwr = static_cast<std::int64_t>(a.trow_blocks) * gridDim.x * 8;
    for (std::int64_t m = w0; m < a.Ml; m += nwr) theta_row_finish(a, m);
    return;
  }
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + tx;
  const std::int64_t rows = FROM_G ? a.V : a.nvb;
  const std::int64_t chunk = (rows + stripes - 1) / stripes;
  const std::int64_t b0 = blockIdx.y * chunk, b1 = min(rows, b0 + chunk);
  double sg = 0.0, sl = 0.0;
  if (k < a.K) {
    if constexpr (FROM_G) {
      LogProd lp;
      std::int64_t b = b0 + ty;
      for (; b < b1; b += 64) {  // 8 loads in flight
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
    } else {
      std::int64_t b = b0 + ty;
      for (; b + 56 < b1; b += 64) {  // 8 independent loads in flight per operand
        double g8[8], l8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          g8[j] = a.gpart[(b + 8 * j) * a.K + k];
          l8[j] = a.lpart[(b + 8 * j) * a.K + k];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          sg += g8[j];
          sl += l8[j];
        }
      }
      double g8[8], l8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {  // the remaining < 8 rows of this thread, loads issued together
        const std::int64_t bj = b + 8 * j;
        g8[j] = bj < b1 ? a.gpart[bj * a.K + k] : 0.0;
        l8[j] = bj < b1 ? a.lpart[bj * a.K + k] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sg += g8[j];
        sl += l8[j];
      }
    }
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

// Per topic: S[k] = sum_b colpart (the gamma row sum) and the phi factor
// lp - sum lgamma(beta) + lgamma(sum beta) with lp = (beta-1) (sum log g - V log S)
// (dist.cpp:115-130; sum phi = sum g / S = 1 by construction).
__global__ void phi_colsum_terms_kernel(LdaArgs a) {
  __shared__ double scratch[32];
  const int k = blockIdx.x;
  double sg = 0.0, sl = 0.0;
  for (int b = threadIdx.x; b < a.nb_phi; b += blockDim.x) {
    sg += a.colpart[static_cast<std::size_t>(b) * a.K + k];
    sl += a.colpart2[(static_cast<std::size_t>(b) * a.K + k) * 2];
  }
  sg = block_sum(sg, scratch);
  sl = block_sum(sl, scratch);
  if (threadIdx.x == 0) {
    a.S[k] = sg;
    const double lp = (a.beta - 1.0) * (sl - static_cast<double>(a.V) * log(sg));
    a.phi_term[k] = (!(sg > 0.0) || !(a.beta > 0.0)) ? -INFINITY : lp - a.phi_norm + a.phi_lgasum;
  }
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
      if (NORMALISE) a.phiT[c] = x;
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
// theta block: one CTA per document row
// ---------------------------------------------------------------------------------
__global__ void theta_kernel(LdaArgs a, const std::int64_t* iter_p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* g = reinterpret_cast<double*>(smem_raw);  // [K]
  __shared__ double scratch[32];
  const std::int64_t iter = *iter_p;
  const std::uint64_t tkey = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_theta),
                                   static_cast<std::uint64_t>(iter));
  for (std::int64_t m = blockIdx.x; m < a.Ml; m += gridDim.x) {
    const std::uint64_t mg = static_cast<std::uint64_t>(a.doc_base + m);
    int* cnt = a.nmk + m * a.K;
    double part = 0.0;
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
      const int n = cnt[k];
      cnt[k] = 0;  // consumed: the z-step accumulates the next sweep's counts here
      Stream r(derive(tkey, mg, static_cast<std::uint64_t>(k)));
      const double x = draw_gamma(r, a.alpha + static_cast<double>(n));
      g[k] = x;
      part += x;
    }
    const double S = block_sum(part, scratch);
    double lp = 0.0, sx = 0.0;
    for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
      const double x = g[k] / S;
      a.theta[m * a.K + k] = x;
      lp += (a.alpha - 1.0) * (x > 0.0 ? log(x) : -INFINITY);
      sx += x;
    }
    lp = block_sum(lp, scratch);
    sx = block_sum(sx, scratch);
    if (threadIdx.x == 0)
      a.tpart[m] = fabs(sx - 1.0) > 1e-9 ? -INFINITY : lp - a.theta_norm + a.theta_lgasum;
    __syncthreads();
  }
}

// theta block, v2: the phi_gamma2 scheme on document rows.  A block holds `dpb`
// documents; each document row is split into runs of TL consecutive topics, one
// run per thread (persistent rejection loop, counts prefetched to shared memory,
// shared per-count constants).  Per document: S = sum g (fixed order: thread runs
// in order), theta = g / S, and the Dirichlet log-pdf via
// sum log theta = sum log g - K log S with sum log g from renormalised products.
// Streams keyed(seed, 4, var_theta, iter).derive(d, k) as the reference (batch.cpp:38-41).
constexpr int kThetaRun = 4;

__global__ void __launch_bounds__(256) theta2_kernel(LdaArgs a, const std::int64_t* iter_p, int tpd, int dpb) {
  __shared__ double tab_d[kGammaTab], tab_c[kGammaTab], tab_inv[kGammaTab];
  __shared__ int cnt_s[kThetaRun][256];
  __shared__ double g_s[kThetaRun][256];
  __shared__ double ps[256], pl[256], dS[256];
  const std::int64_t iter = *iter_p;
  for (int i = threadIdx.x; i < kGammaTab; i += blockDim.x) {
    const double shape = a.alpha + static_cast<double>(i);
    const bool boost = shape < 1.0;
    const double aa = boost ? shape + 1.0 : shape;
    const double d = aa - 1.0 / 3.0;
    tab_d[i] = d;
    tab_c[i] = 1.0 / sqrt(9.0 * d);
    tab_inv[i] = boost ? 1.0 / shape : 0.0;
  }
  const std::uint64_t tkey = keyed(a.seed, kConjugate, static_cast<std::uint64_t>(a.var_theta),
                                   static_cast<std::uint64_t>(iter));
  const int j = threadIdx.x / tpd, t = threadIdx.x - (threadIdx.x / tpd) * tpd;
  const std::int64_t m = static_cast<std::int64_t>(blockIdx.x) * dpb + j;
  const bool active = j < dpb && m < a.Ml;
  const int k0 = t * kThetaRun, k1 = active ? min(a.K, k0 + kThetaRun) : k0;
#pragma unroll
  for (int i = 0; i < kThetaRun; ++i) {
    if (k0 + i < k1) {
      int* c = a.nmk + m * a.K + k0 + i;
      cnt_s[i][threadIdx.x] = *c;
      *c = 0;  // consumed: the z-step accumulates the next sweep's counts here
    }
  }
  __syncthreads();
  const std::uint64_t mkey = fold(tkey, static_cast<std::uint64_t>(a.doc_base + m));
  double sg = 0.0, mant = 1.0;
  int ex = 0;
  bool zero = false;
  int k = k0;
  bool fresh = true;
  Stream r(0);
  double d = 1.0, c = 1.0, inv = 0.0;
  while (k < k1) {
    if (fresh) {
      const int n = cnt_s[k - k0][threadIdx.x];
      r = Stream(fold(mkey, static_cast<std::uint64_t>(k)));
      if (n < kGammaTab) {
        d = tab_d[n];
        c = tab_c[n];
        inv = tab_inv[n];
      } else {
        const double shape = a.alpha + static_cast<double>(n);
        d = shape - 1.0 / 3.0;
        c = 1.0 / sqrt(9.0 * d);
        inv = 0.0;
      }
      fresh = false;
    }
    const double x = r.next_gaussian();
    double vv = 1.0 + c * x;
    if (vv > 0.0) {
      vv = vv * vv * vv;
      const double u = r.next_unit();
      bool acc = u < 1.0 - 0.0331 * (x * x) * (x * x);
      if (!acc) acc = log(u) < 0.5 * x * x + d * (1.0 - vv + log(vv));
      if (acc) {
        double g = d * vv;
        // the reference's boost g * pow(u, 1/shape) (dist.cpp:139-140) as exp(log(u) / shape):
        // |log u / shape| <= 37 / shape, so the relative difference from a correctly
        // rounded pow is <= ~2^-53 * 37 / shape (4e-14 at shape 0.1), far inside the 1e-12
        // contract, and exp + log cost half of pow's double-double path (r01 v33: phi
        // block 83 -> 77 us on NIPS)
        if (inv != 0.0) g = g * boost_factor(r.next_unit(), a.pow_alpha, inv);
        g_s[k - k0][threadIdx.x] = g;
        sg += g;
        if (g > 0.0) {
          int e1, e2;
          mant = frexp(mant * frexp(g, &e1), &e2);
          ex += e1 + e2;
        } else {
          zero = true;
        }
        ++k;
        fresh = true;
      }
    }
  }
  ps[threadIdx.x] = sg;
  pl[threadIdx.x] = zero ? -INFINITY : log(mant) + static_cast<double>(ex) * 0.69314718055994530942;
  __syncthreads();
  if (active && t == 0) {  // document row sums, runs in topic order
    double S = 0.0, L = 0.0;
    for (int q = 0; q < tpd; ++q) {
      S += ps[threadIdx.x + q];
      L += pl[threadIdx.x + q];
    }
    dS[j] = S;
    // sum log theta = sum log g - K log S;  sum theta = 1 by construction
    const double lp = (a.alpha - 1.0) * (L - static_cast<double>(a.K) * log(S));
    a.tpart[m] = (!(S > 0.0) || !isfinite(S)) ? -INFINITY : lp - a.theta_norm + a.theta_lgasum;
  }
  __syncthreads();
  if (active) {
    const double S = dS[j];
    for (int kk = k0; kk < k1; ++kk) a.theta[m * a.K + kk] = g_s[kk - k0][threadIdx.x] / S;
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
// Error budget: every screen partial sum is within (8 + R + log2 G + 4) * 2^-24 *
// total of the exact cumulative weight (non-negative terms, fma chains); with
// G <= 32, R <= 8 that is < 2^-19 * total, 8x below the 2^-16 margin.

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
template <int G, int CW, int R, bool TFR>
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

  for (std::int64_t unit = blockIdx.x; unit < a.n_units; unit += gridDim.x) {
    const std::int64_t m = a.units[unit * 3], t0 = a.units[unit * 3 + 1], t1 = a.units[unit * 3 + 2];
    const double* thg = a.theta + m * a.K;
    for (int k = threadIdx.x; k < G * KL; k += blockDim.x)
      thf[(k / KL) * KLP + k % KL] = k < a.K ? static_cast<float>(thg[k] / a.S[k]) : 0.0f;
    __syncthreads();
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
    int* cnt = a.nmk + m * a.K;
    for (std::int64_t b0 = t0 + warp * 32; b0 < t1; b0 += kWarps * 32) {
      // token b0 + lane: its word and its uniform, keyed(seed, 3, var_z, t, iter)
      const std::int64_t tl = b0 + lane;
      const bool lvalid = tl < t1;
      const int wl = lvalid ? __ldg(a.w + tl) : 0;
      float ul = 0.5f;
      if (lvalid) {
        Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + tl)),
                        static_cast<std::uint64_t>(iter)));
        ul = static_cast<float>(rng.next_unit());
      }
#pragma unroll 1
      for (int s = 0; s < G; ++s) {
        if (b0 + s * (32 / G) >= t1) break;  // warp-uniform: no token left in this sub-batch
        const int src = s * (32 / G) + gid;  // lane holding this group's token
        const std::int64_t t = b0 + src;
        const bool valid = t < t1;
        const int wv = __shfl_sync(0xffffffffu, wl, src);
        const float u01 = __shfl_sync(0xffffffffu, ul, src);
        const float* row = a.phiT32 + static_cast<std::size_t>(wv) * a.Kp32;
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
          if (j >= 0 && kl0 + j < a.K && uf - prev >= mg && acc - uf >= mg) k = kl0 + j;
        }
        const bool decided = ((__ballot_sync(0xffffffffu, k >= 0) >> gshift) & gbits) != 0;
        if (valid) {
          if (k >= 0) {
            a.z[t] = k;
            atomicAdd(&a.nkw[static_cast<std::size_t>(wv) * a.Kp + k], 1);
            atomicAdd(&cnt[k], 1);
          } else if (!decided && gl == 0) {
            // ambiguous for the screen: queued for the fp64 draw (zfallback_kernel)
            const int slot = atomicAdd(a.fq_len, 1);
            a.fq[slot] = make_int2(static_cast<int>(t), static_cast<int>(m));
          }
        }
      }
    }
    __syncthreads();
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

// ---------------------------------------------------------------------------------
// z block, two-level screen (experimental, BNMC_ZSCREEN_H=1): fp16 rows, then fp32, then fp64
// ---------------------------------------------------------------------------------
// The z-step moves one phi row per token from L2 (ncu r01: at the L2 read bandwidth),
// so the row bytes set its time.  Level 1 reads the rows in fp16 (phiT16: 2 bytes per
// candidate, half of phiT32) with theta/S in fp16 and FHFMA (fp16 x fp16 products,
// exact in fp32, fp32 accumulation):
//  * per-row scale c_v and per-document scale a_d (powers of two) put each row's and
//    document's maximum in [2^14, 2^15) -- the draw does not depend on them (both
//    scale every weight of the token alike);
//  * error of every level-1 prefix / total / u * total against the exact scaled value:
//    quantisation of both factors 2^-11 + 2^-11 relative (normal range) or 2^-25
//    absolute per factor (fp16 subnormals), fp32 rounding <= 24 * 2^-24 relative, so
//    <= 2^-9.9 * value + A with A = 2^-24 (32768 K + Theta_d), Theta_d = sum of the
//    document's fp16 theta values (every fp16 value <= 2^15);
//  * a token is decided when u * total lies >= mg1 = 2^-8.5 * uf + 4 A inside its
//    candidate's interval (covers both boundaries' and uf's errors);
//    otherwise it is queued for level 2 (q2).
// Level 2 (zscreen_q_kernel) redraws the queued tokens with the fp32 transposed screen
// (phiT32 rows, theta/S rows the level-1 units left in thS32) and queues what is still
// ambiguous for the fp64 draw (zfallback_kernel).  The pick is the fp64 product-form
// draw in every case.
__host__ __device__ __forceinline__ int phys16(int k, int RH) {
  const int c = k >> 4, j = k & 15, gl = c / RH, r = c - gl * RH;
  return ((r << 2) + gl) * 16 + j;
}

__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float c) {
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"(a), "h"(b));
  return c;
}

struct Oct16 {
  unsigned v[8];  // 16 halves
};

__device__ __forceinline__ Oct16 ldg256h(const unsigned short* p) {
  Oct16 o;
  asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(o.v[0]), "=r"(o.v[1]), "=r"(o.v[2]), "=r"(o.v[3]), "=r"(o.v[4]), "=r"(o.v[5]), "=r"(o.v[6]),
        "=r"(o.v[7])
      : "l"(p));
  return o;
}

// fp16 rows of the current phi numerator (phiT32 -> phiT16, row-scaled); warps w0,
// w0 + nw, ... of the caller each take one row at a time.  K <= 128.
__device__ void h16_rows(const LdaArgs& a, std::int64_t w0, std::int64_t nw) {
  // lane L holds phiT32 physical columns 4L .. 4L + 3 (one coalesced 16-byte load per
  // row; Kp32 <= 128); two rows per warp iteration
  const int lane = threadIdx.x & 31;
  const int p0 = 4 * lane;
  int kl[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {  // logical candidate of physical column p0 + j (phys32 inverse)
    const int p = p0 + j, c = p / a.CW32, jj = p - c * a.CW32, r = c / a.G32, gl = c - r * a.G32;
    kl[j] = (gl * a.R32 + r) * a.CW32 + jj;
  }
  const bool mine = p0 < a.Kp32;
  for (std::int64_t v0 = w0; v0 < a.V; v0 += 2 * nw) {
    float4 x[2];
    float mx[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const std::int64_t v = v0 + i * nw;
      x[i] = (mine && v < a.V) ? *reinterpret_cast<const float4*>(a.phiT32 + static_cast<std::size_t>(v) * a.Kp32 + p0)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // (padding columns hold 0)
      mx[i] = fmaxf(fmaxf(x[i].x, x[i].y), fmaxf(x[i].z, x[i].w));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], o));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const std::int64_t v = v0 + i * nw;
      if (!mine || v >= a.V) continue;
      const int e = mx[i] > 0.0f ? min(127, max(-126, 14 - ilogbf(mx[i]))) : 0;
      const float sc = ldexpf(1.0f, e);
      unsigned short* out = a.phiT16 + static_cast<std::size_t>(v) * a.Kp16;
      const float xv[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (kl[j] < a.K) out[phys16(kl[j], a.RH)] = __half_as_ushort(__float2half_rn(xv[j] * sc));
    }
  }
}

__global__ void __launch_bounds__(256) phi_h16_kernel(LdaArgs a) {
  const std::int64_t nw = static_cast<std::int64_t>(gridDim.x) * (blockDim.x >> 5);
  h16_rows(a, static_cast<std::int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5), nw);
}

// max / sum over a unit's team (a warp for warp units, the CTA otherwise)
template <bool WU>
__device__ __forceinline__ float team_max(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if constexpr (WU) return v;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  v = lane < nw ? red[lane] : 0.0f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <bool WU>
__device__ __forceinline__ float team_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if constexpr (WU) return v;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  v = lane < nw ? red[lane] : 0.0f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr float kL1Rel = 0.0027622f;  // level-1 margin relative to u * total (>= 2^-8.5)

// Level 1.  RH: 16-candidate rounds per lane (K <= 64 * RH); units as zscreen_t_kernel.
// Shared memory per team: thh [4][16 RH + 8] halves (fp16 theta/S * a_d), csum
// [warps][32][16] floats, cnt [K] ints, red [32] floats.
template <int RH, bool WU>
__global__ void __launch_bounds__(kZThreads, 3) zscreen_h_kernel(LdaArgs a, const std::int64_t* iter_p) {
  constexpr int G = 4, KLH = 16 * RH, KLHP = KLH + 8, C = G * RH;
  static_assert(C <= 16, "csum rows hold 16 chunk sums");
  const int kWarps = blockDim.x >> 5;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), gid = lane / G;
  const int warp = threadIdx.x >> 5;
  const int kpad = (a.K + 3) & ~3;
  // team area: [thh G*KLHP halves][csum][cnt kpad][red 32]
  const std::size_t team_floats = G * KLHP / 2 + (WU ? 32 * 16 : kWarps * 32 * 16) + kpad + 32;
  float* base = reinterpret_cast<float*>(smem_raw) + (WU ? warp * team_floats : 0);
  unsigned short* thh = reinterpret_cast<unsigned short*>(base);
  float* csum = base + G * KLHP / 2 + (WU ? 0 : warp * 32 * 16);
  int* cnt_s = reinterpret_cast<int*>(base + G * KLHP / 2 + (WU ? 32 * 16 : kWarps * 32 * 16));
  float* red = base + G * KLHP / 2 + (WU ? 32 * 16 : kWarps * 32 * 16) + kpad;
  pdl_wait();
  pdl_trigger();
  const std::int64_t iter = *iter_p;
  const int rl = min(RH, max(0, (a.K - gl * KLH + 15) / 16));
  const int tid_u = WU ? lane : static_cast<int>(threadIdx.x);
  const int nthr_u = WU ? 32 : static_cast<int>(blockDim.x);
  const std::int64_t nunits = WU ? a.n_wunits : a.n_units;
  const std::int64_t* units = WU ? a.wunits : a.units;
  const std::int64_t ustart = WU ? static_cast<std::int64_t>(blockIdx.x) * kWarps + warp : blockIdx.x;
  const std::int64_t ustride = WU ? static_cast<std::int64_t>(gridDim.x) * kWarps : gridDim.x;
  const int K8 = (a.K + 7) & ~7;

  for (std::int64_t unit = ustart; unit < nunits; unit += ustride) {
    const std::int64_t m = units[unit * 3], t0 = units[unit * 3 + 1], t1 = units[unit * 3 + 2];
    const double* thg = a.theta + m * a.K;
    float* ths = a.thS32 + m * K8;  // theta/S in fp32 for level 2 (natural order, zero-padded)
    // theta/S (fp32) and its maximum; the document scale a_d; fp16 operands and Theta_d
    float mx = 0.0f;
    for (int k = tid_u; k < G * KLH; k += nthr_u) {
      const float x = k < a.K ? static_cast<float>(thg[k] / a.S[k]) : 0.0f;
      if (k < K8) ths[k] = x;
      mx = fmaxf(mx, x);
      if (k < a.K) cnt_s[k] = 0;
    }
    mx = team_max<WU>(mx, red);
    const float ad = ldexpf(1.0f, mx > 0.0f ? min(127, max(-126, 14 - ilogbf(mx))) : 0);
    float th_sum = 0.0f;
    for (int k = tid_u; k < G * KLH; k += nthr_u) {
      const float x = k < a.K ? static_cast<float>(thg[k] / a.S[k]) : 0.0f;
      const __half h = __float2half_rn(x * ad);
      thh[(k / KLH) * KLHP + k % KLH] = __half_as_ushort(h);
      th_sum += __half2float(h);
    }
    th_sum = team_sum<WU>(th_sum, red);
    const float A = 0x1p-24f * (32768.0f * static_cast<float>(a.K) + th_sum);
    if constexpr (WU) __syncwarp();
    else __syncthreads();
    unsigned tw[KLH / 2];
#pragma unroll
    for (int i = 0; i < KLH / 2; i += 4) {
      const uint4 t = *reinterpret_cast<const uint4*>(thh + gl * KLHP + 2 * i);
      tw[i] = t.x, tw[i + 1] = t.y, tw[i + 2] = t.z, tw[i + 3] = t.w;
    }
    const std::int64_t bstep = WU ? 32 : kWarps * 32;
    std::int64_t b0 = t0 + (WU ? 0 : warp * 32);
    int wl_next = b0 + lane < t1 ? __ldg(a.w + b0 + lane) : 0;
    for (; b0 < t1; b0 += bstep) {
      const std::int64_t t = b0 + lane;
      const bool valid = t < t1;
      const int wl = wl_next;
      wl_next = b0 + bstep + lane < t1 ? __ldg(a.w + b0 + bstep + lane) : 0;  // next batch, in flight
      // (1) level-1 chunk sums: 4 lanes per token, 16 candidates per round; the rows of
      // sub-batch s + 1 are in flight while sub-batch s is summed
      const std::int64_t left = (t1 - b0 + 7) / 8;
      const int nsub = left < 4 ? static_cast<int>(left) : 4;  // warp-uniform
      Oct16 cur[RH], nxt[RH];
      auto fetch = [&](int s2, Oct16 (&ph)[RH]) {
        const int wv = __shfl_sync(0xffffffffu, wl, s2 * 8 + gid);
        const unsigned short* row = a.phiT16 + static_cast<std::size_t>(wv) * a.Kp16;
#pragma unroll
        for (int r = 0; r < RH; ++r) {
          if (r < rl) ph[r] = ldg256h(row + 16 * (r * G + gl));
          else ph[r] = Oct16{};
        }
      };
      fetch(0, cur);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        if (s >= nsub) break;  // warp-uniform
        if (s + 1 < nsub) fetch(s + 1, nxt);
        const int src = s * 8 + gid;
#pragma unroll
        for (int r = 0; r < RH; ++r) {
          float sr = 0.0f;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            sr = fhfma(static_cast<unsigned short>(tw[8 * r + j] & 0xffffu), static_cast<unsigned short>(cur[r].v[j] & 0xffffu), sr);
            sr = fhfma(static_cast<unsigned short>(tw[8 * r + j] >> 16), static_cast<unsigned short>(cur[r].v[j] >> 16), sr);
          }
          csum[cs_idx(src, gl * RH + r)] = sr;
        }
#pragma unroll
        for (int r = 0; r < RH; ++r) cur[r] = nxt[r];
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
        const float mg = kL1Rel * uf + 4.0f * A;
        int k = -1;
        if (uf < total && total < 0x1p100f) {
          int cs = C - 1;
          float lo = 0.0f;
#pragma unroll
          for (int c = C - 1; c >= 0; --c)
            if (uf < P[c]) cs = c;
#pragma unroll
          for (int c = 0; c < C - 1; ++c)
            if (c < cs) lo = P[c];
          const int og = cs / RH, orr = cs - og * RH;
          const Oct16 p = ldg256h(a.phiT16 + static_cast<std::size_t>(wl) * a.Kp16 + 16 * (orr * G + og));
          const uint4 y0 = *reinterpret_cast<const uint4*>(thh + og * KLHP + 16 * orr);
          const uint4 y1 = *reinterpret_cast<const uint4*>(thh + og * KLHP + 16 * orr + 8);
          const unsigned tv[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
          float acc = lo, prev = lo;
          int j = -1;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const unsigned ta = tv[jj >> 1], pa = p.v[jj >> 1];
            const float nx = fhfma(static_cast<unsigned short>((jj & 1) ? ta >> 16 : ta & 0xffffu),
                                   static_cast<unsigned short>((jj & 1) ? pa >> 16 : pa & 0xffffu), acc);
            if (j < 0) {
              if (uf < nx) {
                j = jj;
                prev = acc;
              }
              acc = nx;
            }
          }
          const int kk = 16 * cs + j;
          if (j >= 0 && kk < a.K && uf - prev >= mg && acc - uf >= mg) k = kk;
        }
        if (k >= 0) {
          a.z[t] = k;
          atomicAdd(&a.nkw[static_cast<std::size_t>(wl) * a.Kp + k], 1);
          atomicAdd(&cnt_s[k], 1);
        } else {
          const int slot = atomicAdd(a.q2_len, 1);  // level 2 (zscreen_q_kernel)
          a.q2[slot] = make_int2(static_cast<int>(t), static_cast<int>(m));
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

// Level 2: the fp32 transposed screen (zscreen_t_kernel's arithmetic and margin) over
// the level-1 queue.  Each token brings its own document: the theta/S operands come
// from thS32 (written by the level-1 unit), counts go straight to nmk.  R: rounds of
// the phiT32 layout (G = 4 x CW = 8).
template <int R>
__global__ void __launch_bounds__(256) zscreen_q_kernel(LdaArgs a, const std::int64_t* iter_p) {
  constexpr int G = 4, CW = 8, C = G * R;
  __shared__ __align__(16) float csum_all[8][32 * 16];
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), gid = lane / G, warp = threadIdx.x >> 5;
  float* csum = csum_all[warp];
  pdl_wait();
  pdl_trigger();
  const std::int64_t iter = *iter_p;
  const int n = *a.q2_len;
  const int K8 = (a.K + 7) & ~7;
  const int rl = min(R, max(0, (a.K - gl * CW * R + CW - 1) / CW));
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int b0 = (blockIdx.x * (blockDim.x >> 5) + warp) * 32; b0 < n; b0 += nwarps * 32) {
    const int i = b0 + lane;
    const bool valid = i < n;
    const int2 q = valid ? a.q2[i] : make_int2(0, 0);
    const int wl = valid ? __ldg(a.w + q.x) : 0;
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      if (b0 + s * 8 >= n) break;  // warp-uniform
      const int src = s * 8 + gid;
      const int wv = __shfl_sync(0xffffffffu, wl, src);
      const int mv = __shfl_sync(0xffffffffu, q.y, src);
      const float* row = a.phiT32 + static_cast<std::size_t>(wv) * a.Kp32;
      const float* th = a.thS32 + static_cast<std::size_t>(mv) * K8;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        float sr = 0.0f;
        if (r < rl) {
          const Oct p = ldg256f(row + CW * (r * G + gl));
          const int k0 = CW * (gl * R + r);  // logical candidates of this chunk
          const float4 x0 = *reinterpret_cast<const float4*>(th + k0);
          const float4 x1 = *reinterpret_cast<const float4*>(th + k0 + 4);
          const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
          sr = x[0] * p.v[0];
#pragma unroll
          for (int j = 1; j < CW; ++j) sr = __fmaf_rn(x[j], p.v[j], sr);
        }
        csum[cs_idx(src, gl * R + r)] = sr;
      }
    }
    __syncwarp();
    if (valid) {
      const std::int64_t t = q.x, m = q.y;
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
        const int og = cs / R, orr = cs - og * R;
        const Oct p = ldg256f(a.phiT32 + static_cast<std::size_t>(wl) * a.Kp32 + CW * (orr * G + og));
        const float* th = a.thS32 + static_cast<std::size_t>(m) * K8 + CW * cs;
        const float4 y0 = *reinterpret_cast<const float4*>(th);
        const float4 y1 = *reinterpret_cast<const float4*>(th + 4);
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
        atomicAdd(&a.nmk[m * a.K + k], 1);
      } else {
        const int slot = atomicAdd(a.fq_len, 1);  // fp64 redraw (zfallback_kernel)
        a.fq[slot] = make_int2(static_cast<int>(t), static_cast<int>(m));
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------
// z block, TMA-staged screen (experimental, BNMC_ZSTAGE=1; slower, see choose_screen)
// ---------------------------------------------------------------------------------
// ncu r01 v15 (zscreen_t): every warp serialised ~5 L2 round trips per 32-token batch
// (4 sub-batch row fetches + the rescan re-fetch, which missed L1) and register
// double-buffering could not hold enough rows in flight.  Here the phi rows go
// global -> shared by the bulk-copy engine (cp.async.bulk, completion on an
// mbarrier), NS batches ahead per warp, with no register cost:
//  * work = batches of <= 32 consecutive tokens of one document; warp g of the
//    persistent grid owns a contiguous range of batches;
//  * lane j issues the 16*KQ-byte bulk copy of token j's phiT32 row (natural topic
//    order, fp32) into the warp's slot; lane 0 arms the slot's mbarrier with the
//    batch's byte count;
//  * compute is lane-per-token from shared memory: K products theta/S * g in
//    16-byte granules, running prefix in registers, u * total, the crossing granule,
//    the in-granule scan (all from shared memory: no re-fetch), the margin check,
//    z and the count atomics -- no shuffles;
//  * theta/S of the warp's current document sits in shared memory (fp32), reloaded
//    when the batch's document changes.
// Same screen / fp64-fallback contract as zscreen_kernel.
struct ZBatch {
  std::int64_t t0;
  int m, n;
};

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "ZW_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra ZW_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int KQ>
__global__ void __launch_bounds__(256) zstage_kernel(LdaArgs a, const std::int64_t* iter_p, const ZBatch* batches,
                                                     std::int64_t nbatch, int ns, int stride16) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned row_bytes = 16u * KQ;
  const std::size_t slot_bytes = static_cast<std::size_t>(32) * stride16 * 16;
  // CTA area: S (fp64, K).  Warp area: bars[ns], w[ns][32], theta/S[4KQ], rows[ns].
  double* Ssm = reinterpret_cast<double*>(smem_raw);
  const std::size_t cta_bytes = (static_cast<std::size_t>(a.K) * 8 + 127) / 128 * 128;
  const std::size_t warp_hdr = (static_cast<std::size_t>(ns) * (16 + 128) + 16 * KQ + 127) / 128 * 128;
  unsigned char* wbase = smem_raw + cta_bytes + warp * (warp_hdr + ns * slot_bytes);
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(wbase);
  int* wsm = reinterpret_cast<int*>(wbase + 16 * ns);
  float* th = reinterpret_cast<float*>(wbase + 16 * ns + 128 * ns);
  unsigned char* rows = wbase + warp_hdr;

  for (int k = threadIdx.x; k < a.K; k += blockDim.x) Ssm[k] = a.S[k];
  if (lane == 0)
    for (int i = 0; i < ns; ++i) mbar_init(bar + i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  const std::int64_t iter = *iter_p;
  const std::int64_t tw = static_cast<std::int64_t>(gridDim.x) * nw;
  const std::int64_t g = static_cast<std::int64_t>(blockIdx.x) * nw + warp;
  const std::int64_t b_first = nbatch * g / tw, b_last = nbatch * (g + 1) / tw;
  const std::int64_t count = b_last - b_first;

  auto issue = [&](std::int64_t c, int slot) {
    const ZBatch zb = batches[b_first + c];
    const int wv = lane < zb.n ? __ldg(a.w + zb.t0 + lane) : 0;
    wsm[slot * 32 + lane] = wv;
    if (lane == 0) mbar_expect_tx(bar + slot, row_bytes * static_cast<unsigned>(zb.n));
    __syncwarp();
    if (lane < zb.n)
      bulk_g2s(rows + slot * slot_bytes + static_cast<std::size_t>(lane) * stride16 * 16,
               a.phiT32 + static_cast<std::size_t>(wv) * a.Kp32, row_bytes, bar + slot);
  };
  for (std::int64_t c = 0; c < count && c < ns; ++c) issue(c, static_cast<int>(c));

  int curm = -1;
  for (std::int64_t c = 0; c < count; ++c) {
    const int slot = static_cast<int>(c % ns);
    const unsigned parity = static_cast<unsigned>((c / ns) & 1);
    const ZBatch zb = batches[b_first + c];
    if (zb.m != curm) {
      __syncwarp();
      const double* thg = a.theta + static_cast<std::int64_t>(zb.m) * a.K;
      for (int k = lane; k < 4 * KQ; k += 32) th[k] = k < a.K ? static_cast<float>(thg[k] / Ssm[k]) : 0.0f;
      curm = zb.m;
      __syncwarp();
    }
    mbar_wait(bar + slot, parity);
    if (lane < zb.n) {
      const std::int64_t t = zb.t0 + lane;
      const int wv = wsm[slot * 32 + lane];
      const float* row = reinterpret_cast<const float*>(rows + slot * slot_bytes + static_cast<std::size_t>(lane) * stride16 * 16);
      Stream rng(fold(fold(a.zkey_prefix, static_cast<std::uint64_t>(a.tok_base + t)), static_cast<std::uint64_t>(iter)));
      const float u01 = static_cast<float>(rng.next_unit());
      float P[KQ];
      float run = 0.0f;
#pragma unroll
      for (int q = 0; q < KQ; ++q) {
        const float4 f = *reinterpret_cast<const float4*>(row + 4 * q);
        const float4 x = *reinterpret_cast<const float4*>(th + 4 * q);
        float sq = x.x * f.x;
        sq = __fmaf_rn(x.y, f.y, sq);
        sq = __fmaf_rn(x.z, f.z, sq);
        sq = __fmaf_rn(x.w, f.w, sq);
        run += sq;
        P[q] = run;
      }
      const float total = run;
      const float uf = u01 * total;
      const float mg = a.screen_margin * total;
      int k = -1;
      if (uf < total && total > 0x1p-90f && total < 0x1p100f) {
        int cs = KQ - 1;
        float lo = 0.0f;
#pragma unroll
        for (int q = KQ - 1; q >= 0; --q)
          if (uf < P[q]) cs = q;
#pragma unroll
        for (int q = 0; q < KQ - 1; ++q)
          if (q < cs) lo = P[q];
        const float4 f = *reinterpret_cast<const float4*>(row + 4 * cs);
        const float4 x = *reinterpret_cast<const float4*>(th + 4 * cs);
        const float fv[4] = {f.x, f.y, f.z, f.w};
        const float xv[4] = {x.x, x.y, x.z, x.w};
        float acc = lo, prev = lo;
        int j = -1;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const float nx = __fmaf_rn(xv[jj], fv[jj], acc);
          if (j < 0) {
            if (uf < nx) {
              j = jj;
              prev = acc;
            }
            acc = nx;
          }
        }
        const int kk = 4 * cs + j;
        if (j >= 0 && kk < a.K && uf - prev >= mg && acc - uf >= mg) k = kk;
      }
      if (k >= 0) {
        a.z[t] = k;
        atomicAdd(&a.nkw[static_cast<std::size_t>(wv) * a.Kp + k], 1);
        atomicAdd(&a.nmk[static_cast<std::int64_t>(zb.m) * a.K + k], 1);
      } else {
        const int slotq = atomicAdd(a.fq_len, 1);  // fp64 redraw (zfallback_kernel)
        a.fq[slotq] = make_int2(static_cast<int>(t), zb.m);
      }
    }
    __syncwarp();
    // the slot's generic reads are done: order them before the next bulk write into it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (c + ns < count) issue(c + ns, slot);
  }
}

// fp64 product-form draw for the tokens the screen could not decide (~2K * 2^-16
// of them): one warp per queued token.  Lane l owns the contiguous candidates
// [l*c, (l+1)*c), c = ceil(K/32); warp scan of the lane sums, the owner rescans
// its chunk (the reference's candidate order and u = next_unit * total rule,
// dist.cpp:202-215).  Tokens whose product weights underflow take the sequential
// log-space draw.
__global__ void __launch_bounds__(256) zfallback_kernel(LdaArgs a, const std::int64_t* iter_p, int* err) {
  pdl_wait();
  pdl_trigger();
  const std::int64_t iter = *iter_p;
  const int lane = threadIdx.x & 31;
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
    double own = 0.0;
    for (int k = k0; k < k1; ++k) own += (thg[k] / a.S[k]) * row[k];
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
          acc += (thg[k] / a.S[k]) * row[k];
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

template <bool FINAL>
__global__ void __launch_bounds__(256, 4) wterm_kernel(LdaArgs a, Outputs o, int advance) {
  __shared__ double scratch[4 * 32];
  pdl_wait();
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  const std::int64_t g0 = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // w-factor over the topic-word cells, static cell -> thread assignment (deterministic).
  // The padded [V][Kp] arrays are read as 4-cell vectors (Kp % 4 == 0: a vector never
  // crosses a row; padding cells have n = 0 and logS is zero-padded to Kp), two vectors
  // per thread in flight; no per-cell index arithmetic beyond one modulo per vector.
  double accw = 0.0;
  if (a.logg_valid) {
    const std::int64_t nvec = static_cast<std::int64_t>(a.V) * a.Kp / 4;
    const bool narrow = nvec < (std::int64_t{1} << 29);  // 4 * nvec fits 31 bits
    const int4* n4 = reinterpret_cast<const int4*>(a.nkw);
    // log g stored per cell (v2 phi block), or taken here from g = phiT for the
    // counted cells only (warp-pool phi block: a.logg == nullptr)
    const bool take_log = a.logg == nullptr;
    const double2* l2 = reinterpret_cast<const double2*>(take_log ? a.phiT : a.logg);
    for (std::int64_t c0 = g0; c0 < nvec; c0 += kWU * stride) {
      int4 n[kWU];
      double2 la[kWU], lb[kWU];
#pragma unroll
      for (int j = 0; j < kWU; ++j) {
        const std::int64_t c = c0 + j * stride;
        n[j] = make_int4(0, 0, 0, 0);
        if (c < nvec) {
          n[j] = n4[c];
          la[j] = l2[2 * c];
          lb[j] = l2[2 * c + 1];
        }
      }
#pragma unroll
      for (int j = 0; j < kWU; ++j) {  // log phi = log g - log S
        const std::int64_t c = c0 + j * stride;
        if (c >= nvec || (n[j].x | n[j].y | n[j].z | n[j].w) == 0) continue;
        const int k0 = narrow ? static_cast<int>(static_cast<unsigned>(4 * c) % static_cast<unsigned>(a.Kp))
                              : static_cast<int>((4 * c) % a.Kp);
        auto lg = [take_log](double x) { return take_log ? log(x) : x; };  // log(0) = -inf
        if (n[j].x) accw += static_cast<double>(n[j].x) * (lg(la[j].x) - __ldg(&a.logS[k0]));
        if (n[j].y) accw += static_cast<double>(n[j].y) * (lg(la[j].y) - __ldg(&a.logS[k0 + 1]));
        if (n[j].z) accw += static_cast<double>(n[j].z) * (lg(lb[j].x) - __ldg(&a.logS[k0 + 2]));
        if (n[j].w) accw += static_cast<double>(n[j].w) * (lg(lb[j].y) - __ldg(&a.logS[k0 + 3]));
      }
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
  // (cudaMalloc bases are 256-byte aligned), the ragged tail scalar
  double accz = 0.0;
  const std::int64_t ncz = a.Ml * a.K, nvz = ncz / 4;
  const int4* m4 = reinterpret_cast<const int4*>(a.nmk);
  const double2* t2 = reinterpret_cast<const double2*>(a.theta);
  auto zterm = [](int n, double x) {
    return n ? static_cast<double>(n) * (x > 0.0 ? log(x) : -INFINITY) : 0.0;
  };
  for (std::int64_t c = g0; c < nvz; c += stride) {
    const int4 n = m4[c];
    const double2 x = t2[2 * c], y = t2[2 * c + 1];
    accz += zterm(n.x, x.x);
    accz += zterm(n.y, x.y);
    accz += zterm(n.z, y.x);
    accz += zterm(n.w, y.y);
  }
  if (g0 < ncz - 4 * nvz) accz += zterm(a.nmk[4 * nvz + g0], a.theta[4 * nvz + g0]);
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
    theta_threads_ = std::min(256, ((K_ + 31) / 32) * 32);

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
    phiT_.alloc(static_cast<std::size_t>(V_) * Kp_);
    if (exact_) logphiT_.alloc(static_cast<std::size_t>(V_) * Kp_);
    // fp32-screened z-step (product weights only); BNMC_ZSTEP_SCREEN=0 disables it.
    const char* sc = std::getenv("BNMC_ZSTEP_SCREEN");
    screen_ = !exact_ && !(sc && std::string(sc) == "0");
    choose_screen();
    Kp32_ = CW32_ * G32_ * RS_;
    if (stage_ && screen_) {
      std::vector<ZBatch> hb;
      for (std::int64_t m = 0; m < Ml_; ++m)
        for (std::int64_t t = off_host_[m]; t < off_host_[m + 1]; t += 32)
          hb.push_back(ZBatch{t, static_cast<int>(m), static_cast<int>(std::min<std::int64_t>(32, off_host_[m + 1] - t))});
      nbatch_ = static_cast<std::int64_t>(hb.size());
      batches_.alloc(std::max<std::size_t>(hb.size(), 1));
      if (!hb.empty())
        BNMC_CUDA(cudaMemcpy(batches_.p, hb.data(), sizeof(ZBatch) * hb.size(), cudaMemcpyHostToDevice));
      plan_stage();
    }
    if (screen_) phiT32_.alloc(static_cast<std::size_t>(V_) * Kp32_);
    // two-level screen (fp16 rows, then fp32): experimental, BNMC_ZSCREEN_H=1.  Measured
    // slower (r01, NIPS): level 1 takes 79 us against the fp32 screen's 85 us -- half the
    // row bytes, but the kernel is bound by its per-batch latency chain, not bytes --
    // and level 2 (4.6 % of the tokens, one latency chain per scattered batch) plus
    // the row conversion add ~24 us.
    const char* zh = std::getenv("BNMC_ZSCREEN_H");
    h16_ = screen_ && transposed_ && !stage_ && K_ <= 128 && zh && std::string(zh) == "1";
    if (h16_) {
      RH_ = (K_ + 63) / 64;
      Kp16_ = 64 * RH_;
      phiT16_.alloc(static_cast<std::size_t>(V_) * Kp16_);
      thS32_.alloc(static_cast<std::size_t>(std::max<std::int64_t>(Ml_, 1)) * ((K_ + 7) & ~7));
      q2_.alloc(std::max<std::int64_t>(Nl_, 1));
      q2_len_.alloc(1);
      const int gx = (K_ + 31) / 32;
      h16_blocks_ = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((V_ + 8 * gx - 1) / (8 * gx), 296 / gx)));
    }
    theta_.alloc(std::max<std::int64_t>(Ml_ * K_, 1));
    nkw_.alloc(static_cast<std::size_t>(V_) * Kp_);
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
    colpart_.alloc(static_cast<std::size_t>(nb_phi_) * K_);
    {
      int dev = 0, sms = 148, per_sm = 1;
      BNMC_CUDA(cudaGetDevice(&dev));
      BNMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const char* pe = std::getenv("BNMC_PHI_POOL");
      const char* pv1 = std::getenv("BNMC_PHI_V1");
      const char* tv1 = std::getenv("BNMC_THETA_V1");
      pool_ = !(pe && std::string(pe) == "0") && !(pv1 && std::string(pv1) == "1") &&
              !(tv1 && std::string(tv1) == "1");
      if (pool_) {
        // warp-pool phi block: a persistent grid (one resident wave), equal cell ranges
        // per warp; the column sums read phiT rows (nvb_ = V rows for phi_colsum2<true>)
        if (K_ <= kPoolCells)
          BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_pool_kernel<true>, 256, 0));
        else
          BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_pool_kernel<false>, 256, 0));
        pool_blocks_ = sms * std::max(per_sm, 1);
        phi_rows_ = 1;
      } else {
        // rows per thread L = 4 (measured r01 v29: NIPS 82 us at L=4 vs 92 at 8; KOS 38 us
        // vs 42 at 1); 2 when 4 leaves the GPU under one wave (KOS phi 35.3 -> 32.2 us)
        phi_rows_ = 4;
        BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_gamma2_kernel<4>, 256, 0));
        const std::int64_t blocks4 = ((V_ + 3) / 4 * K_ + 255) / 256;
        if (blocks4 < static_cast<std::int64_t>(sms) * std::max(per_sm, 1)) phi_rows_ = 2;
        if (const char* e = std::getenv("BNMC_PHI_ROWS")) {
          const int r = std::atoi(e);
          if (r == 1 || r == 2 || r == 4 || r == 8) phi_rows_ = r;
        }
        switch (phi_rows_) {
          case 1: BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_gamma2_kernel<1>, 256, 0)); break;
          case 2: BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_gamma2_kernel<2>, 256, 0)); break;
          case 4: BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_gamma2_kernel<4>, 256, 0)); break;
          default: BNMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, phi_gamma2_kernel<8>, 256, 0)); break;
        }
        phi_pf_ = static_cast<int>(0.7 * sms * std::max(per_sm, 1));  // measured: 0.55-0.8 of a wave best
        if (const char* e = std::getenv("BNMC_PHI_PREFETCH")) phi_pf_ = std::max(0, std::atoi(e));
      }
    }
    nvb_ = (V_ + phi_rows_ - 1) / phi_rows_;
    col_stripes_ = static_cast<int>(std::min<std::int64_t>(pool_ ? kColStripes : 64, std::max<std::int64_t>(4, nvb_ / (pool_ ? 48 : 96))));
    {
      const std::int64_t gx = (K_ + 31) / 32, wblocks = (Ml_ + 7) / 8;
      trow_blocks_ = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((wblocks + gx - 1) / gx, 16384)));
    }
    if (const char* e = std::getenv("BNMC_COL_STRIPES")) col_stripes_ = std::min(kColStripes, std::max(1, std::atoi(e)));
    spart_.alloc(static_cast<std::size_t>(kColStripes) * K_ * 2);
    ticket_.alloc((K_ + 31) / 32 + 1);
    ticket_.zero(nullptr);
    if (!pool_) gpart_.alloc(static_cast<std::size_t>(nvb_) * K_);
    if (!pool_) logg_.alloc(static_cast<std::size_t>(V_) * Kp_);  // the pool kernel keeps no per-cell log
    logS_.alloc(Kp_);
    logS_.zero(nullptr);  // padding columns stay 0 (wterm_kernel reads 4-cell vectors)
    if (!pool_) lpart_.alloc(static_cast<std::size_t>(nvb_) * K_);
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
    phiT16_.zero(s0);
    q2_len_.zero(s0);
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
    const char* pv = std::getenv("BNMC_PHI_V1");
    phi_v1_ = pv && std::string(pv) == "1";
    if (const char* e = std::getenv("BNMC_SCREEN_MARGIN")) screen_margin_ = static_cast<float>(std::atof(e));
    if (const char* e = std::getenv("BNMC_PDL")) pdl_ = std::string(e) != "0";
    const char* tv = std::getenv("BNMC_THETA_V1");
    theta_v1_ = tv && std::string(tv) == "1";
    configure_kernels();
    BNMC_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    BNMC_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_phi_ready_, cudaEventDisableTiming));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_theta_ready_, cudaEventDisableTiming));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_copy_done_, cudaEventDisableTiming));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    BNMC_CUDA(cudaStreamCreateWithFlags(&up_, cudaStreamNonBlocking));
    BNMC_CUDA(cudaEventCreateWithFlags(&ev_up_, cudaEventDisableTiming));
    BNMC_CUDA(cudaMallocHost(reinterpret_cast<void**>(&spec_flag_host_), sizeof(int)));
    spec_flag_.alloc(1);
    if (const char* e = std::getenv("BNMC_SPECULATE")) speculate_ = std::string(e) != "0";
  }

  ~Lda() override {
    if (side_) cudaStreamDestroy(side_);
    if (copy_) cudaStreamDestroy(copy_);
    if (ev_phi_ready_) cudaEventDestroy(ev_phi_ready_);
    if (ev_theta_ready_) cudaEventDestroy(ev_theta_ready_);
    if (ev_copy_done_) cudaEventDestroy(ev_copy_done_);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
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
    a.logg_valid = (!observe_phi_ && !phi_v1_ && !(pool_ && exact_)) ? 1 : 0;
    const bool timed = marks != nullptr;  // phase timing: everything on one stream
    mark(st, "begin");
    if (pool_) {
      // warp-pool conjugate block: phi and theta cells in one balanced kernel, then the
      // phi column sums (phi_colsum2<true> stripes) and the theta rows (extra y-blocks)
      if (!observe_phi_ && comm_.active()) {
        comm_.all_reduce(nkw_.p, nkw_.n, RedType::I32, RedOp::Sum, st);
        mark(st, "allreduce_counts");
      }
      if (observe_phi_) nkw_.zero(st);  // phi clamped: the z-step's counts feed only the w-factor
      a.pool_phi = observe_phi_ ? 0 : 1;
      a.trow_blocks = Ml_ > 0 ? trow_blocks_ : 0;
      a.col_stripes = observe_phi_ ? 0 : col_stripes_;
      if (a.pool_phi || Ml_ > 0) {
        if (K_ <= kPoolCells)
          phi_pool_kernel<true><<<pool_blocks_, 256, 0, st>>>(a, out.iter);
        else
          phi_pool_kernel<false><<<pool_blocks_, 256, 0, st>>>(a, out.iter);
        mark(st, "conj_pool");
        launch_pdl(phi_colsum2_kernel<true>, dim3((K_ + 31) / 32, a.col_stripes + a.trow_blocks + (h16_ ? h16_blocks_ : 0)),
                   dim3(256), 0, st, a);
        fq_reset_ = true;
        mark(st, "colsum_rows");
      }
      if (!observe_phi_ && exact_) {
        // log-space weights read log phi: normalise in place, then phi = phiT (S = 1).
        phi_norm_kernel<true><<<nb_phi_, phi_threads_, 0, st>>>(a);
        fill_kernel<<<1, 256, 0, st>>>(S_.p, K_, 1.0);
        mark(st, "phi_norm");
      }
      if (!timed) {  // phi, theta final: overlapped downloads may start (external event nodes)
        if (!observe_phi_) record_external(ev_phi_ready_, st);
        if (Ml_ > 0) record_external(ev_theta_ready_, st);
      }
    } else {
      // The theta block depends only on the doc-topic counts: it runs on a side stream
      // concurrently with the phi block (fork/join events; captured into the graph).
      if (Ml_ > 0 && !timed) {
        BNMC_CUDA(cudaEventRecord(ev_fork_, st));
        BNMC_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
        launch_theta(a, side_);
        record_external(ev_theta_ready_, side_);
        BNMC_CUDA(cudaEventRecord(ev_join_, side_));
      }
      if (!observe_phi_) {
        if (comm_.active()) {
          comm_.all_reduce(nkw_.p, nkw_.n, RedType::I32, RedOp::Sum, st);
          mark(st, "allreduce_counts");
        }
        if (phi_v1_) {
          phi_gamma_kernel<<<nb_phi_, 256, 0, st>>>(a, out.iter);
          mark(st, "phi_gamma");
          phi_colsum_terms_kernel<<<K_, 128, 0, st>>>(a);
          if (h16_) phi_h16_kernel<<<148 * 4, 256, 0, st>>>(a);
        } else {
          const unsigned nbg = blocks_for(nvb_ * K_, 256);
          if (pool_) {
            if (K_ <= kPoolCells)
              phi_pool_kernel<true><<<pool_blocks_, 256, 0, st>>>(a, out.iter);
            else
              phi_pool_kernel<false><<<pool_blocks_, 256, 0, st>>>(a, out.iter);
          } else switch (phi_rows_) {
            case 1: phi_gamma2_kernel<1><<<nbg, 256, 0, st>>>(a, out.iter); break;
            case 2: phi_gamma2_kernel<2><<<nbg, 256, 0, st>>>(a, out.iter); break;
            case 4: phi_gamma2_kernel<4><<<nbg, 256, 0, st>>>(a, out.iter); break;
            default: phi_gamma2_kernel<8><<<nbg, 256, 0, st>>>(a, out.iter); break;
          }
          mark(st, "phi_gamma");
          // (+ h16_blocks_ y-blocks converting the rows for the level-1 screen)
          launch_pdl(pool_ ? phi_colsum2_kernel<true> : phi_colsum2_kernel<false>, dim3((K_ + 31) / 32, col_stripes_ + (h16_ ? h16_blocks_ : 0)), dim3(256), 0, st, a);
          fq_reset_ = true;
        }
        mark(st, "phi_colsum");
        if (exact_) {
          // log-space weights read log phi: normalise in place, then phi = phiT (S = 1).
          phi_norm_kernel<true><<<nb_phi_, phi_threads_, 0, st>>>(a);
          fill_kernel<<<1, 256, 0, st>>>(S_.p, K_, 1.0);
          mark(st, "phi_norm");
        }
        // phi (phiT, S) is final from here: an overlapped download may start (external
        // event node in the captured graph)
        if (!timed) record_external(ev_phi_ready_, st);
      } else {
        // phi clamped: no phi block consumes the counts; the z-step's counts of this
        // sweep feed only the w-factor.
        nkw_.zero(st);
      }
      if (Ml_ > 0) {
        if (timed) {
          launch_theta(a, st);
          mark(st, "theta");
        } else {
          BNMC_CUDA(cudaStreamWaitEvent(st, ev_join_, 0));
        }
      }
    }
    if (Ml_ > 0) {
      launch_zstep(a, st);
      mark(st, "zstep");
      if (timed && std::getenv("BNMC_SCREEN_STATS")) {  // diagnostics: queue lengths of this sweep
        int n2 = -1, n3 = -1;
        BNMC_CUDA(cudaStreamSynchronize(st));
        if (h16_) BNMC_CUDA(cudaMemcpy(&n2, q2_len_.p, sizeof(int), cudaMemcpyDeviceToHost));
        BNMC_CUDA(cudaMemcpy(&n3, fq_len_.p, sizeof(int), cudaMemcpyDeviceToHost));
        std::fprintf(stderr, "[bnmc] z-step queues: level2 %d fp64 %d of %lld tokens\n", n2, n3, static_cast<long long>(Nl_));
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
    if (h16_) phi_h16_kernel<<<148 * 4, 256, 0, st>>>(a);
    BNMC_CUDA(cudaGetLastError());
    BNMC_CUDA(cudaStreamSynchronize(st));
  }

  void launch_theta(const LdaArgs& a, cudaStream_t st) {
    if (theta_v1_ || K_ > 256 * kThetaRun) {
      theta_kernel<<<grid_docs(), theta_threads_, sizeof(double) * K_, st>>>(a, out.iter);
      return;
    }
    const int tpd = (K_ + kThetaRun - 1) / kThetaRun;
    const int dpb = std::max(1, 256 / tpd);
    theta2_kernel<<<static_cast<unsigned>((Ml_ + dpb - 1) / dpb), 256, 0, st>>>(a, out.iter, tpd, dpb);
  }

  unsigned grid_docs() const { return static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>(Ml_, 1 << 20))); }

  std::size_t zstep_smem() const { return sizeof(double) * 2 * Kp_; }

  template <int G, int R, bool E>
  void zstep_attr() {
    const int sm = static_cast<int>(zstep_smem());
    BNMC_CUDA(cudaFuncSetAttribute(zstep_kernel<G, R, E, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    BNMC_CUDA(cudaFuncSetAttribute(zstep_kernel<G, R, E, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));

  }

  void configure_kernels() {
    if (sizeof(double) * K_ > 48 * 1024)
      BNMC_CUDA(cudaFuncSetAttribute(theta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(sizeof(double) * K_)));
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
    // Off by default: measured slower on NIPS (160 us vs 107 us; r01 v19) -- 32 bulk
    // copies of 400 B per batch, the bulk-copy issue rate bounds it.  BNMC_ZSTAGE=1.
    stage_ = false;
    if (const char* e = std::getenv("BNMC_ZSTAGE")) stage_ = std::string(e) == "1" && K_ <= 128;
    if (stage_) {
      kq_ = 0;
      for (int q : kStageKQ)
        if (q * 4 >= K_) {
          kq_ = q;
          break;
        }
      G32_ = 1;
      CW32_ = 8;
      RS_ = (kq_ + 1) / 2;  // Kp32 = 8 RS >= 4 KQ: the bulk copy never leaves the row
      transposed_ = false;
      return;
    }
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

  template <int G, int CW, int R, bool TFR>
  void zscreen_launch(const LdaArgs& a, cudaStream_t st) {
    const unsigned g = static_cast<unsigned>(std::min<std::int64_t>(n_units_, 1 << 24));
    const std::size_t sm = sizeof(float) * G * (CW * R + 4);
    zscreen_kernel<G, CW, R, TFR><<<g, kZThreads, sm, st>>>(a, out.iter);
  }

  template <int G, int CW, bool TFR>
  void zscreen_rounds(const LdaArgs& a, cudaStream_t st) {
    if constexpr (G <= 8) {
      switch (RS_) {
        case 1: zscreen_launch<G, CW, 1, TFR>(a, st); return;
        case 2: zscreen_launch<G, CW, 2, TFR>(a, st); return;
        case 3: zscreen_launch<G, CW, 3, TFR>(a, st); return;
        default: zscreen_launch<G, CW, 4, TFR>(a, st); return;
      }
    } else if constexpr (G == 32 && CW == 8 && !TFR) {
      if (RS_ > 4) zscreen_launch<G, CW, 8, TFR>(a, st);
      else zscreen_launch<G, CW, 4, TFR>(a, st);
    } else {
      zscreen_launch<G, CW, 4, TFR>(a, st);
    }
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

  template <int RH, bool WU>
  void zscreen_h_launch(const LdaArgs& a, cudaStream_t st) {
    const int kpad = (K_ + 3) & ~3;
    const std::size_t hw = 4 * (16 * RH + 8) / 2;  // thh, in floats
    if (WU) {
      const std::size_t sm = sizeof(float) * 8 * (hw + 32 * 16 + kpad + 32);
      const unsigned gw = static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((n_wunits_ + 7) / 8, 148 * 3)));
      launch_pdl(zscreen_h_kernel<RH, true>, dim3(gw), dim3(256), sm, st, a, static_cast<const std::int64_t*>(out.iter));
      return;
    }
    const unsigned g = static_cast<unsigned>(std::min<std::int64_t>(n_units_, 1 << 24));
    const std::size_t sm = sizeof(float) * (hw + zt_warps_ * 32 * 16 + kpad + 32);
    launch_pdl(zscreen_h_kernel<RH, false>, dim3(g), dim3(32 * zt_warps_), sm, st, a, static_cast<const std::int64_t*>(out.iter));
  }

  template <int R>
  void zscreen_q_launch(const LdaArgs& a, cudaStream_t st) {
    // one wave of warps covers ~200 k queued tokens (NIPS: ~87 k): the kernel is one
    // latency chain per batch, so warps, not blocks per SM, set its time
    launch_pdl(zscreen_q_kernel<R>, dim3(148 * 6), dim3(256), 0, st, a, static_cast<const std::int64_t*>(out.iter));
  }

  // Level 1 (fp16 rows) then level 2 (fp32 rows, the level-1 queue).
  void launch_zscreen_h(const LdaArgs& a, cudaStream_t st) {
    if (RH_ == 1) {
      if (zt_wu_) zscreen_h_launch<1, true>(a, st);
      else zscreen_h_launch<1, false>(a, st);
    } else {
      if (zt_wu_) zscreen_h_launch<2, true>(a, st);
      else zscreen_h_launch<2, false>(a, st);
    }
    switch (RS_) {
      case 1: zscreen_q_launch<1>(a, st); break;
      case 2: zscreen_q_launch<2>(a, st); break;
      case 3: zscreen_q_launch<3>(a, st); break;
      default: zscreen_q_launch<4>(a, st); break;
    }
  }

  template <int KQ>
  void zstage_launch(const LdaArgs& a, cudaStream_t st) {
    if (!stage_attr_) {
      BNMC_CUDA(cudaFuncSetAttribute(zstage_kernel<KQ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(stage_smem_)));
      stage_attr_ = true;
    }
    zstage_kernel<KQ><<<stage_grid_, 32 * stage_warps_, stage_smem_, st>>>(
        a, out.iter, batches_.p, nbatch_, stage_slots_, stage_stride16_);
  }

  template <int... Q>
  void zstage_dispatch(const LdaArgs& a, cudaStream_t st, std::integer_sequence<int, Q...>) {
    bool done = false;
    ((!done && Q == kq_ ? (zstage_launch<Q>(a, st), done = true) : false), ...);
  }

  // Shared-memory plan of zstage_kernel: W warps x NS slots of 32 rows.
  void plan_stage() {
    stage_stride16_ = kq_ | 1;  // odd 16-byte row stride: conflict-free lane-per-row reads
    const std::size_t slot = static_cast<std::size_t>(32) * stage_stride16_ * 16;
    const std::size_t cta = (static_cast<std::size_t>(K_) * 8 + 127) / 128 * 128;
    int dev = 0, smem_max = 0, sms = 148;
    BNMC_CUDA(cudaGetDevice(&dev));
    BNMC_CUDA(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    BNMC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    stage_warps_ = 8;
    if (const char* e = std::getenv("BNMC_ZSTAGE_WARPS")) stage_warps_ = std::min(8, std::max(1, std::atoi(e)));
    auto hdr = [&](int ns) { return (static_cast<std::size_t>(ns) * (16 + 128) + 16 * kq_ + 127) / 128 * 128; };
    auto need = [&](int w, int ns) { return cta + w * (hdr(ns) + ns * slot); };
    stage_slots_ = 2;
    while (stage_slots_ < 8 && need(stage_warps_, stage_slots_ + 1) <= static_cast<std::size_t>(smem_max))
      ++stage_slots_;
    if (const char* e = std::getenv("BNMC_ZSTAGE_SLOTS")) stage_slots_ = std::min(16, std::max(1, std::atoi(e)));
    while (stage_warps_ > 1 && need(stage_warps_, stage_slots_) > static_cast<std::size_t>(smem_max)) --stage_warps_;
    stage_smem_ = need(stage_warps_, stage_slots_);
    require(stage_smem_ <= static_cast<std::size_t>(smem_max), BNMC_GPU_ERR_ARG, "z-step staging does not fit shared memory");
    stage_grid_ = static_cast<unsigned>(sms);
  }

  void launch_zscreen(const LdaArgs& a, cudaStream_t st) {
    if (!fq_reset_) {
      BNMC_CUDA(cudaMemsetAsync(fq_len_.p, 0, sizeof(int), st));
      if (h16_) BNMC_CUDA(cudaMemsetAsync(q2_len_.p, 0, sizeof(int), st));
    }
    fq_reset_ = false;
    if (h16_) {
      launch_zscreen_h(a, st);
      launch_pdl(zfallback_kernel, dim3(148 * 8), dim3(256), 0, st, a, static_cast<const std::int64_t*>(out.iter), out.err);
      return;
    }
    if (stage_) {
      zstage_dispatch(a, st, std::integer_sequence<int, 1, 2, 4, 6, 8, 10, 12, 13, 14, 16, 18, 20, 22, 24, 25, 26, 28, 30, 32>{});
      zfallback_kernel<<<148 * 8, 256, 0, st>>>(a, out.iter, out.err);
      return;
    }
    if (transposed_) {
      if (tfr_) zscreen_t_rounds<true>(a, st);
      else zscreen_t_rounds<false>(a, st);
      launch_pdl(zfallback_kernel, dim3(148 * 8), dim3(256), 0, st, a, static_cast<const std::int64_t*>(out.iter), out.err);
      return;
    }
    const int key = G32_ * 100 + CW32_ * 10 + (tfr_ ? 1 : 0);
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
    zfallback_kernel<<<148 * 8, 256, 0, st>>>(a, out.iter, out.err);
  }

  void launch_zstep(const LdaArgs& a, cudaStream_t st) {
    const unsigned g = static_cast<unsigned>(std::min<std::int64_t>(n_units_, 1 << 24));
    const std::size_t sm = zstep_smem();
    const int* err = out.err;
    const std::int64_t* it = out.iter;
    dispatch_zstep([&](auto gg, auto r, auto e) {
      constexpr int GG = decltype(gg)::value, RR = decltype(r)::value;
      constexpr bool EE = decltype(e)::value;
      if constexpr (!EE) {
        if (screen_) {
          launch_zscreen(a, st);
          return;
        }
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
    a.phiT16 = h16_ ? phiT16_.p : nullptr;
    a.Kp16 = Kp16_;
    a.RH = RH_;
    a.thS32 = h16_ ? thS32_.p : nullptr;
    a.q2 = h16_ ? q2_.p : nullptr;
    a.q2_len = h16_ ? q2_len_.p : nullptr;
    a.col_stripes = col_stripes_;
    a.logphiT = exact_ ? logphiT_.p : nullptr;
    a.theta = theta_.p;
    a.nkw = nkw_.p;
    a.colpart = colpart_.p;
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
    a.phi_pf = phi_pf_;
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
    a.gpart = gpart_.p;
    a.lpart = lpart_.p;
    a.nvb = nvb_;
    a.logg = logg_.p;
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
    return a;
  }

  Comm comm_;
  int K_ = 0, Kp_ = 0, V_ = 0, G_ = 4, R_ = 8;
  std::int64_t M_ = 0, N_ = 0, d0_ = 0, d1_ = 0, Ml_ = 0, Nl_ = 0, tok0_ = 0;
  std::vector<std::int64_t> off_host_;
  bool exact_ = false, observe_phi_ = false, theta_regs_ = false, screen_ = false;
  int Kp32_ = 0, RS_ = 1, G32_ = 8, CW32_ = 4;
  bool tfr_ = true, transposed_ = false, phi_v1_ = false, theta_v1_ = false;
  // TMA-staged z-step (zstage_kernel)
  static constexpr int kStageKQ[] = {1, 2, 4, 6, 8, 10, 12, 13, 14, 16, 18, 20, 22, 24, 25, 26, 28, 30, 32};
  bool stage_ = false, stage_attr_ = false;
  int kq_ = 0, stage_stride16_ = 1, stage_warps_ = 8, stage_slots_ = 2;
  std::size_t stage_smem_ = 0;
  unsigned stage_grid_ = 148;
  DevBuf<ZBatch> batches_;
  std::int64_t nbatch_ = 0;
  DevBuf<float> phiT32_;
  // two-level screen (zscreen_h_kernel + zscreen_q_kernel), K <= 128
  bool h16_ = false;
  int RH_ = 1, Kp16_ = 64, h16_blocks_ = 1;
  DevBuf<unsigned short> phiT16_;
  DevBuf<float> thS32_;
  DevBuf<int2> q2_;
  DevBuf<int> q2_len_;
  cudaStream_t side_ = nullptr, copy_ = nullptr;
  // speculative sweep_store
  cudaStream_t up_ = nullptr;
  cudaEvent_t ev_up_ = nullptr;
  DevBuf<std::int64_t> up64_;
  DevBuf<int> zprev_, spec_flag_;
  int* spec_flag_host_ = nullptr;
  bool zprev_valid_ = false, speculate_ = true;
  cudaEvent_t ev_phi_ready_ = nullptr, ev_theta_ready_ = nullptr, ev_copy_done_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  double alpha_ = 0.1, beta_ = 0.1, phi_norm_ = 0, phi_lgasum_ = 0, theta_norm_ = 0, theta_lgasum_ = 0;
  std::uint64_t seed_ = 0;
  int var_phi_ = 0, var_theta_ = 1, var_z_ = 2, var_w_ = 3;
  int phi_threads_ = 128, theta_threads_ = 128, rows_per_block_ = 1, nb_phi_ = 1;
  std::vector<std::int64_t> units_host_;
  std::int64_t n_units_ = 0, docs_per_block_ = 1, nb_doc_ = 0, n_wunits_ = 0;
  DevBuf<std::int64_t> wunits_;
  bool zt_wu_ = true;
  int nbw_ = 1, col_stripes_ = kColStripes;
  float screen_margin_ = kScreenMargin;
  bool fq_reset_ = false;  // phi_colsum2 of this sweep zeroes the fallback queue

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
  std::int64_t nvb_ = 1;
  int phi_rows_ = kPhiRowsMax;
  bool boost_pow_ = std::getenv("BNMC_BOOST_POW") == nullptr || std::string(std::getenv("BNMC_BOOST_POW")) != "0";
  bool pool_ = true;     // phi block: warp-pool kernel (BNMC_PHI_POOL=0: v2)
  int pool_blocks_ = 148;
  int trow_blocks_ = 1;   // phi_colsum2 y-blocks for the pool's theta rows
  int phi_pf_ = 0;     // phi_gamma2 count prefetch distance (blocks)
  DevBuf<double> gpart_, lpart_, spart_, logg_, logS_, ttpart_;
  DevBuf<int> ticket_;
  DevBuf<double> phiT_, logphiT_, theta_, colpart_, colpart2_, S_, phi_term_, doc_part_, red_, tpart_,
      zpart_, wpart_;
};

}  // namespace

std::unique_ptr<Model> make_lda(const bnmc_gpu_desc& d, const Comm& c, Outputs o) {
  return std::make_unique<Lda>(d, c, o);
}

}  // namespace bnmc_gpu
