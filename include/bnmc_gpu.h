/* include/bnmc_gpu.h -- C-ABI of the B200-native MCMC sweep (libbnmc_gpu.so).
 *
 * The drop-in boundary for the reference's hot path.  A host caller (the
 * reference's C++ Engine via the adapter in INTEGRATION.md, the C++ mirror in
 * include/bnmc_gpu.hpp, or Python through ctypes) hands over plain host pointers
 * laid out exactly like the reference's ParamStore, and every sweep runs on the
 * GPU.  There is no CPU fallback: every entry point fails with a non-zero code
 * when the device path cannot run.
 *
 * Reference interfaces each entry point replaces (paths under /root/reference/proj):
 *   bnmc_gpu_create        Engine::Engine            include/bnmc/sampler.hpp:47
 *                          (plan for LDA/GMM Gibbs or MH, src/plan.cpp:110-166)
 *   bnmc_gpu_upload        the ParamStore the caller lends to Engine::sweep
 *                          include/bnmc/store.hpp:74-83
 *   bnmc_gpu_sweep         Engine::sweep             include/bnmc/sampler.hpp:60 (src/sampler.cpp:390-405)
 *   bnmc_gpu_run           Engine::run's sweep loop  include/bnmc/sampler.hpp:63 (src/sampler.cpp:426-455)
 *   bnmc_gpu_run_trace     Engine::run (Trace: samples, MAP, log-joints, timings) sampler.hpp:63
 *   bnmc_gpu_eval_log_joint Engine::eval_log_joint   include/bnmc/sampler.hpp:56 (src/sampler.cpp:44-46)
 *   bnmc_gpu_download      writes back the unobserved variables of the ParamStore
 *   bnmc_gpu_prior_init    prior_init                include/bnmc/sampler.hpp:97-99 (src/sampler.cpp:542-555)
 *   bnmc_gpu_dirichlet_batch sample_dirichlet_batch  include/bnmc/batch.hpp:33-34
 *   bnmc_gpu_probe_*       RngStream / draw_gamma / draw_from_log_weights
 *                          include/bnmc/rng.hpp:12-51, include/bnmc/dist.hpp:51,63
 *   bnmc_gpu_lpp           log_predictive_probability include/bnmc/metrics.hpp:16-18
 *   bnmc_gpu_partition     (new) document sharding across GPUs
 *
 * Error behaviour mirrors the reference's exceptions: the return code names the
 * C++ exception type the adapter rethrows (BNMC_GPU_ERR_RUNTIME -> RuntimeError,
 * BNMC_GPU_ERR_DOMAIN -> std::domain_error, BNMC_GPU_ERR_ARG ->
 * std::invalid_argument); bnmc_gpu_last_error() holds the message.
 */
#ifndef BNMC_GPU_H
#define BNMC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BNMC_GPU_ABI_VERSION 2

typedef enum {
  BNMC_GPU_LDA = 1,       /* proj/models/lda.bn, Gibbs: blocks phi, theta, z */
  BNMC_GPU_GMM = 2,       /* proj/models/gmm.bn, Gibbs: blocks pi, mu, sigma2, z */
  BNMC_GPU_MH_LINREG = 3, /* proj/models/regression.bn, method MH (one block w, b, tau) */
  BNMC_GPU_MH_LOGREG = 4, /* logistic twin of regression.bn (no reference model) */
  BNMC_GPU_CATMIX = 5,    /* proj/models/catmix.bn, Gibbs: theta, phi, z.  K, V, N */
  BNMC_GPU_NAIVEBAYES = 6,/* proj/models/naivebayes.bn, Gibbs: pC, pF (c, f observed).  K, N */
  BNMC_GPU_HMM = 7,       /* proj/models/hmm.bn, Gibbs: T, bias, s (sequential scan).  K = S states, N */
  BNMC_GPU_MH_POLYREG = 8 /* proj/models/polyreg.bn, method MH (one block w, bias).  K = M order, N */
} bnmc_gpu_kind;

typedef enum {
  BNMC_GPU_OBSERVE_PHI = 1u << 0,    /* LDA: phi clamped (RunConfig::observe_extra = {"phi"}) */
  BNMC_GPU_EXACT_WEIGHTS = 1u << 1,  /* LDA: log-space weights exactly as the reference
                                        (default: product-form theta*phi, same draws) */
  BNMC_GPU_NO_GRAPH = 1u << 2,       /* launch kernels directly instead of a CUDA graph */
  BNMC_GPU_GIBBS = 1u << 3,          /* regression / polyreg: Method::Gibbs plan -- one MH
                                        block per non-conjugate variable (w, b), conjugate
                                        tau (plan.cpp:139-164) -- instead of one MH block */
  BNMC_GPU_MWG = 1u << 4,            /* regression / polyreg: Method::MWG plan -- single-site
                                        blocks per element (run_mwg_block, sampler.cpp:342-388) */
  BNMC_GPU_TAU_PRECISION = 1u << 5   /* regression: tau is the noise PRECISION with a Gamma(shape,
                                        scale) prior, y ~ N(mean, pow(tau, -1)) -- the
                                        GammaPrecision conjugate kind (rewrite.cpp:538-549,
                                        sampler.cpp:205-207); hyper[4], hyper[5] = shape, scale */
} bnmc_gpu_flag;

typedef enum {
  BNMC_GPU_OK = 0,
  BNMC_GPU_ERR_ARG = 1,     /* std::invalid_argument */
  BNMC_GPU_ERR_RUNTIME = 2, /* bnmc::RuntimeError (shapes, bins out of range) */
  BNMC_GPU_ERR_DOMAIN = 3,  /* std::domain_error (all candidate log-weights -inf) */
  BNMC_GPU_ERR_CUDA = 4,    /* CUDA runtime failure / no device */
  BNMC_GPU_ERR_NCCL = 5
} bnmc_gpu_status;

/* Model description: what the reference Engine derives from (CheckedModel,
 * HyperValues, RunConfig).  Sizes are GLOBAL (all ranks). */
/* A peer group: W contexts of ONE process (one host thread per rank; one GPU per rank,
 * or several ranks sharing a GPU) whose collectives run as libbnmc_gpu's own all-reduce
 * kernel over peer memory instead of NCCL (see bnmc_gpu_group_create). */
typedef struct bnmc_gpu_group bnmc_gpu_group;

typedef struct bnmc_gpu_desc {
  int32_t abi_version;  /* = BNMC_GPU_ABI_VERSION */
  int32_t kind;         /* bnmc_gpu_kind */
  uint64_t seed;        /* RunConfig::seed -- every RNG key starts from it */
  int32_t device;       /* CUDA ordinal; -1 = current device */
  uint32_t flags;       /* bnmc_gpu_flag */
  /* LDA: K topics, V vocabulary, M documents, N tokens.
   * GMM: K components, N points.   MH: K features, N rows. */
  int64_t K, V, M, N;
  const int64_t* doc_offsets; /* LDA: M+1 prefix sums of N[i] (VarLayout::offsets), host */
  /* LDA: {alpha, beta}; GMM: {alpha, mu0, v0, a0, b0};
   * MH:  {lo, hi, w_var, b_var, tau_a, tau_b} */
  double hyper[8];
  /* Reference variable ids (declaration order; they are RNG key components):
   * LDA {phi, theta, z, w}; GMM {pi, mu, sigma2, z, x}; LINREG {w, b, tau, x, y};
   * LOGREG {w, b, x, y}; CATMIX {theta, phi, z, x}; NAIVEBAYES {pC, c, pF, f};
   * HMM {T, bias, s, flips}; POLYREG {w, bias, x, y}. */
  int32_t var_ids[8];
  double mh_scale;      /* RunConfig::mh_scale (PlanConfig, plan.hpp:31-33) */
  int32_t rank;         /* this process's shard (documents / rows) */
  int32_t world_size;   /* number of GPUs sharing the model; 1 = unsharded */
  const void* nccl_id;  /* 128-byte ncclUniqueId: world_size > 1 over NCCL (one process per GPU) */
  void* stream;         /* cudaStream_t to enqueue on; NULL = context-owned stream */
  bnmc_gpu_group* group;/* world_size > 1 inside one process: the ranks' shared group (instead
                           of nccl_id); such contexts launch without CUDA graphs */
} bnmc_gpu_desc;

/* A view of the reference ParamStore (store.hpp:74-83): flat arrays indexed by
 * variable id.  Arrays are GLOBAL; a sharded context reads/writes its slice. */
typedef struct bnmc_gpu_store {
  int32_t n_vars;
  double* const* real;   /* ParamStore::real[id].data() or NULL */
  int64_t* const* ival;  /* ParamStore::ival[id].data() or NULL */
  const int64_t* len;    /* flat length of each variable (VarLayout::flat_values) */
  const char* observed;  /* ParamStore::observed */
} bnmc_gpu_store;

typedef struct bnmc_gpu_ctx bnmc_gpu_ctx;

int bnmc_gpu_abi_version(void);
/* Peer groups (single-process sharding, e.g. one host thread per GPU of a node, or the
 * ranks of a sharded run emulated on one GPU).  Every collective of the W member
 * contexts is a rendezvous of their host threads: each rank must issue its calls from its
 * own thread, in the same order as the others (as with NCCL).  The group must outlive its
 * contexts.  Ranks on different GPUs need peer access (NVLink / NVSwitch). */
int bnmc_gpu_group_create(int32_t world_size, bnmc_gpu_group** out);
void bnmc_gpu_group_destroy(bnmc_gpu_group* group);
/* Thread-local message of the last failure (ctx may be NULL). */
const char* bnmc_gpu_last_error(const bnmc_gpu_ctx* ctx);

int bnmc_gpu_create(const bnmc_gpu_desc* desc, bnmc_gpu_ctx** out);
void bnmc_gpu_destroy(bnmc_gpu_ctx* ctx);

/* Copies the latent state and the observed data of `store` to the device. */
int bnmc_gpu_upload(bnmc_gpu_ctx* ctx, const bnmc_gpu_store* store);
/* Copies only the latent (unobserved) variables; observed data already on the
 * device is kept.  The per-call path of a bound store (Engine::sweep borrow). */
int bnmc_gpu_upload_state(bnmc_gpu_ctx* ctx, const bnmc_gpu_store* store);
/* Copies only the latent variables the next sweep reads (LDA: z -- the phi and theta
 * blocks redraw phi and theta from the counts first; other models: all latent
 * variables).  The per-call upload of Engine::sweep on a bound store. */
int bnmc_gpu_upload_sweep_inputs(bnmc_gpu_ctx* ctx, const bnmc_gpu_store* store);
/* Writes the device state back into the unobserved variables of `store`
 * (observed variables are never written, test_runtime.cpp:214-233). */
int bnmc_gpu_download(bnmc_gpu_ctx* ctx, const bnmc_gpu_store* store);

/* One sweep (all plan blocks + log-joint) for iteration `iter`; synchronous. */
int bnmc_gpu_sweep(bnmc_gpu_ctx* ctx, int64_t iter, double* log_joint, int* mh_accepted);
/* Engine::sweep on a caller's store in one call: upload what the sweep reads
 * (bnmc_gpu_upload_sweep_inputs), sweep, and write the latent state back -- LDA copies
 * phi and theta back while the z-step still runs.  LDA: when no other call ran on the
 * context since the previous sweep_store (on every rank: the decision is collective), the
 * sweep starts from the device
 * state (the z last written back to the caller) while the store's z is uploaded; the
 * upload is then compared with that z and, if the caller changed the store, the sweep
 * is redone from the upload -- results equal the non-speculative path's
 * (BNMC_SPECULATE=0) in every case.  On an error the store's latent variables are
 * unspecified. */
int bnmc_gpu_sweep_store(bnmc_gpu_ctx* ctx, const bnmc_gpu_store* store, int64_t iter, double* log_joint,
                         int* mh_accepted);
/* Page-locks the arrays of `store` (cudaHostRegister) for this context's copies, and
 * releases ranges registered earlier that the view no longer holds (a new or
 * reallocated store).  The reference's ParamStore is pageable std::vector memory; an
 * Engine that keeps borrowing the same store registers it once at binding.  The arrays
 * must stay allocated until bnmc_gpu_unregister_host / bnmc_gpu_destroy (or the next
 * register call with a different view).  Ranges already page-locked by their owner are
 * used as they are and never released here. */
int bnmc_gpu_register_host(bnmc_gpu_ctx* ctx, const bnmc_gpu_store* store);
int bnmc_gpu_unregister_host(bnmc_gpu_ctx* ctx);
/* Host <-> device bytes moved by the last bnmc_gpu_sweep_store call (LDA: z up; z,
 * theta, phi and the log-joint / accept ring entry down).  Models other than LDA
 * report only the ring entry. */
int bnmc_gpu_transfer_stats(bnmc_gpu_ctx* ctx, int64_t* h2d_bytes, int64_t* d2h_bytes);
/* n sweeps iter0..iter0+n-1 with one host sync; per-sweep outputs optional. */
int bnmc_gpu_run(bnmc_gpu_ctx* ctx, int64_t iter0, int64_t n, double* log_joints, int* accepted);
/* Engine::run (sampler.cpp:426-455) with a device-resident trace: burn-in + n kept
 * sweeps; the MAP state is tracked on the device (a conditional device copy after
 * every kept sweep whose log-joint beats the best so far, strict >, as the
 * reference), thinned samples (kept index % thin == 0) are written into
 * samples[i], the MAP state into map_state at the end.  No host round trip per
 * sweep except for the thinned downloads.  timing_ms[i] = device time of kept
 * sweep i (the reference times sweep() only).  Optional outputs may be NULL. */
typedef struct bnmc_gpu_trace {
  int64_t burnin, n, thin;
  double* log_joints;              /* [n] */
  double* timing_ms;               /* [n] */
  int* accepted;                   /* [n] MH accept flags */
  const bnmc_gpu_store* samples;   /* [ceil(n / thin)] host views to write */
  const bnmc_gpu_store* map_state; /* host view to write */
  double* map_log_joint;           /* -inf when no kept sweep */
} bnmc_gpu_trace;
int bnmc_gpu_run_trace(bnmc_gpu_ctx* ctx, int64_t iter0, bnmc_gpu_trace* trace);
/* Asynchronous variant of bnmc_gpu_run (no host sync); pair with bnmc_gpu_synchronize. */
int bnmc_gpu_enqueue(bnmc_gpu_ctx* ctx, int64_t iter0, int64_t n);
int bnmc_gpu_synchronize(bnmc_gpu_ctx* ctx, double* last_log_joint, int* last_accepted);
/* One sweep launched kernel by kernel with CUDA events between phases; ms[i] is
 * the device time of phase names[i] (for the roofline of the dominant kernel). */
int bnmc_gpu_sweep_phases(bnmc_gpu_ctx* ctx, int64_t iter, double* ms, const char** names, int cap,
                          int* n_phases);
/* ncclGetUniqueId for the rank-0 process of a sharded run (128 bytes). */
int bnmc_gpu_nccl_unique_id(void* out128);
/* Engine::eval_log_joint of the current device state. */
int bnmc_gpu_eval_log_joint(bnmc_gpu_ctx* ctx, double* log_joint);
/* prior_init(skip_observed = true) on the device (sampler.cpp:542-555). */
int bnmc_gpu_prior_init(bnmc_gpu_ctx* ctx, uint64_t seed);

/* Checkpoint / resume (the reference has none): the device state
 * of the model (state_buffers: LDA z, theta, phi draws + row sums; GMM z, pi, mu,
 * sigma2; MH w, b, tau; zoo models likewise) and the next iteration, in a binary file.
 * Loading into a context of the same model, sizes, shard and seed resumes the chain
 * exactly: the RNG streams are keyed by (seed, iteration, site). */
int bnmc_gpu_save_checkpoint(bnmc_gpu_ctx* ctx, const char* path);
int bnmc_gpu_load_checkpoint(bnmc_gpu_ctx* ctx, const char* path);
/* The iteration the next sweep will run (after a load: the checkpoint's). */
int bnmc_gpu_checkpoint_iter(const bnmc_gpu_ctx* ctx, int64_t* next_iter);
/* LDA binary corpus (.bnc) -- SURVEY.md 8f row 1, the format for corpora the JSON path
 * (data.cpp:27-136) cannot carry: "BNMCCORP", uint32 version = 1, uint32 0, int64 M,
 * int64 N, int64 V, int64 offsets[M + 1], int32 w[N].  This shard's tokens are streamed
 * to the device (range-checked); the offsets must equal the context's.  Observed data
 * only: follow with bnmc_gpu_prior_init (or an upload of the latent state). */
int bnmc_gpu_lda_load_corpus(bnmc_gpu_ctx* ctx, const char* path);
/* LDA diagnostics: topic-word counts of the current z, row-major K x V (global,
 * after the all-reduce), and this shard's doc-topic counts (local docs x K). */
int bnmc_gpu_lda_counts(bnmc_gpu_ctx* ctx, int32_t* nkw, int32_t* nmk);
/* LDA synthetic corpus on the device, following gen_lda's generative process
 * (gen.cpp:21-60) with per-token counter streams (not the reference's single
 * serial stream); fills w, then prior_init.  For configs the host cannot hold. */
int bnmc_gpu_lda_generate(bnmc_gpu_ctx* ctx, uint64_t seed, double phi_conc, double theta_conc);
/* Documents [begin, end) owned by `rank` under the balanced-token partition. */
int bnmc_gpu_partition(const int64_t* doc_offsets, int64_t M, int32_t world_size, int32_t rank,
                       int64_t* begin, int64_t* end);

/* log_predictive_probability (metrics.cpp:9-34) on the device: sum over held-out
 * tokens of log10 sum_k theta[d,k] phi[k,w]; phi K x V, theta docs x K, host. */
int bnmc_gpu_lpp(const double* phi, const double* theta, int64_t K, int64_t V, const int64_t* w,
                 const int64_t* offsets, int64_t docs, double* out);

/* sample_dirichlet_batch with per-row concentrations (batch.cpp:45-83) on the device. */
int bnmc_gpu_dirichlet_batch(int64_t rows, int64_t cols, const double* alpha, uint64_t key,
                             double* out);
/* Device read bandwidth (GB/s) over a `bytes` buffer read `reps` times by ONE persistent
 * launch: inside the 126 MB L2 it measures L2 -> SM bandwidth (bench.py's secondary
 * roofline), a multi-GB buffer HBM read bandwidth. */
int bnmc_gpu_probe_read_bandwidth(int64_t bytes, int32_t reps, double* gbps);
/* Primitive probes for known-answer parity (device RNG and draws). */
int bnmc_gpu_probe_rng(const uint64_t* keys, int64_t n, int64_t per_key, uint64_t* u64,
                       double* unit, double* gauss);
int bnmc_gpu_probe_gamma(const uint64_t* keys, const double* shapes, int64_t n, double* out,
                         uint64_t* counters);
int bnmc_gpu_probe_log_weights(const uint64_t* keys, const double* logw, int64_t rows,
                               int64_t cols, int64_t* picks);

#ifdef __cplusplus
}
#endif
#endif /* BNMC_GPU_H */
