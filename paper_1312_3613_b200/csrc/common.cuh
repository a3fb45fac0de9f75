// csrc/common.cuh -- shared internals of libbnmc_gpu.so (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bnmc_gpu.h"

namespace bnmc_gpu {

// Internal failures carry the C-ABI status they map to.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define BNMC_CUDA(x)                                                                   \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw ::bnmc_gpu::Error(BNMC_GPU_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define BNMC_NCCL(x)                                                                   \
  do {                                                                                 \
    ncclResult_t r_ = (x);                                                             \
    if (r_ != ncclSuccess)                                                             \
      throw ::bnmc_gpu::Error(BNMC_GPU_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

inline void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

// Device-side error flags, checked by the host at every synchronisation point.
enum : int {
  kErrBin = 1,     // conjugate update bin out of range  -> RuntimeError (sampler.cpp:89-91)
  kErrDomain = 2,  // all candidate log-weights -inf     -> std::domain_error (dist.cpp:205)
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  std::size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void alloc(std::size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count) BNMC_CUDA(cudaMalloc(&p, sizeof(T) * count));
  }
  void zero(cudaStream_t s) {
    if (n) BNMC_CUDA(cudaMemsetAsync(p, 0, sizeof(T) * n, s));
  }
  std::size_t bytes() const { return sizeof(T) * n; }
};

// Ring of per-sweep outputs; the finalize kernel of every model writes
// lj[iter % kRing], acc[iter % kRing] and then advances *iter.
constexpr int kRing = 4096;

struct Outputs {
  double* lj;
  int* acc;
  std::int64_t* iter;
  int* err;
};

// Deterministic block-wide sum (fixed butterfly + fixed warp order): the result
// depends only on the inputs and blockDim, never on scheduling.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// scratch: >= 32 doubles of shared memory. Result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double t = lane < nw ? scratch[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

// N block sums with one pair of barriers. scratch: >= 32 * N doubles. Results valid in
// every thread; fixed order as block_sum.
template <int N>
__device__ __forceinline__ void block_sum_n(double (&v)[N], double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) scratch[i * 32 + wid] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_sum(lane < nw ? scratch[i * 32 + lane] : 0.0);
}

// Model-specific device state behind one context.
struct Model {
  virtual ~Model() = default;
  // host <-> device bytes of the current Engine::sweep call (bnmc_gpu_transfer_stats);
  // counted by the models that implement the bound-store path
  std::int64_t h2d_bytes = 0, d2h_bytes = 0;
  // Speculative bound-store sweeps (bnmc_gpu_sweep_store).  `epoch` counts C-ABI calls
  // on the context; `spec_epoch` is the epoch of the last completed sweep_store.  When
  // nothing ran in between, the device state is the one the caller's store was last
  // written from, so the sweep may start from it while the store's latent state
  // crosses PCIe; the upload is then compared with that state and, if the caller
  // changed it, the sweep is redone from the upload.
  std::uint64_t epoch = 0, spec_epoch = ~std::uint64_t{0};
  // set by sweep_store around upload_sweep_inputs / spec_begin: no other call ran since
  // the previous sweep_store, so the device state is the one last written back
  bool quiet = false;
  // enqueue the upload of the sweep inputs into staging (side stream); false: no speculation
  virtual bool spec_begin(const bnmc_gpu_store&, cudaStream_t) { return false; }
  // enqueue: wait for the upload, compare it with the state the sweep started from
  virtual void spec_verify(cudaStream_t) {}
  // after a stream sync: did the store differ (the speculative sweep must be redone)?
  virtual bool spec_failed() { return false; }
  // the staged upload becomes the state (with upload_sweep_inputs' checks and counts)
  virtual void spec_adopt(cudaStream_t) {}
  virtual void upload(const bnmc_gpu_store& s, cudaStream_t st) = 0;
  virtual void download(const bnmc_gpu_store& s, cudaStream_t st) = 0;
  // Uploads only the latent (unobserved) variables: the observed data already on
  // the device is kept (the engine never writes observed arrays).
  virtual void upload_state(const bnmc_gpu_store& s, cudaStream_t st) { upload(s, st); }
  // Uploads the latent variables the next sweep actually reads (a bound store's
  // per-call path of Engine::sweep); the default is every latent variable.
  virtual void upload_sweep_inputs(const bnmc_gpu_store& s, cudaStream_t st) { upload_state(s, st); }
  // Enqueues one sweep (reads the iteration from *out.iter, advances it).
  virtual void enqueue_sweep(cudaStream_t st) = 0;
  // Enqueues Engine::eval_log_joint of the current state into lj[iter % kRing]
  // without advancing the iteration.
  virtual void enqueue_log_joint(cudaStream_t st) = 0;
  virtual void prior_init(std::uint64_t seed, cudaStream_t st) = 0;
  virtual void lda_counts(std::int32_t*, std::int32_t*, cudaStream_t) {
    throw Error(BNMC_GPU_ERR_ARG, "counts are only defined for LDA");
  }
  virtual void lda_generate(std::uint64_t, double, double, cudaStream_t) {
    throw Error(BNMC_GPU_ERR_ARG, "generate is only defined for LDA");
  }
  // The device buffers that fully determine the latent state (what download()
  // reads).  The trace run keeps a device copy of the MAP state by copying them
  // and downloads it by swapping the pointers in (bnmc_gpu_run_trace).
  struct StateBuf {
    void** p;
    std::size_t bytes;
  };
  virtual std::vector<StateBuf> state_buffers() { return {}; }
  // Download whose copies of variables finished early in the sweep overlap the rest of
  // it (the sweep was just enqueued on `st`); returns false when the model has no such
  // schedule (the caller then downloads after the sweep).
  virtual bool download_overlapped(const bnmc_gpu_store&, cudaStream_t) { return false; }
  // After state_buffers() were overwritten (checkpoint restore): rebuild whatever the
  // model derives from them (counts, caches).
  virtual void on_state_restored(cudaStream_t) {}
  // LDA: stream this shard's tokens of a binary corpus file into device memory.
  virtual void lda_load_corpus(const char*, cudaStream_t) {
    throw Error(BNMC_GPU_ERR_ARG, "binary corpora are only defined for LDA");
  }
  Outputs out{};

  // Per-phase timing (bnmc_gpu_sweep_phases): when `marks` is set, every phase
  // boundary records an event on the launching stream.
  struct Mark {
    const char* name;
    cudaEvent_t ev;
  };
  std::vector<Mark>* marks = nullptr;
  void mark(cudaStream_t st, const char* name) {
    if (!marks) return;
    cudaEvent_t e;
    BNMC_CUDA(cudaEventCreate(&e));
    BNMC_CUDA(cudaEventRecord(e, st));
    marks->push_back({name, e});
  }
};

// Collectives of a sharded model, over one of two transports:
//  * NCCL: one process per GPU (an ncclUniqueId in the desc); or a 1-rank communicator
//    forced with BNMC_FORCE_NCCL=1 (the sharded code path on one GPU);
//  * a peer group (bnmc_gpu_group, comm.cu): the ranks are contexts of ONE process, one
//    host thread each, on one GPU or several; the all-reduce is our own kernel over peer
//    memory (rank r reduces chunk r of every rank's buffer and stores the result into
//    every rank's buffer: P2P loads / stores over NVLink, plain loads when the ranks share
//    a GPU), ordered against the ranks' streams by events and a host rendezvous.
enum class RedType { I32, F64 };
enum class RedOp { Sum, Min, Max };
struct PeerGroup;

struct Comm {
  ncclComm_t comm = nullptr;
  PeerGroup* group = nullptr;
  int rank = 0, world = 1;
  // the sharded code paths run whenever a transport exists (world > 1 or forced NCCL)
  bool active() const { return comm != nullptr || group != nullptr; }
  // in-place all-reduce of n elements on stream st (collective: every rank calls it)
  void all_reduce(void* buf, std::size_t n, RedType t, RedOp op, cudaStream_t st) const;
  // in place over world chunks of `chunk` elements: rank r keeps the sum of chunk r /
  // every rank receives each rank's own chunk (collective: every rank calls it)
  void reduce_scatter(void* buf, std::size_t chunk, RedType t, cudaStream_t st) const;
  void all_gather(void* buf, std::size_t chunk, RedType t, cudaStream_t st) const;
};

// Peer groups (comm.cu): join at context creation, leave at destruction.
PeerGroup* group_of(bnmc_gpu_group* g);
void peer_group_join(PeerGroup* g, int rank, int world, int device);
void peer_group_leave(PeerGroup* g, int rank);

std::unique_ptr<Model> make_lda(const bnmc_gpu_desc& d, const Comm& c, Outputs o);
std::unique_ptr<Model> make_gmm(const bnmc_gpu_desc& d, const Comm& c, Outputs o);
std::unique_ptr<Model> make_mh(const bnmc_gpu_desc& d, const Comm& c, Outputs o);
std::unique_ptr<Model> make_zoo(const bnmc_gpu_desc& d, const Comm& c, Outputs o);

// Balanced-token document partition (shared by the C-ABI and the models).
void partition_docs(const std::int64_t* off, std::int64_t M, int world, int rank, std::int64_t* b,
                    std::int64_t* e);

inline unsigned blocks_for(std::int64_t n, int bt) {
  return static_cast<unsigned>((n + bt - 1) / bt);
}

}  // namespace bnmc_gpu
