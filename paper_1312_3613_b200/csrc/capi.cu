// csrc/capi.cu -- the extern "C" boundary (include/bnmc_gpu.h).
//
// A context owns one CUDA stream, the device state of one model, an optional NCCL
// communicator over NVLink (document / row sharding), and a CUDA graph of one
// sweep.  The iteration number lives on the device (*iter) and the graph's last
// kernel advances it, so n sweeps are n graph launches with no host round trip;
// log-joints land in a device ring read back at synchronisation points.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "rng.cuh"

namespace bnmc_gpu {
void probe_rng(const std::uint64_t*, std::int64_t, std::int64_t, std::uint64_t*, double*, double*);
void probe_gamma(const std::uint64_t*, const double*, std::int64_t, double*, std::uint64_t*);
void probe_log_weights(const std::uint64_t*, const double*, std::int64_t, std::int64_t, std::int64_t*);
double probe_read_bandwidth(std::size_t, int);
void dirichlet_batch(std::int64_t, std::int64_t, const double*, std::uint64_t, double*);
double lpp(const double*, const double*, std::int64_t, std::int64_t, const std::int64_t*,
           const std::int64_t*, std::int64_t);

void partition_docs(const std::int64_t* off, std::int64_t M, int world, int rank, std::int64_t* b,
                    std::int64_t* e) {
  // Contiguous documents balanced by token count: rank r owns the documents whose
  // first token lies in [r*N/world, (r+1)*N/world) (lower_bound on the prefix sums).
  const std::int64_t N = off[M];
  auto bound = [&](int r) -> std::int64_t {
    if (r <= 0) return 0;
    if (r >= world) return M;
    const std::int64_t target = static_cast<std::int64_t>((static_cast<__int128>(N) * r) / world);
    return static_cast<std::int64_t>(std::lower_bound(off, off + M, target) - off);
  };
  *b = bound(rank);
  *e = bound(rank + 1);
}
}  // namespace bnmc_gpu

using namespace bnmc_gpu;

struct bnmc_gpu_ctx {
  bnmc_gpu_desc desc{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  Comm comm;
  std::unique_ptr<Model> model;
  DevBuf<double> lj;
  DevBuf<int> acc;
  DevBuf<std::int64_t> iter;
  DevBuf<int> err;
  std::int64_t* host_iter = nullptr;  // pinned
  int* host_err = nullptr;            // pinned: the device error word, fetched by read_ring
  bool err_fetched = false;           // host_err holds the word as of the last stream sync
  std::int64_t next_iter = -1;        // device *iter value after the enqueued work
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::string last_error;
  // host ranges this context page-locked (bnmc_gpu_register_host): the caller's store
  std::vector<std::pair<void*, std::size_t>> registered;
};

namespace {

thread_local std::string g_last_error;

int fail(bnmc_gpu_ctx* ctx, int code, const std::string& msg) {
  g_last_error = msg;
  if (ctx) ctx->last_error = msg;
  return code;
}

template <class F>
int guarded(bnmc_gpu_ctx* ctx, F&& f) {
  try {
    if (ctx) BNMC_CUDA(cudaSetDevice(ctx->device));
    if (ctx && ctx->model) ++ctx->model->epoch;  // any call may change the device state
    if (ctx) ctx->err_fetched = false;
    f();
    return BNMC_GPU_OK;
  } catch (const Error& e) {
    return fail(ctx, e.code, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ctx, BNMC_GPU_ERR_RUNTIME, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, BNMC_GPU_ERR_RUNTIME, e.what());
  }
}

void check_device_error(bnmc_gpu_ctx* c) {
  int e = 0;
  if (c->err_fetched) {  // read_ring already brought the word back with its sync
    e = *c->host_err;
    c->err_fetched = false;
  } else {
    BNMC_CUDA(cudaMemcpyAsync(&e, c->err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    BNMC_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (e) {
    BNMC_CUDA(cudaMemsetAsync(c->err.p, 0, sizeof(int), c->stream));
    BNMC_CUDA(cudaStreamSynchronize(c->stream));
    if (e & kErrBin) throw Error(BNMC_GPU_ERR_RUNTIME, "conjugate update bin out of range (assignment outside the support)");
    if (e & kErrDomain) throw Error(BNMC_GPU_ERR_DOMAIN, "all candidate log-weights are -inf");
    throw Error(BNMC_GPU_ERR_RUNTIME, "device reported an invalid state");
  }
}

void set_iter(bnmc_gpu_ctx* c, std::int64_t it) {
  if (c->next_iter == it) return;
  BNMC_CUDA(cudaStreamSynchronize(c->stream));
  *c->host_iter = it;
  BNMC_CUDA(cudaMemcpyAsync(c->iter.p, c->host_iter, sizeof(std::int64_t), cudaMemcpyHostToDevice, c->stream));
  BNMC_CUDA(cudaStreamSynchronize(c->stream));
  c->next_iter = it;
}

void launch_sweep(bnmc_gpu_ctx* c) {
  c->err_fetched = false;  // work enqueued after the last fetch of the error word
  if (c->desc.flags & BNMC_GPU_NO_GRAPH) {
    c->model->enqueue_sweep(c->stream);
  } else {
    if (!c->exec) {
      BNMC_CUDA(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
      try {
        c->model->enqueue_sweep(c->stream);
      } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(c->stream, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      BNMC_CUDA(cudaStreamEndCapture(c->stream, &c->graph));
      BNMC_CUDA(cudaGraphInstantiate(&c->exec, c->graph, 0));
    }
    BNMC_CUDA(cudaGraphLaunch(c->exec, c->stream));
  }
  c->next_iter += 1;
}

void read_ring(bnmc_gpu_ctx* c, std::int64_t it0, std::int64_t n, double* lj, int* acc, bool sync = true) {
  // Entries it0 .. it0+n-1 (n <= kRing), possibly wrapping.
  const std::int64_t s = it0 & (kRing - 1);
  const std::int64_t first = std::min<std::int64_t>(n, kRing - s);
  if (lj) {
    BNMC_CUDA(cudaMemcpyAsync(lj, c->lj.p + s, sizeof(double) * first, cudaMemcpyDeviceToHost, c->stream));
    if (n > first)
      BNMC_CUDA(cudaMemcpyAsync(lj + first, c->lj.p, sizeof(double) * (n - first), cudaMemcpyDeviceToHost, c->stream));
  }
  if (acc) {
    BNMC_CUDA(cudaMemcpyAsync(acc, c->acc.p + s, sizeof(int) * first, cudaMemcpyDeviceToHost, c->stream));
    if (n > first)
      BNMC_CUDA(cudaMemcpyAsync(acc + first, c->acc.p, sizeof(int) * (n - first), cudaMemcpyDeviceToHost, c->stream));
  }
  BNMC_CUDA(cudaMemcpyAsync(c->host_err, c->err.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (!sync) return;  // the caller's next stream synchronisation completes the copies
  BNMC_CUDA(cudaStreamSynchronize(c->stream));
  c->err_fetched = true;
}

// MAP tracking on the device (bnmc_gpu_run_trace): the sweep just advanced *iter;
// its log-joint sits in lj[(*iter - 1) % kRing].
__global__ void map_check_kernel(const double* lj, const std::int64_t* iter, double* map_lj, int* flag) {
  const double v = lj[(*iter - 1) & (kRing - 1)];
  const bool better = v > *map_lj;  // strict, NaN never better (sampler.cpp:449)
  if (better) *map_lj = v;
  *flag = better ? 1 : 0;
}

struct CopyTab {
  const unsigned* src[8];
  unsigned* dst[8];
  std::size_t words[8];
  int n;
};

__global__ void cond_copy_kernel(CopyTab t, const int* flag) {  // flag == nullptr: always
  if (flag && !*flag) return;
  const std::size_t stride = static_cast<std::size_t>(gridDim.x) * blockDim.x;
  for (int b = 0; b < t.n; ++b)
    for (std::size_t i = blockIdx.x * static_cast<std::size_t>(blockDim.x) + threadIdx.x; i < t.words[b]; i += stride)
      t.dst[b][i] = t.src[b][i];
}

}  // namespace

extern "C" {

int bnmc_gpu_abi_version(void) { return BNMC_GPU_ABI_VERSION; }

const char* bnmc_gpu_last_error(const bnmc_gpu_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : g_last_error.c_str();
}

int bnmc_gpu_create(const bnmc_gpu_desc* desc, bnmc_gpu_ctx** out) {
  if (!desc || !out) return fail(nullptr, BNMC_GPU_ERR_ARG, "null argument");
  *out = nullptr;
  auto c = std::make_unique<bnmc_gpu_ctx>();
  const int rc = guarded(nullptr, [&] {
    require(desc->abi_version == BNMC_GPU_ABI_VERSION, BNMC_GPU_ERR_ARG, "ABI version mismatch");
    int ndev = 0;
    BNMC_CUDA(cudaGetDeviceCount(&ndev));
    require(ndev > 0, BNMC_GPU_ERR_CUDA, "no CUDA device");
    c->desc = *desc;
    c->desc.doc_offsets = nullptr;  // not retained
    c->desc.nccl_id = nullptr;
    c->desc.group = nullptr;
    if (desc->device >= 0) {
      c->device = desc->device;
    } else {
      BNMC_CUDA(cudaGetDevice(&c->device));
    }
    BNMC_CUDA(cudaSetDevice(c->device));
    cudaDeviceProp prop{};
    BNMC_CUDA(cudaGetDeviceProperties(&prop, c->device));
    require(prop.major >= 10, BNMC_GPU_ERR_CUDA,
            std::string("libbnmc_gpu is built for sm_100a; device is ") + prop.name);
    if (desc->stream) {
      c->stream = static_cast<cudaStream_t>(desc->stream);
    } else {
      BNMC_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    c->comm.world = std::max(1, desc->world_size);
    c->comm.rank = desc->rank;
    require(c->comm.rank >= 0 && c->comm.rank < c->comm.world, BNMC_GPU_ERR_ARG, "rank out of range");
    const char* fn = std::getenv("BNMC_FORCE_NCCL");
    const bool force = fn && std::string(fn) == "1" && c->comm.world == 1 &&
                       (desc->kind == BNMC_GPU_LDA || desc->kind == BNMC_GPU_MH_LINREG ||
                        desc->kind == BNMC_GPU_MH_LOGREG || desc->kind == BNMC_GPU_MH_POLYREG);
    if (desc->group) {  // single-process ranks: our peer-memory all-reduce (comm.cu)
      require(c->comm.world > 1, BNMC_GPU_ERR_ARG, "a peer group needs world_size > 1");
      require(desc->nccl_id == nullptr, BNMC_GPU_ERR_ARG, "give either an ncclUniqueId or a peer group");
      c->comm.group = group_of(desc->group);
      peer_group_join(c->comm.group, c->comm.rank, c->comm.world, c->device);
      c->desc.flags |= BNMC_GPU_NO_GRAPH;  // cross-context event waits cannot be captured
    } else if (c->comm.world > 1 || force) {
      ncclUniqueId id;
      if (c->comm.world > 1) {
        require(desc->nccl_id != nullptr, BNMC_GPU_ERR_ARG, "world_size > 1 needs an ncclUniqueId");
        std::memcpy(&id, desc->nccl_id, sizeof(id));
      } else {
        BNMC_NCCL(ncclGetUniqueId(&id));  // a 1-rank communicator (test hook)
      }
      BNMC_NCCL(ncclCommInitRank(&c->comm.comm, c->comm.world, id, c->comm.rank));
    }
    c->lj.alloc(kRing);
    c->acc.alloc(kRing);
    c->iter.alloc(1);
    c->err.alloc(1);
    c->lj.zero(c->stream);
    c->acc.zero(c->stream);
    c->iter.zero(c->stream);
    c->err.zero(c->stream);
    BNMC_CUDA(cudaMallocHost(&c->host_iter, sizeof(std::int64_t)));
    BNMC_CUDA(cudaMallocHost(&c->host_err, sizeof(int)));
    c->next_iter = 0;
    Outputs o{c->lj.p, c->acc.p, c->iter.p, c->err.p};
    switch (desc->kind) {
      case BNMC_GPU_LDA: c->model = make_lda(*desc, c->comm, o); break;
      case BNMC_GPU_GMM: c->model = make_gmm(*desc, c->comm, o); break;
      case BNMC_GPU_MH_LINREG:
      case BNMC_GPU_MH_LOGREG:
      case BNMC_GPU_MH_POLYREG: c->model = make_mh(*desc, c->comm, o); break;
      case BNMC_GPU_CATMIX:
      case BNMC_GPU_NAIVEBAYES:
      case BNMC_GPU_HMM: c->model = make_zoo(*desc, c->comm, o); break;
      default: throw Error(BNMC_GPU_ERR_ARG, "unknown model kind");
    }
    BNMC_CUDA(cudaStreamSynchronize(c->stream));
  });
  if (rc != BNMC_GPU_OK) {
    bnmc_gpu_destroy(c.release());
    return rc;
  }
  *out = c.release();
  return BNMC_GPU_OK;
}

void bnmc_gpu_destroy(bnmc_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& r : c->registered) cudaHostUnregister(r.first);
  if (c->exec) cudaGraphExecDestroy(c->exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  c->model.reset();
  if (c->comm.comm) ncclCommDestroy(c->comm.comm);
  if (c->comm.group) peer_group_leave(c->comm.group, c->comm.rank);
  if (c->host_iter) cudaFreeHost(c->host_iter);
  if (c->host_err) cudaFreeHost(c->host_err);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int bnmc_gpu_upload(bnmc_gpu_ctx* c, const bnmc_gpu_store* s) {
  if (!c || !s) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    require(s->len != nullptr && s->real != nullptr && s->ival != nullptr, BNMC_GPU_ERR_ARG,
            "store view is incomplete");
    c->model->upload(*s, c->stream);
    check_device_error(c);
  });
}

int bnmc_gpu_upload_state(bnmc_gpu_ctx* c, const bnmc_gpu_store* s) {
  if (!c || !s) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    require(s->len != nullptr && s->real != nullptr && s->ival != nullptr, BNMC_GPU_ERR_ARG,
            "store view is incomplete");
    c->model->upload_state(*s, c->stream);
    check_device_error(c);
  });
}

int bnmc_gpu_upload_sweep_inputs(bnmc_gpu_ctx* c, const bnmc_gpu_store* s) {
  if (!c || !s) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    require(s->len != nullptr && s->real != nullptr && s->ival != nullptr, BNMC_GPU_ERR_ARG,
            "store view is incomplete");
    c->model->upload_sweep_inputs(*s, c->stream);  // range errors surface at the sweep's check
  });
}

int bnmc_gpu_sweep_phases(bnmc_gpu_ctx* c, std::int64_t iter, double* ms, const char** names, int cap,
                          int* n_out) {
  if (!c || !ms || !n_out) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    set_iter(c, iter);
    std::vector<Model::Mark> marks;
    c->model->marks = &marks;
    try {
      c->model->enqueue_sweep(c->stream);
    } catch (...) {
      c->model->marks = nullptr;
      for (auto& m : marks) cudaEventDestroy(m.ev);
      throw;
    }
    c->model->marks = nullptr;
    c->next_iter += 1;
    BNMC_CUDA(cudaStreamSynchronize(c->stream));
    int n = 0;
    for (std::size_t i = 1; i < marks.size() && n < cap; ++i, ++n) {
      float t = 0.f;
      BNMC_CUDA(cudaEventElapsedTime(&t, marks[i - 1].ev, marks[i].ev));
      ms[n] = t;
      if (names) names[n] = marks[i].name;
    }
    for (auto& m : marks) cudaEventDestroy(m.ev);
    *n_out = n;
    check_device_error(c);
  });
}

int bnmc_gpu_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(nullptr, [&] {
    ncclUniqueId id;
    BNMC_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int bnmc_gpu_download(bnmc_gpu_ctx* c, const bnmc_gpu_store* s) {
  if (!c || !s) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    c->model->download(*s, c->stream);
    check_device_error(c);
  });
}

int bnmc_gpu_sweep(bnmc_gpu_ctx* c, std::int64_t iter, double* log_joint, int* mh_accepted) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    require(iter >= 0, BNMC_GPU_ERR_ARG, "iteration must be non-negative");
    set_iter(c, iter);
    launch_sweep(c);
    read_ring(c, iter, 1, log_joint, mh_accepted);
    check_device_error(c);
  });
}

int bnmc_gpu_sweep_store(bnmc_gpu_ctx* c, const bnmc_gpu_store* s, std::int64_t iter, double* log_joint,
                         int* mh_accepted) {
  if (!c || !s) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    require(iter >= 0, BNMC_GPU_ERR_ARG, "iteration must be non-negative");
    require(s->len != nullptr && s->real != nullptr && s->ival != nullptr, BNMC_GPU_ERR_ARG,
            "store view is incomplete");
    Model* m = c->model.get();
    m->h2d_bytes = m->d2h_bytes = 0;
    // speculative when no other call ran since the last sweep_store (see Model::epoch)
    m->quiet = m->spec_epoch + 1 == m->epoch;
    const bool spec = m->spec_begin(*s, c->stream);  // (collective for sharded models)
    if (!spec) m->upload_sweep_inputs(*s, c->stream);
    m->quiet = false;
    auto sweep_and_write_back = [&](bool verify) {
      set_iter(c, iter);
      launch_sweep(c);
      if (verify) m->spec_verify(c->stream);
      if (!m->download_overlapped(*s, c->stream)) {
        read_ring(c, iter, 1, log_joint, mh_accepted, false);
        m->download(*s, c->stream);  // synchronises the stream: the ring entry and error word too
        BNMC_CUDA(cudaStreamSynchronize(c->stream));  // (idle already: guards a model that did not)
        c->err_fetched = true;
        check_device_error(c);
        return;
      }
      read_ring(c, iter, 1, log_joint, mh_accepted);  // synchronises the stream (and the copies)
      check_device_error(c);
    };
    sweep_and_write_back(spec);
    if (spec && m->spec_failed()) {  // the caller changed the store: redo from its state
      m->spec_adopt(c->stream);
      sweep_and_write_back(false);
    }
    m->d2h_bytes += static_cast<std::int64_t>(sizeof(double) + sizeof(int));  // the ring entry
    m->spec_epoch = m->epoch;
  });
}

int bnmc_gpu_register_host(bnmc_gpu_ctx* c, const bnmc_gpu_store* s) {
  if (!c || !s) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  // Host-side only: the device state is untouched, so no epoch bump (a following
  // bnmc_gpu_sweep_store may still start speculatively).
  try {
    BNMC_CUDA(cudaSetDevice(c->device));
    require(s->len != nullptr && s->real != nullptr && s->ival != nullptr, BNMC_GPU_ERR_ARG,
            "store view is incomplete");
    std::vector<std::pair<void*, std::size_t>> want;
    for (int i = 0; i < s->n_vars; ++i) {
      void* p = s->real[i] ? static_cast<void*>(s->real[i]) : static_cast<void*>(s->ival[i]);
      if (p && s->len[i] > 0) want.emplace_back(p, static_cast<std::size_t>(s->len[i]) * 8);
    }
    std::vector<std::pair<void*, std::size_t>> keep;
    for (auto& r : c->registered) {
      if (std::find(want.begin(), want.end(), r) != want.end()) {
        keep.push_back(r);
      } else {
        cudaHostUnregister(r.first);  // a range of a store no longer bound (or reallocated)
        cudaGetLastError();
      }
    }
    c->registered = keep;
    for (auto& r : want) {
      if (std::find(c->registered.begin(), c->registered.end(), r) != c->registered.end()) continue;
      cudaPointerAttributes pa{};
      if (cudaPointerGetAttributes(&pa, r.first) == cudaSuccess && pa.type == cudaMemoryTypeHost) continue;
      cudaGetLastError();  // (pageable memory: "not a CUDA pointer" on older drivers)
      const cudaError_t e = cudaHostRegister(r.first, r.second, cudaHostRegisterDefault);
      if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();  // page-locked by its owner already: not ours to release
        continue;
      }
      BNMC_CUDA(e);
      c->registered.push_back(r);
    }
    return BNMC_GPU_OK;
  } catch (const Error& e) {
    return fail(c, e.code, e.what());
  }
}

int bnmc_gpu_unregister_host(bnmc_gpu_ctx* c) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& r : c->registered) cudaHostUnregister(r.first);
  cudaGetLastError();
  c->registered.clear();
  return BNMC_GPU_OK;
}

int bnmc_gpu_transfer_stats(bnmc_gpu_ctx* c, int64_t* h2d_bytes, int64_t* d2h_bytes) {
  if (!c || !h2d_bytes || !d2h_bytes) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    require(c->model != nullptr, BNMC_GPU_ERR_RUNTIME, "no model");
    *h2d_bytes = c->model->h2d_bytes;
    *d2h_bytes = c->model->d2h_bytes;
  });
}

int bnmc_gpu_run(bnmc_gpu_ctx* c, std::int64_t iter0, std::int64_t n, double* log_joints, int* accepted) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    require(iter0 >= 0 && n >= 0, BNMC_GPU_ERR_ARG, "bad iteration range");
    set_iter(c, iter0);
    for (std::int64_t done = 0; done < n;) {
      const std::int64_t chunk = std::min<std::int64_t>(n - done, kRing);
      for (std::int64_t i = 0; i < chunk; ++i) launch_sweep(c);
      read_ring(c, iter0 + done, chunk, log_joints ? log_joints + done : nullptr,
                accepted ? accepted + done : nullptr);
      check_device_error(c);
      done += chunk;
    }
  });
}

int bnmc_gpu_run_trace(bnmc_gpu_ctx* c, std::int64_t iter0, bnmc_gpu_trace* tr) {
  if (!c || !tr) return fail(c, BNMC_GPU_ERR_ARG, "null context or trace");
  return guarded(c, [&] {
    require(iter0 >= 0 && tr->n >= 0 && tr->burnin >= 0 && tr->thin >= 1, BNMC_GPU_ERR_ARG,
            "bad trace arguments (n, burnin >= 0, thin >= 1)");
    auto bufs = c->model->state_buffers();
    require(bufs.size() <= 8, BNMC_GPU_ERR_RUNTIME, "too many state buffers");
    // device MAP copy of the state + best log-joint + flag
    std::vector<DevBuf<unsigned>> map(bufs.size());
    CopyTab tab{};
    tab.n = static_cast<int>(bufs.size());
    for (std::size_t i = 0; i < bufs.size(); ++i) {
      map[i].alloc((bufs[i].bytes + 3) / 4);
      tab.words[i] = bufs[i].bytes / 4;
    }
    DevBuf<double> map_lj;
    DevBuf<int> flag;
    map_lj.alloc(1);
    flag.alloc(1);
    const double ninf = -INFINITY;
    BNMC_CUDA(cudaMemcpyAsync(map_lj.p, &ninf, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    std::vector<cudaEvent_t> ev;
    // Thinned samples: the state is copied on the device into one of two snapshot slots
    // (stream order), and the slot is written into the caller's sample store by the
    // model's download on a copy stream at the next sample point -- while the sweeps
    // launched since run on the GPU -- instead of a synchronous download per sample.
    std::vector<DevBuf<unsigned>> slot[2];
    cudaEvent_t ev_snap[2] = {nullptr, nullptr};
    cudaStream_t cp = nullptr;
    std::int64_t pending = -1;  // sample index whose snapshot awaits its download
    int pending_slot = 0;
    auto cleanup = [&] {
      for (auto e : ev) cudaEventDestroy(e);
      for (auto e : ev_snap)
        if (e) cudaEventDestroy(e);
      if (cp) cudaStreamDestroy(cp);
    };
    auto with_state = [&](std::vector<DevBuf<unsigned>>& bufs_in, auto&& f) {
      // the model's download reads its state buffers: swap a copy in and out
      for (std::size_t i = 0; i < bufs.size(); ++i) std::swap(*bufs[i].p, *reinterpret_cast<void**>(&bufs_in[i].p));
      try {
        f();
      } catch (...) {
        for (std::size_t i = 0; i < bufs.size(); ++i) std::swap(*bufs[i].p, *reinterpret_cast<void**>(&bufs_in[i].p));
        throw;
      }
      for (std::size_t i = 0; i < bufs.size(); ++i) std::swap(*bufs[i].p, *reinterpret_cast<void**>(&bufs_in[i].p));
    };
    auto flush_sample = [&] {
      if (pending < 0) return;
      BNMC_CUDA(cudaStreamWaitEvent(cp, ev_snap[pending_slot], 0));
      with_state(slot[pending_slot], [&] { c->model->download(tr->samples[pending], cp); });
      pending = -1;
    };
    try {
      set_iter(c, iter0);
      for (std::int64_t i = 0; i < tr->burnin; ++i) launch_sweep(c);
      if (tr->timing_ms) {
        ev.resize(static_cast<std::size_t>(2 * tr->n));
        for (auto& e : ev) BNMC_CUDA(cudaEventCreate(&e));
      }
      std::int64_t read = 0;  // kept log-joints already copied out
      auto drain = [&](std::int64_t upto) {
        if (upto > read) {
          read_ring(c, iter0 + tr->burnin + read, upto - read, tr->log_joints ? tr->log_joints + read : nullptr,
                    tr->accepted ? tr->accepted + read : nullptr);
          read = upto;
        }
      };
      std::int64_t sample = 0;
      for (std::int64_t s = 0; s < tr->n; ++s) {
        if (s - read >= kRing) drain(s);
        if (tr->timing_ms) BNMC_CUDA(cudaEventRecord(ev[2 * s], c->stream));
        launch_sweep(c);
        if (tr->timing_ms) BNMC_CUDA(cudaEventRecord(ev[2 * s + 1], c->stream));
        if (tr->map_state || tr->map_log_joint) {
          map_check_kernel<<<1, 1, 0, c->stream>>>(c->lj.p, c->iter.p, map_lj.p, flag.p);
          for (std::size_t i = 0; i < bufs.size(); ++i) {
            tab.src[i] = static_cast<const unsigned*>(*bufs[i].p);
            tab.dst[i] = map[i].p;
          }
          cond_copy_kernel<<<148 * 4, 256, 0, c->stream>>>(tab, flag.p);
        }
        if (tr->samples && s % tr->thin == 0) {
          flush_sample();  // the previous sample, overlapping the sweep just launched
          const int j = static_cast<int>(sample & 1);
          if (slot[j].empty()) {
            slot[j] = std::vector<DevBuf<unsigned>>(bufs.size());
            for (std::size_t i = 0; i < bufs.size(); ++i) slot[j][i].alloc((bufs[i].bytes + 3) / 4);
            if (!cp) BNMC_CUDA(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
            BNMC_CUDA(cudaEventCreateWithFlags(&ev_snap[j], cudaEventDisableTiming));
          }
          CopyTab snap{};
          snap.n = static_cast<int>(bufs.size());
          for (std::size_t i = 0; i < bufs.size(); ++i) {
            snap.src[i] = static_cast<const unsigned*>(*bufs[i].p);
            snap.dst[i] = slot[j][i].p;
            snap.words[i] = bufs[i].bytes / 4;
          }
          cond_copy_kernel<<<148 * 4, 256, 0, c->stream>>>(snap, nullptr);
          BNMC_CUDA(cudaEventRecord(ev_snap[j], c->stream));
          pending = sample++;
          pending_slot = j;
        }
      }
      flush_sample();
      drain(tr->n);
      check_device_error(c);
      if (tr->timing_ms)
        for (std::int64_t s = 0; s < tr->n; ++s) {
          float ms = 0.f;
          BNMC_CUDA(cudaEventElapsedTime(&ms, ev[2 * s], ev[2 * s + 1]));
          tr->timing_ms[s] = ms;
        }
      if (tr->map_log_joint)
        BNMC_CUDA(cudaMemcpy(tr->map_log_joint, map_lj.p, sizeof(double), cudaMemcpyDeviceToHost));
      if (tr->map_state && tr->n > 0) {
        with_state(map, [&] { c->model->download(*tr->map_state, c->stream); });
      }
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

namespace {
struct CkptHeader {
  char magic[8];
  std::uint32_t version;
  std::int32_t kind;
  std::int64_t K, V, M, N;
  std::uint64_t seed;
  std::int64_t next_iter;
  std::int32_t rank, world;
  std::uint32_t nbufs, pad;
  // version 2: the configuration that shapes the chain -- a checkpoint resumes only into
  // a context with the same flags (exact weights, observed phi, Gibbs / MWG plan), MH
  // proposal scale and hyperparameters
  std::uint32_t flags, pad2;
  double mh_scale;
  double hyper[8];
};
constexpr std::uint32_t kCkptVersion = 2;
// flags that do not change the chain (launch mode only)
constexpr std::uint32_t kCkptIgnoredFlags = BNMC_GPU_NO_GRAPH;

struct FileCloser {
  std::FILE* f;
  ~FileCloser() {
    if (f) std::fclose(f);
  }
};

CkptHeader ckpt_header(const bnmc_gpu_ctx* c, std::uint32_t nbufs) {
  CkptHeader h{};
  std::memcpy(h.magic, "BNMCCKPT", 8);
  h.version = kCkptVersion;
  h.kind = c->desc.kind;
  h.K = c->desc.K;
  h.V = c->desc.V;
  h.M = c->desc.M;
  h.N = c->desc.N;
  h.seed = c->desc.seed;
  h.next_iter = c->next_iter;
  h.rank = c->comm.rank;
  h.world = c->comm.world;
  h.nbufs = nbufs;
  h.flags = c->desc.flags & ~kCkptIgnoredFlags;
  h.mh_scale = c->desc.mh_scale;
  for (int i = 0; i < 8; ++i) h.hyper[i] = c->desc.hyper[i];
  return h;
}
}  // namespace

int bnmc_gpu_save_checkpoint(bnmc_gpu_ctx* c, const char* path) {
  if (!c || !path) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    BNMC_CUDA(cudaStreamSynchronize(c->stream));
    check_device_error(c);
    auto bufs = c->model->state_buffers();
    require(!bufs.empty(), BNMC_GPU_ERR_ARG, "this model has no checkpointable state");
    std::FILE* f = std::fopen(path, "wb");
    require(f != nullptr, BNMC_GPU_ERR_RUNTIME, std::string("cannot write ") + path);
    FileCloser fc{f};
    const CkptHeader h = ckpt_header(c, static_cast<std::uint32_t>(bufs.size()));
    require(std::fwrite(&h, sizeof(h), 1, f) == 1, BNMC_GPU_ERR_RUNTIME, "checkpoint write failed");
    std::vector<unsigned char> host;
    for (const auto& b : bufs) {
      const std::uint64_t n = b.bytes;
      host.resize(static_cast<std::size_t>(n));
      if (n) BNMC_CUDA(cudaMemcpy(host.data(), *b.p, n, cudaMemcpyDeviceToHost));
      require(std::fwrite(&n, 8, 1, f) == 1 && (n == 0 || std::fwrite(host.data(), 1, n, f) == n), BNMC_GPU_ERR_RUNTIME,
              "checkpoint write failed");
    }
  });
}

int bnmc_gpu_load_checkpoint(bnmc_gpu_ctx* c, const char* path) {
  if (!c || !path) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    BNMC_CUDA(cudaStreamSynchronize(c->stream));
    auto bufs = c->model->state_buffers();
    std::FILE* f = std::fopen(path, "rb");
    require(f != nullptr, BNMC_GPU_ERR_RUNTIME, std::string("cannot read ") + path);
    FileCloser fc{f};
    CkptHeader h{};
    require(std::fread(&h, sizeof(h), 1, f) == 1 && std::memcmp(h.magic, "BNMCCKPT", 8) == 0 && h.version == kCkptVersion,
            BNMC_GPU_ERR_RUNTIME, "not a bnmc checkpoint (or written by an older version)");
    const CkptHeader want = ckpt_header(c, static_cast<std::uint32_t>(bufs.size()));
    require(h.kind == want.kind && h.K == want.K && h.V == want.V && h.M == want.M && h.N == want.N &&
                h.rank == want.rank && h.world == want.world && h.nbufs == want.nbufs,
            BNMC_GPU_ERR_RUNTIME, "checkpoint was written by a different model / shard");
    require(h.seed == want.seed, BNMC_GPU_ERR_RUNTIME,
            "checkpoint seed differs (the RNG streams are keyed by the seed: the chain would not resume)");
    bool same_hyper = h.mh_scale == want.mh_scale;
    for (int i = 0; i < 8; ++i) same_hyper = same_hyper && h.hyper[i] == want.hyper[i];
    require(h.flags == want.flags && same_hyper, BNMC_GPU_ERR_RUNTIME,
            "checkpoint was written under a different configuration (flags, mh_scale or hyperparameters): "
            "the chain would not resume");
    std::vector<unsigned char> host;
    for (const auto& b : bufs) {
      std::uint64_t n = 0;
      require(std::fread(&n, 8, 1, f) == 1 && n == b.bytes, BNMC_GPU_ERR_RUNTIME, "checkpoint buffer size mismatch");
      host.resize(static_cast<std::size_t>(n));
      require(n == 0 || std::fread(host.data(), 1, n, f) == n, BNMC_GPU_ERR_RUNTIME, "truncated checkpoint");
      if (n) BNMC_CUDA(cudaMemcpy(*b.p, host.data(), n, cudaMemcpyHostToDevice));
    }
    c->model->on_state_restored(c->stream);
    c->next_iter = -1;
    set_iter(c, h.next_iter < 0 ? 0 : h.next_iter);
    check_device_error(c);
  });
}

int bnmc_gpu_checkpoint_iter(const bnmc_gpu_ctx* c, int64_t* next_iter) {
  if (!c || !next_iter) return fail(nullptr, BNMC_GPU_ERR_ARG, "null argument");
  *next_iter = c->next_iter;
  return BNMC_GPU_OK;
}

int bnmc_gpu_lda_load_corpus(bnmc_gpu_ctx* c, const char* path) {
  if (!c || !path) return fail(c, BNMC_GPU_ERR_ARG, "null argument");
  return guarded(c, [&] {
    c->model->lda_load_corpus(path, c->stream);
    check_device_error(c);
  });
}

int bnmc_gpu_enqueue(bnmc_gpu_ctx* c, std::int64_t iter0, std::int64_t n) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    require(iter0 >= 0 && n >= 0, BNMC_GPU_ERR_ARG, "bad iteration range");
    set_iter(c, iter0);
    for (std::int64_t i = 0; i < n; ++i) launch_sweep(c);
  });
}

int bnmc_gpu_synchronize(bnmc_gpu_ctx* c, double* last_log_joint, int* last_accepted) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    BNMC_CUDA(cudaStreamSynchronize(c->stream));
    if (c->next_iter > 0) read_ring(c, c->next_iter - 1, 1, last_log_joint, last_accepted);
    check_device_error(c);
  });
}

int bnmc_gpu_eval_log_joint(bnmc_gpu_ctx* c, double* log_joint) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    c->model->enqueue_log_joint(c->stream);
    read_ring(c, c->next_iter, 1, log_joint, nullptr);
    check_device_error(c);
  });
}

int bnmc_gpu_prior_init(bnmc_gpu_ctx* c, std::uint64_t seed) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    c->model->prior_init(seed, c->stream);
    check_device_error(c);
  });
}

int bnmc_gpu_lda_counts(bnmc_gpu_ctx* c, std::int32_t* nkw, std::int32_t* nmk) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    c->model->lda_counts(nkw, nmk, c->stream);
    check_device_error(c);
  });
}

int bnmc_gpu_lda_generate(bnmc_gpu_ctx* c, std::uint64_t seed, double phi_conc, double theta_conc) {
  if (!c) return fail(c, BNMC_GPU_ERR_ARG, "null context");
  return guarded(c, [&] {
    require(phi_conc > 0 && theta_conc > 0, BNMC_GPU_ERR_ARG, "concentrations must be positive");
    c->model->lda_generate(seed, phi_conc, theta_conc, c->stream);
    check_device_error(c);
  });
}

int bnmc_gpu_partition(const std::int64_t* off, std::int64_t M, std::int32_t world, std::int32_t rank,
                       std::int64_t* begin, std::int64_t* end) {
  if (!off || !begin || !end || M < 0 || world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, BNMC_GPU_ERR_ARG, "bad partition arguments");
  partition_docs(off, M, world, rank, begin, end);
  return BNMC_GPU_OK;
}

int bnmc_gpu_lpp(const double* phi, const double* theta, std::int64_t K, std::int64_t V,
                 const std::int64_t* w, const std::int64_t* offsets, std::int64_t docs, double* out) {
  return guarded(nullptr, [&] { *out = lpp(phi, theta, K, V, w, offsets, docs); });
}

int bnmc_gpu_dirichlet_batch(std::int64_t rows, std::int64_t cols, const double* alpha, std::uint64_t key,
                             double* out) {
  return guarded(nullptr, [&] { dirichlet_batch(rows, cols, alpha, key, out); });
}

int bnmc_gpu_probe_rng(const std::uint64_t* keys, std::int64_t n, std::int64_t per, std::uint64_t* u64,
                       double* unit, double* gauss) {
  return guarded(nullptr, [&] { probe_rng(keys, n, per, u64, unit, gauss); });
}

int bnmc_gpu_probe_gamma(const std::uint64_t* keys, const double* shapes, std::int64_t n, double* out,
                         std::uint64_t* counters) {
  return guarded(nullptr, [&] { probe_gamma(keys, shapes, n, out, counters); });
}

int bnmc_gpu_probe_read_bandwidth(int64_t bytes, int32_t reps, double* gbps) {
  if (bytes <= 0 || reps <= 0 || !gbps) return fail(nullptr, BNMC_GPU_ERR_ARG, "bad probe arguments");
  return guarded(nullptr, [&] { *gbps = probe_read_bandwidth(static_cast<std::size_t>(bytes), reps); });
}

int bnmc_gpu_probe_log_weights(const std::uint64_t* keys, const double* logw, std::int64_t rows,
                               std::int64_t cols, std::int64_t* picks) {
  return guarded(nullptr, [&] { probe_log_weights(keys, logw, rows, cols, picks); });
}

}  // extern "C"
