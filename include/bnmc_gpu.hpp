// include/bnmc_gpu.hpp -- header-only C++ host mirror of the reference sampler API
// (proj/include/bnmc/sampler.hpp, store.hpp) over the C-ABI in bnmc_gpu.h.
//
// Same names, argument meaning and error behaviour as the reference for the
// plans the GPU path serves (LDA and GMM Gibbs, regression / logistic MH):
//
//   bnmc::gpu::RunConfig       ~ bnmc::RunConfig        sampler.hpp:14-22
//   bnmc::gpu::ParamStore      ~ bnmc::ParamStore       store.hpp:74-83
//   bnmc::gpu::Engine          ~ bnmc::Engine           sampler.hpp:45-86
//       sweep(store, iter, mh_accepted)                 sampler.hpp:60
//       run(store, n) -> Trace                          sampler.hpp:63
//       eval_log_joint(store)                           sampler.hpp:56
//   bnmc::gpu::RuntimeError    ~ bnmc::RuntimeError     store.hpp:14-16
//   std::domain_error / std::invalid_argument as in dist.cpp / batch.cpp
//
// Link with -lbnmc_gpu (paper_1312_3613_b200/libbnmc_gpu.so).
#pragma once

#include <chrono>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bnmc_gpu.h"

namespace bnmc::gpu {

struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc, const bnmc_gpu_ctx* ctx = nullptr) {
  if (rc == BNMC_GPU_OK) return;
  const std::string msg = bnmc_gpu_last_error(ctx);
  switch (rc) {
    case BNMC_GPU_ERR_ARG: throw std::invalid_argument(msg);
    case BNMC_GPU_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw RuntimeError(msg);
  }
}

struct RunConfig {
  std::uint64_t seed = 0;
  long long thin = 1;
  long long burnin = 0;
  double mh_scale = 0.5;
  std::vector<std::string> observe_extra;  // "phi" clamps LDA's phi (lpp protocol)
  bool exact_weights = false;              // LDA: reference log-space weights
  int device = -1;
};

// Flat arrays per variable id, declaration order (the reference's var ids).
struct ParamStore {
  std::vector<std::vector<double>> real;
  std::vector<std::vector<long long>> ival;
  std::vector<char> observed;

  bnmc_gpu_store view() {
    ptr_real.assign(real.size(), nullptr);
    ptr_int.assign(ival.size(), nullptr);
    lens.assign(real.size(), 0);
    for (std::size_t i = 0; i < real.size(); ++i) {
      if (!real[i].empty()) {
        ptr_real[i] = real[i].data();
        lens[i] = static_cast<int64_t>(real[i].size());
      }
      if (!ival[i].empty()) {
        ptr_int[i] = reinterpret_cast<int64_t*>(ival[i].data());
        lens[i] = static_cast<int64_t>(ival[i].size());
      }
    }
    return bnmc_gpu_store{static_cast<int32_t>(real.size()), ptr_real.data(), ptr_int.data(), lens.data(),
                          observed.data()};
  }

 private:
  std::vector<double*> ptr_real;
  std::vector<int64_t*> ptr_int;
  std::vector<int64_t> lens;
};

struct Snapshot {
  std::vector<std::vector<double>> real;
  std::vector<std::vector<long long>> ints;
};

struct Trace {
  std::uint64_t seed = 0;
  std::vector<Snapshot> samples;
  std::vector<double> log_joint;
  Snapshot map_state;
  double map_log_joint = 0.0;
  std::vector<double> timing_ms;
};

// LDA (proj/models/lda.bn): vars phi=0, theta=1, z=2, w=3.
inline bnmc_gpu_desc lda_desc(long long K, long long V, const std::vector<long long>& doc_lengths,
                              std::vector<int64_t>& offsets_out, const RunConfig& cfg) {
  bnmc_gpu_desc d{};
  d.abi_version = BNMC_GPU_ABI_VERSION;
  d.kind = BNMC_GPU_LDA;
  d.seed = cfg.seed;
  d.device = cfg.device;
  for (const auto& o : cfg.observe_extra)
    if (o == "phi") d.flags |= BNMC_GPU_OBSERVE_PHI;
  if (cfg.exact_weights) d.flags |= BNMC_GPU_EXACT_WEIGHTS;
  offsets_out.assign(doc_lengths.size() + 1, 0);
  for (std::size_t i = 0; i < doc_lengths.size(); ++i) offsets_out[i + 1] = offsets_out[i] + doc_lengths[i];
  d.K = K;
  d.V = V;
  d.M = static_cast<int64_t>(doc_lengths.size());
  d.N = offsets_out.back();
  d.doc_offsets = offsets_out.data();
  d.hyper[0] = 0.1;  // alpha = vector(K, 0.1)
  d.hyper[1] = 0.1;  // beta  = vector(V, 0.1)
  for (int i = 0; i < 4; ++i) d.var_ids[i] = i;
  d.mh_scale = cfg.mh_scale;
  d.world_size = 1;
  return d;
}

class Engine {
 public:
  Engine(const bnmc_gpu_desc& desc, const RunConfig& cfg) : cfg_(cfg) {
    bnmc_gpu_ctx* c = nullptr;
    check(bnmc_gpu_create(&desc, &c));
    ctx_.reset(c);
  }

  // Engine::sweep: the store is advanced in place; returns the post-sweep log-joint.
  double sweep(ParamStore& store, long long iter, bool* mh_accepted = nullptr) {
    double lj = 0.0;
    int acc = 0;
    if (bound_ != &store) {
      bind(store);
      check(bnmc_gpu_sweep(ctx_.get(), iter, &lj, &acc), ctx_.get());
      download(store);
    } else {
      // upload what the sweep reads, sweep, write back in one call (bnmc_gpu_sweep_store)
      bnmc_gpu_store v = store.view();
      check(bnmc_gpu_sweep_store(ctx_.get(), &v, iter, &lj, &acc), ctx_.get());
    }
    if (mh_accepted) *mh_accepted = acc != 0;
    return lj;
  }

  // prior_init(skip_observed = true) on the device, written back into the store
  // (sampler.hpp:97-99).
  void prior_init(ParamStore& store, std::uint64_t seed) {
    bind(store);
    check(bnmc_gpu_prior_init(ctx_.get(), seed), ctx_.get());
    download(store);
  }

  double eval_log_joint(ParamStore& store) {
    bind(store);
    double lj = 0.0;
    check(bnmc_gpu_eval_log_joint(ctx_.get(), &lj), ctx_.get());
    return lj;
  }

  // Engine::run: burn-in + n kept sweeps through bnmc_gpu_run_trace -- the MAP state
  // is tracked on the device, thinned samples are downloaded into copies of the store.
  Trace run(ParamStore& store, long long n) {
    bind(store);
    Trace t;
    t.seed = cfg_.seed;
    const long long thin = cfg_.thin > 0 ? cfg_.thin : 1;
    const long long ns = n > 0 ? (n + thin - 1) / thin : 0;
    std::vector<ParamStore> samples(static_cast<std::size_t>(ns), store);
    ParamStore map_store = store;
    std::vector<bnmc_gpu_store> views;
    views.reserve(samples.size());
    for (auto& s : samples) views.push_back(s.view());
    bnmc_gpu_store mv = map_store.view();
    t.log_joint.assign(static_cast<std::size_t>(n > 0 ? n : 0), 0.0);
    t.timing_ms.assign(t.log_joint.size(), 0.0);
    bnmc_gpu_trace tr{};
    tr.burnin = cfg_.burnin;
    tr.n = n;
    tr.thin = thin;
    tr.log_joints = t.log_joint.data();
    tr.timing_ms = t.timing_ms.data();
    tr.samples = views.empty() ? nullptr : views.data();
    tr.map_state = &mv;
    tr.map_log_joint = &t.map_log_joint;
    check(bnmc_gpu_run_trace(ctx_.get(), 0, &tr), ctx_.get());
    for (auto& s : samples) t.samples.push_back(Snapshot{s.real, s.ival});
    if (n > 0) t.map_state = Snapshot{map_store.real, map_store.ival};
    download(store);
    return t;
  }

  bnmc_gpu_ctx* handle() { return ctx_.get(); }

 private:
  void bind(ParamStore& store, bool sweep_inputs = false) {
    bnmc_gpu_store v = store.view();
    if (bound_ != &store) {
      check(bnmc_gpu_upload(ctx_.get(), &v), ctx_.get());
      bound_ = &store;
    } else if (sweep_inputs) {
      check(bnmc_gpu_upload_sweep_inputs(ctx_.get(), &v), ctx_.get());
    } else {
      check(bnmc_gpu_upload_state(ctx_.get(), &v), ctx_.get());
    }
  }
  void download(ParamStore& store) {
    bnmc_gpu_store v = store.view();
    check(bnmc_gpu_download(ctx_.get(), &v), ctx_.get());
  }

  struct Del {
    void operator()(bnmc_gpu_ctx* c) const { bnmc_gpu_destroy(c); }
  };
  RunConfig cfg_;
  std::unique_ptr<bnmc_gpu_ctx, Del> ctx_;
  ParamStore* bound_ = nullptr;
};

}  // namespace bnmc::gpu
