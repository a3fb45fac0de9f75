// integration/gpu_backend.hpp -- the B200 backend of the reference's bnmc::Engine.
//
// Compiled INTO the reference (integration/Makefile copies /root/reference/proj, applies
// reference_b200.patch and builds it with this file).  The patch gives RunConfig a
// `device` field and Engine a `gpu_` member; when cfg.device == Device::B200 the Engine
// constructor (sampler.cpp:34-42) creates a GpuBackend, and Engine::sweep
// (sampler.cpp:390-405), Engine::eval_log_joint (:44-46) and Engine::run (:426-455)
// forward to it.  Everything above Engine -- sample(), map_estimate(), lpp_curve(), the
// bench protocols, the CLI -- is the reference's own code, unchanged.
//
// The backend maps the reference's types onto the C-ABI of libbnmc_gpu.so
// (include/bnmc_gpu.h): the plan onto a model kind, Bindings/VarLayouts onto
// bnmc_gpu_desc, a ParamStore onto a bnmc_gpu_store view.  Plans it has no kernels for
// throw bnmc::RuntimeError -- there is no silent CPU fallback.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "bnmc/sampler.hpp"
#include "bnmc_gpu.h"

namespace bnmc {

class GpuBackend {
 public:
  static std::shared_ptr<GpuBackend> create(const CheckedModel& model, const Bindings& bind,
                                            const std::vector<VarLayout>& layouts, const SamplerPlan& plan,
                                            const std::vector<char>& observed, const RunConfig& cfg);
  ~GpuBackend();
  GpuBackend(const GpuBackend&) = delete;
  GpuBackend& operator=(const GpuBackend&) = delete;

  // Engine::sweep: the store is advanced in place; returns the post-sweep log-joint.
  double sweep(ParamStore& store, long long iter, bool* mh_accepted);
  // Engine::eval_log_joint of the store's current state.
  double eval_log_joint(const ParamStore& store);
  // Engine::run: burn-in + n kept sweeps with a device-resident trace (MAP state tracked
  // on the device, thinned samples downloaded as they are taken); `trace` arrives with
  // its header (model, method, seed, var ids / names) filled by Engine::run.
  void run(ParamStore& store, long long n, Trace& trace);

  bnmc_gpu_ctx* handle() const { return ctx_; }
  int kind() const { return kind_; }

 private:
  GpuBackend() = default;
  struct View {
    std::vector<double*> real;
    std::vector<int64_t*> ival;
    std::vector<int64_t> len;
    std::vector<char> obs;
    bnmc_gpu_store store{};
    void seal() {
      store = bnmc_gpu_store{static_cast<int32_t>(len.size()), real.data(), ival.data(), len.data(), obs.data()};
    }
  };
  void make_view(const ParamStore& s, View& v) const;
  void bind(const ParamStore& s, bool latent_only);
  void check(int rc) const;

  bnmc_gpu_ctx* ctx_ = nullptr;
  int kind_ = 0;
  long long burnin_ = 0, thin_ = 1;
  std::vector<char> observed_;  // the Engine's mask (model observe() + observe_extra)
  const ParamStore* bound_ = nullptr;
  View view_;
};

}  // namespace bnmc
