// integration/gpu_backend.cpp -- see gpu_backend.hpp.  Built into the patched reference
// by integration/Makefile; links against paper_1312_3613_b200/libbnmc_gpu.so.
#include "gpu_backend.hpp"

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>
#include <stdexcept>

#include "bnmc/density.hpp"
#include "bnmc/dist.hpp"
#include "bnmc/expr.hpp"
#include "bnmc/parser.hpp"
#include "bnmc/plan.hpp"
#include "bnmc/rewrite.hpp"

// The canonical zoo sources (proj/models/*.bn), embedded into the build by the Makefile
// (generated into the git-ignored build directory; no model text is committed).
extern "C" const char* bnmc_b200_canonical_model(const char* name);

namespace bnmc {

// --- Device selection (RunConfig::device default) ------------------------------------------
namespace {
std::atomic<int> g_device{-1};  // -1: not decided yet (read BNMC_DEVICE once)
}

bool lookup_device(std::string_view name, Device* out) {
  if (name == "cpu") {
    *out = Device::Cpu;
    return true;
  }
  if (name == "b200" || name == "gpu" || name == "cuda") {
    *out = Device::B200;
    return true;
  }
  return false;
}

Device default_device() {
  int d = g_device.load();
  if (d < 0) {
    Device dev = Device::Cpu;
    if (const char* e = std::getenv("BNMC_DEVICE")) {
      if (!lookup_device(e, &dev)) throw RuntimeError(std::string("BNMC_DEVICE: unknown device '") + e + "'");
    }
    d = static_cast<int>(dev);
    g_device.store(d);
  }
  return static_cast<Device>(d);
}

void set_default_device(Device d) { g_device.store(static_cast<int>(d)); }

// --- Which device kernel serves this plan ---------------------------------------------------
namespace {

std::string R(const ExprPtr& e) { return e ? render(e) : std::string("-"); }

// A structural rendering of a checked model and its plan: every hyperparameter,
// deterministic declaration, variable (plates, clauses, distribution families and their
// parameter expressions, literal constants included) and plan block.  Two models with
// equal fingerprints are the same model up to hyperparameter VALUES (sizes, l, u), so the
// device kernel written for the canonical zoo model computes exactly the reference plan.
std::string fingerprint(const CheckedModel& m, const SamplerPlan& p, const std::vector<char>& observed) {
  std::ostringstream os;
  for (const auto& h : m.hypers) os << "hyper " << h.name << ' ' << static_cast<int>(h.type) << '\n';
  for (const auto& d : m.dets)
    os << "det " << d.name << ' ' << d.is_vector << ' ' << R(d.len) << ' ' << R(d.fill) << ' ' << R(d.value) << '\n';
  for (const auto& v : m.vars) {
    os << "var " << v.name << ' ' << v.is_int << ' ' << v.vector_elem << ' ' << v.observed_in_model << ' '
       << R(v.elem_dim) << " obs=" << int(observed[static_cast<std::size_t>(v.id)]) << '\n';
    for (const auto& pl : v.plates) os << "  plate " << pl.index << ' ' << R(pl.count) << '\n';
    for (const auto& c : v.clauses) {
      os << "  clause " << (c.guard_value ? R(*c.guard_value) : std::string("none")) << ' ' << c.guard_negated << ' '
         << family_name(c.dist.family) << ' ' << R(c.dist.dim);
      if (c.dist.vec)
        os << " vec " << static_cast<int>(c.dist.vec->kind) << ' ' << c.dist.vec->name << ' ' << R(c.dist.vec->row);
      for (const auto& s : c.dist.scalars) os << " s " << R(s);
      os << '\n';
    }
  }
  os << "method " << method_name(p.method) << '\n';
  for (const auto& b : p.blocks) {
    os << "block " << static_cast<int>(b.strategy) << ' ' << b.parallelizable << ' ' << b.one_at_a_time;
    for (int v : b.vars) os << ' ' << v;
    if (b.conj) os << " conj " << posterior_kind_name(b.conj->kind);
    os << '\n';
  }
  return os.str();
}

struct ZooEntry {
  const char* name;
  int kind;
  const char* methods;  // plans the device kernels implement
  unsigned flags = 0;   // extra bnmc_gpu_flag bits of the model
};
constexpr ZooEntry kZoo[] = {
    {"lda", BNMC_GPU_LDA, "gibbs"},
    {"gmm", BNMC_GPU_GMM, "gibbs"},
    {"regression", BNMC_GPU_MH_LINREG, "mh gibbs mwg"},
    {"catmix", BNMC_GPU_CATMIX, "gibbs"},
    {"naivebayes", BNMC_GPU_NAIVEBAYES, "gibbs"},
    {"hmm", BNMC_GPU_HMM, "gibbs"},
    {"polyreg", BNMC_GPU_MH_POLYREG, "mh gibbs mwg"},
    // regression with a Gamma noise precision (oracle/models/regprec.bn): the GammaPrecision kind
    {"regprec", BNMC_GPU_MH_LINREG, "mh gibbs mwg", BNMC_GPU_TAU_PRECISION},
};

int var_id(const CheckedModel& m, const char* name) {
  const RandomVar* v = m.find_var(name);
  if (!v) throw RuntimeError(std::string("B200 backend: model has no variable '") + name + "'");
  return v->id;
}

double det_fill(const CheckedModel& m, const Bindings& b, const char* name) {
  const auto it = m.det_ix.find(name);
  if (it == m.det_ix.end()) throw RuntimeError(std::string("B200 backend: model has no declaration '") + name + "'");
  const auto& v = b.det_vec[static_cast<std::size_t>(it->second)];
  if (v.empty()) throw RuntimeError(std::string("B200 backend: empty vector '") + name + "'");
  for (double x : v)
    if (x != v[0]) throw RuntimeError(std::string("B200 backend: '") + name + "' must be a constant vector");
  return v[0];
}

double hyper_real(const CheckedModel& m, const Bindings& b, const char* name) {
  const auto it = m.hyper_ix.find(name);
  if (it == m.hyper_ix.end()) throw RuntimeError(std::string("B200 backend: missing hyperparameter '") + name + "'");
  return b.hyper_real[static_cast<std::size_t>(it->second)];
}

}  // namespace

// --- GpuBackend ---------------------------------------------------------------------------
std::shared_ptr<GpuBackend> GpuBackend::create(const CheckedModel& model, const Bindings& bind,
                                               const std::vector<VarLayout>& L, const SamplerPlan& plan,
                                               const std::vector<char>& observed, const RunConfig& cfg) {
  const std::string want = fingerprint(model, plan, observed);
  const ZooEntry* hit = nullptr;
  for (const auto& z : kZoo) {
    const char* src = bnmc_b200_canonical_model(z.name);
    if (!src) continue;
    const CheckedModel cm = validate_model(parse_model(src), z.name);
    if (cm.vars.size() != model.vars.size()) continue;
    std::vector<char> obs(cm.vars.size(), 0);
    bool names_match = true;
    for (const auto& v : cm.vars) {
      const RandomVar* u = model.find_var(v.name);
      if (!u || u->id != v.id) {
        names_match = false;
        break;
      }
      obs[static_cast<std::size_t>(v.id)] = observed[static_cast<std::size_t>(u->id)];
    }
    if (!names_match) continue;
    const JointDensity j = lower(cm);
    const SamplerPlan cp = plan_inference(cm, j, cfg.method, obs, PlanConfig{cfg.mh_scale});
    if (fingerprint(cm, cp, obs) == want) {
      hit = &z;
      break;
    }
  }
  if (!hit)
    throw RuntimeError("B200 backend: no device kernels for model '" + model.name + "' under method " +
                       method_name(cfg.method) + " (the device serves the zoo models lda, gmm, regression, "
                       "catmix, naivebayes, hmm and polyreg as written)");
  const std::string mname = method_name(cfg.method);
  if (std::string(" ") .append(hit->methods).append(" ").find(" " + mname + " ") == std::string::npos)
    throw RuntimeError(std::string("B200 backend: model '") + hit->name + "' runs method " + hit->methods +
                       " on the device, not " + mname);
  // Clamped variables beyond the model's observe(): only LDA's phi (the lpp protocol).
  for (const auto& v : model.vars) {
    const bool extra = observed[static_cast<std::size_t>(v.id)] && !v.observed_in_model;
    if (extra && !(hit->kind == BNMC_GPU_LDA && v.name == "phi"))
      throw RuntimeError("B200 backend: observing '" + v.name + "' is not supported on the device for '" +
                         hit->name + "'");
  }

  bnmc_gpu_desc d{};
  d.abi_version = BNMC_GPU_ABI_VERSION;
  d.kind = hit->kind;
  d.seed = cfg.seed;
  d.device = -1;
  d.mh_scale = cfg.mh_scale;
  d.world_size = 1;
  if (const char* e = std::getenv("BNMC_B200_EXACT_WEIGHTS"); e && std::string(e) == "1")
    d.flags |= BNMC_GPU_EXACT_WEIGHTS;  // LDA: the reference's log-space arithmetic
  if (cfg.method == Method::Gibbs && (hit->kind == BNMC_GPU_MH_LINREG || hit->kind == BNMC_GPU_MH_POLYREG))
    d.flags |= BNMC_GPU_GIBBS;
  if (cfg.method == Method::MWG) d.flags |= BNMC_GPU_MWG;
  d.flags |= hit->flags;
  for (std::size_t i = 0; i < model.vars.size() && i < 8; ++i) d.var_ids[i] = static_cast<int32_t>(i);
  std::vector<int64_t> offsets;
  auto lay = [&](const char* n) -> const VarLayout& { return L[static_cast<std::size_t>(var_id(model, n))]; };
  switch (hit->kind) {
    case BNMC_GPU_LDA: {
      const VarLayout& zl = lay("z");
      d.K = lay("phi").total;
      d.V = lay("phi").width;
      d.M = lay("theta").total;
      d.N = zl.total;
      offsets.resize(static_cast<std::size_t>(d.M) + 1);
      for (long long i = 0; i <= d.M; ++i)
        offsets[static_cast<std::size_t>(i)] = zl.uniform1 >= 0 ? i * zl.uniform1 : zl.offsets[static_cast<std::size_t>(i)];
      d.doc_offsets = offsets.data();
      d.hyper[0] = det_fill(model, bind, "alpha");
      d.hyper[1] = det_fill(model, bind, "beta");
      if (observed[static_cast<std::size_t>(var_id(model, "phi"))]) d.flags |= BNMC_GPU_OBSERVE_PHI;
      break;
    }
    case BNMC_GPU_GMM:  // gmm.bn: alpha = vector(K, 0.1), mu ~ Gaussian(0, 10), sigma2 ~ InvGamma(1, 1)
      d.K = lay("mu").total;
      d.N = lay("z").total;
      d.hyper[0] = det_fill(model, bind, "alpha");
      d.hyper[1] = 0.0;
      d.hyper[2] = 10.0;
      d.hyper[3] = 1.0;
      d.hyper[4] = 1.0;
      break;
    case BNMC_GPU_MH_LINREG:  // regression.bn: w, b ~ Gaussian(0, 10), tau ~ InvGamma(3, 1), x ~ U(l, u)
                              // (regprec.bn: tau ~ Gamma(3, 1), a precision)
      d.K = lay("w").total;
      d.N = lay("y").total;
      d.hyper[0] = hyper_real(model, bind, "l");
      d.hyper[1] = hyper_real(model, bind, "u");
      d.hyper[2] = 10.0;
      d.hyper[3] = 10.0;
      d.hyper[4] = 3.0;
      d.hyper[5] = 1.0;
      break;
    case BNMC_GPU_CATMIX:
      d.K = lay("theta").total;
      d.V = lay("theta").width;
      d.N = lay("z").total;
      d.hyper[0] = det_fill(model, bind, "alpha");
      d.hyper[1] = det_fill(model, bind, "beta");
      break;
    case BNMC_GPU_NAIVEBAYES:
      d.K = lay("pF").total / 2;
      d.N = lay("c").total;
      break;
    case BNMC_GPU_HMM:
      d.K = lay("bias").total;
      d.N = lay("s").total;
      d.hyper[0] = det_fill(model, bind, "v");
      break;
    case BNMC_GPU_MH_POLYREG:  // polyreg.bn: w, bias ~ Gaussian(0, 1), x ~ U(0, 2), noise 1
      d.K = lay("w").total;
      d.N = lay("y").total;
      d.hyper[0] = 0.0;
      d.hyper[1] = 2.0;
      d.hyper[2] = 1.0;
      d.hyper[3] = 1.0;
      break;
    default: throw RuntimeError("B200 backend: unhandled kind");
  }
  std::shared_ptr<GpuBackend> g(new GpuBackend);
  g->kind_ = hit->kind;
  g->burnin_ = cfg.burnin;
  g->thin_ = cfg.thin > 0 ? cfg.thin : 1;
  g->observed_ = observed;
  g->check(bnmc_gpu_create(&d, &g->ctx_));
  return g;
}

GpuBackend::~GpuBackend() {
  if (ctx_) bnmc_gpu_destroy(ctx_);  // also releases the page-locked store ranges
}

void GpuBackend::check(int rc) const {  // C-ABI status -> the reference's exception types
  if (rc == BNMC_GPU_OK) return;
  const std::string msg = bnmc_gpu_last_error(ctx_);
  if (rc == BNMC_GPU_ERR_DOMAIN) throw std::domain_error(msg);
  if (rc == BNMC_GPU_ERR_ARG) throw std::invalid_argument(msg);
  throw RuntimeError("B200 backend: " + msg);
}

// ParamStore (store.hpp:74-83) -> bnmc_gpu_store: the same flat arrays, by variable id.
// Observed = the Engine's mask OR the store's (observed arrays are never written).
void GpuBackend::make_view(const ParamStore& s, View& v) const {
  const std::size_t n = observed_.size();
  if (s.real.size() != n || s.ival.size() != n || s.observed.size() != n)
    throw RuntimeError("B200 backend: store does not match the model's variables");
  v.real.assign(n, nullptr);
  v.ival.assign(n, nullptr);
  v.len.assign(n, 0);
  v.obs.assign(n, 0);
  for (std::size_t i = 0; i < n; ++i) {
    auto& re = const_cast<std::vector<double>&>(s.real[i]);
    auto& iv = const_cast<std::vector<long long>&>(s.ival[i]);
    if (!re.empty()) {
      v.real[i] = re.data();
      v.len[i] = static_cast<int64_t>(re.size());
    }
    if (!iv.empty()) {
      v.ival[i] = reinterpret_cast<int64_t*>(iv.data());
      v.len[i] = static_cast<int64_t>(iv.size());
    }
    v.obs[i] = static_cast<char>(observed_[i] || s.observed[i]);
  }
  v.seal();
}

// The store is borrowed per call (sampler.hpp:43-44).  A new store is bound: its arrays are
// page-locked once (the reference's ParamStore is pageable std::vector memory) and the
// observed data crosses PCIe; later calls on the same store move only the latent state.
void GpuBackend::bind(const ParamStore& s, bool latent_only) {
  make_view(s, view_);
  check(bnmc_gpu_register_host(ctx_, &view_.store));
  if (bound_ == &s && latent_only) {
    check(bnmc_gpu_upload_state(ctx_, &view_.store));
  } else {
    check(bnmc_gpu_upload(ctx_, &view_.store));
    bound_ = &s;
  }
}

double GpuBackend::sweep(ParamStore& store, long long iter, bool* mh_accepted) {
  double lj = 0.0;
  int acc = 0;
  if (bound_ != &store) {
    bind(store, false);
    check(bnmc_gpu_sweep(ctx_, iter, &lj, &acc));
    check(bnmc_gpu_download(ctx_, &view_.store));
  } else {
    // the fast path: upload what the sweep reads, sweep, write back in one call (LDA: the
    // z upload overlaps a sweep started from the z written back last time, verified)
    make_view(store, view_);
    check(bnmc_gpu_register_host(ctx_, &view_.store));  // no-op unless an array moved
    check(bnmc_gpu_sweep_store(ctx_, &view_.store, iter, &lj, &acc));
  }
  if (mh_accepted) *mh_accepted = acc != 0;
  return lj;
}

double GpuBackend::eval_log_joint(const ParamStore& store) {
  bind(store, true);  // the store's current state, as the reference evaluates it
  double lj = 0.0;
  check(bnmc_gpu_eval_log_joint(ctx_, &lj));
  return lj;
}

// Engine::run through bnmc_gpu_run_trace: the device keeps the MAP state and writes each
// thinned sample into a host snapshot while the next sweeps run.  timing_ms holds the
// device time of each kept sweep (the reference's wall clock per sweep() call).
void GpuBackend::run(ParamStore& store, long long n, Trace& trace) {
  bind(store, true);
  const long long ns = n > 0 ? (n + thin_ - 1) / thin_ : 0;
  struct Snap {
    std::vector<std::vector<double>> real;
    std::vector<std::vector<long long>> ints;
    View view;
  };
  // Each snapshot owns arrays for the unobserved variables; its view shares the store's
  // observed arrays (read-only: never written).
  auto make_snap = [&](Snap& sn) {
    sn.real.resize(trace.var_ids.size());
    sn.ints.resize(trace.var_ids.size());
    sn.view = view_;
    for (std::size_t k = 0; k < trace.var_ids.size(); ++k) {
      const auto i = static_cast<std::size_t>(trace.var_ids[k]);
      if (!store.ival[i].empty()) {
        sn.ints[k].resize(store.ival[i].size());
        sn.view.ival[i] = reinterpret_cast<int64_t*>(sn.ints[k].data());
      } else {
        sn.real[k].resize(store.real[i].size());
        sn.view.real[i] = sn.real[k].data();
      }
    }
    sn.view.seal();
  };
  std::vector<Snap> samples(static_cast<std::size_t>(ns));
  for (auto& sn : samples) make_snap(sn);
  Snap map;
  make_snap(map);
  std::vector<bnmc_gpu_store> views;
  for (auto& sn : samples) views.push_back(sn.view.store);
  std::vector<double> lj(static_cast<std::size_t>(n > 0 ? n : 0)), ms(lj.size());
  double map_lj = -std::numeric_limits<double>::infinity();
  bnmc_gpu_trace tr{};
  tr.burnin = burnin_;
  tr.n = n > 0 ? n : 0;
  tr.thin = thin_;
  tr.log_joints = lj.data();
  tr.timing_ms = ms.data();
  tr.samples = views.empty() ? nullptr : views.data();
  tr.map_state = &map.view.store;
  tr.map_log_joint = &map_lj;
  check(bnmc_gpu_run_trace(ctx_, 0, &tr));
  trace.log_joint = lj;
  trace.timing_ms = ms;
  for (auto& sn : samples) trace.samples.push_back(Snapshot{std::move(sn.real), std::move(sn.ints)});
  trace.map_log_joint = map_lj;
  if (map_lj > -std::numeric_limits<double>::infinity())
    trace.map_state = Snapshot{std::move(map.real), std::move(map.ints)};
  check(bnmc_gpu_download(ctx_, &view_.store));  // the store ends at the last sweep's state
}

}  // namespace bnmc
