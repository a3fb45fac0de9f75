// integration/b200_driver.cpp -- TEST / BENCH SHIM over the PATCHED reference (the
// reference's own sources + reference_b200.patch + gpu_backend.cpp, built by
// integration/Makefile into _build/libbnmc_b200ref.so).
//
// It drives the reference's public API -- Engine (sampler.hpp:45-86), sample()
// (:103-104), map_estimate() (:108-110), prior_init (:97-99), lpp_curve (bench.hpp) --
// with RunConfig::device = Cpu or B200, so the GPU tests compare the reference's own code
// on the device against the same code on the CPU, and bench.py times Engine::sweep on the
// reference's pageable ParamStore.  Nothing here computes samples.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "bnmc/bench.hpp"
#include "bnmc/data.hpp"
#include "bnmc/metrics.hpp"
#include "bnmc/parser.hpp"
#include "bnmc/sampler.hpp"
#include "json.hpp"

extern "C" const char* bnmc_b200_canonical_model(const char* name);  // models_gen.cpp

namespace {

thread_local std::string g_err;

struct Handle {
  bnmc::CheckedModel model;
  bnmc::HyperValues hyper;
  bnmc::Bindings bind;
  std::vector<bnmc::VarLayout> layouts;
  bnmc::RunConfig cfg;
  std::unique_ptr<bnmc::Engine> engine;
  bnmc::ParamStore store;
  bnmc::Trace trace;
  std::vector<bnmc::LppPoint> lpp;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const bnmc::RuntimeError& e) {
    g_err = std::string("RuntimeError: ") + e.what();
    return 2;
  } catch (const std::domain_error& e) {
    g_err = std::string("domain_error: ") + e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

bnmc::HyperValues hyper_from_json(const std::string& text) {
  bnmc::HyperValues h;
  const auto j = nlohmann::json::parse(text);
  for (auto it = j.begin(); it != j.end(); ++it) {
    if (it->is_array()) {
      h.set_array(it.key(), it->get<std::vector<long long>>());
    } else if (it->is_number_integer()) {
      h.set_int(it.key(), it->get<long long>());
    } else {
      h.set_real(it.key(), it->get<double>());
    }
  }
  return h;
}

std::vector<std::string> split_csv(const char* s) {
  std::vector<std::string> out;
  std::stringstream ss(s ? s : "");
  std::string x;
  while (std::getline(ss, x, ','))
    if (!x.empty()) out.push_back(x);
  return out;
}

int var_of(const Handle& h, const char* name) {
  const bnmc::RandomVar* v = h.model.find_var(name);
  if (!v) throw bnmc::RuntimeError(std::string("unknown variable '") + name + "'");
  return v->id;
}

int trace_pos(const Handle& h, const char* name) {
  for (std::size_t i = 0; i < h.trace.var_names.size(); ++i)
    if (h.trace.var_names[i] == name) return static_cast<int>(i);
  throw bnmc::RuntimeError(std::string("trace does not carry '") + name + "'");
}

}  // namespace

extern "C" {

const char* b2r_last_error() { return g_err.c_str(); }

const char* b2r_canonical_model(const char* name) { return bnmc_b200_canonical_model(name); }

void b2r_set_default_device(int b200) { bnmc::set_default_device(b200 ? bnmc::Device::B200 : bnmc::Device::Cpu); }

// Opens an Engine over a model source (the canonical zoo model when `source` is NULL).
void* b2r_open(const char* name, const char* source, const char* hyper_json, const char* method,
               std::uint64_t seed, int threads, double mh_scale, const char* observe_csv, int b200,
               long long thin, long long burnin) {
  std::unique_ptr<Handle> h(new Handle);
  const int rc = guarded([&] {
    const char* src = source ? source : bnmc_b200_canonical_model(name);
    if (!src) throw std::invalid_argument(std::string("no model '") + name + "'");
    h->model = bnmc::validate_model(bnmc::parse_model(src), name);
    h->hyper = hyper_from_json(hyper_json);
    h->bind = bnmc::make_bindings(h->model, h->hyper);
    h->layouts = bnmc::make_layouts(h->model, h->bind);
    if (!bnmc::lookup_method(method, &h->cfg.method))
      throw std::invalid_argument(std::string("unknown method '") + method + "'");
    h->cfg.seed = seed;
    h->cfg.threads = threads;
    h->cfg.mh_scale = mh_scale;
    h->cfg.thin = thin;
    h->cfg.burnin = burnin;
    h->cfg.device = b200 ? bnmc::Device::B200 : bnmc::Device::Cpu;
    h->cfg.observe_extra = split_csv(observe_csv);
    h->store = bnmc::allocate_store(h->model, h->layouts);
    for (const auto& n : h->cfg.observe_extra) h->store.observed[static_cast<std::size_t>(var_of(*h, n.c_str()))] = 1;
    h->engine = std::make_unique<bnmc::Engine>(h->model, h->hyper, h->cfg);
  });
  return rc == 0 ? h.release() : nullptr;
}

void b2r_close(void* hp) { delete static_cast<Handle*>(hp); }

int b2r_on_device(void* hp) { return static_cast<Handle*>(hp)->engine->on_device() ? 1 : 0; }

int b2r_var_info(void* hp, const char* name, std::int64_t* id, std::int64_t* len, int* is_int, int* observed) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const int v = var_of(*h, name);
    *id = v;
    *len = h->layouts[static_cast<std::size_t>(v)].flat_values();
    *is_int = h->model.vars[static_cast<std::size_t>(v)].is_int ? 1 : 0;
    *observed = h->store.observed[static_cast<std::size_t>(v)];
  });
}

int b2r_set(void* hp, const char* name, const void* p, std::int64_t n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto v = static_cast<std::size_t>(var_of(*h, name));
    if (h->model.vars[v].is_int) {
      auto& a = h->store.ival[v];
      if (static_cast<std::int64_t>(a.size()) != n) throw bnmc::RuntimeError("length mismatch");
      std::memcpy(a.data(), p, sizeof(long long) * static_cast<std::size_t>(n));  // in place: same buffer
    } else {
      auto& a = h->store.real[v];
      if (static_cast<std::int64_t>(a.size()) != n) throw bnmc::RuntimeError("length mismatch");
      std::memcpy(a.data(), p, sizeof(double) * static_cast<std::size_t>(n));
    }
  });
}

int b2r_get(void* hp, const char* name, void* p, std::int64_t n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto v = static_cast<std::size_t>(var_of(*h, name));
    if (h->model.vars[v].is_int) {
      const auto& a = h->store.ival[v];
      if (static_cast<std::int64_t>(a.size()) != n) throw bnmc::RuntimeError("length mismatch");
      std::memcpy(p, a.data(), sizeof(long long) * static_cast<std::size_t>(n));
    } else {
      const auto& a = h->store.real[v];
      if (static_cast<std::int64_t>(a.size()) != n) throw bnmc::RuntimeError("length mismatch");
      std::memcpy(p, a.data(), sizeof(double) * static_cast<std::size_t>(n));
    }
  });
}

int b2r_prior_init(void* hp, std::uint64_t seed) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] { bnmc::prior_init(h->model, h->bind, h->layouts, h->store, seed, true); });
}

int b2r_sweep(void* hp, std::int64_t iter, double* lj, int* accepted) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    bool acc = false;
    *lj = h->engine->sweep(h->store, iter, &acc);
    if (accepted) *accepted = acc ? 1 : 0;
  });
}

// Engine::sweep n times on the reference's own (pageable) ParamStore, wall-clocked per
// call: the end-to-end cost a caller of the reference API sees.
int b2r_sweeps_timed(void* hp, std::int64_t iter0, std::int64_t n, double* lj, double* ms) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    for (std::int64_t i = 0; i < n; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      lj[i] = h->engine->sweep(h->store, iter0 + i);
      ms[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

int b2r_log_joint(void* hp, double* out) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] { *out = h->engine->eval_log_joint(h->store); });
}

int b2r_run(void* hp, long long n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] { h->trace = h->engine->run(h->store, n); });
}

// The reference's free functions: each builds its own Engine from cfg (device included).
int b2r_sample(void* hp, long long n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] { h->trace = bnmc::sample(h->model, h->hyper, h->store, n, h->cfg); });
}

int b2r_map_estimate(void* hp, long long n, const char* observe_csv) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto v = split_csv(observe_csv);
    bnmc::map_estimate(h->model, std::set<std::string>(v.begin(), v.end()), h->hyper, h->store, n, h->cfg);
  });
}

int b2r_trace_info(void* hp, std::int64_t* n_lj, std::int64_t* n_samples, double* map_lj, int* has_map) {
  auto* h = static_cast<Handle*>(hp);
  *n_lj = static_cast<std::int64_t>(h->trace.log_joint.size());
  *n_samples = static_cast<std::int64_t>(h->trace.samples.size());
  *map_lj = h->trace.map_log_joint;
  *has_map = h->trace.map_state.real.empty() && h->trace.map_state.ints.empty() ? 0 : 1;
  return 0;
}

int b2r_trace_lj(void* hp, double* lj, double* ms) {
  auto* h = static_cast<Handle*>(hp);
  for (std::size_t i = 0; i < h->trace.log_joint.size(); ++i) {
    lj[i] = h->trace.log_joint[i];
    if (ms) ms[i] = i < h->trace.timing_ms.size() ? h->trace.timing_ms[i] : 0.0;
  }
  return 0;
}

// Sample j of the last trace (j < 0: the MAP state), variable `name`, into out[n].
int b2r_trace_value(void* hp, std::int64_t j, const char* name, void* out, std::int64_t n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto k = static_cast<std::size_t>(trace_pos(*h, name));
    const bnmc::Snapshot& s = j < 0 ? h->trace.map_state : h->trace.samples.at(static_cast<std::size_t>(j));
    if (h->model.vars[static_cast<std::size_t>(var_of(*h, name))].is_int) {
      const auto& a = s.ints.at(k);
      if (static_cast<std::int64_t>(a.size()) != n) throw bnmc::RuntimeError("length mismatch");
      std::memcpy(out, a.data(), sizeof(long long) * a.size());
    } else {
      const auto& a = s.real.at(k);
      if (static_cast<std::int64_t>(a.size()) != n) throw bnmc::RuntimeError("length mismatch");
      std::memcpy(out, a.data(), sizeof(double) * a.size());
    }
  });
}

// lpp_curve (bench.cpp:30-77) over the handle's last trace: held-out documents to fit
// (w, lengths) and held-out test tokens (w, offsets).  Each checkpoint runs the
// reference's map_estimate, whose Engine follows the process default device.
int b2r_lpp_curve(void* hp, const long long* fit_w, const long long* fit_lengths, std::int64_t fit_docs,
                  const long long* test_w, const std::int64_t* test_off, std::int64_t test_docs, long long fit_sweeps,
                  std::uint64_t seed, int threads, std::int64_t* count) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    bnmc::DataFile held;
    long long K = 0, V = 0;
    for (const auto& d : h->model.hypers) {
      if (d.name == "K") K = h->bind.hyper_int[static_cast<std::size_t>(h->model.hyper_ix.at("K"))];
      if (d.name == "V") V = h->bind.hyper_int[static_cast<std::size_t>(h->model.hyper_ix.at("V"))];
    }
    std::vector<long long> lengths(fit_lengths, fit_lengths + fit_docs);
    long long ntok = 0;
    for (long long l : lengths) ntok += l;
    held.hyper.set_int("K", K);
    held.hyper.set_int("V", V);
    held.hyper.set_int("M", fit_docs);
    held.hyper.set_array("N", lengths);
    held.int_arrays["w"] = std::vector<long long>(fit_w, fit_w + ntok);
    bnmc::HeldoutCorpus docs;
    for (std::int64_t d = 0; d < test_docs; ++d) docs.docs.emplace_back(test_w + test_off[d], test_w + test_off[d + 1]);
    h->lpp = bnmc::lpp_curve(h->model, h->trace, held, docs, fit_sweeps, seed, threads);
    *count = static_cast<std::int64_t>(h->lpp.size());
  });
}

int b2r_lpp_point(void* hp, std::int64_t i, long long* samples, double* lpp, double* seconds) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto& p = h->lpp.at(static_cast<std::size_t>(i));
    *samples = p.samples;
    *lpp = p.lpp;
    *seconds = p.seconds;
  });
}

}  // extern "C"
