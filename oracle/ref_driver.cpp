// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" shim over the UNMODIFIED reference sampler (`bnmc`, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the parity tests, the golden-vector generator and bench.py's reference arm
// drive the reference's own public API -- parse_model / validate_model /
// make_bindings / make_layouts / allocate_store / prior_init / Engine::sweep
// (proj/include/bnmc/sampler.hpp:45-110) -- through ctypes.
//
// Nothing here re-implements sampler arithmetic: every number comes out of the
// reference library.  The model sources (proj/models/*.bn) are embedded at build
// time by the Makefile into oracle/_ref/models_gen.cpp (git-ignored), so no
// reference source text is committed to this repository.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "bnmc/batch.hpp"
#include "bnmc/data.hpp"
#include "bnmc/dist.hpp"
#include "bnmc/gen.hpp"
#include "bnmc/metrics.hpp"
#include "bnmc/parser.hpp"
#include "bnmc/plan.hpp"
#include "bnmc/sampler.hpp"
#include "json.hpp"

extern "C" const char* bref_model_source(const char* name);  // models_gen.cpp

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
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown C++ exception";
    return 1;
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

const bnmc::RandomVar& var_of(const Handle& h, const char* name) {
  const bnmc::RandomVar* v = h.model.find_var(name);
  if (!v) throw bnmc::RuntimeError(std::string("unknown variable '") + name + "'");
  return *v;
}

}  // namespace

extern "C" {

const char* bref_last_error() { return g_err.c_str(); }

// Opens an Engine over one of the embedded models ("lda", "gmm", "regression", ...).
// hyper_json: {"K": 5, "N": [..], "l": -1.0, ...}; observe_csv: extra observed vars.
void* bref_open(const char* model_name, const char* hyper_json, const char* method,
                std::uint64_t seed, int threads, double mh_scale, const char* observe_csv) {
  std::unique_ptr<Handle> h(new Handle);
  const int rc = guarded([&] {
    const char* src = bref_model_source(model_name);
    if (!src) throw std::invalid_argument(std::string("no embedded model '") + model_name + "'");
    h->model = bnmc::validate_model(bnmc::parse_model(src), model_name);
    h->hyper = hyper_from_json(hyper_json);
    h->bind = bnmc::make_bindings(h->model, h->hyper);
    h->layouts = bnmc::make_layouts(h->model, h->bind);
    if (!bnmc::lookup_method(method, &h->cfg.method)) {
      throw std::invalid_argument(std::string("unknown method '") + method + "'");
    }
    h->cfg.seed = seed;
    h->cfg.threads = threads;
    h->cfg.mh_scale = mh_scale;
    std::stringstream ss(observe_csv ? observe_csv : "");
    std::string name;
    while (std::getline(ss, name, ',')) {
      if (!name.empty()) h->cfg.observe_extra.push_back(name);
    }
    h->store = bnmc::allocate_store(h->model, h->layouts);
    for (const auto& n : h->cfg.observe_extra) {
      h->store.observed[static_cast<std::size_t>(var_of(*h, n.c_str()).id)] = 1;
    }
    h->engine = std::make_unique<bnmc::Engine>(h->model, h->hyper, h->cfg);
  });
  return rc == 0 ? h.release() : nullptr;
}

void bref_close(void* hp) { delete static_cast<Handle*>(hp); }

// id, flat length, is_int, observed (model-level OR call-time).
int bref_var_info(void* hp, const char* name, std::int64_t* id, std::int64_t* len, int* is_int,
                  int* observed) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto& v = var_of(*h, name);
    *id = v.id;
    *len = h->layouts[static_cast<std::size_t>(v.id)].flat_values();
    *is_int = v.is_int ? 1 : 0;
    *observed = h->store.observed[static_cast<std::size_t>(v.id)];
  });
}

int bref_set_real(void* hp, const char* name, const double* p, std::int64_t n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    auto& arr = h->store.real[static_cast<std::size_t>(var_of(*h, name).id)];
    if (static_cast<std::int64_t>(arr.size()) != n) throw bnmc::RuntimeError("length mismatch");
    std::memcpy(arr.data(), p, sizeof(double) * static_cast<std::size_t>(n));
  });
}

int bref_get_real(void* hp, const char* name, double* p, std::int64_t n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto& arr = h->store.real[static_cast<std::size_t>(var_of(*h, name).id)];
    if (static_cast<std::int64_t>(arr.size()) != n) throw bnmc::RuntimeError("length mismatch");
    std::memcpy(p, arr.data(), sizeof(double) * static_cast<std::size_t>(n));
  });
}

int bref_set_int(void* hp, const char* name, const std::int64_t* p, std::int64_t n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    auto& arr = h->store.ival[static_cast<std::size_t>(var_of(*h, name).id)];
    if (static_cast<std::int64_t>(arr.size()) != n) throw bnmc::RuntimeError("length mismatch");
    for (std::int64_t i = 0; i < n; ++i) arr[static_cast<std::size_t>(i)] = p[i];
  });
}

int bref_get_int(void* hp, const char* name, std::int64_t* p, std::int64_t n) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const auto& arr = h->store.ival[static_cast<std::size_t>(var_of(*h, name).id)];
    if (static_cast<std::int64_t>(arr.size()) != n) throw bnmc::RuntimeError("length mismatch");
    for (std::int64_t i = 0; i < n; ++i) p[i] = arr[static_cast<std::size_t>(i)];
  });
}

// prior_init(skip_observed=true), the usual chain initialisation (tools/main.cpp:91-92).
int bref_prior_init(void* hp, std::uint64_t seed) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] { bnmc::prior_init(h->model, h->bind, h->layouts, h->store, seed, true); });
}

int bref_sweep(void* hp, std::int64_t iter, double* log_joint, int* accepted) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    bool acc = false;
    *log_joint = h->engine->sweep(h->store, iter, &acc);
    if (accepted) *accepted = acc ? 1 : 0;
  });
}

// n consecutive sweeps from iter0; per-sweep wall time (ms) like Trace::timing_ms.
int bref_sweeps_timed(void* hp, std::int64_t iter0, std::int64_t n, double* lj, double* ms) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    for (std::int64_t i = 0; i < n; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      lj[i] = h->engine->sweep(h->store, iter0 + i);
      const auto t1 = std::chrono::steady_clock::now();
      ms[i] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    }
  });
}

int bref_log_joint(void* hp, double* out) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] { *out = h->engine->eval_log_joint(h->store); });
}

// The `describe` report (plan, block order, strategies).
int bref_describe(void* hp, char* buf, std::int64_t cap) {
  auto* h = static_cast<Handle*>(hp);
  return guarded([&] {
    const std::string s =
        bnmc::describe_plan(h->model, h->engine->joint(), h->engine->plan());
    std::snprintf(buf, static_cast<std::size_t>(cap), "%s", s.c_str());
  });
}

// --- generators (proj/src/gen.cpp) -------------------------------------------

int bref_gen_lda(std::int64_t docs, std::int64_t vocab, std::int64_t topics, std::int64_t len,
                 std::int64_t heldout, std::uint64_t seed, std::int64_t* w, double* true_phi,
                 std::int64_t* w_heldout) {
  return guarded([&] {
    const bnmc::LdaCorpus c = bnmc::gen_lda(docs, vocab, topics, len, heldout, seed);
    const auto& tw = c.train.int_arrays.at("w");
    std::memcpy(w, tw.data(), tw.size() * sizeof(std::int64_t));
    if (true_phi) std::memcpy(true_phi, c.true_phi.data(), c.true_phi.size() * sizeof(double));
    if (w_heldout && heldout > 0) {
      const auto& hw = c.heldout.int_arrays.at("w");
      std::memcpy(w_heldout, hw.data(), hw.size() * sizeof(std::int64_t));
    }
  });
}

int bref_gen_gmm(std::int64_t n, const double* centers, const double* stds, std::int64_t k,
                 std::uint64_t seed, double* x) {
  return guarded([&] {
    const bnmc::GmmTruth t = bnmc::gen_gmm(n, std::vector<double>(centers, centers + k),
                                           std::vector<double>(stds, stds + k), seed);
    const auto& xs = t.data.real_arrays.at("x");
    std::memcpy(x, xs.data(), xs.size() * sizeof(double));
  });
}

int bref_gen_regression(std::int64_t n, std::int64_t k, double noise_var, std::uint64_t seed,
                        double* x, double* y, double* w_true, double* b_true) {
  return guarded([&] {
    const bnmc::RegressionTruth t = bnmc::gen_regression(n, k, noise_var, seed);
    const auto& xs = t.data.real_arrays.at("x");
    const auto& ys = t.data.real_arrays.at("y");
    std::memcpy(x, xs.data(), xs.size() * sizeof(double));
    std::memcpy(y, ys.data(), ys.size() * sizeof(double));
    std::memcpy(w_true, t.w.data(), t.w.size() * sizeof(double));
    *b_true = t.b;
  });
}

// --- primitive known-answer probes (rng.hpp, dist.cpp, batch.cpp, metrics.cpp) -----

std::uint64_t bref_keyed(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c,
                         std::uint64_t d) {
  return bnmc::RngStream::keyed(seed, a, b, c, d).key;
}

std::uint64_t bref_derive(std::uint64_t key, std::uint64_t a, std::uint64_t b) {
  return bnmc::RngStream{key, 0}.derive(a, b).key;
}

void bref_stream_u64(std::uint64_t key, std::int64_t n, std::uint64_t* out) {
  bnmc::RngStream r{key, 0};
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

void bref_stream_unit(std::uint64_t key, std::int64_t n, double* out) {
  bnmc::RngStream r{key, 0};
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_unit();
}

void bref_stream_gaussian(std::uint64_t key, std::int64_t n, double* out) {
  bnmc::RngStream r{key, 0};
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.next_gaussian();
}

// draw_gamma from a fresh stream; *counter_out = counters consumed.
double bref_draw_gamma(std::uint64_t key, double shape, std::uint64_t* counter_out) {
  bnmc::RngStream r{key, 0};
  double g = 0.0;
  if (guarded([&] { g = bnmc::draw_gamma(r, shape); }) != 0) return -1.0;
  if (counter_out) *counter_out = r.counter;
  return g;
}

std::int64_t bref_draw_from_log_weights(std::uint64_t key, const double* logw, std::int64_t n) {
  bnmc::RngStream r{key, 0};
  std::int64_t out = -1;
  if (guarded([&] { out = bnmc::draw_from_log_weights(r, {logw, static_cast<std::size_t>(n)}); }) !=
      0)
    return -1;
  return out;
}

int bref_dirichlet_batch(std::int64_t rows, std::int64_t cols, const double* alpha, int per_row,
                         std::uint64_t key, int threads, int strategy, double* out) {
  return guarded([&] {
    bnmc::BatchSpec spec;
    spec.rows = rows;
    spec.cols = cols;
    spec.per_row = per_row != 0;
    spec.alpha = {alpha, static_cast<std::size_t>(per_row ? rows * cols : cols)};
    spec.strategy = static_cast<bnmc::BatchStrategy>(strategy);
    bnmc::ParallelExecutor pool(threads);
    bnmc::sample_dirichlet_batch(spec, bnmc::RngStream{key, 0}, pool,
                                 {out, static_cast<std::size_t>(rows * cols)});
  });
}

double bref_log_pdf_dirichlet(const double* x, const double* alpha, std::int64_t n) {
  return bnmc::log_pdf_dirichlet({x, static_cast<std::size_t>(n)},
                                 {alpha, static_cast<std::size_t>(n)});
}

double bref_log_pdf_gaussian(double x, double mean, double var) {
  return bnmc::log_pdf_gaussian(x, mean, var);
}

// log_predictive_probability over a uniform-length held-out corpus (metrics.cpp:9-34).
int bref_lpp(const double* phi, const double* theta, std::int64_t topics, std::int64_t vocab,
             const std::int64_t* w, const std::int64_t* offsets, std::int64_t docs, double* out) {
  return guarded([&] {
    bnmc::HeldoutCorpus hc;
    for (std::int64_t d = 0; d < docs; ++d) {
      hc.docs.emplace_back(w + offsets[d], w + offsets[d + 1]);
    }
    *out = bnmc::log_predictive_probability(
        {phi, static_cast<std::size_t>(topics * vocab)},
        {theta, static_cast<std::size_t>(docs * topics)}, topics, vocab, hc);
  });
}

}  // extern "C"
