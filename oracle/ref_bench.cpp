// oracle/ref_bench.cpp -- TEST/BENCH INFRASTRUCTURE ONLY.
//
// Times the UNMODIFIED reference sampler's Engine::sweep (proj/src/sampler.cpp:390-405)
// on the reference's own synthetic generators (proj/src/gen.cpp), initialised with
// prior_init (sampler.cpp:542-555).  bench.py's `--impl reference` arm and
// `cpu_baseline` leg run this binary in a subprocess (with a timeout, because the
// reference thread pool can crash or hang at threads > 1: SURVEY.md section 5).
//
// usage: ref_bench lda  DOCS VOCAB TOPICS LEN SEED THREADS WARMUP SWEEPS
//        ref_bench gmm  N SEED THREADS WARMUP SWEEPS
//        ref_bench regression N K SEED THREADS WARMUP SWEEPS MH_SCALE
// prints one JSON object: {"sites": S, "ms": [...], "log_joint": [...]}
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "bnmc/data.hpp"
#include "bnmc/gen.hpp"
#include "bnmc/parser.hpp"
#include "bnmc/sampler.hpp"

extern "C" const char* bref_model_source(const char* name);

namespace {

struct Run {
  long long sites = 0;
  std::vector<double> ms, lj;
};

Run time_engine(const char* model_name, const bnmc::DataFile& data, bnmc::Method method,
                std::uint64_t seed, int threads, long long warmup, long long sweeps,
                double mh_scale, long long sites) {
  const bnmc::CheckedModel model =
      bnmc::validate_model(bnmc::parse_model(bref_model_source(model_name)), model_name);
  const bnmc::Bindings bind = bnmc::make_bindings(model, data.hyper);
  const auto layouts = bnmc::make_layouts(model, bind);
  bnmc::ParamStore store = bnmc::allocate_store(model, layouts);
  bnmc::apply_data(model, layouts, data, store);
  bnmc::prior_init(model, bind, layouts, store, seed, true);
  bnmc::RunConfig cfg;
  cfg.method = method;
  cfg.seed = seed;
  cfg.threads = threads;
  cfg.mh_scale = mh_scale;
  bnmc::Engine engine(model, data.hyper, cfg);
  Run r;
  r.sites = sites;
  for (long long it = 0; it < warmup + sweeps; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    const double lj = engine.sweep(store, it);
    const auto t1 = std::chrono::steady_clock::now();
    if (it < warmup) continue;
    r.ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    r.lj.push_back(lj);
  }
  return r;
}

void print(const Run& r) {
  std::printf("{\"sites\": %lld, \"ms\": [", r.sites);
  for (std::size_t i = 0; i < r.ms.size(); ++i) std::printf("%s%.6f", i ? ", " : "", r.ms[i]);
  std::printf("], \"log_joint\": [");
  for (std::size_t i = 0; i < r.lj.size(); ++i) std::printf("%s%.17g", i ? ", " : "", r.lj[i]);
  std::printf("]}\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_bench lda|gmm|regression ...\n");
    return 2;
  }
  const std::string which = argv[1];
  try {
    if (which == "lda" && argc == 10) {
      const long long docs = std::atoll(argv[2]), vocab = std::atoll(argv[3]),
                      topics = std::atoll(argv[4]), len = std::atoll(argv[5]);
      const std::uint64_t seed = std::strtoull(argv[6], nullptr, 10);
      const bnmc::LdaCorpus c = bnmc::gen_lda(docs, vocab, topics, len, 0, seed);
      print(time_engine("lda", c.train, bnmc::Method::Gibbs, seed, std::atoi(argv[7]),
                        std::atoll(argv[8]), std::atoll(argv[9]), 0.5, docs * len));
      return 0;
    }
    if (which == "gmm" && argc == 7) {
      const long long n = std::atoll(argv[2]);
      const std::uint64_t seed = std::strtoull(argv[3], nullptr, 10);
      const bnmc::GmmTruth t = bnmc::gen_gmm(n, {-5.0, -1.0, 1.0, 5.0}, {1.0, 0.1, 2.0, 1.0}, seed);
      print(time_engine("gmm", t.data, bnmc::Method::Gibbs, seed, std::atoi(argv[4]),
                        std::atoll(argv[5]), std::atoll(argv[6]), 0.5, n));
      return 0;
    }
    if (which == "regression" && argc == 9) {
      const long long n = std::atoll(argv[2]), k = std::atoll(argv[3]);
      const std::uint64_t seed = std::strtoull(argv[4], nullptr, 10);
      const bnmc::RegressionTruth t = bnmc::gen_regression(n, k, 0.1, seed);
      print(time_engine("regression", t.data, bnmc::Method::MH, seed, std::atoi(argv[5]),
                        std::atoll(argv[6]), std::atoll(argv[7]), std::atof(argv[8]), n));
      return 0;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_bench: %s\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "ref_bench: bad arguments\n");
  return 2;
}
