// oracle/ref_bench.cpp -- TEST/BENCH INFRASTRUCTURE ONLY.
//
// Times the UNMODIFIED reference sampler's Engine::sweep (proj/src/sampler.cpp:390-405)
// on the reference's own synthetic generators (proj/src/gen.cpp), initialised with
// prior_init (sampler.cpp:542-555).  bench.py's `--impl reference` arm and
// `cpu_baseline` leg run this binary in a subprocess (with a timeout, because the
// reference thread pool can crash or hang at threads > 1: SURVEY.md section 5).
//
// usage: ref_bench lda  DOCS VOCAB TOPICS LEN SEED THREADS WARMUP SWEEPS
//        ref_bench lda-file CORPUS.bnc TOPICS SEED THREADS WARMUP SWEEPS DOCS
//        ref_bench gmm  N SEED THREADS WARMUP SWEEPS
//        ref_bench gmm-file X.f64 SEED THREADS WARMUP SWEEPS
//        ref_bench regression N K SEED THREADS WARMUP SWEEPS MH_SCALE
// The *-file forms run the reference on the corpus / points bench.py's GPU arm uses
// (the binary corpus format of include/bnmc_gpu.h; raw float64 points), so both arms
// of the bench see identical inputs; DOCS takes the first DOCS documents (a sample).
// prints one JSON object: {"sites": S, "ms": [...], "log_joint": [...]}
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
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

// The binary LDA corpus of bnmc_gpu_lda_load_corpus (include/bnmc_gpu.h): "BNMCCORP",
// u32 version 1, u32 0, i64 M, N, V, i64 offsets[M + 1], i32 w[N].  The first `docs`
// documents become a DataFile as gen_lda's (gen.cpp:44-58: hyper K, V, M, N; array w).
bnmc::DataFile load_corpus(const char* path, long long topics, long long docs) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string("cannot open ") + path);
  char magic[8];
  std::uint32_t ver[2];
  std::int64_t hdr[3];
  f.read(magic, 8);
  f.read(reinterpret_cast<char*>(ver), sizeof ver);
  f.read(reinterpret_cast<char*>(hdr), sizeof hdr);
  if (!f || std::memcmp(magic, "BNMCCORP", 8) != 0 || ver[0] != 1) throw std::runtime_error("not a BNMCCORP v1 corpus");
  const long long M = hdr[0], N = hdr[1], V = hdr[2];
  std::vector<std::int64_t> off(static_cast<std::size_t>(M + 1));
  std::vector<std::int32_t> w(static_cast<std::size_t>(N));
  f.read(reinterpret_cast<char*>(off.data()), static_cast<std::streamsize>(sizeof(std::int64_t) * off.size()));
  f.read(reinterpret_cast<char*>(w.data()), static_cast<std::streamsize>(sizeof(std::int32_t) * w.size()));
  if (!f) throw std::runtime_error("truncated corpus");
  if (docs <= 0 || docs > M) docs = M;
  bnmc::DataFile d;
  std::vector<long long> lengths;
  for (long long m = 0; m < docs; ++m) lengths.push_back(off[m + 1] - off[m]);
  d.hyper.set_int("K", topics);
  d.hyper.set_int("V", V);
  d.hyper.set_int("M", docs);
  d.hyper.set_array("N", std::move(lengths));
  d.int_arrays["w"] = std::vector<long long>(w.begin(), w.begin() + off[docs]);
  return d;
}

bnmc::DataFile load_points(const char* path) {
  std::ifstream f(path, std::ios::binary | std::ios::ate);
  if (!f) throw std::runtime_error(std::string("cannot open ") + path);
  const std::streamsize bytes = f.tellg();
  f.seekg(0);
  std::vector<double> x(static_cast<std::size_t>(bytes / 8));
  f.read(reinterpret_cast<char*>(x.data()), static_cast<std::streamsize>(8 * x.size()));
  bnmc::DataFile d;
  d.hyper.set_int("N", static_cast<long long>(x.size()));
  d.hyper.set_int("K", 4);
  d.real_arrays["x"] = std::move(x);
  return d;
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
    if (which == "lda-file" && argc == 9) {
      const bnmc::DataFile d = load_corpus(argv[2], std::atoll(argv[3]), std::atoll(argv[8]));
      const std::uint64_t seed = std::strtoull(argv[4], nullptr, 10);
      const auto& w = d.int_arrays.at("w");
      print(time_engine("lda", d, bnmc::Method::Gibbs, seed, std::atoi(argv[5]), std::atoll(argv[6]),
                        std::atoll(argv[7]), 0.5, static_cast<long long>(w.size())));
      return 0;
    }
    if (which == "gmm-file" && argc == 7) {
      const bnmc::DataFile d = load_points(argv[2]);
      const std::uint64_t seed = std::strtoull(argv[3], nullptr, 10);
      print(time_engine("gmm", d, bnmc::Method::Gibbs, seed, std::atoi(argv[4]), std::atoll(argv[5]),
                        std::atoll(argv[6]), 0.5, static_cast<long long>(d.real_arrays.at("x").size())));
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
