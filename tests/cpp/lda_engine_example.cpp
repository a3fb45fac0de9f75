// tests/cpp/lda_engine_example.cpp -- the C++ host mirror (include/bnmc_gpu.hpp) driving
// the GPU path the way a reference caller drives bnmc::Engine (sampler.hpp:45-86).
//
//   lda_engine_example <w.bin> <K> <V> <doc_len> <seed>
//
// w.bin: int64 word ids, doc-major, equal-length documents.  Prints one line per value:
// "prior <lj>", "sweep <i> <lj>" x 5, "run <i> <lj>" x 4, "map <lj>", "eval <lj>",
// "z0 <first assignment>".  tests/test_host.py compiles it; tests/test_gpu_parity.py runs
// it and compares every value with the Python engine over the same library.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "bnmc_gpu.hpp"

int main(int argc, char** argv) {
  if (argc != 6) {
    std::fprintf(stderr, "usage: %s w.bin K V doc_len seed\n", argv[0]);
    return 2;
  }
  std::ifstream f(argv[1], std::ios::binary);
  std::vector<char> raw((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  std::vector<long long> w(raw.size() / sizeof(long long));
  std::copy(raw.begin(), raw.begin() + static_cast<long>(w.size() * sizeof(long long)),
            reinterpret_cast<char*>(w.data()));
  const long long K = std::stoll(argv[2]), V = std::stoll(argv[3]), L = std::stoll(argv[4]);
  const unsigned long long seed = std::stoull(argv[5]);
  const long long M = static_cast<long long>(w.size()) / L;

  bnmc::gpu::RunConfig cfg;
  cfg.seed = seed;
  cfg.thin = 2;
  std::vector<long long> lengths(static_cast<std::size_t>(M), L);
  std::vector<int64_t> offsets;
  const bnmc_gpu_desc desc = bnmc::gpu::lda_desc(K, V, lengths, offsets, cfg);
  try {
    bnmc::gpu::Engine e(desc, cfg);
    // the reference's var order for lda.bn: phi, theta, z, w
    bnmc::gpu::ParamStore s;
    s.real = {std::vector<double>(static_cast<std::size_t>(K * V)), std::vector<double>(static_cast<std::size_t>(M * K)), {}, {}};
    s.ival = {{}, {}, std::vector<long long>(w.size()), w};
    s.observed = {0, 0, 0, 1};
    e.prior_init(s, seed);
    std::printf("prior %.17g\n", e.eval_log_joint(s));
    for (int i = 0; i < 5; ++i) std::printf("sweep %d %.17g\n", i, e.sweep(s, i));
    bnmc::gpu::Trace t = e.run(s, 4);
    for (std::size_t i = 0; i < t.log_joint.size(); ++i) std::printf("run %zu %.17g\n", i, t.log_joint[i]);
    std::printf("map %.17g\n", t.map_log_joint);
    std::printf("samples %zu\n", t.samples.size());
    std::printf("eval %.17g\n", e.eval_log_joint(s));
    std::printf("z0 %lld\n", s.ival[2][0]);
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "error: %s\n", ex.what());
    return 1;
  }
  return 0;
}
