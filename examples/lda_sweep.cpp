// examples/lda_sweep.cpp -- the reference's Engine API shape, on the GPU path.
//
//   g++ -std=c++17 -Iinclude examples/lda_sweep.cpp -Lpaper_1312_3613_b200 -lbnmc_gpu
//       -Wl,-rpath,$PWD/paper_1312_3613_b200 -o lda_sweep && ./lda_sweep
//
// Builds a small LDA store (var ids phi=0, theta=1, z=2, w=3 as lda.bn declares),
// initialises it with the device prior_init and runs Engine::sweep 5 times.
#include <cstdio>
#include <random>

#include "bnmc_gpu.hpp"

int main() {
  using namespace bnmc::gpu;
  const long long K = 8, V = 200, M = 50, L = 40;
  RunConfig cfg;
  cfg.seed = 7;
  std::vector<long long> lengths(M, L);
  std::vector<int64_t> offsets;
  const bnmc_gpu_desc desc = lda_desc(K, V, lengths, offsets, cfg);
  ParamStore store;
  store.real = {std::vector<double>(K * V), std::vector<double>(M * K), {}, {}};
  store.ival = {{}, {}, std::vector<long long>(M * L), std::vector<long long>(M * L)};
  store.observed = {0, 0, 0, 1};
  std::mt19937_64 rng(1);
  for (auto& w : store.ival[3]) w = static_cast<long long>(rng() % V);
  try {
    Engine engine(desc, cfg);
    engine.prior_init(store, cfg.seed);
    for (long long it = 0; it < 5; ++it) {
      const double lj = engine.sweep(store, it);
      std::printf("sweep %lld  log-joint %.6f  z[0..3] = %lld %lld %lld %lld\n", it, lj, store.ival[2][0],
                  store.ival[2][1], store.ival[2][2], store.ival[2][3]);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
