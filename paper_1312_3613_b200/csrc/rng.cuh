// csrc/rng.cuh -- device port of the reference counter RNG.
//
// Bit-exact restatement of RngStream (proj/include/bnmc/rng.hpp:12-51): splitmix64
// finalizer `mix`, `fold`, `keyed` (always five folds), `derive`, next_u64,
// next_unit ((u >> 11) + 0.5) * 2^-53 and Box-Muller next_gaussian (cos branch,
// two counters).  Integer paths are exact; next_gaussian goes through the device
// log/cos, which may differ from glibc by an ulp (parity is tolerance-based there).
#pragma once
#include <cstdint>

namespace bnmc_gpu {

constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// RNG purposes (proj/src/sampler.cpp:12-17, prior_init's kInit at :545).
enum : std::uint64_t { kProposal = 1, kAccept = 2, kDiscrete = 3, kConjugate = 4, kInit = 5 };

__host__ __device__ __forceinline__ std::uint64_t mix(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ std::uint64_t fold(std::uint64_t k, std::uint64_t v) {
  return mix(k * kGolden + v + 0x632BE59BD9B4E019ull);
}

__host__ __device__ __forceinline__ std::uint64_t keyed(std::uint64_t seed, std::uint64_t a = 0,
                                                        std::uint64_t b = 0, std::uint64_t c = 0,
                                                        std::uint64_t d = 0) {
  return fold(fold(fold(fold(fold(1, seed), a), b), c), d);
}

__host__ __device__ __forceinline__ std::uint64_t derive(std::uint64_t key, std::uint64_t a,
                                                         std::uint64_t b = 0) {
  return fold(fold(key, a), b);
}

struct Stream {
  std::uint64_t key;
  std::uint64_t counter;
  std::uint64_t pos;  // key + kGolden * counter (mod 2^64), advanced by addition

  __device__ __forceinline__ explicit Stream(std::uint64_t k) : key(k), counter(0), pos(k) {}
  // the stream after `at` draws (counter-based: no draws replayed)
  __device__ __forceinline__ Stream(std::uint64_t k, std::uint64_t at)
      : key(k), counter(at), pos(k + kGolden * at) {}

  // mix(key + kGolden * ++counter) (rng.hpp:40); the product is carried incrementally
  // (one 64-bit add instead of a 64-bit multiply per draw; identical modulo 2^64).
  __device__ __forceinline__ std::uint64_t next_u64() {
    ++counter;
    pos += kGolden;
    return mix(pos);
  }

  __device__ __forceinline__ double next_unit() {
    return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1p-53;
  }

  __device__ __forceinline__ double next_gaussian() {
    const double u1 = next_unit();
    const double u2 = next_unit();
    return sqrt(-2.0 * log(u1)) * cos(6.28318530717958647692529 * u2);
  }
};

}  // namespace bnmc_gpu
