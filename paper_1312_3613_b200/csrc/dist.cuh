// csrc/dist.cuh -- device draws and log-densities used by the sweep kernels.
//
// Each function restates the reference routine named beside it, expression for
// expression (the library is compiled with --fmad=false so nvcc does not contract
// a*b+c where the reference, built without -march, performs two roundings).
#pragma once
#include <cmath>
#include <cstdint>

#include "rng.cuh"

namespace bnmc_gpu {

constexpr double kLog2Pi = 1.8378770664093454835606594728112;

// draw_gamma (proj/src/dist.cpp:136-155): Marsaglia-Tsang squeeze; shape < 1 draws
// at shape+1 and applies the u^(1/shape) boost (the recursion is one level deep,
// so it is unrolled here).  Returns NaN for a non-positive shape.
__device__ __forceinline__ double draw_gamma(Stream& rng, double shape) {
  if (!(shape > 0.0)) return __longlong_as_double(0x7ff8000000000000ll);  // NaN
  const bool boost = shape < 1.0;
  const double a = boost ? shape + 1.0 : shape;
  const double d = a - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  double g;
  for (;;) {
    double x, v;
    do {
      x = rng.next_gaussian();
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = rng.next_unit();
    if (u < 1.0 - 0.0331 * (x * x) * (x * x)) {
      g = d * v;
      break;
    }
    if (log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) {
      g = d * v;
      break;
    }
  }
  if (boost) g = g * pow(rng.next_unit(), 1.0 / shape);
  return g;
}

// The counters draw_gamma(rng, shape) consumes, without its value: the same attempt
// sequence (the acceptance tests need x, v, u), no d * v and no boost power.
__device__ __forceinline__ void skip_gamma(Stream& rng, double shape) {
  if (!(shape > 0.0)) return;
  const bool boost = shape < 1.0;
  const double a = boost ? shape + 1.0 : shape;
  const double d = a - 1.0 / 3.0;
  const double c = 1.0 / sqrt(9.0 * d);
  for (;;) {
    double x, v;
    do {
      x = rng.next_gaussian();
      v = 1.0 + c * x;
    } while (v <= 0.0);
    v = v * v * v;
    const double u = rng.next_unit();
    if (u < 1.0 - 0.0331 * (x * x) * (x * x)) break;
    if (log(u) < 0.5 * x * x + d * (1.0 - v + log(v))) break;
  }
  if (boost) rng.next_u64();
}

// log_pdf_gaussian (dist.cpp:61-68); variance parameterisation.
__device__ __forceinline__ double log_pdf_gaussian(double x, double mean, double var) {
  if (!(var > 0.0)) return -INFINITY;
  const double d = x - mean;
  return -0.5 * (d * d / var + log(var) + kLog2Pi);
}

// log_pdf_gamma (dist.cpp:85-90); shape / scale parameterisation.
__device__ __forceinline__ double log_pdf_gamma(double x, double shape, double scale) {
  if (!(shape > 0.0) || !(scale > 0.0)) return -INFINITY;
  if (!(x > 0.0)) return -INFINITY;
  return (shape - 1.0) * log(x) - x / scale - shape * log(scale) - lgamma(shape);
}

// log_pdf_inverse_gamma (dist.cpp:92-97).
__device__ __forceinline__ double log_pdf_inverse_gamma(double x, double shape, double scale) {
  if (!(shape > 0.0) || !(scale > 0.0)) return -INFINITY;
  if (!(x > 0.0)) return -INFINITY;
  return shape * log(scale) - lgamma(shape) - (shape + 1.0) * log(x) - scale / x;
}

// log_pmf_categorical at a known in-range index (dist.cpp:107-113).
__device__ __forceinline__ double log_prob(double p) { return p > 0.0 ? log(p) : -INFINITY; }

}  // namespace bnmc_gpu
