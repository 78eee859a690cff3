// profiler.h -- host side of the offline layer profiler (profiler.cpp).
#pragma once
#include <cstdint>
#include <vector>

#include "internal.h"

namespace rk {
namespace prof {

// LayerCurve (metrics.hpp:178-182)
struct Curve {
  std::vector<double> s, rho;
  std::vector<uint8_t> deg;
};

void validate_params(const rk_profiler_params& p);  // ProfilerParams::validate (profiler.cpp:16-26)
void validate_calib(const rk_two_stage_config& c);  // TwoStageConfig::validate (metrics.cpp:272-279)
Curve layer_curve(const double* value_cos, size_t n, size_t L);  // make_layer_curve
Curve average(const std::vector<Curve>& curves);                 // average_curves
// profile_from_curve (profiler.cpp:123-155); curve_rho: [L-1]
rk_profile_result from_curve(const Curve& c, const rk_profiler_params& p, std::vector<double>* curve_rho);
std::vector<int32_t> synthetic_tokens(uint64_t seed, uint64_t salt, size_t count, size_t vocab);
size_t pick_length(uint64_t seed, uint64_t salt, size_t lo, size_t hi);

}  // namespace prof
}  // namespace rk
