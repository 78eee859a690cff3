// relaykv/profiler.hpp -- the layer window of the reference
// (/root/reference/proj/include/relaykv/profiler.hpp:30-43). The offline
// profiler itself runs on the device through rk_profile_model
// (include/relaykv_b200.h); the drop-in carries the profile type the relay
// path consumes.
#pragma once

#include <cstddef>
#include <string>
#include <vector>

namespace relaykv {

struct ProfilerParams {
  double tau_start = 0.99;
  std::size_t tail_layers = 5;
  double stability_lambda = 2.0;
  std::size_t consecutive = 2;
  std::size_t min_rise = 3;
  bool first_negative_alpha = false;
};

struct LayerProfile {
  std::string model_id;
  std::size_t l_start = 0;
  std::size_t l_det = 0;
  std::size_t l_end = 0;
  ProfilerParams params;
  std::vector<double> curve_s;
  std::vector<double> curve_rho;
  std::vector<std::string> warnings;

  // 0 <= l_start <= l_det <= l_end < num_layers, else SchemaError (profiler.cpp:28-35).
  void validate(std::size_t num_layers) const;
};

}  // namespace relaykv
