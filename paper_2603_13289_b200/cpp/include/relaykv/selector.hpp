// relaykv/selector.hpp -- selection types of the reference
// (/root/reference/proj/include/relaykv/selector.hpp:13-54). The selection
// itself (select_deviation / select_influence / suffix_set / final_selection /
// top_k_by_score, selector.cpp:32-105) runs on the device inside
// relay_extend (K2b select_relay_kernel, topk_flags_kernel).
#pragma once

#include <cstddef>
#include <vector>

namespace relaykv {

struct SelectionThresholds {
  double tau_dev = 1.5;
  double tau_inf = 1.45;
  std::size_t suffix_k = 10;

  void validate() const;  // tau_dev > 0, tau_inf > 0 (std::invalid_argument)
};

enum SelectionTag : unsigned {
  kSelDeviation = 1u << 0,
  kSelInfluenceScore = 1u << 1,
  kSelInfluenceSuffix = 1u << 2,
  kSelBlendTopK = 1u << 3,
};

struct SelectionSet {
  std::vector<std::size_t> indices;  // ascending
  std::vector<unsigned> tags;        // parallel to indices

  std::size_t size() const { return indices.size(); }
  bool contains(std::size_t idx) const;
  std::size_t count_tag(unsigned tag) const;
};

}  // namespace relaykv
