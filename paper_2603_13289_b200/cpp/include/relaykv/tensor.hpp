// relaykv/tensor.hpp -- the reference's host tensor
// (/root/reference/proj/include/relaykv/tensor.hpp:17-40): dense row-major
// fp32, shape + data, 2-D row helpers. In the drop-in it is only the
// host-side container of weights, caches, traces and results; the
// arithmetic runs on the B200 behind include/relaykv_b200.h.
#pragma once

#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <span>
#include <vector>

namespace relaykv {

using TokenId = std::int32_t;

struct Tensor {
  std::vector<std::size_t> shape;
  std::vector<float> data;

  Tensor() = default;
  explicit Tensor(std::vector<std::size_t> s);
  Tensor(std::initializer_list<std::size_t> s) : Tensor(std::vector<std::size_t>(s)) {}

  std::size_t numel() const { return data.size(); }
  bool empty() const { return data.empty(); }
  std::size_t rows() const { return shape.empty() ? 0 : shape[0]; }
  std::size_t cols() const;  // trailing dims flattened

  float& at(std::size_t r, std::size_t c) { return data[r * cols() + c]; }
  float at(std::size_t r, std::size_t c) const { return data[r * cols() + c]; }
  std::span<float> row(std::size_t r) { return {data.data() + r * cols(), cols()}; }
  std::span<const float> row(std::size_t r) const { return {data.data() + r * cols(), cols()}; }

  // Bitwise comparison (distinguishes -0.0f, NaN payloads literally).
  bool bit_equal(const Tensor& other) const;
};

}  // namespace relaykv
