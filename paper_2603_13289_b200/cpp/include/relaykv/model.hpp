// relaykv/model.hpp -- C++ drop-in for the reference's model API
// (/root/reference/proj/include/relaykv/model.hpp:21-175), implemented over
// the C ABI of include/relaykv_b200.h: same type and function names, same
// argument meaning, same exception types. The arithmetic runs on the B200:
//   Precision::kFp32Exact (default): bit-identical to the reference CPU path;
//   Precision::kBf16: the tensor-core throughput mode.
// Host-visible differences, by design:
//   - Weights carries a handle to its device copy (uploaded on first use,
//     freed with the object). A tensor edited IN PLACE after first use must
//     be followed by release_device_weights(w); replacing a tensor's storage
//     is detected.
//   - KVContext rows live on the device; key_row()/value_row() read a host
//     mirror refreshed after every call that mutates the context.
//   - set_prefill_logits(kLastRow) makes prefill() compute only the last row's
//     logits (the only row run_workflow / relay_prefill ever read); the default
//     kAllRows returns every row like the reference.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "relaykv/errors.hpp"
#include "relaykv/tensor.hpp"

struct rk_context;
struct rk_weights;

namespace relaykv {

enum class Precision { kFp32Exact = 0, kBf16 = 1, kFp32Tc = 2 };  // = rk_precision
enum class PrefillLogits { kAllRows = 0, kLastRow = 1 };
// Device and numerics of subsequent calls (process-wide; default 0, exact, all rows).
void set_device(int device);
void set_precision(Precision p);
void set_prefill_logits(PrefillLogits mode);

struct ModelSpec {
  std::size_t num_layers = 0;
  std::size_t d_model = 0;
  std::size_t num_heads = 0;
  std::size_t num_kv_heads = 0;
  std::size_t d_head = 0;
  std::size_t d_ff = 0;
  std::size_t vocab_size = 0;
  float theta_base = 10000.0f;
  std::size_t max_positions = 0;
  float norm_eps = 1e-5f;

  std::size_t q_dim() const { return num_heads * d_head; }
  std::size_t kv_dim() const { return num_kv_heads * d_head; }
  std::size_t head_group() const { return num_heads / num_kv_heads; }

  void validate() const;  // throws SchemaError (model.cpp:19-34)
  std::string summary_id(std::uint64_t seed) const;
};

struct LayerWeights {
  Tensor attn_norm_gain;  // [d_model]
  Tensor w_q;             // [d_model x q_dim]
  Tensor w_k, w_v;        // [d_model x kv_dim]
  Tensor w_o;             // [q_dim x d_model]
  Tensor mlp_norm_gain;   // [d_model]
  Tensor w_gate, w_up;    // [d_model x d_ff]
  Tensor w_down;          // [d_ff x d_model]
};

namespace detail {
struct DeviceWeights;  // device copies of one Weights object, per precision
// Owned by one Weights object: a copy of the Weights starts without device
// copies (its tensors live elsewhere), a move takes them along.
struct DeviceWeightsHandle {
  std::shared_ptr<DeviceWeights> p;
  DeviceWeightsHandle() = default;
  DeviceWeightsHandle(const DeviceWeightsHandle&) {}
  DeviceWeightsHandle& operator=(const DeviceWeightsHandle&) {
    p.reset();
    return *this;
  }
  DeviceWeightsHandle(DeviceWeightsHandle&&) noexcept = default;
  DeviceWeightsHandle& operator=(DeviceWeightsHandle&&) noexcept = default;
};
}  // namespace detail

struct Weights {
  ModelSpec spec;
  std::string model_id;
  Tensor embedding;  // [vocab x d_model]
  std::vector<LayerWeights> layers;
  Tensor final_norm_gain;  // [d_model]
  Tensor output_head;      // [d_model x vocab]
  mutable detail::DeviceWeightsHandle device;  // drop-in: the B200 copies (uploaded on first use)
};

// == init_weights (model.cpp:81-114): generated on the device (SplitMix64,
// bit-identical to the reference) and copied back; the device copy is kept.
Weights init_weights(const ModelSpec& spec, std::uint64_t seed);
// Drop the device copies of w (call after editing its tensors in place).
void release_device_weights(const Weights& w);

class KVContext {
 public:
  KVContext() = default;
  KVContext(std::size_t num_layers, std::size_t kv_dim);
  explicit KVContext(const ModelSpec& spec);
  KVContext(const KVContext& o);  // deep copy on the device (rk_context_clone)
  KVContext& operator=(const KVContext& o);
  KVContext(KVContext&&) noexcept = default;
  KVContext& operator=(KVContext&&) noexcept = default;

  std::size_t size() const;
  std::size_t num_layers() const { return num_layers_; }
  std::size_t kv_dim() const { return kv_dim_; }
  std::span<const float> key_row(std::size_t layer, std::size_t pos) const;
  std::span<const float> value_row(std::size_t layer, std::size_t pos) const;

  // drop-in plumbing: the device context, created/bound on first use
  rk_context* handle(const Weights& w);
  rk_context* handle() const { return ctx_.get(); }
  void invalidate() const {
    mirror_k_.clear();
    mirror_v_.clear();
  }

 private:
  void fetch() const;
  std::size_t num_layers_ = 0, kv_dim_ = 0;
  std::shared_ptr<rk_weights> bound_;  // device weights the context was created for (outlives ctx_)
  std::shared_ptr<rk_context> ctx_;
  mutable std::vector<std::vector<float>> mirror_k_, mirror_v_;
};

// Opt-in, chunk-scoped capture (model.hpp:89-111).
struct CaptureFlags {
  bool hidden = false;         // residual-stream input to every layer
  bool pre_rope_keys = false;  // K before rotation, plus V as produced
  bool attention = false;      // per-head attention rows
};

struct StepTrace {
  std::vector<Tensor> hidden;  // [L] chunk x d_model
  std::vector<Tensor> k_pre;   // [L] chunk x kv_dim
  std::vector<Tensor> v;       // [L] chunk x kv_dim
  // attn[layer][chunk_row] is H x (ctx_len_at_row).
  std::vector<std::vector<Tensor>> attn;
  Tensor logits;  // chunk x vocab
};

struct PrefillResult {
  Tensor logits;  // chunk x vocab (kLastRow: only the last row is filled)
  StepTrace trace;
};

// Causal forward over past + chunk (model.cpp:305-331). base_position must
// equal ctx.size(). Throws std::invalid_argument like the reference.
PrefillResult prefill(const Weights& w, std::span<const TokenId> tokens, KVContext& ctx,
                      std::size_t base_position, const CaptureFlags& capture = {});
PrefillResult decode_step(const Weights& w, TokenId token, KVContext& ctx, std::size_t position,
                          const CaptureFlags& capture = {});

// Layers [first_layer, L) for one row as a pure query (model.cpp:339-362).
Tensor row_logits_from_layer(const Weights& w, std::span<const float> hidden_row, std::size_t first_layer,
                             const KVContext& ctx, std::size_t position);

struct GenerateResult {
  std::vector<TokenId> tokens;
};

// Called once per decode step with the step trace, the token that was fed,
// and its absolute position. The trace is only alive during the call.
using StepHook = std::function<void(const StepTrace&, TokenId, std::size_t)>;

// Greedy continuation (model.cpp:364-389): exactly max_new_tokens decode steps.
GenerateResult greedy_generate(const Weights& w, KVContext& ctx, std::span<const float> prompt_end_logits,
                               std::size_t max_new_tokens, const CaptureFlags& capture = {},
                               const StepHook& hook = {});

std::size_t argmax(std::span<const float> values);

}  // namespace relaykv
