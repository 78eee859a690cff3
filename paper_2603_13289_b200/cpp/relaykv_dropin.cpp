// relaykv_dropin.cpp -- the reference's relaykv C++ API over the C ABI of
// include/relaykv_b200.h (see cpp/include/relaykv/*.hpp for the mapping and
// the deliberate differences). Error statuses are re-thrown as the
// reference's exception types. Every computation on a
// tensor runs on the device; host code here validates, marshals and keeps
// the reference's bookkeeping (RelayRecorder's trace accumulation).
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

#include "relaykv/relay_engine.hpp"
#include "relaykv_b200.h"

namespace relaykv {

namespace detail {
// Device copies of one Weights object, per precision. `sig` records the
// storage of every host tensor at upload: a tensor whose vector was replaced
// (new storage) forces a re-upload; in-place edits need release_device_weights.
struct DeviceWeights {
  struct Entry {
    int precision;
    std::vector<const float*> sig;
    std::shared_ptr<rk_weights> dev;
  };
  std::mutex mu;
  std::vector<Entry> entries;
};
}  // namespace detail

namespace {

std::mutex g_mu;
int g_device = 0;
Precision g_prec = Precision::kFp32Exact;
PrefillLogits g_logits = PrefillLogits::kAllRows;
std::map<int, rk_engine*> g_engines;

void check(int st) {
  if (st == RK_OK) return;
  const std::string msg = rk_last_error();
  switch (st) {
    case RK_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case RK_ERR_SCHEMA: throw SchemaError(msg);
    case RK_ERR_LOGIC: throw std::logic_error(msg);
    case RK_ERR_IO: throw IoError(msg);
    default: throw std::runtime_error(msg);
  }
}

rk_engine* engine() {
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_engines.find(g_device);
  if (it != g_engines.end()) return it->second;
  rk_engine* e = nullptr;
  check(rk_engine_create(g_device, &e));
  g_engines[g_device] = e;
  return e;
}

rk_model_spec to_c(const ModelSpec& s) {
  return rk_model_spec{s.num_layers, s.d_model, s.num_heads, s.num_kv_heads, s.d_head, s.d_ff, s.vocab_size,
                       s.theta_base, s.max_positions, s.norm_eps};
}

const Tensor& tensor_at(const Weights& w, std::size_t idx) {  // weights_io.cpp:21-38 order
  if (idx == 0) return w.embedding;
  idx -= 1;
  if (idx < 9 * w.layers.size()) {
    const LayerWeights& l = w.layers[idx / 9];
    const Tensor* t[] = {&l.attn_norm_gain, &l.w_q, &l.w_k, &l.w_v, &l.w_o, &l.mlp_norm_gain, &l.w_gate, &l.w_up,
                         &l.w_down};
    return *t[idx % 9];
  }
  idx -= 9 * w.layers.size();
  return idx == 0 ? w.final_norm_gain : w.output_head;
}

std::size_t num_tensors(const Weights& w) { return 3 + 9 * w.layers.size(); }

std::vector<const float*> signature(const Weights& w) {
  std::vector<const float*> sig;
  for (std::size_t i = 0; i < num_tensors(w); ++i) sig.push_back(tensor_at(w, i).data.data());
  return sig;
}

std::shared_ptr<rk_weights> wrap(rk_weights* dw) { return std::shared_ptr<rk_weights>(dw, rk_weights_destroy); }

// The device copy of w in the current precision (uploaded on first use).
std::shared_ptr<rk_weights> device_weights(const Weights& w) {
  rk_engine* e = engine();
  if (w.layers.size() != w.spec.num_layers) throw std::invalid_argument("weights: layer count does not match spec");
  if (!w.device.p) w.device.p = std::make_shared<detail::DeviceWeights>();
  detail::DeviceWeights& D = *w.device.p;
  const int prec = (int)g_prec;
  const std::vector<const float*> sig = signature(w);
  std::lock_guard<std::mutex> lock(D.mu);
  for (auto& en : D.entries)
    if (en.precision == prec && en.sig == sig) return en.dev;
  const rk_model_spec s = to_c(w.spec);
  rk_weights* dw = nullptr;
  check(rk_weights_upload(e, &s, sig.data(), sig.size(), prec, &dw));
  auto dev = wrap(dw);
  D.entries.erase(std::remove_if(D.entries.begin(), D.entries.end(),
                                 [&](const detail::DeviceWeights::Entry& en) { return en.precision == prec; }),
                  D.entries.end());
  D.entries.push_back({prec, sig, dev});
  return dev;
}

// Host view of a RelayCache for the C ABI; validates like the reference
// before any pointer is handed over (relay_cache.cpp:18-49).
struct CacheView {
  std::vector<const float*> kp, vp;
  rk_relay_cache_view view{};
  explicit CacheView(const RelayCache& c) {
    c.validate();
    for (std::size_t l = 0; l < c.num_layers(); ++l) {
      kp.push_back(c.k_pre[l].data.data());
      vp.push_back(c.v[l].data.data());
    }
    view = rk_relay_cache_view{c.num_layers(), c.num_kv_heads, c.d_head, c.d_model, c.theta_base, c.max_positions,
                               c.segment_len(), c.segment_tokens.data(), c.source_base_position, c.snapshot_layer,
                               c.decode_steps_observed, kp.data(), vp.data(), c.hidden_snapshot.data.data(),
                               c.influence.data()};
  }
};

// Per-call upload: layer-streamed on the engine's copy stream
// (rk_cache_upload_async), so the relay starts while later layers cross PCIe;
// from page-locked memory (PinnedRelayCache) at full speed.
struct CacheUpload : CacheView {
  rk_cache* dev = nullptr;
  CacheUpload(const RelayCache& c, rk_weights* w) : CacheView(c) {
    check(rk_cache_upload_async(engine(), w, &view, &dev));
  }
  ~CacheUpload() {
    rk_cache_wait(dev);  // the host arrays may go away after the call
    rk_cache_destroy(dev);
  }
};

rk_relay_options to_c(const RelayOptions& o) {
  const int mode = o.mode == RelayMode::kFull ? RK_MODE_FULL
                   : o.mode == RelayMode::kZero ? RK_MODE_ZERO
                   : o.mode == RelayMode::kRelay ? RK_MODE_RELAY
                                                 : RK_MODE_BLEND;
  return rk_relay_options{mode, o.thresholds.tau_dev, o.thresholds.tau_inf, o.thresholds.suffix_k, o.blend_alpha,
                          o.rectify_above_end ? 1 : 0};
}

// Host buffers for an rk_relay_output of a segment of n rows.
struct OutBufs {
  std::vector<uint64_t> sel, depth;
  std::vector<uint32_t> tags;
  std::vector<double> s_dev, s_key;
  std::vector<uint8_t> origin;
  Tensor hidden;
  rk_relay_output out{};
  OutBufs(std::size_t n, const ModelSpec& s)
      : sel(n), depth(n), tags(n), s_dev(n), s_key(n), origin(s.num_layers * n), hidden({n, s.d_model}) {
    out.selection_indices = sel.data();
    out.selection_tags = tags.data();
    out.s_dev = s_dev.data();
    out.s_key_dev = s_key.data();
    out.segment_hidden = hidden.data.data();
    out.hidden_depth = depth.data();
    out.origin = origin.data();
  }
  RelayOutput to_output() {
    RelayOutput r;
    const rk_reuse_stats& st = out.stats;
    r.stats.total_entries = st.total_entries;
    r.stats.recomputed_entries = st.recomputed_entries;
    r.stats.reuse_rate = st.reuse_rate;
    r.stats.selected_count = st.selected_count;
    r.stats.selected_deviation = st.selected_deviation;
    r.stats.selected_influence_score = st.selected_influence_score;
    r.stats.selected_influence_suffix = st.selected_influence_suffix;
    r.stats.selected_blend = st.selected_blend;
    r.stats.flops_cost = st.flops_cost;
    r.stats.flops_selection = st.flops_selection;
    r.stats.flops_realign = st.flops_realign;
    r.stats.flops_full_equiv = st.flops_full_equiv;
    r.stats.wall = PhaseTimings{st.wall.fresh_ms, st.wall.realign_ms, st.wall.recompute_ms, st.wall.selection_ms,
                                st.wall.rectify_ms, st.wall.total_ms};
    for (std::size_t i = 0; i < out.selection_count; ++i) {
      r.selection.indices.push_back(sel[i]);
      r.selection.tags.push_back(tags[i]);
    }
    r.s_dev.assign(s_dev.begin(), s_dev.begin() + out.s_dev_len);
    r.s_key_dev.assign(s_key.begin(), s_key.begin() + out.s_dev_len);
    r.segment_hidden = std::move(hidden);
    r.hidden_depth.assign(depth.begin(), depth.end());
    return r;
  }
  SegmentMarks marks() const {
    SegmentMarks m;
    m.base = out.segment_base;
    m.len = out.segment_len;
    for (uint8_t o : origin) m.origin.push_back(static_cast<CellOrigin>(o));
    return m;
  }
};

}  // namespace

void set_device(int device) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_device = device;
}
void set_precision(Precision p) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_prec = p;
}
void set_prefill_logits(PrefillLogits mode) {
  std::lock_guard<std::mutex> lock(g_mu);
  g_logits = mode;
}

// ---- model ------------------------------------------------------------------
void ModelSpec::validate() const {
  std::ostringstream err;
  if (num_layers < 6) err << "num_layers must be >= 6 (profiling needs a usable curve); ";
  if (d_model == 0 || num_heads == 0 || num_kv_heads == 0 || d_head == 0 || d_ff == 0 || vocab_size == 0 ||
      max_positions == 0) {
    err << "all extents must be >= 1; ";
  } else {
    if (num_heads % num_kv_heads != 0) err << "num_heads must be divisible by num_kv_heads; ";
    if (d_model != num_heads * d_head) err << "d_model must equal num_heads * d_head; ";
    if (d_head % 2 != 0) err << "d_head must be even for rotary embedding; ";
  }
  if (!(theta_base > 0.0f)) err << "theta_base must be positive; ";
  if (!(norm_eps > 0.0f)) err << "norm_eps must be positive; ";
  const std::string msg = err.str();
  if (!msg.empty()) throw SchemaError("invalid model spec: " + msg);
}

std::string ModelSpec::summary_id(std::uint64_t seed) const {
  std::ostringstream os;
  os << "toy-L" << num_layers << "-d" << d_model << "-h" << num_heads << "-kv" << num_kv_heads << "-ff" << d_ff
     << "-v" << vocab_size << "-s" << seed;
  return os.str();
}

Tensor::Tensor(std::vector<std::size_t> s) : shape(std::move(s)) {
  std::size_t n = 1;
  for (std::size_t e : shape) n *= e;
  data.assign(shape.empty() ? 0 : n, 0.0f);
}
std::size_t Tensor::cols() const {
  if (shape.size() < 2) return shape.size() == 1 ? 1 : 0;
  std::size_t c = 1;
  for (std::size_t i = 1; i < shape.size(); ++i) c *= shape[i];
  return c;
}
bool Tensor::bit_equal(const Tensor& o) const {
  return shape == o.shape && data.size() == o.data.size() &&
         std::memcmp(data.data(), o.data.data(), data.size() * sizeof(float)) == 0;
}

Weights init_weights(const ModelSpec& spec, std::uint64_t seed) {
  spec.validate();
  const rk_model_spec s = to_c(spec);
  rk_weights* raw = nullptr;
  check(rk_weights_init(engine(), &s, seed, RK_FP32_EXACT, &raw));
  auto dev = wrap(raw);
  Weights w;
  w.spec = spec;
  w.model_id = spec.summary_id(seed);
  const std::size_t d = spec.d_model, q = spec.q_dim(), kv = spec.kv_dim(), ff = spec.d_ff, V = spec.vocab_size;
  auto fetch = [&](std::size_t idx, std::vector<std::size_t> shape) {
    Tensor t(std::move(shape));
    check(rk_weights_export(raw, idx, t.data.data(), t.data.size()));
    return t;
  };
  w.embedding = fetch(0, {V, d});
  w.layers.resize(spec.num_layers);
  for (std::size_t l = 0; l < spec.num_layers; ++l) {
    const std::size_t b = 1 + 9 * l;
    LayerWeights& L = w.layers[l];
    L.attn_norm_gain = fetch(b, {d});
    L.w_q = fetch(b + 1, {d, q});
    L.w_k = fetch(b + 2, {d, kv});
    L.w_v = fetch(b + 3, {d, kv});
    L.w_o = fetch(b + 4, {q, d});
    L.mlp_norm_gain = fetch(b + 5, {d});
    L.w_gate = fetch(b + 6, {d, ff});
    L.w_up = fetch(b + 7, {d, ff});
    L.w_down = fetch(b + 8, {ff, d});
  }
  w.final_norm_gain = fetch(1 + 9 * spec.num_layers, {d});
  w.output_head = fetch(2 + 9 * spec.num_layers, {d, V});
  // keep the exact device copy we already have (the vectors keep their storage when w is moved out)
  w.device.p = std::make_shared<detail::DeviceWeights>();
  w.device.p->entries.push_back({(int)Precision::kFp32Exact, signature(w), dev});
  return w;
}

void release_device_weights(const Weights& w) { w.device.p.reset(); }

// ---- KVContext --------------------------------------------------------------
KVContext::KVContext(std::size_t num_layers, std::size_t kv_dim) : num_layers_(num_layers), kv_dim_(kv_dim) {}
KVContext::KVContext(const ModelSpec& spec) : KVContext(spec.num_layers, spec.kv_dim()) {}
KVContext::KVContext(const KVContext& o) : num_layers_(o.num_layers_), kv_dim_(o.kv_dim_), bound_(o.bound_) {
  if (o.ctx_) {
    rk_context* c = nullptr;
    check(rk_context_clone(o.ctx_.get(), &c));
    ctx_.reset(c, rk_context_destroy);
  }
}
KVContext& KVContext::operator=(const KVContext& o) {
  if (this != &o) {
    KVContext tmp(o);
    *this = std::move(tmp);
    invalidate();
  }
  return *this;
}
std::size_t KVContext::size() const { return ctx_ ? rk_context_size(ctx_.get()) : 0; }
rk_context* KVContext::handle(const Weights& w) {
  auto dw = device_weights(w);
  if (ctx_ && bound_ != dw) {
    if (size() != 0)
      throw std::invalid_argument("KVContext holds positions computed with other weights (or another precision)");
    ctx_.reset();
  }
  if (!ctx_) {
    num_layers_ = w.spec.num_layers;
    kv_dim_ = w.spec.kv_dim();
    rk_context* c = nullptr;
    check(rk_context_create(engine(), dw.get(), &c));
    bound_ = dw;
    ctx_.reset(c, rk_context_destroy);
  }
  invalidate();
  return ctx_.get();
}
void KVContext::fetch() const {
  if (!mirror_k_.empty() || !ctx_) return;
  const std::size_t n = size(), w = kv_dim_;
  mirror_k_.assign(num_layers_, std::vector<float>(n * w));
  mirror_v_.assign(num_layers_, std::vector<float>(n * w));
  for (std::size_t l = 0; l < num_layers_; ++l)
    check(rk_context_export(ctx_.get(), l, 0, n, mirror_k_[l].data(), mirror_v_[l].data()));
}
std::span<const float> KVContext::key_row(std::size_t layer, std::size_t pos) const {
  if (layer >= num_layers_ || pos >= size()) throw std::out_of_range("KVContext::key_row out of range");
  fetch();
  return {mirror_k_[layer].data() + pos * kv_dim_, kv_dim_};
}
std::span<const float> KVContext::value_row(std::size_t layer, std::size_t pos) const {
  if (layer >= num_layers_ || pos >= size()) throw std::out_of_range("KVContext::value_row out of range");
  fetch();
  return {mirror_v_[layer].data() + pos * kv_dim_, kv_dim_};
}

// ---- prefill / decode -------------------------------------------------------
PrefillResult prefill(const Weights& w, std::span<const TokenId> tokens, KVContext& ctx, std::size_t base,
                      const CaptureFlags& capture) {
  const ModelSpec& s = w.spec;
  // model.cpp:307-315: the reference checks before touching the context
  if (tokens.empty()) throw std::invalid_argument("prefill: empty token chunk");
  rk_context* c = ctx.handle(w);
  const std::size_t n = tokens.size(), L = s.num_layers, keys = base + n;
  PrefillResult r;
  r.logits = Tensor({n, s.vocab_size});
  const bool any = capture.hidden || capture.pre_rope_keys || capture.attention;
  if (!any && g_logits == PrefillLogits::kLastRow) {
    check(rk_prefill(engine(), device_weights(w).get(), c, tokens.data(), n, base,
                     r.logits.data.data() + (n - 1) * s.vocab_size));
  } else {
    std::vector<float> hid, kp, vv, at;
    rk_trace_request req{};
    req.logits = r.logits.data.data();
    if (capture.hidden) req.hidden = (hid.resize(L * n * s.d_model), hid.data());
    if (capture.pre_rope_keys) {
      req.k_pre = (kp.resize(L * n * s.kv_dim()), kp.data());
      req.v = (vv.resize(L * n * s.kv_dim()), vv.data());
    }
    if (capture.attention) req.attn = (at.resize(L * n * s.num_heads * keys), at.data());
    check(rk_prefill_trace(engine(), device_weights(w).get(), c, tokens.data(), n, base, &req));
    StepTrace& t = r.trace;
    auto slab = [&](const std::vector<float>& src, std::size_t l, std::size_t width) {
      Tensor x({n, width});
      std::copy(src.begin() + l * n * width, src.begin() + (l + 1) * n * width, x.data.begin());
      return x;
    };
    for (std::size_t l = 0; l < L; ++l) {
      if (capture.hidden) t.hidden.push_back(slab(hid, l, s.d_model));
      if (capture.pre_rope_keys) {
        t.k_pre.push_back(slab(kp, l, s.kv_dim()));
        t.v.push_back(slab(vv, l, s.kv_dim()));
      }
      if (capture.attention) {
        std::vector<Tensor> rows;
        for (std::size_t i = 0; i < n; ++i) {  // H x (ctx_len_at_row)
          const std::size_t len = base + i + 1;
          Tensor a({s.num_heads, len});
          for (std::size_t h = 0; h < s.num_heads; ++h) {
            const float* src = at.data() + ((l * n + i) * s.num_heads + h) * keys;
            std::copy(src, src + len, a.row(h).begin());
          }
          rows.push_back(std::move(a));
        }
        t.attn.push_back(std::move(rows));
      }
    }
    t.logits = r.logits;
  }
  ctx.invalidate();
  return r;
}

PrefillResult decode_step(const Weights& w, TokenId token, KVContext& ctx, std::size_t position,
                          const CaptureFlags& capture) {
  const TokenId one[1] = {token};
  return prefill(w, one, ctx, position, capture);
}

Tensor row_logits_from_layer(const Weights& w, std::span<const float> hidden_row, std::size_t first_layer,
                             const KVContext& ctx, std::size_t position) {
  if (hidden_row.size() != w.spec.d_model) throw std::invalid_argument("row_logits_from_layer: row width");
  Tensor out({1, w.spec.vocab_size});
  // a pure query: nothing is committed, so the const context's device copy is used as is
  KVContext& c = const_cast<KVContext&>(ctx);
  check(rk_row_logits_from_layer(engine(), device_weights(w).get(), c.handle(w), hidden_row.data(), first_layer,
                                 position, out.data.data()));
  return out;
}

std::size_t argmax(std::span<const float> values) {  // model.cpp:364-370 (first maximum wins)
  std::size_t best = 0;
  for (std::size_t i = 1; i < values.size(); ++i)
    if (values[i] > values[best]) best = i;
  return best;
}

GenerateResult greedy_generate(const Weights& w, KVContext& ctx, std::span<const float> prompt_end_logits,
                               std::size_t max_new_tokens, const CaptureFlags& capture, const StepHook& hook) {
  GenerateResult out;
  if (max_new_tokens == 0) return out;
  TokenId next = static_cast<TokenId>(argmax(prompt_end_logits));
  for (std::size_t t = 0; t < max_new_tokens; ++t) {
    const std::size_t pos = ctx.size();
    const PrefillResult step = decode_step(w, next, ctx, pos, capture);
    out.tokens.push_back(next);
    if (hook) hook(step.trace, next, pos);
    if (t + 1 < max_new_tokens) next = static_cast<TokenId>(argmax(step.logits.row(0)));
  }
  return out;
}

// ---- relay caches -----------------------------------------------------------
void RelayCache::validate() const {  // relay_cache.cpp:18-41
  const std::size_t n = segment_len();
  if (n == 0) throw std::invalid_argument("relay cache: empty segment");
  if (k_pre.size() != v.size() || k_pre.empty()) throw std::invalid_argument("relay cache: per-layer K/V tables disagree");
  if (snapshot_layer >= num_layers()) throw std::invalid_argument("relay cache: snapshot layer out of range");
  for (std::size_t l = 0; l < num_layers(); ++l) {
    if (k_pre[l].rows() != n || v[l].rows() != n || k_pre[l].cols() != kv_dim() || v[l].cols() != kv_dim() ||
        k_pre[l].data.size() != n * kv_dim() || v[l].data.size() != n * kv_dim())
      throw std::invalid_argument("relay cache: layer " + std::to_string(l) + " tensor shape mismatch");
  }
  if (hidden_snapshot.rows() != n || hidden_snapshot.cols() != d_model || hidden_snapshot.data.size() != n * d_model)
    throw std::invalid_argument("relay cache: hidden snapshot shape mismatch");
  if (influence.size() != n) throw std::invalid_argument("relay cache: influence length mismatch");
  for (float s : influence)
    if (!(s >= 0.0f)) throw std::invalid_argument("relay cache: negative influence score");
}

void RelayCache::validate_for(const ModelSpec& spec) const {  // relay_cache.cpp:43-49
  validate();
  if (num_layers() != spec.num_layers || num_kv_heads != spec.num_kv_heads || d_head != spec.d_head ||
      d_model != spec.d_model || theta_base != spec.theta_base)
    throw std::invalid_argument("relay cache geometry does not match model spec");
}

// RelayRecorder (relay_cache.cpp:51-136): the reference's streaming recorder
// over host step traces, kept for StepHook callers. Influence sums follow the
// reference's order (layer -> head -> position, double), so the result is
// bit-identical to the reference's and to rk_cache_capture_decode.
RelayRecorder::RelayRecorder(const ModelSpec& spec, std::size_t source_base_position, std::size_t snapshot_layer,
                             bool include_self)
    : spec_(spec), include_self_(include_self) {
  if (snapshot_layer >= spec.num_layers) throw std::invalid_argument("recorder: snapshot layer out of range");
  cache_.num_kv_heads = spec.num_kv_heads;
  cache_.d_head = spec.d_head;
  cache_.d_model = spec.d_model;
  cache_.theta_base = spec.theta_base;
  cache_.max_positions = spec.max_positions;
  cache_.source_base_position = source_base_position;
  cache_.snapshot_layer = snapshot_layer;
  cache_.k_pre.assign(spec.num_layers, Tensor{});
  cache_.v.assign(spec.num_layers, Tensor{});
}

void RelayRecorder::feed(const StepTrace& trace, TokenId token, std::size_t position) {
  const std::size_t t = cache_.segment_tokens.size(), L = spec_.num_layers;
  if (position != cache_.source_base_position + t) throw std::invalid_argument("recorder: step position out of sequence");
  if (trace.k_pre.size() != L || trace.v.size() != L)
    throw std::invalid_argument("recorder: capture missing field 'pre_rope_keys'");
  if (trace.hidden.size() != L) throw std::invalid_argument("recorder: capture missing field 'hidden'");
  if (trace.attn.size() != L) throw std::invalid_argument("recorder: capture missing field 'attention'");
  if (t == 0) {
    for (std::size_t l = 0; l < L; ++l) {
      cache_.k_pre[l] = Tensor({0, spec_.kv_dim()});
      cache_.v[l] = Tensor({0, spec_.kv_dim()});
    }
    cache_.hidden_snapshot = Tensor({0, spec_.d_model});
  }
  for (std::size_t l = 0; l < L; ++l) {
    if (trace.k_pre[l].rows() != 1 || trace.v[l].rows() != 1)
      throw std::invalid_argument("recorder: expected single-row decode trace");
    cache_.k_pre[l].shape[0] = t + 1;
    cache_.k_pre[l].data.insert(cache_.k_pre[l].data.end(), trace.k_pre[l].data.begin(), trace.k_pre[l].data.end());
    cache_.v[l].shape[0] = t + 1;
    cache_.v[l].data.insert(cache_.v[l].data.end(), trace.v[l].data.begin(), trace.v[l].data.end());
  }
  const Tensor& snap = trace.hidden[cache_.snapshot_layer];
  cache_.hidden_snapshot.shape[0] = t + 1;
  cache_.hidden_snapshot.data.insert(cache_.hidden_snapshot.data.end(), snap.data.begin(), snap.data.end());
  influence_acc_.resize(t + 1, 0.0);
  const std::size_t upto = include_self_ ? t + 1 : t;
  for (std::size_t l = 0; l < L; ++l) {
    if (trace.attn[l].size() != 1) throw std::invalid_argument("recorder: capture missing field 'attention'");
    const Tensor& rows = trace.attn[l][0];  // H x (position+1)
    for (std::size_t h = 0; h < spec_.num_heads; ++h) {
      const auto row = rows.row(h);
      for (std::size_t j = 0; j < upto; ++j)
        influence_acc_[j] += static_cast<double>(row[cache_.source_base_position + j]);
    }
  }
  cache_.segment_tokens.push_back(token);
  cache_.decode_steps_observed = t + 1;
}

RelayCache RelayRecorder::finalize() {
  cache_.influence.resize(cache_.segment_tokens.size());
  for (std::size_t j = 0; j < cache_.influence.size(); ++j) cache_.influence[j] = static_cast<float>(influence_acc_[j]);
  cache_.validate();
  return std::move(cache_);
}

RelayCache record_from_decode(const ModelSpec& spec, std::span<const StepTrace> traces,
                              std::span<const TokenId> segment_tokens, std::size_t source_base_position,
                              std::size_t snapshot_layer, bool include_self) {
  if (traces.size() != segment_tokens.size())
    throw std::invalid_argument("record_from_decode: traces do not cover the segment (" +
                                std::to_string(traces.size()) + " steps for " + std::to_string(segment_tokens.size()) +
                                " tokens)");
  RelayRecorder rec(spec, source_base_position, snapshot_layer, include_self);
  for (std::size_t t = 0; t < traces.size(); ++t) rec.feed(traces[t], segment_tokens[t], source_base_position + t);
  return rec.finalize();
}

PinnedRelayCache::PinnedRelayCache(const RelayCache& c) {
  auto pin = [&](const void* p, std::size_t bytes) {
    if (!p || bytes == 0) return;
    check(rk_host_pin(const_cast<void*>(p), bytes));
    pinned_.push_back(const_cast<void*>(p));
  };
  try {
    for (std::size_t l = 0; l < c.num_layers(); ++l) {
      pin(c.k_pre[l].data.data(), c.k_pre[l].data.size() * sizeof(float));
      pin(c.v[l].data.data(), c.v[l].data.size() * sizeof(float));
    }
    pin(c.hidden_snapshot.data.data(), c.hidden_snapshot.data.size() * sizeof(float));
  } catch (...) {
    for (void* p : pinned_) rk_host_unpin(p);
    throw;
  }
}
PinnedRelayCache::~PinnedRelayCache() {
  for (void* p : pinned_) rk_host_unpin(p);
}

namespace {
// A decoded RKRC file (rk_cache_file) -> RelayCache, freeing the file.
RelayCache take_file(rk_cache_file* f, const rk_relay_cache_view& v) {
  RelayCache c;
  const std::size_t n = v.segment_len, kv = v.num_kv_heads * v.d_head;
  c.num_kv_heads = v.num_kv_heads;
  c.d_head = v.d_head;
  c.d_model = v.d_model;
  c.theta_base = v.theta_base;
  c.max_positions = v.max_positions;
  c.segment_tokens.assign(v.segment_tokens, v.segment_tokens + n);
  c.source_base_position = v.source_base_position;
  c.snapshot_layer = v.snapshot_layer;
  c.decode_steps_observed = v.decode_steps_observed;
  for (std::size_t l = 0; l < v.num_layers; ++l) {
    Tensor k({n, kv}), vv({n, kv});
    std::copy(v.k_pre[l], v.k_pre[l] + n * kv, k.data.begin());
    std::copy(v.v[l], v.v[l] + n * kv, vv.data.begin());
    c.k_pre.push_back(std::move(k));
    c.v.push_back(std::move(vv));
  }
  c.hidden_snapshot = Tensor({n, v.d_model});
  std::copy(v.hidden_snapshot, v.hidden_snapshot + n * v.d_model, c.hidden_snapshot.data.begin());
  c.influence.assign(v.influence, v.influence + n);
  rk_cache_file_free(f);
  return c;
}
}  // namespace

std::vector<std::uint8_t> export_relay_cache(const RelayCache& cache) {
  const CacheView v(cache);  // validates (relay_cache.cpp:177)
  uint64_t size = 0;
  check(rk_cache_file_encode(&v.view, nullptr, 0, &size));
  std::vector<std::uint8_t> out(size);
  check(rk_cache_file_encode(&v.view, out.data(), out.size(), &size));
  return out;
}

RelayCache import_relay_cache(std::vector<std::uint8_t> bytes) {
  rk_cache_file* f = nullptr;
  rk_relay_cache_view v{};
  check(rk_cache_file_decode(bytes.data(), bytes.size(), &f, &v));
  return take_file(f, v);
}

void save_relay_cache(const RelayCache& cache, const std::filesystem::path& path) {
  const CacheView v(cache);
  check(rk_cache_file_write(&v.view, path.c_str()));
}

RelayCache load_relay_cache(const std::filesystem::path& path) {
  rk_cache_file* f = nullptr;
  rk_relay_cache_view v{};
  check(rk_cache_file_read(path.c_str(), &f, &v));
  return take_file(f, v);
}

RelayCache capture_relay_cache(const Weights& w, std::span<const TokenId> prompt, std::size_t n,
                               std::size_t snapshot_layer, KVContext* decode_ctx) {
  KVContext local(w.spec);
  KVContext& ctx = decode_ctx ? *decode_ctx : local;
  ctx = KVContext(w.spec);
  std::vector<float> last(w.spec.vocab_size);
  if (prompt.empty()) throw std::invalid_argument("prefill: empty token chunk");
  check(rk_prefill(engine(), device_weights(w).get(), ctx.handle(w), prompt.data(), prompt.size(), 0, last.data()));
  rk_cache* c = nullptr;
  check(rk_cache_capture_decode(engine(), device_weights(w).get(), ctx.handle(w), last.data(), n, snapshot_layer, 0,
                                &c));
  ctx.invalidate();
  RelayCache out;
  const ModelSpec& s = w.spec;
  out.num_kv_heads = s.num_kv_heads;
  out.d_head = s.d_head;
  out.d_model = s.d_model;
  out.theta_base = s.theta_base;
  out.max_positions = s.max_positions;
  out.segment_tokens.resize(n);
  out.k_pre.assign(s.num_layers, Tensor({n, s.kv_dim()}));
  out.v.assign(s.num_layers, Tensor({n, s.kv_dim()}));
  out.hidden_snapshot = Tensor({n, s.d_model});
  out.influence.resize(n);
  std::vector<float*> kp, vp;
  for (std::size_t l = 0; l < s.num_layers; ++l) {
    kp.push_back(out.k_pre[l].data.data());
    vp.push_back(out.v[l].data.data());
  }
  uint64_t src = 0, snap = 0;
  const int st = rk_cache_export(c, out.segment_tokens.data(), kp.data(), vp.data(), out.hidden_snapshot.data.data(),
                                 out.influence.data(), &src, &snap);
  rk_cache_destroy(c);
  check(st);
  out.source_base_position = src;
  out.snapshot_layer = snap;
  out.decode_steps_observed = n;
  return out;
}

// ---- selection / profile / marks ------------------------------------------------
void SelectionThresholds::validate() const {
  if (!(tau_dev > 0.0)) throw std::invalid_argument("thresholds: tau_dev must be > 0");
  if (!(tau_inf > 0.0)) throw std::invalid_argument("thresholds: tau_inf must be > 0");
}
bool SelectionSet::contains(std::size_t idx) const { return std::binary_search(indices.begin(), indices.end(), idx); }
std::size_t SelectionSet::count_tag(unsigned tag) const {
  std::size_t n = 0;
  for (unsigned t : tags) n += (t & tag) != 0;
  return n;
}
void LayerProfile::validate(std::size_t num_layers) const {
  if (!(l_start <= l_det && l_det <= l_end && l_end < num_layers))
    throw SchemaError("layer profile violates l_start <= l_det <= l_end < num_layers (" + std::to_string(l_start) +
                      ", " + std::to_string(l_det) + ", " + std::to_string(l_end) + ") for " +
                      std::to_string(num_layers) + " layers");
}
std::size_t SegmentMarks::recomputed() const {
  return static_cast<std::size_t>(std::count(origin.begin(), origin.end(), CellOrigin::kRecomputed));
}

// ---- relay ------------------------------------------------------------------------
RelayOutput relay_extend(const Weights& w, MergedKVContext& ctx, const RelayCache& cache, const LayerProfile& profile,
                         const RelayOptions& opts) {
  cache.validate_for(w.spec);  // relay_engine.cpp:186
  auto dw = device_weights(w);
  rk_context* c = ctx.kv.handle(w);
  CacheUpload up(cache, dw.get());
  OutBufs b(cache.segment_len(), w.spec);
  const rk_layer_profile p{profile.l_start, profile.l_det, profile.l_end};
  const rk_relay_options o = to_c(opts);
  check(rk_relay_extend(engine(), dw.get(), c, up.dev, &p, &o, &b.out));
  ctx.kv.invalidate();
  ctx.segments.push_back(b.marks());
  return b.to_output();
}

RelayPrefillResult relay_prefill(const Weights& w, std::span<const TokenId> prefix, const RelayCache& cache,
                                 const LayerProfile& profile, const RelayOptions& opts) {
  cache.validate_for(w.spec);
  auto dw = device_weights(w);
  RelayPrefillResult r;
  r.ctx.kv = KVContext(w.spec);
  rk_context* c = r.ctx.kv.handle(w);
  CacheUpload up(cache, dw.get());
  OutBufs b(cache.segment_len(), w.spec);
  const rk_layer_profile p{profile.l_start, profile.l_det, profile.l_end};
  const rk_relay_options o = to_c(opts);
  r.segment_end_logits = Tensor({1, w.spec.vocab_size});
  check(rk_relay_prefill(engine(), dw.get(), c, prefix.data(), prefix.size(), up.dev, &p, &o, &b.out,
                         r.segment_end_logits.data.data()));
  r.ctx.kv.invalidate();
  r.ctx.segments.push_back(b.marks());
  r.segment = b.to_output();
  return r;
}

RelayPrefillResult blend_baseline(const Weights& w, std::span<const TokenId> prefix, const RelayCache& cache,
                                  double alpha) {
  RelayOptions opts;
  opts.mode = RelayMode::kBlend;
  opts.blend_alpha = alpha;
  return relay_prefill(w, prefix, cache, LayerProfile{}, opts);
}

// ---- FLOP model (relay_engine.cpp:72-128) -------------------------------------------
double flops_proj_mlp_per_token_layer(const ModelSpec& spec) {
  const double d = (double)spec.d_model, kv = (double)spec.kv_dim(), ff = (double)spec.d_ff;
  return 2.0 * d * (2.0 * d + 2.0 * kv) + 6.0 * d * ff;
}
double flops_attn_term(const ModelSpec& spec, std::size_t base, std::size_t n) {
  const double b = (double)base, nn = (double)n, dhH = (double)(spec.d_head * spec.num_heads);
  return 4.0 * dhH * (nn * b + nn * (nn + 1.0) / 2.0);
}
double flops_span_full(const ModelSpec& spec, std::size_t base, std::size_t n) {
  const rk_model_spec s = to_c(spec);
  return rk_flops_span_full(&s, base, n);
}
double flops_segment_schedule(const ModelSpec& spec, std::size_t base, std::size_t n, std::size_t lo, std::size_t hi,
                              std::size_t sparse_hi, std::size_t selected) {
  const rk_model_spec s = to_c(spec);
  return rk_flops_segment_schedule(&s, base, n, lo, hi, sparse_hi, selected);
}
double flops_selection_overhead(const ModelSpec& spec, std::size_t n) {
  const double nn = (double)n, kv = (double)spec.kv_dim();
  return nn * (6.0 * kv + 10.0) + 4.0 * nn;
}
double flops_realign_cost(const ModelSpec& spec, std::size_t n) {
  return 3.0 * (double)spec.kv_dim() * (double)n * (double)spec.num_layers;
}
FlopEstimate flops_estimate(const ModelSpec& spec, std::size_t prefix_len, std::size_t segment_len,
                            const LayerProfile& profile, std::size_t selected_count) {
  profile.validate(spec.num_layers);
  FlopEstimate est;
  est.relay = flops_span_full(spec, 0, prefix_len) +
              flops_segment_schedule(spec, prefix_len, segment_len, profile.l_start, profile.l_det, profile.l_end,
                                     selected_count);
  est.selection = flops_selection_overhead(spec, segment_len);
  est.realign = flops_realign_cost(spec, segment_len);
  est.full_equiv = flops_span_full(spec, 0, prefix_len + segment_len);
  return est;
}

}  // namespace relaykv
