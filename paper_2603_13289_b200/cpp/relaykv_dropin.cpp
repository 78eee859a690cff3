// relaykv_dropin.cpp -- the reference's relay-prefill C++ API over the C ABI.
// See include/relaykv/relay_engine.hpp for the mapping and the two deliberate
// differences. Error statuses are re-thrown as the reference's exception
// types.
#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>

#include "relaykv/relay_engine.hpp"
#include "relaykv_b200.h"

namespace relaykv {
namespace {

std::mutex g_mu;
int g_device = 0;
Precision g_prec = Precision::kFp32Exact;
std::map<int, rk_engine*> g_engines;
struct WeightsKey {
  std::string id;
  const float* emb;
  int prec;
  bool operator<(const WeightsKey& o) const {
    return std::tie(id, emb, prec) < std::tie(o.id, o.emb, o.prec);
  }
};
std::map<WeightsKey, rk_weights*> g_weights;

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

rk_weights* device_weights(const Weights& w) {
  rk_engine* e = engine();
  const WeightsKey key{w.model_id, w.embedding.data.data(), (int)g_prec};
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = g_weights.find(key);
    if (it != g_weights.end()) return it->second;
  }
  const rk_model_spec s = to_c(w.spec);
  const std::size_t n = rk_weights_num_tensors(&s);
  std::vector<const float*> ptrs(n);
  for (std::size_t i = 0; i < n; ++i) ptrs[i] = tensor_at(w, i).data.data();
  rk_weights* dw = nullptr;
  check(rk_weights_upload(e, &s, ptrs.data(), n, (int)g_prec, &dw));
  std::lock_guard<std::mutex> lock(g_mu);
  g_weights[key] = dw;
  return dw;
}

struct CacheView {
  std::vector<const float*> kp, vp;
  rk_relay_cache_view view{};
  explicit CacheView(const RelayCache& c) {
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

struct CacheUpload : CacheView {
  rk_cache* dev = nullptr;
  CacheUpload(const RelayCache& c, rk_weights* w) : CacheView(c) { check(rk_cache_upload(engine(), w, &view, &dev)); }
  ~CacheUpload() { rk_cache_destroy(dev); }
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

Weights init_weights(const ModelSpec& spec, std::uint64_t seed) {
  spec.validate();
  const rk_model_spec s = to_c(spec);
  rk_weights* dw = nullptr;
  check(rk_weights_init(engine(), &s, seed, RK_FP32_EXACT, &dw));
  Weights w;
  w.spec = spec;
  w.model_id = spec.summary_id(seed);
  const std::size_t d = spec.d_model, q = spec.q_dim(), kv = spec.kv_dim(), ff = spec.d_ff, V = spec.vocab_size;
  auto fetch = [&](std::size_t idx, std::vector<std::size_t> shape) {
    Tensor t(std::move(shape));
    check(rk_weights_export(dw, idx, t.data.data(), t.data.size()));
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
  if (g_prec == Precision::kFp32Exact) {  // keep the device copy we already have
    std::lock_guard<std::mutex> lock(g_mu);
    g_weights[WeightsKey{w.model_id, w.embedding.data.data(), (int)g_prec}] = dw;
  } else {
    rk_weights_destroy(dw);
  }
  return w;
}

// ---- KVContext --------------------------------------------------------------
KVContext::KVContext(const ModelSpec& spec) : spec_(spec) {}
KVContext::KVContext(const KVContext& o) : spec_(o.spec_) {
  if (o.ctx_) {
    rk_context* c = nullptr;
    check(rk_context_clone(o.ctx_.get(), &c));
    ctx_.reset(c, rk_context_destroy);
  }
}
KVContext& KVContext::operator=(const KVContext& o) {
  if (this != &o) {
    KVContext tmp(o);
    spec_ = tmp.spec_;
    ctx_ = tmp.ctx_;
    invalidate();
  }
  return *this;
}
std::size_t KVContext::size() const { return ctx_ ? rk_context_size(ctx_.get()) : 0; }
rk_context* KVContext::handle(const Weights& w) {
  if (!ctx_) {
    spec_ = w.spec;
    rk_context* c = nullptr;
    check(rk_context_create(engine(), device_weights(w), &c));
    ctx_.reset(c, rk_context_destroy);
  }
  invalidate();
  return ctx_.get();
}
void KVContext::fetch() const {
  if (!mirror_k_.empty() || !ctx_) return;
  const std::size_t n = size(), w = spec_.kv_dim();
  mirror_k_.assign(spec_.num_layers, std::vector<float>(n * w));
  mirror_v_.assign(spec_.num_layers, std::vector<float>(n * w));
  for (std::size_t l = 0; l < spec_.num_layers; ++l)
    check(rk_context_export(ctx_.get(), l, 0, n, mirror_k_[l].data(), mirror_v_[l].data()));
}
std::span<const float> KVContext::key_row(std::size_t layer, std::size_t pos) const {
  fetch();
  return {mirror_k_[layer].data() + pos * spec_.kv_dim(), spec_.kv_dim()};
}
std::span<const float> KVContext::value_row(std::size_t layer, std::size_t pos) const {
  fetch();
  return {mirror_v_[layer].data() + pos * spec_.kv_dim(), spec_.kv_dim()};
}

PrefillResult prefill(const Weights& w, std::span<const TokenId> tokens, KVContext& ctx, std::size_t base) {
  PrefillResult r;
  r.logits = Tensor({1, w.spec.vocab_size});
  check(rk_prefill(engine(), device_weights(w), ctx.handle(w), tokens.data(), tokens.size(), base,
                   r.logits.data.data()));
  return r;
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
  const CacheView v(cache);
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
  const PrefillResult p = prefill(w, prompt, ctx, 0);
  rk_cache* c = nullptr;
  check(rk_cache_capture_decode(engine(), device_weights(w), ctx.handle(w), p.logits.data.data(), n,
                                snapshot_layer, 0, &c));
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

void SelectionThresholds::validate() const {
  if (!(tau_dev > 0.0)) throw std::invalid_argument("thresholds: tau_dev must be > 0");
  if (!(tau_inf > 0.0)) throw std::invalid_argument("thresholds: tau_inf must be > 0");
}
bool SelectionSet::contains(std::size_t idx) const {
  return std::binary_search(indices.begin(), indices.end(), idx);
}
std::size_t SelectionSet::count_tag(unsigned tag) const {
  std::size_t n = 0;
  for (unsigned t : tags) n += (t & tag) != 0;
  return n;
}
void LayerProfile::validate(std::size_t num_layers) const {
  if (!(l_start <= l_det && l_det <= l_end && l_end < num_layers))
    throw SchemaError("layer profile violates l_start <= l_det <= l_end < num_layers");
}
std::size_t SegmentMarks::recomputed() const {
  return static_cast<std::size_t>(std::count(origin.begin(), origin.end(), CellOrigin::kRecomputed));
}

RelayOutput relay_extend(const Weights& w, MergedKVContext& ctx, const RelayCache& cache,
                         const LayerProfile& profile, const RelayOptions& opts) {
  rk_weights* dw = device_weights(w);
  CacheUpload up(cache, dw);
  OutBufs b(cache.segment_len(), w.spec);
  const rk_layer_profile p{profile.l_start, profile.l_det, profile.l_end};
  const rk_relay_options o = to_c(opts);
  check(rk_relay_extend(engine(), dw, ctx.kv.handle(w), up.dev, &p, &o, &b.out));
  ctx.segments.push_back(b.marks());
  return b.to_output();
}

RelayPrefillResult relay_prefill(const Weights& w, std::span<const TokenId> prefix, const RelayCache& cache,
                                 const LayerProfile& profile, const RelayOptions& opts) {
  rk_weights* dw = device_weights(w);
  CacheUpload up(cache, dw);
  OutBufs b(cache.segment_len(), w.spec);
  const rk_layer_profile p{profile.l_start, profile.l_det, profile.l_end};
  const rk_relay_options o = to_c(opts);
  RelayPrefillResult r;
  r.ctx.kv = KVContext(w.spec);
  r.segment_end_logits = Tensor({1, w.spec.vocab_size});
  check(rk_relay_prefill(engine(), dw, r.ctx.kv.handle(w), prefix.data(), prefix.size(), up.dev, &p, &o, &b.out,
                         r.segment_end_logits.data.data()));
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

double flops_span_full(const ModelSpec& spec, std::size_t base, std::size_t n) {
  const rk_model_spec s = to_c(spec);
  return rk_flops_span_full(&s, base, n);
}
double flops_segment_schedule(const ModelSpec& spec, std::size_t base, std::size_t n, std::size_t lo,
                              std::size_t hi, std::size_t sparse_hi, std::size_t selected) {
  const rk_model_spec s = to_c(spec);
  return rk_flops_segment_schedule(&s, base, n, lo, hi, sparse_hi, selected);
}

}  // namespace relaykv
