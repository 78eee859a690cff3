// ref_capi.cpp -- C ABI harness over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY. Linked (by oracle/Makefile) against the reference
// sources compiled where they lie under /root/reference/proj/src into
// oracle/_ref/librelaykv_ref.so. Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg and --impl reference) load it, as the checker /
// the reference CPU arm, never as the product path.
//
// Every entry point calls the reference's own public API; the only code here
// that is not a call into the reference is (a) the unchecked init mirror for
// specs the reference's ModelSpec::validate() rejects (num_layers < 6,
// model.cpp:21) -- pinned bit-equal to init_weights for num_layers >= 6 by
// tests/test_oracle_pins.py -- and (b) marshalling between the reference's
// structs and the rk_* plain-C structs of include/relaykv_b200.h.

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "relaykv/errors.hpp"
#include "relaykv/metrics.hpp"
#include "relaykv/model.hpp"
#include "relaykv/profiler.hpp"
#include "relaykv/relay_cache.hpp"
#include "relaykv/relay_engine.hpp"
#include "relaykv/selector.hpp"
#include "relaykv_b200.h"

using namespace relaykv;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return RK_OK;
  } catch (const SchemaError& e) {
    g_err = e.what();
    return RK_ERR_SCHEMA;
  } catch (const IoError& e) {
    g_err = e.what();
    return RK_ERR_IO;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RK_ERR_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return RK_ERR_LOGIC;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return std::string(e.what()).find("non-finite") != std::string::npos ? RK_ERR_NONFINITE
                                                                           : RK_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RK_ERR_RUNTIME;
  }
}

ModelSpec to_spec(const rk_model_spec& s) {
  ModelSpec m;
  m.num_layers = s.num_layers;
  m.d_model = s.d_model;
  m.num_heads = s.num_heads;
  m.num_kv_heads = s.num_kv_heads;
  m.d_head = s.d_head;
  m.d_ff = s.d_ff;
  m.vocab_size = s.vocab_size;
  m.theta_base = s.theta_base;
  m.max_positions = s.max_positions;
  m.norm_eps = s.norm_eps;
  return m;
}

// Unchecked mirror of init_weights (model.cpp:81-114) minus spec.validate()
// (model.cpp:82). Same SplitMix64 stream (model.cpp:49-62), same draw order.
struct Mix {
  std::uint64_t state;
  std::uint64_t next() {
    std::uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  float symmetric() {
    const float u = static_cast<float>(next() >> 40) * 0x1p-24f;
    return 2.0f * u - 1.0f;
  }
};

Tensor uniform(Mix& rng, std::vector<std::size_t> shape, float sd) {
  Tensor t(std::move(shape));
  const float scale = sd * 1.7320508f;
  for (float& v : t.data) v = rng.symmetric() * scale;
  return t;
}

Tensor ones(std::vector<std::size_t> shape) {
  Tensor t(std::move(shape));
  for (float& v : t.data) v = 1.0f;
  return t;
}

Weights init_unchecked(const ModelSpec& spec, std::uint64_t seed) {
  Mix rng{seed ^ 0x72656c6179ull};
  Weights w;
  w.spec = spec;
  w.model_id = spec.summary_id(seed);
  w.embedding = uniform(rng, {spec.vocab_size, spec.d_model}, 0.02f);
  const float d_in = 1.0f / std::sqrt(static_cast<float>(spec.d_model));
  const float ff_in = 1.0f / std::sqrt(static_cast<float>(spec.d_ff));
  const float q_in = 1.0f / std::sqrt(static_cast<float>(spec.q_dim())) /
                     (2.0f * static_cast<float>(spec.num_layers));
  w.layers.resize(spec.num_layers);
  for (auto& layer : w.layers) {
    layer.attn_norm_gain = ones({spec.d_model});
    layer.w_q = uniform(rng, {spec.d_model, spec.q_dim()}, d_in);
    layer.w_k = uniform(rng, {spec.d_model, spec.kv_dim()}, d_in);
    layer.w_v = uniform(rng, {spec.d_model, spec.kv_dim()}, d_in);
    layer.w_o = uniform(rng, {spec.q_dim(), spec.d_model}, q_in);
    layer.mlp_norm_gain = ones({spec.d_model});
    layer.w_gate = uniform(rng, {spec.d_model, spec.d_ff}, d_in);
    layer.w_up = uniform(rng, {spec.d_model, spec.d_ff}, d_in);
    layer.w_down = uniform(rng, {spec.d_ff, spec.d_model}, ff_in);
  }
  w.final_norm_gain = ones({spec.d_model});
  w.output_head = uniform(rng, {spec.d_model, spec.vocab_size}, d_in);
  return w;
}

// tensor_table order (weights_io.cpp:21-38)
const Tensor& tensor_at(const Weights& w, std::size_t idx) {
  if (idx == 0) return w.embedding;
  idx -= 1;
  const std::size_t per = 9;
  if (idx < w.layers.size() * per) {
    const LayerWeights& l = w.layers[idx / per];
    switch (idx % per) {
      case 0: return l.attn_norm_gain;
      case 1: return l.w_q;
      case 2: return l.w_k;
      case 3: return l.w_v;
      case 4: return l.w_o;
      case 5: return l.mlp_norm_gain;
      case 6: return l.w_gate;
      case 7: return l.w_up;
      default: return l.w_down;
    }
  }
  idx -= w.layers.size() * per;
  if (idx == 0) return w.final_norm_gain;
  return w.output_head;
}

RelayOptions to_opts(const rk_relay_options& o) {
  RelayOptions r;
  r.mode = static_cast<RelayMode>(o.mode == RK_MODE_FULL    ? 0
                                  : o.mode == RK_MODE_ZERO  ? 1
                                  : o.mode == RK_MODE_RELAY ? 2
                                                            : 3);
  r.thresholds.tau_dev = o.tau_dev;
  r.thresholds.tau_inf = o.tau_inf;
  r.thresholds.suffix_k = o.suffix_k;
  r.blend_alpha = o.blend_alpha;
  r.rectify_above_end = o.rectify_above_end != 0;
  return r;
}

LayerProfile to_profile(const rk_layer_profile* p) {
  LayerProfile lp;
  if (p) {
    lp.l_start = p->l_start;
    lp.l_det = p->l_det;
    lp.l_end = p->l_end;
  }
  return lp;
}

void fill_output(const RelayOutput& o, const SegmentMarks& marks, std::size_t L,
                 rk_relay_output* out) {
  if (!out) return;
  const std::size_t n = marks.len;
  out->segment_base = marks.base;
  out->segment_len = n;
  out->selection_count = o.selection.size();
  out->s_dev_len = o.s_dev.size();
  for (std::size_t i = 0; i < o.selection.size(); ++i) {
    if (out->selection_indices) out->selection_indices[i] = o.selection.indices[i];
    if (out->selection_tags) out->selection_tags[i] = o.selection.tags[i];
  }
  for (std::size_t j = 0; j < o.s_dev.size(); ++j) {
    if (out->s_dev) out->s_dev[j] = o.s_dev[j];
    if (out->s_key_dev) out->s_key_dev[j] = o.s_key_dev[j];
  }
  if (out->segment_hidden)
    std::memcpy(out->segment_hidden, o.segment_hidden.data.data(),
                o.segment_hidden.data.size() * sizeof(float));
  if (out->hidden_depth)
    for (std::size_t j = 0; j < o.hidden_depth.size(); ++j) out->hidden_depth[j] = o.hidden_depth[j];
  if (out->origin)
    for (std::size_t i = 0; i < L * n; ++i) out->origin[i] = static_cast<uint8_t>(marks.origin[i]);
  const ReuseStats& s = o.stats;
  rk_reuse_stats& r = out->stats;
  r.total_entries = s.total_entries;
  r.recomputed_entries = s.recomputed_entries;
  r.reuse_rate = s.reuse_rate;
  r.selected_count = s.selected_count;
  r.selected_deviation = s.selected_deviation;
  r.selected_influence_score = s.selected_influence_score;
  r.selected_influence_suffix = s.selected_influence_suffix;
  r.selected_blend = s.selected_blend;
  r.flops_cost = s.flops_cost;
  r.flops_selection = s.flops_selection;
  r.flops_realign = s.flops_realign;
  r.flops_full_equiv = s.flops_full_equiv;
  r.wall = {s.wall.fresh_ms, s.wall.realign_ms, s.wall.recompute_ms,
            s.wall.selection_ms, s.wall.rectify_ms, s.wall.total_ms};
}

struct RefCtx {
  MergedKVContext ctx;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// checked != 0: the reference's own init_weights (validates the spec).
int ref_weights_create(const rk_model_spec* spec, uint64_t seed, int checked, void** out) {
  return guard([&] {
    const ModelSpec s = to_spec(*spec);
    *out = new Weights(checked ? init_weights(s, seed) : init_unchecked(s, seed));
  });
}
void ref_weights_destroy(void* w) { delete static_cast<Weights*>(w); }
// Build reference Weights from host tensors in tensor_table order.
int ref_weights_from_tensors(const rk_model_spec* spec, const float* const* tensors, void** out) {
  return guard([&] {
    const ModelSpec s = to_spec(*spec);
    auto* w = new Weights(init_unchecked(s, 0));
    const std::size_t count = 1 + 9 * s.num_layers + 2;
    for (std::size_t i = 0; i < count; ++i) {
      Tensor& t = const_cast<Tensor&>(tensor_at(*w, i));
      std::memcpy(t.data.data(), tensors[i], t.data.size() * sizeof(float));
    }
    *out = w;
  });
}
const float* ref_weights_tensor(void* w, uint64_t idx, uint64_t* numel) {
  const Tensor& t = tensor_at(*static_cast<Weights*>(w), idx);
  if (numel) *numel = t.data.size();
  return t.data.data();
}

// ---- relay caches -------------------------------------------------------
// Decode-with-capture scenario exactly as the reference tests build it
// (test_engine.cpp:43-62): prefill old_prefix, greedy-decode segment_len
// tokens with RelayRecorder at snapshot_layer. Returns a RelayCache*.
// decode_ctx_out (optional) receives the decode-time context.
int ref_scenario_create(void* w, const int32_t* old_prefix, uint64_t n_prefix,
                        uint64_t segment_len, uint64_t snapshot_layer, int include_self,
                        void** cache_out, void** decode_ctx_out) {
  return guard([&] {
    const Weights& W = *static_cast<Weights*>(w);
    auto ctx = std::make_unique<RefCtx>();
    ctx->ctx.kv = KVContext(W.spec);
    std::vector<TokenId> pre(old_prefix, old_prefix + n_prefix);
    const PrefillResult p = prefill(W, pre, ctx->ctx.kv, 0);
    CaptureFlags cap;
    cap.hidden = cap.pre_rope_keys = cap.attention = true;
    RelayRecorder rec(W.spec, n_prefix, snapshot_layer, include_self != 0);
    const StepHook hook = [&](const StepTrace& tr, TokenId tok, std::size_t pos) {
      rec.feed(tr, tok, pos);
    };
    greedy_generate(W, ctx->ctx.kv, p.logits.row(n_prefix - 1), segment_len, cap, hook);
    *cache_out = new RelayCache(rec.finalize());
    if (decode_ctx_out) *decode_ctx_out = ctx.release();
  });
}
int ref_cache_from_view(const rk_relay_cache_view* v, void** out) {
  return guard([&] {
    auto* c = new RelayCache();
    c->num_kv_heads = v->num_kv_heads;
    c->d_head = v->d_head;
    c->d_model = v->d_model;
    c->theta_base = v->theta_base;
    c->max_positions = v->max_positions;
    c->segment_tokens.assign(v->segment_tokens, v->segment_tokens + v->segment_len);
    c->source_base_position = v->source_base_position;
    c->snapshot_layer = v->snapshot_layer;
    c->decode_steps_observed = v->decode_steps_observed;
    const std::size_t n = v->segment_len, kv = v->num_kv_heads * v->d_head;
    for (std::size_t l = 0; l < v->num_layers; ++l) {
      Tensor k({n, kv}), vv({n, kv});
      std::memcpy(k.data.data(), v->k_pre[l], n * kv * sizeof(float));
      std::memcpy(vv.data.data(), v->v[l], n * kv * sizeof(float));
      c->k_pre.push_back(std::move(k));
      c->v.push_back(std::move(vv));
    }
    c->hidden_snapshot = Tensor({n, v->d_model});
    std::memcpy(c->hidden_snapshot.data.data(), v->hidden_snapshot, n * v->d_model * sizeof(float));
    c->influence.assign(v->influence, v->influence + n);
    *out = c;
  });
}
void ref_cache_destroy(void* c) { delete static_cast<RelayCache*>(c); }
// View into the cache's storage; k_ptrs/v_ptrs: caller arrays of L pointers.
int ref_cache_view(void* c, rk_relay_cache_view* v, const float** k_ptrs, const float** v_ptrs) {
  const RelayCache& C = *static_cast<RelayCache*>(c);
  v->num_layers = C.num_layers();
  v->num_kv_heads = C.num_kv_heads;
  v->d_head = C.d_head;
  v->d_model = C.d_model;
  v->theta_base = C.theta_base;
  v->max_positions = C.max_positions;
  v->segment_len = C.segment_len();
  v->segment_tokens = C.segment_tokens.data();
  v->source_base_position = C.source_base_position;
  v->snapshot_layer = C.snapshot_layer;
  v->decode_steps_observed = C.decode_steps_observed;
  for (std::size_t l = 0; l < C.num_layers(); ++l) {
    k_ptrs[l] = C.k_pre[l].data.data();
    v_ptrs[l] = C.v[l].data.data();
  }
  v->k_pre = k_ptrs;
  v->v = v_ptrs;
  v->hidden_snapshot = C.hidden_snapshot.data.data();
  v->influence = C.influence.data();
  return RK_OK;
}
// save_relay_cache / load_relay_cache (relay_cache.cpp:238-253).
int ref_cache_save(void* c, const char* path) {
  return guard([&] { save_relay_cache(*static_cast<RelayCache*>(c), path); });
}
int ref_cache_load(const char* path, void** out) {
  return guard([&] { *out = new RelayCache(load_relay_cache(path)); });
}
// realign (relay_cache.cpp:154-174) of every layer into out[L][n x kv].
int ref_realign(void* c, uint64_t base, float* const* out) {
  return guard([&] {
    const RealignedKeys k = realign(*static_cast<RelayCache*>(c), base);
    for (std::size_t l = 0; l < k.k.size(); ++l)
      std::memcpy(out[l], k.k[l].data.data(), k.k[l].data.size() * sizeof(float));
  });
}

// ---- contexts and the hot path -----------------------------------------
int ref_ctx_create(void* w, void** out) {
  return guard([&] {
    auto* c = new RefCtx();
    c->ctx.kv = KVContext(static_cast<Weights*>(w)->spec);
    *out = c;
  });
}
int ref_ctx_clone(void* c, void** out) {
  return guard([&] { *out = new RefCtx(*static_cast<RefCtx*>(c)); });
}
void ref_ctx_destroy(void* c) { delete static_cast<RefCtx*>(c); }
uint64_t ref_ctx_size(void* c) { return static_cast<RefCtx*>(c)->ctx.kv.size(); }
uint64_t ref_ctx_num_segments(void* c) { return static_cast<RefCtx*>(c)->ctx.segments.size(); }
int ref_ctx_segment(void* c, uint64_t i, uint64_t* base, uint64_t* len, uint8_t* origin) {
  const RefCtx& C = *static_cast<RefCtx*>(c);
  if (i >= C.ctx.segments.size()) return RK_ERR_INVALID_ARGUMENT;
  const SegmentMarks& m = C.ctx.segments[i];
  *base = m.base;
  *len = m.len;
  if (origin)
    for (std::size_t k = 0; k < m.origin.size(); ++k) origin[k] = static_cast<uint8_t>(m.origin[k]);
  return RK_OK;
}
int ref_ctx_export(void* c, uint64_t layer, uint64_t pos, uint64_t count, float* k, float* v) {
  const KVContext& kv = static_cast<RefCtx*>(c)->ctx.kv;
  if (layer >= kv.num_layers() || pos + count > kv.size()) return RK_ERR_INVALID_ARGUMENT;
  const std::size_t w = kv.kv_dim();
  for (std::size_t i = 0; i < count; ++i) {
    if (k) std::memcpy(k + i * w, kv.key_row(layer, pos + i).data(), w * sizeof(float));
    if (v) std::memcpy(v + i * w, kv.value_row(layer, pos + i).data(), w * sizeof(float));
  }
  return RK_OK;
}

// prefill (model.cpp:305-331); last_logits: last row [V] or NULL.
int ref_prefill(void* w, void* ctx, const int32_t* tokens, uint64_t n, uint64_t base,
                float* last_logits) {
  return guard([&] {
    const Weights& W = *static_cast<Weights*>(w);
    std::vector<TokenId> t(tokens, tokens + n);
    const PrefillResult r = prefill(W, t, static_cast<RefCtx*>(ctx)->ctx.kv, base);
    if (last_logits && n > 0)
      std::memcpy(last_logits, r.logits.row(n - 1).data(), W.spec.vocab_size * sizeof(float));
  });
}

int ref_relay_extend(void* w, void* ctx, void* cache, const rk_layer_profile* prof,
                     const rk_relay_options* opts, rk_relay_output* out) {
  return guard([&] {
    const Weights& W = *static_cast<Weights*>(w);
    RefCtx& C = *static_cast<RefCtx*>(ctx);
    const RelayOutput o = relay_extend(W, C.ctx, *static_cast<RelayCache*>(cache),
                                       to_profile(prof), to_opts(*opts));
    fill_output(o, C.ctx.segments.back(), W.spec.num_layers, out);
  });
}

// relay_prefill (relay_engine.cpp:363-395); returns the merged ctx as a new handle.
int ref_relay_prefill(void* w, const int32_t* prefix, uint64_t n_prefix, void* cache,
                      const rk_layer_profile* prof, const rk_relay_options* opts,
                      rk_relay_output* out, float* end_logits, void** ctx_out) {
  return guard([&] {
    const Weights& W = *static_cast<Weights*>(w);
    std::vector<TokenId> p(prefix, prefix + n_prefix);
    RelayPrefillResult r = relay_prefill(W, p, *static_cast<RelayCache*>(cache),
                                         to_profile(prof), to_opts(*opts));
    fill_output(r.segment, r.ctx.segments.back(), W.spec.num_layers, out);
    if (end_logits)
      std::memcpy(end_logits, r.segment_end_logits.data.data(), W.spec.vocab_size * sizeof(float));
    if (ctx_out) {
      auto* c = new RefCtx();
      c->ctx = std::move(r.ctx);
      *ctx_out = c;
    }
  });
}

// row_logits_from_layer (model.cpp:339-362).
int ref_row_logits_from_layer(void* w, const float* hidden_row, uint64_t first_layer, void* ctx,
                              uint64_t position, float* logits) {
  return guard([&] {
    const Weights& W = *static_cast<Weights*>(w);
    const Tensor t = row_logits_from_layer(
        W, std::span<const float>(hidden_row, W.spec.d_model), first_layer,
        static_cast<RefCtx*>(ctx)->ctx.kv, position);
    std::memcpy(logits, t.data.data(), W.spec.vocab_size * sizeof(float));
  });
}

// The downstream agent's TTFT sequence, written with the reference's public
// functions exactly as run_workflow's relay branch calls them
// (workflow.cpp:316-369); FULL = workflow.cpp:301-315.
int ref_agent_prefill(void* w, void* ctx, const int32_t* prefix, uint64_t n_prefix,
                      void* const* caches, uint64_t n_up, const int32_t* suffix,
                      uint64_t n_suffix, const rk_layer_profile* prof,
                      const rk_relay_options* opts, float* end_logits, int32_t* first_token) {
  return guard([&] {
    const Weights& W = *static_cast<Weights*>(w);
    const ModelSpec& ms = W.spec;
    RefCtx& C = *static_cast<RefCtx*>(ctx);
    std::vector<float> logits;
    std::vector<TokenId> pre(prefix, prefix + n_prefix), suf(suffix, suffix + n_suffix);
    if (opts->mode == RK_MODE_FULL) {
      std::vector<TokenId> full = pre;
      for (std::size_t u = 0; u < n_up; ++u) {
        const auto& t = static_cast<RelayCache*>(caches[u])->segment_tokens;
        full.insert(full.end(), t.begin(), t.end());
      }
      full.insert(full.end(), suf.begin(), suf.end());
      const PrefillResult pr = prefill(W, full, C.ctx.kv, 0);
      const auto row = pr.logits.row(full.size() - 1);
      logits.assign(row.begin(), row.end());
    } else {
      prefill(W, pre, C.ctx.kv, 0);
      const LayerProfile lp = to_profile(prof);
      const RelayOptions ro = to_opts(*opts);
      RelayOutput last_seg;
      for (std::size_t u = 0; u < n_up; ++u)
        last_seg = relay_extend(W, C.ctx, *static_cast<RelayCache*>(caches[u]), lp, ro);
      if (n_suffix > 0) {
        const std::size_t base = C.ctx.kv.size();
        const PrefillResult sr = prefill(W, suf, C.ctx.kv, base);
        const auto row = sr.logits.row(n_suffix - 1);
        logits.assign(row.begin(), row.end());
      } else {
        const std::size_t n = last_seg.hidden_depth.size();
        const std::size_t depth = last_seg.hidden_depth[n - 1];
        const std::size_t pos = C.ctx.kv.size() - 1;
        Tensor lg;
        if (depth >= ms.num_layers) {
          Tensor last({1, ms.d_model});
          std::memcpy(last.row(0).data(), last_seg.segment_hidden.row(n - 1).data(),
                      ms.d_model * sizeof(float));
          lg = output_logits(W, last);
        } else {
          lg = row_logits_from_layer(W, last_seg.segment_hidden.row(n - 1), depth, C.ctx.kv, pos);
        }
        logits.assign(lg.data.begin(), lg.data.end());
      }
    }
    if (end_logits) std::memcpy(end_logits, logits.data(), logits.size() * sizeof(float));
    if (first_token) *first_token = static_cast<int32_t>(argmax(logits));
  });
}

// Throughput harness for the reference CPU arm: `threads` independent
// sessions (the reference's only parallelism), each running the
// agent sequence above on its own context; weights and caches are shared
// read-only. Returns wall milliseconds for all sessions.
int ref_agent_prefill_parallel(void* w, uint64_t threads, const int32_t* prefix, uint64_t n_prefix,
                               void* const* caches, uint64_t n_up, const int32_t* suffix,
                               uint64_t n_suffix, const rk_layer_profile* prof,
                               const rk_relay_options* opts, int32_t* first_tokens,
                               double* wall_ms) {
  std::vector<int> status(threads, RK_OK);
  std::vector<std::string> errs(threads);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (std::size_t t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      void* ctx = nullptr;
      status[t] = ref_ctx_create(w, &ctx);
      if (status[t] == RK_OK)
        status[t] = ref_agent_prefill(w, ctx, prefix, n_prefix, caches, n_up, suffix, n_suffix,
                                      prof, opts, nullptr, first_tokens ? first_tokens + t : nullptr);
      if (status[t] != RK_OK) errs[t] = g_err;
      ref_ctx_destroy(ctx);
    });
  }
  for (auto& th : pool) th.join();
  *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  for (std::size_t t = 0; t < threads; ++t)
    if (status[t] != RK_OK) {
      g_err = errs[t];
      return status[t];
    }
  return RK_OK;
}

// Analytic FLOP model pass-throughs (relay_engine.cpp:72-128).
double ref_flops_span_full(const rk_model_spec* s, uint64_t base, uint64_t n) {
  return flops_span_full(to_spec(*s), base, n);
}
double ref_flops_segment_schedule(const rk_model_spec* s, uint64_t base, uint64_t n, uint64_t lo,
                                  uint64_t hi, uint64_t sparse_hi, uint64_t selected) {
  return flops_segment_schedule(to_spec(*s), base, n, lo, hi, sparse_hi, selected);
}

// libm expf of this host, for checking the device restatement of it.
float ref_host_expf(float x) { return std::exp(x); }

// ---- offline profiler (profiler.cpp:155-175, metrics.cpp:118-238) ----------
namespace {
ProfilerParams to_params(const rk_profiler_params& p) {
  ProfilerParams q;
  q.tau_start = p.tau_start;
  q.tail_layers = p.tail_layers;
  q.stability_lambda = p.stability_lambda;
  q.consecutive = p.consecutive;
  q.min_rise = p.min_rise;
  q.first_negative_alpha = p.first_negative_alpha != 0;
  return q;
}
void put_profile(const LayerProfile& lp, rk_profile_result* out, double* curve_s, double* curve_rho) {
  out->l_start = lp.l_start;
  out->l_det = lp.l_det;
  out->l_end = lp.l_end;
  out->end_fallback = 0;
  out->det_fallback = 0;
  for (const auto& w : lp.warnings) {
    if (w.find("end-layer") != std::string::npos) out->end_fallback = 1;
    if (w.find("detection") != std::string::npos) out->det_fallback = 1;
  }
  if (curve_s) std::copy(lp.curve_s.begin(), lp.curve_s.end(), curve_s);
  if (curve_rho) std::copy(lp.curve_rho.begin(), lp.curve_rho.end(), curve_rho);
}
LayerCurve to_curve(const double* s, const double* rho, const uint8_t* deg, uint64_t L) {
  LayerCurve c;
  c.s.assign(s, s + L);
  c.rho.assign(rho, rho + L);
  for (uint64_t l = 0; l < L; ++l) c.rho_degenerate.push_back(deg[l] != 0);
  return c;
}
}  // namespace

int ref_profile_model(void* w, const rk_two_stage_config* c, const rk_profiler_params* p, rk_profile_result* out,
                      double* curve_s, double* curve_rho) {
  return guard([&] {
    TwoStageConfig cfg;
    cfg.seed = c->seed;
    cfg.instances = c->instances;
    cfg.stage1_prefix_min = c->stage1_prefix_min;
    cfg.stage1_prefix_max = c->stage1_prefix_max;
    cfg.stage2_prefix_min = c->stage2_prefix_min;
    cfg.stage2_prefix_max = c->stage2_prefix_max;
    cfg.segment_len = c->segment_len;
    cfg.stage2_suffix_len = c->stage2_suffix_len;
    cfg.sweep_instances = c->sweep_instances;
    cfg.identical_prefix = c->identical_prefix != 0;
    cfg.snapshot_layer = c->snapshot_layer;
    put_profile(profile_model(*static_cast<Weights*>(w), cfg, to_params(*p)), out, curve_s, curve_rho);
  });
}
// token_deviation of two caches' (k_pre, v); outputs [n x L].
int ref_token_deviation(void* reuse, void* full, double* vc, double* kc, double* vn, double* kn) {
  return guard([&] {
    const RelayCache& a = *static_cast<RelayCache*>(reuse);
    const RelayCache& b = *static_cast<RelayCache*>(full);
    SegmentKV ra{a.k_pre, a.v}, fb{b.k_pre, b.v};
    const DeviationMatrix m = token_deviation(ra, fb, a.num_kv_heads);
    std::copy(m.value_cos.begin(), m.value_cos.end(), vc);
    std::copy(m.key_cos.begin(), m.key_cos.end(), kc);
    std::copy(m.value_norm.begin(), m.value_norm.end(), vn);
    std::copy(m.key_norm.begin(), m.key_norm.end(), kn);
  });
}
int ref_layer_curve(const double* value_cos, uint64_t n, uint64_t L, double* s, double* rho, uint8_t* deg) {
  return guard([&] {
    DeviationMatrix m;
    m.segment_len = n;
    m.num_layers = L;
    m.value_cos.assign(value_cos, value_cos + n * L);
    m.key_cos = m.value_norm = m.key_norm = m.value_cos;
    const LayerCurve c = make_layer_curve(m);
    for (uint64_t l = 0; l < L; ++l) {
      s[l] = c.s[l];
      rho[l] = c.rho[l];
      deg[l] = c.rho_degenerate[l];
    }
  });
}
int ref_profile_from_curve(const double* s, const double* rho, const uint8_t* deg, uint64_t L,
                           const rk_profiler_params* p, rk_profile_result* out, double* curve_rho) {
  return guard([&] { put_profile(profile_from_curve(to_curve(s, rho, deg, L), to_params(*p), "m"), out, nullptr,
                                 curve_rho); });
}
int ref_average_curves(const double* s, const double* rho, const uint8_t* deg, uint64_t k, uint64_t L, double* so,
                       double* ro, uint8_t* dout) {
  return guard([&] {
    std::vector<LayerCurve> cs;
    for (uint64_t i = 0; i < k; ++i) cs.push_back(to_curve(s + i * L, rho + i * L, deg + i * L, L));
    const LayerCurve a = average_curves(cs);
    for (uint64_t l = 0; l < L; ++l) {
      so[l] = a.s[l];
      ro[l] = a.rho[l];
      dout[l] = a.rho_degenerate[l];
    }
  });
}

}  // extern "C"
