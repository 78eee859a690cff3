// test_dropin.cpp -- the reference's relay-engine test scenarios
// (/root/reference/proj/tests/test_engine.cpp:101-324), rewritten against the
// C++ drop-in (paper_2603_13289_b200/cpp) running on the B200, plus a bitwise
// cross-check against the oracle restatement (oracle/build/liboracle.so).
// Built by paper_2603_13289_b200/build.py; run by tests/test_gpu_dropin.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <algorithm>
#include <cmath>
#include <cstring>

#include "relaykv/relay_engine.hpp"
#include "relaykv_b200.h"

using namespace relaykv;

extern "C" {  // oracle restatement (test infrastructure)
struct orc_weights;
struct orc_ctx;
struct orc_cache;
orc_weights* orc_weights_init(const rk_model_spec*, uint64_t);
void orc_weights_destroy(orc_weights*);
orc_ctx* orc_ctx_create(orc_weights*);
void orc_ctx_destroy(orc_ctx*);
int orc_cache_from_view(const rk_relay_cache_view*, orc_cache**);
void orc_cache_destroy(orc_cache*);
int orc_relay_prefill(orc_weights*, orc_ctx*, const int32_t*, uint64_t, orc_cache*, const rk_layer_profile*,
                      const rk_relay_options*, rk_relay_output*, float*);
int orc_ctx_export(orc_ctx*, uint64_t, uint64_t, uint64_t, float*, float*);
}

namespace {

ModelSpec spec_of(std::size_t layers, std::size_t d_model, std::size_t heads) {
  ModelSpec s;
  s.num_layers = layers;
  s.d_model = d_model;
  s.num_heads = heads;
  s.num_kv_heads = heads;
  s.d_head = d_model / heads;
  s.d_ff = 2 * d_model;
  s.vocab_size = 64;
  s.max_positions = 4096;
  return s;
}

std::vector<TokenId> pattern_tokens(std::size_t n, std::size_t vocab, std::size_t salt) {
  std::vector<TokenId> t(n);
  for (std::size_t i = 0; i < n; ++i) t[i] = static_cast<TokenId>((i * 13 + salt * 7 + 1) % vocab);
  return t;
}

LayerProfile triple(std::size_t a, std::size_t b, std::size_t c) {
  LayerProfile p;
  p.l_start = a;
  p.l_det = b;
  p.l_end = c;
  return p;
}

double max_abs(std::span<const float> a, std::span<const float> b) {
  double mx = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) mx = std::max(mx, std::abs(static_cast<double>(a[i]) - b[i]));
  return mx;
}

bool ctx_bit_equal(const KVContext& a, const KVContext& b, std::size_t upto = SIZE_MAX) {
  if (upto == SIZE_MAX && a.size() != b.size()) return false;
  const std::size_t n = std::min(upto, a.size());
  for (std::size_t l = 0; l < a.num_layers(); ++l)
    for (std::size_t p = 0; p < n; ++p) {
      const auto ka = a.key_row(l, p), kb = b.key_row(l, p);
      const auto va = a.value_row(l, p), vb = b.value_row(l, p);
      if (std::memcmp(ka.data(), kb.data(), ka.size_bytes()) || std::memcmp(va.data(), vb.data(), va.size_bytes()))
        return false;
    }
  return true;
}

}  // namespace

TEST_CASE("init_weights validates the spec like the reference") {
  CHECK_THROWS_AS(init_weights(spec_of(2, 32, 4), 1), SchemaError);
  const Weights a = init_weights(spec_of(6, 32, 4), 5), b = init_weights(spec_of(6, 32, 4), 5);
  CHECK(a.output_head.data == b.output_head.data);
  CHECK(a.model_id == "toy-L6-d32-h4-kv4-ff64-v64-s5");
}

TEST_CASE("degenerate full-range relay with select-all reduces to full recomputation") {
  const Weights w = init_weights(spec_of(8, 32, 4), 101);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(12, 64, 0), 10, 0);
  const auto new_prefix = pattern_tokens(9, 64, 5);
  RelayOptions ro;
  ro.thresholds.suffix_k = 10;
  const RelayPrefillResult relay = relay_prefill(w, new_prefix, cache, triple(0, 0, 7), ro);
  RelayOptions fo;
  fo.mode = RelayMode::kFull;
  const RelayPrefillResult full = relay_prefill(w, new_prefix, cache, triple(0, 0, 7), fo);
  CHECK(ctx_bit_equal(relay.ctx.kv, full.ctx.kv));
  CHECK(max_abs(relay.segment_end_logits.row(0), full.segment_end_logits.row(0)) <= 1e-5);
  CHECK(relay.segment.stats.recomputed_entries == 8 * 10);
  CHECK(relay.segment.stats.reuse_rate == 0.0);
}

TEST_CASE("zero mode with unchanged prefix reproduces decode-time KV bit-exactly") {
  const Weights w = init_weights(spec_of(8, 32, 4), 102);
  const auto old_prefix = pattern_tokens(10, 64, 0);
  KVContext decode_ctx;
  const RelayCache cache = capture_relay_cache(w, old_prefix, 8, 2, &decode_ctx);
  RelayOptions opts;
  opts.mode = RelayMode::kZero;
  const RelayPrefillResult zero = relay_prefill(w, old_prefix, cache, LayerProfile{}, opts);
  CHECK(ctx_bit_equal(zero.ctx.kv, decode_ctx));
  CHECK(zero.segment.stats.recomputed_entries == 0);
  CHECK(zero.segment.stats.reuse_rate == 1.0);
  for (const auto o : zero.ctx.segments[0].origin) CHECK(o == CellOrigin::kReused);
}

TEST_CASE("reuse accounting matches the counting formula exactly") {
  const Weights w = init_weights(spec_of(32, 16, 2), 103);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(8, 64, 0), 100, 1);
  RelayOptions opts;
  opts.thresholds.tau_dev = 1e9;
  opts.thresholds.tau_inf = 1e9;
  opts.thresholds.suffix_k = 10;
  const RelayPrefillResult r = relay_prefill(w, pattern_tokens(12, 64, 3), cache, triple(1, 3, 18), opts);
  const ReuseStats& st = r.segment.stats;
  CHECK(st.selected_count == 10);
  CHECK(st.total_entries == 3200);
  CHECK(st.recomputed_entries == 450);
  CHECK(st.reuse_rate == 0.859375);
  const SegmentMarks& marks = r.ctx.segments[0];
  CHECK(marks.recomputed() == st.recomputed_entries);
  for (std::size_t l = 4; l <= 18; ++l)
    for (std::size_t j = 0; j < 100; ++j)
      CHECK(marks.at(l, j) == (j >= 90 ? CellOrigin::kRecomputed : CellOrigin::kReused));
}

TEST_CASE("blend baseline: alpha=1 equals full, small alpha keeps only bootstrap layers") {
  const Weights w = init_weights(spec_of(8, 32, 4), 104);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(10, 64, 0), 12, 0);
  const auto new_prefix = pattern_tokens(7, 64, 9);
  const RelayPrefillResult all = blend_baseline(w, new_prefix, cache, 1.0);
  RelayOptions fo;
  fo.mode = RelayMode::kFull;
  const RelayPrefillResult full = relay_prefill(w, new_prefix, cache, LayerProfile{}, fo);
  CHECK(ctx_bit_equal(all.ctx.kv, full.ctx.kv));
  const RelayPrefillResult tiny = blend_baseline(w, new_prefix, cache, 0.05);
  CHECK(tiny.segment.stats.selected_count == 0);
  CHECK(tiny.segment.stats.recomputed_entries == 2 * 12);
  CHECK_THROWS_AS(blend_baseline(w, new_prefix, cache, 0.0), std::invalid_argument);
}

TEST_CASE("suffix processing never touches segment cells") {
  const Weights w = init_weights(spec_of(8, 32, 4), 106);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(10, 64, 0), 8, 1);
  const RelayPrefillResult r = relay_prefill(w, pattern_tokens(6, 64, 4), cache, triple(1, 2, 5), RelayOptions{});
  const auto run_suffix = [&](std::size_t salt) {
    MergedKVContext ctx = r.ctx;
    prefill(w, pattern_tokens(5, 64, salt), ctx.kv, ctx.kv.size());
    return ctx;
  };
  const MergedKVContext a = run_suffix(11), b = run_suffix(12);
  CHECK(ctx_bit_equal(a.kv, b.kv, 6 + 8));
}

TEST_CASE("relay validates profile, snapshot layer and capacity") {
  const Weights w = init_weights(spec_of(8, 32, 4), 107);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(10, 64, 0), 8, 2);
  const auto prefix = pattern_tokens(4, 64, 1);
  CHECK_THROWS(relay_prefill(w, prefix, cache, triple(1, 2, 20), RelayOptions{}));
  CHECK_THROWS_AS(relay_prefill(w, prefix, cache, triple(1, 2, 5), RelayOptions{}), std::invalid_argument);
  ModelSpec tiny = w.spec;
  tiny.max_positions = 10;
  const Weights w2 = init_weights(tiny, 107);
  const RelayCache c2 = capture_relay_cache(w2, pattern_tokens(4, 64, 0), 4, 0);
  RelayOptions zero;
  zero.mode = RelayMode::kZero;
  CHECK_THROWS_AS(relay_prefill(w2, pattern_tokens(8, 64, 2), c2, LayerProfile{}, zero), std::invalid_argument);
}

TEST_CASE("selection diagnostics are exposed and consistent with the marks") {
  const Weights w = init_weights(spec_of(8, 32, 4), 108);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(14, 64, 0), 20, 1);
  RelayOptions opts;
  opts.thresholds.suffix_k = 4;
  const RelayPrefillResult r = relay_prefill(w, pattern_tokens(10, 64, 8), cache, triple(1, 3, 6), opts);
  CHECK(r.segment.s_dev.size() == 20);
  CHECK(r.segment.s_key_dev.size() == 20);
  for (double d : r.segment.s_dev) CHECK(d >= 0.0);
  const SegmentMarks& marks = r.ctx.segments[0];
  for (std::size_t j = 0; j < 20; ++j)
    CHECK((marks.at(5, j) == CellOrigin::kRecomputed) == r.segment.selection.contains(j));
  CHECK(r.segment.stats.selected_influence_suffix == 4);
  for (std::size_t j = 0; j < 20; ++j)
    CHECK(r.segment.hidden_depth[j] == (r.segment.selection.contains(j) ? 7u : 4u));
}

TEST_CASE("drop-in relay_prefill is bit-identical to the oracle restatement") {
  const ModelSpec spec = spec_of(8, 32, 4);
  const Weights w = init_weights(spec, 55);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(12, 64, 1), 24, 1);
  const auto prefix = pattern_tokens(9, 64, 2);
  RelayOptions opts;
  opts.thresholds.suffix_k = 3;
  const RelayPrefillResult r = relay_prefill(w, prefix, cache, triple(1, 2, 5), opts);
  // oracle
  const rk_model_spec s{8, 32, 4, 4, 8, 64, 64, 10000.0f, 4096, 1e-5f};
  orc_weights* ow = orc_weights_init(&s, 55);
  std::vector<const float*> kp, vp;
  for (std::size_t l = 0; l < 8; ++l) {
    kp.push_back(cache.k_pre[l].data.data());
    vp.push_back(cache.v[l].data.data());
  }
  const rk_relay_cache_view view{8, 4, 8, 32, 10000.0f, 4096, 24, cache.segment_tokens.data(),
                                 cache.source_base_position, 1, 24, kp.data(), vp.data(),
                                 cache.hidden_snapshot.data.data(), cache.influence.data()};
  orc_cache* oc = nullptr;
  REQUIRE(orc_cache_from_view(&view, &oc) == 0);
  orc_ctx* octx = orc_ctx_create(ow);
  std::vector<uint64_t> sel(24);
  rk_relay_output out{};
  out.selection_indices = sel.data();
  std::vector<float> logits(64);
  const rk_layer_profile p{1, 2, 5};
  const rk_relay_options o{RK_MODE_RELAY, 1.5, 1.45, 3, 0.2, 0};
  REQUIRE(orc_relay_prefill(ow, octx, prefix.data(), prefix.size(), oc, &p, &o, &out, logits.data()) == 0);
  CHECK(out.selection_count == r.segment.selection.size());
  for (std::size_t i = 0; i < out.selection_count; ++i) CHECK(sel[i] == r.segment.selection.indices[i]);
  CHECK(std::memcmp(logits.data(), r.segment_end_logits.data.data(), 64 * 4) == 0);
  std::vector<float> k(r.ctx.kv.size() * 32), v(k.size());
  for (std::size_t l = 0; l < 8; ++l) {
    REQUIRE(orc_ctx_export(octx, l, 0, r.ctx.kv.size(), k.data(), v.data()) == 0);
    for (std::size_t pos = 0; pos < r.ctx.kv.size(); ++pos) {
      CHECK(std::memcmp(r.ctx.kv.key_row(l, pos).data(), k.data() + pos * 32, 32 * 4) == 0);
      CHECK(std::memcmp(r.ctx.kv.value_row(l, pos).data(), v.data() + pos * 32, 32 * 4) == 0);
    }
  }
  orc_ctx_destroy(octx);
  orc_cache_destroy(oc);
  orc_weights_destroy(ow);
}

// test_relay_cache.cpp:251-276 "cache export/import is the identity", plus the
// file round trip (relay_cache.cpp:238-253).
TEST_CASE("cache export/import is the identity") {
  const Weights w = init_weights(spec_of(6, 32, 4), 31);
  const RelayCache cache = capture_relay_cache(w, pattern_tokens(7, 64, 0), 5, 1);
  const auto bytes = export_relay_cache(cache);
  const RelayCache back = import_relay_cache(bytes);
  CHECK(back.segment_tokens == cache.segment_tokens);
  CHECK(back.source_base_position == cache.source_base_position);
  CHECK(back.snapshot_layer == cache.snapshot_layer);
  CHECK(back.decode_steps_observed == cache.decode_steps_observed);
  CHECK(back.influence == cache.influence);
  CHECK(std::memcmp(back.hidden_snapshot.data.data(), cache.hidden_snapshot.data.data(),
                    cache.hidden_snapshot.data.size() * 4) == 0);
  for (std::size_t l = 0; l < cache.num_layers(); ++l) {
    CHECK(std::memcmp(back.k_pre[l].data.data(), cache.k_pre[l].data.data(), cache.k_pre[l].data.size() * 4) == 0);
    CHECK(std::memcmp(back.v[l].data.data(), cache.v[l].data.data(), cache.v[l].data.size() * 4) == 0);
  }
  auto truncated = bytes;
  truncated.resize(truncated.size() - 3);
  CHECK_THROWS_AS(import_relay_cache(truncated), SchemaError);
  RelayCache empty;
  CHECK_THROWS_AS(export_relay_cache(empty), std::invalid_argument);

  const std::filesystem::path p = std::filesystem::temp_directory_path() / "relaykv_dropin_cache.rkrc";
  save_relay_cache(cache, p);
  const RelayCache again = load_relay_cache(p);
  CHECK(export_relay_cache(again) == bytes);
  std::filesystem::remove(p);
  CHECK_THROWS_AS(load_relay_cache(p), IoError);
}

// model.hpp:108-111 + workflow.cpp:304,343: PrefillResult.logits is chunk x
// vocab and callers index row(n-1); every row equals a prefill ending there.
TEST_CASE("prefill returns every row's logits (chunk x vocab)") {
  const Weights w = init_weights(spec_of(6, 32, 4), 61);
  const auto toks = pattern_tokens(9, 64, 3);
  KVContext a(w.spec);
  const PrefillResult all = prefill(w, toks, a, 0);
  REQUIRE(all.logits.rows() == 9);
  REQUIRE(all.logits.cols() == 64);
  for (std::size_t n = 1; n <= 9; ++n) {  // row n-1 == the last row of a prefill of the first n tokens
    KVContext b(w.spec);
    const PrefillResult part = prefill(w, std::span<const TokenId>(toks.data(), n), b, 0);
    CHECK(std::memcmp(part.logits.row(n - 1).data(), all.logits.row(n - 1).data(), 64 * 4) == 0);
  }
  set_prefill_logits(PrefillLogits::kLastRow);
  KVContext c(w.spec);
  const PrefillResult last = prefill(w, toks, c, 0);
  set_prefill_logits(PrefillLogits::kAllRows);
  CHECK(std::memcmp(last.logits.row(8).data(), all.logits.row(8).data(), 64 * 4) == 0);
  CHECK(ctx_bit_equal(a, c));
}

// relay_cache.cpp:51-136 through the StepHook API (test_engine.cpp:43-62):
// greedy_generate + RelayRecorder over host traces == the device recorder.
TEST_CASE("RelayRecorder over greedy_generate traces equals the device capture") {
  const Weights w = init_weights(spec_of(6, 32, 4), 62);
  const auto old = pattern_tokens(11, 64, 4);
  KVContext dctx(w.spec);
  const PrefillResult p = prefill(w, old, dctx, 0);
  CaptureFlags cap;
  cap.hidden = cap.pre_rope_keys = cap.attention = true;
  RelayRecorder rec(w.spec, old.size(), 1);
  std::size_t steps = 0;
  const StepHook hook = [&](const StepTrace& tr, TokenId tok, std::size_t pos) {
    REQUIRE(tr.attn.size() == w.spec.num_layers);
    CHECK(tr.attn[0][0].cols() == pos + 1);
    rec.feed(tr, tok, pos);
    ++steps;
  };
  const auto gen = greedy_generate(w, dctx, p.logits.row(old.size() - 1), 13, cap, hook);
  const RelayCache host = rec.finalize();
  KVContext dev_ctx;
  const RelayCache dev = capture_relay_cache(w, old, 13, 1, &dev_ctx);
  CHECK(steps == 13);
  CHECK(gen.tokens == dev.segment_tokens);
  CHECK(host.segment_tokens == dev.segment_tokens);
  CHECK(host.influence == dev.influence);
  CHECK(export_relay_cache(host) == export_relay_cache(dev));
  CHECK(ctx_bit_equal(dctx, dev_ctx));
  // a trace without attention is rejected by name (relay_cache.cpp:75-84)
  RelayRecorder bad(w.spec, 0, 0);
  CHECK_THROWS_AS(bad.feed(StepTrace{}, 1, 0), std::invalid_argument);
}

TEST_CASE("relay caches are validated before any pointer reaches the device") {
  const Weights w = init_weights(spec_of(6, 32, 4), 63);
  RelayCache c = capture_relay_cache(w, pattern_tokens(8, 64, 1), 6, 1);
  RelayOptions opts;
  RelayCache short_v = c;
  short_v.v[2].data.resize(5);  // malformed: would be a heap over-read
  short_v.v[2].shape = {1, 5};
  CHECK_THROWS_AS(relay_prefill(w, pattern_tokens(4, 64, 2), short_v, triple(1, 2, 4), opts), std::invalid_argument);
  CHECK_THROWS_AS(export_relay_cache(short_v), std::invalid_argument);
  RelayCache wrong_geom = c;
  wrong_geom.theta_base = 500000.0f;
  CHECK_THROWS_AS(relay_prefill(w, pattern_tokens(4, 64, 2), wrong_geom, triple(1, 2, 4), opts),
                  std::invalid_argument);
  RelayCache neg = c;
  neg.influence[0] = -1.0f;
  CHECK_THROWS_AS(relay_prefill(w, pattern_tokens(4, 64, 2), neg, triple(1, 2, 4), opts), std::invalid_argument);
}

TEST_CASE("device weights follow the Weights object: in-place edits need release, new storage re-uploads") {
  Weights w = init_weights(spec_of(6, 32, 4), 64);
  const auto toks = pattern_tokens(7, 64, 5);
  KVContext a(w.spec);
  const PrefillResult base = prefill(w, toks, a, 0);
  w.output_head.data[3] += 1.0f;  // in place: the device copy is now stale ...
  release_device_weights(w);      // ... until released
  KVContext b(w.spec);
  const PrefillResult edited = prefill(w, toks, b, 0);
  CHECK(std::memcmp(base.logits.row(6).data(), edited.logits.row(6).data(), 64 * 4) != 0);
  w.output_head.data = std::vector<float>(w.output_head.data);  // new storage: detected without a release
  w.output_head.data[3] -= 1.0f;
  KVContext c(w.spec);
  const PrefillResult restored = prefill(w, toks, c, 0);
  CHECK(std::memcmp(base.logits.row(6).data(), restored.logits.row(6).data(), 64 * 4) == 0);
  const Weights copy = w;  // a copy owns its own device copies
  KVContext d(copy.spec);
  const PrefillResult from_copy = prefill(copy, toks, d, 0);
  CHECK(std::memcmp(base.logits.row(6).data(), from_copy.logits.row(6).data(), 64 * 4) == 0);
}

TEST_CASE("page-locked relay caches give the same relay") {
  const Weights w = init_weights(spec_of(6, 32, 4), 65);
  const RelayCache c = capture_relay_cache(w, pattern_tokens(9, 64, 1), 16, 1);
  RelayOptions opts;
  const RelayPrefillResult a = relay_prefill(w, pattern_tokens(5, 64, 2), c, triple(1, 2, 4), opts);
  {
    PinnedRelayCache pin(c);
    const RelayPrefillResult b = relay_prefill(w, pattern_tokens(5, 64, 2), c, triple(1, 2, 4), opts);
    CHECK(a.segment.selection.indices == b.segment.selection.indices);
    CHECK(a.segment_end_logits.bit_equal(b.segment_end_logits));
    CHECK(ctx_bit_equal(a.ctx.kv, b.ctx.kv));
  }
}

// model.cpp:339-362 through the ABI (rk_row_logits_from_layer)
TEST_CASE("row_logits_from_layer equals relay_prefill's segment-end logits") {
  const Weights w = init_weights(spec_of(6, 32, 4), 66);
  const RelayCache c = capture_relay_cache(w, pattern_tokens(9, 64, 1), 12, 1);
  RelayOptions opts;
  const RelayPrefillResult r = relay_prefill(w, pattern_tokens(5, 64, 2), c, triple(1, 2, 4), opts);
  const std::size_t n = c.segment_len(), depth = r.segment.hidden_depth[n - 1];
  REQUIRE(depth < w.spec.num_layers);
  const Tensor lg = row_logits_from_layer(w, r.segment.segment_hidden.row(n - 1), depth, r.ctx.kv,
                                          r.ctx.kv.size() - 1);
  CHECK(lg.bit_equal(r.segment_end_logits));
}
