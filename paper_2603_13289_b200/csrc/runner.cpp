// runner.cpp -- per-call orchestration of the relay-prefill path.
//
// Control flow follows the reference line by line (cited per function); the
// device work is enqueued on the engine stream without host round trips
// except where the reference's control flow needs a device value (the depth
// of the last segment row for relay_prefill's pure-query pass). Selection
// counts stay on the device: the sparse passes read |I| from device memory.
#include <cmath>
#include <cstring>

#include <cstdlib>

#include "layer.h"
#include "layer_tc.h"
#include "prof.h"

namespace rk {
namespace {
void require(bool ok, int code, const std::string& msg) {
  if (!ok) raise(code, msg);
}
float* fptr(void* p, size_t off_elems = 0) { return static_cast<float*>(p) + off_elems; }
}  // namespace

Runner::Runner(rk_engine* e, rk_weights* w) : e_(e), w_(w), st_(e->stream) {
  require(e != nullptr && w != nullptr, RK_ERR_INVALID_ARGUMENT, "null engine / weights");
  require(w->e == e, RK_ERR_INVALID_ARGUMENT, "weights belong to another engine");
  k::zero_dev(st_, e->status.p, 64);
  e->launches += 1;
  // side-stream reporting work of the previous call must finish before its
  // buffers (selection slots) are reused
  if (e->side_join) RK_CUDA(cudaStreamWaitEvent(st_, e->side_join, 0));
}
Runner::~Runner() = default;

int Runner::event() {
  if (next_event_ >= (int)e_->events.size()) {
    cudaEvent_t ev;
    RK_CUDA(cudaEventCreate(&ev));
    e_->events.push_back(ev);
  }
  RK_CUDA(cudaEventRecord(e_->events[next_event_], st_));
  return next_event_++;
}

// Asynchronously uploaded caches: the compute stream waits (on the device)
// for the pieces it is about to read.
void Runner::wait_cache_meta(rk_cache* c) {
  if (c->async) RK_CUDA(cudaStreamWaitEvent(st_, c->ev_meta, 0));
}
void Runner::wait_cache_layer(rk_cache* c, uint64_t l) {
  ensure_cache_layer(c, l);
  if (c->async) RK_CUDA(cudaStreamWaitEvent(st_, c->ev_layer[l], 0));
}

ExtendSlot& Runner::slot(int i) {
  while ((int)e_->slots.size() <= i) e_->slots.emplace_back(new ExtendSlot());
  return *e_->slots[i];
}

void Runner::begin_timer() { timer_ev_ = event(); }
float Runner::lap_ms() {
  const int ev = event();
  RK_CUDA(cudaEventSynchronize(e_->events[ev]));
  float ms = 0.f;
  RK_CUDA(cudaEventElapsedTime(&ms, e_->events[timer_ev_], e_->events[ev]));
  return ms;
}

void Runner::ensure_rows(size_t R) {
  Scratch& S = *e_->scratch;
  const rk_model_spec& s = w_->s;
  const size_t d = s.d_model, q = w_->q(), kv = w_->kv(), ff = s.d_ff;
  R = std::max<size_t>(R, 1);
  S.hidden.ensure(R * d * 4);
  S.normed.ensure(R * d * 4);
  S.qkv.ensure(R * (q + 2 * kv) * 4);
  S.attn.ensure(R * q * 4);
  S.act.ensure(R * ff * 4);
  S.positions.ensure(std::max<size_t>(R, s.max_positions) * 4);
  S.sub_positions.ensure(64);
  S.logits.ensure(s.vocab_size * 4);
  S.argmax.ensure(64 + 148 * 8);  // [0] result, +64: argmax partials
  S.seg_hidden_out.ensure(d * 4);
  S.tokens.ensure((s.max_positions + 64) * 4);
}

void Runner::check_tokens(const int32_t* tokens, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (tokens[i] < 0 || (uint64_t)tokens[i] >= w_->s.vocab_size)
      raise(RK_ERR_INVALID_ARGUMENT, "token id " + std::to_string(tokens[i]) + " outside vocab of " +
                                         std::to_string(w_->s.vocab_size));
}

// Stage host tokens through pinned memory; `slot` is an offset in tokens.
int* Runner::upload_tokens(const int32_t* tokens, uint64_t n, int off) {
  Scratch& S = *e_->scratch;
  const size_t need = (off + n) * 4;
  if (need > e_->pinned_bytes) {
    RK_CUDA(cudaStreamSynchronize(st_));
    cudaFreeHost(e_->pinned);
    e_->pinned = nullptr;
    e_->pinned_bytes = std::max(need, e_->pinned_bytes * 2);
    RK_CUDA(cudaMallocHost(&e_->pinned, e_->pinned_bytes));
  }
  S.tokens.ensure(need + 256);
  int32_t* pin = static_cast<int32_t*>(e_->pinned) + off;
  std::memcpy(pin, tokens, n * 4);
  int* dev = S.tokens.as<int>() + off;
  // a kernel reads the (mapped) pinned tokens over PCIe instead of a copy:
  // the copy engine may be busy streaming relay caches (rk_cache_upload_async)
  // and a memcpy would queue behind them
  int32_t* mapped = nullptr;
  RK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&mapped), pin, 0));
  k::copy_i32(st_, dev, mapped, (int)n);
  e_->launches += 1;
  return dev;
}

// ---------------------------------------------------------------------------
// one decoder layer (run_layer_rows, model.cpp:237-280)
// ---------------------------------------------------------------------------
void Runner::run_layer(rk_context* ctx, int l, float* hidden, Rows rows, bool commit, int max_ctx,
                       float* probs, int key_lo, int key_n, int tail) {
  if (w_->precision == RK_BF16) {
    run_layer_bf16(e_, w_, ctx, l, hidden, rows, commit, max_ctx, probs, key_lo, key_n, cap_k_, cap_v_, prepared_,
                   tail);
    prepared_ = true;
    return;
  }
  Scratch& S = *e_->scratch;
  const rk_model_spec& s = w_->s;
  const rk_layer_dev& ly = w_->layers[l];
  const int d = s.d_model, q = w_->q(), kv = w_->kv(), ff = s.d_ff;
  const int H = s.num_heads, Hkv = s.num_kv_heads, dh = s.d_head;
  int* status = e_->status.as<int>();
  float* ck = static_cast<float*>(ctx->k_layer(l));
  float* cv = static_cast<float*>(ctx->v_layer(l));
  const double2* rope = w_->rope->cs.as<double2>();
  const bool tcm = w_->precision == RK_FP32_TC;  // 3xTF32 matmuls + fp32 flash attention (layer_tc.cu)
  {
    ProfScope ps(e_, "norm_exact", 0, 0);
    k::rmsnorm_exact(st_, hidden, ly.attn_norm, s.norm_eps, S.normed.as<float>(), rows, d);
  }
  if (tcm) {
    tc::gemm(e_, S.normed.as<float>(), d, rows, ly.tc_qkv, q + 2 * kv, d, S.qkv.as<float>(), q + 2 * kv, false);
  } else {
    ProfScope ps(e_, "gemm_exact_qkv", 0, 0);
    k::gemm_exact(st_, S.normed.as<float>(), static_cast<const float*>(ly.w_qkv), S.qkv.as<float>(), rows,
                  q + 2 * kv, d, k::EPI_STORE, status);
  }
  if (cap_k_) {  // decode-time capture of pre-rotation K and V (model.cpp:254-257)
    k::copy2d_f32(st_, cap_k_, kv, 1, S.qkv.as<float>() + q, q + 2 * kv, 1, rows.rows_max, kv);
    k::copy2d_f32(st_, cap_v_, kv, 1, S.qkv.as<float>() + q + kv, q + 2 * kv, 1, rows.rows_max, kv);
    e_->launches += 2;
  }
  {
    ProfScope ps(e_, "rope_commit_exact", 0, 0);
    k::rope_commit_exact(st_, S.qkv.as<float>(), rows, H, Hkv, dh, rope, ck, cv, commit ? 1 : 0);
  }
  const float* qkv = S.qkv.as<float>();
  if (tail >= 0 && commit && !rows.rows_dev && tail < rows.rows_max) {
    // only the last `tail` rows continue (see run_layer_bf16)
    if (tail == 0) {
      e_->launches += 3;
      return;
    }
    const int off = rows.rows_max - tail;
    hidden += (size_t)off * d;
    qkv += (size_t)off * (q + 2 * kv);
    rows = Rows{tail, nullptr, rows.pos + off};
  }
  if (tcm && commit && !probs) {  // (the pure-query pass and the capture keep the exact kernel)
    tc::attention(e_, qkv, q + 2 * kv, rows, H, Hkv, dh, ck, cv, S.attn.as<float>());
  } else {
    ProfScope ps(e_, "attn_exact", 0, 0);
    k::attn_exact(st_, qkv, rows, H, Hkv, dh, ck, cv, S.attn.as<float>(), commit ? 0 : 1,
                  max_ctx, probs, key_lo, key_n);
  }
  if (tcm) {
    tc::gemm(e_, S.attn.as<float>(), q, rows, ly.tc_o, d, q, hidden, d, true);
    k::rmsnorm_exact(st_, hidden, ly.mlp_norm, s.norm_eps, S.normed.as<float>(), rows, d);
    S.tc_gu.ensure((size_t)rows.rows_max * 2 * ff * 4);
    tc::gemm(e_, S.normed.as<float>(), d, rows, ly.tc_gu, 2 * ff, d, S.tc_gu.as<float>(), 2 * ff, false);
    tc::silu(e_, S.tc_gu.as<float>(), S.act.as<float>(), rows, ff);
    tc::gemm(e_, S.act.as<float>(), ff, rows, ly.tc_down, d, ff, hidden, d, true);
    e_->launches += 3;
    return;
  }
  {
    ProfScope ps(e_, "gemm_exact_o", 0, 0);
    k::gemm_exact(st_, S.attn.as<float>(), static_cast<const float*>(ly.w_o), hidden, rows, d, q,
                  k::EPI_ADD, status);
  }
  k::rmsnorm_exact(st_, hidden, ly.mlp_norm, s.norm_eps, S.normed.as<float>(), rows, d);
  {
    ProfScope ps(e_, "gemm_exact_mlp", 0, 0);
    k::gemm_exact(st_, S.normed.as<float>(), static_cast<const float*>(ly.w_gu), S.act.as<float>(), rows,
                  2 * ff, d, k::EPI_SILU_PAIR, status);
    k::gemm_exact(st_, S.act.as<float>(), static_cast<const float*>(ly.w_down), hidden, rows, d, ff,
                  k::EPI_ADD, status);
  }
  e_->launches += 8;
}

// output_logits (model.cpp:282-288) of one row into scratch logits.
void Runner::last_row_logits(const float* hidden_row) {
  Scratch& S = *e_->scratch;
  const rk_model_spec& s = w_->s;
  if (w_->precision == RK_BF16) {
    last_row_logits_bf16(e_, w_, hidden_row, S.logits.as<float>());
  } else {
    Rows one{1, nullptr, S.sub_positions.as<int>()};
    k::rmsnorm_exact(st_, hidden_row, w_->final_norm, s.norm_eps, S.normed.as<float>(), one, s.d_model);
    k::gemm_exact(st_, S.normed.as<float>(), static_cast<const float*>(w_->head), S.logits.as<float>(), one,
                  s.vocab_size, s.d_model, k::EPI_STORE, e_->status.as<int>());
    e_->launches += 2;
  }
  have_logits_ = true;
}

// row_logits_from_layer (model.cpp:339-362): the row as a pure query, its
// own cell overridden by fresh K/V, nothing committed.
void Runner::row_logits_from_layer(rk_context* ctx, const float* hidden_row, uint64_t first_layer,
                                   uint64_t position) {
  Scratch& S = *e_->scratch;
  const rk_model_spec& s = w_->s;
  float* row = S.seg_hidden_out.as<float>();
  k::copy_dev(st_, row, hidden_row, s.d_model * 4);
  k::iota_positions(st_, S.sub_positions.as<int>(), 1, (int)position);
  e_->launches += 1;
  Rows one{1, nullptr, S.sub_positions.as<int>()};
  prepared_ = false;
  for (uint64_t l = first_layer; l < s.num_layers; ++l)
    run_layer(ctx, (int)l, row, one, /*commit=*/false, (int)position + 1);
  last_row_logits(row);
}

// ---------------------------------------------------------------------------
// prefill (model.cpp:305-331)
// ---------------------------------------------------------------------------
void Runner::prefill(rk_context* ctx, const int32_t* tokens, uint64_t n, uint64_t base, bool want_logits) {
  const rk_model_spec& s = w_->s;
  require(ctx != nullptr && ctx->w == w_, RK_ERR_INVALID_ARGUMENT, "context belongs to other weights");
  require(n > 0, RK_ERR_INVALID_ARGUMENT, "prefill: empty token chunk");
  require(base == ctx->size, RK_ERR_INVALID_ARGUMENT,
          "prefill: base_position " + std::to_string(base) + " != context size " + std::to_string(ctx->size));
  require(base + n <= s.max_positions, RK_ERR_INVALID_ARGUMENT,
          "prefill: position overflow beyond max_positions " + std::to_string(s.max_positions));
  require(tokens != nullptr, RK_ERR_INVALID_ARGUMENT, "null tokens");
  check_tokens(tokens, n);
  ensure_rows(n);
  Scratch& S = *e_->scratch;
  int* dev_tok = upload_tokens(tokens, n, tok_cursor_);
  tok_cursor_ += (int)n;
  k::embed(st_, S.hidden.as<float>(), w_->emb, w_->elem, dev_tok, (int)n, (int)s.d_model, 0, nullptr);
  ctx->resize(base + n);
  k::iota_positions(st_, S.positions.as<int>(), (int)n, (int)base);
  e_->launches += 2;
  Rows rows{(int)n, nullptr, S.positions.as<int>()};
  prepared_ = false;
  for (uint64_t l = 0; l < s.num_layers; ++l)  // top layer: only the last row's output is ever read
    run_layer(ctx, (int)l, S.hidden.as<float>(), rows, true, (int)(base + n), nullptr, 0, 0,
              l + 1 == s.num_layers ? (want_logits ? 1 : 0) : -1);
  if (want_logits) last_row_logits(S.hidden.as<float>() + (n - 1) * s.d_model);
}

// prefill with capture (model.cpp:305-331, CaptureFlags/StepTrace): the same
// layer pass with the top layer over all rows, each layer's input rows, pre-RoPE
// K/V and full-context attention rows copied out per layer, and every row's
// logits (output_logits over the chunk, model.cpp:328).
void Runner::prefill_trace(rk_context* ctx, const int32_t* tokens, uint64_t n, uint64_t base,
                           const rk_trace_request& rq) {
  const rk_model_spec& s = w_->s;
  require(ctx != nullptr && ctx->w == w_, RK_ERR_INVALID_ARGUMENT, "context belongs to other weights");
  require(n > 0, RK_ERR_INVALID_ARGUMENT, "prefill: empty token chunk");
  require(base == ctx->size, RK_ERR_INVALID_ARGUMENT,
          "prefill: base_position " + std::to_string(base) + " != context size " + std::to_string(ctx->size));
  require(base + n <= s.max_positions, RK_ERR_INVALID_ARGUMENT,
          "prefill: position overflow beyond max_positions " + std::to_string(s.max_positions));
  require(tokens != nullptr, RK_ERR_INVALID_ARGUMENT, "null tokens");
  check_tokens(tokens, n);
  ensure_rows(n);
  Scratch& S = *e_->scratch;
  const uint64_t L = s.num_layers, d = s.d_model, kv = w_->kv(), H = s.num_heads, V = s.vocab_size;
  const uint64_t keys = base + n, el = w_->elem;
  int* dev_tok = upload_tokens(tokens, n, tok_cursor_);
  tok_cursor_ += (int)n;
  k::embed(st_, S.hidden.as<float>(), w_->emb, w_->elem, dev_tok, (int)n, (int)d, 0, nullptr);
  ctx->resize(base + n);
  k::iota_positions(st_, S.positions.as<int>(), (int)n, (int)base);
  e_->launches += 2;
  Rows rows{(int)n, nullptr, S.positions.as<int>()};
  const bool kvcap = rq.k_pre || rq.v;
  DevBuf kst, vst, f32, probs;
  if (kvcap) {
    kst.alloc(n * kv * el);
    vst.alloc(n * kv * el);
    if (el == 2) f32.alloc(n * kv * 4);
  }
  if (rq.attn) probs.alloc(n * H * keys * 4);
  auto kv_out = [&](float* dst, const DevBuf& src) {
    if (!dst) return;
    if (el == 4) {
      RK_CUDA(cudaMemcpyAsync(dst, src.p, n * kv * 4, cudaMemcpyDeviceToHost, st_));
    } else {
      k::bf16_to_f32(st_, f32.as<float>(), static_cast<const __nv_bfloat16*>(src.p), n * kv);
      RK_CUDA(cudaMemcpyAsync(dst, f32.p, n * kv * 4, cudaMemcpyDeviceToHost, st_));
      e_->launches += 1;
    }
    RK_CUDA(cudaStreamSynchronize(st_));
  };
  prepared_ = false;
  for (uint64_t l = 0; l < L; ++l) {
    if (rq.hidden) {
      RK_CUDA(cudaMemcpyAsync(rq.hidden + l * n * d, S.hidden.p, n * d * 4, cudaMemcpyDeviceToHost, st_));
      RK_CUDA(cudaStreamSynchronize(st_));
    }
    if (kvcap) {
      cap_k_ = static_cast<float*>(kst.p);
      cap_v_ = static_cast<float*>(vst.p);
    }
    run_layer(ctx, (int)l, S.hidden.as<float>(), rows, true, (int)(base + n), rq.attn ? probs.as<float>() : nullptr,
              0, (int)keys, -1);
    cap_k_ = cap_v_ = nullptr;
    if (kvcap) {
      kv_out(rq.k_pre ? rq.k_pre + l * n * kv : nullptr, kst);
      kv_out(rq.v ? rq.v + l * n * kv : nullptr, vst);
    }
    if (rq.attn) {
      RK_CUDA(cudaMemcpyAsync(rq.attn + l * n * H * keys, probs.p, n * H * keys * 4, cudaMemcpyDeviceToHost, st_));
      RK_CUDA(cudaStreamSynchronize(st_));
    }
  }
  if (rq.logits) {  // output_logits over every row (model.cpp:282-288)
    DevBuf lg(n * V * 4);
    if (w_->precision == RK_BF16) {
      rows_logits_bf16(e_, w_, S.hidden.as<float>(), rows, lg.as<float>());
    } else {
      k::rmsnorm_exact(st_, S.hidden.as<float>(), w_->final_norm, s.norm_eps, S.normed.as<float>(), rows, (int)d);
      k::gemm_exact(st_, S.normed.as<float>(), static_cast<const float*>(w_->head), lg.as<float>(), rows, (int)V,
                    (int)d, k::EPI_STORE, e_->status.as<int>());
    }
    e_->launches += 2;
    RK_CUDA(cudaMemcpyAsync(rq.logits, lg.p, n * V * 4, cudaMemcpyDeviceToHost, st_));
    RK_CUDA(cudaStreamSynchronize(st_));
  }
}

// Validation of one relay_extend (relay_engine.cpp:186-192, 236-243, 296-298;
// relay_cache.cpp:43-49, 157-161) and its layer window.
ExtendPlan Runner::plan_extend(uint64_t base, rk_cache* cache, const rk_layer_profile* prof,
                               const rk_relay_options& opts) {
  const rk_model_spec& s = w_->s;
  require(cache != nullptr, RK_ERR_INVALID_ARGUMENT, "null relay cache");
  require(cache->L == s.num_layers && cache->Hkv == s.num_kv_heads && cache->dh == s.d_head &&
              cache->d == s.d_model && cache->theta == s.theta_base,
          RK_ERR_INVALID_ARGUMENT, "relay cache geometry does not match model spec");
  require(cache->elem == w_->elem, RK_ERR_INVALID_ARGUMENT,
          "relay cache was uploaded for weights of another precision");
  const uint64_t n = cache->n, L = s.num_layers;
  require(base + n <= s.max_positions, RK_ERR_INVALID_ARGUMENT, "relay_extend: segment overflows max_positions");
  const int mode = opts.mode;
  require(mode >= RK_MODE_FULL && mode <= RK_MODE_BLEND, RK_ERR_INVALID_ARGUMENT, "unknown relay mode");
  ExtendPlan p;
  if (mode == RK_MODE_RELAY) {
    require(prof != nullptr, RK_ERR_INVALID_ARGUMENT, "null layer profile");
    // LayerProfile::validate (profiler.cpp:28-35) -> SchemaError
    if (!(prof->l_start <= prof->l_det && prof->l_det <= prof->l_end && prof->l_end < L))
      raise(RK_ERR_SCHEMA, "layer profile violates l_start <= l_det <= l_end < num_layers (" +
                               std::to_string(prof->l_start) + ", " + std::to_string(prof->l_det) + ", " +
                               std::to_string(prof->l_end) + ") for " + std::to_string(L) + " layers");
    require(opts.tau_dev > 0.0, RK_ERR_INVALID_ARGUMENT, "thresholds: tau_dev must be > 0");
    require(opts.tau_inf > 0.0, RK_ERR_INVALID_ARGUMENT, "thresholds: tau_inf must be > 0");
    require(cache->snapshot == prof->l_start, RK_ERR_INVALID_ARGUMENT,
            "relay_extend: cache snapshot layer " + std::to_string(cache->snapshot) +
                " does not match profile l_start " + std::to_string(prof->l_start));
    p.l_start = prof->l_start;
    p.l_det = prof->l_det;
    p.sparse_hi = opts.rectify_above_end ? L - 1 : prof->l_end;
  }
  if (mode == RK_MODE_BLEND) {
    require(opts.blend_alpha > 0.0 && opts.blend_alpha <= 1.0, RK_ERR_INVALID_ARGUMENT,
            "relay_extend: blend alpha must be in (0, 1]");
    require(L >= 2, RK_ERR_INVALID_ARGUMENT, "blend needs at least 2 layers");
    p.l_start = 0;
    p.l_det = 1;
    p.sparse_hi = L - 1;
  }
  if (mode != RK_MODE_FULL)
    require(base + n <= cache->maxpos, RK_ERR_INVALID_ARGUMENT,
            "realign: base " + std::to_string(base) + " overflows max_positions " + std::to_string(cache->maxpos));
  if (mode == RK_MODE_FULL || mode == RK_MODE_BLEND) check_tokens(cache->host_tokens.data(), n);
  return p;
}

// ---------------------------------------------------------------------------
// relay_extend (relay_engine.cpp:183-361)
// ---------------------------------------------------------------------------
ExtendResult Runner::relay_extend(rk_context* ctx, rk_cache* cache, const rk_layer_profile* prof,
                                  const rk_relay_options& opts) {
  const rk_model_spec& s = w_->s;
  require(ctx != nullptr && ctx->w == w_, RK_ERR_INVALID_ARGUMENT, "context belongs to other weights");
  const ExtendPlan plan = plan_extend(ctx->size, cache, prof, opts);
  // wait only for what this extend reads: RELAY/BLEND never read cache layers
  // l_start..l_det-1 (the band recomputes them; l_det feeds the deviation
  // score), FULL reads no layer at all -- deferred uploads of the others stay deferred
  if (cache->async) {
    wait_cache_meta(cache);
    if (opts.mode != RK_MODE_FULL)
      for (uint64_t l = 0; l < s.num_layers; ++l)
        if (opts.mode == RK_MODE_ZERO || l < plan.l_start || l >= plan.l_det) wait_cache_layer(cache, l);
  }
  const uint64_t n = cache->n, base = ctx->size, L = s.num_layers;
  const int mode = opts.mode;
  const uint64_t l_start = plan.l_start, l_det = plan.l_det, sparse_hi = plan.sparse_hi;
  ExtendResult r;
  r.mode = mode;
  r.base = base;
  r.n = n;
  r.L = L;
  r.l_start = l_start;
  r.l_det = l_det;
  r.sparse_hi = sparse_hi;

  r.slot = next_slot_++;
  ExtendSlot& X = slot(r.slot);
  const size_t d = s.d_model, kv = w_->kv();
  X.hidden.ensure(n * d * 4);
  X.sub_hidden.ensure(n * d * 4);
  X.depth.ensure(n * 8);
  X.s_dev.ensure(n * 8);
  X.s_key.ensure(n * 8);
  X.sel_idx.ensure(n * 4);
  X.sel_tags.ensure(2 * n * 4);
  X.info.ensure(64);
  X.dinfo.ensure(64);
  X.sub_pos.ensure(n * 4);
  X.score.ensure(n * 8);
  k::zero_dev(st_, X.info.p, 64);
  k::zero_dev(st_, X.dinfo.p, 64);
  ensure_rows(n);
  Scratch& S = *e_->scratch;

  rk_segment_marks marks;
  marks.base = base;
  marks.len = n;
  marks.origin.alloc_pooled(&e_->cache_pool, L * n);  // pooled: freeing would sync the device
  k::zero_dev(st_, marks.origin.p, L * n);
  uint8_t* origin = marks.origin.as<uint8_t>();
  float* hidden = X.hidden.as<float>();
  uint64_t* depth = X.depth.as<uint64_t>();
  const double2* rope = w_->rope->cs.as<double2>();
  const size_t lstride = ctx->cap;  // placeholder, recomputed after resize
  (void)lstride;

  r.ev_begin = event();
  ctx->resize(base + n);
  const size_t layer_stride = ctx->cap * kv;  // elements between layers
  k::iota_positions(st_, S.positions.as<int>(), (int)n, (int)base);
  e_->launches += 1;
  Rows band_rows{(int)n, nullptr, S.positions.as<int>()};
  const int max_ctx = (int)(base + n);

  if (mode != RK_MODE_FULL) {
    // realign + graft (relay_engine.cpp:226-229, 252-256, 301-305); band
    // layers are skipped because the recompute overwrites every one of their
    // segment cells before anything reads them.
    int skip_lo = 1, skip_hi = 0;
    if (mode == RK_MODE_RELAY) { skip_lo = (int)l_start; skip_hi = (int)l_det; }
    if (mode == RK_MODE_BLEND) { skip_lo = 0; skip_hi = 1; }
    const int grafted = (int)L - (skip_hi >= skip_lo ? skip_hi - skip_lo + 1 : 0);
    ProfScope ps(e_, "realign_graft", 3.0 * kv * n * grafted, 4.0 * grafted * n * kv * w_->elem);
    k::realign_graft(st_, cache->k_pre.p, cache->v.p, w_->elem, (int)L, (int)n, (int)kv, (int)s.d_head,
                     rope, (int)base, ctx->k.p, ctx->v.p, layer_stride, skip_lo, skip_hi);
    e_->launches += 1;
  }
  r.ev_realign = event();

  switch (mode) {
    case RK_MODE_FULL: {  // relay_engine.cpp:210-222
      int* dev_tok = cache->tokens.as<int>();
      k::embed(st_, hidden, w_->emb, w_->elem, dev_tok, (int)n, (int)d, 0, nullptr);
      e_->launches += 1;
      prepared_ = false;
      for (uint64_t l = 0; l < L; ++l) run_layer(ctx, (int)l, hidden, band_rows, true, max_ctx);
      k::mark_layers(st_, origin, (int)n, 0, (int)L - 1);
      k::set_depth(st_, depth, (int)n, L);
      e_->launches += 2;
      r.band_layers = L;
      r.ev_band = r.ev_select = r.ev_end = event();
      break;
    }
    case RK_MODE_ZERO: {  // relay_engine.cpp:224-234
      k::copy_dev(st_, hidden, cache->hidden.p, n * d * 4);
      k::set_depth(st_, depth, (int)n, cache->snapshot);
      e_->launches += 1;
      r.ev_band = r.ev_select = r.ev_end = event();
      break;
    }
    default: {  // RELAY (236-293) and BLEND (295-344)
      if (mode == RK_MODE_RELAY) {
        k::copy_dev(st_, hidden, cache->hidden.p, n * d * 4);
      } else {
        k::embed(st_, hidden, w_->emb, w_->elem, cache->tokens.as<int>(), (int)n, (int)d, 0, nullptr);
        e_->launches += 1;
      }
      // full-recompute band: every segment row, layers [l_start, l_det]
      prepared_ = false;
      for (uint64_t l = l_start; l <= l_det; ++l) run_layer(ctx, (int)l, hidden, band_rows, true, max_ctx);
      k::mark_layers(st_, origin, (int)n, (int)l_start, (int)l_det);
      k::set_depth(st_, depth, (int)n, l_det + 1);
      e_->launches += 2;
      r.band_layers = l_det - l_start + 1;
      r.ev_band = event();
      const size_t el = w_->elem;
      const char* ctx_v_det = static_cast<const char*>(ctx->v_layer(l_det)) + base * kv * el;
      const char* cache_v_det = static_cast<const char*>(cache->v.p) + l_det * n * kv * el;
      if (mode == RK_MODE_RELAY) {
        // one-shot selection at the detection layer (relay_engine.cpp:266-282)
        const char* ctx_k_det = static_cast<const char*>(ctx->k_layer(l_det)) + base * kv * el;
        const char* cache_k_det = static_cast<const char*>(cache->k_pre.p) + l_det * n * kv * el;
        {
          ProfScope ps(e_, "score_deviation", 0, 4.0 * n * kv * el);
          k::score_deviation(st_, ctx_v_det, cache_v_det, ctx_k_det, cache_k_det, el, (int)n, (int)kv,
                             (int)s.num_kv_heads, (int)s.d_head, rope, (int)base, X.s_dev.as<double>(),
                             X.s_key.as<double>());
        }
        {
          ProfScope ps(e_, "select_relay", 0, n * 20.0);
          k::select_relay(st_, X.s_dev.as<double>(), cache->influence.as<float>(), cache->infl_mean.as<double>(),
                          (int)n, opts.tau_dev, opts.tau_inf, (int)std::min<uint64_t>(opts.suffix_k, 0x7fffffff),
                          X.sel_idx.as<int>(), X.sel_tags.as<uint32_t>(), X.info.as<int>(), X.dinfo.as<double>(),
                          e_->side, e_->side_fork, e_->side_join);
          e_->launches += 1;  // the side-stream report kernel
        }
        e_->launches += 2;
      } else {
        // CacheBlend ranking at layer 1 (relay_engine.cpp:318-332)
        k::blend_scores(st_, ctx_v_det, cache_v_det, el, (int)n, (int)kv, X.score.as<double>());
        size_t count = static_cast<size_t>(opts.blend_alpha * static_cast<double>(n));
        if (count > n) count = n;
        r.blend_count = (int)count;
        k::select_topk(st_, X.score.as<double>(), (int)n, (int)count, X.sel_idx.as<int>(),
                       X.sel_tags.as<uint32_t>(), X.info.as<int>());
        e_->launches += 3;
      }
      r.ev_select = event();
      // sparse_rectify (relay_engine.cpp:156-179): selected rows through
      // (l_det, sparse_hi], |I| read from device memory by every kernel.
      if (sparse_hi > l_det) {
        const int* count = X.info.as<int>();
        k::gather_rows(st_, X.sub_hidden.as<float>(), hidden, X.sel_idx.as<int>(), count, (int)n, (int)d);
        k::positions_from_sel(st_, X.sub_pos.as<int>(), X.sel_idx.as<int>(), count, (int)n, (int)base);
        e_->launches += 2;
        Rows sparse_rows{(int)n, count, X.sub_pos.as<int>()};
        sparse_rows.hint = live_hint(0, n);
        prepared_ = false;
        for (uint64_t l = l_det + 1; l <= sparse_hi; ++l)
          run_layer(ctx, (int)l, X.sub_hidden.as<float>(), sparse_rows, true, max_ctx);
        k::mark_rows(st_, origin, (int)n, (int)l_det + 1, (int)sparse_hi, X.sel_idx.as<int>(), count, (int)n);
        k::scatter_rows(st_, hidden, X.sub_hidden.as<float>(), X.sel_idx.as<int>(), count, (int)n, (int)d,
                        depth, sparse_hi + 1);
        e_->launches += 2;
        r.sparse_layers = sparse_hi - l_det;
      }
      r.ev_end = event();
      break;
    }
  }
  ctx->segs.push_back(std::move(marks));
  r.seg_index = ctx->segs.size() - 1;
  return r;
}

void Runner::stage_results(std::vector<ExtendResult>& rs, bool token) {
  if (!e_->results_host) RK_CUDA(cudaMallocHost(&e_->results_host, rk_engine::kResultsBytes));
  uint8_t* h = nullptr;  // the device's view of the pinned area (a kernel writes it over PCIe)
  RK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h), e_->results_host, 0));
  k::SmallCopies c;
  auto add = [&](void* dst, const void* src, int bytes) {
    c.src[c.n] = src;
    c.dst[c.n] = dst;
    c.bytes[c.n] = bytes;
    ++c.n;
  };
  size_t off = 64;  // [0, 4): first token, [8, 16): status flags
  for (auto& r : rs) {
    if (!(r.mode == RK_MODE_RELAY || r.mode == RK_MODE_BLEND)) continue;
    if (c.n + 3 > 16 || off + sizeof r.info + sizeof r.dinfo > rk_engine::kResultsBytes) break;  // (rest: resolve copies)
    ExtendSlot& X = slot(r.slot);
    add(h + off, X.info.p, (int)sizeof r.info);
    add(h + off + sizeof r.info, X.dinfo.p, (int)sizeof r.dinfo);
    r.staged = (int)off;
    off += sizeof r.info + sizeof r.dinfo;
  }
  if (token && e_->scratch->argmax.p) {
    add(h, e_->scratch->argmax.p, 4);
    token_staged_ = true;
  }
  add(h + 8, e_->status.p, 8);  // the non-finite flags finish() checks
  status_staged_ = true;
  // the threshold report (dinfo) runs on the side stream (k::select_relay)
  if (e_->side_join) RK_CUDA(cudaStreamWaitEvent(st_, e_->side_join, 0));
  k::small_copies(st_, c);
  e_->launches += c.n > 0;
}

void Runner::resolve(ExtendResult& r, bool timings) {
  const rk_model_spec& s = w_->s;
  ExtendSlot& X = slot(r.slot);
  if (r.mode == RK_MODE_RELAY || r.mode == RK_MODE_BLEND) {
    if (r.staged >= 0) {  // landed with finish()'s synchronize
      const uint8_t* h = static_cast<const uint8_t*>(e_->results_host) + r.staged;
      std::memcpy(r.info, h, sizeof r.info);
      std::memcpy(r.dinfo, h + sizeof r.info, sizeof r.dinfo);
    } else {
      RK_CUDA(cudaMemcpy(r.info, X.info.p, sizeof r.info, cudaMemcpyDeviceToHost));
      RK_CUDA(cudaMemcpy(r.dinfo, X.dinfo.p, sizeof r.dinfo, cudaMemcpyDeviceToHost));
    }
  }
  const uint64_t count = (r.mode == RK_MODE_RELAY || r.mode == RK_MODE_BLEND) ? (uint64_t)r.info[0] : 0;
  rk_reuse_stats& st = r.stats;
  st = rk_reuse_stats{};
  st.total_entries = r.L * r.n;
  st.recomputed_entries = r.n * r.band_layers + count * r.sparse_layers;
  st.reuse_rate = st.total_entries == 0 ? 0.0
                                        : 1.0 - static_cast<double>(st.recomputed_entries) /
                                                    static_cast<double>(st.total_entries);
  st.selected_count = count;
  if ((r.mode == RK_MODE_RELAY || r.mode == RK_MODE_BLEND) && r.n > 0)
    e_->sel_frac = static_cast<double>(count) / static_cast<double>(r.n);
  st.selected_deviation = count ? (uint64_t)r.info[1] : 0;
  st.selected_influence_score = count ? (uint64_t)r.info[2] : 0;
  st.selected_influence_suffix = count ? (uint64_t)r.info[3] : 0;
  st.selected_blend = count ? (uint64_t)r.info[4] : 0;
  st.flops_full_equiv = rk_flops_span_full(&s, r.base, r.n);
  const double kvd = static_cast<double>(w_->kv()), nn = static_cast<double>(r.n);
  if (r.mode != RK_MODE_FULL) st.flops_realign = 3.0 * kvd * nn * static_cast<double>(s.num_layers);
  if (r.mode == RK_MODE_RELAY || r.mode == RK_MODE_BLEND) st.flops_selection = nn * (6.0 * kvd + 10.0) + 4.0 * nn;
  if (r.mode == RK_MODE_FULL) st.flops_cost = rk_flops_span_full(&s, r.base, r.n);
  if (r.mode == RK_MODE_RELAY || r.mode == RK_MODE_BLEND)
    st.flops_cost = rk_flops_segment_schedule(&s, r.base, r.n, r.l_start, r.l_det, r.sparse_hi, count);
  auto ms = [&](int a, int b) {
    float v = 0.f;
    if (timings && a >= 0 && b >= 0) RK_CUDA(cudaEventElapsedTime(&v, e_->events[a], e_->events[b]));
    return static_cast<double>(v);
  };
  st.wall.realign_ms = ms(r.ev_begin, r.ev_realign);
  st.wall.recompute_ms = ms(r.ev_realign, r.ev_band);
  st.wall.selection_ms = ms(r.ev_band, r.ev_select);
  st.wall.rectify_ms = ms(r.ev_select, r.ev_end);
  st.wall.total_ms = ms(r.ev_begin, r.ev_end);
  // ReuseStats::check_identity (relay_engine.cpp:57-66)
  if (st.recomputed_entries > st.total_entries) raise(RK_ERR_LOGIC, "reuse stats: recomputed exceeds total");
  r.resolved = true;
}

void Runner::segment_end_logits(rk_context* ctx, const ExtendResult& r) {
  const rk_model_spec& s = w_->s;
  ExtendSlot& X = slot(r.slot);
  uint64_t dep = 0;
  RK_CUDA(cudaMemcpyAsync(&dep, X.depth.as<uint64_t>() + (r.n - 1), 8, cudaMemcpyDeviceToHost, st_));
  RK_CUDA(cudaStreamSynchronize(st_));
  const float* row = X.hidden.as<float>() + (r.n - 1) * s.d_model;
  const uint64_t last_pos = r.base + r.n - 1;
  if (dep >= s.num_layers) last_row_logits(row);
  else row_logits_from_layer(ctx, row, dep, last_pos);
}

// run_workflow relay branch (workflow.cpp:316-369) / FULL (301-315)
void Runner::agent_prefill(rk_context* ctx, const int32_t* prefix, uint64_t n_prefix,
                           rk_cache* const* ups, uint64_t n_up, const int32_t* suffix, uint64_t n_suffix,
                           const rk_layer_profile* prof, const rk_relay_options& opts,
                           std::vector<ExtendResult>& results) {
  require(n_up == 0 || ups != nullptr, RK_ERR_INVALID_ARGUMENT, "null upstream caches");
  if (opts.mode == RK_MODE_FULL) {
    std::vector<int32_t> full(prefix, prefix + n_prefix);
    for (uint64_t u = 0; u < n_up; ++u) full.insert(full.end(), ups[u]->host_tokens.begin(), ups[u]->host_tokens.end());
    if (n_suffix) full.insert(full.end(), suffix, suffix + n_suffix);
    prefill(ctx, full.data(), full.size(), 0, true);
  } else if (e_->fused && n_up <= (uint64_t)k::kMaxFusedSegments) {
    agent_fused(ctx, prefix, n_prefix, ups, n_up, suffix, n_suffix, prof, opts, results);
  } else {
    prefill(ctx, prefix, n_prefix, 0, false);
    for (uint64_t u = 0; u < n_up; ++u) results.push_back(relay_extend(ctx, ups[u], prof, opts));
    if (n_suffix > 0) {
      prefill(ctx, suffix, n_suffix, ctx->size, true);
    } else {
      require(!results.empty(), RK_ERR_INVALID_ARGUMENT, "agent prefill: no suffix and no upstream segment");
      segment_end_logits(ctx, results.back());
    }
  }
  k::argmax(st_, e_->scratch->logits.as<float>(), (int)w_->s.vocab_size, e_->scratch->argmax.as<int>(),
            e_->scratch->argmax.as<char>() + 64);
  e_->launches += 2;
}

// ---------------------------------------------------------------------------
// Layer-major fused schedule of the downstream agent's prompt
// (run_workflow relay branch, workflow.cpp:316-369).
//
// The reference runs prefill(prefix), relay_extend per segment, prefill(suffix)
// one after another, each through all its layers. Each of those is a set of
// rows passing through run_layer_rows, which commits all rows' K/V before any
// attention and lets row r see exactly the cells at positions <= pos_r. So at
// every layer the rows of all phases can run as ONE row set: a row's inputs
// (its own hidden state, and the layer-l cells at earlier positions: fresh
// prefix K/V, band K/V, rectified K/V of selected rows, grafted K/V of the
// rest) are the same values the sequential order gives it -- later phases only
// ever read earlier positions, earlier phases only earlier positions. Results
// are identical (bit-identical in RK_FP32_EXACT; tests compare against the
// oracle's sequential order), with 16 layer passes instead of ~50 and weights
// streamed once per layer.
//
// Row layout of the pass buffer: [prefix | suffix | segment rows], where the
// segment rows are all segment rows during the band [l_start, l_det] and the
// compacted selected rows during (l_det, sparse_hi] (live count on the device).
// ---------------------------------------------------------------------------
void Runner::agent_fused(rk_context* ctx, const int32_t* prefix, uint64_t P, rk_cache* const* ups, uint64_t U,
                         const int32_t* suffix, uint64_t S, const rk_layer_profile* prof,
                         const rk_relay_options& opts, std::vector<ExtendResult>& results) {
  const rk_model_spec& s = w_->s;
  const int mode = opts.mode;
  const uint64_t L = s.num_layers, d = s.d_model;
  require(ctx != nullptr && ctx->w == w_, RK_ERR_INVALID_ARGUMENT, "context belongs to other weights");
  require(ctx->size == 0, RK_ERR_INVALID_ARGUMENT, "agent prefill: context must be empty");
  // prefill(prefix) checks (model.cpp:309-316)
  require(P > 0 && prefix != nullptr, RK_ERR_INVALID_ARGUMENT, "prefill: empty token chunk");
  require(P <= s.max_positions, RK_ERR_INVALID_ARGUMENT,
          "prefill: position overflow beyond max_positions " + std::to_string(s.max_positions));
  check_tokens(prefix, P);
  std::vector<uint64_t> base(U), n(U);
  std::vector<ExtendPlan> plan(U);
  uint64_t off = P;
  for (uint64_t u = 0; u < U; ++u) {
    plan[u] = plan_extend(off, ups[u], prof, opts);
    base[u] = off;
    n[u] = ups[u]->n;
    off += n[u];
  }
  if (S > 0) {
    require(suffix != nullptr, RK_ERR_INVALID_ARGUMENT, "null suffix");
    require(off + S <= s.max_positions, RK_ERR_INVALID_ARGUMENT,
            "prefill: position overflow beyond max_positions " + std::to_string(s.max_positions));
    check_tokens(suffix, S);
  }
  require(S > 0 || U > 0, RK_ERR_INVALID_ARGUMENT, "agent prefill: no suffix and no upstream segment");
  const uint64_t sbase = off, total = off + S, head = P + S, segrows = sbase - P;
  const bool segs = mode != RK_MODE_ZERO && U > 0;
  const uint64_t l_start = U ? plan[0].l_start : 0, l_det = U ? plan[0].l_det : 0;
  const uint64_t sparse_hi = U ? plan[0].sparse_hi : 0;

  ensure_rows(head + segrows);
  Scratch& Sc = *e_->scratch;
  float* H = Sc.hidden.as<float>();
  int* pos = Sc.positions.as<int>();
  Sc.sel_info.ensure(64 * 4);
  int* offs = Sc.sel_info.as<int>();  // [U+1]: row offset of each segment's selected rows, live count
  int* dtok_p = upload_tokens(prefix, P, tok_cursor_);
  tok_cursor_ += (int)P;
  int* dtok_s = nullptr;
  if (S) {
    dtok_s = upload_tokens(suffix, S, tok_cursor_);
    tok_cursor_ += (int)S;
  }

  results.clear();
  std::vector<rk_segment_marks> marks(U);
  std::vector<std::pair<void*, size_t>> zeros;
  for (uint64_t u = 0; u < U; ++u) {
    ExtendResult r;
    r.mode = mode;
    r.base = base[u];
    r.n = n[u];
    r.L = L;
    r.l_start = plan[u].l_start;
    r.l_det = plan[u].l_det;
    r.sparse_hi = plan[u].sparse_hi;
    r.slot = next_slot_++;
    ExtendSlot& X = slot(r.slot);
    X.hidden.ensure(n[u] * d * 4);
    X.depth.ensure(n[u] * 8);
    X.s_dev.ensure(n[u] * 8);
    X.s_key.ensure(n[u] * 8);
    X.sel_idx.ensure(n[u] * 4);
    X.sel_tags.ensure(2 * n[u] * 4);
    X.info.ensure(64);
    X.dinfo.ensure(64);
    X.score.ensure(n[u] * 8);
    zeros.emplace_back(X.info.p, 64);
    zeros.emplace_back(X.dinfo.p, 64);
    marks[u].base = base[u];
    marks[u].len = n[u];
    marks[u].origin.alloc_pooled(&e_->cache_pool, L * n[u]);  // pooled: freeing would sync the device
    zeros.emplace_back(marks[u].origin.p, L * n[u]);
    results.push_back(r);
  }
  static const bool zm = [] {
    const char* v = std::getenv("RK_ZERO_MANY");
    return v ? std::atoi(v) != 0 : true;
  }();
  if (zm) {
    k::zero_many(st_, zeros);  // selection counters, diagnostics and marks of every segment in one launch
    e_->launches += 1;
  } else {
    for (auto& z : zeros) k::zero_dev(st_, z.first, z.second);
    e_->launches += zeros.size();
  }
  const int ev_begin = event();
  // every cell is written before it is read: prefix / suffix rows by each
  // layer's QKV pass, segment rows by the graft (reused layers) or the band
  // recompute -- no zero fill needed
  ctx->resize(total, /*zero_fill=*/false);
  const size_t layer_stride = ctx->cap * w_->kv();
  const double2* rope = w_->rope->cs.as<double2>();
  int skip_lo = 1, skip_hi = 0;  // band layers are recomputed, never grafted
  if (mode == RK_MODE_RELAY) { skip_lo = (int)l_start; skip_hi = (int)l_det; }
  if (mode == RK_MODE_BLEND) { skip_lo = 0; skip_hi = 1; }
  bool streamed = false;  // some cache still arriving: graft layer by layer as the pass reaches it
  for (uint64_t u = 0; u < U; ++u) {
    streamed |= ups[u]->async;
    wait_cache_meta(ups[u]);
  }
  const size_t el = w_->elem, kvd = w_->kv();
  uint64_t n_all = 0;
  for (uint64_t u = 0; u < U; ++u) n_all += n[u];
  auto graft_layer = [&](uint64_t l) {  // realign + graft of layer l of every segment, one launch
    if ((int)l >= skip_lo && (int)l <= skip_hi) return;
    std::vector<k::RealignJob> jobs(U);
    for (uint64_t u = 0; u < U; ++u) {
      rk_cache* c = ups[u];
      wait_cache_layer(c, l);
      jobs[u] = {static_cast<char*>(c->k_pre.p) + l * n[u] * kvd * el, static_cast<char*>(c->v.p) + l * n[u] * kvd * el,
                 (int)n[u], (int)base[u]};
    }
    ProfScope ps(e_, "realign_graft", 3.0 * kvd * n_all, 4.0 * n_all * kvd * el);
    k::realign_graft_batch(st_, jobs.data(), (int)U, el, 1, (int)kvd, (int)s.d_head, rope,
                           static_cast<char*>(ctx->k.p) + l * layer_stride * el,
                           static_cast<char*>(ctx->v.p) + l * layer_stride * el, layer_stride, 1, 0);
    e_->launches += 1;
  };
  if (!streamed) {  // one launch: every segment, every grafted layer
    std::vector<k::RealignJob> jobs(U);
    for (uint64_t u = 0; u < U; ++u) jobs[u] = {ups[u]->k_pre.p, ups[u]->v.p, (int)n[u], (int)base[u]};
    const int grafted = (int)L - (skip_hi >= skip_lo ? skip_hi - skip_lo + 1 : 0);
    ProfScope ps(e_, "realign_graft", 3.0 * kvd * n_all * grafted, 4.0 * grafted * n_all * kvd * el);
    k::realign_graft_batch(st_, jobs.data(), (int)U, el, (int)L, (int)kvd, (int)s.d_head, rope, ctx->k.p, ctx->v.p,
                           layer_stride, skip_lo, skip_hi);
    e_->launches += 1;
  }
  const int ev_realign = event();
  // pass inputs: prefix / suffix embeddings, segment snapshots (or embeddings for BLEND)
  k::embed(st_, H, w_->emb, w_->elem, dtok_p, (int)P, (int)d, 0, nullptr);
  k::iota_positions(st_, pos, (int)P, 0);
  e_->launches += 2;
  if (S) {
    k::embed(st_, H + P * d, w_->emb, w_->elem, dtok_s, (int)S, (int)d, 0, nullptr);
    k::iota_positions(st_, pos + P, (int)S, (int)sbase);
    e_->launches += 2;
  }
  if (segs) {
    for (uint64_t u = 0; u < U; ++u) {
      float* dst = H + (head + base[u] - P) * d;
      if (mode == RK_MODE_RELAY)
        k::copy_dev(st_, dst, ups[u]->hidden.p, n[u] * d * 4);
      else
        k::embed(st_, dst, w_->emb, w_->elem, ups[u]->tokens.as<int>(), (int)n[u], (int)d, 0, nullptr);
      k::iota_positions(st_, pos + head + (base[u] - P), (int)n[u], (int)base[u]);
      e_->launches += 2;
    }
  }
  int ev_band = -1, ev_select = -1;
  for (uint64_t l = 0; l < L; ++l) {
    Rows rows{(int)head, nullptr, pos};
    if (segs && l >= l_start && l <= l_det) rows = Rows{(int)(head + segrows), nullptr, pos};
    else if (segs && l > l_det && l <= sparse_hi) {
      rows = Rows{(int)(head + segrows), offs + U, pos};
      rows.hint = live_hint(head, segrows);
    }
    rows.g1 = (int)P;
    rows.g2 = (int)head;
    // the row set grows at l = 0, at the band start and after the selected
    // rows are gathered (it only shrinks, to the head rows, after sparse_hi)
    if (l == 0 || (segs && (l == l_start || l == l_det + 1))) prepared_ = false;
    if (streamed) graft_layer(l);
    // top layer over the head rows only: just the suffix's last row feeds the
    // logits (no rows at all when the logits come from the segment end)
    const bool top_head = l + 1 == L && rows.rows_dev == nullptr && rows.rows_max == (int)head;
    run_layer(ctx, (int)l, H, rows, true, (int)total, nullptr, 0, 0, top_head ? (S > 0 ? 1 : 0) : -1);
    if (segs && l == l_det) {
      ev_band = event();
      for (uint64_t u = 0; u < U; ++u) {
        ExtendSlot& X = slot(results[u].slot);
        rk_cache* c = ups[u];
        k::copy_dev(st_, X.hidden.p, H + (head + base[u] - P) * d, n[u] * d * 4);
        k::set_depth(st_, X.depth.as<uint64_t>(), (int)n[u], l_det + 1);
        k::mark_layers(st_, marks[u].origin.as<uint8_t>(), (int)n[u], (int)l_start, (int)l_det);
        const size_t kv = w_->kv();
        wait_cache_layer(c, l_det);
        const char* ctx_v_det = static_cast<const char*>(ctx->v_layer(l_det)) + base[u] * kv * el;
        const char* cache_v_det = static_cast<const char*>(c->v.p) + l_det * n[u] * kv * el;
        if (mode == RK_MODE_RELAY) {
          const char* ctx_k_det = static_cast<const char*>(ctx->k_layer(l_det)) + base[u] * kv * el;
          const char* cache_k_det = static_cast<const char*>(c->k_pre.p) + l_det * n[u] * kv * el;
          {
            ProfScope ps(e_, "score_deviation", 0, 4.0 * n[u] * kv * el);
            k::score_deviation(st_, ctx_v_det, cache_v_det, ctx_k_det, cache_k_det, el, (int)n[u], (int)kv,
                               (int)s.num_kv_heads, (int)s.d_head, rope, (int)base[u], X.s_dev.as<double>(),
                               X.s_key.as<double>());
          }
          ProfScope ps(e_, "select_relay", 0, n[u] * 20.0);
          k::select_relay(st_, X.s_dev.as<double>(), c->influence.as<float>(), c->infl_mean.as<double>(),
                          (int)n[u], opts.tau_dev, opts.tau_inf, (int)std::min<uint64_t>(opts.suffix_k, 0x7fffffff),
                          X.sel_idx.as<int>(), X.sel_tags.as<uint32_t>(), X.info.as<int>(), X.dinfo.as<double>(),
                          e_->side, e_->side_fork, e_->side_join);
          e_->launches += 1;  // the side-stream report kernel
        } else {
          k::blend_scores(st_, ctx_v_det, cache_v_det, el, (int)n[u], (int)kv, X.score.as<double>());
          size_t count = static_cast<size_t>(opts.blend_alpha * static_cast<double>(n[u]));
          if (count > n[u]) count = n[u];
          results[u].blend_count = (int)count;
          k::select_topk(st_, X.score.as<double>(), (int)n[u], (int)count, X.sel_idx.as<int>(),
                         X.sel_tags.as<uint32_t>(), X.info.as<int>());
          e_->launches += 1;
        }
        e_->launches += 5;
        results[u].band_layers = l_det - l_start + 1;
      }
      ev_select = event();
      if (sparse_hi > l_det) {  // compact the selected rows of every segment after [prefix | suffix]
        k::SegCounts cnt{};
        for (uint64_t u = 0; u < U; ++u) cnt.count[u] = slot(results[u].slot).info.as<int>();
        k::segment_offsets(st_, cnt, (int)U, (int)head, offs);
        e_->launches += 1;
        for (uint64_t u = 0; u < U; ++u) {
          ExtendSlot& X = slot(results[u].slot);
          k::gather_rows_to(st_, H, offs + u, X.hidden.as<float>(), X.sel_idx.as<int>(), X.info.as<int>(), (int)n[u],
                            (int)d, pos, (int)base[u]);
          e_->launches += 1;
        }
      }
    }
    if (segs && l == sparse_hi && sparse_hi > l_det) {
      for (uint64_t u = 0; u < U; ++u) {
        ExtendSlot& X = slot(results[u].slot);
        k::scatter_rows_from(st_, X.hidden.as<float>(), H, offs + u, X.sel_idx.as<int>(), X.info.as<int>(), (int)n[u],
                             (int)d, X.depth.as<uint64_t>(), sparse_hi + 1);
        k::mark_rows(st_, marks[u].origin.as<uint8_t>(), (int)n[u], (int)l_det + 1, (int)sparse_hi,
                     X.sel_idx.as<int>(), X.info.as<int>(), (int)n[u]);
        e_->launches += 2;
        results[u].sparse_layers = sparse_hi - l_det;
      }
    }
  }
  if (!segs) {  // ZERO (relay_engine.cpp:224-234): the segment keeps its snapshot
    for (uint64_t u = 0; u < U; ++u) {
      ExtendSlot& X = slot(results[u].slot);
      k::copy_dev(st_, X.hidden.p, ups[u]->hidden.p, n[u] * d * 4);
      k::set_depth(st_, X.depth.as<uint64_t>(), (int)n[u], ups[u]->snapshot);
      e_->launches += 1;
    }
  }
  const int ev_end = event();
  for (uint64_t u = 0; u < U; ++u) {
    ExtendResult& r = results[u];
    r.ev_begin = ev_begin;
    r.ev_realign = ev_realign;
    r.ev_band = ev_band >= 0 ? ev_band : ev_end;
    r.ev_select = ev_select >= 0 ? ev_select : r.ev_band;
    r.ev_end = ev_end;
    ctx->segs.push_back(std::move(marks[u]));
    r.seg_index = ctx->segs.size() - 1;
  }
  if (S > 0) last_row_logits(H + (head - 1) * d);
  else segment_end_logits(ctx, results.back());
}

// ---------------------------------------------------------------------------
// device capture (RelayRecorder, relay_cache.cpp:52-136)
// ---------------------------------------------------------------------------
static rk_cache* new_cache(rk_engine* e, rk_weights* w, uint64_t n, uint64_t src, uint64_t snapshot) {
  const rk_model_spec& s = w->s;
  auto c = std::make_unique<rk_cache>();
  c->e = e;
  c->precision = w->precision;
  c->elem = w->elem;
  c->L = s.num_layers;
  c->Hkv = s.num_kv_heads;
  c->dh = s.d_head;
  c->d = s.d_model;
  c->n = n;
  c->maxpos = s.max_positions;
  c->theta = s.theta_base;
  c->src_base = src;
  c->snapshot = snapshot;
  c->steps = n;
  const size_t kv = c->kv();
  BlockPool* pl = &e->cache_pool;
  c->tokens.alloc_pooled(pl, n * 4);
  c->k_pre.alloc_pooled(pl, c->L * n * kv * c->elem);
  c->v.alloc_pooled(pl, c->L * n * kv * c->elem);
  c->hidden.alloc_pooled(pl, n * c->d * 4);
  c->influence.alloc_pooled(pl, n * 4);
  c->infl_mean.alloc_pooled(pl, 8);
  c->host_tokens.resize(n);
  return c.release();
}

rk_cache* Runner::capture_prefill(rk_context* ctx, const int32_t* tokens, uint64_t n, uint64_t snapshot,
                                  bool include_self) {
  const rk_model_spec& s = w_->s;
  require(snapshot < s.num_layers, RK_ERR_INVALID_ARGUMENT, "recorder: snapshot layer out of range");
  require(n > 0 && tokens != nullptr, RK_ERR_INVALID_ARGUMENT, "prefill: empty token chunk");
  const uint64_t src = ctx->size;
  require(src + n <= s.max_positions, RK_ERR_INVALID_ARGUMENT, "prefill: position overflow beyond max_positions");
  check_tokens(tokens, n);
  std::unique_ptr<rk_cache> c(new_cache(e_, w_, n, src, snapshot));
  std::memcpy(c->host_tokens.data(), tokens, n * 4);
  RK_CUDA(cudaMemcpyAsync(c->tokens.p, tokens, n * 4, cudaMemcpyHostToDevice, st_));
  const size_t d = s.d_model, kv = w_->kv(), H = s.num_heads;
  // chunked prefill == one-shot prefill (test_model.cpp:102-115); chunks
  // bound the captured attention rows to chunk x H x n floats.
  const uint64_t chunk = std::min<uint64_t>(n, std::max<uint64_t>(1, (256ull << 20) / (H * n * 4)));
  ensure_rows(chunk);
  Scratch& S = *e_->scratch;
  DevBuf acc(n * 8), probs(chunk * H * n * 4);
  k::zero_dev(st_, acc.p, n * 8);
  ctx->resize(src + n);
  for (uint64_t c0 = 0; c0 < n; c0 += chunk) {
    const uint64_t m = std::min(chunk, n - c0);
    k::embed(st_, S.hidden.as<float>(), w_->emb, w_->elem, c->tokens.as<int>() + c0, (int)m, (int)d, 0, nullptr);
    k::iota_positions(st_, S.positions.as<int>(), (int)m, (int)(src + c0));
    e_->launches += 2;
    Rows rows{(int)m, nullptr, S.positions.as<int>()};
    prepared_ = false;
    for (uint64_t l = 0; l < s.num_layers; ++l) {
      if (l == snapshot)
        k::copy_dev(st_, c->hidden.as<float>() + c0 * d, S.hidden.p, m * d * 4);
      cap_k_ = static_cast<float*>(static_cast<void*>(static_cast<char*>(c->k_pre.p) + (l * n + c0) * kv * c->elem));
      cap_v_ = static_cast<float*>(static_cast<void*>(static_cast<char*>(c->v.p) + (l * n + c0) * kv * c->elem));
      run_layer(ctx, (int)l, S.hidden.as<float>(), rows, true, (int)(src + c0 + m), probs.as<float>(), (int)src, (int)n);
      cap_k_ = cap_v_ = nullptr;
      k::influence_accum(st_, acc.as<double>(), probs.as<float>(), rows, (int)H, (int)src, (int)n, include_self);
      e_->launches += 1;
    }
  }
  k::doubles_to_floats(st_, c->influence.as<float>(), acc.as<double>(), (int)n);
  k::seq_mean(st_, c->influence.as<float>(), (int)n, c->infl_mean.as<double>());
  e_->launches += 2;
  RK_CUDA(cudaStreamSynchronize(st_));
  return c.release();
}

// Greedy decode with capture, one row per step (greedy_generate,
// model.cpp:372-389, feeding RelayRecorder, relay_cache.cpp:68-127). A step's
// ~10 kernels per layer are launch-bound on the host, so the step is recorded
// once as a CUDA graph and replayed: its position, token and capture slots come
// from a device step counter (decode_step_begin/end), the context is sized for
// all n steps up front (keys past a step's position are masked by causality),
// and the captured K_pre / V / snapshot rows go through fixed staging buffers.
// Step 0 runs eagerly (it sizes every buffer the graph then reuses); the last
// step, which needs no next-token logits, too. RK_DECODE_GRAPH=0: all eager.
rk_cache* Runner::capture_decode(rk_context* ctx, const float* first_logits, uint64_t n, uint64_t snapshot,
                                 bool include_self) {
  const rk_model_spec& s = w_->s;
  require(snapshot < s.num_layers, RK_ERR_INVALID_ARGUMENT, "recorder: snapshot layer out of range");
  require(n > 0, RK_ERR_INVALID_ARGUMENT, "capture: zero decode steps");
  const uint64_t src = ctx->size;
  require(src + n <= s.max_positions, RK_ERR_INVALID_ARGUMENT, "prefill: position overflow beyond max_positions");
  std::unique_ptr<rk_cache> c(new_cache(e_, w_, n, src, snapshot));
  ensure_rows(1);
  Scratch& S = *e_->scratch;
  const size_t d = s.d_model, kv = w_->kv(), H = s.num_heads, V = s.vocab_size, L = s.num_layers, el = c->elem;
  if (first_logits) RK_CUDA(cudaMemcpyAsync(S.logits.p, first_logits, V * 4, cudaMemcpyHostToDevice, st_));
  DevBuf acc(n * 8), probs(H * n * 4);
  const size_t row_bytes = kv * el;
  DevBuf stage(2 * L * row_bytes + d * 4 + 64);  // [K_pre rows | V rows | snapshot row | step, token, next token]
  char* sk = static_cast<char*>(stage.p);
  char* sv = sk + L * row_bytes;
  char* sh = sv + L * row_bytes;
  int* ints = reinterpret_cast<int*>(sh + d * 4);
  int *step = ints, *cur_tok = ints + 1, *next_tok = ints + 2;
  k::zero_dev(st_, acc.p, n * 8);
  k::zero_dev(st_, ints, 16);
  int* tok = c->tokens.as<int>();
  // greedy_generate (model.cpp:372-389): next = argmax(prompt-end logits)
  k::argmax(st_, S.logits.as<float>(), (int)V, tok, S.argmax.as<char>() + 64);
  e_->launches += 4;
  ctx->resize(src + n);
  auto one_step = [&](bool logits) {
    k::decode_step_begin(st_, step, (int)src, tok, cur_tok, S.positions.as<int>());
    k::embed(st_, S.hidden.as<float>(), w_->emb, w_->elem, cur_tok, 1, (int)d, 0, nullptr);
    e_->launches += 2;
    Rows rows{1, nullptr, S.positions.as<int>()};
    prepared_ = false;
    for (uint64_t l = 0; l < L; ++l) {
      if (l == snapshot) {
        k::copy_dev(st_, sh, S.hidden.p, d * 4);
        e_->launches += 1;
      }
      cap_k_ = reinterpret_cast<float*>(sk + l * row_bytes);
      cap_v_ = reinterpret_cast<float*>(sv + l * row_bytes);
      run_layer(ctx, (int)l, S.hidden.as<float>(), rows, true, (int)(src + n), probs.as<float>(), (int)src, (int)n);
      cap_k_ = cap_v_ = nullptr;
      k::influence_accum(st_, acc.as<double>(), probs.as<float>(), rows, (int)H, (int)src, (int)n, include_self);
      e_->launches += 1;
    }
    if (logits) {
      last_row_logits(S.hidden.as<float>());
      k::argmax(st_, S.logits.as<float>(), (int)V, next_tok, S.argmax.as<char>() + 64);
      e_->launches += 2;
    }
    k::decode_step_end(st_, step, (int)n, (int)L, row_bytes, sk, sv, c->k_pre.p, c->v.p, d * 4, sh, c->hidden.p,
                       logits ? next_tok : nullptr, tok);
    e_->launches += 1;
  };
  static const bool graph_env = [] {
    const char* v = std::getenv("RK_DECODE_GRAPH");
    return v ? std::atoi(v) != 0 : true;
  }();
  const bool graph = graph_env && n >= 4 && !(e_->prof && e_->prof->on);
  if (!graph) {
    for (uint64_t t = 0; t < n; ++t) one_step(t + 1 < n);
  } else {
    one_step(true);  // step 0, eagerly: every buffer and kernel attribute the graph reuses is set up here
    const uint64_t l0 = e_->launches;
    cudaGraph_t g = nullptr;
    RK_CUDA(cudaStreamBeginCapture(st_, cudaStreamCaptureModeRelaxed));
    try {
      one_step(true);
    } catch (...) {
      cudaGraph_t tmp = nullptr;
      cudaStreamEndCapture(st_, &tmp);
      if (tmp) cudaGraphDestroy(tmp);
      throw;
    }
    RK_CUDA(cudaStreamEndCapture(st_, &g));
    const uint64_t per_step = e_->launches - l0;
    cudaGraphExec_t ge = nullptr;
    const cudaError_t ierr = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    RK_CUDA(ierr);
    for (uint64_t t = 1; t + 1 < n; ++t) {
      const cudaError_t lerr = cudaGraphLaunch(ge, st_);
      if (lerr != cudaSuccess) {
        cudaGraphExecDestroy(ge);
        RK_CUDA(lerr);
      }
    }
    e_->launches += per_step * (n - 3);  // (the captured step's launches were counted once already)
    one_step(false);                     // the last step: no next-token logits
    RK_CUDA(cudaStreamSynchronize(st_));
    RK_CUDA(cudaGraphExecDestroy(ge));
  }
  k::doubles_to_floats(st_, c->influence.as<float>(), acc.as<double>(), (int)n);
  k::seq_mean(st_, c->influence.as<float>(), (int)n, c->infl_mean.as<double>());
  e_->launches += 2;
  RK_CUDA(cudaMemcpyAsync(c->host_tokens.data(), tok, n * 4, cudaMemcpyDeviceToHost, st_));
  RK_CUDA(cudaStreamSynchronize(st_));
  return c.release();
}

// ---------------------------------------------------------------------------
void Runner::finish() {
  RK_CUDA(cudaStreamSynchronize(st_));
  if (e_->side) RK_CUDA(cudaStreamSynchronize(e_->side));
  RK_CUDA(cudaGetLastError());
  int flags[2] = {0, 0};
  if (status_staged_) std::memcpy(flags, static_cast<const uint8_t*>(e_->results_host) + 8, sizeof flags);
  else RK_CUDA(cudaMemcpy(flags, e_->status.p, sizeof flags, cudaMemcpyDeviceToHost));
  if (flags[0]) raise(RK_ERR_NONFINITE, "matmul: non-finite value");
}

void Runner::fill_output(ExtendResult& r, rk_context* ctx, rk_relay_output* out) {
  if (!r.resolved) resolve(r);
  if (!out) return;
  const rk_model_spec& s = w_->s;
  ExtendSlot& X = slot(r.slot);
  const uint64_t n = r.n, count = r.stats.selected_count;
  out->segment_base = r.base;
  out->segment_len = n;
  out->selection_count = count;
  out->s_dev_len = r.mode == RK_MODE_RELAY ? n : 0;
  out->dev_threshold = r.mode == RK_MODE_RELAY ? r.dinfo[0] : 0.0;
  out->min_dev_margin = r.mode == RK_MODE_RELAY ? r.dinfo[1] : 0.0;
  out->stats = r.stats;
  if (count && (out->selection_indices || out->selection_tags)) {
    std::vector<int> idx(count);
    std::vector<uint32_t> tags(count);
    RK_CUDA(cudaMemcpy(idx.data(), X.sel_idx.p, count * 4, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(tags.data(), X.sel_tags.p, count * 4, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < count; ++i) {
      if (out->selection_indices) out->selection_indices[i] = (uint64_t)idx[i];
      if (out->selection_tags) out->selection_tags[i] = tags[i];
    }
  }
  if (r.mode == RK_MODE_RELAY) {
    if (out->s_dev) RK_CUDA(cudaMemcpy(out->s_dev, X.s_dev.p, n * 8, cudaMemcpyDeviceToHost));
    if (out->s_key_dev) RK_CUDA(cudaMemcpy(out->s_key_dev, X.s_key.p, n * 8, cudaMemcpyDeviceToHost));
  }
  if (out->segment_hidden) RK_CUDA(cudaMemcpy(out->segment_hidden, X.hidden.p, n * s.d_model * 4, cudaMemcpyDeviceToHost));
  if (out->hidden_depth) RK_CUDA(cudaMemcpy(out->hidden_depth, X.depth.p, n * 8, cudaMemcpyDeviceToHost));
  if (out->origin) RK_CUDA(cudaMemcpy(out->origin, ctx->segs[r.seg_index].origin.p, s.num_layers * n, cudaMemcpyDeviceToHost));
}

void Runner::download_logits(float* dst) {
  require(have_logits_, RK_ERR_LOGIC, "no logits were computed");
  RK_CUDA(cudaMemcpy(dst, e_->scratch->logits.p, w_->s.vocab_size * 4, cudaMemcpyDeviceToHost));
}

int32_t Runner::first_token() {
  int32_t t = 0;
  if (token_staged_) std::memcpy(&t, e_->results_host, 4);
  else RK_CUDA(cudaMemcpy(&t, e_->scratch->argmax.p, 4, cudaMemcpyDeviceToHost));
  return t;
}

// ---------------------------------------------------------------------------
void layer_unpack_tensor(rk_weights* w, size_t idx, float* dst, size_t rows, size_t cols) {
  const rk_model_spec& s = w->s;
  cudaStream_t st = w->e->stream;
  const size_t d = s.d_model, q = w->q(), kv = w->kv(), ff = s.d_ff;
  const bool bf = w->precision == RK_BF16;
  auto plain = [&](const void* src) {
    if (bf) k::bf16_to_f32(st, dst, static_cast<const __nv_bfloat16*>(src), rows * cols);
    else RK_CUDA(cudaMemcpyAsync(dst, src, rows * cols * 4, cudaMemcpyDeviceToDevice, st));
  };
  auto strided = [&](const void* src, size_t ld_exact, size_t c0, size_t cs, size_t ld_t,
                     const float* gain = nullptr) {
    if (bf) k::untranspose_bf16(st, dst, static_cast<const __nv_bfloat16*>(src), ld_t, c0, cs, rows, cols, gain);
    else k::copy2d_f32(st, dst, cols, 1, static_cast<const float*>(src) + c0, ld_exact, cs, rows, cols);
  };
  auto f32 = [&](const float* src) { RK_CUDA(cudaMemcpyAsync(dst, src, rows * cols * 4, cudaMemcpyDeviceToDevice, st)); };
  if (idx == 0) { plain(w->emb); return; }
  size_t i = idx - 1;
  if (i < 9 * s.num_layers) {
    const rk_layer_dev& ly = w->layers[i / 9];
    switch (i % 9) {
      case 0: f32(ly.attn_norm); break;
      case 1: strided(ly.w_qkv, q + 2 * kv, 0, 1, d, ly.attn_norm); break;
      case 2: strided(ly.w_qkv, q + 2 * kv, q, 1, d, ly.attn_norm); break;
      case 3: strided(ly.w_qkv, q + 2 * kv, q + kv, 1, d, ly.attn_norm); break;
      case 4: strided(ly.w_o, d, 0, 1, q); break;
      case 5: f32(ly.mlp_norm); break;
      case 6: strided(ly.w_gu, 2 * ff, 0, 2, d, ly.mlp_norm); break;
      case 7: strided(ly.w_gu, 2 * ff, 1, 2, d, ly.mlp_norm); break;
      default: strided(ly.w_down, d, 0, 1, ff); break;
    }
    return;
  }
  i -= 9 * s.num_layers;
  if (i == 0) { f32(w->final_norm); return; }
  strided(w->head, s.vocab_size, 0, 1, d);
}

}  // namespace rk
