// layer.h -- per-call orchestration (Runner) shared by the C ABI entry points.
#pragma once

#include <vector>

#include "internal.h"

namespace rk {

// Device-side state of one relay_extend, resolved on the host by finish().
struct ExtendResult {
  int mode = RK_MODE_RELAY;
  uint64_t base = 0, n = 0, L = 0;
  uint64_t band_layers = 0, sparse_layers = 0;  // recomputed = n*band + |I|*sparse
  int slot = 0;                                 // scratch slot holding device buffers
  size_t seg_index = 0;                         // SegmentMarks index in the context
  int ev_begin = -1, ev_realign = -1, ev_band = -1, ev_select = -1, ev_end = -1;
  int blend_count = 0;
  uint64_t l_start = 0, l_det = 0, sparse_hi = 0;
  bool resolved = false;
  // host copies after finish()
  int info[8] = {0};
  double dinfo[2] = {0, 0};
  int staged = -1;  // byte offset of info/dinfo in rk_engine::results_host (stage_results), -1: not staged
  rk_reuse_stats stats{};
};

struct ExtendPlan {
  uint64_t l_start = 0, l_det = 0, sparse_hi = 0;
};

// Grow-only device buffers of one extend slot.
struct ExtendSlot {
  DevBuf hidden, sub_hidden, depth, s_dev, s_key, sel_idx, sel_tags, info, dinfo, sub_pos, score;
};

class Runner {
 public:
  Runner(rk_engine* e, rk_weights* w);
  ~Runner();

  void prefill(rk_context* ctx, const int32_t* tokens, uint64_t n, uint64_t base, bool want_logits);
  // prefill with capture into host buffers (rk_prefill_trace)
  void prefill_trace(rk_context* ctx, const int32_t* tokens, uint64_t n, uint64_t base,
                     const rk_trace_request& req);
  ExtendResult relay_extend(rk_context* ctx, rk_cache* cache, const rk_layer_profile* prof,
                            const rk_relay_options& opts);
  // relay_prefill's next-token logits at the segment end (relay_engine.cpp:381-393)
  void segment_end_logits(rk_context* ctx, const ExtendResult& res);
  void agent_prefill(rk_context* ctx, const int32_t* prefix, uint64_t n_prefix,
                     rk_cache* const* ups, uint64_t n_up, const int32_t* suffix, uint64_t n_suffix,
                     const rk_layer_profile* prof, const rk_relay_options& opts,
                     std::vector<ExtendResult>& results);
  rk_cache* capture_prefill(rk_context* ctx, const int32_t* tokens, uint64_t n, uint64_t snapshot,
                            bool include_self);
  rk_cache* capture_decode(rk_context* ctx, const float* first_logits, uint64_t n,
                           uint64_t snapshot, bool include_self);

  // Synchronize, raise on device-side errors, resolve pending ExtendResults.
  // queue the results' small device values (and the first token) for one
  // asynchronous copy each into pinned memory ahead of finish(), so resolve()
  // and first_token() need no further device round trips
  void stage_results(std::vector<ExtendResult>& rs, bool token);
  void finish();
  void resolve(ExtendResult& r, bool timings = true);  // after finish(): counts, stats (+ event timings)
  // expected live rows of a sparse pass over `head` fixed rows plus the
  // selected ones of `seg` segment rows: the last observed selection fraction,
  // 0 when none was observed yet (the grids cover rows_max regardless; the
  // hint only picks tile shapes and the split-KV plan)
  int live_hint(uint64_t head, uint64_t seg) const {
    if (e_->sel_frac < 0) return 0;
    const double sel = e_->sel_frac * static_cast<double>(seg) + 0.5;
    return static_cast<int>(std::min<double>(static_cast<double>(head + seg), static_cast<double>(head) + sel));
  }
  void fill_output(ExtendResult& res, rk_context* ctx, rk_relay_output* out);
  void download_logits(float* dst);
  // row_logits_from_layer (model.cpp:339-362) of a device hidden row into scratch logits
  void row_logits_from_layer(rk_context* ctx, const float* hidden_row, uint64_t first_layer,
                             uint64_t position);
  int32_t first_token();

  void begin_timer();
  float lap_ms();  // ms since begin_timer (synchronizes)

 private:
  // one decoder layer over a row set (run_layer_rows, model.cpp:237-280)
  void run_layer(rk_context* ctx, int layer, float* hidden, Rows rows, bool commit, int max_ctx,
                 float* probs = nullptr, int key_lo = 0, int key_n = 0, int tail = -1);
  void last_row_logits(const float* hidden_row);  // output_logits (model.cpp:282-288)
  ExtendPlan plan_extend(uint64_t base, rk_cache* cache, const rk_layer_profile* prof,
                         const rk_relay_options& opts);
  void agent_fused(rk_context* ctx, const int32_t* prefix, uint64_t P, rk_cache* const* ups, uint64_t U,
                   const int32_t* suffix, uint64_t S, const rk_layer_profile* prof, const rk_relay_options& opts,
                   std::vector<ExtendResult>& results);
  void ensure_rows(size_t rows);
  int* upload_tokens(const int32_t* tokens, uint64_t n, int slot);
  void check_tokens(const int32_t* tokens, uint64_t n);
  int event();
  ExtendSlot& slot(int i);
  void wait_cache_meta(rk_cache* c);
  void wait_cache_layer(rk_cache* c, uint64_t layer);

  rk_engine* e_;
  rk_weights* w_;
  cudaStream_t st_;
  std::vector<ExtendResult*> pending_;
  int next_event_ = 0;
  int next_slot_ = 0;
  int timer_ev_ = -1;
  bool have_logits_ = false;
  int tok_cursor_ = 0;
  float* cap_k_ = nullptr;  // capture destinations for pre-RoPE K / V rows
  float* cap_v_ = nullptr;
  // bf16 path: the last layer left its rows' fused-RMSNorm inputs (bf16 rows,
  // 1/rms) for the same row set; cleared whenever the rows or hidden change.
  bool prepared_ = false;
  bool token_staged_ = false, status_staged_ = false;
};

// weights_export helper: unpack tensor idx of the engine layout to fp32 [rows x cols].
void layer_unpack_tensor(rk_weights* w, size_t idx, float* dst, size_t rows, size_t cols);

// bf16 layer path (layer_bf16.cu)
// prepared: the rows' bf16 copy and 1/rms were left by the previous layer's
// residual GEMM (same row set); otherwise they are computed first.
// tail >= 0: only the last `tail` rows go past the QKV GEMM (all rows' K/V are
// still committed) -- the top layer when only the last row's output is used.
void run_layer_bf16(rk_engine* e, rk_weights* w, rk_context* ctx, int layer, float* hidden,
                    Rows rows, bool commit, int max_ctx, float* probs, int key_lo, int key_n,
                    void* cap_k, void* cap_v, bool prepared, int tail = -1);
void last_row_logits_bf16(rk_engine* e, rk_weights* w, const float* hidden_row, float* logits);
// output_logits over a row set (model.cpp:282-288): logits [rows][V] fp32
void rows_logits_bf16(rk_engine* e, rk_weights* w, const float* hidden, Rows rows, float* logits);

}  // namespace rk
