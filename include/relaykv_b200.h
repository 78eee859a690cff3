/*
 * relaykv_b200.h -- C ABI of the B200-native RelayCaching relay-prefill engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (BASELINE.json north_star). The reference exposes a
 * C++ API only (/root/reference/proj/include/relaykv/relay_engine.hpp:142-163,
 * model.hpp:116-152); every entry point below replaces one reference function
 * and is cited next to it. Plain pointers and sizes only: no torch or CUDA
 * types cross this boundary. The C++ drop-in (namespace relaykv, same headers
 * as the reference) and the Python host mirror both sit on top of it.
 *
 * Conventions
 *  - Every call returns an rk_status. A non-zero status maps 1:1 to the
 *    exception type the reference throws on the same condition (see
 *    rk_status); rk_last_error() returns the message (thread-local).
 *  - Host output pointers are optional: NULL means "do not copy back". With all
 *    output pointers NULL a call is device-resident end to end.
 *  - Layouts are the reference's: row-major fp32, x.W convention,
 *    KVContext rows [layer][pos][kv_dim] with head h at [h*d_head,(h+1)*d_head),
 *    SegmentMarks origin layer-major [L x n] (relay_engine.hpp:26-35).
 */
#ifndef RELAYKV_B200_H_
#define RELAYKV_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RK_ABI_VERSION 1

/* Status codes, one per reference exception type on this path
 * (SURVEY.md 8(b) "Errors"). */
typedef enum rk_status {
  RK_OK = 0,
  RK_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (shapes, capacity, snapshot, alpha) */
  RK_ERR_SCHEMA = 2,           /* relaykv::SchemaError (profile window, profiler.cpp:28-35) */
  RK_ERR_LOGIC = 3,            /* std::logic_error (accounting, relay_engine.cpp:57-66) */
  RK_ERR_NONFINITE = 4,        /* std::runtime_error "<what>: non-finite value" (tensor.cpp:58-64) */
  RK_ERR_RUNTIME = 5,          /* other std::runtime_error: CUDA failure, out of memory */
  RK_ERR_IO = 6                /* relaykv::IoError (errors.hpp:12): cannot open / read / write a file */
} rk_status;

/* Numerics of a weights object (and of everything computed with it).
 *  RK_FP32_EXACT: fp32 storage; every kernel replays the reference's
 *    operation order (sequential-k matmul without FMA, glibc-identical expf,
 *    double RoPE from a host cos/sin table) so results are bit-identical to
 *    the reference CPU path.
 *  RK_BF16: bf16 weights and KV context, tcgen05 tensor-core GEMMs with fp32
 *    accumulation, flash attention; throughput mode, reports its own error.
 *  RK_FP32_TC: fp32-accurate tensor-core mode: RK_FP32_EXACT's storage and
 *    relay kernels, matmuls as 3xTF32 on tcgen05 (hi/lo split, fp32
 *    accumulation) and an fp32 flash attention; not bit-identical, relative
 *    error ~1e-6 (north_star's "fp32-accumulate mode <= 1e-4 relative"). */
typedef enum rk_precision { RK_FP32_EXACT = 0, RK_BF16 = 1, RK_FP32_TC = 2 } rk_precision;

/* RelayMode (relay_engine.hpp:17-22). */
typedef enum rk_relay_mode {
  RK_MODE_FULL = 0,
  RK_MODE_ZERO = 1,
  RK_MODE_RELAY = 2,
  RK_MODE_BLEND = 3
} rk_relay_mode;

/* SelectionTag bits (selector.hpp:21-26). */
enum {
  RK_SEL_DEVIATION = 1u << 0,
  RK_SEL_INFLUENCE_SCORE = 1u << 1,
  RK_SEL_INFLUENCE_SUFFIX = 1u << 2,
  RK_SEL_BLEND_TOPK = 1u << 3
};

/* ModelSpec (model.hpp:21-38). */
typedef struct rk_model_spec {
  uint64_t num_layers;
  uint64_t d_model;
  uint64_t num_heads;
  uint64_t num_kv_heads;
  uint64_t d_head;
  uint64_t d_ff;
  uint64_t vocab_size;
  float theta_base;
  uint64_t max_positions;
  float norm_eps;
} rk_model_spec;

/* LayerProfile's window (profiler.hpp:30-43): l_start <= l_det <= l_end < L. */
typedef struct rk_layer_profile {
  uint64_t l_start;
  uint64_t l_det;
  uint64_t l_end;
} rk_layer_profile;

/* RelayOptions + SelectionThresholds (relay_engine.hpp:119-126, selector.hpp:13-19). */
typedef struct rk_relay_options {
  int32_t mode;              /* rk_relay_mode */
  double tau_dev;            /* 1.5 */
  double tau_inf;            /* 1.45 */
  uint64_t suffix_k;         /* 10 */
  double blend_alpha;        /* 0.2, BLEND only: recompute ratio */
  int32_t rectify_above_end; /* ablation flag */
} rk_relay_options;

/* Host view of a RelayCache (relay_cache.hpp:23-46); all arrays fp32 / int32. */
typedef struct rk_relay_cache_view {
  uint64_t num_layers;
  uint64_t num_kv_heads;
  uint64_t d_head;
  uint64_t d_model;
  float theta_base;
  uint64_t max_positions;
  uint64_t segment_len;
  const int32_t* segment_tokens; /* [n] */
  uint64_t source_base_position;
  uint64_t snapshot_layer;
  uint64_t decode_steps_observed;
  const float* const* k_pre;    /* [L] -> [n x kv_dim], keys BEFORE rotation */
  const float* const* v;        /* [L] -> [n x kv_dim] */
  const float* hidden_snapshot; /* [n x d_model], input to snapshot_layer */
  const float* influence;       /* [n], >= 0 */
} rk_relay_cache_view;

/* PhaseTimings (relay_engine.hpp:42-49). Device phases are CUDA-event times. */
typedef struct rk_phase_timings {
  double fresh_ms, realign_ms, recompute_ms, selection_ms, rectify_ms, total_ms;
} rk_phase_timings;

/* ReuseStats (relay_engine.hpp:53-71). */
typedef struct rk_reuse_stats {
  uint64_t total_entries;
  uint64_t recomputed_entries;
  double reuse_rate;
  uint64_t selected_count;
  uint64_t selected_deviation;
  uint64_t selected_influence_score;
  uint64_t selected_influence_suffix;
  uint64_t selected_blend;
  double flops_cost;
  double flops_selection;
  double flops_realign;
  double flops_full_equiv;
  rk_phase_timings wall;
} rk_reuse_stats;

/* RelayOutput (relay_engine.hpp:128-137) + SegmentMarks of the new segment.
 * Caller-owned host buffers sized for the segment length n; any may be NULL. */
typedef struct rk_relay_output {
  uint64_t* selection_indices; /* [n] sorted ascending */
  uint32_t* selection_tags;    /* [n] RK_SEL_* bits */
  double* s_dev;               /* [n] value deviation at l_det (RELAY only) */
  double* s_key_dev;           /* [n] key deviation at l_det (RELAY only) */
  float* segment_hidden;       /* [n x d_model] */
  uint64_t* hidden_depth;      /* [n] */
  uint8_t* origin;             /* [L x n] layer-major, 0 reused / 1 recomputed */
  /* filled by the call */
  uint64_t segment_base;
  uint64_t segment_len;
  uint64_t selection_count;
  uint64_t s_dev_len;          /* n in RELAY mode, else 0 (reference leaves them empty) */
  double dev_threshold;        /* tau_dev * mean(s_dev), or 0 */
  double min_dev_margin;       /* min_j |s_dev[j]-thr|/thr: selection certification margin */
  rk_reuse_stats stats;
} rk_relay_output;

typedef struct rk_engine rk_engine;
typedef struct rk_weights rk_weights;
typedef struct rk_cache rk_cache;
typedef struct rk_context rk_context;

/* ---- engine ------------------------------------------------------------ */
int rk_abi_version(void);
const char* rk_last_error(void);
/* One engine per device: owns a stream, scratch arena, RoPE cos/sin tables. */
int rk_engine_create(int device, rk_engine** out);
void rk_engine_destroy(rk_engine* e);
int rk_engine_synchronize(rk_engine* e);
/* Opaque cudaStream_t of the engine (for external event timing). */
void* rk_engine_stream(rk_engine* e);
/* Number of engine kernel launches issued so far (instrumentation). */
uint64_t rk_engine_launch_count(rk_engine* e);
/* rk_agent_prefill schedule: 1 (default) = layer-major fused schedule (all
 * phases of the prompt share one pass per layer; identical results), 0 = the
 * reference's sequential prefill / relay_extend / prefill order. */
int rk_engine_set_fused(rk_engine* e, int enable);
/* Reserved for CUDA-graph replay of repeated identical rk_agent_prefill calls;
 * currently accepted and ignored: on c2 the step's 145 kernels run 4.11 ms
 * back to back inside a 4.21 ms step, so replay could save < 3%. */
int rk_engine_set_graphs(rk_engine* e, int enable);

/* Per-kernel instrumentation: when enabled, each hot-kernel launch is
 * bracketed by CUDA events on the engine stream and tagged with its
 * algorithmic FLOPs / bytes (for roofline reporting). Enabling clears. */
typedef struct rk_kernel_stat {
  char name[32];
  uint64_t launches;
  double total_ms;
  double flops;
  double bytes;
} rk_kernel_stat;
int rk_engine_profile(rk_engine* e, int enable);
int rk_engine_profile_read(rk_engine* e, rk_kernel_stat* out, uint64_t cap, uint64_t* count);

/* ---- weights (model.hpp:42-58) ----------------------------------------- */
/* == init_weights(spec, seed) (model.cpp:81-114) computed on the device,
 * without spec.validate() (model.cpp:82) so 2-layer specs are accepted. */
int rk_weights_init(rk_engine* e, const rk_model_spec* spec, uint64_t seed, int precision,
                    rk_weights** out);
/* Upload host tensors in weights_io.cpp tensor_table order (weights_io.cpp:21-38). */
int rk_weights_upload(rk_engine* e, const rk_model_spec* spec, const float* const* tensors,
                      uint64_t n_tensors, int precision, rk_weights** out);
uint64_t rk_weights_num_tensors(const rk_model_spec* spec);
/* Copy tensor #index (tensor_table order) back to host as fp32. */
int rk_weights_export(rk_weights* w, uint64_t index, float* out, uint64_t count);
void rk_weights_destroy(rk_weights* w);

/* ---- relay cache (relay_cache.hpp:23-46) ------------------------------- */
/* Validates like RelayCache::validate (relay_cache.cpp:18-41), then uploads. */
int rk_cache_upload(rk_engine* e, rk_weights* w, const rk_relay_cache_view* view,
                    rk_cache** out);
/* Decode-time capture on the device (relay_cache.cpp:68-136 via
 * model.cpp:372-389): greedy-decodes n tokens after ctx, recording pre-RoPE
 * K, V, the hidden input of snapshot_layer and influence. first_logits: the
 * prompt-end logits row [V] on the host, or NULL to use the context's last
 * computed row. */
int rk_cache_capture_decode(rk_engine* e, rk_weights* w, rk_context* ctx,
                            const float* first_logits, uint64_t n, uint64_t snapshot_layer,
                            int include_self, rk_cache** out);
/* Capture by chunked prefill of given segment tokens (prefill == decode, test_model.cpp:78-101). */
int rk_cache_capture_prefill(rk_engine* e, rk_weights* w, rk_context* ctx,
                             const int32_t* segment_tokens, uint64_t n, uint64_t snapshot_layer,
                             int include_self, rk_cache** out);
/* Asynchronous upload: validates and returns at once; the layers stream to
 * the device in layer order on the engine's copy stream, and every later call
 * that reads layer l of this cache waits (on the device) for that layer only,
 * so a relay prefill starts while the cache is still arriving. The view's host
 * arrays must stay valid until rk_cache_wait or rk_cache_destroy; pinned host
 * memory makes the copies truly asynchronous. */
int rk_cache_upload_async(rk_engine* e, rk_weights* w, const rk_relay_cache_view* view,
                          rk_cache** out);
/* rk_cache_upload_async with layers [defer_lo, defer_hi] held back: each of
 * them crosses PCIe only when a later call first reads it (a relay with
 * profile (l_start, l_det, l_end) never reads layers l_start..l_det-1). */
int rk_cache_upload_async_defer(rk_engine* e, rk_weights* w, const rk_relay_cache_view* view,
                                uint64_t defer_lo, uint64_t defer_hi, rk_cache** out);
/* Block until an asynchronous upload has landed, deferred layers included
 * (the host arrays may be freed afterwards). */
int rk_cache_wait(rk_cache* c);
/* Block until the copies issued so far have landed; deferred layers stay
 * deferred (the host arrays must stay valid). */
int rk_cache_sync(rk_cache* c);
uint64_t rk_cache_segment_len(const rk_cache* c);
/* Copy a cache back to host (fp32). Any pointer may be NULL. k_pre/v: [L] arrays of [n x kv]. */
int rk_cache_export(rk_cache* c, int32_t* tokens, float* const* k_pre, float* const* v,
                    float* hidden_snapshot, float* influence, uint64_t* source_base,
                    uint64_t* snapshot_layer);
void rk_cache_destroy(rk_cache* c);

/* ---- RKRC relay-cache files (relay_cache.cpp:176-253, serialize.cpp:45-117)
 * "RKRC" | u32 1 | u64 manifest length | JSON manifest | fp32 blob, FNV-1a-64
 * blob checksum. Files are byte-identical to the reference's
 * save_relay_cache; corrupt files fail with RK_ERR_SCHEMA, unreadable paths
 * with RK_ERR_IO, exactly where load_relay_cache throws. */
/* save_relay_cache (relay_cache.cpp:238-245). A bf16 cache saves its bf16
 * values widened to fp32. */
int rk_cache_save(rk_cache* c, const char* path);
/* load_relay_cache (relay_cache.cpp:247-253) straight onto the device.
 * asynchronous != 0: the blob is read into pinned memory owned by the cache
 * and streamed layer by layer as in rk_cache_upload_async. */
int rk_cache_load(rk_engine* e, rk_weights* w, const char* path, int asynchronous, rk_cache** out);
/* Host-only codec (no device work): a host view to a file, a file to a view
 * whose arrays live until rk_cache_file_free. */
typedef struct rk_cache_file rk_cache_file;
int rk_cache_file_write(const rk_relay_cache_view* view, const char* path);
int rk_cache_file_read(const char* path, rk_cache_file** out, rk_relay_cache_view* view);
/* export_relay_cache / import_relay_cache (relay_cache.cpp:176-236) on byte
 * buffers. encode: out == NULL queries *size; capacity < *size fails. */
int rk_cache_file_encode(const rk_relay_cache_view* view, uint8_t* out, uint64_t capacity, uint64_t* size);
int rk_cache_file_decode(const uint8_t* bytes, uint64_t size, rk_cache_file** out, rk_relay_cache_view* view);
void rk_cache_file_free(rk_cache_file* f);

/* ---- offline layer profiler (profiler.cpp:155-175, metrics.cpp:118-238) --
 * Calibrates a LayerProfile: per calibration instance, a decode-time capture
 * of a segment under one prefix (reuse side) against a full prefill of the
 * same segment under another (full side), token_deviation over all layers,
 * layer curves (similarity s, adjacent-layer Spearman rho), averaged, then the
 * start / end / detection scans. In RK_FP32_EXACT every number is
 * bit-identical to the reference. */
/* ProfilerParams (profiler.hpp:19-28). */
typedef struct rk_profiler_params {
  double tau_start;           /* 0.99 */
  uint64_t tail_layers;       /* 5 */
  double stability_lambda;    /* 2.0 */
  uint64_t consecutive;       /* 2 */
  uint64_t min_rise;          /* 3 */
  int32_t first_negative_alpha; /* 0 */
} rk_profiler_params;
/* TwoStageConfig (metrics.hpp:93-107). */
typedef struct rk_two_stage_config {
  uint64_t seed;              /* 1 */
  uint64_t instances;         /* 8 */
  uint64_t stage1_prefix_min, stage1_prefix_max; /* 32, 64 */
  uint64_t stage2_prefix_min, stage2_prefix_max; /* 24, 72 */
  uint64_t segment_len;       /* 48 */
  uint64_t stage2_suffix_len; /* 16 */
  uint64_t sweep_instances;   /* 2 */
  int32_t identical_prefix;   /* 0 */
  uint64_t snapshot_layer;    /* 0 */
} rk_two_stage_config;
/* The scans' result (LayerProfile window + the two fallback warnings). */
typedef struct rk_profile_result {
  uint64_t l_start, l_det, l_end;
  int32_t end_fallback;       /* "end-layer scan found no stable window; using last layer" */
  int32_t det_fallback;       /* "no correlation-trend transition; detection at l_start + 1" */
} rk_profile_result;
/* token_deviation (metrics.cpp:118-159) of two caches of one segment (reuse
 * side, full side) on the device; outputs [n x L] row-major (position, layer),
 * any may be NULL. */
int rk_token_deviation(rk_cache* reuse, rk_cache* full, double* value_cos, double* key_cos,
                       double* value_norm, double* key_norm);
/* Host-only: make_layer_curve (metrics.cpp:191-213) of a value-cosine
 * deviation matrix [n x L]: s[L], rho[L] (rho[0] = NaN), rho_degenerate[L]. */
int rk_layer_curve(const double* value_cos, uint64_t n, uint64_t L, double* s, double* rho,
                   uint8_t* rho_degenerate);
/* Host-only: average_curves (metrics.cpp:215-238) of k curves laid out [k][L]. */
int rk_average_curves(const double* s, const double* rho, const uint8_t* rho_degenerate, uint64_t k,
                      uint64_t L, double* s_out, double* rho_out, uint8_t* rho_degenerate_out);
/* Host-only: profile_from_curve (profiler.cpp:123-155); curve_rho_out [L-1]
 * (curve_rho[i] correlates layers i and i+1) may be NULL. */
int rk_profile_from_curve(const double* s, const double* rho, const uint8_t* rho_degenerate, uint64_t L,
                          const rk_profiler_params* params, rk_profile_result* out, double* curve_rho_out);
/* profile_model (profiler.cpp:157-175) with every instance's captures,
 * prefills and deviations on the device. curve_s [L], curve_rho [L-1] may be NULL. */
int rk_profile_model(rk_engine* e, rk_weights* w, const rk_two_stage_config* calib,
                     const rk_profiler_params* params, rk_profile_result* out, double* curve_s,
                     double* curve_rho);

/* ---- merged KV context (model.hpp:68-87, relay_engine.hpp:37-40) ------- */
int rk_context_create(rk_engine* e, rk_weights* w, rk_context** out);
int rk_context_clone(rk_context* src, rk_context** out);
/* Empty the context (size 0, no segments), keeping its device allocation. */
int rk_context_reset(rk_context* c);
uint64_t rk_context_size(const rk_context* c);
uint64_t rk_context_num_segments(const rk_context* c);
int rk_context_segment(rk_context* c, uint64_t index, uint64_t* base, uint64_t* len,
                       uint8_t* origin /* [L x len] or NULL */);
/* Rows [pos_begin, pos_begin+count) of one layer, fp32. */
int rk_context_export(rk_context* c, uint64_t layer, uint64_t pos_begin, uint64_t count,
                      float* k, float* v);
void rk_context_destroy(rk_context* c);

/* ---- hot path ------------------------------------------------------------ */
/* prefill (model.cpp:305-331): fresh rows at base_position == ctx size.
 * last_logits: logits of the last row [V] (NULL = not computed). */
int rk_prefill(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* tokens, uint64_t n,
               uint64_t base_position, float* last_logits);
/* prefill with capture (model.cpp:305-331 with CaptureFlags/StepTrace,
 * model.hpp:89-111) -- what decode_step / greedy_generate hand to a StepHook
 * (model.cpp:364-389) and what the reference's PrefillResult carries.
 * Every destination is a HOST buffer and may be NULL (= not captured):
 *   logits  [n][V]            every row's logits (output_logits over all rows)
 *   hidden  [L][n][d_model]   each layer's input rows (CaptureFlags::hidden)
 *   k_pre   [L][n][kv]        K before rotation      (CaptureFlags::pre_rope_keys)
 *   v       [L][n][kv]        V as produced          (CaptureFlags::pre_rope_keys)
 *   attn    [L][n][H][base+n] softmax rows over the causal context, zero past
 *                             each row's own position (CaptureFlags::attention)
 * Rows are committed to ctx exactly as rk_prefill does. */
typedef struct rk_trace_request {
  float* logits;
  float* hidden;
  float* k_pre;
  float* v;
  float* attn;
} rk_trace_request;
int rk_prefill_trace(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* tokens, uint64_t n,
                     uint64_t base_position, const rk_trace_request* req);
/* row_logits_from_layer (model.cpp:339-362): one HOST hidden row [d_model]
 * run as a pure query from first_layer to the top at `position` (its own
 * context cell overridden by the fresh K/V, nothing committed), then
 * output_logits; logits [V] (host). workflow.cpp:347-354 uses it when an
 * agent has no suffix. */
int rk_row_logits_from_layer(rk_engine* e, rk_weights* w, rk_context* ctx, const float* hidden_row,
                             uint64_t first_layer, uint64_t position, float* logits);
/* Page-lock caller-owned host memory (cudaHostRegister) so uploads from it
 * (rk_cache_upload_async) stream at full PCIe speed and overlap compute;
 * rk_host_unpin releases it. */
int rk_host_pin(void* ptr, uint64_t bytes);
int rk_host_unpin(void* ptr);
/* relay_extend (relay_engine.cpp:183-361): appends one relayed segment at ctx size. */
int rk_relay_extend(rk_engine* e, rk_weights* w, rk_context* ctx, rk_cache* cache,
                    const rk_layer_profile* profile, const rk_relay_options* opts,
                    rk_relay_output* out);
/* relay_prefill (relay_engine.cpp:363-395): fresh prefix prefill into an empty
 * ctx, relay_extend, then the segment-end logits (row_logits_from_layer,
 * model.cpp:339-362). */
int rk_relay_prefill(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* prefix,
                     uint64_t n_prefix, rk_cache* cache, const rk_layer_profile* profile,
                     const rk_relay_options* opts, rk_relay_output* out,
                     float* segment_end_logits);
/* The downstream agent's TTFT sequence of run_workflow's relay branch
 * (workflow.cpp:316-369): prefix prefill, relay_extend per upstream cache in
 * order, then the suffix prefill's last-row logits (or, with no suffix, the
 * last segment row as a pure query), then argmax (model.cpp:364-370).
 * mode RK_MODE_FULL prefills prefix ++ segments ++ suffix from scratch
 * (workflow.cpp:301-315). outs: [n_upstream] or NULL. */
int rk_agent_prefill(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* prefix,
                     uint64_t n_prefix, rk_cache* const* upstream, uint64_t n_upstream,
                     const int32_t* suffix, uint64_t n_suffix, const rk_layer_profile* profile,
                     const rk_relay_options* opts, rk_relay_output* outs, float* end_logits,
                     int32_t* first_token);

/* ---- analytic FLOP model (relay_engine.cpp:72-128) ---------------------- */
double rk_flops_span_full(const rk_model_spec* s, uint64_t base, uint64_t n);
double rk_flops_segment_schedule(const rk_model_spec* s, uint64_t base, uint64_t n,
                                 uint64_t band_lo, uint64_t band_hi, uint64_t sparse_hi,
                                 uint64_t selected);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* RELAYKV_B200_H_ */
