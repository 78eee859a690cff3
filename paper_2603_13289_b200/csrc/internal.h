// internal.h -- engine objects and kernel launchers (not part of the ABI).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <future>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hostconv.h"
#include "relaykv_b200.h"

namespace rk {

// Internal error carrying the rk_status of the reference exception type.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
void set_last_error(const std::string& msg);
#define RK_CUDA(x) ::rk::cuda_check((x), #x, __FILE__, __LINE__)

// Free device blocks kept for reuse (exact-size match), so per-call objects
// (relay caches uploaded every agent hop) do not pay cudaMalloc/cudaFree --
// cudaFree synchronizes the whole device.
using BlockPool = std::multimap<size_t, void*>;

// Owning device allocation (optionally drawn from / returned to a BlockPool).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  BlockPool* pool = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), pool(o.pool) { o.p = nullptr; o.bytes = 0; o.pool = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; bytes = o.bytes; pool = o.pool;
      o.p = nullptr; o.bytes = 0; o.pool = nullptr;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t n);
  // take an exact-size block from `pl` if one is free (callers must have
  // synchronized the stream that last used blocks returned to it)
  void alloc_pooled(BlockPool* pl, size_t n);
  void release();
  // grow (contents discarded) to at least n bytes
  void ensure(size_t n) { if (n > bytes) { release(); alloc(n); } }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// Double-precision RoPE table built on the host with glibc exactly as
// rope_rotate does (tensor.cpp:134-142): cs[pos][i] = {cos, sin}(pos * pow(theta, -2i/dh)).
struct RopeTable {
  float theta = 0;
  uint64_t d_head = 0, positions = 0;
  DevBuf cs;   // double2 [positions][d_head/2]
  DevBuf csf;  // float2, same angles (bf16 path)
};

struct Scratch;
struct ExtendSlot;
struct Profiler;

}  // namespace rk

struct rk_engine {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  // side stream for off-critical-path reporting kernels (joined at the next call)
  cudaStream_t side = nullptr;
  cudaEvent_t side_fork = nullptr, side_join = nullptr;
  // copy streams of asynchronous relay-cache uploads (round-robin per cache, so
  // the layers of several upstream caches arrive interleaved)
  static constexpr int kXfer = 4;
  cudaStream_t xfer[kXfer] = {};
  int next_xfer = 0;
  std::unique_ptr<rk::HostPool> host_pool;
  std::unique_ptr<rk::Uploader> uploader;
  rk::PinnedPool pinned_pool;
  uint64_t launches = 0;
  int use_graphs = 0;
  // fraction of a relayed segment's rows the last RELAY/BLEND selection kept
  // (-1: none yet). The live row count of a sparse pass exists only on the
  // device; the host plans its GEMM tiles / attention split from this
  // (Rows::hint) instead of a fixed guess.
  double sel_frac = -1.0;
  int fused = 1;  // layer-major fused agent schedule (runner.cpp agent_fused)
  std::vector<std::unique_ptr<rk::RopeTable>> rope;
  std::unique_ptr<rk::Scratch> scratch;
  // pinned host staging
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // pinned landing area of a call's small results (selection counts, threshold,
  // first token), copied in stream order before the call's final synchronize
  void* results_host = nullptr;
  static constexpr size_t kResultsBytes = 4096;
  rk::DevBuf status;  // int flags: [0] non-finite
  std::vector<cudaEvent_t> events;
  std::vector<std::unique_ptr<rk::ExtendSlot>> slots;
  rk::BlockPool cache_pool;  // device blocks of destroyed relay caches
  std::unique_ptr<rk::Profiler> prof;
  rk_engine();
  ~rk_engine();
};

// Per-layer weights on the device.
//  FP32_EXACT: reference layout [K x N] row-major fp32, Q|K|V concatenated
//    along N, gate/up interleaved along N (col 2j = gate j, 2j+1 = up j).
//  BF16: the same logical matrices stored transposed, [N x K] K-major bf16,
//    the tcgen05 B-operand layout.
struct rk_layer_dev {
  float* attn_norm = nullptr;  // [d]
  float* mlp_norm = nullptr;   // [d]
  void* w_qkv = nullptr;       // [d x (q+2kv)]
  void* w_o = nullptr;         // [q x d]
  void* w_gu = nullptr;        // [d x 2ff] interleaved
  void* w_down = nullptr;      // [ff x d]
  // RK_FP32_TC: 3xTF32 packings [N x 3K] = [hi | lo | hi] of the transposed weights
  float* tc_qkv = nullptr;
  float* tc_o = nullptr;
  float* tc_gu = nullptr;
  float* tc_down = nullptr;
};

struct rk_weights {
  rk_engine* e = nullptr;
  rk_model_spec s{};
  int precision = RK_FP32_EXACT;
  size_t elem = 4;             // bytes per stored weight element
  rk::DevBuf blob;             // all tensors
  rk::DevBuf tc_blob;          // RK_FP32_TC packed weights (layer_tc.cu)
  void* emb = nullptr;         // [V x d] (fp32 exact; bf16 in BF16)
  float* final_norm = nullptr; // [d]
  void* head = nullptr;        // exact: [d x V]; bf16: [V x d]
  std::vector<rk_layer_dev> layers;
  rk::RopeTable* rope = nullptr;
  size_t q() const { return s.num_heads * s.d_head; }
  size_t kv() const { return s.num_kv_heads * s.d_head; }
};

struct rk_cache {
  rk_engine* e = nullptr;
  int precision = RK_FP32_EXACT;
  size_t elem = 4;
  uint64_t L = 0, Hkv = 0, dh = 0, d = 0, n = 0, maxpos = 0;
  float theta = 0;
  uint64_t src_base = 0, snapshot = 0, steps = 0;
  rk::DevBuf tokens;     // int32 [n]
  rk::DevBuf k_pre, v;   // elem [L][n][kv]
  rk::DevBuf hidden;     // fp32 [n x d]
  rk::DevBuf influence;  // fp32 [n]
  rk::DevBuf infl_mean;  // double [1], sequential mean (selector.cpp:37-39)
  std::vector<int32_t> host_tokens;
  // asynchronous upload (rk_cache_upload_async): per-layer readiness on the
  // engine's copy stream; ev_meta covers tokens / hidden / influence
  bool async = false;
  cudaStream_t xfer = nullptr;
  cudaEvent_t ev_meta = nullptr;
  std::vector<cudaEvent_t> ev_layer;
  // deferred layers (rk_cache_upload_async_defer): uploaded from the host view
  // the first time a call reads them
  std::vector<uint8_t> deferred;
  std::vector<const float*> host_k, host_v;
  rk::DevBuf staging;  // fp32 layer staging of the bf16 conversion
  // host-converted upload (bf16 weights, async): the engine's uploader thread
  // converts layer l into a ring of pinned bf16 slots and sets flags[l]; the
  // copy stream waits on the flag (cuStreamWaitValue32) before copying it
  void* stage_host = nullptr;
  size_t stage_host_bytes = 0;
  volatile uint32_t* flags = nullptr;  // in stage_host, [L]
  std::shared_future<void> conv_done;
  std::shared_ptr<void> host_keep;  // host source of an async upload owned by the cache (rk_cache_load)
  size_t kv() const { return Hkv * dh; }
  ~rk_cache();
};

struct rk_segment_marks {
  uint64_t base = 0, len = 0;
  rk::DevBuf origin;  // uint8 [L x len]
};

struct rk_context {
  rk_engine* e = nullptr;
  rk_weights* w = nullptr;
  uint64_t size = 0, cap = 0;
  size_t elem = 4;
  rk::DevBuf k, v;  // elem [L][cap][kv]
  std::vector<rk_segment_marks> segs;
  void* k_layer(size_t l) const { return static_cast<char*>(k.p) + l * cap * w->kv() * elem; }
  void* v_layer(size_t l) const { return static_cast<char*>(v.p) + l * cap * w->kv() * elem; }
  void reserve(uint64_t positions);
  // zero_fill=false: the caller writes every new cell of every layer before
  // anything reads it (the fused agent schedule), so the fill is skipped
  void resize(uint64_t positions, bool zero_fill = true);
};

namespace rk {

// Grow-only scratch buffers reused across calls.
struct Scratch {
  DevBuf hidden, sub_hidden, normed, qkv, attn, act, logits, tokens, positions, sub_positions;
  DevBuf s_dev, s_key, sel_idx, sel_tags, sel_info, depth, argmax, seg_hidden_out;
  DevBuf gemm_tmp, attn_ws, attn_cnt, gemm_ws;
  DevBuf tc_split, tc_gu;  // RK_FP32_TC: [hi|hi|lo] GEMM operand, gate/up output
  DevBuf norm_inv, norm_part, norm_cnt;  // fused RMSNorm (layer_bf16.cu)
};

RopeTable* rope_table(rk_engine* e, float theta, uint64_t d_head, uint64_t positions);

// Row set of a layer pass: rows_max bounds the launch; rows_dev (optional)
// holds the true count on the device (sparse passes after selection).
struct Rows {
  int rows_max = 0;
  const int* rows_dev = nullptr;
  const int* pos = nullptr;  // int32 [rows_max] absolute positions
  // Row groups of the fused schedule ([prefix | suffix | segment rows]):
  // rows [0, g1), [g1, g2), [g2, live). Attention tiles never straddle a
  // group boundary, so a tile's key range follows its own rows' positions.
  int g1 = 0, g2 = 0;
  int hint = 0;  // expected live rows when rows_dev is set (0: unknown -> rows_max / 3)
};

void ensure_cache_layer(rk_cache* c, uint64_t l);  // engine.cpp: upload a deferred layer now
void ensure_cache_all(rk_cache* c);
bool pdl_enabled();  // programmatic dependent launch (RK_PDL, default on), gemm_sm100.cu

// ---- kernel launchers (kernels_*.cu) -------------------------------------
namespace k {
// weights
void init_uniform(cudaStream_t s, float* dst, size_t n, uint64_t state0, float scale);
void fill(cudaStream_t s, float* dst, size_t n, float v);
// dst[r * ldd + c0 + c] = src[r * lds + c] for c < cols  (fp32)
void copy_cols_f32(cudaStream_t s, float* dst, size_t ldd, size_t c0, const float* src, size_t lds,
                   size_t rows, size_t cols, size_t dst_col_stride);
// dst[(c0 + c*cstride) * ldd + r] = bf16(src[r * lds + c])  (transpose to K-major bf16)
void transpose_to_bf16(cudaStream_t s, __nv_bfloat16* dst, size_t ldd, size_t c0, size_t cstride,
                       const float* src, size_t rows, size_t cols, const float* row_gain = nullptr);
void f32_to_bf16(cudaStream_t s, __nv_bfloat16* dst, const float* src, size_t n);
void bf16_to_f32(cudaStream_t s, float* dst, const __nv_bfloat16* src, size_t n);

// model building blocks (elem = 4 fp32 exact, 2 bf16)
void embed(cudaStream_t s, float* hidden, const void* emb, size_t elem, const int32_t* tokens,
           int n, int d, int vocab, int* status);
void gather_rows(cudaStream_t s, float* dst, const float* src, const int* idx, const int* count,
                 int rows_max, int d);
void scatter_rows(cudaStream_t s, float* dst, const float* src, const int* idx, const int* count,
                  int rows_max, int d, uint64_t* depth, uint64_t depth_value);
void positions_from_sel(cudaStream_t s, int* pos, const int* sel, const int* count, int rows_max, int base);
void iota_positions(cudaStream_t s, int* pos, int n, int base);
void mark_rows(cudaStream_t s, uint8_t* origin, int len, int layer_lo, int layer_hi, const int* sel,
               const int* count, int rows_max);
void mark_layers(cudaStream_t s, uint8_t* origin, int len, int layer_lo, int layer_hi);
// device memset / memcpy / 2-D row zero as kernels (see kernels_common.cu)
void zero_dev(cudaStream_t s, void* dst, size_t bytes);
void zero_many(cudaStream_t s, const std::vector<std::pair<void*, size_t>>& bufs);  // one launch
void copy_dev(cudaStream_t s, void* dst, const void* src, size_t bytes);
// up to 16 small copies (e.g. into mapped pinned host memory) in one launch:
// no copy engine, so they never queue behind bulk uploads
struct SmallCopies {
  const void* src[16];
  void* dst[16];
  int bytes[16];
  int n = 0;
};
void small_copies(cudaStream_t s, const SmallCopies& c);
// decode capture (graph-replayed steps; see Runner::capture_decode)
void decode_step_begin(cudaStream_t s, const int* step, int src, const int* tokens, int* cur_tok, int* pos);
void decode_step_end(cudaStream_t s, int* step, int n, int L, size_t row_bytes, const void* stage_k,
                     const void* stage_v, void* k_pre, void* v, size_t hid_bytes, const void* stage_h, void* hidden,
                     const int* next_tok, int* tokens);
void zero_rows(cudaStream_t s, void* dst, size_t pitch, size_t width, size_t rows);
void copy_i32(cudaStream_t s, int* dst, const int* src, int n);  // src may be mapped host memory
void fill_doubles(cudaStream_t s, double* dst, int n, double v);
void set_depth(cudaStream_t s, uint64_t* depth, int n, uint64_t v);
// ws: >= 148 float2 of scratch
void argmax(cudaStream_t s, const float* x, int n, int* out, void* ws);

// relay (both precisions)
void realign_graft(cudaStream_t s, const void* k_pre, const void* v_src, size_t elem, int L,
                   int n, int kv, int dh, const double2* rope, int base, void* ctx_k, void* ctx_v,
                   size_t ctx_layer_stride, int skip_lo, int skip_hi);
// several segments (caches k_pre/v [L][n][kv] grafted at ctx rows base..) in one launch
struct RealignJob {
  const void* k_pre;
  const void* v;
  int n, base;
};
constexpr int kMaxRealignJobs = 8;
struct RealignJobs {
  const void* k_pre[kMaxRealignJobs];
  const void* v[kMaxRealignJobs];
  int n[kMaxRealignJobs], base[kMaxRealignJobs], blk0[kMaxRealignJobs + 1];
  int count;
};
void realign_graft_batch(cudaStream_t s, const RealignJob* jobs, int count, size_t elem, int L, int kv, int dh,
                         const double2* rope, void* ctx_k, void* ctx_v, size_t ctx_layer_stride, int skip_lo,
                         int skip_hi);
void score_deviation(cudaStream_t s, const void* ctx_v, const void* cache_v, const void* ctx_k,
                     const void* cache_kpre, size_t elem, int n, int kv, int heads, int dh,
                     const double2* rope, int base, double* s_dev, double* s_key);
// Selection (certified parallel threshold) on s; the exact reported threshold
// and margin (dinfo) on `side` (forked from s via `fork`, recorded on `join`).
void select_relay(cudaStream_t s, const double* s_dev, const float* influence,
                  const double* infl_mean, int n, double tau_dev, double tau_inf, int suffix_k,
                  int* sel_idx, uint32_t* sel_tags, int* info, double* dinfo, cudaStream_t side = nullptr,
                  cudaEvent_t fork = nullptr, cudaEvent_t join = nullptr);
// offline profiler: token_deviation (metrics.cpp:118-159); out [4][n][L]
void token_deviation(cudaStream_t s, const void* reuse_k, const void* reuse_v, const void* full_k,
                     const void* full_v, size_t elem, int L, int n, int kv, int heads, double* out);
void blend_scores(cudaStream_t s, const void* ctx_v, const void* cache_v, size_t elem, int n,
                  int kv, double* score);
void select_topk(cudaStream_t s, const double* score, int n, int count, int* sel_idx,
                 uint32_t* sel_tags, int* info);
void seq_mean(cudaStream_t s, const float* x, int n, double* out);

// fused agent schedule
constexpr int kMaxFusedSegments = 32;  // upstream segments of one layer-major fused agent prefill
struct SegCounts {
  const int* count[kMaxFusedSegments];
};
void segment_offsets(cudaStream_t s, const SegCounts& c, int U, int start, int* offs);
void gather_rows_to(cudaStream_t s, float* H, const int* off, const float* src, const int* idx, const int* count,
                    int rows_max, int d, int* pos, int base);
void scatter_rows_from(cudaStream_t s, float* dst, const float* H, const int* off, const int* idx, const int* count,
                       int rows_max, int d, uint64_t* depth, uint64_t value);

// fp32 exact path
void rmsnorm_exact(cudaStream_t s, const float* x, const float* gain, float eps, float* out,
                   Rows rows, int d);
enum EpiMode { EPI_STORE = 0, EPI_ADD = 1, EPI_SILU_PAIR = 2 };
void gemm_exact(cudaStream_t s, const float* A, const float* B, float* C, Rows rows, int N, int K,
                int epi, int* status);
void rope_commit_exact(cudaStream_t s, float* qkv, Rows rows, int H, int Hkv, int dh,
                       const double2* rope, float* ctx_k, float* ctx_v, int commit);
void attn_exact(cudaStream_t s, const float* qkv, Rows rows, int H, int Hkv, int dh,
                const float* ctx_k, const float* ctx_v, float* out, int self_override, int max_ctx,
                float* probs, int key_lo, int key_n);
// influence accumulation of RelayRecorder::feed (relay_cache.cpp:108-123)
void influence_accum(cudaStream_t s, double* acc, const float* probs, Rows rows, int H, int key_lo,
                     int key_n, int include_self);
void copy2d_f32(cudaStream_t s, float* dst, size_t dld, size_t dcs, const float* src, size_t sld,
                size_t scs, size_t rows, size_t cols);
void untranspose_bf16(cudaStream_t s, float* dst, const __nv_bfloat16* src, size_t ld, size_t c0,
                      size_t cstride, size_t rows, size_t cols, const float* row_gain = nullptr);
void doubles_to_floats(cudaStream_t s, float* dst, const double* src, int n);

// bf16 tensor-core path
void rmsnorm_bf16(cudaStream_t s, const float* x, const float* gain, float eps,
                  __nv_bfloat16* out, Rows rows, int d);
}  // namespace k

}  // namespace rk
