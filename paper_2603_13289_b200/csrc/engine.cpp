// engine.cpp -- C ABI implementation and the relay-prefill orchestration.
//
// Host-side control flow mirrors the reference function by function
// (relay_engine.cpp:183-395, model.cpp:305-362, workflow.cpp:316-369); the
// arithmetic runs in the CUDA kernels of kernels_*.cu / gemm_sm100.cu /
// attn_sm100.cu. Compiled with -ffp-contract=off: the few float expressions
// evaluated here (init scales, thresholds) must round as the reference's.
#include <cuda.h>

#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <atomic>
#include <future>
#include <mutex>
#include <thread>

#include "internal.h"
#include "layer_tc.h"
#include "layer.h"
#include "prof.h"
#include "profiler.h"
#include "rkrc.h"

using namespace rk;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return RK_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return RK_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RK_ERR_RUNTIME;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev, bool nothrow = false) {
    cudaGetDevice(&prev);
    if (prev != dev) {
      const cudaError_t err = cudaSetDevice(dev);
      if (!nothrow) RK_CUDA(err);
    }
  }
  ~DeviceGuard() {
    int cur;
    if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void require(bool ok, int code, const std::string& msg) {
  if (!ok) raise(code, msg);
}

size_t num_tensors(const rk_model_spec& s) { return 1 + 9 * s.num_layers + 2; }

}  // namespace

namespace rk {

void set_last_error(const std::string& msg) { g_err = msg; }

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
             cudaGetErrorString(e), file, line, what);
    throw Error(RK_ERR_RUNTIME, buf);
  }
}

void DevBuf::alloc(size_t n) {
  bytes = n;
  p = nullptr;
  if (n == 0) return;
  cudaError_t e = cudaMalloc(&p, n);
  if (e != cudaSuccess) {
    p = nullptr;
    bytes = 0;
    cudaGetLastError();
    throw Error(RK_ERR_RUNTIME, "device allocation of " + std::to_string(n) + " bytes failed: " +
                                    cudaGetErrorString(e));
  }
}
void DevBuf::alloc_pooled(BlockPool* pl, size_t n) {
  release();
  pool = pl;
  auto it = pl->find(n);
  if (it != pl->end()) {
    p = it->second;
    bytes = n;
    pl->erase(it);
    return;
  }
  alloc(n);
  pool = pl;
}

void DevBuf::release() {
  if (p) {
    if (pool) pool->emplace(bytes, p);
    else cudaFree(p);
  }
  p = nullptr;
  bytes = 0;
  pool = nullptr;
}

RopeTable* rope_table(rk_engine* e, float theta, uint64_t d_head, uint64_t positions) {
  for (auto& t : e->rope)
    if (t->theta == theta && t->d_head == d_head && t->positions >= positions) return t.get();
  auto t = std::make_unique<RopeTable>();
  t->theta = theta;
  t->d_head = d_head;
  t->positions = positions;
  const uint64_t half = d_head / 2;
  std::vector<double2> h(positions * half);
  const double d = static_cast<double>(d_head);
  for (uint64_t i = 0; i < half; ++i) {
    // exactly rope_rotate's expressions (tensor.cpp:135-137), glibc pow/cos/sin
    const double freq = std::pow(static_cast<double>(theta), -2.0 * static_cast<double>(i) / d);
    for (uint64_t p = 0; p < positions; ++p) {
      const double angle = static_cast<double>(static_cast<int64_t>(p)) * freq;
      h[p * half + i] = make_double2(std::cos(angle), std::sin(angle));
    }
  }
  t->cs.alloc(h.size() * sizeof(double2));
  // (stream-ordered: a pageable cudaMemcpy may return before its DMA lands,
  // and the kernels reading the table run on the non-blocking engine stream)
  RK_CUDA(cudaMemcpyAsync(t->cs.p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, e->stream));
  std::vector<float2> hf(h.size());
  for (size_t i = 0; i < h.size(); ++i) hf[i] = make_float2((float)h[i].x, (float)h[i].y);
  t->csf.alloc(hf.size() * sizeof(float2));
  RK_CUDA(cudaMemcpyAsync(t->csf.p, hf.data(), hf.size() * sizeof(float2), cudaMemcpyHostToDevice, e->stream));
  e->rope.push_back(std::move(t));
  return e->rope.back().get();
}

}  // namespace rk

rk_engine::rk_engine() : scratch(new Scratch()) {}
rk_engine::~rk_engine() {
  for (auto& kv : cache_pool) cudaFree(kv.second);
  cache_pool.clear();
  scratch.reset();
  rope.clear();
  if (pinned) cudaFreeHost(pinned);
  if (results_host) cudaFreeHost(results_host);
  if (side) {
    cudaStreamSynchronize(side);
    cudaStreamDestroy(side);
  }
  for (auto& x : xfer)
    if (x) {
      cudaStreamSynchronize(x);
      cudaStreamDestroy(x);
    }
  uploader.reset();  // drains queued conversion jobs
  if (side_fork) cudaEventDestroy(side_fork);
  if (side_join) cudaEventDestroy(side_join);
  if (stream) cudaStreamDestroy(stream);
}

void rk_context::reserve(uint64_t positions) {
  if (positions <= cap) return;
  uint64_t ncap = cap ? cap : 256;
  while (ncap < positions) ncap *= 2;
  if (ncap > w->s.max_positions) ncap = std::max<uint64_t>(w->s.max_positions, positions);
  const size_t L = w->s.num_layers, row = w->kv() * elem;
  DevBuf nk(L * ncap * row), nv(L * ncap * row);
  // zero-fill: masked keys beyond the live size must be finite (0 * NaN = NaN in P.V)
  RK_CUDA(cudaMemsetAsync(nk.p, 0, nk.bytes, e->stream));
  RK_CUDA(cudaMemsetAsync(nv.p, 0, nv.bytes, e->stream));
  if (size > 0) {
    RK_CUDA(cudaMemcpy2DAsync(nk.p, ncap * row, k.p, cap * row, size * row, L, cudaMemcpyDeviceToDevice, e->stream));
    RK_CUDA(cudaMemcpy2DAsync(nv.p, ncap * row, v.p, cap * row, size * row, L, cudaMemcpyDeviceToDevice, e->stream));
    RK_CUDA(cudaStreamSynchronize(e->stream));
  }
  k = std::move(nk);
  v = std::move(nv);
  cap = ncap;
}

void rk_context::resize(uint64_t positions, bool zero_fill) {  // KVContext::resize (model.cpp:124-131)
  if (positions < size) raise(RK_ERR_INVALID_ARGUMENT, "KVContext::resize: cannot shrink");
  if (positions == size) return;
  reserve(positions);
  const size_t L = w->s.num_layers, row = w->kv() * elem;
  if (!zero_fill) {
    size = positions;
    return;
  }
  rk::k::zero_rows(e->stream, static_cast<char*>(k.p) + size * row, cap * row, (positions - size) * row, L);
  rk::k::zero_rows(e->stream, static_cast<char*>(v.p) + size * row, cap * row, (positions - size) * row, L);
  size = positions;
}

// ============================================================================
// weights
// ============================================================================
namespace {

struct TensorDesc {
  size_t rows, cols;  // reference shape [rows x cols]
};

// Allocate the device layout for a spec/precision; returns total bytes.
void layout_weights(rk_weights* w) {
  const rk_model_spec& s = w->s;
  const size_t d = s.d_model, q = w->q(), kv = w->kv(), ff = s.d_ff, V = s.vocab_size, L = s.num_layers;
  const size_t el = w->elem;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  size_t total = al(V * d * el) + al(d * 4) + al(d * V * el);
  const size_t per_layer = al(d * 4) * 2 + al(d * (q + 2 * kv) * el) + al(q * d * el) + al(d * 2 * ff * el) + al(ff * d * el);
  total += L * per_layer;
  w->blob.alloc(total);
  char* p = static_cast<char*>(w->blob.p);
  auto take = [&](size_t b) { void* r = p; p += al(b); return r; };
  w->emb = take(V * d * el);
  w->final_norm = static_cast<float*>(take(d * 4));
  w->head = take(d * V * el);
  w->layers.resize(L);
  for (auto& ly : w->layers) {
    ly.attn_norm = static_cast<float*>(take(d * 4));
    ly.mlp_norm = static_cast<float*>(take(d * 4));
    ly.w_qkv = take(d * (q + 2 * kv) * el);
    ly.w_o = take(q * d * el);
    ly.w_gu = take(d * 2 * ff * el);
    ly.w_down = take(ff * d * el);
  }
}

// Reference shape of tensor_table entry idx (weights_io.cpp:21-38).
TensorDesc tensor_desc(const rk_model_spec& s, size_t idx) {
  const size_t d = s.d_model, q = s.num_heads * s.d_head, kv = s.num_kv_heads * s.d_head;
  if (idx == 0) return {s.vocab_size, d};
  idx -= 1;
  if (idx < 9 * s.num_layers) {
    switch (idx % 9) {
      case 0: case 5: return {1, d};
      case 1: return {d, q};
      case 2: case 3: return {d, kv};
      case 4: return {q, d};
      case 6: case 7: return {d, s.d_ff};
      default: return {s.d_ff, d};
    }
  }
  idx -= 9 * s.num_layers;
  if (idx == 0) return {1, d};
  return {d, s.vocab_size};
}

// Place one reference-layout fp32 tensor (device, [rows x cols]) into the
// engine layout.
void pack_tensor(rk_weights* w, size_t idx, const float* src) {
  const rk_model_spec& s = w->s;
  cudaStream_t st = w->e->stream;
  const size_t d = s.d_model, q = w->q(), kv = w->kv(), ff = s.d_ff, V = s.vocab_size;
  const bool bf = w->precision == RK_BF16;
  const TensorDesc td = tensor_desc(s, idx);
  auto copy_plain = [&](void* dst, size_t n) {
    if (bf) k::f32_to_bf16(st, static_cast<__nv_bfloat16*>(dst), src, n);
    else RK_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToDevice, st));
  };
  // exact: dst[r][c0 + c*cs] (row length ldd); bf16: transposed dst[c0 + c*cs][r] (row length ld_t)
  // bf16: the RMSNorm gain feeding W_q/W_k/W_v (attn_norm) or W_gate/W_up
  // (mlp_norm) is folded into the weight rows; the GEMM epilogue applies 1/rms
  auto place = [&](void* dst, size_t ldd, size_t c0, size_t cs, size_t ld_t, const float* gain = nullptr) {
    if (bf) k::transpose_to_bf16(st, static_cast<__nv_bfloat16*>(dst), ld_t, c0, cs, src, td.rows, td.cols, gain);
    else k::copy_cols_f32(st, static_cast<float*>(dst), ldd, c0, src, td.cols, td.rows, td.cols, cs);
  };
  if (idx == 0) { copy_plain(w->emb, V * d); return; }
  size_t i = idx - 1;
  if (i < 9 * s.num_layers) {
    rk_layer_dev& ly = w->layers[i / 9];
    switch (i % 9) {
      case 0: RK_CUDA(cudaMemcpyAsync(ly.attn_norm, src, d * 4, cudaMemcpyDeviceToDevice, st)); break;
      case 1: place(ly.w_qkv, q + 2 * kv, 0, 1, d, ly.attn_norm); break;
      case 2: place(ly.w_qkv, q + 2 * kv, q, 1, d, ly.attn_norm); break;
      case 3: place(ly.w_qkv, q + 2 * kv, q + kv, 1, d, ly.attn_norm); break;
      case 4: place(ly.w_o, d, 0, 1, q); break;
      case 5: RK_CUDA(cudaMemcpyAsync(ly.mlp_norm, src, d * 4, cudaMemcpyDeviceToDevice, st)); break;
      case 6: place(ly.w_gu, 2 * ff, 0, 2, d, ly.mlp_norm); break;
      case 7: place(ly.w_gu, 2 * ff, 1, 2, d, ly.mlp_norm); break;
      default: place(ly.w_down, d, 0, 1, ff); break;
    }
    return;
  }
  i -= 9 * s.num_layers;
  if (i == 0) { RK_CUDA(cudaMemcpyAsync(w->final_norm, src, d * 4, cudaMemcpyDeviceToDevice, st)); return; }
  if (bf) k::transpose_to_bf16(st, static_cast<__nv_bfloat16*>(w->head), d, 0, 1, src, d, V);
  else RK_CUDA(cudaMemcpyAsync(w->head, src, d * V * 4, cudaMemcpyDeviceToDevice, st));
}

// RK_FP32_TC: the 3xTF32 packings [N x 3K] of the four layer matmuls, built
// from the fp32 reference-layout tensors (layer_tc.cu).
void build_tc_weights(rk_weights* w) {
  const rk_model_spec& s = w->s;
  const size_t d = s.d_model, q = w->q(), kv = w->kv(), ff = s.d_ff;
  const size_t per = 3 * (d * (q + 2 * kv) + q * d + d * 2 * ff + ff * d);
  w->tc_blob.alloc(per * s.num_layers * 4);
  float* p = w->tc_blob.as<float>();
  cudaStream_t st = w->e->stream;
  for (auto& ly : w->layers) {
    ly.tc_qkv = p, p += 3 * d * (q + 2 * kv);
    ly.tc_o = p, p += 3 * q * d;
    ly.tc_gu = p, p += 3 * d * 2 * ff;
    ly.tc_down = p, p += 3 * ff * d;
    tc::pack_weight(st, ly.tc_qkv, static_cast<const float*>(ly.w_qkv), (int)(q + 2 * kv), 0, 1, (int)d,
                    (int)(q + 2 * kv));
    tc::pack_weight(st, ly.tc_o, static_cast<const float*>(ly.w_o), (int)d, 0, 1, (int)q, (int)d);
    tc::pack_weight(st, ly.tc_gu, static_cast<const float*>(ly.w_gu), (int)(2 * ff), 0, 1, (int)d, (int)(2 * ff));
    tc::pack_weight(st, ly.tc_down, static_cast<const float*>(ly.w_down), (int)d, 0, 1, (int)ff, (int)d);
  }
}

void check_spec(const rk_model_spec& s) {
  require(s.num_layers >= 1 && s.d_model > 0 && s.num_heads > 0 && s.num_kv_heads > 0 &&
              s.d_head > 0 && s.d_ff > 0 && s.vocab_size > 0 && s.max_positions > 0,
          RK_ERR_SCHEMA, "invalid model spec: all extents must be >= 1");
  require(s.num_heads % s.num_kv_heads == 0, RK_ERR_SCHEMA,
          "invalid model spec: num_heads must be divisible by num_kv_heads");
  require(s.d_head % 2 == 0, RK_ERR_SCHEMA, "invalid model spec: d_head must be even for rotary embedding");
  require((s.num_kv_heads * s.d_head) % 8 == 0, RK_ERR_INVALID_ARGUMENT,
          "engine requires kv_dim to be a multiple of 8 (16-byte rows)");
}

rk_weights* new_weights(rk_engine* e, const rk_model_spec* spec, int precision) {
  require(spec != nullptr, RK_ERR_INVALID_ARGUMENT, "null spec");
  check_spec(*spec);
  require(precision == RK_FP32_EXACT || precision == RK_BF16 || precision == RK_FP32_TC, RK_ERR_INVALID_ARGUMENT,
          "bad precision");
  auto w = std::make_unique<rk_weights>();
  w->e = e;
  w->s = *spec;
  w->precision = precision;
  w->elem = precision == RK_BF16 ? 2 : 4;
  if (precision == RK_FP32_TC) {
    require(spec->d_model % 64 == 0 && (spec->num_heads * spec->d_head) % 64 == 0 && spec->d_ff % 64 == 0 &&
                (spec->num_heads * spec->d_head + 2 * spec->num_kv_heads * spec->d_head) % 64 == 0,
            RK_ERR_INVALID_ARGUMENT, "fp32-tc mode requires d_model, q_dim, qkv width and d_ff to be multiples of 64");
    require(spec->d_head == 64 || spec->d_head == 128, RK_ERR_INVALID_ARGUMENT,
            "fp32-tc mode supports d_head 64 or 128");
  }
  if (precision == RK_BF16) {
    require(spec->d_model % 64 == 0 && (spec->num_heads * spec->d_head) % 64 == 0 && spec->d_ff % 64 == 0 &&
                spec->vocab_size % 64 == 0,
            RK_ERR_INVALID_ARGUMENT, "bf16 mode requires d_model, q_dim, d_ff and vocab to be multiples of 64");
    require(spec->d_head == 64 || spec->d_head == 128, RK_ERR_INVALID_ARGUMENT,
            "bf16 mode supports d_head 64 or 128");
  }
  layout_weights(w.get());
  w->rope = rope_table(e, spec->theta_base, spec->d_head, spec->max_positions);
  return w.release();
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
namespace rk {
// Upload a deferred layer (rk_cache_upload_async_defer) on the cache's copy
// stream the first time something reads it.
void ensure_cache_layer(rk_cache* c, uint64_t l) {
  if (c->deferred.empty() || !c->deferred[l]) return;
  const size_t n = c->n, kv = c->kv();
  for (int which = 0; which < 2; ++which) {
    const float* src = which == 0 ? c->host_k[l] : c->host_v[l];
    char* dst = static_cast<char*>(which == 0 ? c->k_pre.p : c->v.p) + l * n * kv * c->elem;
    if (c->elem == 4) {
      RK_CUDA(cudaMemcpyAsync(dst, src, n * kv * 4, cudaMemcpyHostToDevice, c->xfer));
    } else {
      float* stage = c->staging.as<float>() + (size_t)which * n * kv;
      RK_CUDA(cudaMemcpyAsync(stage, src, n * kv * 4, cudaMemcpyHostToDevice, c->xfer));
      k::f32_to_bf16(c->xfer, reinterpret_cast<__nv_bfloat16*>(dst), stage, n * kv);
    }
  }
  RK_CUDA(cudaEventCreateWithFlags(&c->ev_layer[l], cudaEventDisableTiming));
  RK_CUDA(cudaEventRecord(c->ev_layer[l], c->xfer));
  c->deferred[l] = 0;
}
void ensure_cache_all(rk_cache* c) {
  for (uint64_t l = 0; l < c->deferred.size(); ++l) ensure_cache_layer(c, l);
}
}  // namespace rk

extern "C" {

int rk_abi_version(void) { return RK_ABI_VERSION; }
const char* rk_last_error(void) { return g_err.c_str(); }

int rk_engine_create(int device, rk_engine** out) {
  return guard([&] {
    require(out != nullptr, RK_ERR_INVALID_ARGUMENT, "null out");
    int n = 0;
    RK_CUDA(cudaGetDeviceCount(&n));
    require(device >= 0 && device < n, RK_ERR_INVALID_ARGUMENT, "no such CUDA device");
    DeviceGuard g(device);
    auto e = std::make_unique<rk_engine>();
    e->device = device;
    RK_CUDA(cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, device));
    int major = 0;
    RK_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    require(major == 10, RK_ERR_RUNTIME, "relaykv-b200 kernels are built for sm_100a (B200)");
    RK_CUDA(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    RK_CUDA(cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking));
    // copy streams at the highest priority: their small fp32->bf16 convert
    // kernels take the next free SM slot instead of queueing behind the pass
    int prio_lo = 0, prio_hi = 0;
    RK_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    for (auto& x : e->xfer) RK_CUDA(cudaStreamCreateWithPriority(&x, cudaStreamNonBlocking, prio_hi));
    {
      const char* env = std::getenv("RK_HOST_THREADS");
      int t = env ? std::atoi(env) : (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
      e->host_pool = std::make_unique<HostPool>(std::max(1, t));
    }
    RK_CUDA(cudaEventCreateWithFlags(&e->side_fork, cudaEventDisableTiming));
    RK_CUDA(cudaEventCreateWithFlags(&e->side_join, cudaEventDisableTiming));
    e->status.alloc(64);
    RK_CUDA(cudaMemset(e->status.p, 0, 64));
    e->pinned_bytes = 1 << 20;
    RK_CUDA(cudaMallocHost(&e->pinned, e->pinned_bytes));
    *out = e.release();
  });
}

void rk_engine_destroy(rk_engine* e) {
  if (!e) return;
  DeviceGuard g(e->device, true);
  cudaStreamSynchronize(e->stream);
  delete e;
}

int rk_engine_synchronize(rk_engine* e) {
  return guard([&] {
    DeviceGuard g(e->device);
    RK_CUDA(cudaStreamSynchronize(e->stream));
    if (e->side) RK_CUDA(cudaStreamSynchronize(e->side));
  });
}
void* rk_engine_stream(rk_engine* e) { return e ? (void*)e->stream : nullptr; }
uint64_t rk_engine_launch_count(rk_engine* e) { return e ? e->launches : 0; }
int rk_engine_set_fused(rk_engine* e, int enable) {
  return guard([&] { e->fused = enable; });
}

int rk_engine_set_graphs(rk_engine* e, int enable) {
  return guard([&] { e->use_graphs = enable; });
}

uint64_t rk_weights_num_tensors(const rk_model_spec* s) { return s ? num_tensors(*s) : 0; }

int rk_weights_init(rk_engine* e, const rk_model_spec* spec, uint64_t seed, int precision,
                    rk_weights** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    std::unique_ptr<rk_weights> w(new_weights(e, spec, precision));
    const rk_model_spec& s = *spec;
    // init_weights (model.cpp:81-114): one SplitMix64 stream, draw order
    // embedding, per layer (w_q, w_k, w_v, w_o, w_gate, w_up, w_down), head;
    // gains are ones and draw nothing.
    uint64_t state = seed ^ 0x72656c6179ull;
    const float kSqrt3 = 1.7320508f;
    const float d_in = 1.0f / std::sqrt(static_cast<float>(s.d_model));
    const float ff_in = 1.0f / std::sqrt(static_cast<float>(s.d_ff));
    const float q_in = 1.0f / std::sqrt(static_cast<float>(s.num_heads * s.d_head)) /
                       (2.0f * static_cast<float>(s.num_layers));
    size_t maxn = 0;
    for (size_t i = 0; i < num_tensors(s); ++i) {
      const TensorDesc td = tensor_desc(s, i);
      maxn = std::max(maxn, td.rows * td.cols);
    }
    DevBuf tmp(maxn * 4);
    float* t = tmp.as<float>();
    cudaStream_t st = e->stream;
    auto gen = [&](size_t idx, float sd) {
      const TensorDesc td = tensor_desc(s, idx);
      const size_t n = td.rows * td.cols;
      k::init_uniform(st, t, n, state, sd * kSqrt3);
      state += static_cast<uint64_t>(n) * 0x9e3779b97f4a7c15ull;
      pack_tensor(w.get(), idx, t);
    };
    auto ones = [&](size_t idx) {
      const TensorDesc td = tensor_desc(s, idx);
      k::fill(st, t, td.rows * td.cols, 1.0f);
      pack_tensor(w.get(), idx, t);
    };
    gen(0, 0.02f);
    for (size_t l = 0; l < s.num_layers; ++l) {
      const size_t b = 1 + 9 * l;
      ones(b + 0);
      gen(b + 1, d_in);
      gen(b + 2, d_in);
      gen(b + 3, d_in);
      gen(b + 4, q_in);
      ones(b + 5);
      gen(b + 6, d_in);
      gen(b + 7, d_in);
      gen(b + 8, ff_in);
    }
    ones(1 + 9 * s.num_layers);
    gen(2 + 9 * s.num_layers, d_in);
    if (precision == RK_FP32_TC) build_tc_weights(w.get());
    RK_CUDA(cudaStreamSynchronize(st));
    *out = w.release();
  });
}

int rk_weights_upload(rk_engine* e, const rk_model_spec* spec, const float* const* tensors,
                      uint64_t n_tensors, int precision, rk_weights** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    require(tensors != nullptr && n_tensors == num_tensors(*spec), RK_ERR_INVALID_ARGUMENT,
            "weights upload: expected tensor_table order with " + std::to_string(num_tensors(*spec)) + " tensors");
    std::unique_ptr<rk_weights> w(new_weights(e, spec, precision));
    size_t maxn = 0;
    for (size_t i = 0; i < n_tensors; ++i) {
      const TensorDesc td = tensor_desc(*spec, i);
      maxn = std::max(maxn, td.rows * td.cols);
    }
    DevBuf tmp(maxn * 4);
    for (size_t i = 0; i < n_tensors; ++i) {
      const TensorDesc td = tensor_desc(*spec, i);
      require(tensors[i] != nullptr, RK_ERR_INVALID_ARGUMENT, "null tensor");
      RK_CUDA(cudaMemcpyAsync(tmp.p, tensors[i], td.rows * td.cols * 4, cudaMemcpyHostToDevice, e->stream));
      pack_tensor(w.get(), i, tmp.as<float>());
    }
    if (precision == RK_FP32_TC) build_tc_weights(w.get());
    RK_CUDA(cudaStreamSynchronize(e->stream));
    *out = w.release();
  });
}

int rk_weights_export(rk_weights* w, uint64_t idx, float* out, uint64_t count) {
  return guard([&] {
    DeviceGuard g(w->e->device);
    const rk_model_spec& s = w->s;
    require(idx < num_tensors(s), RK_ERR_INVALID_ARGUMENT, "tensor index out of range");
    const TensorDesc td = tensor_desc(s, idx);
    require(count >= td.rows * td.cols, RK_ERR_INVALID_ARGUMENT, "output buffer too small");
    DevBuf tmp(td.rows * td.cols * 4);
    layer_unpack_tensor(w, idx, tmp.as<float>(), td.rows, td.cols);
    RK_CUDA(cudaMemcpyAsync(out, tmp.p, td.rows * td.cols * 4, cudaMemcpyDeviceToHost, w->e->stream));
    RK_CUDA(cudaStreamSynchronize(w->e->stream));
  });
}

void rk_weights_destroy(rk_weights* w) {
  if (!w) return;
  DeviceGuard g(w->e->device, true);
  cudaStreamSynchronize(w->e->stream);
  delete w;
}

// ---- relay caches ---------------------------------------------------------
namespace {
typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
// cuStreamWaitValue32 through the runtime's driver entry point (no libcuda link)
PFN_waitValue32 wait_value_fn() {
  static PFN_waitValue32 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (PFN_waitValue32) nullptr;
    }
    return reinterpret_cast<PFN_waitValue32>(f);
  }();
  return fn;
}
inline uint32_t* c_flags_of(char* stage, uint64_t R, size_t slot) {
  return reinterpret_cast<uint32_t*>(stage + R * slot);
}
// RelayCache::validate + upload (relay_cache.cpp:18-41). async: everything on
// the copy stream with per-layer events, no host synchronization.
rk_cache* upload_cache(rk_engine* e, rk_weights* w, const rk_relay_cache_view* v, bool async, uint64_t defer_lo = 1,
                       uint64_t defer_hi = 0) {
  require(v != nullptr && w != nullptr, RK_ERR_INVALID_ARGUMENT, "null cache view / weights");
  const uint64_t n = v->segment_len;
  require(n > 0, RK_ERR_INVALID_ARGUMENT, "relay cache: empty segment");
  require(v->num_layers > 0 && v->k_pre && v->v, RK_ERR_INVALID_ARGUMENT,
          "relay cache: per-layer K/V tables disagree");
  require(v->snapshot_layer < v->num_layers, RK_ERR_INVALID_ARGUMENT,
          "relay cache: snapshot layer out of range");
  for (uint64_t j = 0; j < n; ++j)
    require(v->influence[j] >= 0.0f, RK_ERR_INVALID_ARGUMENT, "relay cache: negative influence score");
  auto c = std::make_unique<rk_cache>();
  c->e = e;
  c->precision = w->precision;
  c->elem = w->elem;
  c->L = v->num_layers;
  c->Hkv = v->num_kv_heads;
  c->dh = v->d_head;
  c->d = v->d_model;
  c->n = n;
  c->maxpos = v->max_positions;
  c->theta = v->theta_base;
  c->src_base = v->source_base_position;
  c->snapshot = v->snapshot_layer;
  c->steps = v->decode_steps_observed;
  const size_t kv = c->kv();
  BlockPool* pl = &e->cache_pool;
  c->tokens.alloc_pooled(pl, n * 4);
  c->host_tokens.assign(v->segment_tokens, v->segment_tokens + n);
  c->k_pre.alloc_pooled(pl, c->L * n * kv * c->elem);
  c->v.alloc_pooled(pl, c->L * n * kv * c->elem);
  c->hidden.alloc_pooled(pl, n * c->d * 4);
  c->influence.alloc_pooled(pl, n * 4);
  c->infl_mean.alloc_pooled(pl, 8);
  // (pooled blocks are idle: rk_cache_destroy synchronized their last reader)
  cudaStream_t st = e->stream;
  if (async) {
    st = e->xfer[e->next_xfer];
    e->next_xfer = (e->next_xfer + 1) % rk_engine::kXfer;
    c->xfer = st;
  }
  // influence mean, sequential in double (selector.cpp:37-39) -- cache-static
  double mean = 0.0;
  for (uint64_t j = 0; j < n; ++j) mean += static_cast<double>(v->influence[j]);
  mean /= static_cast<double>(n);
  RK_CUDA(cudaMemcpyAsync(c->tokens.p, v->segment_tokens, n * 4, cudaMemcpyHostToDevice, st));
  RK_CUDA(cudaMemcpyAsync(c->hidden.p, v->hidden_snapshot, n * c->d * 4, cudaMemcpyHostToDevice, st));
  RK_CUDA(cudaMemcpyAsync(c->influence.p, v->influence, n * 4, cudaMemcpyHostToDevice, st));
  k::fill_doubles(st, c->infl_mean.as<double>(), 1, mean);
  if (async) {
    c->async = true;
    RK_CUDA(cudaEventCreateWithFlags(&c->ev_meta, cudaEventDisableTiming));
    RK_CUDA(cudaEventRecord(c->ev_meta, st));
    c->ev_layer.resize(c->L);
  }
  // bf16, asynchronous: the engine's uploader thread converts each layer to
  // bf16 on the host worker pool into a ring of pinned slots and raises a
  // per-layer flag; the copy stream waits on that flag (cuStreamWaitValue32)
  // and moves half the fp32 bytes across PCIe. The conversion of layer l+R
  // waits for the copy that frees its slot. The call returns at once.
  // Opt-in (RK_HOST_CONVERT=1): on the 16-vCPU B200 hosts measured so far the
  // conversion (72 GB/s alone, less next to the running step) is slower than
  // letting PCIe carry fp32 (~50 GB/s) and converting on the device.
  static const bool host_conv_env = [] {
    const char* v = std::getenv("RK_HOST_CONVERT");
    return v ? std::atoi(v) != 0 : false;
  }();
  if (async && c->elem == 2 && host_conv_env && wait_value_fn()) {
    const uint64_t L = c->L, R = std::min<uint64_t>(L, 4);
    const size_t cnt = n * kv, slot = 2 * cnt * 2;
    c->stage_host = e->pinned_pool.acquire(R * slot + L * 4 + 64, &c->stage_host_bytes);
    char* stage = static_cast<char*>(c->stage_host);
    c->flags = reinterpret_cast<volatile uint32_t*>(stage + R * slot);
    for (uint64_t l = 0; l < L; ++l) c->flags[l] = 0;
    void* dflags = nullptr;
    RK_CUDA(cudaHostGetDevicePointer(&dflags, const_cast<uint32_t*>(c->flags), 0));
    auto release_all = [flags = c->flags, L] {
      for (uint64_t l = 0; l < L; ++l) __atomic_store_n(const_cast<uint32_t*>(flags + l), 1u, __ATOMIC_SEQ_CST);
    };
    for (uint64_t l = 0; l < L; ++l) {
      const uint16_t* sk = reinterpret_cast<const uint16_t*>(stage + (l % R) * slot);
      const CUresult r = wait_value_fn()(st, reinterpret_cast<CUdeviceptr>(dflags) + 4 * l, 1u, CU_STREAM_WAIT_VALUE_GEQ);
      if (r != CUDA_SUCCESS) {
        release_all();  // nothing may stay blocked on a flag
        raise(RK_ERR_RUNTIME, "cuStreamWaitValue32 failed: " + std::to_string((int)r));
      }
      RK_CUDA(cudaMemcpyAsync(static_cast<char*>(c->k_pre.p) + l * cnt * 2, sk, cnt * 2, cudaMemcpyHostToDevice, st));
      RK_CUDA(cudaMemcpyAsync(static_cast<char*>(c->v.p) + l * cnt * 2, sk + cnt, cnt * 2, cudaMemcpyHostToDevice, st));
      RK_CUDA(cudaEventCreateWithFlags(&c->ev_layer[l], cudaEventDisableTiming));
      RK_CUDA(cudaEventRecord(c->ev_layer[l], st));
    }
    std::vector<const float*> ks(v->k_pre, v->k_pre + L), vs(v->v, v->v + L);
    std::vector<cudaEvent_t> evs = c->ev_layer;
    HostPool* pool = e->host_pool.get();
    auto task = std::make_shared<std::packaged_task<void()>>([=] {
      try {
        for (uint64_t l = 0; l < L; ++l) {
          if (l >= R && cudaEventSynchronize(evs[l - R]) != cudaSuccess) break;  // slot l % R is free
          uint16_t* dk = reinterpret_cast<uint16_t*>(stage + (l % R) * slot);
          const float* srck = ks[l];
          const float* srcv = vs[l];
          pool->parallel_for(2 * cnt, size_t{1} << 16, [&](size_t b, size_t end) {
            if (b < cnt) f32_to_bf16_host(srck + b, dk + b, std::min(end, cnt) - b);
            if (end > cnt) {
              const size_t b2 = b > cnt ? b - cnt : 0;
              f32_to_bf16_host(srcv + b2, dk + cnt + b2, end - cnt - b2);
            }
          });
          std::atomic_thread_fence(std::memory_order_seq_cst);
          __atomic_store_n(const_cast<uint32_t*>(c_flags_of(stage, R, slot) + l), 1u, __ATOMIC_SEQ_CST);
        }
      } catch (...) {
      }
      release_all();  // (no-op when every layer went through)
    });
    c->conv_done = task->get_future().share();
    if (!e->uploader) e->uploader = std::make_unique<Uploader>(e->device);
    e->uploader->submit([task] { (*task)(); });
    return c.release();
  }
  // bf16: each fp32 layer lands in a staging buffer and is converted on the
  // device; two staging buffers alternate (stream order keeps them safe, no
  // host round trip), so pinned sources stream at copy-engine speed
  if (c->elem == 2) c->staging.alloc_pooled(pl, 2 * n * kv * 4);
  if (async && defer_lo <= defer_hi) {  // these layers cross PCIe only if a later call reads them
    c->deferred.assign(c->L, 0);
    c->host_k.assign(v->k_pre, v->k_pre + c->L);
    c->host_v.assign(v->v, v->v + c->L);
  }
  int flip = 0;
  for (uint64_t l = 0; l < c->L; ++l) {
    if (!c->deferred.empty() && l >= defer_lo && l <= defer_hi) {
      c->deferred[l] = 1;
      continue;
    }
    for (int which = 0; which < 2; ++which) {
      const float* src = which == 0 ? v->k_pre[l] : v->v[l];
      char* dst = static_cast<char*>(which == 0 ? c->k_pre.p : c->v.p) + l * n * kv * c->elem;
      if (c->elem == 4) {
        RK_CUDA(cudaMemcpyAsync(dst, src, n * kv * 4, cudaMemcpyHostToDevice, st));
      } else {
        float* stage = c->staging.as<float>() + (size_t)flip * n * kv;
        flip ^= 1;
        RK_CUDA(cudaMemcpyAsync(stage, src, n * kv * 4, cudaMemcpyHostToDevice, st));
        k::f32_to_bf16(st, reinterpret_cast<__nv_bfloat16*>(dst), stage, n * kv);
      }
    }
    if (async) {
      RK_CUDA(cudaEventCreateWithFlags(&c->ev_layer[l], cudaEventDisableTiming));
      RK_CUDA(cudaEventRecord(c->ev_layer[l], st));
    }
  }
  if (!async) {
    RK_CUDA(cudaStreamSynchronize(st));
    c->staging.release();
  }
  return c.release();
}
}  // namespace

int rk_cache_upload(rk_engine* e, rk_weights* w, const rk_relay_cache_view* v, rk_cache** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    *out = upload_cache(e, w, v, false);
  });
}

int rk_cache_upload_async(rk_engine* e, rk_weights* w, const rk_relay_cache_view* v, rk_cache** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    *out = upload_cache(e, w, v, true);
  });
}

int rk_cache_upload_async_defer(rk_engine* e, rk_weights* w, const rk_relay_cache_view* v, uint64_t defer_lo,
                                uint64_t defer_hi, rk_cache** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    require(v != nullptr && defer_lo <= defer_hi && defer_hi < v->num_layers, RK_ERR_INVALID_ARGUMENT,
            "deferred layer range out of bounds");
    *out = upload_cache(e, w, v, true, defer_lo, defer_hi);
  });
}



int rk_cache_wait(rk_cache* c) {
  return guard([&] {
    require(c != nullptr, RK_ERR_INVALID_ARGUMENT, "null cache");
    DeviceGuard g(c->e->device);
    ensure_cache_all(c);  // the host arrays may be freed after this call
    if (c->async) RK_CUDA(cudaStreamSynchronize(c->xfer));
  });
}

int rk_cache_sync(rk_cache* c) {
  return guard([&] {
    require(c != nullptr, RK_ERR_INVALID_ARGUMENT, "null cache");
    DeviceGuard g(c->e->device);
    if (c->async) RK_CUDA(cudaStreamSynchronize(c->xfer));
  });
}

uint64_t rk_cache_segment_len(const rk_cache* c) { return c ? c->n : 0; }

namespace {
void export_cache(rk_cache* c, int32_t* tokens, float* const* k_pre, float* const* v, float* hidden,
                  float* influence) {
  DeviceGuard g(c->e->device);
  ensure_cache_all(c);
  if (c->async) RK_CUDA(cudaStreamSynchronize(c->xfer));
  cudaStream_t st = c->e->stream;
  const size_t kv = c->kv(), n = c->n;
  if (tokens) RK_CUDA(cudaMemcpyAsync(tokens, c->tokens.p, n * 4, cudaMemcpyDeviceToHost, st));
  if (hidden) RK_CUDA(cudaMemcpyAsync(hidden, c->hidden.p, n * c->d * 4, cudaMemcpyDeviceToHost, st));
  if (influence) RK_CUDA(cudaMemcpyAsync(influence, c->influence.p, n * 4, cudaMemcpyDeviceToHost, st));
  DevBuf tmp;
  if (c->elem == 2) tmp.alloc(n * kv * 4);
  for (uint64_t l = 0; l < c->L; ++l)
    for (int which = 0; which < 2; ++which) {
      float* dst = which == 0 ? (k_pre ? k_pre[l] : nullptr) : (v ? v[l] : nullptr);
      if (!dst) continue;
      const char* src = static_cast<const char*>(which == 0 ? c->k_pre.p : c->v.p) + l * n * kv * c->elem;
      if (c->elem == 4) {
        RK_CUDA(cudaMemcpyAsync(dst, src, n * kv * 4, cudaMemcpyDeviceToHost, st));
      } else {
        k::bf16_to_f32(st, tmp.as<float>(), reinterpret_cast<const __nv_bfloat16*>(src), n * kv);
        RK_CUDA(cudaMemcpyAsync(dst, tmp.p, n * kv * 4, cudaMemcpyDeviceToHost, st));
        RK_CUDA(cudaStreamSynchronize(st));
      }
    }
  RK_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

int rk_cache_export(rk_cache* c, int32_t* tokens, float* const* k_pre, float* const* v,
                    float* hidden, float* influence, uint64_t* src_base, uint64_t* snapshot) {
  return guard([&] {
    require(c != nullptr, RK_ERR_INVALID_ARGUMENT, "null cache");
    export_cache(c, tokens, k_pre, v, hidden, influence);
    if (src_base) *src_base = c->src_base;
    if (snapshot) *snapshot = c->snapshot;
  });
}

// ---- RKRC files (relay_cache.cpp:176-253) ---------------------------------
int rk_cache_save(rk_cache* c, const char* path) {
  return guard([&] {
    require(c != nullptr && path != nullptr, RK_ERR_INVALID_ARGUMENT, "null cache / path");
    const size_t n = c->n, kv = c->kv();
    std::vector<int32_t> tokens(n);
    std::vector<std::vector<float>> kb(c->L, std::vector<float>(n * kv)), vb(c->L, std::vector<float>(n * kv));
    std::vector<float*> kp(c->L), vp(c->L);
    for (uint64_t l = 0; l < c->L; ++l) {
      kp[l] = kb[l].data();
      vp[l] = vb[l].data();
    }
    std::vector<float> hidden(n * c->d), infl(n);
    export_cache(c, tokens.data(), kp.data(), vp.data(), hidden.data(), infl.data());
    std::vector<const float*> kc(kp.begin(), kp.end()), vc(vp.begin(), vp.end());
    rk_relay_cache_view view{c->L, c->Hkv, c->dh, c->d, c->theta, c->maxpos, n, tokens.data(),
                             c->src_base, c->snapshot, c->steps, kc.data(), vc.data(), hidden.data(), infl.data()};
    rkrc_write(path, rkrc_encode(view));
  });
}

int rk_cache_load(rk_engine* e, rk_weights* w, const char* path, int asynchronous, rk_cache** out) {
  return guard([&] {
    require(e != nullptr && path != nullptr && out != nullptr, RK_ERR_INVALID_ARGUMENT, "null engine / path");
    DeviceGuard g(e->device);
    auto file = std::make_shared<HostCacheFile>(rkrc_read(path, asynchronous != 0));
    rk_cache* c = upload_cache(e, w, &file->view, asynchronous != 0);
    if (asynchronous) c->host_keep = file;  // the pinned blob outlives the copies
    *out = c;
  });
}

struct rk_cache_file {
  HostCacheFile f;
};

namespace {
// export_relay_cache validates first (relay_cache.cpp:177)
std::vector<uint8_t> encode_checked(const rk_relay_cache_view* view) {
  require(view != nullptr, RK_ERR_INVALID_ARGUMENT, "null view");
  const rk_relay_cache_view& v = *view;
  require(v.segment_len > 0, RK_ERR_INVALID_ARGUMENT, "relay cache: empty segment");
  require(v.num_layers > 0 && v.k_pre && v.v, RK_ERR_INVALID_ARGUMENT, "relay cache: per-layer K/V tables disagree");
  require(v.snapshot_layer < v.num_layers, RK_ERR_INVALID_ARGUMENT, "relay cache: snapshot layer out of range");
  for (uint64_t j = 0; j < v.segment_len; ++j)
    require(v.influence[j] >= 0.0f, RK_ERR_INVALID_ARGUMENT, "relay cache: negative influence score");
  return rkrc_encode(v);
}
}  // namespace

int rk_cache_file_write(const rk_relay_cache_view* view, const char* path) {
  return guard([&] {
    require(path != nullptr, RK_ERR_INVALID_ARGUMENT, "null path");
    rkrc_write(path, encode_checked(view));
  });
}

int rk_cache_file_encode(const rk_relay_cache_view* view, uint8_t* out, uint64_t capacity, uint64_t* size) {
  return guard([&] {
    require(size != nullptr, RK_ERR_INVALID_ARGUMENT, "null size");
    const std::vector<uint8_t> b = encode_checked(view);
    *size = b.size();
    if (out) {
      require(capacity >= b.size(), RK_ERR_INVALID_ARGUMENT, "rk_cache_file_encode: buffer too small");
      std::memcpy(out, b.data(), b.size());
    }
  });
}

int rk_cache_file_decode(const uint8_t* bytes, uint64_t size, rk_cache_file** out, rk_relay_cache_view* view) {
  return guard([&] {
    require((bytes != nullptr || size == 0) && out != nullptr && view != nullptr, RK_ERR_INVALID_ARGUMENT,
            "null argument");
    auto f = std::make_unique<rk_cache_file>();
    f->f = rkrc_decode(bytes, size);
    *view = f->f.view;
    *out = f.release();
  });
}

int rk_cache_file_read(const char* path, rk_cache_file** out, rk_relay_cache_view* view) {
  return guard([&] {
    require(path != nullptr && out != nullptr && view != nullptr, RK_ERR_INVALID_ARGUMENT, "null argument");
    auto f = std::make_unique<rk_cache_file>();
    f->f = rkrc_read(path, false);
    *view = f->f.view;
    *out = f.release();
  });
}

void rk_cache_file_free(rk_cache_file* f) { delete f; }

rk_cache::~rk_cache() {
  if (conv_done.valid()) conv_done.wait();  // the uploader job is done with the staging ring and events
  if (stage_host) e->pinned_pool.release(stage_host, stage_host_bytes);
  if (ev_meta) cudaEventDestroy(ev_meta);
  for (cudaEvent_t ev : ev_layer)
    if (ev) cudaEventDestroy(ev);
}

void rk_cache_destroy(rk_cache* c) {
  if (!c) return;
  DeviceGuard g(c->e->device, true);
  cudaStreamSynchronize(c->e->stream);
  if (c->async) cudaStreamSynchronize(c->xfer);
  delete c;
}

// ---- contexts -------------------------------------------------------------
int rk_context_create(rk_engine* e, rk_weights* w, rk_context** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    auto c = std::make_unique<rk_context>();
    c->e = e;
    c->w = w;
    c->elem = w->elem;
    *out = c.release();
  });
}

int rk_context_clone(rk_context* src, rk_context** out) {
  return guard([&] {
    DeviceGuard g(src->e->device);
    auto c = std::make_unique<rk_context>();
    c->e = src->e;
    c->w = src->w;
    c->elem = src->elem;
    c->reserve(src->cap);
    c->size = src->size;
    if (src->cap) {
      RK_CUDA(cudaMemcpyAsync(c->k.p, src->k.p, src->k.bytes, cudaMemcpyDeviceToDevice, src->e->stream));
      RK_CUDA(cudaMemcpyAsync(c->v.p, src->v.p, src->v.bytes, cudaMemcpyDeviceToDevice, src->e->stream));
    }
    for (const auto& m : src->segs) {
      rk_segment_marks nm;
      nm.base = m.base;
      nm.len = m.len;
      nm.origin.alloc(m.origin.bytes);
      RK_CUDA(cudaMemcpyAsync(nm.origin.p, m.origin.p, m.origin.bytes, cudaMemcpyDeviceToDevice, src->e->stream));
      c->segs.push_back(std::move(nm));
    }
    RK_CUDA(cudaStreamSynchronize(src->e->stream));
    *out = c.release();
  });
}

uint64_t rk_context_size(const rk_context* c) { return c ? c->size : 0; }
uint64_t rk_context_num_segments(const rk_context* c) { return c ? c->segs.size() : 0; }

int rk_context_segment(rk_context* c, uint64_t index, uint64_t* base, uint64_t* len, uint8_t* origin) {
  return guard([&] {
    require(index < c->segs.size(), RK_ERR_INVALID_ARGUMENT, "segment index out of range");
    const rk_segment_marks& m = c->segs[index];
    if (base) *base = m.base;
    if (len) *len = m.len;
    if (origin && m.origin.bytes) {
      DeviceGuard g(c->e->device);
      RK_CUDA(cudaMemcpyAsync(origin, m.origin.p, c->w->s.num_layers * m.len, cudaMemcpyDeviceToHost, c->e->stream));
      RK_CUDA(cudaStreamSynchronize(c->e->stream));
    }
  });
}

int rk_context_export(rk_context* c, uint64_t layer, uint64_t pos, uint64_t count, float* k, float* v) {
  return guard([&] {
    DeviceGuard g(c->e->device);
    require(layer < c->w->s.num_layers && pos + count <= c->size, RK_ERR_INVALID_ARGUMENT,
            "context export out of range");
    const size_t kv = c->w->kv();
    cudaStream_t st = c->e->stream;
    DevBuf tmp;
    if (c->elem == 2) tmp.alloc(count * kv * 4);
    for (int which = 0; which < 2; ++which) {
      float* dst = which == 0 ? k : v;
      if (!dst || count == 0) continue;
      const char* src = static_cast<const char*>(which == 0 ? c->k_layer(layer) : c->v_layer(layer)) + pos * kv * c->elem;
      if (c->elem == 4) {
        RK_CUDA(cudaMemcpyAsync(dst, src, count * kv * 4, cudaMemcpyDeviceToHost, st));
      } else {
        k::bf16_to_f32(st, tmp.as<float>(), reinterpret_cast<const __nv_bfloat16*>(src), count * kv);
        RK_CUDA(cudaMemcpyAsync(dst, tmp.p, count * kv * 4, cudaMemcpyDeviceToHost, st));
        RK_CUDA(cudaStreamSynchronize(st));
      }
    }
    RK_CUDA(cudaStreamSynchronize(st));
  });
}

void rk_context_destroy(rk_context* c) {
  if (!c) return;
  DeviceGuard g(c->e->device, true);
  cudaStreamSynchronize(c->e->stream);
  delete c;
}

// ---- hot path --------------------------------------------------------------
int rk_prefill(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* tokens, uint64_t n,
               uint64_t base, float* last_logits) {
  return guard([&] {
    DeviceGuard g(e->device);
    Runner r(e, w);
    r.prefill(ctx, tokens, n, base, last_logits != nullptr);
    r.finish();
    if (last_logits) r.download_logits(last_logits);
  });
}

int rk_prefill_trace(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* tokens, uint64_t n,
                     uint64_t base, const rk_trace_request* req) {
  return guard([&] {
    DeviceGuard g(e->device);
    const rk_trace_request none{};
    Runner r(e, w);
    r.prefill_trace(ctx, tokens, n, base, req ? *req : none);
    r.finish();
  });
}

int rk_row_logits_from_layer(rk_engine* e, rk_weights* w, rk_context* ctx, const float* hidden_row,
                             uint64_t first_layer, uint64_t position, float* logits) {
  return guard([&] {
    DeviceGuard g(e->device);
    require(ctx != nullptr && ctx->w == w, RK_ERR_INVALID_ARGUMENT, "context belongs to other weights");
    require(hidden_row != nullptr && logits != nullptr, RK_ERR_INVALID_ARGUMENT, "null hidden row or logits");
    require(first_layer <= w->s.num_layers, RK_ERR_INVALID_ARGUMENT, "row_logits_from_layer: first_layer out of range");
    require(position < ctx->size, RK_ERR_INVALID_ARGUMENT, "row_logits_from_layer: position outside the context");
    DevBuf row(w->s.d_model * 4);
    RK_CUDA(cudaMemcpyAsync(row.p, hidden_row, w->s.d_model * 4, cudaMemcpyHostToDevice, e->stream));
    Runner r(e, w);
    r.row_logits_from_layer(ctx, row.as<float>(), first_layer, position);
    r.finish();
    r.download_logits(logits);
  });
}

int rk_host_pin(void* ptr, uint64_t bytes) {
  return guard([&] {
    require(ptr != nullptr && bytes > 0, RK_ERR_INVALID_ARGUMENT, "rk_host_pin: empty range");
    RK_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
  });
}

int rk_host_unpin(void* ptr) {
  return guard([&] { RK_CUDA(cudaHostUnregister(ptr)); });
}

int rk_relay_extend(rk_engine* e, rk_weights* w, rk_context* ctx, rk_cache* cache,
                    const rk_layer_profile* profile, const rk_relay_options* opts, rk_relay_output* out) {
  return guard([&] {
    DeviceGuard g(e->device);
    require(opts != nullptr, RK_ERR_INVALID_ARGUMENT, "null options");
    Runner r(e, w);
    ExtendResult res = r.relay_extend(ctx, cache, profile, *opts);
    r.finish();
    r.resolve(res);
    r.fill_output(res, ctx, out);
  });
}

int rk_relay_prefill(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* prefix,
                     uint64_t n_prefix, rk_cache* cache, const rk_layer_profile* profile,
                     const rk_relay_options* opts, rk_relay_output* out, float* end_logits) {
  return guard([&] {
    DeviceGuard g(e->device);
    require(opts != nullptr && ctx != nullptr && cache != nullptr, RK_ERR_INVALID_ARGUMENT, "null argument");
    require(ctx->size == 0, RK_ERR_INVALID_ARGUMENT, "relay_prefill: context must be empty");
    Runner r(e, w);
    r.begin_timer();
    if (n_prefix > 0) r.prefill(ctx, prefix, n_prefix, 0, false);
    const float prefix_ms = r.lap_ms();
    ExtendResult res = r.relay_extend(ctx, cache, profile, *opts);
    r.segment_end_logits(ctx, res);
    r.finish();
    r.resolve(res);
    res.stats.wall.fresh_ms = prefix_ms;
    res.stats.wall.total_ms += prefix_ms;
    res.stats.flops_cost += rk_flops_span_full(&w->s, 0, n_prefix);
    res.stats.flops_full_equiv += rk_flops_span_full(&w->s, 0, n_prefix);
    r.fill_output(res, ctx, out);
    if (end_logits) r.download_logits(end_logits);
  });
}

int rk_agent_prefill(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* prefix,
                     uint64_t n_prefix, rk_cache* const* ups, uint64_t n_up, const int32_t* suffix,
                     uint64_t n_suffix, const rk_layer_profile* profile, const rk_relay_options* opts,
                     rk_relay_output* outs, float* end_logits, int32_t* first_token) {
  return guard([&] {
    DeviceGuard g(e->device);
    require(opts != nullptr && ctx != nullptr, RK_ERR_INVALID_ARGUMENT, "null argument");
    require(ctx->size == 0, RK_ERR_INVALID_ARGUMENT, "agent prefill: context must be empty");
    static const bool host_timing = std::getenv("RK_HOST_TIMING") != nullptr;  // (diagnostic: stderr)
    const auto t0 = std::chrono::steady_clock::now();
    Runner r(e, w);
    std::vector<ExtendResult> results;
    r.agent_prefill(ctx, prefix, n_prefix, ups, n_up, suffix, n_suffix, profile, *opts, results);
    r.stage_results(results, first_token != nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    r.finish();
    const auto t2 = std::chrono::steady_clock::now();
    for (auto& res : results) r.resolve(res, outs != nullptr);  // (wall timings only reach the caller via outs)
    if (outs)
      for (size_t u = 0; u < results.size(); ++u) r.fill_output(results[u], ctx, &outs[u]);
    if (end_logits) r.download_logits(end_logits);
    if (first_token) *first_token = r.first_token();
    if (host_timing) {
      const auto t3 = std::chrono::steady_clock::now();
      auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
      std::fprintf(stderr, "[host] agent_prefill enqueue %.1f us, wait %.1f us, after %.1f us\n", us(t0, t1),
                   us(t1, t2), us(t2, t3));
    }
  });
}

int rk_cache_capture_prefill(rk_engine* e, rk_weights* w, rk_context* ctx, const int32_t* tokens,
                             uint64_t n, uint64_t snapshot, int include_self, rk_cache** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    Runner r(e, w);
    *out = r.capture_prefill(ctx, tokens, n, snapshot, include_self != 0);
    r.finish();
  });
}

int rk_cache_capture_decode(rk_engine* e, rk_weights* w, rk_context* ctx, const float* first_logits,
                            uint64_t n, uint64_t snapshot, int include_self, rk_cache** out) {
  return guard([&] {
    DeviceGuard g(e->device);
    Runner r(e, w);
    *out = r.capture_decode(ctx, first_logits, n, snapshot, include_self != 0);
    r.finish();
  });
}

// FLOP model (relay_engine.cpp:72-110)
double rk_flops_span_full(const rk_model_spec* s, uint64_t base, uint64_t n) {
  const double d = (double)s->d_model, kv = (double)(s->num_kv_heads * s->d_head), ff = (double)s->d_ff;
  const double pm = 2.0 * d * (2.0 * d + 2.0 * kv) + 6.0 * d * ff;
  const double b = (double)base, nn = (double)n, dhH = (double)(s->d_head * s->num_heads);
  const double attn = 4.0 * dhH * (nn * b + nn * (nn + 1.0) / 2.0);
  const double layers = (double)s->num_layers;
  return layers * nn * pm + layers * attn;
}
double rk_flops_segment_schedule(const rk_model_spec* s, uint64_t base, uint64_t n, uint64_t lo,
                                 uint64_t hi, uint64_t sparse_hi, uint64_t selected) {
  const double d = (double)s->d_model, kv = (double)(s->num_kv_heads * s->d_head), ff = (double)s->d_ff;
  const double pm = 2.0 * d * (2.0 * d + 2.0 * kv) + 6.0 * d * ff;
  const double band_layers = (double)(hi - lo + 1), sparse_layers = (double)(sparse_hi - hi);
  const double dhH = (double)(s->d_head * s->num_heads);
  const double avg_ctx = (double)base + ((double)n + 1.0) / 2.0;
  const double b = (double)base, nn = (double)n;
  const double attn = 4.0 * dhH * (nn * b + nn * (nn + 1.0) / 2.0);
  const double band = band_layers * (nn * pm + attn);
  const double sparse = sparse_layers * (double)selected * (pm + 4.0 * dhH * avg_ctx);
  return band + sparse;
}

}  // extern "C"

// ============================================================================
// profiling + context reset
// ============================================================================
namespace rk {
const char* intern(const std::string& s) {
  static std::set<std::string> pool;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  return pool.insert(s).first->c_str();
}
Profiler& profiler(rk_engine* e) {
  if (!e->prof) e->prof.reset(new Profiler());
  return *e->prof;
}
ProfScope::ProfScope(rk_engine* eng, const char* name, double flops, double bytes) : e(eng) {
  on = eng->prof && eng->prof->on;
  rec.name = name;
  rec.flops = flops;
  rec.bytes = bytes;
  if (on) rec.ev0 = eng->prof->ev(eng->stream);
}
ProfScope::~ProfScope() {
  if (!on) return;
  try {
    rec.ev1 = e->prof->ev(e->stream);
    e->prof->recs.push_back(rec);
  } catch (...) {
  }
}
}  // namespace rk

extern "C" {
int rk_engine_profile(rk_engine* e, int enable) {
  return guard([&] {
    DeviceGuard g(e->device);
    RK_CUDA(cudaStreamSynchronize(e->stream));
    Profiler& p = profiler(e);
    p.on = enable != 0;
    p.recs.clear();
    p.next = 0;
  });
}

int rk_engine_profile_read(rk_engine* e, rk_kernel_stat* out, uint64_t cap, uint64_t* count) {
  return guard([&] {
    DeviceGuard g(e->device);
    RK_CUDA(cudaStreamSynchronize(e->stream));
    Profiler& p = profiler(e);
    std::vector<rk_kernel_stat> agg;
    for (const ProfRec& r : p.recs) {
      float ms = 0.f;
      RK_CUDA(cudaEventElapsedTime(&ms, p.pool[r.ev0], p.pool[r.ev1]));
      double flops = r.flops, bytes = r.bytes;
      if (r.kind != 0) {
        int M = r.rows_max;
        if (r.rows_dev) RK_CUDA(cudaMemcpy(&M, r.rows_dev, 4, cudaMemcpyDeviceToHost));
        if (r.kind == 1) {
          flops = 2.0 * M * r.N * r.K;
        } else {
          std::vector<int> pos(M);
          if (M) RK_CUDA(cudaMemcpy(pos.data(), r.pos, M * 4, cudaMemcpyDeviceToHost));
          double ctx = 0;
          for (int v : pos) ctx += v + 1;
          flops = 4.0 * r.dh * r.H * ctx;
        }
      }
      rk_kernel_stat* st = nullptr;
      for (auto& a : agg)
        if (std::strncmp(a.name, r.name, sizeof a.name) == 0) st = &a;
      if (!st) {
        agg.push_back(rk_kernel_stat{});
        st = &agg.back();
        std::strncpy(st->name, r.name, sizeof st->name - 1);
      }
      st->launches += 1;
      st->total_ms += ms;
      st->flops += flops;
      st->bytes += bytes;
    }
    if (count) *count = agg.size();
    for (size_t i = 0; i < agg.size() && i < cap; ++i) out[i] = agg[i];
  });
}

int rk_context_reset(rk_context* c) {
  return guard([&] {
    DeviceGuard g(c->e->device);
    RK_CUDA(cudaStreamSynchronize(c->e->stream));
    c->size = 0;
    c->segs.clear();
  });
}
}  // extern "C"

// ---- offline layer profiler (profiler.cpp:155-175, metrics.cpp:118-238) -----
int rk_token_deviation(rk_cache* reuse, rk_cache* full, double* value_cos, double* key_cos, double* value_norm,
                       double* key_norm) {
  return guard([&] {
    require(reuse != nullptr && full != nullptr, RK_ERR_INVALID_ARGUMENT, "null cache");
    // token_deviation's shape checks (metrics.cpp:120-147)
    require(reuse->L == full->L && reuse->L > 0, RK_ERR_INVALID_ARGUMENT, "token_deviation: layer count mismatch");
    require(reuse->n == full->n && reuse->kv() == full->kv() && reuse->elem == full->elem, RK_ERR_INVALID_ARGUMENT,
            "token_deviation: shape mismatch at layer 0");
    require(reuse->Hkv > 0 && reuse->kv() % reuse->Hkv == 0, RK_ERR_INVALID_ARGUMENT,
            "token_deviation: kv width not divisible by head count");
    DeviceGuard g(reuse->e->device);
    rk_engine* e = reuse->e;
    ensure_cache_all(reuse);
    ensure_cache_all(full);
    if (reuse->async) RK_CUDA(cudaStreamSynchronize(reuse->xfer));
    if (full->async) RK_CUDA(cudaStreamSynchronize(full->xfer));
    const size_t n = reuse->n, L = reuse->L;
    DevBuf out(4 * n * L * sizeof(double));
    k::token_deviation(e->stream, reuse->k_pre.p, reuse->v.p, full->k_pre.p, full->v.p, reuse->elem, (int)L, (int)n,
                       (int)reuse->kv(), (int)reuse->Hkv, out.as<double>());
    e->launches += 1;
    double* dst[4] = {value_cos, key_cos, value_norm, key_norm};
    for (int m = 0; m < 4; ++m)
      if (dst[m])
        RK_CUDA(cudaMemcpyAsync(dst[m], out.as<double>() + m * n * L, n * L * sizeof(double), cudaMemcpyDeviceToHost,
                                e->stream));
    RK_CUDA(cudaStreamSynchronize(e->stream));
  });
}

namespace {
void put_curve(const prof::Curve& c, double* s, double* rho, uint8_t* deg) {
  for (size_t l = 0; l < c.s.size(); ++l) {
    if (s) s[l] = c.s[l];
    if (rho) rho[l] = c.rho[l];
    if (deg) deg[l] = c.deg[l];
  }
}
}  // namespace

int rk_layer_curve(const double* value_cos, uint64_t n, uint64_t L, double* s, double* rho, uint8_t* deg) {
  return guard([&] {
    require(value_cos != nullptr || n * L == 0, RK_ERR_INVALID_ARGUMENT, "null deviation matrix");
    put_curve(prof::layer_curve(value_cos, n, L), s, rho, deg);
  });
}

int rk_average_curves(const double* s, const double* rho, const uint8_t* deg, uint64_t k, uint64_t L, double* s_out,
                      double* rho_out, uint8_t* deg_out) {
  return guard([&] {
    std::vector<prof::Curve> cs(k);
    for (uint64_t i = 0; i < k; ++i) {
      cs[i].s.assign(s + i * L, s + (i + 1) * L);
      cs[i].rho.assign(rho + i * L, rho + (i + 1) * L);
      cs[i].deg.assign(deg + i * L, deg + (i + 1) * L);
    }
    put_curve(prof::average(cs), s_out, rho_out, deg_out);
  });
}

int rk_profile_from_curve(const double* s, const double* rho, const uint8_t* deg, uint64_t L,
                          const rk_profiler_params* params, rk_profile_result* out, double* curve_rho_out) {
  return guard([&] {
    require(s && rho && deg && params && out, RK_ERR_INVALID_ARGUMENT, "null argument");
    prof::Curve c;
    c.s.assign(s, s + L);
    c.rho.assign(rho, rho + L);
    c.deg.assign(deg, deg + L);
    std::vector<double> crho;
    *out = prof::from_curve(c, *params, &crho);
    if (curve_rho_out) std::copy(crho.begin(), crho.end(), curve_rho_out);
  });
}

int rk_profile_model(rk_engine* e, rk_weights* w, const rk_two_stage_config* calib, const rk_profiler_params* params,
                     rk_profile_result* out, double* curve_s, double* curve_rho) {
  return guard([&] {
    require(e && w && calib && params && out, RK_ERR_INVALID_ARGUMENT, "null argument");
    prof::validate_params(*params);
    prof::validate_calib(*calib);
    DeviceGuard g(e->device);
    const rk_model_spec& spec = w->s;
    const size_t L = spec.num_layers, V = spec.vocab_size;
    struct CacheDel {
      void operator()(rk_cache* c) const { rk_cache_destroy(c); }
    };
    std::vector<prof::Curve> curves;
    std::vector<float> logits(V);
    for (uint64_t i = 0; i < calib->instances; ++i) {
      try {
        // make_two_stage_instance (metrics.cpp:280-322)
        const uint64_t seed = calib->seed + 0x9e37u * (i + 1);
        const size_t p1 = prof::pick_length(seed, 11, calib->stage1_prefix_min, calib->stage1_prefix_max);
        const std::vector<int32_t> pre1 = prof::synthetic_tokens(seed, 21, p1, V);
        const std::vector<int32_t> pre2 =
            calib->identical_prefix
                ? pre1
                : prof::synthetic_tokens(seed, 22,
                                         prof::pick_length(seed, 12, calib->stage2_prefix_min, calib->stage2_prefix_max),
                                         V);
        auto make_ctx = [&] {
          auto c = std::make_unique<rk_context>();
          c->e = e;
          c->w = w;
          c->elem = w->elem;
          return c;
        };
        // stage 1: prompt prefill, then greedy decode of the segment with capture
        auto ctx1 = make_ctx();
        std::unique_ptr<rk_cache, CacheDel> reuse, full;
        {
          Runner r(e, w);
          r.prefill(ctx1.get(), pre1.data(), pre1.size(), 0, true);
          r.finish();
          r.download_logits(logits.data());
        }
        {
          Runner r(e, w);
          reuse.reset(r.capture_decode(ctx1.get(), logits.data(), calib->segment_len, calib->snapshot_layer, false));
          r.finish();
        }
        // full side: prefill of (stage-2 prefix + segment), pre-RoPE keys of
        // the segment rows (build_comparison_setting kDecoding, metrics.cpp:336-352)
        auto ctx2 = make_ctx();
        {
          Runner r(e, w);
          r.prefill(ctx2.get(), pre2.data(), pre2.size(), 0, false);
          full.reset(r.capture_prefill(ctx2.get(), reuse->host_tokens.data(), reuse->n, calib->snapshot_layer, false));
          r.finish();
        }
        const size_t n = reuse->n;
        std::vector<double> vc(n * L);
        const int st = rk_token_deviation(reuse.get(), full.get(), vc.data(), nullptr, nullptr, nullptr);
        if (st != RK_OK) raise(st, rk_last_error());
        curves.push_back(prof::layer_curve(vc.data(), n, L));
      } catch (const Error& ex) {
        raise(RK_ERR_RUNTIME, "calibration instance " + std::to_string(i) + ": " + ex.what());
      }
    }
    const prof::Curve avg = prof::average(curves);
    std::vector<double> crho;
    *out = prof::from_curve(avg, *params, &crho);
    if (curve_s) std::copy(avg.s.begin(), avg.s.end(), curve_s);
    if (curve_rho) std::copy(crho.begin(), crho.end(), curve_rho);
  });
}
