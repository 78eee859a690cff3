// layer_bf16.cu -- RK_BF16 decoder layer (run_layer_rows, model.cpp:237-280):
//   RMSNorm (fp32 -> bf16) -> QKV GEMM [RoPE, K/V scatter into the context]
//   -> tcgen05 attention -> O GEMM (+= hidden) -> RMSNorm -> gate/up GEMM
//   [SiLU(g)*u] -> down GEMM (+= hidden).
// The residual stream stays fp32; GEMM operands are bf16 with fp32 accumulation.
#include <cmath>

#include "layer.h"
#include "layer_bf16.h"
#include "sm100.cuh"

namespace rk {
namespace {
// 256-thread launch with programmatic stream serialization (sm100.cuh pdl_*).
template <typename... KArgs, typename... Args>
void launch_pdl1(void (*kern)(KArgs...), dim3 grid, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  RK_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}


__device__ __forceinline__ int live(const Rows& r) { return r.rows_dev ? *r.rows_dev : r.rows_max; }

// rms_norm (tensor.cpp:109-119) in fp32, output bf16 (GEMM operand). One warp per row.
__global__ void rmsnorm_bf16_kernel(const float* __restrict__ x, const float* __restrict__ gain, float eps,
                                    __nv_bfloat16* __restrict__ out, Rows rows, int d) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int M = live(rows);
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= M) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * d);
  float ss = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / (float)d + eps);
  const float4* g = reinterpret_cast<const float4*>(gain);
  uint2* o = reinterpret_cast<uint2*>(out + (size_t)row * d);
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i], gg = g[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x * inv * gg.x, v.y * inv * gg.y);
    __nv_bfloat162 b = __floats2bfloat162_rn(v.z * inv * gg.z, v.w * inv * gg.w);
    o[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
}

// First layer of a row set (rows not produced by the previous residual GEMM):
// bf16 copy of the residual rows (the GEMM operand; the norm gain is folded
// into the weights) and 1/rms per row, applied in the consumer's epilogue.
__global__ void norm_prep_kernel(const float* __restrict__ x, float eps, __nv_bfloat16* __restrict__ out,
                                 float* __restrict__ inv, Rows rows, int d) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int M = live(rows);
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= M) return;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * d);
  uint2* o = reinterpret_cast<uint2*>(out + (size_t)row * d);
  float ss = 0.f;
  for (int i = lane; i < d / 4; i += 32) {
    const float4 v = xr[i];
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    o[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  }
  for (int m = 16; m; m >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, m);
  if (lane == 0) inv[row] = rsqrtf(ss / (float)d + eps);
}

// Pure-query pass (row_logits_from_layer, model.cpp:339-362): the row's own
// context cell is temporarily replaced by its fresh K/V and restored after
// the attention, so nothing is committed.
__global__ void swap_row_kernel(__nv_bfloat16* ctx_k, __nv_bfloat16* ctx_v, const int* pos, int kv,
                                __nv_bfloat16* save, int restore) {
  const size_t base = (size_t)pos[0] * kv;
  for (int i = threadIdx.x; i < kv; i += blockDim.x) {
    if (restore) {
      ctx_k[base + i] = save[i];
      ctx_v[base + i] = save[kv + i];
    } else {
      save[i] = ctx_k[base + i];
      save[kv + i] = ctx_v[base + i];
    }
  }
}

}  // namespace

static int* split_flags(rk_engine* e) {
  Scratch& S = *e->scratch;
  constexpr size_t kFlags = 1 << 16;
  if (S.gemm_tmp.bytes < kFlags * 4) {
    S.gemm_tmp.ensure(kFlags * 4);
    RK_CUDA(cudaMemsetAsync(S.gemm_tmp.p, 0, kFlags * 4, e->stream));
  }
  return S.gemm_tmp.as<int>();
}

void rmsnorm_bf16(cudaStream_t st, const float* x, const float* gain, float eps, __nv_bfloat16* out, Rows rows,
                  int d) {
  if (rows.rows_max <= 0) return;
  launch_pdl1(rmsnorm_bf16_kernel, dim3((rows.rows_max + 7) / 8), st, x, gain, eps, out, rows, d);
}

// Fused-RMSNorm buffers (scratch): per-row 1/rms, partial sums, m-tile counters.
struct NormBufs {
  float* inv;
  float* part;
  int* cnt;
};
static NormBufs norm_bufs(rk_engine* e, size_t rows) {
  Scratch& S = *e->scratch;
  S.norm_inv.ensure(rows * 4 + 256);
  S.norm_part.ensure(rows * kNormSlots * 4 + 256);
  const size_t cnt_bytes = ((rows + 127) / 128 * 8 + 64) * 4;  // [m tile][quarter or cluster owner]
  if (S.norm_cnt.bytes < cnt_bytes) {
    S.norm_cnt.ensure(cnt_bytes);
    RK_CUDA(cudaMemsetAsync(S.norm_cnt.p, 0, S.norm_cnt.bytes, e->stream));
  }
  return {S.norm_inv.as<float>(), S.norm_part.as<float>(), S.norm_cnt.as<int>()};
}

void run_layer_bf16(rk_engine* e, rk_weights* w, rk_context* ctx, int l, float* hidden, Rows rows, bool commit,
                    int max_ctx, float* probs, int key_lo, int key_n, void* cap_k, void* cap_v, bool prepared,
                    int tail) {
  (void)max_ctx;
  Scratch& S = *e->scratch;
  const rk_model_spec& s = w->s;
  const rk_layer_dev& ly = w->layers[l];
  const int d = s.d_model, q = (int)w->q(), kv = (int)w->kv(), ff = s.d_ff;
  cudaStream_t st = e->stream;
  auto* normed = S.normed.as<__nv_bfloat16>();
  auto* qbuf = S.qkv.as<__nv_bfloat16>();
  auto* attn = S.attn.as<__nv_bfloat16>();
  auto* act = S.act.as<__nv_bfloat16>();
  auto* ck = static_cast<__nv_bfloat16*>(ctx->k_layer(l));
  auto* cv = static_cast<__nv_bfloat16*>(ctx->v_layer(l));
  // live rows of a sparse pass are known only on the device: plan tiles for ~1/3
  int hint = rows.rows_dev ? (rows.hint > 0 ? rows.hint : std::max(1, rows.rows_max / 3)) : rows.rows_max;
  int* flags = split_flags(e);
  __nv_bfloat16* save = reinterpret_cast<__nv_bfloat16*>(S.seg_hidden_out.as<char>() + 0);
  if (!commit) {
    S.sub_hidden.ensure((size_t)2 * kv * 2 + 256);
    save = S.sub_hidden.as<__nv_bfloat16>();
    swap_row_kernel<<<1, 256, 0, st>>>(ck, cv, rows.pos, kv, save, 0);
    e->launches += 1;
  }

  const NormBufs nb = norm_bufs(e, (size_t)rows.rows_max);
  if (!prepared) {  // else the previous layer's down GEMM left bf16 rows + 1/rms
    launch_pdl1(norm_prep_kernel, dim3((rows.rows_max + 7) / 8), st, hidden, s.norm_eps, normed, nb.inv, rows, d);
    e->launches += 1;
  }
  GemmArgs g;
  g.row_scale = nb.inv;
  g.rows_max = rows.rows_max;
  g.rows_dev = rows.rows_dev;
  g.N = q + 2 * kv;
  g.K = d;
  g.epi = EPI_QKV;
  g.out_bf16 = qbuf;
  g.ld_bf16 = q;
  g.pos = rows.pos;
  g.rope = w->rope->csf.as<float2>();
  g.dh = s.d_head;
  g.q = q;
  g.kv = kv;
  g.ctx_k = ck;
  g.ctx_v = cv;
  g.commit = 1;
  g.cap_k = static_cast<__nv_bfloat16*>(cap_k);
  g.cap_v = static_cast<__nv_bfloat16*>(cap_v);
  gemm_bf16(e, normed, d, static_cast<const __nv_bfloat16*>(ly.w_qkv), g, hint);

  NormBufs tb = nb;
  if (tail >= 0 && commit && !rows.rows_dev && tail < rows.rows_max) {
    // only the last `tail` rows continue (their outputs are the only ones used)
    if (tail == 0) return;
    const int off = rows.rows_max - tail;
    hidden += (size_t)off * d;
    qbuf += (size_t)off * q;
    normed += (size_t)off * d;
    tb.inv += off;
    rows = Rows{tail, nullptr, rows.pos + off};
    rows.g1 = rows.g2 = 0;
    hint = tail;
  }

  AttnArgs a;
  a.q = qbuf;
  a.out = attn;
  a.pos = rows.pos;
  a.rows_max = rows.rows_max;
  a.rows_dev = rows.rows_dev;
  a.g1 = rows.g1;
  a.g2 = rows.g2;
  a.rows_hint = rows.rows_dev ? rows.hint : 0;
  a.H = s.num_heads;
  a.Hkv = s.num_kv_heads;
  a.dh = s.d_head;
  a.scale_log2 = 1.4426950408889634f / std::sqrt((float)s.d_head);
  a.probs = probs;
  a.key_lo = key_lo;
  a.key_n = key_n;
  attention_bf16(e, a, ck, cv, (int)ctx->size);

  GemmArgs o;
  o.rows_max = rows.rows_max;
  o.rows_dev = rows.rows_dev;
  o.N = d;
  o.K = q;
  o.epi = EPI_ADD;
  o.out_f32 = hidden;
  o.ld_out = d;
  o.split_flags = flags;
  o.norm_bf16 = normed;  // mlp RMSNorm fused: bf16 rows + 1/rms for the gate/up GEMM
  o.norm_part = tb.part;
  o.norm_inv = tb.inv;
  o.norm_cnt = tb.cnt;
  o.norm_eps = s.norm_eps;
  gemm_bf16(e, attn, q, static_cast<const __nv_bfloat16*>(ly.w_o), o, hint);

  GemmArgs gu;
  gu.row_scale = tb.inv;
  gu.rows_max = rows.rows_max;
  gu.rows_dev = rows.rows_dev;
  gu.N = 2 * ff;
  gu.K = d;
  gu.epi = EPI_SILU;
  gu.out_bf16 = act;
  gu.ld_bf16 = ff;
  gemm_bf16(e, normed, d, static_cast<const __nv_bfloat16*>(ly.w_gu), gu, hint);

  GemmArgs dn;
  dn.rows_max = rows.rows_max;
  dn.rows_dev = rows.rows_dev;
  dn.N = d;
  dn.K = ff;
  dn.epi = EPI_ADD;
  dn.out_f32 = hidden;
  dn.ld_out = d;
  dn.split_flags = flags;
  dn.norm_bf16 = normed;  // next layer's attention RMSNorm fused likewise
  dn.norm_part = tb.part;
  dn.norm_inv = tb.inv;
  dn.norm_cnt = tb.cnt;
  dn.norm_eps = s.norm_eps;
  gemm_bf16(e, act, ff, static_cast<const __nv_bfloat16*>(ly.w_down), dn, hint);

  if (!commit) {
    swap_row_kernel<<<1, 256, 0, st>>>(ck, cv, rows.pos, kv, save, 1);
    e->launches += 1;
  }
}

void last_row_logits_bf16(rk_engine* e, rk_weights* w, const float* hidden_row, float* logits) {
  Scratch& S = *e->scratch;
  const rk_model_spec& s = w->s;
  Rows one{1, nullptr, S.sub_positions.as<int>()};
  auto* normed = S.normed.as<__nv_bfloat16>();
  rmsnorm_bf16(e->stream, hidden_row, w->final_norm, s.norm_eps, normed, one, s.d_model);
  GemmArgs g;
  g.rows_max = 1;
  g.N = s.vocab_size;
  g.K = s.d_model;
  g.epi = EPI_F32;
  g.out_f32 = logits;
  g.ld_out = s.vocab_size;
  gemm_bf16(e, normed, s.d_model, static_cast<const __nv_bfloat16*>(w->head), g, 1);
  e->launches += 1;
}

void rows_logits_bf16(rk_engine* e, rk_weights* w, const float* hidden, Rows rows, float* logits) {
  Scratch& S = *e->scratch;
  const rk_model_spec& s = w->s;
  auto* normed = S.normed.as<__nv_bfloat16>();
  rmsnorm_bf16(e->stream, hidden, w->final_norm, s.norm_eps, normed, rows, s.d_model);
  GemmArgs g;
  g.rows_max = rows.rows_max;
  g.N = s.vocab_size;
  g.K = s.d_model;
  g.epi = EPI_F32;
  g.out_f32 = logits;
  g.ld_out = s.vocab_size;
  gemm_bf16(e, normed, s.d_model, static_cast<const __nv_bfloat16*>(w->head), g, rows.rows_max);
  e->launches += 1;
}

}  // namespace rk
