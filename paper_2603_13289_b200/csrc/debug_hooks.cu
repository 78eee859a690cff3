// debug_hooks.cu -- kernel-level test entry points (relaykv_b200_debug.h).
#include <string>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "glibc_expf.h"
#include "layer_bf16.h"
#include "layer_tc.h"
#include "relaykv_b200_debug.h"

using namespace rk;

namespace {
template <class F>
int guard(F&& f) {
  try {
    f();
    return RK_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return RK_ERR_RUNTIME;
  }
}
__global__ void expf_kernel(const float* x, float* y, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    y[i] = glibc_expf(x[i]);
}
DevBuf to_bf16(cudaStream_t st, const float* h, size_t n) {
  DevBuf f(n * 4), b(n * 2);
  RK_CUDA(cudaMemcpyAsync(f.p, h, n * 4, cudaMemcpyHostToDevice, st));
  k::f32_to_bf16(st, b.as<__nv_bfloat16>(), f.as<float>(), n);
  RK_CUDA(cudaStreamSynchronize(st));
  return b;
}
}  // namespace

extern "C" {

int rk_debug_gemm_tc(rk_engine* e, const float* A, const float* B, float* C, int M, int N, int K, int add) {
  return guard([&] {
    cudaStream_t st = e->stream;
    DevBuf a((size_t)M * K * 4), b((size_t)K * N * 4), bt((size_t)3 * K * N * 4), c((size_t)M * N * 4);
    RK_CUDA(cudaMemcpyAsync(a.p, A, (size_t)M * K * 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(b.p, B, (size_t)K * N * 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(c.p, C, (size_t)M * N * 4, cudaMemcpyHostToDevice, e->stream));
    tc::pack_weight(st, bt.as<float>(), b.as<float>(), N, 0, 1, K, N);
    Rows rows{M, nullptr, nullptr};
    tc::gemm(e, a.as<float>(), K, rows, bt.as<float>(), N, K, c.as<float>(), N, add != 0);
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(C, c.p, (size_t)M * N * 4, cudaMemcpyDeviceToHost));
  });
}

int rk_debug_gemm_bf16(rk_engine* e, const float* A, const float* B, float* C, int rows_max, int live_rows, int N,
                       int K, int epi) {
  return guard([&] {
    cudaStream_t st = e->stream;
    DevBuf a = to_bf16(st, A, (size_t)rows_max * K), b = to_bf16(st, B, (size_t)N * K);
    DevBuf c((size_t)rows_max * N * 4), live(4), flags(1 << 18);
    RK_CUDA(cudaMemcpyAsync(c.p, C, (size_t)rows_max * N * 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(live.p, &live_rows, 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemset(flags.p, 0, 1 << 18));
    GemmArgs g;
    g.rows_max = rows_max;
    g.rows_dev = live_rows == rows_max ? nullptr : live.as<int>();
    g.N = N;
    g.K = K;
    g.epi = epi;
    g.out_f32 = c.as<float>();
    g.ld_out = N;
    g.split_flags = flags.as<int>();
    gemm_bf16(e, a.as<__nv_bfloat16>(), K, b.as<__nv_bfloat16>(), g, live_rows);
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(C, c.p, (size_t)rows_max * N * 4, cudaMemcpyDeviceToHost));
  });
}

int rk_debug_attention_bf16(rk_engine* e, const float* q, const float* kk, const float* v, const int32_t* pos,
                            int M, int live, int g1, int g2, int T, int H, int Hkv, int dh, float* out) {
  return guard([&] {
    cudaStream_t st = e->stream;
    DevBuf qb = to_bf16(st, q, (size_t)M * H * dh), kb = to_bf16(st, kk, (size_t)T * Hkv * dh),
           vb = to_bf16(st, v, (size_t)T * Hkv * dh);
    DevBuf p(M * 4 + 16), o((size_t)M * H * dh * 2), of((size_t)M * H * dh * 4);
    RK_CUDA(cudaMemcpyAsync(p.p, pos, M * 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(p.as<int>() + M, &live, 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemsetAsync(o.p, 0, (size_t)M * H * dh * 2, st));
    AttnArgs a;
    a.q = qb.as<__nv_bfloat16>();
    a.out = o.as<__nv_bfloat16>();
    a.pos = p.as<int>();
    a.rows_max = M;
    a.rows_dev = live < M ? p.as<int>() + M : nullptr;
    a.g1 = g1;
    a.g2 = g2;
    a.H = H;
    a.Hkv = Hkv;
    a.dh = dh;
    a.scale_log2 = 1.4426950408889634f / std::sqrt((float)dh);
    attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);
    k::bf16_to_f32(st, of.as<float>(), o.as<__nv_bfloat16>(), (size_t)M * H * dh);
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(out, of.p, (size_t)M * H * dh * 4, cudaMemcpyDeviceToHost));
  });
}

// Device-resident timing of one kernel shape (random bf16 operands), avg ms per call.
int rk_debug_bench_attention(rk_engine* e, int M, int T, int H, int Hkv, int dh, int iters, float* ms) {
  return guard([&] {
    cudaStream_t st = e->stream;
    const size_t nq = (size_t)M * H * dh, nk = (size_t)T * Hkv * dh;
    DevBuf f((nq > nk ? nq : nk) * 4), qb(nq * 2), kb(nk * 2), vb(nk * 2), o(nq * 2), p(M * 4);
    k::init_uniform(st, f.as<float>(), nq, 11, 1.0f);
    k::f32_to_bf16(st, qb.as<__nv_bfloat16>(), f.as<float>(), nq);
    k::init_uniform(st, f.as<float>(), nk, 12, 1.0f);
    k::f32_to_bf16(st, kb.as<__nv_bfloat16>(), f.as<float>(), nk);
    k::init_uniform(st, f.as<float>(), nk, 13, 1.0f);
    k::f32_to_bf16(st, vb.as<__nv_bfloat16>(), f.as<float>(), nk);
    k::iota_positions(st, p.as<int>(), M, T - M);
    AttnArgs a;
    a.q = qb.as<__nv_bfloat16>();
    a.out = o.as<__nv_bfloat16>();
    a.pos = p.as<int>();
    a.rows_max = M;
    a.H = H;
    a.Hkv = Hkv;
    a.dh = dh;
    a.scale_log2 = 1.4426950408889634f / std::sqrt((float)dh);
    attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);
    cudaEvent_t e0, e1;
    RK_CUDA(cudaEventCreate(&e0));
    RK_CUDA(cudaEventCreate(&e1));
    RK_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);
    RK_CUDA(cudaEventRecord(e1, st));
    RK_CUDA(cudaEventSynchronize(e1));
    RK_CUDA(cudaEventElapsedTime(ms, e0, e1));
    *ms /= iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    RK_CUDA(cudaGetLastError());
  });
}

int rk_debug_bench_attention_rows(rk_engine* e, const int32_t* pos, int M, int live, int g1, int g2, int T, int H,
                                  int Hkv, int dh, int iters, float* ms) {
  return guard([&] {
    cudaStream_t st = e->stream;
    const size_t nq = (size_t)M * H * dh, nk = (size_t)T * Hkv * dh;
    DevBuf f((nq > nk ? nq : nk) * 4), qb(nq * 2), kb(nk * 2), vb(nk * 2), o(nq * 2), p(M * 4 + 16);
    k::init_uniform(st, f.as<float>(), nq, 11, 1.0f);
    k::f32_to_bf16(st, qb.as<__nv_bfloat16>(), f.as<float>(), nq);
    k::init_uniform(st, f.as<float>(), nk, 12, 1.0f);
    k::f32_to_bf16(st, kb.as<__nv_bfloat16>(), f.as<float>(), nk);
    k::init_uniform(st, f.as<float>(), nk, 13, 1.0f);
    k::f32_to_bf16(st, vb.as<__nv_bfloat16>(), f.as<float>(), nk);
    RK_CUDA(cudaMemcpyAsync(p.p, pos, M * 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(p.as<int>() + M, &live, 4, cudaMemcpyHostToDevice, e->stream));
    AttnArgs a;
    a.q = qb.as<__nv_bfloat16>();
    a.out = o.as<__nv_bfloat16>();
    a.pos = p.as<int>();
    a.rows_max = M;
    a.rows_dev = live < M ? p.as<int>() + M : nullptr;
    a.g1 = g1;
    a.g2 = g2;
    a.H = H;
    a.Hkv = Hkv;
    a.dh = dh;
    a.scale_log2 = 1.4426950408889634f / std::sqrt((float)dh);
    attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);
    cudaEvent_t e0, e1;
    RK_CUDA(cudaEventCreate(&e0));
    RK_CUDA(cudaEventCreate(&e1));
    RK_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);
    RK_CUDA(cudaEventRecord(e1, st));
    RK_CUDA(cudaEventSynchronize(e1));
    RK_CUDA(cudaEventElapsedTime(ms, e0, e1));
    *ms /= iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    RK_CUDA(cudaGetLastError());
  });
}

// Per-CTA global-timer spans of one attention launch over a rows layout (as
// rk_debug_bench_attention_rows): out[4 * cta] = {entry, after the dependency
// wait, end, nk | partial << 8 | parts << 16 | rows << 32}; CTAs that exit
// early (dead tiles / parts) stay 0; out[0, 1536) holds CTA (0,0,0)'s event slots
// (rk_debug_trace_attention layout) first. out must hold 1536 + 4 * max_ctas.
int rk_debug_trace_attention_rows(rk_engine* e, const int32_t* pos, int M, int live, int g1, int g2, int T, int H,
                                  int Hkv, int dh, unsigned long long* out, int max_ctas, int* n) {
  return guard([&] {
    cudaStream_t st = e->stream;
    const size_t nq = (size_t)M * H * dh, nk = (size_t)T * Hkv * dh;
    DevBuf f((nq > nk ? nq : nk) * 4), qb(nq * 2), kb(nk * 2), vb(nk * 2), o(nq * 2), p(M * 4 + 16),
        tr((1536 + 4 * (size_t)max_ctas) * 8);
    k::init_uniform(st, f.as<float>(), nq, 11, 1.0f);
    k::f32_to_bf16(st, qb.as<__nv_bfloat16>(), f.as<float>(), nq);
    k::init_uniform(st, f.as<float>(), nk, 12, 1.0f);
    k::f32_to_bf16(st, kb.as<__nv_bfloat16>(), f.as<float>(), nk);
    k::init_uniform(st, f.as<float>(), nk, 13, 1.0f);
    k::f32_to_bf16(st, vb.as<__nv_bfloat16>(), f.as<float>(), nk);
    RK_CUDA(cudaMemcpyAsync(p.p, pos, M * 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(p.as<int>() + M, &live, 4, cudaMemcpyHostToDevice, e->stream));
    AttnArgs a;
    a.q = qb.as<__nv_bfloat16>();
    a.out = o.as<__nv_bfloat16>();
    a.pos = p.as<int>();
    a.rows_max = M;
    a.rows_dev = live < M ? p.as<int>() + M : nullptr;
    a.g1 = g1;
    a.g2 = g2;
    a.H = H;
    a.Hkv = Hkv;
    a.dh = dh;
    a.scale_log2 = 1.4426950408889634f / std::sqrt((float)dh);
    attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);  // warm
    RK_CUDA(cudaMemsetAsync(tr.p, 0, tr.bytes, st));
    RK_CUDA(cudaStreamSynchronize(st));
    a.trace = tr.as<unsigned long long>();
    attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(out, tr.p, tr.bytes, cudaMemcpyDeviceToHost));  // event slots, then the CTA spans
    *n = max_ctas;
  });
}

int rk_debug_trace_attention(rk_engine* e, int M, int T, int H, int Hkv, int dh, unsigned long long* out) {
  return guard([&] {
    cudaStream_t st = e->stream;
    const size_t nq = (size_t)M * H * dh, nk = (size_t)T * Hkv * dh;
    DevBuf f((nq > nk ? nq : nk) * 4), qb(nq * 2), kb(nk * 2), vb(nk * 2), o(nq * 2), p(M * 4), tr(3 * 64 * 8 * 8);
    k::init_uniform(st, f.as<float>(), nq, 11, 1.0f);
    k::f32_to_bf16(st, qb.as<__nv_bfloat16>(), f.as<float>(), nq);
    k::init_uniform(st, f.as<float>(), nk, 12, 1.0f);
    k::f32_to_bf16(st, kb.as<__nv_bfloat16>(), f.as<float>(), nk);
    k::init_uniform(st, f.as<float>(), nk, 13, 1.0f);
    k::f32_to_bf16(st, vb.as<__nv_bfloat16>(), f.as<float>(), nk);
    k::iota_positions(st, p.as<int>(), M, T - M);
    RK_CUDA(cudaMemsetAsync(tr.p, 0, tr.bytes, st));
    AttnArgs a;
    a.q = qb.as<__nv_bfloat16>();
    a.out = o.as<__nv_bfloat16>();
    a.pos = p.as<int>();
    a.rows_max = M;
    a.H = H;
    a.Hkv = Hkv;
    a.dh = dh;
    a.scale_log2 = 1.4426950408889634f / std::sqrt((float)dh);
    attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);  // warm
    a.trace = tr.as<unsigned long long>();
    attention_bf16(e, a, kb.as<__nv_bfloat16>(), vb.as<__nv_bfloat16>(), T);
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(out, tr.p, tr.bytes, cudaMemcpyDeviceToHost));
  });
}

int rk_debug_bench_gemm(rk_engine* e, int M, int N, int K, int epi, int iters, float* ms) {
  return guard([&] {
    cudaStream_t st = e->stream;
    // the weights rotate over enough copies (>= 256 MB) that every iteration
    // streams them from HBM, as each layer's weights are in a relay step
    const size_t wbytes = (size_t)N * K * 2;
    int copies = (int)std::min<size_t>(16, std::max<size_t>(1, ((size_t)256 << 20) / wbytes + 1));
    if (const char* c = std::getenv("RK_BENCH_COPIES")) copies = std::max(1, std::atoi(c));  // 1: L2-resident weights
    DevBuf f((size_t)(M > N ? M : N) * K * 4), a((size_t)M * K * 2), b(wbytes * copies), c((size_t)M * N * 4),
        flags(1 << 18);
    k::init_uniform(st, f.as<float>(), (size_t)M * K, 21, 1.0f);
    k::f32_to_bf16(st, a.as<__nv_bfloat16>(), f.as<float>(), (size_t)M * K);
    k::init_uniform(st, f.as<float>(), (size_t)N * K, 22, 0.02f);
    for (int i = 0; i < copies; ++i)
      k::f32_to_bf16(st, b.as<__nv_bfloat16>() + (size_t)i * N * K, f.as<float>(), (size_t)N * K);
    RK_CUDA(cudaMemsetAsync(c.p, 0, c.bytes, st));
    RK_CUDA(cudaMemsetAsync(flags.p, 0, flags.bytes, st));
    GemmArgs g;
    g.rows_max = M;
    g.N = N;
    g.K = K;
    g.epi = epi;
    g.out_f32 = c.as<float>();
    g.ld_out = N;
    g.out_bf16 = reinterpret_cast<__nv_bfloat16*>(c.p);
    g.ld_bf16 = N / 2;
    g.split_flags = flags.as<int>();
    // RK_BENCH_NORM=1 (residual epi): the fused RMSNorm producer of the layer
    // pass (bf16 row copy, per-tile sums of squares, last tile writes 1/rms)
    DevBuf nbf, npart, ninv, ncnt;
    if (epi == EPI_ADD && std::getenv("RK_BENCH_NORM")) {
      nbf.alloc((size_t)M * N * 2);
      npart.alloc((size_t)M * kNormSlots * 4 + 256);
      ninv.alloc((size_t)M * 4 + 256);
      ncnt.alloc(((size_t)(M + 127) / 128 * 8 + 64) * 4);
      RK_CUDA(cudaMemsetAsync(ncnt.p, 0, ncnt.bytes, st));
      g.norm_bf16 = nbf.as<__nv_bfloat16>();
      g.norm_part = npart.as<float>();
      g.norm_inv = ninv.as<float>();
      g.norm_cnt = ncnt.as<int>();
    }
    // epi 0: the real QKV epilogue (c2-like heads: d_head 64, kv 512): 1/rms row
    // scale, RoPE on Q/K, Q as bf16, K/V scattered into a context at positions 0..M-1
    DevBuf pos, ctxk, ctxv, rs;
    if (epi == EPI_QKV) {
      const int dh = 64, kv = 512;
      pos.alloc((size_t)M * 4);
      k::iota_positions(st, pos.as<int>(), M, 0);
      ctxk.alloc((size_t)M * kv * 2);
      ctxv.alloc((size_t)M * kv * 2);
      rs.alloc((size_t)M * 4);
      k::fill(st, rs.as<float>(), M, 1.0f);
      g.pos = pos.as<int>();
      g.rope = rope_table(e, 10000.0f, dh, (uint64_t)M)->csf.as<float2>();
      g.dh = dh;
      g.kv = kv;
      g.q = N - 2 * kv;
      g.ctx_k = ctxk.as<__nv_bfloat16>();
      g.ctx_v = ctxv.as<__nv_bfloat16>();
      g.commit = 1;
      g.row_scale = rs.as<float>();
      g.ld_bf16 = g.q;
    }
    gemm_bf16(e, a.as<__nv_bfloat16>(), K, b.as<__nv_bfloat16>(), g, M);
    cudaEvent_t e0, e1;
    RK_CUDA(cudaEventCreate(&e0));
    RK_CUDA(cudaEventCreate(&e1));
    RK_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i)
      gemm_bf16(e, a.as<__nv_bfloat16>(), K, b.as<__nv_bfloat16>() + (size_t)(i % copies) * N * K, g, M);
    RK_CUDA(cudaEventRecord(e1, st));
    RK_CUDA(cudaEventSynchronize(e1));
    RK_CUDA(cudaEventElapsedTime(ms, e0, e1));
    *ms /= iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    RK_CUDA(cudaGetLastError());
  });
}

int rk_debug_trace_gemm(rk_engine* e, int M, int N, int K, int epi, unsigned long long* out) {
  return guard([&] {
    cudaStream_t st = e->stream;
    DevBuf f((size_t)(M > N ? M : N) * K * 4), a((size_t)M * K * 2), b((size_t)N * K * 2), c((size_t)M * N * 4),
        flags(1 << 18), tr(3 * 512 * 8);
    k::init_uniform(st, f.as<float>(), (size_t)M * K, 21, 1.0f);
    k::f32_to_bf16(st, a.as<__nv_bfloat16>(), f.as<float>(), (size_t)M * K);
    k::init_uniform(st, f.as<float>(), (size_t)N * K, 22, 0.02f);
    k::f32_to_bf16(st, b.as<__nv_bfloat16>(), f.as<float>(), (size_t)N * K);
    RK_CUDA(cudaMemsetAsync(c.p, 0, c.bytes, st));
    RK_CUDA(cudaMemsetAsync(flags.p, 0, flags.bytes, st));
    RK_CUDA(cudaMemsetAsync(tr.p, 0, tr.bytes, st));
    GemmArgs g;
    g.rows_max = M;
    g.N = N;
    g.K = K;
    g.epi = epi;
    g.out_f32 = c.as<float>();
    g.ld_out = N;
    g.out_bf16 = reinterpret_cast<__nv_bfloat16*>(c.p);
    g.ld_bf16 = N / 2;
    g.split_flags = flags.as<int>();
    DevBuf nbf, npart, ninv, ncnt;
    if (epi == EPI_ADD && std::getenv("RK_BENCH_NORM")) {  // the layer pass's fused RMSNorm producer
      nbf.alloc((size_t)M * N * 2);
      npart.alloc((size_t)M * kNormSlots * 4 + 256);
      ninv.alloc((size_t)M * 4 + 256);
      ncnt.alloc(((size_t)(M + 127) / 128 * 8 + 64) * 4);
      RK_CUDA(cudaMemsetAsync(ncnt.p, 0, ncnt.bytes, st));
      g.norm_bf16 = nbf.as<__nv_bfloat16>();
      g.norm_part = npart.as<float>();
      g.norm_inv = ninv.as<float>();
      g.norm_cnt = ncnt.as<int>();
    }
    gemm_bf16(e, a.as<__nv_bfloat16>(), K, b.as<__nv_bfloat16>(), g, M);  // warm
    g.trace = tr.as<unsigned long long>();
    gemm_bf16(e, a.as<__nv_bfloat16>(), K, b.as<__nv_bfloat16>(), g, M);
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(out, tr.p, tr.bytes, cudaMemcpyDeviceToHost));
  });
}

// K2 deviation scores (k::score_deviation) on host rows: elem 2 = bf16 rows
// (uint16 bit patterns), 4 = fp32; rope = [base + n][dh / 2] {cos, sin} doubles.
int rk_debug_score_deviation(rk_engine* e, const void* ctx_v, const void* cache_v, const void* ctx_k,
                             const void* cache_kpre, int elem, int n, int heads, int dh, const double* rope, int base,
                             double* s_dev, double* s_key) {
  return guard([&] {
    cudaStream_t st = e->stream;
    const size_t bytes = (size_t)n * heads * dh * elem, rbytes = (size_t)(base + n) * dh / 2 * 16;
    DevBuf a(bytes), b(bytes), c(bytes), d(bytes), r(rbytes), sd((size_t)n * 8), sk((size_t)n * 8);
    RK_CUDA(cudaMemcpyAsync(a.p, ctx_v, bytes, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(b.p, cache_v, bytes, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(c.p, ctx_k, bytes, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(d.p, cache_kpre, bytes, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(r.p, rope, rbytes, cudaMemcpyHostToDevice, e->stream));
    k::score_deviation(st, a.p, b.p, c.p, d.p, (size_t)elem, n, heads * dh, heads, dh, r.as<double2>(), base,
                       sd.as<double>(), sk.as<double>());
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(s_dev, sd.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(s_key, sk.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
  });
}

int rk_debug_select_topk(rk_engine* e, const double* score, int n, int count, int32_t* sel_idx, int32_t* out_count) {
  return guard([&] {
    cudaStream_t st = e->stream;
    DevBuf sc((size_t)n * 8 + 8), idx((size_t)n * 4 + 4), tags((size_t)2 * n * 4 + 8), info(64);
    RK_CUDA(cudaMemcpyAsync(sc.p, score, (size_t)n * 8, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemset(info.p, 0, 64));
    k::select_topk(st, sc.as<double>(), n, count, idx.as<int>(), tags.as<uint32_t>(), info.as<int>());
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(out_count, info.p, 4, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(sel_idx, idx.p, (size_t)*out_count * 4, cudaMemcpyDeviceToHost));
  });
}

int rk_debug_select_relay(rk_engine* e, const double* s_dev, const float* influence, double infl_mean, int n,
                          double tau_dev, double tau_inf, int suffix_k, int32_t* sel_idx, uint32_t* sel_tags,
                          int32_t* count, double* dinfo) {
  return guard([&] {
    cudaStream_t st = e->stream;
    DevBuf sd(n * 8), inf(n * 4), im(8), idx(n * 4), tags(2 * n * 4), info(64), di(64);
    RK_CUDA(cudaMemcpyAsync(sd.p, s_dev, n * 8, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(inf.p, influence, n * 4, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemcpyAsync(im.p, &infl_mean, 8, cudaMemcpyHostToDevice, e->stream));
    RK_CUDA(cudaMemset(info.p, 0, 64));
    k::select_relay(st, sd.as<double>(), inf.as<float>(), im.as<double>(), n, tau_dev, tau_inf, suffix_k,
                    idx.as<int>(), tags.as<uint32_t>(), info.as<int>(), di.as<double>(), e->side, e->side_fork,
                    e->side_join);
    RK_CUDA(cudaStreamSynchronize(st));
    RK_CUDA(cudaStreamSynchronize(e->side));
    RK_CUDA(cudaGetLastError());
    RK_CUDA(cudaMemcpy(count, info.p, 4, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(sel_idx, idx.p, (size_t)*count * 4, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(sel_tags, tags.p, (size_t)*count * 4, cudaMemcpyDeviceToHost));
    RK_CUDA(cudaMemcpy(dinfo, di.p, 16, cudaMemcpyDeviceToHost));
  });
}

int rk_debug_expf(rk_engine* e, const float* x, float* y, uint64_t n) {
  return guard([&] {
    DevBuf dx(n * 4), dy(n * 4);
    RK_CUDA(cudaMemcpyAsync(dx.p, x, n * 4, cudaMemcpyHostToDevice, e->stream));
    expf_kernel<<<1024, 256, 0, e->stream>>>(dx.as<float>(), dy.as<float>(), n);
    RK_CUDA(cudaStreamSynchronize(e->stream));
    RK_CUDA(cudaMemcpy(y, dy.p, n * 4, cudaMemcpyDeviceToHost));
  });
}

int rk_debug_f32_to_bf16_host(const float* x, uint16_t* y, uint64_t n, int threads) {
  return guard([&] {
    HostPool pool(threads);
    pool.parallel_for(n, 4096, [&](size_t b, size_t e) { f32_to_bf16_host(x + b, y + b, e - b); });
  });
}

}  // extern "C"
