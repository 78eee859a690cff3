/*
 * relaykv_b200_debug.h -- kernel-level test hooks (not part of the drop-in
 * boundary). Used by tests/test_gpu_kernels.py to check the bf16 tensor-core
 * GEMM and attention kernels in isolation against fp32 numpy references.
 */
#ifndef RELAYKV_B200_DEBUG_H_
#define RELAYKV_B200_DEBUG_H_
#include "relaykv_b200.h"
#ifdef __cplusplus
extern "C" {
#endif
/* C[M x N] (+)= A[M x K] . B[N x K]^T with bf16-rounded operands; epi 1 adds
 * into C (residual epilogue, deterministic split-K), 3 stores. live_rows <=
 * rows_max is passed through device memory like a sparse pass. */
/* RK_FP32_TC matmul: C (+)= A[M x K] . B[K x N] (reference layouts, fp32)
 * as 3xTF32 on tcgen05 (layer_tc.cu). */
int rk_debug_gemm_tc(rk_engine* e, const float* A, const float* B, float* C, int M, int N, int K, int add);
int rk_debug_gemm_bf16(rk_engine* e, const float* A, const float* B, float* C, int rows_max, int live_rows,
                       int N, int K, int epi);
/* out[M x H*dh] = causal attention of q rows at positions pos over ctx rows
 * [T x Hkv*dh]; bf16 operands. Rows [live, M) are not computed (live passed
 * through device memory like a sparse pass); row groups [0,g1) [g1,g2)
 * [g2,live) as in the fused schedule (0, 0 = one group). */
int rk_debug_attention_bf16(rk_engine* e, const float* q, const float* k, const float* v, const int32_t* pos,
                            int M, int live, int g1, int g2, int T, int H, int Hkv, int dh, float* out);
/* Device-resident timing (random operands, CUDA events): avg ms per call.
 * attention: band rows at positions T-M..T-1 over T context rows. */
int rk_debug_bench_attention(rk_engine* e, int M, int T, int H, int Hkv, int dh, int iters, float* ms);
/* Same, on a given row layout (positions, live count, row groups as in
 * rk_debug_attention_bf16): the c2 sparse / prefix+suffix passes. */
int rk_debug_bench_attention_rows(rk_engine* e, const int32_t* pos, int M, int live, int g1, int g2, int T, int H,
                                  int Hkv, int dh, int iters, float* ms);
/* clock64 timeline of one attention CTA (the last query tiles of head 0) on
 * the band case: out[3 roles][64 steps][8 events] (see attn_sm100.cu). */
int rk_debug_trace_attention(rk_engine* e, int M, int T, int H, int Hkv, int dh, unsigned long long* out);
int rk_debug_trace_attention_rows(rk_engine* e, const int32_t* pos, int M, int live, int g1, int g2, int T, int H,
                                  int Hkv, int dh, unsigned long long* out, int max_ctas, int* n);
int rk_debug_bench_gemm(rk_engine* e, int M, int N, int K, int epi, int iters, float* ms);
/* clock64 timeline of CTA 0 of one GEMM: out[3][512] (role 0: producer, per
 * k-block slot acquired; 1: MMA issuer, per k-block stage full; 2: epilogue,
 * per unit accumulator ready / drained). */
int rk_debug_trace_gemm(rk_engine* e, int M, int N, int K, int epi, unsigned long long* out);
/* K2b selection (select_relay) on host-given scores: sorted indices + tags,
 * count, dinfo = {exact threshold, min relative margin}. */
int rk_debug_select_relay(rk_engine* e, const double* s_dev, const float* influence, double infl_mean, int n,
                          double tau_dev, double tau_inf, int suffix_k, int32_t* sel_idx, uint32_t* sel_tags,
                          int32_t* count, double* dinfo);
/* top_k_by_score (selector.cpp:90-105) on the device (radix select):
   the `count` largest scores, ties by ascending index, as an ascending list */
int rk_debug_select_topk(rk_engine* e, const double* score, int n, int count, int32_t* sel_idx, int32_t* out_count);
/* K2 deviation scores at l_det (k::score_deviation) on host rows: elem 2 =
   bf16 bit patterns, 4 = fp32; rope = [base + n][dh / 2] {cos, sin} doubles */
int rk_debug_score_deviation(rk_engine* e, const void* ctx_v, const void* cache_v, const void* ctx_k,
                             const void* cache_kpre, int elem, int n, int heads, int dh, const double* rope, int base,
                             double* s_dev, double* s_key);
/* y[i] = device glibc_expf(x[i]) */
int rk_debug_expf(rk_engine* e, const float* x, float* y, uint64_t n);
/* Host only: the upload path's fp32 -> bf16 conversion on a `threads`-worker pool. */
int rk_debug_f32_to_bf16_host(const float* x, uint16_t* y, uint64_t n, int threads);
#ifdef __cplusplus
}
#endif
#endif
