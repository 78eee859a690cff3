// layer_bf16.h -- argument blocks of the bf16 tensor-core kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"

namespace rk {

// EPI_PART: raw fp32 split-K partials to ws_part[split][row][N] (the residual
// add and fused RMSNorm then run in splitk_reduce_add_kernel)
enum GemmEpi { EPI_QKV = 0, EPI_ADD = 1, EPI_SILU = 2, EPI_F32 = 3, EPI_PART = 4 };

struct GemmArgs {
  int rows_max = 0;             // launch bound on M (tensor-map rows)
  const int* rows_dev = nullptr;  // live M on the device (sparse passes)
  int N = 0, K = 0;
  int epi = EPI_F32;
  int bn = 128, splits = 1;     // chosen by gemm_bf16 (splits re-chosen on the device for live rows)
  int sms = 148;
  int dbg = 0;                  // experiments (RK_GEMM_DBG): 1 = every k-block loads tile (0,0), 2 = no MMAs
  unsigned long long* trace = nullptr;  // debug: clock64 timeline of CTA 0 ([role 0..2][event < 512])
  int pair = 1;                 // 2: CTA-pair kernel (256-row tiles, cta_group::2), chosen by gemm_bf16
  // swap-AB (short static M): the weights are the MMA's M side (256 rows per
  // CTA pair), the M tokens its N side in nc chunks of tc (<= 256) columns
  int swap = 0, tc = 0, nc = 1;
  int m_hint = 0;  // live-row launches: m tiles of the host's row estimate (L2 warm-up of the first weight tiles)
  // tf32: operands are fp32 viewed as bf16 pairs (K, lda in bf16 units = 2x
  // the fp32 count), kind::tf32 MMAs (the 3xTF32 mode's K-concatenated
  // [hi|lo|hi] x [hi|hi|lo] operands); EPI_ADD / EPI_F32 only
  int tf32 = 0;
  int* split_flags = nullptr;   // non-null: a residual GEMM may run split-K (EPI_PART partials + reduce)
  // outputs
  float* out_f32 = nullptr;     // EPI_ADD / EPI_F32, row stride ld_out
  int ld_out = 0;
  __nv_bfloat16* out_bf16 = nullptr;  // EPI_SILU (act) / EPI_QKV (Q), row stride ld_bf16
  int ld_bf16 = 0;
  // EPI_QKV
  const int* pos = nullptr;
  const float2* rope = nullptr;  // [positions][dh/2] {cos, sin}
  int dh = 0, q = 0, kv = 0;
  __nv_bfloat16* ctx_k = nullptr;
  __nv_bfloat16* ctx_v = nullptr;
  int commit = 1;
  __nv_bfloat16* self_k = nullptr;
  __nv_bfloat16* self_v = nullptr;
  __nv_bfloat16* cap_k = nullptr;  // pre-RoPE K capture rows [M x kv]
  __nv_bfloat16* cap_v = nullptr;
  // Fused RMSNorm (rms_norm, tensor.cpp:109-119). Consumer side (QKV, SILU):
  // the accumulator row is scaled by row_scale[row] = 1/sqrt(mean(h^2)+eps)
  // before the epilogue (the norm gain is folded into the weights). Producer
  // side (ADD, final split): the new residual row is also written as bf16
  // (norm_bf16, row stride N) and its sum of squares per N tile goes to
  // norm_part[row][nt]; the last tile of each 32-row group to finish sums the
  // partials in tile order and writes norm_inv[row] (deterministic).
  const float* row_scale = nullptr;
  __nv_bfloat16* norm_bf16 = nullptr;
  float* norm_part = nullptr;   // [rows_max][64]
  float* norm_inv = nullptr;    // [rows_max]
  int* norm_cnt = nullptr;      // [m tiles * 4], zero-initialised, self-resetting
  float norm_eps = 1e-5f;
  float* ws_part = nullptr;  // EPI_PART workspace [splits][rows_max][N]
  // ensure_finite (tensor.cpp:58-64, after every matmul): any non-finite
  // product value sets status[0] (engine status flags, set by gemm_bf16);
  // the call then fails with RK_ERR_NONFINITE ("matmul: non-finite value")
  int* status = nullptr;
};
constexpr int kNormSlots = 64;  // max N tiles of a residual GEMM (d_model / BN)

// A: [rows_max x K] bf16 row-major with row stride lda; B: [N x K] bf16.
// rows_hint: expected live rows (tile-shape choice) when rows_dev is set.
bool pdl_enabled();  // programmatic dependent launch of the hot kernels (RK_PDL, default on)

void gemm_bf16(rk_engine* e, const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, GemmArgs p,
               int rows_hint = 0);
void make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
                    uint64_t row_stride_elems);

struct AttnArgs {
  const __nv_bfloat16* q = nullptr;  // [rows_max x H*dh]
  __nv_bfloat16* out = nullptr;      // [rows_max x H*dh]
  const int* pos = nullptr;          // ascending absolute positions
  int rows_max = 0;
  const int* rows_dev = nullptr;
  int g1 = 0, g2 = 0;                // row groups [0,g1) [g1,g2) [g2,live) (Rows::g1/g2)
  int H = 0, Hkv = 0, dh = 0;
  float scale_log2 = 0.f;            // log2(e) / sqrt(dh)
  // probability capture for influence (key window [key_lo, key_lo+key_n))
  float* probs = nullptr;
  int key_lo = 0, key_n = 0;
  // split-KV (set by attention_bf16): partial O / (m, l) workspace
  int splits = 1, tiles_per_split = 1 << 20;
  float* ws_o = nullptr;
  float* ws_ml = nullptr;
  int* tile_cnt = nullptr;    // [tiles x grid.y] zeroed, self-resetting: in-kernel split-KV merge
  // debug: clock64 timeline of the last CTA of head 0 ([role 0..2][step < 64][event < 8];
  // roles: softmax group 0, group 1, MMA issuer)
  unsigned long long* trace = nullptr;
  int coop = 0;  // split parts launched as one cluster: every part merges a slice (set by attention_bf16)
  int group = 1, rq = 128;  // GQA packing (set by attention_bf16): q heads per CTA, rows per head
  int rows_hint = 0;        // expected live rows (Rows::hint) for the split-KV plan
  int* status = nullptr;  // non-finite output flag (engine status[0], set by attention_bf16)
};
// ctx_k / ctx_v: the layer's [ctx_rows x kv] bf16 context rows.
void attention_bf16(rk_engine* e, const AttnArgs& a, const __nv_bfloat16* ctx_k, const __nv_bfloat16* ctx_v,
                    int ctx_rows);

}  // namespace rk
