// attn_sm100.cu -- K4: causal GQA attention for the recomputed rows over the
// mixed (reused + recomputed) KV context, on tcgen05 tensor cores.
//
// Reference semantics: attend_row (model.cpp:170-204) -- query row r at
// absolute position pos_r sees context keys 0..pos_r of its layer, softmax
// over scores scaled by 1/sqrt(d_head), kv head = h / (H / H_kv). Rows may be
// any ascending subset of positions (dense band or gathered sparse rows), so
// the causal limit is per row, by absolute position.
//
// One CTA = 128 query rows x one head, flash-style over 128-key tiles:
//   warp 0      TMA: Q once; K_j and V_j into a 2-stage ring
//   warp 1      TMEM alloc + MMA issue: S_j = Q K_j^T -> TMEM (double buffered);
//               O_j = P_j V_j -> TMEM (P from smem, V as MN-major B operand)
//   warps 2..5  one query row per thread: S_j from TMEM, scale + causal mask,
//               online softmax (exp2), P_j (bf16) into swizzled smem, then
//               acc = acc * corr_j + O_j in registers; finally O = acc / l.
#include <cuda.h>

#include "internal.h"
#include "layer_bf16.h"
#include "prof.h"
#include "sm100.cuh"

namespace rk {
namespace {

using namespace sm100;

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr int kQ = 128;     // query rows per CTA
constexpr int kKeys = 128;  // keys per tile
constexpr int kThreads = 192;

template <int DH>
struct ACfg {
  static constexpr int Q_BYTES = kQ * DH * 2;
  static constexpr int KV_BYTES = kKeys * DH * 2;       // one of K or V
  static constexpr int STAGE_BYTES = 2 * KV_BYTES;      // K + V
  static constexpr int P_BYTES = kQ * kKeys * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = Q_BYTES;
  static constexpr int OFF_P = OFF_KV + 2 * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  // pad to > half the SM's shared memory: one CTA per SM (it owns all of TMEM)
  static constexpr int SMEM_RAW = OFF_BAR + 256 + 1024;
  static constexpr int SMEM = SMEM_RAW < 120 * 1024 ? 120 * 1024 : SMEM_RAW;
  static constexpr uint32_t TMEM_COLS = 512;
  static constexpr uint32_t S_COL0 = 0, S_COL1 = 128, O_COL = 256;
};

template <int DH>
__global__ void __launch_bounds__(kThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using C = ACfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;   // [2]
  uint64_t* kv_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;    // [2]
  uint64_t* s_free = bar + 7;    // [2]
  uint64_t* p_full = bar + 9;
  uint64_t* o_full = bar + 10;
  uint64_t* o_free = bar + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 12);

  const int M = a.rows_dev ? *a.rows_dev : a.rows_max;
  const int m0 = blockIdx.x * kQ;
  if (m0 >= M) return;
  const int h = blockIdx.y;
  const int kvh = h / (a.H / a.Hkv);
  // key range: up to the largest position among the tile's rows (rows need
  // not be sorted: the fused schedule packs prefix, suffix and segment rows)
  __shared__ int s_kmax;
  if (threadIdx.x == 0) s_kmax = 0;
  __syncthreads();
  if (threadIdx.x < kQ && m0 + (int)threadIdx.x < M) atomicMax(&s_kmax, a.pos[m0 + threadIdx.x]);
  __syncthreads();
  const int kmax = s_kmax;
  const int nk = kmax / kKeys + 1;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_free, 4);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int DB = DH / 64;  // 64-wide swizzle blocks along d

  if (warp == 0) {
    if (elect_one()) {  // ------------------------------------------------ TMA
      uint8_t* sq = smem + C::OFF_Q;
      mbar_arrive_expect_tx(q_full, C::Q_BYTES);
      for (int b = 0; b < DB; ++b) tma_load_2d(sq + b * kQ * 128, &tmQ, q_full, h * DH + b * 64, m0);
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* sk = smem + C::OFF_KV + st * C::STAGE_BYTES;
        uint8_t* sv = sk + C::KV_BYTES;
        mbar_arrive_expect_tx(&kv_full[st], C::STAGE_BYTES);
        for (int b = 0; b < DB; ++b) {
          tma_load_2d(sk + b * kKeys * 128, &tmK, &kv_full[st], kvh * DH + b * 64, j * kKeys);
          tma_load_2d(sv + b * kKeys * 128, &tmV, &kv_full[st], kvh * DH + b * 64, j * kKeys);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {  // ------------------------------------------------ MMA
      constexpr uint32_t idesc_s = idesc_bf16(kQ, kKeys);
      constexpr uint32_t idesc_o = idesc_bf16(kQ, DH, /*b_mn_major=*/true);
      const uint32_t sq = smem_u32(smem + C::OFF_Q);
      const uint32_t sp = smem_u32(smem + C::OFF_P);
      mbar_wait(q_full, 0);
      auto issue_pv = [&](int j) {
        const int st = j & 1;
        mbar_wait(p_full, j & 1);
        mbar_wait(o_free, (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t sv = smem_u32(smem + C::OFF_KV + st * C::STAGE_BYTES + C::KV_BYTES);
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          const uint64_t ad = sdesc_sw128(sp + (k >> 2) * (kQ * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sv + k * 2048, kKeys * 128, 1024);
          mma_bf16_ss(tmem + C::O_COL, ad, bd, idesc_o, k > 0 ? 1u : 0u);
        }
        tc_commit(o_full);
        tc_commit(&kv_empty[st]);
      };
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_full[st], (j >> 1) & 1);
        mbar_wait(&s_free[st], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t sk = smem_u32(smem + C::OFF_KV + st * C::STAGE_BYTES);
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = (k >> 2) * (kQ * 128) + (k & 3) * 32;
          const uint32_t offk = (k >> 2) * (kKeys * 128) + (k & 3) * 32;
          mma_bf16_ss(tmem + (st ? C::S_COL1 : C::S_COL0), sdesc_sw128(sq + off, 16, 1024),
                      sdesc_sw128(sk + offk, 16, 1024), idesc_s, k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[st]);
        if (j > 0) issue_pv(j - 1);
      }
      issue_pv(nk - 1);
    }
  } else {  // ------------------------------------------------------ softmax
    const int quarter = warp & 3;
    const int rl = quarter * 32 + lane;  // row within the tile == TMEM lane
    const int row = m0 + rl;
    const bool valid = row < M;
    const int pos = valid ? a.pos[row] : kmax;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    uint8_t* sp = smem + C::OFF_P;
    float acc[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) acc[d] = 0.f;
    float m_run = -INFINITY, l_run = 0.f, corr_pending = 0.f;
    for (int j = 0; j < nk; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t s_col = tmem + lane_base + (st ? C::S_COL1 : C::S_COL0);
      const int kbase = j * kKeys;
      // pass 1: row max of the scaled, causally masked scores
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kKeys; c += 32) {
        uint32_t r[32];
        tmem_ld32(s_col + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (kbase + c + t <= pos) mx = fmaxf(mx, __uint_as_float(r[t]) * a.scale_log2);
      }
      const float m_new = fmaxf(m_run, mx);
      const float corr = fast_exp2(m_run - m_new);  // 0 on the first tile
      float lsum = 0.f;
      // PV_{j-1} done: the P buffer is free and O_{j-1} is ready
      if (j > 0) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < DH; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_base + C::O_COL + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) acc[c + t] = acc[c + t] * corr_pending + __uint_as_float(r[t]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free);
      }
      // pass 2: P_j = exp2(s - m_new) -> bf16, K-major SW128 (2 blocks of 64 keys)
#pragma unroll
      for (int c = 0; c < kKeys; c += 32) {
        uint32_t r[32];
        tmem_ld32(s_col + c, r);
        tmem_ld_wait();
        const int b = c / 64;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t pk[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int i0 = ch * 8 + 2 * t;
            const float v0 = (kbase + c + i0 <= pos) ? __uint_as_float(r[i0]) * a.scale_log2 : -INFINITY;
            const float v1 = (kbase + c + i0 + 1 <= pos) ? __uint_as_float(r[i0 + 1]) * a.scale_log2 : -INFINITY;
            const float p0 = fast_exp2(v0 - m_new), p1 = fast_exp2(v1 - m_new);
            lsum += p0 + p1;
            pk[t] = pack_bf16(p0, p1);
          }
          const int chunk = ((c % 64) / 8) + ch;
          uint4* dst = reinterpret_cast<uint4*>(sp + b * (kQ * 128) + rl * 128 + ((chunk ^ (rl & 7)) * 16));
          *dst = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[st]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      l_run = l_run * corr + lsum;
      m_run = m_new;
      corr_pending = corr;
    }
    mbar_wait(o_full, (nk - 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < DH; c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + C::O_COL + c, r);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 32; ++t) acc[c + t] = acc[c + t] * corr_pending + __uint_as_float(r[t]);
    }
    if (valid) {
      const float inv = 1.f / l_run;
      uint4* dst = reinterpret_cast<uint4*>(a.out + (size_t)row * (a.H * DH) + h * DH);
#pragma unroll
      for (int c = 0; c < DH; c += 8) {
        dst[c / 8] = make_uint4(pack_bf16(acc[c] * inv, acc[c + 1] * inv), pack_bf16(acc[c + 2] * inv, acc[c + 3] * inv),
                                pack_bf16(acc[c + 4] * inv, acc[c + 5] * inv), pack_bf16(acc[c + 6] * inv, acc[c + 7] * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// Normalised attention probabilities over a window of segment keys for the
// decode-time capture (influence, relay_cache.cpp:108-123): SIMT, fp32.
__global__ void attn_probs_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ ck,
                                  const AttnArgs a, float* __restrict__ probs) {
  extern __shared__ float sc[];
  const int r = blockIdx.x, h = blockIdx.y;
  const int M = a.rows_dev ? *a.rows_dev : a.rows_max;
  if (r >= M) return;
  const int kvh = h / (a.H / a.Hkv), kv = a.Hkv * a.dh;
  const int pos = a.pos[r];
  const __nv_bfloat16* qr = q + (size_t)r * a.H * a.dh + h * a.dh;
  __shared__ float red[32];
  float mx = -INFINITY;
  for (int j = threadIdx.x; j <= pos; j += blockDim.x) {
    const __nv_bfloat16* kj = ck + (size_t)j * kv + kvh * a.dh;
    float s = 0.f;
    for (int d = 0; d < a.dh; ++d) s += __bfloat162float(qr[d]) * __bfloat162float(kj[d]);
    s *= a.scale_log2;
    sc[j] = s;
    mx = fmaxf(mx, s);
  }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j <= pos; j += blockDim.x) {
    const float p = exp2f(sc[j] - mx);
    sc[j] = p;
    sum += p;
  }
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  sum = 0.f;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += red[w];
  float* pr = probs + ((size_t)r * a.H + h) * a.key_n;
  for (int jj = threadIdx.x; jj < a.key_n; jj += blockDim.x) {
    const int j = a.key_lo + jj;
    pr[jj] = j <= pos ? sc[j] / sum : 0.f;
  }
}

template <int DH>
void launch_attn(rk_engine* e, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                 const AttnArgs& a) {
  static bool attr = false;
  if (!attr) {
    RK_CUDA(cudaFuncSetAttribute(attn_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<DH>::SMEM));
    attr = true;
  }
  dim3 grid((a.rows_max + kQ - 1) / kQ, a.H);
  attn_kernel<DH><<<grid, kThreads, ACfg<DH>::SMEM, e->stream>>>(tq, tk, tv, a);
}

}  // namespace

void attention_bf16(rk_engine* e, const AttnArgs& a, const __nv_bfloat16* ctx_k, const __nv_bfloat16* ctx_v,
                    int ctx_rows) {
  if (a.rows_max <= 0) return;
  const int q = a.H * a.dh, kv = a.Hkv * a.dh;
  CUtensorMap tq, tk, tv;
  make_tmap_bf16(&tq, a.q, (uint64_t)a.rows_max, (uint64_t)q, kQ, (uint64_t)q);
  make_tmap_bf16(&tk, ctx_k, (uint64_t)ctx_rows, (uint64_t)kv, kKeys, (uint64_t)kv);
  make_tmap_bf16(&tv, ctx_v, (uint64_t)ctx_rows, (uint64_t)kv, kKeys, (uint64_t)kv);
  ProfScope ps(e, "attention_bf16_tcgen05", 0, 0);
  ps.rec.kind = 2;
  ps.rec.rows_dev = a.rows_dev;
  ps.rec.rows_max = a.rows_max;
  ps.rec.pos = a.pos;
  ps.rec.H = a.H;
  ps.rec.dh = a.dh;
  if (a.dh == 64) launch_attn<64>(e, tq, tk, tv, a);
  else if (a.dh == 128) launch_attn<128>(e, tq, tk, tv, a);
  else raise(RK_ERR_INVALID_ARGUMENT, "bf16 attention supports d_head 64 or 128");
  e->launches += 1;
  if (a.probs) {
    const size_t smem = (size_t)ctx_rows * 4;
    if (smem > 200 * 1024) raise(RK_ERR_INVALID_ARGUMENT, "capture: context too long for probability capture");
    static bool attr = false;
    if (!attr) {
      RK_CUDA(cudaFuncSetAttribute(attn_probs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    attn_probs_kernel<<<dim3(a.rows_max, a.H), 256, smem, e->stream>>>(a.q, ctx_k, a, a.probs);
    e->launches += 1;
  }
}

}  // namespace rk
