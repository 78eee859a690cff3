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

#include <algorithm>

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

constexpr int kQ = 128;     // query rows per tile (one softmax warpgroup each)
constexpr int kKeys = 128;  // keys per tile
// query tiles per CTA (ping-pong softmax warpgroups over shared K/V tiles)
template <int DH> constexpr int qtiles() { return DH == 64 ? 2 : 1; }
template <int DH> constexpr int threads() { return 64 + qtiles<DH>() * 128; }  // TMA, MMA, softmax WGs

template <int DH>
struct ACfg {
  static constexpr int kQT = qtiles<DH>();
  static constexpr int Q_TILE = kQ * DH * 2;
  static constexpr int KV_BYTES = kKeys * DH * 2;  // one of K or V
  static constexpr int ONES_BYTES = kKeys * 128;   // 64-wide block of ones after V: P.[V|1] gives row sums
  static constexpr int STAGE_BYTES = 2 * KV_BYTES + ONES_BYTES;
  static constexpr int ON = DH + 16;               // PV MMA N: DH value columns + 16 ones columns
  static constexpr int P_BYTES = kQ * kKeys * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_KV = kQT * Q_TILE;
  static constexpr int OFF_P = OFF_KV + 2 * STAGE_BYTES;
  static constexpr int OFF_BAR = OFF_P + kQT * P_BYTES;
  static constexpr int SMEM = OFF_BAR + 512 + 1024;
  static constexpr uint32_t TMEM_COLS = 512;
  // TMEM columns: S_t at t*128, O_t (DH values + row-sum column) at 256 + t*128
  static constexpr uint32_t S_COL = 0, O_COL = 256;
};

template <int DH>
__global__ void __launch_bounds__(threads<DH>(), 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using C = ACfg<DH>;
  constexpr int kQT = C::kQT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;   // [2]
  uint64_t* kv_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;    // [kQT]
  uint64_t* s_free = bar + 7;    // [kQT]
  uint64_t* p_full = bar + 9;    // [kQT]
  uint64_t* o_full = bar + 11;   // [kQT]
  uint64_t* o_free = bar + 13;   // [kQT]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int M = a.rows_dev ? *a.rows_dev : a.rows_max;
  const int m0 = blockIdx.x * (kQ * kQT);
  if (m0 >= M) return;
  const int h = blockIdx.y;
  const int kvh = h / (a.H / a.Hkv);
  // key range: up to the largest position among the CTA's rows (rows need not
  // be sorted: the fused schedule packs prefix, suffix and segment rows)
  __shared__ int s_kmax;
  if (threadIdx.x == 0) s_kmax = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < kQ * kQT; i += blockDim.x)
    if (m0 + i < M) atomicMax(&s_kmax, a.pos[m0 + i]);
  __syncthreads();
  const int kmax = s_kmax;
  // split-KV: this CTA covers key tiles [j0, j0 + nk)
  const int j0 = blockIdx.z * a.tiles_per_split;
  const int nk = min(kmax / kKeys + 1 - j0, a.tiles_per_split);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (nk <= 0) {  // no keys for this split: an empty partial (m = -inf, l = 0)
    for (int i = threadIdx.x; i < kQ * kQT; i += blockDim.x)
      if (m0 + i < M) {
        float* ml = a.ws_ml + (((size_t)blockIdx.z * a.rows_max + m0 + i) * a.H + h) * 2;
        ml[0] = -INFINITY;
        ml[1] = 0.f;
      }
    return;
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int t = 0; t < kQT; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&s_free[t], 4);
      mbar_init(&p_full[t], 4);
      mbar_init(&o_full[t], 1);
      mbar_init(&o_free[t], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  for (int st = 0; st < 2; ++st) {  // the constant ones block of each K/V stage
    uint4* ones = reinterpret_cast<uint4*>(smem + C::OFF_KV + st * C::STAGE_BYTES + 2 * C::KV_BYTES);
    for (int i = threadIdx.x; i < C::ONES_BYTES / 16; i += blockDim.x) ones[i] = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr int DB = DH / 64;  // 64-wide swizzle blocks along d

  if (warp == 0) {
    if (elect_one()) {  // ------------------------------------------------ TMA
      uint8_t* sq = smem + C::OFF_Q;
      mbar_arrive_expect_tx(q_full, kQT * C::Q_TILE);
      for (int t = 0; t < kQT; ++t)
        for (int b = 0; b < DB; ++b)
          tma_load_2d(sq + t * C::Q_TILE + b * kQ * 128, &tmQ, q_full, h * DH + b * 64, m0 + t * kQ);
      for (int j = 0; j < nk; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        uint8_t* sk = smem + C::OFF_KV + st * C::STAGE_BYTES;
        uint8_t* sv = sk + C::KV_BYTES;
        mbar_arrive_expect_tx(&kv_full[st], 2 * C::KV_BYTES);
        for (int b = 0; b < DB; ++b) {
          tma_load_2d(sk + b * kKeys * 128, &tmK, &kv_full[st], kvh * DH + b * 64, (j0 + j) * kKeys);
          tma_load_2d(sv + b * kKeys * 128, &tmV, &kv_full[st], kvh * DH + b * 64, (j0 + j) * kKeys);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {  // ------------------------------------------------ MMA
      constexpr uint32_t idesc_s = idesc_bf16(kQ, kKeys);
      constexpr uint32_t idesc_o = idesc_bf16(kQ, C::ON, /*b_mn_major=*/true);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j, int t) {
        const int st = j & 1;
        mbar_wait(&s_free[t], (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t sq = smem_u32(smem + C::OFF_Q + t * C::Q_TILE);
        const uint32_t sk = smem_u32(smem + C::OFF_KV + st * C::STAGE_BYTES);
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          const uint32_t off = (k >> 2) * (kQ * 128) + (k & 3) * 32;
          const uint32_t offk = (k >> 2) * (kKeys * 128) + (k & 3) * 32;
          mma_bf16_ss(tmem + C::S_COL + t * 128, sdesc_sw128(sq + off, 16, 1024), sdesc_sw128(sk + offk, 16, 1024),
                      idesc_s, k > 0 ? 1u : 0u);
        }
        tc_commit(&s_full[t]);
      };
      auto issue_pv = [&](int j, int t) {
        const int st = j & 1;
        mbar_wait(&p_full[t], j & 1);
        mbar_wait(&o_free[t], (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t sp = smem_u32(smem + C::OFF_P + t * C::P_BYTES);
        const uint32_t sv = smem_u32(smem + C::OFF_KV + st * C::STAGE_BYTES + C::KV_BYTES);
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          const uint64_t ad = sdesc_sw128(sp + (k >> 2) * (kQ * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc_sw128(sv + k * 2048, kKeys * 128, 1024);
          mma_bf16_ss(tmem + C::O_COL + t * 128, ad, bd, idesc_o, k > 0 ? 1u : 0u);
        }
        tc_commit(&o_full[t]);
      };
      // ping-pong order: as soon as warpgroup t has turned S_t(j) into P_t(j),
      // issue its P.V and its next S, so one group's softmax overlaps the
      // other group's MMAs.
      mbar_wait(&kv_full[0], 0);
      for (int t = 0; t < kQT; ++t) issue_s(0, t);
      for (int j = 0; j < nk; ++j) {
        if (j + 1 < nk) mbar_wait(&kv_full[(j + 1) & 1], ((j + 1) >> 1) & 1);
        for (int t = 0; t < kQT; ++t) {
          if (j + 1 < nk) issue_s(j + 1, t);  // its softmax needs S first; O only later
          issue_pv(j, t);
        }
        tc_commit(&kv_empty[j & 1]);
      }
    }
  } else {  // ----------------------------------------- softmax warpgroups
    const int t = (warp - 2) / 4;        // query tile of this warpgroup
    const int quarter = warp & 3;        // TMEM lane quarter this warp may access
    const int rl = quarter * 32 + lane;  // row within the tile == TMEM lane
    const int row = m0 + t * kQ + rl;
    const bool valid = row < M;
    const int pos = valid ? a.pos[row] : kmax;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_col = tmem + lane_base + C::S_COL + t * 128;
    const uint32_t o_col = tmem + lane_base + C::O_COL + t * 128;
    uint8_t* sp = smem + C::OFF_P + t * C::P_BYTES;
    const float scale = a.scale_log2;
    float acc[DH];
#pragma unroll
    for (int d = 0; d < DH; ++d) acc[d] = 0.f;
    float m_run = -INFINITY, l_run = 0.f, corr_pending = 0.f;
    for (int j = 0; j < nk; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      const int kbase = (j0 + j) * kKeys;
      // warp-uniform: no causal mask anywhere in this tile for this warp's rows
      const bool full = __all_sync(0xffffffffu, kbase + kKeys - 1 <= pos);
      // pass 1: row max of the raw scores (scale > 0 commutes with max); two
      // 32-column TMEM loads per wait, four independent max chains
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int c = 0; c < kKeys; c += 64) {
        uint32_t r[32], q2[32];
        tmem_ld32(s_col + c, r);
        tmem_ld32(s_col + c + 32, q2);
        tmem_ld_wait();
        if (full) {
#pragma unroll
          for (int u = 0; u < 32; u += 4) {
            mx0 = fmaxf(mx0, fmaxf(__uint_as_float(r[u]), __uint_as_float(r[u + 1])));
            mx1 = fmaxf(mx1, fmaxf(__uint_as_float(r[u + 2]), __uint_as_float(r[u + 3])));
            mx2 = fmaxf(mx2, fmaxf(__uint_as_float(q2[u]), __uint_as_float(q2[u + 1])));
            mx3 = fmaxf(mx3, fmaxf(__uint_as_float(q2[u + 2]), __uint_as_float(q2[u + 3])));
          }
        } else {
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            if (kbase + c + u <= pos) mx0 = fmaxf(mx0, __uint_as_float(r[u]));
            if (kbase + c + 32 + u <= pos) mx1 = fmaxf(mx1, __uint_as_float(q2[u]));
          }
        }
      }
      const float mx = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      const float m_new = fmaxf(m_run, mx * scale);
      const float corr = fast_exp2(m_run - m_new);  // 0 on the first tile
      // PV_{j-1} done: P buffer free, O_{j-1} (and its row sum) ready
      if (j > 0) {
        mbar_wait(&o_full[t], (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < DH; c += 32) {
          uint32_t r[32];
          tmem_ld32(o_col + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int u = 0; u < 32; ++u) acc[c + u] = fmaf(acc[c + u], corr_pending, __uint_as_float(r[u]));
        }
        const uint32_t rs = tmem_ld1(o_col + DH);
        tmem_ld_wait();
        l_run = fmaf(l_run, corr_pending, __uint_as_float(rs));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free[t]);
      }
      // pass 2: P = exp2(s*scale - m_new) -> bf16, K-major SW128 (2 blocks of 64 keys)
      const float neg_m = -m_new;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        uint32_t r[64];
        tmem_ld32(s_col + b * 64, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        tmem_ld32(s_col + b * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
        tmem_ld_wait();
        if (!full) {
#pragma unroll
          for (int u = 0; u < 64; ++u)
            if (kbase + b * 64 + u > pos) r[u] = __float_as_uint(-INFINITY);
        }
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t pk[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i0 = ch * 8 + 2 * u;
            const float p0 = fast_exp2(fmaf(__uint_as_float(r[i0]), scale, neg_m));
            const float p1 = fast_exp2(fmaf(__uint_as_float(r[i0 + 1]), scale, neg_m));
            pk[u] = pack_bf16(p0, p1);
          }
          uint4* dst = reinterpret_cast<uint4*>(sp + b * (kQ * 128) + rl * 128 + ((ch ^ (rl & 7)) * 16));
          *dst = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[t]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
      m_run = m_new;
      corr_pending = corr;
    }
    mbar_wait(&o_full[t], (nk - 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < DH; c += 32) {
      uint32_t r[32];
      tmem_ld32(o_col + c, r);
      tmem_ld_wait();
#pragma unroll
      for (int u = 0; u < 32; ++u) acc[c + u] = fmaf(acc[c + u], corr_pending, __uint_as_float(r[u]));
    }
    {
      const uint32_t rs = tmem_ld1(o_col + DH);
      tmem_ld_wait();
      l_run = fmaf(l_run, corr_pending, __uint_as_float(rs));
    }
    if (valid && a.splits > 1) {
      const size_t pr = ((size_t)blockIdx.z * a.rows_max + row) * a.H + h;
      float4* dst = reinterpret_cast<float4*>(a.ws_o + pr * DH);
#pragma unroll
      for (int c = 0; c < DH; c += 4) dst[c / 4] = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
      a.ws_ml[pr * 2] = m_run;
      a.ws_ml[pr * 2 + 1] = l_run;
    } else if (valid) {
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

// Merge split-KV partials: out = sum_z 2^(m_z - m) acc_z / sum_z 2^(m_z - m) l_z.
// One warp per (row, head).
template <int DH>
__global__ void attn_combine_kernel(const AttnArgs a) {
  const int M = a.rows_dev ? *a.rows_dev : a.rows_max;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int row = gw / a.H, h = gw % a.H;
  if (row >= M) return;
  float m = -INFINITY;
  for (int z = 0; z < a.splits; ++z)
    m = fmaxf(m, a.ws_ml[(((size_t)z * a.rows_max + row) * a.H + h) * 2]);
  constexpr int PER = DH / 32;
  float o[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) o[i] = 0.f;
  float lsum = 0.f;
  for (int z = 0; z < a.splits; ++z) {
    const size_t pr = ((size_t)z * a.rows_max + row) * a.H + h;
    const float mz = a.ws_ml[pr * 2];
    if (mz == -INFINITY) continue;
    const float wz = fast_exp2(mz - m);
    lsum += wz * a.ws_ml[pr * 2 + 1];
#pragma unroll
    for (int i = 0; i < PER; ++i) o[i] += wz * a.ws_o[pr * DH + lane * PER + i];
  }
  const float inv = 1.f / lsum;
  __nv_bfloat16* dst = a.out + (size_t)row * (a.H * DH) + h * DH + lane * PER;
#pragma unroll
  for (int i = 0; i < PER; i += 2) *reinterpret_cast<uint32_t*>(dst + i) = pack_bf16(o[i] * inv, o[i + 1] * inv);
}

template <int DH>
void launch_attn(rk_engine* e, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                 const AttnArgs& a) {
  static bool attr = false;
  if (!attr) {
    RK_CUDA(cudaFuncSetAttribute(attn_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<DH>::SMEM));
    attr = true;
  }
  dim3 grid((a.rows_max + kQ * qtiles<DH>() - 1) / (kQ * qtiles<DH>()), a.H, a.splits);
  attn_kernel<DH><<<grid, threads<DH>(), ACfg<DH>::SMEM, e->stream>>>(tq, tk, tv, a);
  if (a.splits > 1) {
    const int warps = a.rows_max * a.H;
    attn_combine_kernel<DH><<<(warps + 7) / 8, 256, 0, e->stream>>>(a);
    e->launches += 1;
  }
}

}  // namespace

void attention_bf16(rk_engine* e, const AttnArgs& a_in, const __nv_bfloat16* ctx_k, const __nv_bfloat16* ctx_v,
                    int ctx_rows) {
  if (a_in.rows_max <= 0) return;
  AttnArgs a = a_in;
  // split-KV when the query tiles alone cannot fill the SMs
  const int qt = a.dh == 64 ? qtiles<64>() : qtiles<128>();
  const int q_tiles = (a.rows_max + kQ * qt - 1) / (kQ * qt);
  const int base = q_tiles * a.H;
  const int nk_max = (ctx_rows + kKeys - 1) / kKeys;
  a.splits = 1;
  a.tiles_per_split = nk_max > 0 ? nk_max : 1;
  if (base < 2 * e->sm_count && nk_max > 2) {
    int splits = std::min((2 * e->sm_count + base - 1) / base, (nk_max + 1) / 2);
    a.tiles_per_split = (nk_max + splits - 1) / splits;
    a.splits = (nk_max + a.tiles_per_split - 1) / a.tiles_per_split;
  }
  if (a.splits > 1) {
    Scratch& S = *e->scratch;
    const size_t per = (size_t)a.splits * a.rows_max * a.H;
    S.attn_ws.ensure(per * (a.dh + 2) * 4);
    a.ws_o = S.attn_ws.as<float>();
    a.ws_ml = a.ws_o + per * a.dh;
  }
  const int q = a.H * a.dh, kv = a.Hkv * a.dh;
  CUtensorMap tq, tk, tv;
  make_tmap_bf16(&tq, a.q, (uint64_t)a.rows_max, (uint64_t)q, kQ, (uint64_t)q);
  make_tmap_bf16(&tk, ctx_k, (uint64_t)ctx_rows, (uint64_t)kv, kKeys, (uint64_t)kv);
  make_tmap_bf16(&tv, ctx_v, (uint64_t)ctx_rows, (uint64_t)kv, kKeys, (uint64_t)kv);
  ProfScope ps(e, (e->prof && e->prof->on)
                      ? intern("attn_m" + std::to_string(a.rows_max) + (a.rows_dev ? "dyn" : "") + "_ctx" +
                               std::to_string(ctx_rows) + "_s" + std::to_string(a.splits))
                      : "attn",
               0, 0);
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
