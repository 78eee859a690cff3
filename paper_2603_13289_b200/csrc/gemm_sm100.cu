// gemm_sm100.cu -- K3: the recompute GEMMs on 5th-gen tensor cores.
//
// D[M x N] = A[M x K] . B[N x K]^T, bf16 operands (both K-major), fp32
// accumulation in TMEM. One persistent CTA per SM, warp-specialized:
//   warp 0      TMA producer (one elected lane): A/B k-blocks into a
//               STAGES-deep shared-memory ring (SWIZZLE_128B), mbarrier-tracked
//   warp 1      TMEM allocator + MMA issuer (one elected lane):
//               tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16
//   warps 2..5  epilogue: tcgen05.ld 32x32b rows -> fused epilogue -> global
// TMEM holds two BN-column accumulators so the epilogue of tile i overlaps
// the MMAs of tile i+1. Rows of A beyond the live row count (read from device
// memory for sparse passes) are computed but never stored.
//
// Fused epilogues (the reference computes these as separate loops over the
// matmul outputs, model.cpp:246-280 / 211-233):
//   EPI_QKV   RoPE on Q and K (adjacent pairs, tensor.cpp:134-142), Q -> bf16
//             buffer, K/V rows scattered into the context at each row's
//             absolute position (model.cpp:266-269), optional capture of
//             pre-RoPE K and V (decode-time capture, model.cpp:254-257)
//   EPI_ADD   hidden += D (residual); split-K partials are added in split
//             order (deterministic) via per-tile flags
//   EPI_SILU  interleaved (gate, up) columns -> bf16 silu(g)*u (model.cpp:226)
//   EPI_F32   plain fp32 store (logits)
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "internal.h"
#include "layer_bf16.h"
#include "prof.h"
#include "sm100.cuh"

namespace rk {
namespace {

using namespace sm100;

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int kThreads = 192;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = BN * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  // per epilogue warp: a 32x32 fp32 staging tile for the coalesced residual epilogue
  static constexpr int EPI_STAGE = 4 * 32 * 32 * 4;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_STAGE;
};

struct Units {
  int num_m, num_n, splits, kb_total, kb_per;
  int total;
};

__device__ __forceinline__ Units units_of(const GemmArgs& p) {
  Units u;
  const int M = p.rows_dev ? *p.rows_dev : p.rows_max;
  u.num_m = (M + kBM - 1) / kBM;
  u.num_n = p.N / p.bn;
  // live row count known only on the device: pick split-K here (grid = all SMs)
  u.splits = p.splits;
  u.kb_total = p.K / kBK;
  u.kb_per = (u.kb_total + u.splits - 1) / u.splits;
  u.total = u.num_m * u.num_n * u.splits;
  return u;
}

// unit -> (m tile, n tile, split); split fastest so the splits of one tile run
// concurrently on different CTAs, then m so CTAs share B tiles in L2.
__device__ __forceinline__ void decode_unit(const Units& u, int unit, int& mt, int& nt, int& s) {
  s = unit % u.splits;
  const int tile = unit / u.splits;
  mt = tile % u.num_m;
  nt = tile / u.num_m;
}

// One accumulator's worth of work: tile (mt, nt), k-blocks [kb0, kb1); s is
// the split index (split-K) or the CTA-local slot (stream-K).
struct Work {
  int mt, nt, s, kb0, kb1;
};

// Stream-K: the tile-major k-block space (tile t = mt + nt*num_m) is cut into
// gridDim.x equal contiguous ranges; CTA g takes range g, touching at most
// kSkSlots tiles (the host uses it only with at most 2 tiles per CTA, counting
// the largest live row count).
constexpr int kSkSlots = 4;
__device__ __forceinline__ long long sk_lo(const Units& u, int g, int G) {
  return (long long)u.num_m * u.num_n * u.kb_total * g / G;
}

// k-th work item of this CTA; false when the CTA is done.
__device__ __forceinline__ bool get_work(const Units& U, bool streamk, int k, Work& w) {
  if (!streamk) {
    const int unit = blockIdx.x + k * gridDim.x;
    if (unit >= U.total) return false;
    decode_unit(U, unit, w.mt, w.nt, w.s);
    w.kb0 = w.s * U.kb_per;
    w.kb1 = min(U.kb_total, w.kb0 + U.kb_per);
    return true;
  }
  const long long lo = sk_lo(U, blockIdx.x, gridDim.x), hi = sk_lo(U, blockIdx.x + 1, gridDim.x);
  const long long t = lo / U.kb_total + k, tlo = t * U.kb_total;
  if (tlo >= hi || lo >= hi) return false;
  w.kb0 = (int)((lo > tlo ? lo : tlo) - tlo);
  w.kb1 = (int)((hi < tlo + U.kb_total ? hi : tlo + U.kb_total) - tlo);
  w.mt = (int)(t % U.num_m);
  w.nt = (int)(t / U.num_m);
  w.s = k;
  return true;
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& p, int row, int col, const uint32_t (&r)[32],
                                               float rs, int split = 0) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * rs;
  if constexpr (EPI == EPI_F32 || EPI == EPI_PART) {
    float* base = EPI != EPI_PART ? p.out_f32 + (size_t)row * p.ld_out + col
                  : p.streamk ? p.ws_part + (((size_t)blockIdx.x * kSkSlots + split) * kBM + row % kBM) * p.bn + col % p.bn
                              : p.ws_part + ((size_t)split * p.rows_max + row) * p.N + col;
    float4* dst = reinterpret_cast<float4*>(base);
#pragma unroll
    for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  } else if constexpr (EPI == EPI_ADD) {
    float4* dst = reinterpret_cast<float4*>(p.out_f32 + (size_t)row * p.ld_out + col);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 h = dst[j];
      h.x += v[4 * j]; h.y += v[4 * j + 1]; h.z += v[4 * j + 2]; h.w += v[4 * j + 3];
      dst[j] = h;
    }
  } else if constexpr (EPI == EPI_SILU) {
    uint32_t packed[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float g0 = v[4 * j], u0 = v[4 * j + 1], g1 = v[4 * j + 2], u1 = v[4 * j + 3];
      const float a0 = g0 / (1.0f + __expf(-g0)) * u0;
      const float a1 = g1 / (1.0f + __expf(-g1)) * u1;
      packed[j] = pack_bf16(a0, a1);
    }
    uint4* dst = reinterpret_cast<uint4*>(p.out_bf16 + (size_t)row * p.ld_bf16 + col / 2);
    dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
  } else {  // EPI_QKV
    const int q = p.q, kv = p.kv, dh = p.dh;
    const int pos = p.pos[row];
    const int region = col < q ? 0 : (col < q + kv ? 1 : 2);
    if (region == 2) {
      const int c = col - q - kv;
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
      if (p.cap_v) {
        uint4* d = reinterpret_cast<uint4*>(p.cap_v + (size_t)row * kv + c);
#pragma unroll
        for (int j = 0; j < 4; ++j) d[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      }
      __nv_bfloat16* base = p.commit ? p.ctx_v + (size_t)pos * kv : p.self_v + (size_t)row * kv;
      uint4* d = reinterpret_cast<uint4*>(base + c);
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
      return;
    }
    const int c = region == 0 ? col : col - q;
    if (region == 1 && p.cap_k) {
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
      uint4* d = reinterpret_cast<uint4*>(p.cap_k + (size_t)row * kv + c);
#pragma unroll
      for (int j = 0; j < 4; ++j) d[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
    }
    const int half = dh / 2;
    const float2* cs = p.rope + (size_t)pos * half + (c % dh) / 2;
    uint32_t pk[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float2 t = cs[j];
      const float x0 = v[2 * j], x1 = v[2 * j + 1];
      pk[j] = pack_bf16(x0 * t.x - x1 * t.y, x0 * t.y + x1 * t.x);
    }
    __nv_bfloat16* base;
    if (region == 0) base = p.out_bf16 + (size_t)row * p.ld_bf16;
    else base = p.commit ? p.ctx_k + (size_t)pos * kv : p.self_k + (size_t)row * kv;
    uint4* d = reinterpret_cast<uint4*>(base + c);
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
  }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs p) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* epi_stage = smem + C::STAGES * C::STAGE_BYTES + 256;  // [4 warps][32 rows][128 B]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const Units U = units_of(p);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      Work w;
      for (int it = 0; get_work(U, p.streamk, it, w); ++it) {
        const int mt = w.mt, nt = w.nt, kb0 = w.kb0, kb1 = w.kb1;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full[stage], kb * kBK, mt * kBM);
          tma_load_2d(sa + C::A_BYTES, &tmB, &full[stage], kb * kBK, nt * BN);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      Work w;
      for (int it = 0; get_work(U, p.streamk, it, w); ++it, ++local) {
        const int kb0 = w.kb0, kb1 = w.kb1;
        const int acc = local & 1;
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t b0 = a0 + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            mma_bf16_ss(d, sdesc_sw128(a0 + k * 32, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                        (kb > kb0 || k > 0) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {  // ------------------------------- epilogue warps 2..5
    const int quarter = warp & 3;
    const int M = p.rows_dev ? *p.rows_dev : p.rows_max;
    int local = 0;
    Work w;
    for (int it = 0; get_work(U, p.streamk, it, w); ++it, ++local) {
      const int mt = w.mt, nt = w.nt, s = w.s;
      const int acc = local & 1;
      const int row = mt * kBM + quarter * 32 + lane;
      int* flag = nullptr;
      if (EPI == EPI_ADD && U.splits > 1) {  // ordered split-K: wait for split s-1 on these rows
        flag = p.split_flags + ((size_t)(nt * U.num_m + mt) * 4 + quarter);
        if (lane == 0)
          while (atomicAdd(flag, 0) != s) __nanosleep(64);
        __syncwarp();
        __threadfence();
      }
      if constexpr (EPI == EPI_ADD) {
        // Coalesced residual epilogue: each 32x32 accumulator chunk (thread =
        // row) goes through a swizzled smem tile so that 8 lanes cover one
        // row's 128 contiguous bytes -- every load/store instruction touches 4
        // full lines instead of 32 partial ones. The residual of the next chunk
        // is prefetched while the current one is written.
        const bool norm = p.norm_part != nullptr && s + 1 == U.splits;  // final values: fused RMSNorm stats
        uint8_t* T = epi_stage + quarter * 4096;
        const int sub = lane >> 3, ch = lane & 7;  // row-within-4 and 16-byte chunk of the read-back layout
        const int row0 = mt * kBM + quarter * 32;
        auto hptr = [&](int i, int c) {  // residual of local row 4i+sub, columns c + 4*ch ..
          const int rr = row0 + 4 * i + sub;
          return reinterpret_cast<float4*>(p.out_f32 + (size_t)(rr < M ? rr : 0) * p.ld_out + nt * BN + c) + ch;
        };
        float4 hb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) hb[i] = (row0 + 4 * i + sub < M) ? __ldcg(hptr(i, 0)) : make_float4(0.f, 0.f, 0.f, 0.f);
        mbar_wait(&tfull[acc], (local >> 1) & 1);
        tc_fence_after();
        float ss[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) ss[i] = 0.f;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + c, r);
          tmem_ld_wait();
          __syncwarp();  // previous chunk's read-back of T is done
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(T + lane * 128 + ((j ^ (lane & 7)) * 16)) =
                make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
          __syncwarp();
          float4 cur[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) cur[i] = hb[i];
          if (c + 32 < BN) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              hb[i] = (row0 + 4 * i + sub < M) ? __ldcg(hptr(i, c + 32)) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rl = 4 * i + sub, rr = row0 + rl;
            const uint4 a4 = *reinterpret_cast<const uint4*>(T + rl * 128 + ((ch ^ (rl & 7)) * 16));
            float4 h = cur[i];
            h.x += __uint_as_float(a4.x);
            h.y += __uint_as_float(a4.y);
            h.z += __uint_as_float(a4.z);
            h.w += __uint_as_float(a4.w);
            if (rr < M) {
              *hptr(i, c) = h;
              if (norm) {
                ss[i] = fmaf(h.x, h.x, fmaf(h.y, h.y, fmaf(h.z, h.z, fmaf(h.w, h.w, ss[i]))));
                *reinterpret_cast<uint2*>(p.norm_bf16 + (size_t)rr * p.N + nt * BN + c + 4 * ch) =
                    make_uint2(pack_bf16(h.x, h.y), pack_bf16(h.z, h.w));
              }
            }
          }
        }
        if (norm) {
          // row sums over the 8 lanes of each row group; lane ch==0 owns rows 4i+sub
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            ss[i] += __shfl_xor_sync(0xffffffffu, ss[i], 1);
            ss[i] += __shfl_xor_sync(0xffffffffu, ss[i], 2);
            ss[i] += __shfl_xor_sync(0xffffffffu, ss[i], 4);
            const int rr = row0 + 4 * i + sub;
            if (ch == 0 && rr < M) p.norm_part[(size_t)rr * kNormSlots + nt] = ss[i];
          }
          // the last of the num_n tiles of these 32 rows turns partials into 1/rms
          __threadfence();
          __syncwarp();
          int done = 0;
          if (lane == 0) done = atomicAdd(p.norm_cnt + (size_t)mt * 4 + quarter, 1) + 1;
          done = __shfl_sync(0xffffffffu, done, 0);
          if (done == U.num_n) {
            __threadfence();
            if (row < M) {
              float tot = 0.f;
              for (int t = 0; t < U.num_n; ++t) tot += __ldcg(p.norm_part + (size_t)row * kNormSlots + t);
              p.norm_inv[row] = rsqrtf(tot / (float)p.N + p.norm_eps);
            }
            if (lane == 0) p.norm_cnt[(size_t)mt * 4 + quarter] = 0;
          }
        }
      } else {
        mbar_wait(&tfull[acc], (local >> 1) & 1);
        tc_fence_after();
        const float rs = (p.row_scale && row < M) ? p.row_scale[row] : 1.0f;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + acc * BN + c, r);
          tmem_ld_wait();
          if (row < M) epilogue_chunk<EPI>(p, row, nt * BN + c, r, rs, s);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (flag) {
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicExch(flag, s + 1 == U.splits ? 0 : s + 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// Split-K reduction + residual epilogue (EPI_PART partials): one CTA per row,
// h[row] += sum_s part[s][row] in split order (deterministic); with the fused
// RMSNorm the bf16 row copy and 1/rms come out of the same pass.
// one row of splitk_reduce_add_kernel
__device__ __forceinline__ void splitk_reduce_row(const GemmArgs& p, int splits, int row, const Units& U,
                                                  int G, const int* sk_tab) {
  const int n4 = p.N / 4;
  float ss = 0.f;
  float4* h = reinterpret_cast<float4*>(p.out_f32 + (size_t)row * p.ld_out);
  for (int c = threadIdx.x; c < n4; c += blockDim.x) {
    float4 acc;
    if (p.streamk) {  // partials of the CTAs whose k-block ranges cover this tile, in CTA order
      const int mt = row / kBM, nt = (4 * c) / p.bn;
      const int t = mt + nt * U.num_m, tlo = t * U.kb_total, thi = tlo + U.kb_total;
      int lo = 0, hi = G - 1;  // last CTA whose range starts at or before tlo (binary search)
      while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (sk_tab[mid] <= tlo) lo = mid;
        else hi = mid - 1;
      }
      acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int g = lo; g < G && sk_tab[g] < thi; ++g) {
        if (sk_tab[g + 1] == sk_tab[g]) continue;  // empty range: no partial
        const int slot = t - sk_tab[g] / U.kb_total;
        const float4 v = __ldcg(reinterpret_cast<const float4*>(
            p.ws_part + (((size_t)g * kSkSlots + slot) * kBM + row % kBM) * p.bn + (4 * c) % p.bn));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    } else {
      acc = __ldcg(reinterpret_cast<const float4*>(p.ws_part + (size_t)row * p.N) + c);
      for (int s = 1; s < splits; ++s) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(p.ws_part + ((size_t)s * p.rows_max + row) * p.N) + c);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    float4 x = h[c];
    x.x += acc.x; x.y += acc.y; x.z += acc.z; x.w += acc.w;
    h[c] = x;
    if (p.norm_bf16) {
      ss += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
      reinterpret_cast<uint2*>(p.norm_bf16 + (size_t)row * p.N)[c] = make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
    }
  }
  if (p.norm_inv) {
    __shared__ float red[8];
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      p.norm_inv[row] = rsqrtf(t / (float)p.N + p.norm_eps);
    }
    __syncthreads();  // red[] is reused by the CTA's next row
  }
}

__global__ void __launch_bounds__(256) splitk_reduce_add_kernel(const GemmArgs p, int splits, int G) {
  const int M = p.rows_dev ? *p.rows_dev : p.rows_max;
  const Units U = units_of(p);
  __shared__ int sk_tab[1025];  // stream-K range starts of the G CTAs (+ end)
  if (p.streamk) {
    for (int g = threadIdx.x; g <= G; g += blockDim.x) sk_tab[g] = (int)sk_lo(U, g, G);
    __syncthreads();
  }
  for (int row = blockIdx.x; row < M; row += gridDim.x)
    splitk_reduce_row(p, splits, row, U, G, sk_tab);
}

template <int BN, int EPI>
void launch(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p, int grid) {
  static bool attr = false;
  if (!attr) {
    RK_CUDA(cudaFuncSetAttribute(gemm_bf16_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
    attr = true;
  }
  gemm_bf16_kernel<BN, EPI><<<grid, kThreads, Cfg<BN>::SMEM, st>>>(a, b, p);
}

template <int EPI>
void launch_bn(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p, int grid) {
  if (p.bn == 256) launch<256, EPI>(st, a, b, p, grid);
  else if (p.bn == 128) launch<128, EPI>(st, a, b, p, grid);
  else launch<64, EPI>(st, a, b, p, grid);
}

}  // namespace

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    RK_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) raise(RK_ERR_RUNTIME, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_encodeTiled>(f);
  }
  return fn;
}

// 2-D bf16 row-major [rows x cols] tensor map, box {64, box_rows}, 128B swizzle.
void make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows,
                    uint64_t row_stride_elems) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(RK_ERR_RUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

// Pick the N tile and split count so the grid fills the SMs: the widest tile
// that still gives a full wave, else BN=64; split-K only while the grid is
// under half the SMs (split_flags present, residual epilogue).
static void choose_config(GemmArgs& p, int sm_count, int rows_hint) {
  const int num_m = (rows_hint + kBM - 1) / kBM;
  p.sms = sm_count;
  int bn = 64;
  for (int cand : {256, 128}) {
    if (p.N % cand == 0 && num_m * (p.N / cand) >= sm_count) { bn = cand; break; }
  }
  if (p.N % bn) raise(RK_ERR_INVALID_ARGUMENT, "bf16 GEMM needs N % 64 == 0");
  p.bn = bn;
  p.splits = 1;
  if (p.epi == EPI_ADD && p.split_flags) {
    // residual GEMMs that cannot fill the SMs: widest tile, K split s ways with
    // the s partials reduced (in order) by splitk_reduce_add_kernel; s picks
    // the best wave efficiency of tiles*s units over the SMs
    // Cost model (calibrated on B200): a 128x256 k-block ~0.45 us per CTA;
    // partials cost s * M * N * 4 B written + read at ~8 TB/s plus ~3 us for
    // the reduce launch.
    const int wide = p.N % 256 == 0 ? 256 : (p.N % 128 == 0 ? 128 : 64);
    const int tiles = num_m * (p.N / wide), kb = p.K / kBK;
    if (4 * tiles < 3 * sm_count) {
      const double t_kb = 0.45 * wide / 256.0;
      // stream-K: every SM gets the same k-block count; partials of the
      // ~tiles + SMs segments go through L2 to the reduce kernel
      // (measured on c2: slower than split-K at these shapes -- opt-in with
      // RK_GEMM_STREAMK=1 for experiments)
      static const bool sk_enabled = [] {
        const char* v = std::getenv("RK_GEMM_STREAMK");
        return v && std::atoi(v) != 0;
      }();
      const int tiles_max = ((p.rows_max + kBM - 1) / kBM) * (p.N / wide);
      const bool sk_ok = sk_enabled && kb >= 2 && tiles_max <= 2 * sm_count;
      const double sk_cost = sk_ok ? ((double)tiles * kb + sm_count - 1) / sm_count * t_kb + 1.0 +
                                         2.0 * (tiles + sm_count) * (double)kBM * wide * 4 / 8e6
                                   : 1e30;
      auto cost = [&](int s) {
        const int units = tiles * s, waves = (units + sm_count - 1) / sm_count;
        const double mma = waves * ((kb + s - 1) / s) * t_kb;
        const double part = s > 1 ? 3.0 + 2.0 * s * (double)rows_hint * p.N * 4 / 8e6 : 0.0;
        return mma + part;
      };
      int best = 1;
      double best_cost = cost(1);
      for (int s = 2; s <= 8 && kb / s >= 4; ++s)
        if (cost(s) < best_cost) { best = s; best_cost = cost(s); }
      if (sk_cost < best_cost) {
        p.bn = wide;
        p.splits = 1;
        p.streamk = 1;
        p.epi = EPI_PART;
      } else if (best > 1) {
        p.bn = wide;
        p.splits = best;
        p.epi = EPI_PART;
      }
    }
  }
}

void gemm_bf16(rk_engine* e, const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, GemmArgs p,
               int rows_hint) {
  if (p.rows_max <= 0) return;
  if (p.K % kBK) raise(RK_ERR_INVALID_ARGUMENT, "bf16 GEMM needs K % 64 == 0");
  choose_config(p, e->sm_count, rows_hint > 0 ? rows_hint : p.rows_max);
  if (p.norm_part && p.N / p.bn > kNormSlots) raise(RK_ERR_INVALID_ARGUMENT, "fused RMSNorm: too many N tiles");
  CUtensorMap ta, tb;
  make_tmap_bf16(&ta, A, (uint64_t)p.rows_max, (uint64_t)p.K, kBM, (uint64_t)lda);
  make_tmap_bf16(&tb, B, (uint64_t)p.N, (uint64_t)p.K, (uint32_t)p.bn, (uint64_t)p.K);
  const int num_m = (p.rows_max + kBM - 1) / kBM;
  const int total = num_m * (p.N / p.bn) * p.splits;
  const int grid = p.streamk ? e->sm_count : (total < e->sm_count ? total : e->sm_count);
  if (p.epi == EPI_PART) {
    e->scratch->gemm_ws.ensure(p.streamk ? (size_t)grid * kSkSlots * kBM * p.bn * 4
                                         : (size_t)p.splits * p.rows_max * p.N * 4);
    p.ws_part = e->scratch->gemm_ws.as<float>();
  }
  static const char* kEpi[] = {"qkv", "add", "silu", "f32", "addsplit"};
  ProfScope ps(e, (e->prof && e->prof->on)
                      ? intern(std::string("gemm_") + kEpi[p.epi] + "_m" + std::to_string(p.rows_max) +
                               (p.rows_dev ? "dyn" : "") + "_n" + std::to_string(p.N) + "_k" + std::to_string(p.K) +
                               "_bn" + std::to_string(p.bn) + (p.streamk ? std::string("_sk") : "_s" + std::to_string(p.splits)))
                      : "gemm",
               0, 0);
  ps.rec.kind = 1;
  ps.rec.rows_dev = p.rows_dev;
  ps.rec.rows_max = rows_hint > 0 && !p.rows_dev ? p.rows_max : p.rows_max;
  ps.rec.N = p.N;
  ps.rec.K = p.K;
  switch (p.epi) {
    case EPI_QKV: launch_bn<EPI_QKV>(e->stream, ta, tb, p, grid); break;
    case EPI_ADD: launch_bn<EPI_ADD>(e->stream, ta, tb, p, grid); break;
    case EPI_SILU: launch_bn<EPI_SILU>(e->stream, ta, tb, p, grid); break;
    case EPI_PART:
      launch_bn<EPI_PART>(e->stream, ta, tb, p, grid);
      splitk_reduce_add_kernel<<<std::min(p.rows_max, 8 * e->sm_count), 256, 0, e->stream>>>(p, p.splits, grid);
      e->launches += 1;
      break;
    default: launch_bn<EPI_F32>(e->stream, ta, tb, p, grid); break;
  }
  e->launches += 1;
}

}  // namespace rk
