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
// Shapes (choose_config picks one per GEMM from a calibrated cost model):
//   1-CTA      128 x BN tiles, persistent, one CTA per SM
//   CTA pair   cluster of 2, tcgen05 cta_group::2, 256 x BN tiles; each CTA
//              stages half of B, halving the L2->SM feed per MMA
//   split-K    residual GEMMs that cannot fill the GPU: fp32 partials reduced
//              in split order (splitk_reduce_add_kernel)
//   swap-AB    (gemm_swap_kernel) wide short-M SiLU GEMMs: weights on the MMA's M side
//   GEMV       M = 1 (top-layer last row, logits head, decode steps): CUDA
//              cores at HBM speed with the same epilogues
//
// Fused epilogues (the reference computes these as separate loops over the
// matmul outputs, model.cpp:246-280 / 211-233):
//   EPI_QKV   RoPE on Q and K (adjacent pairs, tensor.cpp:134-142), Q -> bf16
//             buffer, K/V rows scattered into the context at each row's
//             absolute position (model.cpp:266-269), optional capture of
//             pre-RoPE K and V (decode-time capture, model.cpp:254-257)
//   EPI_ADD   hidden += D (residual) + the next RMSNorm's bf16 rows and 1/rms;
//             split-K residual GEMMs write EPI_PART partials instead, summed
//             in split order (deterministic) by splitk_reduce_add_kernel
//   EPI_SILU  interleaved (gate, up) columns -> bf16 silu(g)*u (model.cpp:226)
//   EPI_F32   plain fp32 store (logits)
#include <cuda.h>
#include <cstdio>
#include <cstring>
#include <vector>

#include <algorithm>
#include <cstdio>
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

// ensure_finite (tensor.cpp:58-64): x * 0 is NaN exactly when x is inf or NaN,
// so one FFMA per value folds a whole chunk into one check.
__device__ __forceinline__ float finite_acc(float acc, float x) { return fmaf(x, 0.0f, acc); }
__device__ __forceinline__ void flag_nonfinite(int* status, float acc) {
  if (acc != acc && status) *reinterpret_cast<volatile int*>(status) = 1;
}
constexpr int kThreads = 192;
// debug timeline (GemmArgs::trace, rk_debug_trace_gemm): CTA 0 only;
// role 0 producer (per k-block: empty slot acquired), role 1 MMA issuer (per
// k-block: stage full), role 2 epilogue warp 2 (per unit: 2u accumulator
// ready, 2u+1 drained)
#define GTRACE(role, i, cond)                                                                  \
  do {                                                                                         \
    if (p.trace && blockIdx.x == 0 && (cond) && (i) < 512) p.trace[(role) * 512 + (i)] = clock64(); \
  } while (0)

// PAIR = 2: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes a
// 256 x BN tile; each CTA stages its own 128 rows of A and HALF of the BN rows
// of B, so a CTA's shared-memory fill per k-block drops from 48 KB to 32 KB
// (BN=256) -- the L2->SM feed, not the tensor pipe, bounds the 1-CTA kernel.
//
// (Variants measured slower on the c2 shapes in round 1-2 and removed: cluster
// split-K over DSMEM, m-grouped short-M tiles, stream-K, L2 weight prefetch,
// in-GEMM split-K fixup -- see DESIGN.md section 11.)
constexpr int pow2_cols(int c) { return c <= 32 ? 32 : (c <= 64 ? 64 : (c <= 128 ? 128 : (c <= 256 ? 256 : 512))); }
template <int BN, int PAIR = 1>
struct Cfg {
  static constexpr int A_BYTES = kBM * kBK * 2;
  static constexpr int B_BYTES = BN / PAIR * kBK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = PAIR == 1 ? ((BN == 256) ? 4 : (BN == 128 ? 6 : 8))
                                           : (BN == 256 ? 6 : (BN == 192 ? 7 : 8));
  static constexpr int NACC = 2;  // TMEM accumulator buffers
  static constexpr int TMEM_COLS = pow2_cols(NACC * BN);
  // per epilogue warp: a 32x32 fp32 staging tile for the coalesced residual epilogue
  static constexpr int EPI_STAGE = 4 * 32 * 32 * 4;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + EPI_STAGE;
};

struct Units {
  int num_m, num_n, splits, kb_total, kb_per;
  int total;
};

template <int PAIR = 1>
__device__ __forceinline__ Units units_of(const GemmArgs& p) {
  Units u;
  const int M = p.rows_dev ? *p.rows_dev : p.rows_max;
  // m tiles of 128 (or 256-row pair tiles)
  u.num_m = (M + kBM * PAIR - 1) / (kBM * PAIR);
  u.num_n = (p.N + p.bn - 1) / p.bn;  // (BN 192: the last N tile may be ragged)
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

// One accumulator's worth of work: tile (mt, nt), k-blocks [kb0, kb1) of split s.
struct Work {
  int mt, nt, s, kb0, kb1;
};

// k-th work item of this CTA (both CTAs of a pair walk the same units);
// false when the CTA is done.
template <int PAIR = 1>
__device__ __forceinline__ bool get_work(const Units& U, int k, Work& w) {
  const int unit = blockIdx.x / PAIR + k * (gridDim.x / PAIR);
  if (unit >= U.total) return false;
  decode_unit(U, unit, w.mt, w.nt, w.s);
  w.kb0 = w.s * U.kb_per;
  w.kb1 = min(U.kb_total, w.kb0 + U.kb_per);
  return true;
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& p, int row, int col, const uint32_t (&r)[32],
                                               float rs, int split = 0, const float2* csv = nullptr, int pos_in = -1) {
  float v[32];
  float chk = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    v[j] = __uint_as_float(r[j]) * rs;
    chk = finite_acc(chk, v[j]);
  }
  flag_nonfinite(p.status, chk);
  if constexpr (EPI == EPI_F32 || EPI == EPI_PART) {
    float* base = EPI != EPI_PART ? p.out_f32 + (size_t)row * p.ld_out + col
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
      const float a0 = __fdividef(g0, 1.0f + __expf(-g0)) * u0;  // (no IEEE-division slow path; bf16 output)
      const float a1 = __fdividef(g1, 1.0f + __expf(-g1)) * u1;
      packed[j] = pack_bf16(a0, a1);
    }
    uint4* dst = reinterpret_cast<uint4*>(p.out_bf16 + (size_t)row * p.ld_bf16 + col / 2);
    dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
    dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
  } else {  // EPI_QKV
    const int q = p.q, kv = p.kv, dh = p.dh;
    const int pos = pos_in >= 0 ? pos_in : p.pos[row];
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
      const float2 t = csv ? csv[j] : cs[j];
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

// Coalesced epilogue stores: a warp's 32 rows (thread = row, the TMEM lane
// layout) are transposed through a per-warp 4 KB shared tile so that each
// store instruction covers whole row segments -- 8 lanes per 128-byte fp32
// segment -- instead of 32 rows x 16 B (r02af trace: the per-row stores made
// the fp32 epilogue of a 256-column pair tile take ~16k cycles and stalled
// the next tile's mainloop; F32 band-shape GEMM 49 -> 42 us). (For the bf16
// QKV / SiLU outputs the extra shared-memory traffic competes with the next
// tile's MMAs and measured slower -- r02ag -- so they store per row.)
// dst(rl) returns the destination of local row rl's segment (nullptr: skip).
template <class Dst>
__device__ __forceinline__ void stage_store128(uint8_t* T, int lane, const float (&v)[32], Dst dst) {
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<uint4*>(T + lane * 128 + ((j ^ (lane & 7)) * 16)) =
        make_uint4(__float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]), __float_as_uint(v[4 * j + 2]),
                   __float_as_uint(v[4 * j + 3]));
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int rl = 4 * i + (lane >> 3), ch = lane & 7;
    const uint4 x = *reinterpret_cast<const uint4*>(T + rl * 128 + ((ch ^ (rl & 7)) * 16));
    uint4* d = dst(rl);
    if (d) d[ch] = x;
  }
}

template <int BN, int EPI, int PAIR, bool TF32 = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmArgs p) {
  using C = Cfg<BN, PAIR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* epi_stage = smem + C::STAGES * C::STAGE_BYTES + 256;  // [4 warps][32 rows][128 B]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = PAIR == 2 ? cluster_ctarank() : 0;  // 0 = leader (issues the MMAs)
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4 * PAIR);  // the epilogue warps of both CTAs drain the leader's accumulator
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR == 2) tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    else tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (PAIR == 2) cluster_sync();  // barriers of both CTAs initialised before any remote use
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // The producer starts streaming the weights (B) of its first STAGES k-blocks
  // before the dependency wait -- they do not depend on the previous kernel --
  // so with programmatic dependent launch the weight stream overlaps the
  // previous kernel's tail; A (activations) follows after the wait.
  int pre = 0;
  if (warp == 0 && !p.rows_dev && !(p.dbg & 1)) {
    const Units Up = units_of<PAIR>(p);
    Work w0;
    if (elect_one() && get_work<PAIR>(Up, 0, w0)) {
      pre = min(C::STAGES, w0.kb1 - w0.kb0);
      for (int i = 0; i < pre; ++i) {
        uint8_t* sa = smem + i * C::STAGE_BYTES;
        const int kx = (w0.kb0 + i) * kBK;
        if constexpr (PAIR == 2) {
          if (rank == 0) mbar_arrive_expect_tx(&full[i], 2 * C::STAGE_BYTES);
          tma_load_2d_pair(sa + C::A_BYTES, &tmB, &full[i], kx, w0.nt * BN + rank * (BN / 2));
        } else {
          mbar_arrive_expect_tx(&full[i], C::STAGE_BYTES);
          tma_load_2d(sa + C::A_BYTES, &tmB, &full[i], kx, w0.nt * BN);
        }
      }
    }
  }
  if (warp == 0 && p.rows_dev && p.m_hint > 0 && !(p.dbg & 1)) {
    // live rows known only on the device: warm L2 with the weight k-blocks of
    // the first unit the host's row estimate predicts (a wrong guess costs L2
    // bandwidth only), so the ring's first loads after the wait hit L2
    Units Uh = units_of<PAIR>(p);
    Uh.num_m = p.m_hint;
    Uh.total = Uh.num_m * Uh.num_n * Uh.splits;
    Work w0;
    if (elect_one() && get_work<PAIR>(Uh, 0, w0))
      for (int i = 0; i < C::STAGES && w0.kb0 + i < w0.kb1; ++i)
        tma_prefetch_2d(&tmB, (w0.kb0 + i) * kBK, w0.nt * BN + (int)rank * (BN / PAIR));
  }
  pdl_wait();  // the prologue above overlapped the previous kernel; its outputs are visible from here
  const Units U = units_of<PAIR>(p);

  if (warp == 0) {
    if (elect_one()) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      Work w;
      int kbn = 0;  // (trace index)
      for (int it = 0; get_work<PAIR>(U, it, w); ++it) {
        const int mt = w.mt, nt = w.nt, kb0 = w.kb0, kb1 = w.kb1;
        for (int kb = kb0; kb < kb1; ++kb, ++kbn) {
          const bool early = it == 0 && kb - kb0 < pre;  // stage armed, its B already in flight
          if (!early) mbar_wait(&empty[stage], phase ^ 1);
          GTRACE(0, kbn, true);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          const bool same = p.dbg & 1;
          const int kx = same ? 0 : kb * kBK, am = same ? 0 : mt, bn_ = same ? 0 : nt;
          if constexpr (PAIR == 2) {
            // the leader's barrier counts both CTAs' bytes
            if (rank == 0 && !early) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            tma_load_2d_pair(sa, &tmA, &full[stage], kx, (am * 2 + rank) * kBM);
            if (!early) tma_load_2d_pair(sa + C::A_BYTES, &tmB, &full[stage], kx, bn_ * BN + rank * (BN / 2));
          } else {
            if (!early) mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(sa, &tmA, &full[stage], kx, am * kBM);
            if (!early) tma_load_2d(sa + C::A_BYTES, &tmB, &full[stage], kx, bn_ * BN);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {  // ---------------- MMA issuer (the pair's leader)
      constexpr uint32_t idesc = TF32 ? idesc_tf32(kBM * PAIR, BN) : idesc_bf16(kBM * PAIR, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0, kbm = 0;
      Work w;
      for (int it = 0; get_work<PAIR>(U, it, w); ++it, ++local) {
        const int kb0 = w.kb0, kb1 = w.kb1;
        const int acc = local % C::NACC;
        mbar_wait(&tempty[acc], ((local / C::NACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++kbm) {
          mbar_wait(&full[stage], phase);
          GTRACE(1, kbm, true);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t b0 = a0 + C::A_BYTES;
          {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              if (p.dbg & 2) break;
              const uint32_t am = a0 + k * 32;
              if constexpr (PAIR == 2 && TF32)
                mma_tf32_ss_pair(d, sdesc_sw128(am, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                                 (kb > kb0 || k > 0) ? 1u : 0u);
              else if constexpr (PAIR == 2)
                mma_bf16_ss_pair(d, sdesc_sw128(am, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                                 (kb > kb0 || k > 0) ? 1u : 0u);
              else if constexpr (TF32)
                mma_tf32_ss(d, sdesc_sw128(am, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                            (kb > kb0 || k > 0) ? 1u : 0u);
              else
                mma_bf16_ss(d, sdesc_sw128(am, 16, 1024), sdesc_sw128(b0 + k * 32, 16, 1024), idesc,
                            (kb > kb0 || k > 0) ? 1u : 0u);
            }
          }
          if constexpr (PAIR == 2) tc_commit_pair(&empty[stage]);
          else tc_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (PAIR == 2) tc_commit_pair(&tfull[acc]);
        else tc_commit(&tfull[acc]);
      }
    }
  } else {  // ------------------------------- epilogue warps 2..5
    const int quarter = warp & 3;
    const int M = p.rows_dev ? *p.rows_dev : p.rows_max;
    int local = 0;
    Work w;
    for (int it = 0; get_work<PAIR>(U, it, w); ++it, ++local) {
      const int acc = local % C::NACC, use = local / C::NACC;
      {
      const int mt = w.mt * PAIR + rank, nt = w.nt, s = w.s;  // this CTA's 128-row tile
      const uint32_t acol = (uint32_t)(acc * BN);  // its accumulator's first TMEM column
      const int row = mt * kBM + quarter * 32 + lane;
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
        const int bn_live = min(BN, p.N - nt * BN);  // (a ragged last N tile stores its live columns only)
        auto hptr = [&](int i, int c) {  // residual of local row 4i+sub, columns c + 4*ch ..
          const int rr = row0 + 4 * i + sub;
          return reinterpret_cast<float4*>(p.out_f32 + (size_t)(rr < M ? rr : 0) * p.ld_out + nt * BN + c) + ch;
        };
        float4 hb[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) hb[i] = (row0 + 4 * i + sub < M) ? __ldcg(hptr(i, 0)) : make_float4(0.f, 0.f, 0.f, 0.f);
        mbar_wait(&tfull[acc], use & 1);
        GTRACE(2, 2 * local, warp == 2 && lane == 0);
        tc_fence_after();
        float ss[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) ss[i] = 0.f;
        float chk = 0.f;  // non-finite matmul values (rows past M are zero-filled A rows: finite)
#pragma unroll 1
        for (int c = 0; c < bn_live; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + acol + c, r);
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
          if (c + 32 < bn_live) {
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
              chk = finite_acc(finite_acc(finite_acc(finite_acc(chk, __uint_as_float(a4.x)), __uint_as_float(a4.y)),
                                          __uint_as_float(a4.z)), __uint_as_float(a4.w));
              *hptr(i, c) = h;
              if (norm) {
                ss[i] = fmaf(h.x, h.x, fmaf(h.y, h.y, fmaf(h.z, h.z, fmaf(h.w, h.w, ss[i]))));
                *reinterpret_cast<uint2*>(p.norm_bf16 + (size_t)rr * p.N + nt * BN + c + 4 * ch) =
                    make_uint2(pack_bf16(h.x, h.y), pack_bf16(h.z, h.w));
              }
            }
          }
        }
        flag_nonfinite(p.status, chk);
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
          fence_acq_rel_gpu();  // (release: this warp's partials and rows)
          __syncwarp();
          int done = 0;
          if (lane == 0) done = atomicAdd(p.norm_cnt + (size_t)mt * 4 + quarter, 1) + 1;
          done = __shfl_sync(0xffffffffu, done, 0);
          if (done == U.num_n) {
            fence_acq_rel_gpu();  // (acquire: the other tiles' partials)
            if (row < M) {
              // all of the row's partials in flight at once (16-byte loads),
              // summed in tile order (a runtime-bounded scalar loop was one
              // L2 round trip per tile: +6 us on the M=320 W_o GEMM, r02ah)
              const float4* pp = reinterpret_cast<const float4*>(p.norm_part + (size_t)row * kNormSlots);
              const int nn = U.num_n, n4 = (nn + 3) / 4;
              float4 v[kNormSlots / 4];
#pragma unroll
              for (int i = 0; i < kNormSlots / 4; ++i)
                if (i < n4) v[i] = __ldcg(pp + i);
              float tot = 0.f;
#pragma unroll
              for (int i = 0; i < kNormSlots / 4; ++i) {
                if (4 * i < nn) tot += v[i].x;
                if (4 * i + 1 < nn) tot += v[i].y;
                if (4 * i + 2 < nn) tot += v[i].z;
                if (4 * i + 3 < nn) tot += v[i].w;
              }
              p.norm_inv[row] = rsqrtf(tot / (float)p.N + p.norm_eps);
            }
            if (lane == 0) p.norm_cnt[(size_t)mt * 4 + quarter] = 0;
          }
        }
      } else {
        mbar_wait(&tfull[acc], use & 1);
        GTRACE(2, 2 * local, warp == 2 && lane == 0);
        tc_fence_after();
        const float rs = (p.row_scale && row < M) ? p.row_scale[row] : 1.0f;
        const int bn_live = min(BN, p.N - nt * BN);  // (ragged last N tile)
        uint8_t* T = epi_stage + quarter * 4096;
        const int row0 = mt * kBM + quarter * 32;  // the warp's first row
        if constexpr (EPI == EPI_QKV) {
          const int pos = row < M ? p.pos[row] : 0;
          const float2* csrow = p.rope + (size_t)pos * (p.dh / 2);
          if (p.dh == 64) {
            // the row's whole RoPE {cos, sin} row (32 pairs, 256 B) once per
            // tile as 16-byte loads; every head of the tile reuses it (chunks
            // c and c+32 of a head take its two halves)
            float2 cs[32];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float4 t = reinterpret_cast<const float4*>(csrow)[j];
              cs[2 * j] = make_float2(t.x, t.y);
              cs[2 * j + 1] = make_float2(t.z, t.w);
            }
#pragma unroll 1
            for (int c = 0; c < bn_live; c += 64) {
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                if (c + 32 * hh >= bn_live) break;
                uint32_t r[32];
                tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + acol + c + 32 * hh, r);
                tmem_ld_wait();
                if (row < M) epilogue_chunk<EPI>(p, row, nt * BN + c + 32 * hh, r, rs, s, cs + 16 * hh, pos);
              }
            }
          } else {
            // RoPE {cos, sin} of the next chunk load while the current one computes
            float2 cur[16], nxt[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) cur[j] = csrow[((nt * BN) % p.dh) / 2 + j];
#pragma unroll 1
            for (int c = 0; c < bn_live; c += 32) {
              if (c + 32 < bn_live) {
#pragma unroll
                for (int j = 0; j < 16; ++j) nxt[j] = csrow[((nt * BN + c + 32) % p.dh) / 2 + j];
              }
              uint32_t r[32];
              tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + acol + c, r);
              tmem_ld_wait();
              if (row < M) epilogue_chunk<EPI>(p, row, nt * BN + c, r, rs, s, cur, pos);
#pragma unroll
              for (int j = 0; j < 16; ++j) cur[j] = nxt[j];
            }
          }
        } else if constexpr (EPI == EPI_SILU) {
#pragma unroll 1
          for (int c = 0; c < bn_live; c += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + acol + c, r);
            tmem_ld_wait();
            if (row < M) epilogue_chunk<EPI>(p, row, nt * BN + c, r, rs, s);
          }
        } else {  // EPI_F32 / EPI_PART: 128-byte fp32 segments
#pragma unroll 1
          for (int c = 0; c < bn_live; c += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + acol + c, r);
            tmem_ld_wait();
            float v[32];
            float chk = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              v[j] = __uint_as_float(r[j]) * rs;
              chk = finite_acc(chk, v[j]);
            }
            if (row < M) flag_nonfinite(p.status, chk);
            const int col = nt * BN + c;
            stage_store128(T, lane, v, [&](int rl) -> uint4* {
              const int rr = row0 + rl;
              if (rr >= M) return nullptr;
              float* base = EPI != EPI_PART ? p.out_f32 + (size_t)rr * p.ld_out + col
                                            : p.ws_part + ((size_t)s * p.rows_max + rr) * p.N + col;
              return reinterpret_cast<uint4*>(base);
            });
          }
        }
      }
      }
      tc_fence_before();
      __syncwarp();
      GTRACE(2, 2 * local + 1, warp == 2 && lane == 0);
      if (lane == 0) {
        if constexpr (PAIR == 2) mbar_arrive_cluster(&tempty[acc], 0);
        else mbar_arrive(&tempty[acc]);
      }
    }
  }
  tc_fence_before();
  if constexpr (PAIR == 2) {
    cluster_sync();  // neither CTA leaves while its peer may still signal its barriers
    if (warp == 1) tmem_dealloc_pair(tmem, C::TMEM_COLS);
  } else {
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// Swap-AB CTA pair for short static M (the prefix/suffix-only layers, M <= 512):
// D^T[N x M] = W[N x K] . X[M x K]^T. The weights take the MMA's M side -- 256
// rows per pair, each CTA staging its own 128 -- and the M tokens its N side,
// nc chunks of tc columns (each CTA staging half of every chunk). The 1-CTA
// 128 x 256 tile stages 48 KB per k-block for 4.2 MFLOP and, at M = 320, reads
// every weight tile three times in two rounds; here a CTA stages 16 + M/16 KB
// for 2*128*M*64 FLOP (M = 320: 36 KB for 5.2 MFLOP) and each weight tile is
// read by exactly one pair in one round. TMEM lane = output feature, column =
// token, so the epilogue walks 32 tokens per tcgen05.ld; residual GEMMs store
// split-K partials (EPI_PART) for splitk_reduce_add_kernel.
// ---------------------------------------------------------------------------
constexpr int kSwStages = 4;      // ring bytes = kSwStages * kSwStage; the ring is cut into
constexpr int kSwMaxStages = 6;   // as many stages of the launch's real size as fit (<= 6)
constexpr int kSwA = kBM * kBK * 2;     // 16 KB: this CTA's 128 weight rows
constexpr int kSwBMax = 256 * kBK * 2;  // 32 KB: half of up to 512 tokens
constexpr int kSwStage = kSwA + kSwBMax;
constexpr int kSwRs = 544;  // row scales of up to 512 tokens (+ one chunk of padding)
constexpr int kSwEpi = 8 * 1024;  // per epilogue warp: 32 tokens x 16 bf16 outputs (SiLU transpose)
constexpr int kSwSmem = kSwStages * kSwStage + 1024 + 256 + kSwRs * 4 + kSwEpi;
constexpr uint32_t kSwTmemCols = 512;
constexpr int kSwThreads = 320;  // producer, MMA issuer, 8 epilogue warps (two per TMEM lane quarter)

// SiLU epilogue of the swap kernel: thread = feature n (gate on even lanes,
// up on odd), 32 tokens per TMEM load. The 16 outputs x 32 tokens of a warp go
// through a 1 KB shared tile so each store is a 16-byte piece of a token's
// 32-byte output segment (2 instructions per chunk instead of 16 2-byte
// scattered stores); row scales come as 16-byte shared loads; full chunks run
// without per-element bounds checks. (r02al trace: the scalar version took
// ~3.5k cycles per 32-token chunk, as long as the whole mainloop.)
__device__ __forceinline__ void swap_silu_epilogue(const GemmArgs& p, uint32_t tbase, int n, int M, int lane, int hw,
                                                   const float* rs_sm, uint8_t* S) {
  const bool odd = lane & 1;
  const int i = lane >> 1;            // output column within the warp's 16
  const int col0 = (n - lane) / 2;    // the warp's first output column
  const uint32_t rs_s = smem_u32(rs_sm), S_s = smem_u32(S);
  float chk = 0.f;
#pragma unroll 1
  for (int t0 = 32 * hw; t0 < M; t0 += 64) {
    uint32_t r[32];
    tmem_ld32(tbase + (uint32_t)t0, r);
    float rs[32];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(rs[4 * q]), "=f"(rs[4 * q + 1]), "=f"(rs[4 * q + 2]), "=f"(rs[4 * q + 3])
                   : "r"(rs_s + (uint32_t)(t0 + 4 * q) * 4u));
    tmem_ld_wait();
    const int lim = M - t0;  // valid tokens in this chunk (>= 32 except the last)
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = __uint_as_float(r[j]) * rs[j];
      chk = finite_acc(chk, j < lim ? v[j] : 0.f);
    }
    // even lane (gate) takes tokens t0..t0+15, odd lane (up) t0+16..t0+31
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float recv = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[16 + j], 1);
      const float g = odd ? recv : v[j], u = odd ? v[16 + j] : recv;
      const float a = __fdividef(g, 1.0f + __expf(-g)) * u;
      const int tl = (odd ? 16 : 0) + j;
      asm volatile("st.shared.b16 [%0], %1;" ::"r"(S_s + (uint32_t)(tl * 32 + i * 2)),
                   "h"(__bfloat16_as_ushort(__float2bfloat16_rn(a))));
    }
    __syncwarp();
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
      const int piece = lane + 32 * rep, tok = piece >> 1, h = piece & 1;
      uint4 x;
      asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                   : "r"(S_s + (uint32_t)(tok * 32 + h * 16)));
      if (tok < lim) *reinterpret_cast<uint4*>(p.out_bf16 + (size_t)(t0 + tok) * p.ld_bf16 + col0 + 8 * h) = x;
    }
    __syncwarp();
  }
  flag_nonfinite(p.status, chk);
}

// Epilogue of one CTA's 128 features (thread = feature n) over the M tokens.
// rs_sm: the M row scales (1.0 without a fused RMSNorm), staged in shared
// memory; warp half `hw` of a lane quarter takes token chunks hw, hw+2, ...
template <int EPI>
__device__ __forceinline__ void swap_epilogue(const GemmArgs& p, uint32_t tbase, int n, int M, int split,
                                              int lane, int hw, const float* rs_sm) {
  const bool odd = lane & 1;  // == n & 1: RoPE pairs and (gate, up) pairs are adjacent lanes
  float chk = 0.f;
#pragma unroll 1
  for (int t0 = 32 * hw; t0 < M; t0 += 64) {
    uint32_t r[32];
    tmem_ld32(tbase + (uint32_t)t0, r);
    tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = __uint_as_float(r[j]) * rs_sm[t0 + j];
      if (t0 + j < M) chk = finite_acc(chk, v[j]);  // (columns past the token tile hold no data)
    }
    if constexpr (EPI == EPI_F32 || EPI == EPI_PART) {
      float* base = EPI == EPI_PART ? p.ws_part + (size_t)split * p.rows_max * p.N + n : p.out_f32 + n;
      const size_t ld = EPI == EPI_PART ? (size_t)p.N : (size_t)p.ld_out;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (t0 + j < M) base[(size_t)(t0 + j) * ld] = v[j];
    } else if constexpr (EPI == EPI_SILU) {
      // even lane (gate) takes tokens t0..t0+15, odd lane (up) t0+16..t0+31
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float recv = __shfl_xor_sync(0xffffffffu, odd ? v[j] : v[16 + j], 1);
        const int t = odd ? t0 + 16 + j : t0 + j;
        const float g = odd ? recv : v[j], u = odd ? v[16 + j] : recv;
        if (t < M) p.out_bf16[(size_t)t * p.ld_bf16 + n / 2] = __float2bfloat16_rn(__fdividef(g, 1.0f + __expf(-g)) * u);
      }
    } else {  // EPI_QKV
      const int q = p.q, kv = p.kv, dh = p.dh;
      if (n >= q + kv) {  // V rows into the context (warp-uniform region: q, kv are multiples of 32)
        const int c = n - q - kv;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int t = t0 + j;
          if (t >= M) break;
          const __nv_bfloat16 b = __float2bfloat16_rn(v[j]);
          if (p.cap_v) p.cap_v[(size_t)t * kv + c] = b;
          (p.commit ? p.ctx_v + (size_t)p.pos[t] * kv : p.self_v + (size_t)t * kv)[c] = b;
        }
      } else {
        const bool is_k = n >= q;
        const int c = is_k ? n - q : n, pi = (c % dh) / 2;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
          const int t = t0 + j;
          if (t < M) {
            if (is_k && p.cap_k) p.cap_k[(size_t)t * kv + c] = __float2bfloat16_rn(v[j]);
            const int pos = p.pos[t];
            const float2 cs = p.rope[(size_t)pos * (dh / 2) + pi];
            const float x0 = odd ? partner : v[j], x1 = odd ? v[j] : partner;
            const float o = odd ? x0 * cs.y + x1 * cs.x : x0 * cs.x - x1 * cs.y;
            __nv_bfloat16* base = !is_k ? p.out_bf16 + (size_t)t * p.ld_bf16
                                        : (p.commit ? p.ctx_k + (size_t)pos * kv : p.self_k + (size_t)t * kv);
            base[c] = __float2bfloat16_rn(o);
          }
        }
      }
    }
  }
  flag_nonfinite(p.status, chk);
}

template <int EPI>
__global__ void __launch_bounds__(kSwThreads, 1)
    gemm_swap_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSwStages * kSwStage);
  uint64_t* empty = full + kSwMaxStages;
  uint64_t* tfull = empty + kSwMaxStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  float* rs_sm = reinterpret_cast<float*>(smem + kSwStages * kSwStage + 256);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the MMAs)
  pdl_trigger();
  const int tc = p.tc, nc = p.nc, half = tc / 2;
  const int sst = kSwA + nc * half * kBK * 2;  // this launch's stage bytes (M = 320: 36 KB of the 48 KB maximum)
  const int nst = min(kSwMaxStages, kSwStages * kSwStage / sst);  // 5 stages at M = 320 instead of 4
  const uint32_t stage_tx = 2u * (uint32_t)sst;  // both CTAs' bytes, on the leader
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
    for (int i = 0; i < nst; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 16);  // the 8 epilogue warps of both CTAs
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, kSwTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int kb_total = p.K / kBK, splits = p.splits, kb_per = (kb_total + splits - 1) / splits;
  const int units = (p.N / 256) * splits;
  // unit -> (weight tile, split), split fastest; both CTAs of a pair walk the same units
  auto unit_of = [&](int k, int& wt, int& s, int& kb0, int& kb1) {
    const int u = (int)blockIdx.x / 2 + k * ((int)gridDim.x / 2);
    if (u >= units) return false;
    s = u % splits;
    wt = u / splits;
    kb0 = s * kb_per;
    kb1 = min(kb_total, kb0 + kb_per);
    return true;
  };
  // the first stages' weights do not depend on the previous kernel: in flight before the wait
  int pre = 0;
  if (warp == 0) {
    int wt, s, kb0, kb1;
    if (elect_one() && unit_of(0, wt, s, kb0, kb1)) {
      pre = min(nst, kb1 - kb0);
      for (int i = 0; i < pre; ++i) {
        if (rank == 0) mbar_arrive_expect_tx(&full[i], stage_tx);
        tma_load_2d_pair(smem + i * sst, &tmW, &full[i], (kb0 + i) * kBK, wt * 256 + (int)rank * kBM);
      }
    }
  }
  pdl_wait();

  if (warp == 0) {
    if (elect_one()) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      int wt, s, kb0, kb1, kbn = 0;
      for (int it = 0; unit_of(it, wt, s, kb0, kb1); ++it) {
        for (int kb = kb0; kb < kb1; ++kb, ++kbn) {
          const bool early = it == 0 && kb - kb0 < pre;
          uint8_t* sa = smem + stage * sst;
          if (!early) {
            mbar_wait(&empty[stage], phase ^ 1);
            GTRACE(0, kbn, true);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], stage_tx);
            tma_load_2d_pair(sa, &tmW, &full[stage], kb * kBK, wt * 256 + (int)rank * kBM);
          }
          for (int c = 0; c < nc; ++c)
            tma_load_2d_pair(sa + kSwA + c * half * (kBK * 2), &tmX, &full[stage], kb * kBK, c * tc + (int)rank * half);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {  // ---------------- MMA issuer (the pair's leader)
      const uint32_t idesc = idesc_bf16(2 * kBM, tc);
      int stage = 0;
      uint32_t phase = 0;
      int wt, s, kb0, kb1, kbm = 0;
      for (int it = 0; unit_of(it, wt, s, kb0, kb1); ++it) {
        mbar_wait(tempty, (it & 1) ^ 1);
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb, ++kbm) {
          mbar_wait(&full[stage], phase);
          GTRACE(1, kbm, true);
          tc_fence_after();
          const uint32_t a0 = smem_u32(smem + stage * sst), b0 = a0 + kSwA;
          for (int c = 0; c < nc; ++c) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              mma_bf16_ss_pair(tmem + (uint32_t)(c * tc), sdesc_sw128(a0 + k * 32, 16, 1024),
                               sdesc_sw128(b0 + c * half * (kBK * 2) + k * 32, 16, 1024), idesc,
                               (kb > kb0 || k > 0) ? 1u : 0u);
          }
          tc_commit_pair(&empty[stage]);
          if (++stage == nst) { stage = 0; phase ^= 1; }
        }
        tc_commit_pair(tfull);
      }
    }
  } else {  // ------------------------------- epilogue warps 2..9
    const int quarter = warp & 3, hw = (warp - 2) >> 2;
    for (int i = threadIdx.x - 64; i < kSwRs; i += 256)
      rs_sm[i] = i < p.rows_max ? (p.row_scale ? p.row_scale[i] : 1.0f) : 0.0f;
    named_bar_sync(1, 256);
    int wt, s, kb0, kb1;
    for (int it = 0; unit_of(it, wt, s, kb0, kb1); ++it) {
      mbar_wait(tfull, it & 1);
      GTRACE(2, 2 * it, warp == 2 && lane == 0);
      tc_fence_after();
      const int n = wt * 256 + (int)rank * kBM + quarter * 32 + lane;
      if constexpr (EPI == EPI_SILU)
        swap_silu_epilogue(p, tmem + ((uint32_t)(quarter * 32) << 16), n, p.rows_max, lane, hw, rs_sm,
                           reinterpret_cast<uint8_t*>(rs_sm + kSwRs) + (warp - 2) * 1024);
      else
        swap_epilogue<EPI>(p, tmem + ((uint32_t)(quarter * 32) << 16), n, p.rows_max, s, lane, hw, rs_sm);
      GTRACE(2, 2 * it + 1, warp == 2 && lane == 0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty, 0);
    }
  }
  tc_fence_before();
  cluster_sync();  // neither CTA leaves while its peer may still signal its barriers
  if (warp == 1) tmem_dealloc_pair(tmem, kSwTmemCols);
}

// Split-K reduction + residual epilogue (EPI_PART partials): one CTA per row,
// h[row] += sum_s part[s][row] in split order (deterministic); with the fused
// RMSNorm the bf16 row copy and 1/rms come out of the same pass.
// one row of splitk_reduce_add_kernel
__device__ __forceinline__ void splitk_reduce_row(const GemmArgs& p, int splits, int row) {
  const int n4 = p.N / 4;
  float ss = 0.f;
  float4* h = reinterpret_cast<float4*>(p.out_f32 + (size_t)row * p.ld_out);
  for (int c = threadIdx.x; c < n4; c += blockDim.x) {
    float4 acc;
    if (splits <= 8) {  // all partials in flight at once, then summed in split order
      float4 v[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < splits) v[s] = __ldcg(reinterpret_cast<const float4*>(p.ws_part + ((size_t)s * p.rows_max + row) * p.N) + c);
      acc = v[0];
#pragma unroll
      for (int s = 1; s < 8; ++s)
        if (s < splits) {
          acc.x += v[s].x; acc.y += v[s].y; acc.z += v[s].z; acc.w += v[s].w;
        }
    } else {  // (the fp32-TC mode's up to 16 K chunks) 8 at a time, in split order
      acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s0 = 0; s0 < splits; s0 += 8) {
        float4 v[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s0 + s < splits)
            v[s] = __ldcg(reinterpret_cast<const float4*>(p.ws_part + ((size_t)(s0 + s) * p.rows_max + row) * p.N) + c);
        if (s0 == 0) acc = v[0];
        else { acc.x += v[0].x; acc.y += v[0].y; acc.z += v[0].z; acc.w += v[0].w; }
#pragma unroll
        for (int s = 1; s < 8; ++s)
          if (s0 + s < splits) {
            acc.x += v[s].x; acc.y += v[s].y; acc.z += v[s].z; acc.w += v[s].w;
          }
      }
    }
    flag_nonfinite(p.status, finite_acc(finite_acc(finite_acc(finite_acc(0.f, acc.x), acc.y), acc.z), acc.w));
    float4 x = h[c];
    x.x += acc.x; x.y += acc.y; x.z += acc.z; x.w += acc.w;
    h[c] = x;
    if (p.norm_bf16) {
      ss += x.x * x.x + x.y * x.y + x.z * x.z + x.w * x.w;
      reinterpret_cast<uint2*>(p.norm_bf16 + (size_t)row * p.N)[c] = make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
    }
  }
  if (p.norm_inv) {
    __shared__ float red[32];
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

__global__ void __launch_bounds__(256) splitk_reduce_add_kernel(const GemmArgs p, int splits) {
  pdl_trigger();
  pdl_wait();
  const int M = p.rows_dev ? *p.rows_dev : p.rows_max;
  for (int row = blockIdx.x; row < M; row += gridDim.x) splitk_reduce_row(p, splits, row);
}

// ---------------------------------------------------------------------------
// M = 1 (the top layer's last row, the logits head): the GEMM is a weight
// stream, so it runs on the CUDA cores as a GEMV at HBM speed instead of as
// one mostly-empty 128-row tensor-core tile per N tile. The activation row is
// staged in shared memory; each warp streams kGvRows weight rows with 16-byte
// loads (kGvUnroll k-chunks of every row in flight), fp32 accumulation, and the
// same epilogues: residual add, SiLU(gate)*up pairs, fp32 store.
// ---------------------------------------------------------------------------
constexpr int kGvWarps = 8;

__device__ __forceinline__ float dot8(uint4 w, uint4 a) {
  const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&w);
  const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 wf = __bfloat1622float2(w2[i]), af = __bfloat1622float2(a2[i]);
    s = fmaf(wf.x, af.x, s);
    s = fmaf(wf.y, af.y, s);
  }
  return s;
}

// Store R consecutive outputs n0.. of the single row (R even: SiLU pairs and
// RoPE pairs stay together) with the GEMM's epilogue semantics.
template <int EPI, int R>
__device__ __forceinline__ void gemv_store(const GemmArgs& p, int n0, const float (&v)[R], float rs) {
  float chk = 0.f;
#pragma unroll
  for (int r = 0; r < R; ++r) chk = finite_acc(chk, v[r] * rs);
  flag_nonfinite(p.status, chk);
  if constexpr (EPI == EPI_SILU) {  // rows (2j, 2j+1) = (gate j, up j)
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const float g = v[r] * rs, u = v[r + 1] * rs;
      p.out_bf16[(n0 + r) / 2] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * u);
    }
  } else if constexpr (EPI == EPI_ADD) {
#pragma unroll
    for (int r = 0; r < R; ++r) p.out_f32[n0 + r] += v[r] * rs;
  } else if constexpr (EPI == EPI_QKV) {  // RoPE on Q/K, K/V rows into the context at the row's position
    const int pos = p.pos[0], q = p.q, kv = p.kv, dh = p.dh;
#pragma unroll
    for (int r = 0; r < R; r += 2) {
      const int col = n0 + r;
      const float x0 = v[r] * rs, x1 = v[r + 1] * rs;
      const __nv_bfloat162 raw = __floats2bfloat162_rn(x0, x1);
      if (col >= q + kv) {
        const int c = col - q - kv;
        if (p.cap_v) *reinterpret_cast<__nv_bfloat162*>(p.cap_v + c) = raw;
        __nv_bfloat16* base = p.commit ? p.ctx_v + (size_t)pos * kv : p.self_v;
        *reinterpret_cast<__nv_bfloat162*>(base + c) = raw;
        continue;
      }
      const bool is_k = col >= q;
      const int c = is_k ? col - q : col;
      if (is_k && p.cap_k) *reinterpret_cast<__nv_bfloat162*>(p.cap_k + c) = raw;
      const float2 t = p.rope[(size_t)pos * (dh / 2) + (c % dh) / 2];
      const __nv_bfloat162 rot = __floats2bfloat162_rn(x0 * t.x - x1 * t.y, x0 * t.y + x1 * t.x);
      __nv_bfloat16* base = !is_k ? p.out_bf16 : (p.commit ? p.ctx_k + (size_t)pos * kv : p.self_k);
      *reinterpret_cast<__nv_bfloat162*>(base + c) = rot;
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) p.out_f32[n0 + r] = v[r] * rs;
  }
}

// EPI_ADD with the fused RMSNorm: the last block to finish turns the new
// residual row into its bf16 copy and 1/rms (norm_cnt[0] is the ticket).
template <int EPI>
__device__ __forceinline__ void gemv_norm_finish(const GemmArgs& p) {
  if constexpr (EPI == EPI_ADD) {
    if (!p.norm_bf16 || !p.norm_inv || !p.norm_cnt) return;
    __shared__ int last;
    __shared__ float red[kGvWarps];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(p.norm_cnt, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    float ss = 0.f;
    for (int i = threadIdx.x; i < p.N; i += blockDim.x) {
      const float x = __ldcg(p.out_f32 + i);
      ss = fmaf(x, x, ss);
      p.norm_bf16[i] = __float2bfloat16_rn(x);
    }
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.f;
      for (int w = 0; w < kGvWarps; ++w) t += red[w];
      p.norm_inv[0] = rsqrtf(t / (float)p.N + p.norm_eps);
      p.norm_cnt[0] = 0;
    }
  }
}

// kGvRows weight rows per warp, kGvUnroll k-chunks of each in flight: 4 x 2 for
// wide N, 2 x 4 when N/32 warps would leave SMs idle (kGvRows even: SiLU pairs)
template <int EPI, int kGvRows, int kGvUnroll>
__global__ void __launch_bounds__(kGvWarps * 32) gemv_bf16_kernel(const __nv_bfloat16* __restrict__ a,
                                                                  const __nv_bfloat16* __restrict__ B, GemmArgs p) {
  extern __shared__ uint4 a_sm[];  // the activation row, K bf16
  pdl_trigger();
  pdl_wait();
  const int K = p.K, k8 = K / 8;
  for (int i = threadIdx.x; i < k8; i += blockDim.x) a_sm[i] = reinterpret_cast<const uint4*>(a)[i];
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float rs = p.row_scale ? p.row_scale[0] : 1.0f;
  for (int n0 = (blockIdx.x * kGvWarps + warp) * kGvRows; n0 < p.N; n0 += gridDim.x * kGvWarps * kGvRows) {
    float acc[kGvRows];
#pragma unroll
    for (int r = 0; r < kGvRows; ++r) acc[r] = 0.f;
    const uint4* w4 = reinterpret_cast<const uint4*>(B + (size_t)n0 * K);
    for (int c = lane; c < k8; c += 32 * kGvUnroll) {
      uint4 wv[kGvUnroll][kGvRows], av[kGvUnroll];
#pragma unroll
      for (int u = 0; u < kGvUnroll; ++u) {
        const int cc = c + 32 * u;
        if (cc < k8) {
          av[u] = a_sm[cc];
#pragma unroll
          for (int r = 0; r < kGvRows; ++r) wv[u][r] = __ldcs(w4 + (size_t)r * k8 + cc);  // streamed once
        }
      }
#pragma unroll
      for (int u = 0; u < kGvUnroll; ++u)
        if (c + 32 * u < k8) {
#pragma unroll
          for (int r = 0; r < kGvRows; ++r) acc[r] += dot8(wv[u][r], av[u]);
        }
    }
#pragma unroll
    for (int r = 0; r < kGvRows; ++r)
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    if (lane == 0) gemv_store<EPI, kGvRows>(p, n0, acc, rs);
  }
  gemv_norm_finish<EPI>(p);
}

// Narrow N (few weight rows, long K): a whole block shares R rows, its 8 warps
// splitting K, so the weight stream still spreads over every SM.
template <int EPI, int R>
__global__ void __launch_bounds__(kGvWarps * 32) gemv_bf16_ksplit_kernel(const __nv_bfloat16* __restrict__ a,
                                                                         const __nv_bfloat16* __restrict__ B,
                                                                         GemmArgs p) {
  extern __shared__ uint4 a_sm[];
  __shared__ float red[kGvWarps][R];
  pdl_trigger();
  pdl_wait();
  const int K = p.K, k8 = K / 8;
  for (int i = threadIdx.x; i < k8; i += blockDim.x) a_sm[i] = reinterpret_cast<const uint4*>(a)[i];
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const float rs = p.row_scale ? p.row_scale[0] : 1.0f;
  constexpr int U = 4;
  for (int n0 = blockIdx.x * R; n0 < p.N; n0 += gridDim.x * R) {
    float acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.f;
    const uint4* w4 = reinterpret_cast<const uint4*>(B + (size_t)n0 * K);
    for (int c = threadIdx.x; c < k8; c += blockDim.x * U) {
      uint4 wv[U][R], av[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int cc = c + blockDim.x * u;
        if (cc < k8) {
          av[u] = a_sm[cc];
#pragma unroll
          for (int r = 0; r < R; ++r) wv[u][r] = __ldcs(w4 + (size_t)r * k8 + cc);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c + blockDim.x * u < k8) {
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] += dot8(wv[u][r], av[u]);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int o = 16; o; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
      if (lane == 0) red[warp][r] = acc[r];
    }
    __syncthreads();
    if (threadIdx.x < R) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < kGvWarps; ++w) t += red[w][threadIdx.x];
      red[0][threadIdx.x] = t;  // (each thread reads its own column before writing row 0 of it)
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = red[0][r];
      gemv_store<EPI, R>(p, n0, v, rs);
    }
    __syncthreads();
  }
  gemv_norm_finish<EPI>(p);
}

// The fused RMSNorm of a residual GEMM for one row: bf16 copy + 1/rms.
__global__ void __launch_bounds__(256) row_norm_kernel(const float* __restrict__ h, int d, float eps,
                                                       __nv_bfloat16* __restrict__ out, float* __restrict__ inv) {
  __shared__ float red[8];
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float x = h[i];
    ss = fmaf(x, x, ss);
    out[i] = __float2bfloat16_rn(x);
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    inv[0] = rsqrtf(t / (float)d + eps);
  }
}

}  // namespace

// Programmatic dependent launch on for the hot kernels (RK_PDL=0 turns it off).
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("RK_PDL");
    return v ? std::atoi(v) != 0 : true;
  }();
  return on;
}

namespace {

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  RK_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <int BN, int EPI, int PAIR, bool TF32 = false>
void launch(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p, int grid) {
  using C = Cfg<BN, PAIR>;
  static bool attr = false;
  if (!attr) {
    RK_CUDA(cudaFuncSetAttribute(gemm_bf16_kernel<BN, EPI, PAIR, TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM));
    attr = true;
  }
  if constexpr (PAIR == 1) {
    launch_pdl(gemm_bf16_kernel<BN, EPI, 1, TF32>, dim3(grid), dim3(kThreads), C::SMEM, st, a, b, p);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    RK_CUDA(cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<BN, EPI, 2, TF32>, a, b, p));
  }
}

template <int EPI, bool TF32>
void launch_tiles(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p, int grid) {
  if (p.pair == 2) {
    if (p.bn == 256) launch<256, EPI, 2, TF32>(st, a, b, p, grid);
    else if (p.bn == 192) launch<192, EPI, 2, TF32>(st, a, b, p, grid);
    else if (p.bn == 128) launch<128, EPI, 2, TF32>(st, a, b, p, grid);
    else launch<64, EPI, 2, TF32>(st, a, b, p, grid);
  } else {
    if (p.bn == 256) launch<256, EPI, 1, TF32>(st, a, b, p, grid);
    else if (p.bn == 128) launch<128, EPI, 1, TF32>(st, a, b, p, grid);
    else launch<64, EPI, 1, TF32>(st, a, b, p, grid);
  }
}

template <int EPI>
void launch_bn(cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& p, int grid) {
  if constexpr (EPI == EPI_ADD || EPI == EPI_F32 || EPI == EPI_PART) {
    if (p.tf32) {  // 3xTF32 mode (kind::tf32)
      launch_tiles<EPI, true>(st, a, b, p, grid);
      return;
    }
  }
  launch_tiles<EPI, false>(st, a, b, p, grid);
}

// CTA pairs the GPU can hold at once (a GPC's odd SM cannot host a pair).
int pair_slots(int sm_count) {
  static int slots = -1;
  if (slots < 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * sm_count);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg<256, 2>::SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    RK_CUDA(cudaFuncSetAttribute(gemm_bf16_kernel<256, EPI_F32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg<256, 2>::SMEM));
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_bf16_kernel<256, EPI_F32, 2>, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 0;
    }
    slots = n;
  }
  return slots;
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

// Pick the kernel shape for one GEMM with a small cost model calibrated on
// B200 (time per k-block of one unit, by the bytes a CTA stages per k-block:
// ~0.0096 us per KB, the L2->SM feed; 1-CTA 128x256 tile = 48 KB = 0.46 us,
// pair = 0.42 us) times the rounds of units over the concurrent slots:
//  - 1-CTA 128xBN tiles (the widest BN that still fills the SMs), or
//  - CTA pairs (256-row tiles), when M >= 640 and the rounds allow, or
//  - m-grouped tiles (MT = 2/3 m tiles per CTA, BN 128) for short M, or
//  - for residual GEMMs that cannot fill the GPU, split-K over any of the
//    1-CTA shapes: EPI_PART partials reduced in split order by
//    splitk_reduce_add_kernel (+ ~3 us and 2*s*M*N*4 B at ~8 TB/s), or the
//    opt-in cluster (DSMEM) reduction / stream-K.
static double choose_config(GemmArgs& p, int sm_count, int rows_hint) {
  auto env = [](const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
  };
  static const int pair_env = env("RK_GEMM_PAIR", 1), dbg_env = env("RK_GEMM_DBG", 0);
  p.dbg = dbg_env;
  p.sms = sm_count;
  p.splits = 1;
  p.pair = 1;
  const int kb = p.K / kBK;
  auto ceil_div = [](long long a, long long b) { return (int)((a + b - 1) / b); };
  // us per k-block of one unit: the staged bytes at the L2->SM feed rate.
  // (RK_GEMM_TKB_FLOOR_NS=450 floors it at a k-block round trip -- closer for
  // narrow tiles, but the extra split-K it then picks measured slower on c2.)
  static const double t_floor = env("RK_GEMM_TKB_FLOOR_NS", 0) * 1e-3;
  // (r02s recalibration on the c2 step: 1-CTA 128x256 ~0.50 us per k-block,
  // CTA pair 256x256 ~0.39 us -- the pair also wins the dynamic-row sparse
  // gate/up and W_down GEMMs, where the old 0.46 / 0.425 picked 1-CTA tiles)
  auto t_kb = [](int a_kb, int b_kb) { return std::max(t_floor, 0.0104 * (a_kb + b_kb)); };
  constexpr double kPairKb = 0.39;  // us per k-block of a 256 x 256 pair unit

  // 1-CTA (or pair) tiles, BN by the fill rule
  const int pslots = pair_env ? pair_slots(sm_count) : 0;
  if (pslots > 0 && rows_hint > kBM) {
    auto rounds = [&](int tm, int slots_) {
      int best = 1 << 30;
      for (int cand : {256, 128})
        if (p.N % cand == 0)
          best = std::min(best, ceil_div((long long)ceil_div(rows_hint, tm) * (p.N / cand), slots_) * (cand / 128));
      return best;
    };
    const double single = rounds(kBM, sm_count) * t_kb(16, 32), pair = rounds(2 * kBM, pslots) * kPairKb;
    if (pair_env == 2 || (rows_hint >= 640 && pair <= single)) p.pair = 2;
  }
  const int slots = p.pair == 2 ? pslots : sm_count;
  const int num_m = ceil_div(rows_hint, kBM * p.pair);
  int bn = 64;
  if (p.pair == 2) {
    // pair tiles: the BN with the fewest unit-rounds x width; on a tie the
    // wider tile (fewer, longer units), except the QKV epilogue (RoPE + K/V
    // scatter) of the sparse passes, whose exposed last epilogue favours two
    // narrower rounds (measured r02s: sparse W_o 256 wins, sparse QKV 128)
    // (192: a ragged last N tile, e.g. N = 2048 = 10 x 192 + 128, when whole
    // 256-column tiles leave a third of the pair slots idle -- c2 sparse W_down:
    // 48 pair units on 74 slots)
    double bc = 1e30;
    for (int cand : {256, 192, 128, 64}) {
      if (cand != 192 && p.N % cand) continue;
      if (cand == 192 && (p.N % 32 || p.N <= 192)) continue;
      const double c = (double)ceil_div((long long)num_m * ceil_div(p.N, cand), slots) *
                       std::max(kPairKb * cand / 256.0, t_kb(16, cand / 16));
      if (c < bc || (c == bc && p.epi == EPI_QKV && p.rows_dev && cand >= 128)) { bc = c; bn = cand; }
    }
  } else {
    for (int cand : {256, 128}) {
      if (p.N % cand == 0 && num_m * (p.N / cand) >= slots) { bn = cand; break; }
    }
  }
  if (p.N % bn && bn != 192) raise(RK_ERR_INVALID_ARGUMENT, "bf16 GEMM needs N % 64 == 0");
  p.bn = bn;
  double best = (double)ceil_div((long long)num_m * ceil_div(p.N, bn), slots) * kb *
                (p.pair == 2 ? std::max(kPairKb * bn / 256.0, t_kb(16, bn / 16)) : t_kb(16, bn / 8));

  const bool residual_split = p.epi == EPI_ADD && p.split_flags;
  auto part_cost = [&](int s) { return s > 1 ? 3.0 + 2.0 * s * (double)rows_hint * p.N * 4 / 8e6 : 0.0; };
  auto split_ok = [&](int s) { return kb / s >= 4 && (s - 1) * ((kb + s - 1) / s) < kb; };
  int pick_bn = -1, pick_splits = 1;
  // split-K over 1-CTA 128 x wide tiles
  if (residual_split) {
    const int wide = p.N % 256 == 0 ? 256 : (p.N % 128 == 0 ? 128 : 64);
    const int tiles1 = ceil_div(rows_hint, kBM) * (p.N / wide);
    const double t1 = t_kb(16, wide / 8);
    for (int sp = 2; sp <= 8; ++sp) {
      if (!split_ok(sp)) continue;
      const double c = (double)ceil_div((long long)tiles1 * sp, sm_count) * ((kb + sp - 1) / sp) * t1 + part_cost(sp);
      if (c < best) { best = c; pick_bn = wide; pick_splits = sp; }
    }
  }
  if (pick_bn > 0) {
    p.pair = 1;
    p.bn = pick_bn;
    p.splits = pick_splits;
    p.epi = EPI_PART;
  }
  return best;
}

// Swap-AB pair (gemm_swap_kernel) for a short static M. Measured (r02g,
// weights streamed from HBM): it wins for the wide SiLU GEMMs of the
// prefix/suffix-only layers -- c2 gate/up M=320 N=16384 30.1 -> 25.2 us, c3
// N=28672 84.6 -> 77.0 us -- where the 1-CTA kernel needs two rounds of
// 128 x 256 tiles and re-reads every weight tile per m tile; it loses on the
// narrow QKV / W_o / down GEMMs (too few 256-row weight tiles to fill the
// SMs, and its single-unit epilogue is exposed). RK_GEMM_SWAP: 0 never,
// 1 (default) wide SiLU GEMMs with 128 < M <= 512, 2 every eligible GEMM
// (tests; residual GEMMs then write split-K partials).
static bool choose_swap(GemmArgs& p, int sm_count, double other_us) {
  static const int swap_env = [] {
    const char* v = std::getenv("RK_GEMM_SWAP");
    return v ? std::atoi(v) : 1;
  }();
  const int M = p.rows_max;
  if (!swap_env || p.rows_dev || M < 2 || M > 512 || p.N % 256 || p.K % kBK) return false;
  if (!(p.epi == EPI_QKV || p.epi == EPI_SILU || p.epi == EPI_F32 || p.epi == EPI_ADD)) return false;
  if (p.epi == EPI_QKV && (p.q % 32 || p.kv % 32)) return false;
  const int pslots = pair_slots(sm_count);
  if (pslots <= 0) return false;
  const int nc = M <= 256 ? 1 : 2;
  const int tc = ((M + nc - 1) / nc + 15) / 16 * 16;
  const int kb = p.K / kBK, tiles = p.N / 256;
  if (swap_env != 2 && !(p.epi == EPI_SILU && M > kBM && 2 * tiles >= pslots)) return false;
  (void)other_us;
  const double t_kb = std::max(0.0096 * (16.0 + nc * tc / 16.0), 2.0 * nc * tc / 1900.0);
  double best = 1e30;
  int best_s = 1;
  for (int s = 1; s <= (p.epi == EPI_ADD ? 8 : 1); ++s) {  // (splitk_reduce_add_kernel: <= 8 partials)
    if (s > 1 && (kb / s < 2 || (s - 1) * ((kb + s - 1) / s) >= kb)) continue;
    const int units = tiles * s;
    double c = (double)((units + pslots - 1) / pslots) * ((kb + s - 1) / s) * t_kb + 1.0;
    if (p.epi == EPI_ADD) c += 3.0 + 2.0 * s * (double)M * p.N * 4 / 8e6;  // partials + reduce kernel
    if (c < best) { best = c; best_s = s; }
  }
  p.swap = 1;
  p.nc = nc;
  p.tc = tc;
  p.pair = 2;
  p.splits = best_s;
  p.bn = 256;
  if (p.epi == EPI_ADD) p.epi = EPI_PART;
  return true;
}

void gemm_bf16(rk_engine* e, const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, GemmArgs p,
               int rows_hint) {
  if (p.rows_max <= 0) return;
  if (p.K % kBK) raise(RK_ERR_INVALID_ARGUMENT, "bf16 GEMM needs K % 64 == 0");
  if (!p.status) p.status = e->status.as<int>();
  static const bool gemv_env = [] {
    const char* v = std::getenv("RK_GEMV");
    return v ? std::atoi(v) != 0 : true;
  }();
  if (p.tf32 && p.epi != EPI_ADD && p.epi != EPI_F32) raise(RK_ERR_INVALID_ARGUMENT, "tf32 GEMM: ADD / F32 epilogues");
  if (gemv_env && !p.tf32 && p.rows_max == 1 && !p.rows_dev &&
      (p.epi == EPI_ADD || p.epi == EPI_SILU || p.epi == EPI_F32 || p.epi == EPI_QKV) && p.N % 4 == 0) {
    const size_t smem = (size_t)p.K * 2;
    const bool narrow = p.N / (kGvWarps * 4) < 2 * e->sm_count;
    const int per_block = kGvWarps * (narrow ? 2 : 4);
    const int blocks = std::min((p.N + per_block - 1) / per_block, 16 * e->sm_count);
    ProfScope ps(e, (e->prof && e->prof->on)
                        ? intern(std::string("gemv_n") + std::to_string(p.N) + "_k" + std::to_string(p.K))
                        : "gemv",
                 0, 2.0 * p.N * p.K);  // the weight stream
    ps.rec.kind = 1;
    ps.rec.rows_max = 1;
    ps.rec.N = p.N;
    ps.rec.K = p.K;
    auto go = [&](auto kern) {
      if (smem > 48 * 1024) RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      launch_pdl(kern, dim3(blocks), dim3(kGvWarps * 32), smem, e->stream, A, B, p);
    };
    if (narrow) {  // a block per 2 rows, K split over its warps
      const int nb = std::min(p.N / 2, 16 * e->sm_count);
      auto go2 = [&](auto kern) {
        if (smem > 48 * 1024) RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        launch_pdl(kern, dim3(nb), dim3(kGvWarps * 32), smem, e->stream, A, B, p);
      };
      if (p.epi == EPI_ADD) go2(gemv_bf16_ksplit_kernel<EPI_ADD, 2>);
      else if (p.epi == EPI_SILU) go2(gemv_bf16_ksplit_kernel<EPI_SILU, 2>);
      else if (p.epi == EPI_QKV) go2(gemv_bf16_ksplit_kernel<EPI_QKV, 2>);
      else go2(gemv_bf16_ksplit_kernel<EPI_F32, 2>);
    } else {
      if (p.epi == EPI_ADD) go(gemv_bf16_kernel<EPI_ADD, 4, 2>);
      else if (p.epi == EPI_SILU) go(gemv_bf16_kernel<EPI_SILU, 4, 2>);
      else if (p.epi == EPI_QKV) go(gemv_bf16_kernel<EPI_QKV, 4, 2>);
      else go(gemv_bf16_kernel<EPI_F32, 4, 2>);
    }
    e->launches += 1;
    if (p.epi == EPI_ADD && p.norm_bf16 && p.norm_inv && !p.norm_cnt) {  // (no ticket: separate pass)
      row_norm_kernel<<<1, 256, 0, e->stream>>>(p.out_f32, p.N, p.norm_eps, p.norm_bf16, p.norm_inv);
      e->launches += 1;
    }
    return;
  }
  {
    const int epi0 = p.epi;
    GemmArgs alt = p;
    const double other = choose_config(alt, e->sm_count, rows_hint > 0 ? rows_hint : p.rows_max);
    if (p.tf32 || !choose_swap(p, e->sm_count, other)) p = alt;
    p.dbg = alt.dbg;
    if (p.tf32) {
      // The tensor core's fp32 accumulation loses ~3.6e-9 (relative, measured)
      // per accumulated element of K, linearly in K (r02v: rel-L2 6e-6 at a
      // 3K of 1536, 8.7e-5 at 24576). So the 3K-long dot products are cut into
      // chunks of <= 48 k-blocks (1536 fp32) accumulated in TMEM, written as
      // split-K partials and summed on the CUDA cores (RN, split order).
      p.epi = epi0;
      const int kb = p.K / kBK;
      int sp = std::min(16, (kb + 47) / 48);
      while (sp > 1 && (sp - 1) * ((kb + sp - 1) / sp) >= kb) --sp;
      p.splits = sp;
      if (sp > 1) {
        p.pair = 1;  // (1-CTA tiles are 256 / 128 / 64 wide; a 192 pair pick maps to the widest that divides N)
        if (p.bn != 256 && p.bn != 128 && p.bn != 64) p.bn = 256;
        while (p.bn > 64 && p.N % p.bn) p.bn /= 2;
        if (epi0 == EPI_F32)  // the reduce adds into the output: start from zero
          RK_CUDA(cudaMemset2DAsync(p.out_f32, (size_t)p.ld_out * 4, 0, (size_t)p.N * 4, p.rows_max, e->stream));
        p.epi = EPI_PART;
      } else {
        p.splits = 1;
      }
    }
    // sweep hook: RK_GEMM_OVERRIDE="M[d]:N:K=bn/pair/splits;..." (d: live rows
    // on the device) forces one shape's tile config (tools/gemm_override_sweep.py)
    struct Ovr {
      int M, dyn, N, K, bn, pair, splits;
    };
    static const std::vector<Ovr> ovr = [] {
      std::vector<Ovr> v;
      const char* s = std::getenv("RK_GEMM_OVERRIDE");
      while (s && *s) {
        Ovr o{};
        char d = 0;
        int n = 0;
        if (std::sscanf(s, "%d%c", &o.M, &d) == 2 && d == 'd') {
          o.dyn = 1;
          std::sscanf(s, "%*dd:%d:%d=%d/%d/%d%n", &o.N, &o.K, &o.bn, &o.pair, &o.splits, &n);
        } else {
          std::sscanf(s, "%*d:%d:%d=%d/%d/%d%n", &o.N, &o.K, &o.bn, &o.pair, &o.splits, &n);
        }
        if (n > 0) v.push_back(o);
        s = std::strchr(s, ';');
        if (s) ++s;
      }
      return v;
    }();
    for (const Ovr& o : ovr) {
      if (o.M == p.rows_max && o.dyn == (p.rows_dev != nullptr) && o.N == p.N && o.K == p.K) {
        p = alt;
        p.swap = 0;
        p.bn = o.bn;
        p.pair = o.pair;
        p.splits = (epi0 == EPI_ADD || epi0 == EPI_PART) ? o.splits : 1;
        p.epi = (o.splits > 1 && (epi0 == EPI_ADD || epi0 == EPI_PART)) ? EPI_PART : epi0;
      }
    }
  }
  static const bool log = std::getenv("RK_GEMM_LOG") != nullptr;
  if (p.swap) {
    if (log)
      std::fprintf(stderr, "[gemm] M=%d N=%d K=%d epi=%d -> swap nc=%d tc=%d splits=%d\n", p.rows_max, p.N, p.K, p.epi,
                   p.nc, p.tc, p.splits);
    CUtensorMap tw, tx;
    make_tmap_bf16(&tw, B, (uint64_t)p.N, (uint64_t)p.K, kBM, (uint64_t)p.K);
    make_tmap_bf16(&tx, A, (uint64_t)p.rows_max, (uint64_t)p.K, (uint32_t)(p.tc / 2), (uint64_t)lda);
    const int units = (p.N / 256) * p.splits;
    const int grid = 2 * std::min(units, pair_slots(e->sm_count));
    if (p.epi == EPI_PART) {
      e->scratch->gemm_ws.ensure((size_t)p.splits * p.rows_max * p.N * 4);
      p.ws_part = e->scratch->gemm_ws.as<float>();
    }
    static const char* kEpiS[] = {"qkv", "add", "silu", "f32", "addsplit"};
    ProfScope ps(e, (e->prof && e->prof->on)
                        ? intern(std::string("gemm_") + kEpiS[p.epi] + "_m" + std::to_string(p.rows_max) + "_n" +
                                 std::to_string(p.N) + "_k" + std::to_string(p.K) + "_swap_s" + std::to_string(p.splits))
                        : "gemm",
                 0, 0);
    ps.rec.kind = 1;
    ps.rec.rows_dev = nullptr;
    ps.rec.rows_max = p.rows_max;
    ps.rec.N = p.N;
    ps.rec.K = p.K;
    static bool attr_done[5] = {false, false, false, false, false};
    auto go = [&](auto kern) {
      if (!attr_done[p.epi]) {
        RK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSwSmem));
        attr_done[p.epi] = true;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(kSwThreads);
      cfg.dynamicSmemBytes = kSwSmem;
      cfg.stream = e->stream;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl_enabled() ? 2 : 1;
      RK_CUDA(cudaLaunchKernelEx(&cfg, kern, tw, tx, p));
    };
    switch (p.epi) {
      case EPI_QKV: go(gemm_swap_kernel<EPI_QKV>); break;
      case EPI_SILU: go(gemm_swap_kernel<EPI_SILU>); break;
      case EPI_PART:
        go(gemm_swap_kernel<EPI_PART>);
        launch_pdl(splitk_reduce_add_kernel, dim3(std::min(p.rows_max, 8 * e->sm_count)), dim3(256), 0, e->stream, p,
                   (int)p.splits);
        e->launches += 1;
        break;
      default: go(gemm_swap_kernel<EPI_F32>); break;
    }
    e->launches += 1;
    return;
  }
  if (log)
    std::fprintf(stderr, "[gemm] M=%d%s N=%d K=%d epi=%d -> bn=%d pair=%d splits=%d tf32=%d\n", p.rows_max,
                 p.rows_dev ? "(dyn)" : "", p.N, p.K, p.epi, p.bn, p.pair, p.splits, p.tf32);
  if (p.norm_part && p.N / p.bn > kNormSlots) raise(RK_ERR_INVALID_ARGUMENT, "fused RMSNorm: too many N tiles");
  CUtensorMap ta, tb;
  make_tmap_bf16(&ta, A, (uint64_t)p.rows_max, (uint64_t)p.K, kBM, (uint64_t)lda);
  make_tmap_bf16(&tb, B, (uint64_t)p.N, (uint64_t)p.K, (uint32_t)(p.bn / p.pair), (uint64_t)p.K);
  const int num_m = (p.rows_max + kBM * p.pair - 1) / (kBM * p.pair);
  const int total = num_m * ((p.N + p.bn - 1) / p.bn) * p.splits;  // units (pair units for the pair kernel)
  p.m_hint = p.rows_dev && rows_hint > 0 ? (rows_hint + kBM * p.pair - 1) / (kBM * p.pair) : 0;
  const int slots = p.pair == 2 ? pair_slots(e->sm_count) : e->sm_count;
  const int grid = p.pair * (total < slots ? total : slots);
  if (p.epi == EPI_PART) {
    e->scratch->gemm_ws.ensure((size_t)p.splits * p.rows_max * p.N * 4);
    p.ws_part = e->scratch->gemm_ws.as<float>();
  }
  static const char* kEpi[] = {"qkv", "add", "silu", "f32", "addsplit"};
  ProfScope ps(e, (e->prof && e->prof->on)
                      ? intern(std::string("gemm_") + kEpi[p.epi] + "_m" + std::to_string(p.rows_max) +
                               (p.rows_dev ? "dyn" : "") + "_n" + std::to_string(p.N) + "_k" + std::to_string(p.K) +
                               "_bn" + std::to_string(p.bn) + "_s" + std::to_string(p.splits) +
                               (p.pair == 2 ? "_pair" : "") + (p.tf32 ? "_tf32" : ""))
                      : "gemm",
               0, 0);
  ps.rec.kind = 1;
  ps.rec.rows_dev = p.rows_dev;
  ps.rec.rows_max = rows_hint > 0 && !p.rows_dev ? p.rows_max : p.rows_max;
  ps.rec.N = p.N;
  ps.rec.K = p.K;
  switch (p.epi) {
    case EPI_QKV: launch_bn<EPI_QKV>(e->stream, ta, tb, p, grid); break;
    case EPI_ADD:  // (unsplit: split-K residual GEMMs run as EPI_PART + splitk_reduce_add_kernel)
      if (p.splits != 1) raise(RK_ERR_LOGIC, "residual GEMM epilogue with split-K");
      launch_bn<EPI_ADD>(e->stream, ta, tb, p, grid);
      break;
    case EPI_SILU: launch_bn<EPI_SILU>(e->stream, ta, tb, p, grid); break;
    case EPI_PART:  // partials, then splitk_reduce_add_kernel sums them in split order
      launch_bn<EPI_PART>(e->stream, ta, tb, p, grid);
      launch_pdl(splitk_reduce_add_kernel, dim3(std::min(p.rows_max, 8 * e->sm_count)), dim3(256), 0, e->stream, p,
                 (int)p.splits);
      e->launches += 1;
      break;
    default: launch_bn<EPI_F32>(e->stream, ta, tb, p, grid); break;
  }
  e->launches += 1;
}

}  // namespace rk
