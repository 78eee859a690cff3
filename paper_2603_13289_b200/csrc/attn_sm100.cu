// attn_sm100.cu -- K4: causal GQA attention for the recomputed rows over the
// mixed (reused + recomputed) KV context, on tcgen05 tensor cores.
//
// Reference semantics: attend_row (model.cpp:170-204) -- query row r at
// absolute position pos_r sees context keys 0..pos_r of its layer, softmax
// over scores scaled by 1/sqrt(d_head), kv head = h / (H / H_kv). Rows may be
// any ascending subset of positions (dense band or gathered sparse rows), so
// the causal limit is per row, by absolute position.
//
// One CTA = one query tile (128 rows) x one head, flash-style over 128-key
// tiles (64-key tiles at d_head 128); two CTAs per SM (112 KB smem, 256 TMEM columns each),
// so one CTA's exponentials overlap the other's MMAs, loads and epilogue.
//   warp 4      TMA: K_j into a 2-stage ring
//   warp 6      TMA: Q once, V_j into a 2-stage ring
//   warp 5      TMEM alloc + MMA issue: S(j+1) = Q K_{j+1}^T -> TMEM as soon
//               as the softmax has pulled S(j) into registers, then
//               O += P(j) V_j -> TMEM (accumulated across key tiles)
//   warps 0-3   softmax, one row per thread: S into registers (TMEM freed at
//               once), scale + causal mask, row max, lazy rescale of O in TMEM
//               only when the max grows by more than 2^8, P = exp2(.) (MUFU +
//               a cubic on the FMA pipe for a quarter of the columns) as bf16
//               into swizzled smem, row sum l in registers.
// Query tiles never straddle a row group (prefix / suffix / segment rows of
// the fused schedule), and each tile stops at its own last key tile.
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

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a pair on the FMA pipe (FADD2/FFMA2): round-to-nearest split
// x = n + f (f in [-0.5, 0.5]), minimax cubic for 2^f (max rel. err 7.5e-5,
// far below bf16's 2^-9), n added straight into the exponent bits. Valid for
// x <= 64; x is clamped at -125 so p * 2^n stays a normal float.
__device__ __forceinline__ void poly_exp2_pair(float x0, float x1, float& e0, float& e1) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: integer part lands in the low mantissa bits
  x0 = fmaxf(x0, -125.0f);
  x1 = fmaxf(x1, -125.0f);
  float t0, t1, r0, r1, f0, f1, p0, p1;
  add2(t0, t1, x0, x1, kMagic, kMagic);
  sub2(r0, r1, t0, t1, kMagic, kMagic);
  sub2(f0, f1, x0, x1, r0, r1);
  fma2(p0, p1, f0, f1, 0.05517166f, 0.05517166f, 0.24261115f, 0.24261115f);
  fma2(p0, p1, p0, p1, f0, f1, 0.69326097f, 0.69326097f);
  fma2(p0, p1, p0, p1, f0, f1, 0.99992806f, 0.99992806f);
  e0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  e1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Debug timeline (AttnArgs::trace): one CTA records clock64 at pipeline events.
#define RK_TRACE(role, step, ev)                                                                           \
  do {                                                                                                   \
    if (TRACE && tracing && (step) < 64) a.trace[((role) * 64 + (step)) * 8 + (ev)] = clock64();         \
  } while (0)

constexpr int kQ = 128;     // query rows per tile (TMEM lanes)
constexpr float kRescaleLog2 = 8.0f;  // lazy O rescale threshold (P <= 2^8)
constexpr int kThreadsA = 256;        // softmax warpgroup + control warpgroup

template <int DH>
struct ACfg {
  // keys per tile: 128 at d_head 64, 64 at d_head 128, so that two CTAs
  // (112 KB smem, 256 TMEM columns each) share every SM and one CTA's softmax
  // overlaps the other's MMAs, loads and epilogue. (Measured: 64-key tiles
  // with three CTAs per SM at d_head 64 are slower -- the per-tile fixed
  // softmax latency dominates.)
  static constexpr int KEYS = DH == 64 ? 128 : 64;
  static constexpr int KB = KEYS / 64;             // 64-key swizzle blocks of S / P
  static constexpr int Q_TILE = kQ * DH * 2;
  static constexpr int KV_BYTES = KEYS * DH * 2;   // one stage of K or V
  static constexpr int KST = 2, VST = 2;
  static constexpr int P_BYTES = kQ * KEYS * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = Q_TILE;
  static constexpr int OFF_V = OFF_K + KST * KV_BYTES;
  static constexpr int OFF_P = OFF_V + VST * KV_BYTES;
  static constexpr int OFF_BAR = OFF_P + P_BYTES;
  static constexpr int SMEM = OFF_BAR + 128;
  static constexpr int CTAS = 2;  // CTAs per SM
  static_assert(CTAS * (SMEM + 1024) <= 233472, "shared memory per SM");
  static constexpr uint32_t TMEM_COLS = KEYS + DH <= 128 ? 128 : 256;
  static_assert(CTAS * TMEM_COLS <= 512, "tensor memory per SM");
  static constexpr uint32_t S_COL = 0, O_COL = KEYS;  // S [0,KEYS), O [KEYS, KEYS+DH)
  // setmaxnreg: control warpgroup down to REG_CTL, softmax up to REG_SM
  static constexpr int REG_LAUNCH = (65536 / (CTAS * 256)) / 8 * 8;
  static constexpr int REG_CTL = CTAS == 3 ? 24 : 56;
  static constexpr int REG_SM = (REG_LAUNCH * 2 - REG_CTL) / 8 * 8;
};

// Query tile `tile` of the launch -> rows [r0, r1) within one row group.
// Tiles are numbered prefix, segment rows, suffix -- ascending key length
// (the suffix sits after every segment) -- so the reversed dispatch order is
// longest-first: the suffix tiles, whose rows see the whole context, start
// at once instead of forming the launch's tail.
__device__ __forceinline__ void tile_rows(const AttnArgs& a, int M, int tile, int& r0, int& r1) {
  const int g1 = min(a.g1, M), g2 = min(max(a.g2, g1), M);
  const int lo[3] = {0, g2, g1}, hi[3] = {g1, M, g2};  // prefix | segment rows | suffix
  const int rq = a.rq;
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    const int b0 = lo[g], b1 = hi[g];
    const int nt = (b1 - b0 + rq - 1) / rq;
    if (tile < nt) {
      r0 = b0 + tile * rq;
      r1 = min(r0 + rq, b1);
      return;
    }
    tile -= nt;
  }
  r0 = r1 = 0;
}

// Query tiles of the live rows (tile_rows numbering).
__device__ __forceinline__ int live_tiles(const AttnArgs& a, int M) {
  const int g1 = min(a.g1, M), g2 = min(max(a.g2, g1), M), rq = a.rq;
  return (g1 + rq - 1) / rq + (M - g2 + rq - 1) / rq + (g2 - g1 + rq - 1) / rq;
}

// 3-input max (FMNMX3 on sm_100): two new values per instruction
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ __forceinline__ void exp2_pair(float x0, float x1, bool poly, float& e0, float& e1) {
  if (poly) {
    poly_exp2_pair(x0, x1, e0, e1);
  } else {
    e0 = fast_exp2(x0);
    e1 = fast_exp2(x1);
  }
}

// Split-KV merge, streaming part: NP >= ts parts, Q float4 per thread per
// round (NP * Q loads in flight); returns the non-finite check value.
template <int DH, int NP>
__device__ __forceinline__ float attn_merge_stream(const AttnArgs& a, const float4* src, const float* wsm, int rl, int ts,
                                                   int r0, int r1, int rq, int G, int h0) {
  constexpr int F4 = DH / 4;  // float4 per lane row
  constexpr int Q = NP <= 4 ? 8 : (NP <= 8 ? 4 : 2);
  float chk = 0.f;
#pragma unroll 1
  for (int i0 = 0; i0 < F4; i0 += Q) {
    float4 v[NP][Q];
#pragma unroll
    for (int z = 0; z < NP; ++z)
#pragma unroll
      for (int q = 0; q < Q; ++q) v[z][q] = __ldcg(src + (size_t)min(z, ts - 1) * kQ * F4 + rl + 128 * (i0 + q));
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const int f = rl + 128 * (i0 + q), ln = f / F4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int z = 0; z < NP; ++z) {
        const float wz = wsm[ln * 16 + z];
        acc.x += wz * v[z][q].x;
        acc.y += wz * v[z][q].y;
        acc.z += wz * v[z][q].z;
        acc.w += wz * v[z][q].w;
      }
      const int hl = ln / rq, row = r0 + ln % rq;
      if (hl < G && row < r1) {
        chk = fmaf(acc.x + acc.y + acc.z + acc.w, 0.f, chk);
        *reinterpret_cast<uint2*>(a.out + (size_t)row * (a.H * DH) + (h0 + hl) * DH + 4 * (f % F4)) =
            make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
      }
    }
  }
  return chk;
}

// Split-KV merge of a lane slice [l0, l1) of the tile (cooperative merge: each
// part of a cluster-launched tile merges its own slice once all parts have
// written their partials); weights wsm[lane][16] as above.
template <int DH, int NP>
__device__ __forceinline__ float attn_merge_slice(const AttnArgs& a, const float4* src, const float* wsm, int rl,
                                                  int ts, int l0, int l1, int r0, int r1, int rq, int G, int h0) {
  constexpr int F4 = DH / 4;
  float chk = 0.f;
#pragma unroll 2
  for (int f = l0 * F4 + rl; f < l1 * F4; f += 128) {
    float4 v[NP];
#pragma unroll
    for (int z = 0; z < NP; ++z) v[z] = __ldcg(src + (size_t)min(z, ts - 1) * kQ * F4 + f);
    const int ln = f / F4;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int z = 0; z < NP; ++z) {
      const float wz = wsm[ln * 16 + z];
      acc.x += wz * v[z].x;
      acc.y += wz * v[z].y;
      acc.z += wz * v[z].z;
      acc.w += wz * v[z].w;
    }
    const int hl = ln / rq, row = r0 + ln % rq;
    if (hl < G && row < r1) {
      chk = fmaf(acc.x + acc.y + acc.z + acc.w, 0.f, chk);
      *reinterpret_cast<uint2*>(a.out + (size_t)row * (a.H * DH) + (h0 + hl) * DH + 4 * (f % F4)) =
          make_uint2(pack_bf16(acc.x, acc.y), pack_bf16(acc.z, acc.w));
    }
  }
  return chk;
}

// POLY: bit c set -> the 4 pairs of 16-byte chunk c (of 8 per 64-key block)
// take the FMA-pipe cubic instead of MUFU.EX2 (0x88: a quarter of the exps).
template <int DH, bool TRACE, int POLY = 0x88>
__global__ void __launch_bounds__(kThreadsA, ACfg<DH>::CTAS)
    attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnArgs a) {
  using C = ACfg<DH>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* k_empty = bar + 3;  // [2]
  uint64_t* v_full = bar + 5;   // [2]
  uint64_t* v_empty = bar + 7;  // [2]
  uint64_t* s_full = bar + 9;
  uint64_t* s_free = bar + 10;
  uint64_t* p_full = bar + 11;
  uint64_t* o_done = bar + 12;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 13);
  int* s_kmax = reinterpret_cast<int*>(bar + 14);

  pdl_trigger();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint64_t t_entry = 0, t_wait = 0;  // (TRACE: per-CTA global-timer span, after the 1536 event slots)
  if (TRACE) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_entry));
  const long long c_entry = TRACE ? clock64() : 0;
  // shared-memory setup overlaps the previous kernel's tail (before the wait)
  if (warp == 4 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();  // SW128 tiles need a 1 KB aligned base
    *s_kmax = -1;
  }
  pdl_wait();  // rows_dev / positions / Q of the previous kernel
  if (TRACE) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_wait));
  const bool tr_cta = TRACE && a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0;
  const int M = a.rows_dev ? *a.rows_dev : a.rows_max;
  // grid (split part, head, tile) with the LIVE tiles in reverse order: the
  // CTAs of the latest (longest) query tiles of every head dispatch first, all
  // parts of a tile together; grid slots past the live tile count (sparse
  // passes size the grid for rows_max) come last and exit at once instead of
  // occupying the first waves
  const int nlive = live_tiles(a, M);
  if ((int)blockIdx.z >= nlive) return;
  int r0, r1;
  tile_rows(a, M, nlive - 1 - (int)blockIdx.z, r0, r1);
  if (r1 <= r0) return;
  // GQA packing: the CTA's 128 TMEM lanes hold rq rows x `group` q heads of
  // one kv head (lane = head_local * rq + row), so every K/V tile is staged
  // once for all heads of its group and a tile spans only rq positions
  // (tighter causal bound for gathered sparse rows). group 1: rq = 128 rows
  // of head blockIdx.y.
  const int G = a.group, rq = a.rq;
  const int part = blockIdx.x;  // split-KV part (fastest grid dim: a tile's parts dispatch together)
  const int kvh = G > 1 ? (int)blockIdx.y : (int)blockIdx.y / (a.H / a.Hkv);
  const int h0 = G > 1 ? kvh * G : (int)blockIdx.y;  // first q head of the CTA
  constexpr int KEYS = C::KEYS;
  constexpr int DB = DH / 64;  // 64-wide swizzle blocks along d
  __syncthreads();  // barriers initialised
  // Part 0 of a live tile always owns key tile 0, so its Q and first K tile
  // go out now; their latency overlaps the key-bound scan and TMEM allocation.
  const bool early = part == 0;
  if (early && warp == 6 && elect_one()) {
    mbar_arrive_expect_tx(q_full, G * rq * DH * 2);
    for (int hl = 0; hl < G; ++hl)
      for (int b = 0; b < DB; ++b)
        tma_load_2d(smem + C::OFF_Q + b * kQ * 128 + hl * rq * 128, &tmQ, q_full, (h0 + hl) * DH + b * 64, r0);
  }
  if (early && warp == 4 && elect_one()) {
    mbar_arrive_expect_tx(&k_full[0], C::KV_BYTES);
    for (int b = 0; b < DB; ++b)
      tma_load_2d(smem + C::OFF_K + b * KEYS * 128, &tmK, &k_full[0], kvh * DH + b * 64, 0);
  }
  for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) atomicMax(s_kmax, a.pos[i]);
  __syncthreads();
  if (tr_cta) {  // prologue marks (role 1 slots: one tile per CTA leaves them free)
    a.trace[(64 + 0) * 8 + 0] = c_entry;
    a.trace[(64 + 0) * 8 + 1] = clock64();
  }
  // Adaptive split-KV: a tile whose key range exceeds tiles_per_split key
  // tiles is cut into ts = ceil(nk_tile / tiles_per_split) (<= gridDim.x)
  // equal parts; CTA x covers part x, and the last part to finish merges them
  // (in-kernel, below). Tiles that fit in one part write their output directly.
  const int nk_tile = *s_kmax / KEYS + 1;
  const int ts = min((int)gridDim.x, (nk_tile + a.tiles_per_split - 1) / a.tiles_per_split);
  const int tps = (nk_tile + ts - 1) / ts;
  const int ts_eff = (nk_tile + tps - 1) / tps;  // parts that own key tiles
  const int j0 = part * tps;
  const int nk = min(nk_tile - j0, tps);
  const bool partial = ts_eff > 1;
  const bool trace_cta = TRACE && a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  if (part >= ts_eff || nk <= 0) return;  // this tile has no such part (never part 0: no TMA in flight)

  if (warp == 5) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (tr_cta) a.trace[(64 + 0) * 8 + 2] = clock64();

  if (warp >= 4) {  // ------------------------------------------ control warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(C::REG_CTL) : "memory");
    if (warp == 4) {
      if (elect_one()) {  // ---------------------------------------- TMA K
        for (int j = early ? 1 : 0; j < nk; ++j) {  // (part 0: K tile 0 already issued)
          const int st = j & 1;
          mbar_wait(&k_empty[st], ((j >> 1) & 1) ^ 1);
          uint8_t* sk = smem + C::OFF_K + st * C::KV_BYTES;
          mbar_arrive_expect_tx(&k_full[st], C::KV_BYTES);
          for (int b = 0; b < DB; ++b)
            tma_load_2d(sk + b * KEYS * 128, &tmK, &k_full[st], kvh * DH + b * 64, (j0 + j) * KEYS);
        }
      }
    } else if (warp == 6) {
      if (elect_one()) {  // ------------------------------------- TMA Q, V
        if (!early) {
          mbar_arrive_expect_tx(q_full, G * rq * DH * 2);
          for (int hl = 0; hl < G; ++hl)
            for (int b = 0; b < DB; ++b)
              tma_load_2d(smem + C::OFF_Q + b * kQ * 128 + hl * rq * 128, &tmQ, q_full, (h0 + hl) * DH + b * 64, r0);
        }
        for (int j = 0; j < nk; ++j) {
          const int st = j & 1;
          mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
          uint8_t* sv = smem + C::OFF_V + st * C::KV_BYTES;
          mbar_arrive_expect_tx(&v_full[st], C::KV_BYTES);
          for (int b = 0; b < DB; ++b)
            tma_load_2d(sv + b * KEYS * 128, &tmV, &v_full[st], kvh * DH + b * 64, (j0 + j) * KEYS);
        }
      }
    } else if (warp == 5) {
      if (elect_one()) {  // ------------------------------------------ MMA
        const bool tracing = trace_cta;
        constexpr uint32_t idesc_s = idesc_bf16(kQ, KEYS);
        constexpr uint32_t idesc_o = idesc_bf16(kQ, DH, /*b_mn_major=*/true);
        const uint32_t sq = smem_u32(smem + C::OFF_Q);
        mbar_wait(q_full, 0);
        auto issue_s = [&](int j) {
          const int st = j & 1;
          mbar_wait(&k_full[st], (j >> 1) & 1);
          mbar_wait(s_free, (j & 1) ^ 1);
          RK_TRACE(2, j, 1);
          tc_fence_after();
          const uint32_t sk = smem_u32(smem + C::OFF_K + st * C::KV_BYTES);
#pragma unroll
          for (int k = 0; k < DH / 16; ++k) {
            const uint32_t off = (k >> 2) * (kQ * 128) + (k & 3) * 32;
            const uint32_t offk = (k >> 2) * (KEYS * 128) + (k & 3) * 32;
            mma_bf16_ss(tmem + C::S_COL, sdesc_sw128(sq + off, 16, 1024), sdesc_sw128(sk + offk, 16, 1024), idesc_s,
                        k > 0 ? 1u : 0u);
          }
          tc_commit(s_full);
          tc_commit(&k_empty[st]);
        };
        auto issue_pv = [&](int j) {
          const int st = j & 1;
          mbar_wait(&v_full[st], (j >> 1) & 1);
          mbar_wait(p_full, j & 1);
          RK_TRACE(2, j, 4);
          tc_fence_after();
          const uint32_t sp = smem_u32(smem + C::OFF_P);
          const uint32_t sv = smem_u32(smem + C::OFF_V + st * C::KV_BYTES);
#pragma unroll
          for (int k = 0; k < KEYS / 16; ++k) {
            const uint64_t ad = sdesc_sw128(sp + (k >> 2) * (kQ * 128) + (k & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc_sw128(sv + k * 2048, KEYS * 128, 1024);
            mma_bf16_ss(tmem + C::O_COL, ad, bd, idesc_o, (j > 0 || k > 0) ? 1u : 0u);
          }
          tc_commit(o_done);
          tc_commit(&v_empty[st]);
        };
        // S(j+1) goes in as soon as the softmax holds S(j) in registers, ahead
        // of P(j) V_j, so the next scores compute while exponentials run
        issue_s(0);
        for (int j = 0; j < nk; ++j) {
          if (j + 1 < nk) issue_s(j + 1);
          issue_pv(j);
        }
      }
    }
  } else {  // ------------------------------------------------ softmax warpgroup
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(C::REG_SM) : "memory");
    const bool tracing = trace_cta && warp == 0 && lane == 0;
    const int rl = warp * 32 + lane;  // TMEM lane
    const int hl = rl / rq;           // head within the group
    const int h = h0 + hl;
    const int row = r0 + rl % rq;
    const bool valid = hl < G && row < r1;
    const int pos = valid ? a.pos[row] : *s_kmax;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t s_col = tmem + lane_base + C::S_COL;
    const uint32_t o_col = tmem + lane_base + C::O_COL;
    uint8_t* sp = smem + C::OFF_P;
    const float scale = a.scale_log2;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < nk; ++j) {
      RK_TRACE(0, j, 0);
      mbar_wait(s_full, j & 1);
      RK_TRACE(0, j, 1);
      tc_fence_after();
      uint32_t r[KEYS];
#pragma unroll
      for (int c = 0; c < KEYS; c += 32) tmem_ld32(s_col + c, *reinterpret_cast<uint32_t(*)[32]>(&r[c]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);  // S(j+1) may overwrite TMEM now
      RK_TRACE(0, j, 2);
      const int kbase = (j0 + j) * KEYS;
      // warp-uniform: no causal mask anywhere in this tile for this warp's rows
      if (!__all_sync(0xffffffffu, kbase + KEYS - 1 <= pos)) {
#pragma unroll
        for (int u = 0; u < KEYS; ++u)
          if (kbase + u > pos) r[u] = __float_as_uint(-INFINITY);
      }
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int u = 0; u < KEYS; u += 8) {
        mx0 = fmax3(mx0, __uint_as_float(r[u]), __uint_as_float(r[u + 1]));
        mx1 = fmax3(mx1, __uint_as_float(r[u + 2]), __uint_as_float(r[u + 3]));
        mx2 = fmax3(mx2, __uint_as_float(r[u + 4]), __uint_as_float(r[u + 5]));
        mx3 = fmax3(mx3, __uint_as_float(r[u + 6]), __uint_as_float(r[u + 7]));
      }
      const float m_new = fmaxf(m_run, fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3)) * scale);
      bool waited = false;  // P(j-1) V_{j-1} known complete (P buffer free, O stable)
      if (j == 0) {
        m_run = m_new;  // O is written (not accumulated) by the first P.V
      } else {
        const bool need = m_new > m_run + kRescaleLog2;
        if (__any_sync(0xffffffffu, need)) {  // rare: rescale O in TMEM once P.V_{j-1} landed
          mbar_wait(o_done, (j - 1) & 1);
          tc_fence_after();
          waited = true;
          const float corr = need ? fast_exp2(m_run - m_new) : 1.0f;
#pragma unroll
          for (int c = 0; c < DH; c += 32) {
            uint32_t o[32];
            tmem_ld32(o_col + c, o);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * corr);
            tmem_st32(o_col + c, o);
          }
          tmem_st_wait();
          l_run *= corr;
          if (need) m_run = m_new;
        }
      }
      RK_TRACE(0, j, 3);
      // P = exp2(s * scale - m_run) -> bf16, K-major SW128 (2 blocks of 64
      // keys, 16-byte chunks swizzled by row); chunks 3 and 7 of each block via
      // the FMA-pipe cubic, the rest on MUFU. The first block is computed
      // before waiting for the previous P.V, so that wait overlaps the exps.
      const float neg_m = m_run == -INFINITY ? 0.f : -m_run;
      float ls0 = 0.f, ls1 = 0.f, ls2 = 0.f, ls3 = 0.f;
#pragma unroll
      for (int b = 0; b < C::KB; ++b) {
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int u = b * 64 + 2 * i;
          float x0, x1, e0, e1;
          fma2(x0, x1, __uint_as_float(r[u]), __uint_as_float(r[u + 1]), scale, scale, neg_m, neg_m);
          exp2_pair(x0, x1, (POLY >> (i >> 2)) & 1, e0, e1);
          if (i & 1) add2(ls2, ls3, ls2, ls3, e0, e1);
          else add2(ls0, ls1, ls0, ls1, e0, e1);
          pk[i] = pack_bf16(e0, e1);
        }
        if (b == 0) RK_TRACE(0, j, 6);  // first block's exps done
        if (b == 0 && j > 0 && !waited) {
          mbar_wait(o_done, (j - 1) & 1);
          tc_fence_after();
        }
        if (b == 0) RK_TRACE(0, j, 7);  // P(j-1) V done (P buffer free)
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint4* dst = reinterpret_cast<uint4*>(sp + b * (kQ * 128) + rl * 128 + ((ch ^ (rl & 7)) * 16));
          *dst = make_uint4(pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
        }
      }
      l_run += (ls0 + ls1) + (ls2 + ls3);
      RK_TRACE(0, j, 4);
      tc_fence_before();
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      RK_TRACE(0, j, 5);
    }
    mbar_wait(o_done, (nk - 1) & 1);
    tc_fence_after();
    if (tracing) a.trace[(64 + 0) * 8 + 3] = clock64();
    if (partial) {
      // in-kernel merge: partials in a tile-contiguous block [tile][part][lane][DH]
      // (one 128 x DH fp32 block per part); the last part of this (tile, kv
      // group) to finish merges them with coalesced streaming reads -- no
      // combine launch
      const size_t tid = (size_t)blockIdx.z * gridDim.y + blockIdx.y;
      const size_t blk = (tid * gridDim.x + part) * kQ;  // lanes of this part's block
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        uint32_t o[32];
        tmem_ld32(o_col + c, o);
        tmem_ld_wait();
        float4* dst = reinterpret_cast<float4*>(a.ws_o + (blk + rl) * DH + c);
#pragma unroll
        for (int u = 0; u < 32; u += 4)
          dst[u / 4] = make_float4(__uint_as_float(o[u]), __uint_as_float(o[u + 1]), __uint_as_float(o[u + 2]),
                                   __uint_as_float(o[u + 3]));
      }
      reinterpret_cast<float2*>(a.ws_ml)[blk + rl] = make_float2(valid ? m_run : -INFINITY, l_run);
      int* s_last = reinterpret_cast<int*>(bar + 15);
      fence_acq_rel_gpu();  // (release: this part's partials)
      named_bar_sync(1, 128);
      int* cnt = a.tile_cnt + tid;
      if (a.coop) {
        // the tile's parts are one cluster (co-scheduled): wait for all of
        // them, then each merges its slice of the 128 lanes in one round of
        // loads -- instead of the last part streaming every lane alone
        if (rl == 0) {
          atomicAdd(cnt, 1);
          uint32_t spins = 0;
          while (*reinterpret_cast<volatile int*>(cnt) < ts_eff) {
            __nanosleep(64);
            if (++spins > (1u << 26)) __trap();  // (a scheduling bug traps instead of hanging)
          }
        }
        named_bar_sync(1, 128);
        fence_acq_rel_gpu();  // (acquire: every part's partials)
        const int l0 = part * kQ / ts_eff, l1 = (part + 1) * kQ / ts_eff;
        float* wsm = reinterpret_cast<float*>(smem + C::OFF_K);  // [lane][16]
        const size_t blk0 = tid * gridDim.x * kQ;
        if (rl < l1 - l0) {
          const int ln = l0 + rl;
          float mz[16], lz[16];
#pragma unroll
          for (int z = 0; z < 16; ++z) {
            const float2 v = __ldcg(reinterpret_cast<const float2*>(a.ws_ml) + blk0 + (size_t)min(z, ts_eff - 1) * kQ + ln);
            mz[z] = z < ts_eff ? v.x : -INFINITY;
            lz[z] = v.y;
          }
          float m = -INFINITY;
#pragma unroll
          for (int z = 0; z < 16; ++z) m = fmaxf(m, mz[z]);
          float lsum = 0.f;
#pragma unroll
          for (int z = 0; z < 16; ++z) {
            mz[z] = mz[z] == -INFINITY ? 0.f : fast_exp2(mz[z] - m);
            lsum += mz[z] * lz[z];
          }
          const float inv = 1.f / lsum;
#pragma unroll
          for (int z = 0; z < 16; ++z) wsm[ln * 16 + z] = mz[z] * inv;
        }
        named_bar_sync(1, 128);
        const float4* src = reinterpret_cast<const float4*>(a.ws_o) + blk0 * (DH / 4);
        float chk = 0.f;
        if (ts_eff <= 4) chk = attn_merge_slice<DH, 4>(a, src, wsm, rl, ts_eff, l0, l1, r0, r1, rq, G, h0);
        else chk = attn_merge_slice<DH, 8>(a, src, wsm, rl, ts_eff, l0, l1, r0, r1, rq, G, h0);
        if (chk != chk && a.status) *reinterpret_cast<volatile int*>(a.status) = 1;
        named_bar_sync(1, 128);
        if (rl == 0 && atomicAdd(cnt, 1) == 2 * ts_eff - 1) *cnt = 0;  // the last to leave resets it
      } else {
      if (rl == 0) *s_last = atomicAdd(cnt, 1) == ts_eff - 1;
      named_bar_sync(1, 128);
      if (tracing) a.trace[(64 + 0) * 8 + 4] = clock64();
      if (*s_last) {
        fence_acq_rel_gpu();  // (acquire: every part's partials)
        if (rl == 0) *cnt = 0;  // self-resetting for the next launch
        // per-lane part weights 2^(m_z - m) / l into smem (the K ring is idle now)
        float* wsm = reinterpret_cast<float*>(smem + C::OFF_K);  // [lane][16]
        const size_t blk0 = tid * gridDim.x * kQ;
        float mz[16], lz[16];
#pragma unroll
        for (int z = 0; z < 16; ++z) {
          const float2 v = __ldcg(reinterpret_cast<const float2*>(a.ws_ml) + blk0 + (size_t)min(z, ts_eff - 1) * kQ + rl);
          mz[z] = z < ts_eff ? v.x : -INFINITY;
          lz[z] = v.y;
        }
        float m = -INFINITY;
#pragma unroll
        for (int z = 0; z < 16; ++z) m = fmaxf(m, mz[z]);
        float lsum = 0.f;
#pragma unroll
        for (int z = 0; z < 16; ++z) {
          mz[z] = mz[z] == -INFINITY ? 0.f : fast_exp2(mz[z] - m);
          lsum += mz[z] * lz[z];
        }
        const float inv = 1.f / lsum;
#pragma unroll
        for (int z = 0; z < 16; ++z) wsm[rl * 16 + z] = mz[z] * inv;
        named_bar_sync(1, 128);
        // stream: thread t takes float4 f = t + 128 i of every part block
        // (lane f / (DH/4), columns 4 (f % (DH/4)) ..), all parts' loads in
        // flight at once (branch-free: part index clamped, weight 0 past ts)
        const float4* src = reinterpret_cast<const float4*>(a.ws_o) + blk0 * (DH / 4);
        float chk = 0.f;
        if (ts_eff <= 4) chk = attn_merge_stream<DH, 4>(a, src, wsm, rl, ts_eff, r0, r1, rq, G, h0);
        else if (ts_eff <= 8) chk = attn_merge_stream<DH, 8>(a, src, wsm, rl, ts_eff, r0, r1, rq, G, h0);
        else chk = attn_merge_stream<DH, 16>(a, src, wsm, rl, ts_eff, r0, r1, rq, G, h0);
        if (chk != chk && a.status) *reinterpret_cast<volatile int*>(a.status) = 1;
        if (tracing) a.trace[(64 + 0) * 8 + 5] = clock64();
      }
      }  // (last-arriver merge)
    } else {
      const float inv = 1.f / l_run;
      uint4* dst = reinterpret_cast<uint4*>(a.out + (size_t)row * (a.H * DH) + h * DH);
      float chk = inv * 0.f;  // non-finite output (x * 0 is NaN iff x is inf/NaN)
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        uint32_t o[32];
        tmem_ld32(o_col + c, o);
        tmem_ld_wait();
        if (valid) {
#pragma unroll
          for (int u = 0; u < 32; ++u) chk = fmaf(__uint_as_float(o[u]), 0.f, chk);
#pragma unroll
          for (int u = 0; u < 32; u += 8)
            dst[(c + u) / 8] = make_uint4(pack_bf16(__uint_as_float(o[u]) * inv, __uint_as_float(o[u + 1]) * inv),
                                          pack_bf16(__uint_as_float(o[u + 2]) * inv, __uint_as_float(o[u + 3]) * inv),
                                          pack_bf16(__uint_as_float(o[u + 4]) * inv, __uint_as_float(o[u + 5]) * inv),
                                          pack_bf16(__uint_as_float(o[u + 6]) * inv, __uint_as_float(o[u + 7]) * inv));
        }
      }
      if (valid && chk != chk && a.status) *reinterpret_cast<volatile int*>(a.status) = 1;
      if (tracing) a.trace[(64 + 0) * 8 + 5] = clock64();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) tmem_dealloc(tmem, C::TMEM_COLS);
  if (tr_cta) a.trace[(64 + 0) * 8 + 6] = clock64();
  if (TRACE && a.trace && threadIdx.x == 0) {
    uint64_t t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    const size_t cid = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    unsigned long long* ct = a.trace + 1536 + 4 * cid;
    ct[0] = t_entry;
    ct[1] = t_wait;
    ct[2] = t_end;
    ct[3] = (unsigned long long)nk | ((unsigned long long)partial << 8) | ((unsigned long long)ts_eff << 16) |
            ((unsigned long long)(r1 - r0) << 32);
  }
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

// Upper bound on query tiles of a launch (row groups split at their bounds).
int max_tiles(const AttnArgs& a) {
  const int M = a.rows_max, g1 = std::min(a.g1, M), g2 = std::min(std::max(a.g2, g1), M), rq = a.rq;
  return (g1 + rq - 1) / rq + (g2 - g1 + rq - 1) / rq + (M - g2 + rq - 1) / rq;
}

template <int DH>
void launch_attn(rk_engine* e, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                 const AttnArgs& a) {
  static bool attr = false;
  // measured: a quarter of the exps on the FMA pipe pays at d_head 64 (MUFU
  // bound, 128-key tiles); at d_head 128 (64-key tiles) MUFU alone is faster
  static const int poly = [] {
    const char* v = std::getenv("RK_ATTN_POLY");
    return v ? (int)std::strtol(v, nullptr, 0) : (DH == 64 ? 0x88 : 0x00);
  }();
  if (!attr) {
    RK_CUDA(cudaFuncSetAttribute(attn_kernel<DH, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<DH>::SMEM));
    RK_CUDA(cudaFuncSetAttribute(attn_kernel<DH, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ACfg<DH>::SMEM));
    RK_CUDA(cudaFuncSetAttribute(attn_kernel<DH, false, 0xAA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 ACfg<DH>::SMEM));
    RK_CUDA(cudaFuncSetAttribute(attn_kernel<DH, false, 0x92>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 ACfg<DH>::SMEM));
    RK_CUDA(cudaFuncSetAttribute(attn_kernel<DH, false, 0x00>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 ACfg<DH>::SMEM));
    attr = true;
  }
  dim3 grid(a.splits, a.group > 1 ? a.Hkv : a.H, max_tiles(a));
  // split launches: a tile's parts form one cluster, so they are co-scheduled
  // and merge cooperatively (RK_ATTN_COOP=0: the last part merges alone)
  static const bool coop_env = [] {
    const char* v = std::getenv("RK_ATTN_COOP");
    return v ? std::atoi(v) != 0 : true;
  }();
  AttnArgs ac = a;
  ac.coop = coop_env && a.splits > 1 && a.splits <= 8 && !a.trace;
  auto go = [&](auto kern) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreadsA);
    cfg.dynamicSmemBytes = ACfg<DH>::SMEM;
    cfg.stream = e->stream;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl_enabled()) {
      at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    if (ac.coop) {
      at[na].id = cudaLaunchAttributeClusterDimension;
      at[na].val.clusterDim.x = (unsigned)a.splits;
      at[na].val.clusterDim.y = 1;
      at[na].val.clusterDim.z = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    RK_CUDA(cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, ac));
  };
  if (a.trace) go(attn_kernel<DH, true>);
  else if (poly == 0xAA) go(attn_kernel<DH, false, 0xAA>);
  else if (poly == 0x92) go(attn_kernel<DH, false, 0x92>);
  else if (poly == 0) go(attn_kernel<DH, false, 0x00>);
  else go(attn_kernel<DH, false>);
}

}  // namespace

void attention_bf16(rk_engine* e, const AttnArgs& a_in, const __nv_bfloat16* ctx_k, const __nv_bfloat16* ctx_v,
                    int ctx_rows) {
  if (a_in.rows_max <= 0) return;
  AttnArgs a = a_in;
  if (!a.status) a.status = e->status.as<int>();

  // GQA packing (RK_ATTN_PACK=0: off): G = H / H_kv q heads share a CTA, rq =
  // the largest power of two rows with G * rq <= 128 (>= 8, so G <= 16)
  static const bool pack_env = [] {
    const char* v = std::getenv("RK_ATTN_PACK");
    return v ? std::atoi(v) != 0 : true;
  }();
  a.group = 1;
  a.rq = kQ;
  if (pack_env && a.Hkv > 0 && a.H % a.Hkv == 0 && a.H / a.Hkv > 1 && a.H / a.Hkv <= 16) {
    a.group = a.H / a.Hkv;
    a.rq = 8;
    while (a.rq * 2 * a.group <= kQ) a.rq *= 2;
  }
  // split-KV when the query tiles alone cannot fill the SMs (sparse passes:
  // plan for ~1/3 of rows_max live). A split covers >= 2 key tiles; CTAs
  // whose rows end before their split exit at once, so long tiles (suffix,
  // late segment rows) spread over many CTAs while short ones stay whole.
  AttnArgs hint = a;
  if (a.rows_dev) hint.rows_max = a.rows_hint > 0 ? std::max(a.g2 + 1, a.rows_hint) : std::max(a.g2 + 1, a.rows_max / 3);
  const int ctas_per_sm = a.dh == 64 ? ACfg<64>::CTAS : ACfg<128>::CTAS;
  const int base = max_tiles(hint) * (a.group > 1 ? a.Hkv : a.H);  // CTAs without splitting
  const int slots = ctas_per_sm * e->sm_count;     // CTAs resident at once
  const int keys = a.dh == 64 ? ACfg<64>::KEYS : ACfg<128>::KEYS;
  const int nk_max = (ctx_rows + keys - 1) / keys;
  a.splits = 1;
  a.tiles_per_split = nk_max > 0 ? nk_max : 1;
  // Adaptive split-KV when the grid cannot fill ~1.5 waves: the longest
  // tile should not walk more key tiles than the average load of a resident
  // slot (~ base * nk_max / (2 * slots), causal), and no part below 6 key
  // tiles (a CTA's fixed cost is a few microseconds). Only tiles longer than
  // that are cut (per tile, on the device); the rest write their output
  // directly. (Measured: a uniform 2-way split of the c2 sparse layers and a
  // column-split softmax with two warpgroups per tile were both slower.)
  static const int min_part = [] {
    const char* v = std::getenv("RK_ATTN_MINPART");
    return v ? std::max(1, std::atoi(v)) : 6;  // (4 before the cooperative merge; 6 measured best with it, r02cd/r02ck)
  }();
  static const double split_div = [] {
    const char* v = std::getenv("RK_ATTN_SPLITDIV");
    return v ? std::atof(v) : 2.0;
  }();
  static const double split_waves = [] {
    const char* v = std::getenv("RK_ATTN_SPLITWAVES");
    return v ? std::atof(v) : 1.0;
  }();
  if (base < split_waves * slots && nk_max >= 2 * min_part) {
    const int target = std::max(min_part, (int)((double)nk_max * base / (split_div * slots) + 0.999));
    if (target < nk_max) {
      a.tiles_per_split = target;
      a.splits = std::min(16, (nk_max + target - 1) / target);
    }
  }
  if (a.splits > 1) {
    Scratch& S = *e->scratch;
    // partials: per (tile, kv group, part) one 128-lane fp32 block + (m, l)
    // per lane, merged in-kernel by the tile's last part (r02r: faster than a
    // separate combine launch, 19.8 vs 20.5 us on the c2 prefix+suffix layer)
    const size_t tiles = (size_t)max_tiles(a) * (a.group > 1 ? a.Hkv : a.H);
    const size_t per = tiles * a.splits * kQ;
    S.attn_ws.ensure(per * (a.dh + 2) * 4 + 256);
    a.ws_o = S.attn_ws.as<float>();
    a.ws_ml = a.ws_o + per * a.dh;
    if (S.attn_cnt.bytes < tiles * 4) {  // arrival counters, zeroed once, self-resetting
      S.attn_cnt.ensure(tiles * 4);
      RK_CUDA(cudaMemsetAsync(S.attn_cnt.p, 0, S.attn_cnt.bytes, e->stream));
    }
    a.tile_cnt = S.attn_cnt.as<int>();
  }
  const int q = a.H * a.dh, kv = a.Hkv * a.dh;
  CUtensorMap tq, tk, tv;
  make_tmap_bf16(&tq, a.q, (uint64_t)a.rows_max, (uint64_t)q, (uint32_t)a.rq, (uint64_t)q);
  make_tmap_bf16(&tk, ctx_k, (uint64_t)ctx_rows, (uint64_t)kv, keys, (uint64_t)kv);
  make_tmap_bf16(&tv, ctx_v, (uint64_t)ctx_rows, (uint64_t)kv, keys, (uint64_t)kv);
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
