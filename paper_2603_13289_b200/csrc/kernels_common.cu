// kernels_common.cu -- kernels shared by both precisions: weight init and
// packing, embedding, row gather/scatter, SegmentMarks, argmax, and the relay
// kernels proper (realign+graft, deviation scoring, selection).
//
// Every floating-point operation that the reference performs is written with
// explicit round-to-nearest intrinsics (__fmul_rn, __dadd_rn, ...) so nvcc
// cannot contract it into an FMA the reference does not have
// (-ffp-contract=off, proj/src/CMakeLists.txt:16-18).
#include <cuda_bf16.h>

#include <algorithm>

#include "internal.h"
#include "sm100.cuh"

namespace rk {
namespace {
// Launch with programmatic stream serialization (see sm100.cuh pdl_*): every
// kernel launched through here starts with pdl_trigger(); pdl_wait().
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


constexpr int kThreads = 256;

inline int blocks_for(size_t n, int threads = kThreads) {
  size_t b = (n + threads - 1) / threads;
  return (int)(b > 0x7fffffff ? 0x7fffffff : (b == 0 ? 1 : b));
}

__device__ __forceinline__ float load_elem(const void* p, size_t i, size_t elem) {
  if (elem == 4) return static_cast<const float*>(p)[i];
  return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}
__device__ __forceinline__ uint32_t load_bits(const void* p, size_t i, size_t elem) {
  if (elem == 4) return __float_as_uint(static_cast<const float*>(p)[i]);
  return static_cast<const unsigned short*>(p)[i];
}

// ---------------------------------------------------------------------------
// weights: init_weights (model.cpp:81-114) as a counter-based stream.
// SplitMix64 (model.cpp:49-56) advances state by a constant, so draw i of a
// tensor whose stream starts at state0 is mix(state0 + (i+1)*gamma).
// ---------------------------------------------------------------------------
__global__ void init_uniform_kernel(float* dst, size_t n, uint64_t state0, float scale) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = state0 + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z = z ^ (z >> 31);
    const float u = __fmul_rn((float)(z >> 40), 0x1p-24f);          // model.cpp:58
    const float sym = __fsub_rn(__fmul_rn(2.0f, u), 1.0f);          // model.cpp:59
    dst[i] = __fmul_rn(sym, scale);                                 // model.cpp:69
  }
}

__global__ void fill_kernel(float* dst, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = v;
}

__global__ void copy_cols_kernel(float* dst, size_t ldd, size_t c0, const float* src, size_t lds,
                                 size_t rows, size_t cols, size_t cstride) {
  const size_t total = rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / cols, c = i % cols;
    dst[r * ldd + c0 + c * cstride] = src[r * lds + c];
  }
}

// src [rows x cols] row-major fp32 -> dst row (c0 + c*cstride), column r, bf16.
// row_gain (optional, [rows]): src row r is multiplied by row_gain[r] (a
// RMSNorm gain folded into the weight that consumes the normalised rows).
__global__ void transpose_bf16_kernel(__nv_bfloat16* dst, size_t ldd, size_t c0, size_t cstride,
                                      const float* src, size_t rows, size_t cols, const float* row_gain) {
  __shared__ float tile[32][33];
  const size_t bc = blockIdx.x * 32, br = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const size_t r = br + i, c = bc + threadIdx.x;
    float v = (r < rows && c < cols) ? src[r * cols + c] : 0.f;
    if (row_gain && r < rows) v = __fmul_rn(v, row_gain[r]);
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const size_t c = bc + i, r = br + threadIdx.x;
    if (r < rows && c < cols) dst[(c0 + c * cstride) * ldd + r] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

__global__ void copy2d_kernel(float* dst, size_t dld, size_t dcs, const float* src, size_t sld,
                              size_t scs, size_t rows, size_t cols) {
  const size_t total = rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / cols, c = i % cols;
    dst[r * dld + c * dcs] = src[r * sld + c * scs];
  }
}
// dst[r][c] = float(src[(c0 + c*cstride) * ld + r])
__global__ void untranspose_bf16_kernel(float* dst, const __nv_bfloat16* src, size_t ld, size_t c0,
                                        size_t cstride, size_t rows, size_t cols, const float* row_gain) {
  const size_t total = rows * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / cols, c = i % cols;
    float v = __bfloat162float(src[(c0 + c * cstride) * ld + r]);
    if (row_gain && row_gain[r] != 0.f) v = __fdiv_rn(v, row_gain[r]);
    dst[i] = v;
  }
}
__global__ void d2f_kernel(float* dst, const double* src, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

__global__ void f32_to_bf16_kernel(__nv_bfloat16* dst, const float* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}
__global__ void bf16_to_f32_kernel(float* dst, const __nv_bfloat16* src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __bfloat162float(src[i]);
}

// ---------------------------------------------------------------------------
// embed_tokens (model.cpp:149-161); token range is validated on the host.
// ---------------------------------------------------------------------------
__global__ void embed_kernel(float* hidden, const void* emb, size_t elem, const int32_t* tokens,
                             int n, int d) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const size_t total = (size_t)n * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / d, c = i % d;
    hidden[i] = load_elem(emb, (size_t)tokens[r] * d + c, elem);
  }
}

// sparse_rectify gather/scatter (relay_engine.cpp:162-178)
__global__ void gather_rows_kernel(float* dst, const float* src, const int* idx, const int* count,
                                   int rows_max, int d) {
  const int rows = count ? *count : rows_max;
  const size_t total = (size_t)rows * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / d, c = i % d;
    dst[i] = src[(size_t)idx[r] * d + c];
  }
}
__global__ void scatter_rows_kernel(float* dst, const float* src, const int* idx, const int* count,
                                    int rows_max, int d, uint64_t* depth, uint64_t depth_value) {
  const int rows = count ? *count : rows_max;
  const size_t total = (size_t)rows * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / d, c = i % d;
    dst[(size_t)idx[r] * d + c] = src[i];
    if (c == 0 && depth) depth[idx[r]] = depth_value;
  }
}
__global__ void positions_from_sel_kernel(int* pos, const int* sel, const int* count, int rows_max,
                                          int base) {
  const int rows = count ? *count : rows_max;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    pos[r] = base + sel[r];
}
__global__ void iota_kernel(int* pos, int n, int base) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    pos[r] = base + r;
}
__global__ void mark_rows_kernel(uint8_t* origin, int len, int lo, int hi, const int* sel,
                                 const int* count, int rows_max) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int rows = count ? *count : rows_max;
  const int layers = hi - lo + 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * layers;
       i += gridDim.x * blockDim.x)
    origin[(size_t)(lo + i / rows) * len + sel[i % rows]] = 1;
}
__global__ void mark_layers_kernel(uint8_t* origin, int len, int lo, int hi) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const size_t total = (size_t)(hi - lo + 1) * len;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x)
    origin[(size_t)lo * len + i] = 1;
}
// Device-side zero fill / copy as kernels (not copy-engine operations, which
// would queue behind relay-cache uploads streaming on the copy engines).
__global__ void zero_bytes_kernel(uint8_t* dst, size_t n) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const size_t i0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x), stride = (size_t)gridDim.x * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (size_t i = i0; i < n / 16; i += stride) d4[i] = make_uint4(0, 0, 0, 0);
    for (size_t i = n / 16 * 16 + i0; i < n; i += stride) dst[i] = 0;
  } else {
    for (size_t i = i0; i < n; i += stride) dst[i] = 0;
  }
}
__global__ void copy_bytes_kernel(uint8_t* dst, const uint8_t* src, size_t n) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const size_t i0 = (blockIdx.x * (size_t)blockDim.x + threadIdx.x), stride = (size_t)gridDim.x * blockDim.x;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    for (size_t i = i0; i < n / 16; i += stride) d4[i] = s4[i];
    for (size_t i = n / 16 * 16 + i0; i < n; i += stride) dst[i] = src[i];
  } else {
    for (size_t i = i0; i < n; i += stride) dst[i] = src[i];
  }
}
// rows x width bytes at pitch
__global__ void zero_rows_kernel(uint8_t* dst, size_t pitch, size_t width, size_t rows) {
  for (size_t r = blockIdx.y; r < rows; r += gridDim.y) {
    uint8_t* d = dst + r * pitch;
    if (((reinterpret_cast<uintptr_t>(d) | width) & 15) == 0) {
      for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < width / 16; i += (size_t)gridDim.x * blockDim.x)
        reinterpret_cast<uint4*>(d)[i] = make_uint4(0, 0, 0, 0);
    } else {
      for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < width; i += (size_t)gridDim.x * blockDim.x)
        d[i] = 0;
    }
  }
}
__global__ void copy_i32_kernel(int* dst, const int* src, int n) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
__global__ void fill_doubles_kernel(double* dst, int n, double v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = v;
}
__global__ void set_depth_kernel(uint64_t* depth, int n, uint64_t v) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) depth[i] = v;
}

// argmax (model.cpp:364-370): first index of the maximum. Two passes: kArgBlocks
// CTAs reduce strided chunks with 16-byte loads, one CTA merges the partials.
constexpr int kArgBlocks = 148;
__device__ __forceinline__ void arg_better(float v, int i, float& bv, int& bi) {
  if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}
__device__ void block_argmax(float& best, int& bi) {
  __shared__ float sv[32];
  __shared__ int si[32];
  for (int o = 16; o; o >>= 1) {
    const float v = __shfl_xor_sync(0xffffffffu, best, o);
    const int i = __shfl_xor_sync(0xffffffffu, bi, o);
    arg_better(v, i, best, bi);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[w] = best; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    best = lane < (int)(blockDim.x >> 5) ? sv[lane] : -__int_as_float(0x7f800000);
    bi = lane < (int)(blockDim.x >> 5) ? si[lane] : 0x7fffffff;
    for (int o = 16; o; o >>= 1) {
      const float v = __shfl_xor_sync(0xffffffffu, best, o);
      const int i = __shfl_xor_sync(0xffffffffu, bi, o);
      arg_better(v, i, best, bi);
    }
  }
}
__global__ void __launch_bounds__(256) argmax_partial_kernel(const float* __restrict__ x, int n,
                                                             float2* __restrict__ part) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  float best = -__int_as_float(0x7f800000);
  int bi = 0x7fffffff;
  const int n4 = (reinterpret_cast<uintptr_t>(x) & 15) ? 0 : n / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const float4 v = x4[i];
    arg_better(v.x, 4 * i, best, bi);
    arg_better(v.y, 4 * i + 1, best, bi);
    arg_better(v.z, 4 * i + 2, best, bi);
    arg_better(v.w, 4 * i + 3, best, bi);
  }
  for (int i = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    arg_better(x[i], i, best, bi);
  block_argmax(best, bi);
  if (threadIdx.x == 0) part[blockIdx.x] = make_float2(best, __int_as_float(bi));
}
__global__ void argmax_final_kernel(const float2* __restrict__ part, int parts, int* out) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  float best = -__int_as_float(0x7f800000);
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < parts; i += blockDim.x)
    arg_better(part[i].x, __float_as_int(part[i].y), best, bi);
  block_argmax(best, bi);
  if (threadIdx.x == 0) *out = bi == 0x7fffffff ? 0 : bi;
}

// ---------------------------------------------------------------------------
// K1 realign + graft (relay_cache.cpp:154-174 + relay_engine.cpp:136-148).
// HBM-bound stream: grid (vector blocks of the segment, grafted layers), one
// 16-byte vector of K_pre and one of V per thread, both loads issued before
// any use so every thread keeps 32 B in flight. K pairs are rotated in double
// without FMA from the host-built glibc cos/sin table (L1/L2-resident), then
// rounded (tensor.cpp:140-141); V is a bit copy. Layers [skip_lo, skip_hi]
// are skipped (the band recompute overwrites them; relay_engine.cpp:261-264).
// ---------------------------------------------------------------------------
// Fast path for d_head 64/128, staged through shared memory by TMA bulk
// copies: a CTA owns P consecutive segment positions of one grafted layer.
// One thread issues two cp.async.bulk loads (the P x kv block of K_pre and of
// V, contiguous in the cache's [L][n][kv] layout) on an mbarrier while the CTA
// stages the P rows of the double cos/sin table; V goes straight back out with
// a bulk store into the context rows [base+p0, base+p0+P) (contiguous in the
// context's [L][cap][kv] layout), K is rotated in shared memory (double, no
// FMA) and follows with a second bulk store. Registers stay low, so many CTAs
// per SM keep their bulk copies in flight.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(sm100::smem_u32(dst)), "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sm100::smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename T, int DH>
__global__ void __launch_bounds__(128) realign_graft_dh_kernel(const __grid_constant__ k::RealignJobs J, int kv,
                                                               const double2* __restrict__ rope, T* __restrict__ ctx_k,
                                                               T* __restrict__ ctx_v, size_t ctx_layer_stride,
                                                               int skip_lo, int skip_hi, int P) {
  extern __shared__ __align__(128) uint8_t sm_raw[];
  constexpr int VEC = 16 / sizeof(T), HALF = DH / 2, CH = DH / VEC;  // CH: 16-byte chunks per head slice
  int u = 0;  // the segment (job) of this CTA
  while (u + 1 < J.count && (int)blockIdx.x >= J.blk0[u + 1]) ++u;
  const int n = J.n[u], base = J.base[u];
  const int p0 = ((int)blockIdx.x - J.blk0[u]) * P, np = min(P, n - p0);
  const uint32_t bytes = (uint32_t)np * kv * sizeof(T);
  T* sk = reinterpret_cast<T*>(sm_raw);
  T* sv = reinterpret_cast<T*>(sm_raw + (size_t)P * kv * sizeof(T));
  double2* cs_sm = reinterpret_cast<double2*>(sm_raw + (size_t)2 * P * kv * sizeof(T));
  uint64_t* bar = reinterpret_cast<uint64_t*>(cs_sm + (size_t)P * HALF);
  int l = blockIdx.y;
  if (skip_hi >= skip_lo && l >= skip_lo) l += skip_hi - skip_lo + 1;
  sm100::pdl_trigger();
  if (threadIdx.x == 0) {
    sm100::mbar_init(bar, 1);
    sm100::fence_barrier_init();
  }
  // the table is host-built and constant: staged before the dependency wait
  for (int i = threadIdx.x; i < np * HALF; i += blockDim.x) cs_sm[i] = rope[(size_t)(base + p0) * HALF + i];
  __syncthreads();
  sm100::pdl_wait();
  const size_t src = ((size_t)l * n + p0) * kv;
  const size_t dst = (size_t)l * ctx_layer_stride + (size_t)(base + p0) * kv;
  if (threadIdx.x == 0) {
    sm100::mbar_arrive_expect_tx(bar, 2 * bytes);
    bulk_g2s(sk, static_cast<const T*>(J.k_pre[u]) + src, bytes, bar);
    bulk_g2s(sv, static_cast<const T*>(J.v[u]) + src, bytes, bar);
  }
  sm100::mbar_wait(bar, 0);
  if (threadIdx.x == 0) bulk_s2g(ctx_v + dst, sv, bytes);  // V: a bit copy
  // thread = (position, 16-byte chunk of the head slice): its cos/sin pairs
  // live in registers across every head
  const int heads = kv / DH;
  for (int it = threadIdx.x; it < np * CH; it += blockDim.x) {
    const int pl = it / CH, ch = it - pl * CH;
    double2 c_s[VEC / 2];
#pragma unroll
    for (int i = 0; i < VEC / 2; ++i) c_s[i] = cs_sm[pl * HALF + ch * (VEC / 2) + i];
    uint4* row = reinterpret_cast<uint4*>(sk + (size_t)pl * kv) + ch;
    for (int h = 0; h < heads; ++h) {
      uint4 raw = row[h * CH];
      const T* kin = reinterpret_cast<const T*>(&raw);
      uint4 out_raw;
      T* kout = reinterpret_cast<T*>(&out_raw);
#pragma unroll
      for (int e = 0; e < VEC; e += 2) {
        double x0, x1;
        if constexpr (sizeof(T) == 4) {
          x0 = (double)kin[e];
          x1 = (double)kin[e + 1];
        } else {
          x0 = (double)__bfloat162float(kin[e]);
          x1 = (double)__bfloat162float(kin[e + 1]);
        }
        const double2 c = c_s[e / 2];
        const double r0 = __dsub_rn(__dmul_rn(c.x, x0), __dmul_rn(c.y, x1));
        const double r1 = __dadd_rn(__dmul_rn(c.y, x0), __dmul_rn(c.x, x1));
        if constexpr (sizeof(T) == 4) {
          kout[e] = __double2float_rn(r0);
          kout[e + 1] = __double2float_rn(r1);
        } else {
          kout[e] = __float2bfloat16_rn(__double2float_rn(r0));
          kout[e + 1] = __float2bfloat16_rn(__double2float_rn(r1));
        }
      }
      row[h * CH] = out_raw;
    }
  }
  sm100::fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk copy
  __syncthreads();
  if (threadIdx.x == 0) {
    bulk_s2g(ctx_k + dst, sk, bytes);
    bulk_commit_wait_read();  // both stores complete (and have read shared memory) before the CTA exits
  }
}

template <typename T>
__global__ void __launch_bounds__(256) realign_graft_kernel(
    const T* __restrict__ k_pre, const T* __restrict__ v_src, int n, int kv, int dh,
    const double2* __restrict__ rope, int base, T* __restrict__ ctx_k, T* __restrict__ ctx_v,
    size_t ctx_layer_stride, int skip_lo, int skip_hi) {
  constexpr int VEC = 16 / sizeof(T);  // elements per 16-byte vector
  int l = blockIdx.y;
  if (skip_hi >= skip_lo && l >= skip_lo) l += skip_hi - skip_lo + 1;
  const int vpr = kv / VEC;  // vectors per row
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)n * vpr) return;
  const int p = (int)(t / vpr);
  const int off = (int)(t % vpr) * VEC;
  const size_t src = (size_t)l * n * kv + (size_t)p * kv + off;
  const uint4 kraw = __ldcs(reinterpret_cast<const uint4*>(k_pre + src));
  const uint4 vraw = __ldcs(reinterpret_cast<const uint4*>(v_src + src));
  const size_t dst = (size_t)l * ctx_layer_stride + (size_t)(base + p) * kv + off;
  *reinterpret_cast<uint4*>(ctx_v + dst) = vraw;
  const double2* cs = rope + (size_t)(base + p) * (dh / 2);
  const T* kin = reinterpret_cast<const T*>(&kraw);
  uint4 kout_raw;
  T* kout = reinterpret_cast<T*>(&kout_raw);
#pragma unroll
  for (int e = 0; e < VEC; e += 2) {
    const double2 c_s = cs[((off + e) % dh) / 2];
    double x0, x1;
    if constexpr (sizeof(T) == 4) {
      x0 = (double)kin[e];
      x1 = (double)kin[e + 1];
    } else {
      x0 = (double)__bfloat162float(kin[e]);
      x1 = (double)__bfloat162float(kin[e + 1]);
    }
    const double r0 = __dsub_rn(__dmul_rn(c_s.x, x0), __dmul_rn(c_s.y, x1));
    const double r1 = __dadd_rn(__dmul_rn(c_s.y, x0), __dmul_rn(c_s.x, x1));
    if constexpr (sizeof(T) == 4) {
      kout[e] = __double2float_rn(r0);
      kout[e + 1] = __double2float_rn(r1);
    } else {
      kout[e] = __float2bfloat16_rn(__double2float_rn(r0));
      kout[e + 1] = __float2bfloat16_rn(__double2float_rn(r1));
    }
  }
  *reinterpret_cast<uint4*>(ctx_k + dst) = kout_raw;
}

// ---------------------------------------------------------------------------
// K2 deviation scoring at l_det (relay_engine.cpp:270-277):
//   s_dev[j]     = mean_head_cosine_deviation(ctx V[l_det][base+j], cache V[l_det][j])
//   s_key_dev[j] = same for ctx K[l_det][base+j] vs realigned cache K (rotated
//                  on the fly from K_pre, bit-identical to realign()).
// cosine_d (metrics.cpp:21-32): sequential double dot/norms per head slice;
// zero-norm -> 0; bit-identical slices -> exactly 1; clamp. Heads are summed
// in order (metrics.cpp:99-102). One thread per (token, head, {V,K}).
// ---------------------------------------------------------------------------
__device__ double cosine_slice(const void* a, size_t ai, const void* b, size_t bi, size_t elem,
                               int dh, const double2* cs, bool rotate_b) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  bool same = true;
  for (int i = 0; i < dh; i += 2) {
    float x0 = load_elem(a, ai + i, elem), x1 = load_elem(a, ai + i + 1, elem);
    float y0 = load_elem(b, bi + i, elem), y1 = load_elem(b, bi + i + 1, elem);
    if (rotate_b) {
      const double2 c = cs[i / 2];
      const double r0 = __dsub_rn(__dmul_rn(c.x, (double)y0), __dmul_rn(c.y, (double)y1));
      const double r1 = __dadd_rn(__dmul_rn(c.y, (double)y0), __dmul_rn(c.x, (double)y1));
      y0 = __double2float_rn(r0);
      y1 = __double2float_rn(r1);
      if (elem == 2) {  // realigned keys are stored in the context's bf16
        y0 = __bfloat162float(__float2bfloat16_rn(y0));
        y1 = __bfloat162float(__float2bfloat16_rn(y1));
      }
    }
    same = same && __float_as_uint(x0) == __float_as_uint(y0) && __float_as_uint(x1) == __float_as_uint(y1);
    const double a0 = x0, a1 = x1, b0 = y0, b1 = y1;
    dot = __dadd_rn(dot, __dmul_rn(a0, b0));
    na = __dadd_rn(na, __dmul_rn(a0, a0));
    nb = __dadd_rn(nb, __dmul_rn(b0, b0));
    dot = __dadd_rn(dot, __dmul_rn(a1, b1));
    na = __dadd_rn(na, __dmul_rn(a1, a1));
    nb = __dadd_rn(nb, __dmul_rn(b1, b1));
  }
  const double sa = __dsqrt_rn(na), sb = __dsqrt_rn(nb);
  if (sa < 1e-12 || sb < 1e-12) return 0.0;
  if (same) return 1.0;
  const double c = __ddiv_rn(dot, __dmul_rn(sa, sb));
  return c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
}

// Copy `bytes` from global to shared with 16-byte vectors when both sides allow.
__device__ __forceinline__ void stage_bytes(void* dst, const void* src, size_t bytes) {
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | bytes) & 15) == 0) {
    const uint4* s4 = static_cast<const uint4*>(src);
    uint4* d4 = static_cast<uint4*>(dst);
    for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) d4[i] = __ldcs(s4 + i);
  } else {
    const unsigned short* s2 = static_cast<const unsigned short*>(src);
    unsigned short* d2 = static_cast<unsigned short*>(dst);
    for (size_t i = threadIdx.x; i < bytes / 2; i += blockDim.x) d2[i] = s2[i];
  }
}

// One CTA scores `tok` consecutive tokens: their four rows (ctx V, cache V,
// ctx K, cache K_pre) are staged in shared memory with coalesced 16-byte loads
// (the HBM-bound part), then one thread per (token, head, {V,K}) runs the
// reference's sequential double loops out of shared memory.
__global__ void __launch_bounds__(256) score_kernel(const void* ctx_v, const void* cache_v, const void* ctx_k,
                                                    const void* cache_kpre, size_t elem, int n, int kv, int heads,
                                                    int dh, const double2* rope, int base, double* s_dev,
                                                    double* s_key, int tok) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int j0 = blockIdx.x * tok;
  const int nt = min(tok, n - j0);
  const size_t row = (size_t)kv * elem, blk = (size_t)tok * row;
  uint8_t* s_cv = sm;             // ctx V rows
  uint8_t* s_rv = sm + blk;       // cache V rows
  uint8_t* s_ck = sm + 2 * blk;   // ctx K rows
  uint8_t* s_rk = sm + 3 * blk;   // cache K_pre rows
  double* cosv = reinterpret_cast<double*>(sm + 4 * blk);  // [tok][2][heads]
  const size_t off = (size_t)j0 * row;
  stage_bytes(s_cv, static_cast<const uint8_t*>(ctx_v) + off, nt * row);
  stage_bytes(s_rv, static_cast<const uint8_t*>(cache_v) + off, nt * row);
  stage_bytes(s_ck, static_cast<const uint8_t*>(ctx_k) + off, nt * row);
  stage_bytes(s_rk, static_cast<const uint8_t*>(cache_kpre) + off, nt * row);
  __syncthreads();
  for (int w = threadIdx.x; w < nt * 2 * heads; w += blockDim.x) {
    const int t = w / (2 * heads), which = (w / heads) % 2, h = w % heads;
    const size_t ai = (size_t)t * kv + h * dh;
    double c;
    if (which == 0)
      c = cosine_slice(s_cv, ai, s_rv, ai, elem, dh, nullptr, false);
    else
      c = cosine_slice(s_ck, ai, s_rk, ai, elem, dh, rope + (size_t)(base + j0 + t) * (dh / 2), true);
    cosv[(t * 2 + which) * heads + h] = c;
  }
  __syncthreads();
  for (int w = threadIdx.x; w < nt * 2; w += blockDim.x) {
    const int t = w / 2, which = w % 2;
    double acc = 0.0;
    for (int hh = 0; hh < heads; ++hh) acc = __dadd_rn(acc, cosv[(t * 2 + which) * heads + hh]);
    (which == 0 ? s_dev : s_key)[j0 + t] = __dsub_rn(1.0, __ddiv_rn(acc, (double)heads));
  }
}

// Fast path for d_head 64/128: one thread per (token, {V,K}, head) holds its
// two head slices in registers (16-byte loads, all in flight at once) and runs
// the reference's sequential double loops (cosine_d) on them; heads are then
// summed in order through shared memory. Same operation order as
// cosine_slice, so the scores are bit-identical.
template <typename T, int DH>
__device__ __forceinline__ float elem_f(const uint4 (&v)[DH * sizeof(T) / 16], int i) {
  const T* p = reinterpret_cast<const T*>(&v[0]);
  if constexpr (sizeof(T) == 4) return p[i];
  else return __bfloat162float(p[i]);
}

template <typename T, int DH>
__global__ void __launch_bounds__(256) score_dh_kernel(const T* __restrict__ ctx_v, const T* __restrict__ cache_v,
                                                       const T* __restrict__ ctx_k, const T* __restrict__ cache_kpre,
                                                       int n, int heads, const double2* __restrict__ rope,
                                                       int base, double* __restrict__ s_dev,
                                                       double* __restrict__ s_key) {
  sm100::pdl_trigger();
  constexpr int NV = DH * sizeof(T) / 16;  // 16-byte vectors per head slice
  extern __shared__ double cosv[];          // [tokens of this CTA][2][heads], then the cos/sin rows
  const int per_tok = 2 * heads;
  const int tok = blockDim.x / per_tok;
  const int t = threadIdx.x / per_tok, which = (threadIdx.x / heads) % 2, h = threadIdx.x % heads;
  const int j = blockIdx.x * tok + t;
  const int kv = heads * DH;
  // the CTA's rows of the (constant, host-built) double cos/sin table, staged
  // before the dependency wait: the K rotation reads them from shared memory
  // instead of 32 dependent L2 loads inside its sequential loop
  double2* cs_sm = reinterpret_cast<double2*>(cosv + (size_t)tok * per_tok);
  {
    const int nt = min(tok, n - (int)blockIdx.x * tok);
    for (int i = threadIdx.x; i < nt * (DH / 2); i += blockDim.x)
      cs_sm[i] = rope[(size_t)(base + blockIdx.x * tok) * (DH / 2) + i];
  }
  __syncthreads();
  sm100::pdl_wait();
  if (t < tok && j < n) {
    const size_t off = (size_t)j * kv + (size_t)h * DH;
    const T* a = which == 0 ? ctx_v : ctx_k;
    const T* b = which == 0 ? cache_v : cache_kpre;
    uint4 x[NV], y[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      x[i] = __ldcs(reinterpret_cast<const uint4*>(a + off) + i);
      y[i] = __ldcs(reinterpret_cast<const uint4*>(b + off) + i);
    }
    const double2* cs = cs_sm + t * (DH / 2);
    double dot = 0.0, na = 0.0, nb = 0.0;
    bool same = true;
#pragma unroll  // fully: the slices stay in registers (compile-time indices)
    for (int i = 0; i < DH; i += 2) {
      const float x0 = elem_f<T, DH>(x, i), x1 = elem_f<T, DH>(x, i + 1);
      float y0 = elem_f<T, DH>(y, i), y1 = elem_f<T, DH>(y, i + 1);
      if (which == 1) {  // realigned key, bit-identical to realign()
        const double2 c = cs[i / 2];
        const double r0 = __dsub_rn(__dmul_rn(c.x, (double)y0), __dmul_rn(c.y, (double)y1));
        const double r1 = __dadd_rn(__dmul_rn(c.y, (double)y0), __dmul_rn(c.x, (double)y1));
        y0 = __double2float_rn(r0);
        y1 = __double2float_rn(r1);
        if constexpr (sizeof(T) == 2) {
          y0 = __bfloat162float(__float2bfloat16_rn(y0));
          y1 = __bfloat162float(__float2bfloat16_rn(y1));
        }
      }
      same = same && __float_as_uint(x0) == __float_as_uint(y0) && __float_as_uint(x1) == __float_as_uint(y1);
      const double a0 = x0, a1 = x1, b0 = y0, b1 = y1;
      dot = __dadd_rn(dot, __dmul_rn(a0, b0));
      na = __dadd_rn(na, __dmul_rn(a0, a0));
      nb = __dadd_rn(nb, __dmul_rn(b0, b0));
      dot = __dadd_rn(dot, __dmul_rn(a1, b1));
      na = __dadd_rn(na, __dmul_rn(a1, a1));
      nb = __dadd_rn(nb, __dmul_rn(b1, b1));
    }
    const double sa = __dsqrt_rn(na), sb = __dsqrt_rn(nb);
    double c;
    if (sa < 1e-12 || sb < 1e-12) c = 0.0;
    else if (same) c = 1.0;
    else {
      c = __ddiv_rn(dot, __dmul_rn(sa, sb));
      c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
    }
    cosv[(t * 2 + which) * heads + h] = c;
  }
  __syncthreads();
  if (threadIdx.x < tok * 2) {
    const int tt = threadIdx.x / 2, w = threadIdx.x % 2;
    const int jj = blockIdx.x * tok + tt;
    if (jj < n) {
      double acc = 0.0;
      for (int hh = 0; hh < heads; ++hh) acc = __dadd_rn(acc, cosv[(tt * 2 + w) * heads + hh]);
      (w == 0 ? s_dev : s_key)[jj] = __dsub_rn(1.0, __ddiv_rn(acc, (double)heads));
    }
  }
}

// bf16 storage (the throughput mode, whose K/V already differ from the
// reference's): one warp per (token, {V,K}) row, EPL = kv/32 elements per lane
// (one head spans DH/EPL lanes), 16-byte loads, per-lane double partial sums
// combined across the head's lanes by shuffles, heads summed in order. The
// key rotation is the double one of realign() (same bf16 rounding), so an
// unchanged key still scores exactly 1. Not the reference's sequential order
// (the fp32-exact path keeps score_dh_kernel): ~1e-16 relative on a cosine.
// The per-thread sequential double loops were latency-bound at ~0.08 of HBM.
template <int DH, int EPL>
__global__ void __launch_bounds__(256) score_bf16_warp_kernel(const __nv_bfloat16* __restrict__ ctx_v,
                                                              const __nv_bfloat16* __restrict__ cache_v,
                                                              const __nv_bfloat16* __restrict__ ctx_k,
                                                              const __nv_bfloat16* __restrict__ cache_kpre, int n,
                                                              int heads, const double2* __restrict__ rope, int base,
                                                              double* __restrict__ s_dev, double* __restrict__ s_key) {
  sm100::pdl_trigger();
  constexpr int LPH = DH / EPL;  // lanes per head
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int j = gw >> 1, which = gw & 1;  // row j, 0 = V, 1 = K
  if (j >= n) return;
  const int e0 = (lane % LPH) * EPL;  // first element within the head
  // the (constant) cos/sin of the key rotation load before the dependency wait
  double2 cs[EPL / 2];
  if (which == 1) {
    const double2* cr = rope + (size_t)(base + j) * (DH / 2) + e0 / 2;
#pragma unroll
    for (int i = 0; i < EPL / 2; ++i) cs[i] = __ldg(cr + i);
  }
  sm100::pdl_wait();
  const int kv = heads * DH;
  const size_t off = (size_t)j * kv + (size_t)lane * EPL;
  const __nv_bfloat16* a = (which == 0 ? ctx_v : ctx_k) + off;
  const __nv_bfloat16* b = (which == 0 ? cache_v : cache_kpre) + off;
  uint4 x[EPL / 8], y[EPL / 8];
#pragma unroll
  for (int i = 0; i < EPL / 8; ++i) {
    x[i] = __ldcs(reinterpret_cast<const uint4*>(a) + i);
    y[i] = __ldcs(reinterpret_cast<const uint4*>(b) + i);
  }
  double dot = 0.0, na = 0.0, nb = 0.0;
  bool same = true;
#pragma unroll
  for (int i = 0; i < EPL; i += 2) {
    const __nv_bfloat16* xp = reinterpret_cast<const __nv_bfloat16*>(x);
    const __nv_bfloat16* yp = reinterpret_cast<const __nv_bfloat16*>(y);
    const float x0 = __bfloat162float(xp[i]), x1 = __bfloat162float(xp[i + 1]);
    float y0 = __bfloat162float(yp[i]), y1 = __bfloat162float(yp[i + 1]);
    if (which == 1) {  // realigned key, bit-identical to realign()
      const double2 c = cs[i / 2];
      const double r0 = __dsub_rn(__dmul_rn(c.x, (double)y0), __dmul_rn(c.y, (double)y1));
      const double r1 = __dadd_rn(__dmul_rn(c.y, (double)y0), __dmul_rn(c.x, (double)y1));
      y0 = __bfloat162float(__float2bfloat16_rn(__double2float_rn(r0)));
      y1 = __bfloat162float(__float2bfloat16_rn(__double2float_rn(r1)));
    }
    same = same && __float_as_uint(x0) == __float_as_uint(y0) && __float_as_uint(x1) == __float_as_uint(y1);
    dot = fma((double)x0, (double)y0, fma((double)x1, (double)y1, dot));
    na = fma((double)x0, (double)x0, fma((double)x1, (double)x1, na));
    nb = fma((double)y0, (double)y0, fma((double)y1, (double)y1, nb));
  }
#pragma unroll
  for (int o = LPH / 2; o; o >>= 1) {  // within the head's lanes
    dot += __shfl_xor_sync(0xffffffffu, dot, o);
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
  }
  // every lane of a head now holds its sums; the head's cosine
  const unsigned head_mask = (LPH == 32 ? 0xffffffffu : ((1u << LPH) - 1u)) << (lane / LPH * LPH);
  same = (__ballot_sync(0xffffffffu, !same) & head_mask) == 0;  // every element of the head unchanged
  const double sa = sqrt(na), sb = sqrt(nb);
  double c;
  if (sa < 1e-12 || sb < 1e-12) c = 0.0;
  else if (same) c = 1.0;
  else c = fmin(1.0, fmax(-1.0, dot / (sa * sb)));
  // heads summed in order by lane 0 (head h's value from lane h * LPH)
  double acc = 0.0;
  for (int h = 0; h < heads; ++h) acc += __shfl_sync(0xffffffffu, c, h * LPH);
  if (lane == 0) (which == 0 ? s_dev : s_key)[j] = 1.0 - acc / (double)heads;
}

// ---------------------------------------------------------------------------
// K2b selection (selector.cpp:32-88): mean-relative thresholds with the
// reference's sequential double mean, suffix window, sorted union with tag
// bits via a block-wide scan compaction. One CTA.
// info: [0] count [1] dev [2] inf-score [3] inf-suffix [4] blend
// dinfo: [0] dev threshold (0 if none) [1] min relative margin
// ---------------------------------------------------------------------------
__device__ void block_compact(const uint32_t* flags_smem_unused, int n, const uint32_t* flags,
                              int* sel_idx, uint32_t* sel_tags, int* info) {
  __shared__ int warp_sums[32];
  __shared__ int running;
  __shared__ int cnt[4];
  if (threadIdx.x == 0) { running = 0; cnt[0] = cnt[1] = cnt[2] = cnt[3] = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (int chunk = 0; chunk < n; chunk += blockDim.x) {
    const int j = chunk + threadIdx.x;
    const uint32_t f = j < n ? flags[j] : 0u;
    const int pred = f != 0;
    c0 += (f & RK_SEL_DEVIATION) != 0;
    c1 += (f & RK_SEL_INFLUENCE_SCORE) != 0;
    c2 += (f & RK_SEL_INFLUENCE_SUFFIX) != 0;
    c3 += (f & RK_SEL_BLEND_TOPK) != 0;
    const unsigned ballot = __ballot_sync(0xffffffffu, pred);
    const int within = __popc(ballot & ((1u << lane) - 1u));
    if (lane == 0) warp_sums[wid] = __popc(ballot);
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane < nw) warp_sums[lane] = v;  // inclusive
    }
    __syncthreads();
    const int warp_off = wid == 0 ? 0 : warp_sums[wid - 1];
    if (pred) {
      const int pos = running + warp_off + within;
      sel_idx[pos] = j;
      sel_tags[pos] = f;
    }
    __syncthreads();
    if (threadIdx.x == 0) running += warp_sums[nw - 1];
    __syncthreads();
  }
  atomicAdd(&cnt[0], c0);
  atomicAdd(&cnt[1], c1);
  atomicAdd(&cnt[2], c2);
  atomicAdd(&cnt[3], c3);
  __syncthreads();
  if (threadIdx.x == 0) {
    info[0] = running;
    info[1] = cnt[0];
    info[2] = cnt[1];
    info[3] = cnt[2];
    info[4] = cnt[3];
  }
}

// mean_relative's threshold (selector.cpp:37-39): sequential double sum, then
// divide, then tau * mean. Warp 0 loads 4 x 32 values per round (coalesced,
// all in flight); the dependent DADD chain walks them in index order via
// shuffles, every lane computing the identical chain.
__device__ double seq_threshold_warp(const double* s_dev, int n, double tau, bool& valid) {
  // The reference's sequential double sum (selector.cpp:37-39): the warp
  // stages 1024 scores at a time in shared memory and lane 0 runs the add
  // chain from there (the loads are off the chain; the chain is DADD-latency bound).
  __shared__ double buf[1024];
  const int lane = threadIdx.x & 31;
  double mean = 0.0;
  for (int b = 0; b < n; b += 1024) {
    const int m = min(1024, n - b);
    __syncwarp();
    for (int i = lane; i < m; i += 32) buf[i] = s_dev[b + i];
    __syncwarp();
    if (lane == 0) {
#pragma unroll 8
      for (int i = 0; i < m; ++i) mean = __dadd_rn(mean, buf[i]);
    }
  }
  mean = __shfl_sync(0xffffffffu, mean, 0);
  mean = __ddiv_rn(mean, (double)n);
  valid = mean > 0.0;
  return __dmul_rn(tau, mean);
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bp = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bp)), __dsub_rn(b, bp));
}

// Selection with a certified parallel threshold: the sequential sum differs
// from the exact sum by at most (n-1) u sum|s_j| (u = 2^-53), and the divide
// and tau-multiply add two roundings. The exact sum comes from a compensated
// (TwoSum) block reduction; any token within that bound of the threshold
// sends the block to the reference's sequential order (rare), otherwise every
// decision s_j >= thr equals the reference's. The exact reported threshold
// and margin are computed off the critical path (seq_threshold_report_kernel
// on the engine's side stream).
__global__ void __launch_bounds__(1024) select_relay_kernel(
    const double* s_dev, const float* influence, const double* infl_mean, int n, double tau_dev,
    double tau_inf, int suffix_k, uint32_t* flags, int* sel_idx, uint32_t* sel_tags, int* info) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  __shared__ double thr[2], margin_abs;
  __shared__ int valid[2], uncertain;
  __shared__ double red_hi[32], red_lo[32];
  double hi = 0.0, lo = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double e;
    two_sum(hi, s_dev[j], hi, e);
    lo = __dadd_rn(lo, e);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o), l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    double e;
    two_sum(hi, h2, hi, e);
    lo = __dadd_rn(__dadd_rn(lo, l2), e);
  }
  if ((threadIdx.x & 31) == 0) {
    red_hi[threadIdx.x >> 5] = hi;
    red_lo[threadIdx.x >> 5] = lo;
  }
  if (threadIdx.x == 0) uncertain = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double H = 0.0, Lo = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      double e;
      two_sum(H, red_hi[w], H, e);
      Lo = __dadd_rn(__dadd_rn(Lo, red_lo[w]), e);
    }
    const double S = __dadd_rn(H, Lo);  // s_dev >= 0: S > 0 iff some s_j > 0 iff the sequential mean > 0
    valid[0] = S > 0.0;
    thr[0] = __dmul_rn(tau_dev, __ddiv_rn(S, (double)n));
    margin_abs = __dmul_rn(thr[0], ((double)n + 16.0) * 2.3e-16);
    const double mi = *infl_mean;
    valid[1] = mi > 0.0;
    thr[1] = __dmul_rn(tau_inf, mi);
  }
  __syncthreads();
  if (valid[0]) {
    bool near = false;
    for (int j = threadIdx.x; j < n; j += blockDim.x) near |= fabs(__dsub_rn(s_dev[j], thr[0])) <= margin_abs;
    if (__any_sync(0xffffffffu, near) && (threadIdx.x & 31) == 0) atomicOr(&uncertain, 1);
  }
  __syncthreads();
  if (uncertain && threadIdx.x < 32) {  // fall back to the reference's sequential order
    bool v;
    const double t = seq_threshold_warp(s_dev, n, tau_dev, v);
    if (threadIdx.x == 0) {
      thr[0] = t;
      valid[0] = v;
    }
  }
  __syncthreads();
  const int start = suffix_k >= n ? 0 : n - suffix_k;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    uint32_t f = 0;
    if (valid[0] && s_dev[j] >= thr[0]) f |= RK_SEL_DEVIATION;
    if (valid[1] && (double)influence[j] >= thr[1]) f |= RK_SEL_INFLUENCE_SCORE;
    if (suffix_k > 0 && j >= start) f |= RK_SEL_INFLUENCE_SUFFIX;
    flags[j] = f;
  }
  __syncthreads();
  block_compact(nullptr, n, flags, sel_idx, sel_tags, info);
}

// Reported values (rk_relay_output::dev_threshold / min_dev_margin): the
// reference's exact sequential threshold and the smallest relative distance of
// any score to it. Runs on the side stream, concurrent with the next layers.
// dinfo: [0] threshold (0 if none) [1] min relative margin
__global__ void __launch_bounds__(1024) seq_threshold_report_kernel(const double* s_dev, int n, double tau_dev,
                                                                    double* dinfo) {
  __shared__ double thr;
  __shared__ int valid;
  __shared__ double mred[32];
  if (threadIdx.x < 32) {
    bool v;
    const double t = seq_threshold_warp(s_dev, n, tau_dev, v);
    if (threadIdx.x == 0) {
      thr = t;
      valid = v;
    }
  }
  __syncthreads();
  double margin = 1e300;
  if (valid)
    for (int j = threadIdx.x; j < n; j += blockDim.x) margin = fmin(margin, fabs(s_dev[j] - thr) / thr);
  for (int o = 16; o > 0; o >>= 1) margin = fmin(margin, __shfl_xor_sync(0xffffffffu, margin, o));
  if ((threadIdx.x & 31) == 0) mred[threadIdx.x >> 5] = margin;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 1e300;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, mred[w]);
    dinfo[0] = valid ? thr : 0.0;
    dinfo[1] = valid ? m : __longlong_as_double(0x7ff0000000000000LL);
  }
}

// BLEND score (relay_engine.cpp:318-330): L2 norm of fresh-vs-stale V at layer 1.
__global__ void blend_score_kernel(const void* ctx_v, const void* cache_v, size_t elem, int n,
                                   int kv, double* score) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
  for (int e = 0; e < kv; ++e) {
    const double diff = __dsub_rn((double)load_elem(ctx_v, (size_t)j * kv + e, elem),
                                  (double)load_elem(cache_v, (size_t)j * kv + e, elem));
    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
  }
  score[j] = __dsqrt_rn(acc);
}

// top_k_by_score (selector.cpp:90-105): the `count` largest scores, ties by
// ascending index (the reference's stable sort by score desc), as a radix
// select in one CTA. Scores are non-negative doubles (L2 norms), so their bit
// patterns order like the values: eight MSB-first passes of an 8-bit digit
// histogram pin the exact key T of the count-th largest score and how many of
// the keys equal to T are still needed; a final pass in index order flags
// every key > T and the first `need` keys == T, then the block compaction
// writes the ascending index list. O(8n) reads instead of O(n^2) rank counting.
__global__ void __launch_bounds__(1024) topk_radix_kernel(const double* __restrict__ score, int n, int count,
                                                          uint32_t* flags, int* sel_idx, uint32_t* sel_tags,
                                                          int* info) {
  __shared__ int hist[256];
  __shared__ unsigned long long s_prefix;
  __shared__ int s_need;
  __shared__ int warp_sums[32];
  __shared__ int running;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int k = count < n ? count : n;
  if (threadIdx.x == 0) { s_prefix = 0ull; s_need = k; running = 0; }
  __syncthreads();
  unsigned long long mask = 0ull;
  if (k > 0 && k < n) {
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
      __syncthreads();
      const unsigned long long prefix = s_prefix;
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const unsigned long long key = (unsigned long long)__double_as_longlong(score[j]);
        if ((key & mask) == prefix) atomicAdd(&hist[(int)((key >> shift) & 255ull)], 1);
      }
      __syncthreads();
      if (wid == 0) {  // lane l covers digits 255-8l .. 248-8l, scanned from the top
        int c[8], sum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) { c[i] = hist[255 - 8 * lane - i]; sum += c[i]; }
        int incl = sum;
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        const int want = s_need, excl = incl - sum;
        if (excl < want && want <= incl) {
          int cum = excl;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (cum + c[i] >= want) {
              s_prefix = prefix | ((unsigned long long)(255 - 8 * lane - i) << shift);
              s_need = want - cum;
              break;
            }
            cum += c[i];
          }
        }
      }
      mask |= 255ull << shift;
      __syncthreads();
    }
  }
  const unsigned long long T = s_prefix;
  const int need = s_need;  // keys == T to take, lowest indices first
  for (int chunk = 0; chunk < n; chunk += blockDim.x) {
    const int j = chunk + threadIdx.x;
    const unsigned long long key = j < n ? (unsigned long long)__double_as_longlong(score[j]) : 0ull;
    const bool eq = j < n && k > 0 && k < n && key == T;
    const unsigned ballot = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) warp_sums[wid] = __popc(ballot);
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (lane < nw) warp_sums[lane] = v;  // inclusive
    }
    __syncthreads();
    const int rank_eq = running + (wid == 0 ? 0 : warp_sums[wid - 1]) + __popc(ballot & ((1u << lane) - 1u));
    if (j < n) {
      const bool take = k >= n || (k > 0 && (key > T || (eq && rank_eq < need)));
      flags[j] = take ? RK_SEL_BLEND_TOPK : 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) running += warp_sums[nw - 1];
    __syncthreads();
  }
  __syncthreads();  // flags (global) written by this CTA are visible to it after the barrier
  block_compact(nullptr, n, flags, sel_idx, sel_tags, info);
}


__global__ void seq_mean_kernel(const float* x, int n, double* out) {
  double m = 0.0;
  for (int j = 0; j < n; ++j) m = __dadd_rn(m, (double)x[j]);
  *out = __ddiv_rn(m, (double)n);
}

// Decode-capture step bookkeeping: a graph-replayed decode step reads its
// index from device memory (step_begin: the row's position and token), and
// step_end moves the step's captured rows from fixed staging buffers to their
// slots in the relay cache, stores the next token and advances the index.
__global__ void decode_step_begin_kernel(const int* step, int src, const int* tokens, int* cur_tok, int* pos) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  if (threadIdx.x == 0) {
    const int t = *step;
    pos[0] = src + t;
    cur_tok[0] = tokens[t];
  }
}
__global__ void decode_step_end_kernel(int* step, int n, int L, int row_words, const uint32_t* stage_k,
                                       const uint32_t* stage_v, uint32_t* k_pre, uint32_t* v, int hid_words,
                                       const uint32_t* stage_h, uint32_t* hidden, const int* next_tok, int* tokens) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int t = *step;
  for (int i = threadIdx.x; i < L * row_words; i += blockDim.x) {
    const int l = i / row_words, w = i - l * row_words;
    const size_t dst = ((size_t)l * n + t) * row_words + w;
    k_pre[dst] = stage_k[i];
    v[dst] = stage_v[i];
  }
  if (hidden)
    for (int i = threadIdx.x; i < hid_words; i += blockDim.x) hidden[(size_t)t * hid_words + i] = stage_h[i];
  __syncthreads();  // every thread has read *step
  if (threadIdx.x == 0) {
    if (next_tok) tokens[t + 1] = *next_tok;
    *step = t + 1;
  }
}

}  // namespace

namespace k {

void init_uniform(cudaStream_t s, float* dst, size_t n, uint64_t state0, float scale) {
  init_uniform_kernel<<<blocks_for(n) < 4096 ? blocks_for(n) : 4096, kThreads, 0, s>>>(dst, n, state0, scale);
}
void fill(cudaStream_t s, float* dst, size_t n, float v) {
  fill_kernel<<<blocks_for(n) < 4096 ? blocks_for(n) : 4096, kThreads, 0, s>>>(dst, n, v);
}
void copy_cols_f32(cudaStream_t s, float* dst, size_t ldd, size_t c0, const float* src, size_t lds,
                   size_t rows, size_t cols, size_t cstride) {
  const size_t n = rows * cols;
  copy_cols_kernel<<<blocks_for(n) < 8192 ? blocks_for(n) : 8192, kThreads, 0, s>>>(dst, ldd, c0, src, lds, rows, cols, cstride);
}
void transpose_to_bf16(cudaStream_t s, __nv_bfloat16* dst, size_t ldd, size_t c0, size_t cstride,
                       const float* src, size_t rows, size_t cols, const float* row_gain) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_bf16_kernel<<<grid, dim3(32, 8), 0, s>>>(dst, ldd, c0, cstride, src, rows, cols, row_gain);
}
void f32_to_bf16(cudaStream_t s, __nv_bfloat16* dst, const float* src, size_t n) {
  f32_to_bf16_kernel<<<blocks_for(n) < 8192 ? blocks_for(n) : 8192, kThreads, 0, s>>>(dst, src, n);
}
void bf16_to_f32(cudaStream_t s, float* dst, const __nv_bfloat16* src, size_t n) {
  bf16_to_f32_kernel<<<blocks_for(n) < 8192 ? blocks_for(n) : 8192, kThreads, 0, s>>>(dst, src, n);
}
void copy2d_f32(cudaStream_t s, float* dst, size_t dld, size_t dcs, const float* src, size_t sld,
                size_t scs, size_t rows, size_t cols) {
  const size_t n = rows * cols;
  copy2d_kernel<<<blocks_for(n) < 8192 ? blocks_for(n) : 8192, kThreads, 0, s>>>(dst, dld, dcs, src, sld, scs, rows, cols);
}
void untranspose_bf16(cudaStream_t s, float* dst, const __nv_bfloat16* src, size_t ld, size_t c0,
                      size_t cstride, size_t rows, size_t cols, const float* row_gain) {
  const size_t n = rows * cols;
  untranspose_bf16_kernel<<<blocks_for(n) < 8192 ? blocks_for(n) : 8192, kThreads, 0, s>>>(dst, src, ld, c0, cstride, rows, cols, row_gain);
}
void doubles_to_floats(cudaStream_t s, float* dst, const double* src, int n) {
  d2f_kernel<<<blocks_for(n), kThreads, 0, s>>>(dst, src, n);
}
void embed(cudaStream_t s, float* hidden, const void* emb, size_t elem, const int32_t* tokens,
           int n, int d, int, int*) {
  const size_t total = (size_t)n * d;
  launch_pdl(embed_kernel, dim3(blocks_for(total) < 4096 ? blocks_for(total) : 4096), dim3(kThreads), 0, s, hidden, emb, elem, tokens, n, d);
}
void gather_rows(cudaStream_t s, float* dst, const float* src, const int* idx, const int* count,
                 int rows_max, int d) {
  const size_t total = (size_t)rows_max * d;
  gather_rows_kernel<<<blocks_for(total) < 4096 ? blocks_for(total) : 4096, kThreads, 0, s>>>(dst, src, idx, count, rows_max, d);
}
void scatter_rows(cudaStream_t s, float* dst, const float* src, const int* idx, const int* count,
                  int rows_max, int d, uint64_t* depth, uint64_t depth_value) {
  const size_t total = (size_t)rows_max * d;
  scatter_rows_kernel<<<blocks_for(total) < 4096 ? blocks_for(total) : 4096, kThreads, 0, s>>>(
      dst, src, idx, count, rows_max, d, depth, depth_value);
}
void positions_from_sel(cudaStream_t s, int* pos, const int* sel, const int* count, int rows_max,
                        int base) {
  positions_from_sel_kernel<<<blocks_for(rows_max), kThreads, 0, s>>>(pos, sel, count, rows_max, base);
}
void iota_positions(cudaStream_t s, int* pos, int n, int base) {
  launch_pdl(iota_kernel, dim3(blocks_for(n)), dim3(kThreads), 0, s, pos, n, base);
}
void mark_rows(cudaStream_t s, uint8_t* origin, int len, int lo, int hi, const int* sel,
               const int* count, int rows_max) {
  if (hi < lo) return;
  launch_pdl(mark_rows_kernel, dim3(blocks_for((size_t)rows_max * (hi - lo + 1))), dim3(kThreads), 0, s, origin, len, lo, hi, sel, count, rows_max);
}
void mark_layers(cudaStream_t s, uint8_t* origin, int len, int lo, int hi) {
  if (hi < lo) return;
  launch_pdl(mark_layers_kernel, dim3(blocks_for((size_t)(hi - lo + 1) * len)), dim3(kThreads), 0, s, origin, len, lo, hi);
}
struct ZeroList {
  uint8_t* p[16];
  size_t n[16];
};
__global__ void zero_many_kernel(ZeroList z) {
  sm100::pdl_trigger();
  sm100::pdl_wait();  // (blockIdx.y = buffer)
  uint8_t* dst = z.p[blockIdx.y];
  const size_t n = z.n[blockIdx.y];
  const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (size_t i = i0; i < n / 16; i += stride) d4[i] = make_uint4(0, 0, 0, 0);
    for (size_t i = n / 16 * 16 + i0; i < n; i += stride) dst[i] = 0;
  } else {
    for (size_t i = i0; i < n; i += stride) dst[i] = 0;
  }
}
void zero_many(cudaStream_t s, const std::vector<std::pair<void*, size_t>>& bufs) {
  for (size_t b = 0; b < bufs.size(); b += 16) {
    ZeroList z{};
    size_t mx = 0;
    const int m = (int)std::min<size_t>(16, bufs.size() - b);
    for (int i = 0; i < m; ++i) {
      z.p[i] = static_cast<uint8_t*>(bufs[b + i].first);
      z.n[i] = bufs[b + i].second;
      mx = std::max(mx, z.n[i]);
    }
    if (!mx) continue;
    const unsigned blocks = (unsigned)std::min<size_t>(256, (mx / 16 + kThreads - 1) / kThreads + 1);
    launch_pdl(zero_many_kernel, dim3(dim3(blocks, m)), dim3(kThreads), 0, s, z);
  }
}
void zero_dev(cudaStream_t s, void* dst, size_t bytes) {
  if (!bytes) return;
  const size_t blocks = std::min<size_t>(1184, (bytes / 16 + kThreads - 1) / kThreads + 1);
  launch_pdl(zero_bytes_kernel, dim3((unsigned)blocks), dim3(kThreads), 0, s, static_cast<uint8_t*>(dst), bytes);
}
void decode_step_begin(cudaStream_t s, const int* step, int src, const int* tokens, int* cur_tok, int* pos) {
  launch_pdl(decode_step_begin_kernel, dim3(1), dim3(32), 0, s, step, src, tokens, cur_tok, pos);
}
void decode_step_end(cudaStream_t s, int* step, int n, int L, size_t row_bytes, const void* stage_k,
                     const void* stage_v, void* k_pre, void* v, size_t hid_bytes, const void* stage_h, void* hidden,
                     const int* next_tok, int* tokens) {
  launch_pdl(decode_step_end_kernel, dim3(1), dim3(1024), 0, s, step, n, L, (int)(row_bytes / 4),
             static_cast<const uint32_t*>(stage_k), static_cast<const uint32_t*>(stage_v), static_cast<uint32_t*>(k_pre),
             static_cast<uint32_t*>(v), (int)(hid_bytes / 4), static_cast<const uint32_t*>(stage_h),
             static_cast<uint32_t*>(hidden), next_tok, tokens);
}
__global__ void small_copies_kernel(const SmallCopies c) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int i = blockIdx.x;
  const uint8_t* src = static_cast<const uint8_t*>(c.src[i]);
  uint8_t* dst = static_cast<uint8_t*>(c.dst[i]);
  for (int b = threadIdx.x; b < c.bytes[i]; b += blockDim.x) dst[b] = src[b];
}
void small_copies(cudaStream_t s, const SmallCopies& c) {
  if (c.n > 0) launch_pdl(small_copies_kernel, dim3((unsigned)c.n), dim3(64), 0, s, c);
}
void copy_dev(cudaStream_t s, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  const size_t blocks = std::min<size_t>(1184, (bytes / 16 + kThreads - 1) / kThreads + 1);
  launch_pdl(copy_bytes_kernel, dim3((unsigned)blocks), dim3(kThreads), 0, s, static_cast<uint8_t*>(dst),
                                                          static_cast<const uint8_t*>(src), bytes);
}
void zero_rows(cudaStream_t s, void* dst, size_t pitch, size_t width, size_t rows) {
  if (!width || !rows) return;
  dim3 grid((unsigned)std::min<size_t>(64, (width / 16 + kThreads - 1) / kThreads + 1),
            (unsigned)std::min<size_t>(rows, 1024));
  zero_rows_kernel<<<grid, kThreads, 0, s>>>(static_cast<uint8_t*>(dst), pitch, width, rows);
}
void copy_i32(cudaStream_t s, int* dst, const int* src, int n) {
  if (n > 0) launch_pdl(copy_i32_kernel, dim3(std::min(64, blocks_for(n))), dim3(kThreads), 0, s, dst, src, n);
}
void fill_doubles(cudaStream_t s, double* dst, int n, double v) {
  fill_doubles_kernel<<<blocks_for(n), kThreads, 0, s>>>(dst, n, v);
}
void set_depth(cudaStream_t s, uint64_t* depth, int n, uint64_t v) {
  launch_pdl(set_depth_kernel, dim3(blocks_for(n)), dim3(kThreads), 0, s, depth, n, v);
}
void argmax(cudaStream_t s, const float* x, int n, int* out, void* ws) {
  const int g = std::min(kArgBlocks, blocks_for((size_t)(n + 3) / 4));
  launch_pdl(argmax_partial_kernel, dim3(g), dim3(kThreads), 0, s, x, n, static_cast<float2*>(ws));
  launch_pdl(argmax_final_kernel, dim3(1), dim3(kThreads), 0, s, static_cast<const float2*>(ws), g, out);
}

void realign_graft(cudaStream_t s, const void* k_pre, const void* v_src, size_t elem, int L, int n,
                   int kv, int dh, const double2* rope, int base, void* ctx_k, void* ctx_v,
                   size_t ctx_layer_stride, int skip_lo, int skip_hi) {
  const RealignJob job{k_pre, v_src, n, base};
  realign_graft_batch(s, &job, 1, elem, L, kv, dh, rope, ctx_k, ctx_v, ctx_layer_stride, skip_lo, skip_hi);
}

void realign_graft_batch(cudaStream_t s, const RealignJob* jobs, int count, size_t elem, int L, int kv, int dh,
                         const double2* rope, void* ctx_k, void* ctx_v, size_t ctx_layer_stride, int skip_lo,
                         int skip_hi) {
  const int skipped = skip_hi >= skip_lo ? skip_hi - skip_lo + 1 : 0;
  const int layers = L - skipped;
  if (layers <= 0 || count <= 0) return;
  bool bulk_ok = (dh == 64 || dh == 128) && ((reinterpret_cast<uintptr_t>(ctx_k) | reinterpret_cast<uintptr_t>(ctx_v) |
                                              (kv * elem)) & 15) == 0;
  for (int u = 0; u < count; ++u)
    bulk_ok = bulk_ok && ((reinterpret_cast<uintptr_t>(jobs[u].k_pre) | reinterpret_cast<uintptr_t>(jobs[u].v)) & 15) == 0;
  if (!bulk_ok) {  // generic d_head / alignment: one thread per 16-byte vector
    for (int u = 0; u < count; ++u) {
      const int n = jobs[u].n;
      if (n <= 0) continue;
      const size_t vecs = (size_t)n * (kv * elem / 16);
      dim3 grid((unsigned)((vecs + 255) / 256), (unsigned)layers);
      if (elem == 4)
        realign_graft_kernel<float><<<grid, 256, 0, s>>>(
            (const float*)jobs[u].k_pre, (const float*)jobs[u].v, n, kv, dh, rope, jobs[u].base, (float*)ctx_k,
            (float*)ctx_v, ctx_layer_stride, skip_lo, skip_hi);
      else
        realign_graft_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
            (const __nv_bfloat16*)jobs[u].k_pre, (const __nv_bfloat16*)jobs[u].v, n, kv, dh, rope, jobs[u].base,
            (__nv_bfloat16*)ctx_k, (__nv_bfloat16*)ctx_v, ctx_layer_stride, skip_lo, skip_hi);
    }
    return;
  }
  // fast path: P positions (~16 KB of K and of V) of one segment and one
  // grafted layer per CTA, every segment of the call in one launch
  const int P = (int)std::max<size_t>(1, 16384 / (kv * elem));
  const size_t smem = (size_t)2 * P * kv * elem + (size_t)P * (dh / 2) * 16 + 16;
  for (int u0 = 0; u0 < count; u0 += kMaxRealignJobs) {
    RealignJobs J{};
    J.count = std::min(kMaxRealignJobs, count - u0);
    int blocks = 0;
    for (int i = 0; i < J.count; ++i) {
      const RealignJob& jb = jobs[u0 + i];
      J.k_pre[i] = jb.k_pre;
      J.v[i] = jb.v;
      J.n[i] = jb.n;
      J.base[i] = jb.base;
      J.blk0[i] = blocks;
      blocks += (jb.n + P - 1) / P;
    }
    J.blk0[J.count] = blocks;
    if (blocks == 0) continue;
#define RK_REALIGN_DH(T, D)                                                                                  \
  do {                                                                                                       \
    static bool attr = false;                                                                                \
    if (!attr) {                                                                                             \
      RK_CUDA(cudaFuncSetAttribute(realign_graft_dh_kernel<T, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
      attr = true;                                                                                           \
    }                                                                                                        \
    launch_pdl(realign_graft_dh_kernel<T, D>, dim3(blocks, layers), dim3(128), smem, s, J, kv, rope, (T*)ctx_k, \
               (T*)ctx_v, ctx_layer_stride, skip_lo, skip_hi, P);                                            \
  } while (0)
    if (elem == 4 && dh == 64) RK_REALIGN_DH(float, 64);
    else if (elem == 4) RK_REALIGN_DH(float, 128);
    else if (dh == 64) RK_REALIGN_DH(__nv_bfloat16, 64);
    else RK_REALIGN_DH(__nv_bfloat16, 128);
#undef RK_REALIGN_DH
  }
}

// ---------------------------------------------------------------------------
// Offline profiler: token_deviation (metrics.cpp:118-159) on the device. For
// every (position j, layer l) and both V and K_pre rows of the reuse-side and
// the full-prefill cache: mean-over-heads cosine deviation (cosine_d,
// metrics.cpp:21-32) and norm-ratio deviation (norm_ratio_d, 40-46), in the
// reference's sequential double order. One CTA per (j, l), one thread per
// (row kind, head); heads are summed in order. out: [4][n][L] doubles
// (value_cos, key_cos, value_norm, key_norm), row-major [position][layer].
// ---------------------------------------------------------------------------
__global__ void token_deviation_kernel(const void* rk, const void* rv, const void* fk, const void* fv, size_t elem,
                                       int L, int n, int kv, int heads, double* out) {
  extern __shared__ double dsh[];  // [2 kinds][heads][cos, ratio]
  const int j = blockIdx.x / L, l = blockIdx.x % L;
  const int dh = kv / heads;
  const size_t rowi = ((size_t)l * n + j) * kv;
  for (int t = threadIdx.x; t < 2 * heads; t += blockDim.x) {
    const int which = t / heads, h = t % heads;  // 0 = V, 1 = K_pre
    const void* a = which == 0 ? rv : rk;  // reuse side (metrics.cpp:151-154: a = reuse, b = full)
    const void* b = which == 0 ? fv : fk;
    const size_t ai = rowi + (size_t)h * dh;
    double dot = 0.0, na = 0.0, nb = 0.0;
    bool same = true;
    for (int i = 0; i < dh; ++i) {
      const float x = load_elem(a, ai + i, elem), y = load_elem(b, ai + i, elem);
      same = same && __float_as_uint(x) == __float_as_uint(y);
      const double xd = x, yd = y;
      dot = __dadd_rn(dot, __dmul_rn(xd, yd));
      na = __dadd_rn(na, __dmul_rn(xd, xd));
      nb = __dadd_rn(nb, __dmul_rn(yd, yd));
    }
    const double sa = __dsqrt_rn(na), sb = __dsqrt_rn(nb);
    double c;
    if (sa < 1e-12 || sb < 1e-12) c = 0.0;
    else if (same) c = 1.0;
    else {
      c = __ddiv_rn(dot, __dmul_rn(sa, sb));
      c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
    }
    const double hi = sa > sb ? sa : sb, lo = sa > sb ? sb : sa;
    const double ratio = hi < 1e-12 ? 1.0 : __ddiv_rn(lo, hi);
    dsh[(which * heads + h) * 2] = c;
    dsh[(which * heads + h) * 2 + 1] = ratio;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    const int which = threadIdx.x & 1, metric = threadIdx.x >> 1;  // metric 0 cos, 1 ratio
    double acc = 0.0;
    for (int h = 0; h < heads; ++h) acc = __dadd_rn(acc, dsh[(which * heads + h) * 2 + metric]);
    // out planes: 0 value_cos, 1 key_cos, 2 value_norm, 3 key_norm
    out[((size_t)(metric * 2 + which) * n + j) * L + l] = __dsub_rn(1.0, __ddiv_rn(acc, (double)heads));
  }
}

void token_deviation(cudaStream_t s, const void* reuse_k, const void* reuse_v, const void* full_k,
                     const void* full_v, size_t elem, int L, int n, int kv, int heads, double* out) {
  if (n <= 0 || L <= 0) return;
  const int threads = std::max(32, ((2 * heads + 31) / 32) * 32);
  token_deviation_kernel<<<n * L, threads, (size_t)4 * heads * sizeof(double), s>>>(reuse_k, reuse_v, full_k, full_v,
                                                                                   elem, L, n, kv, heads, out);
  RK_CUDA(cudaGetLastError());
}

void score_deviation(cudaStream_t s, const void* ctx_v, const void* cache_v, const void* ctx_k,
                     const void* cache_kpre, size_t elem, int n, int kv, int heads, int dh,
                     const double2* rope, int base, double* s_dev, double* s_key) {
  if (n <= 0) return;
  const size_t row = (size_t)kv * elem;
  const bool aligned = ((reinterpret_cast<uintptr_t>(ctx_v) | reinterpret_cast<uintptr_t>(cache_v) |
                         reinterpret_cast<uintptr_t>(ctx_k) | reinterpret_cast<uintptr_t>(cache_kpre)) & 15) == 0;
  if (aligned && elem == 2 && (dh == 64 || dh == 128) && kv % 256 == 0 && kv / 32 <= dh && dh % (kv / 32) == 0 &&
      kv / 32 <= 32) {
    const int warps = 2 * n, grid = (warps * 32 + 255) / 256;
#define RK_SCORE_W(D, E)                                                                                         \
  launch_pdl(score_bf16_warp_kernel<D, E>, dim3(grid), dim3(256), 0, s, (const __nv_bfloat16*)ctx_v,             \
             (const __nv_bfloat16*)cache_v, (const __nv_bfloat16*)ctx_k, (const __nv_bfloat16*)cache_kpre, n,    \
             heads, rope, base, s_dev, s_key)
    const int epl = kv / 32;
    if (dh == 64 && epl == 8) RK_SCORE_W(64, 8);
    else if (dh == 64 && epl == 16) RK_SCORE_W(64, 16);
    else if (dh == 64 && epl == 32) RK_SCORE_W(64, 32);
    else if (dh == 128 && epl == 8) RK_SCORE_W(128, 8);
    else if (dh == 128 && epl == 16) RK_SCORE_W(128, 16);
    else RK_SCORE_W(128, 32);
#undef RK_SCORE_W
    return;
  }
  if (aligned && (dh == 64 || dh == 128) && 2 * heads <= 256) {
    // tokens per CTA: at most 256 threads, and few enough that the grid covers
    // every SM about twice (the per-thread double loops are latency-bound)
    static const int sms = [] {
      int dev = 0, v = 148;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      return v;
    }();
    const int tok = std::max(1, std::min(256 / (2 * heads), (n + 2 * sms - 1) / (2 * sms)));
    const size_t smem = (size_t)tok * 2 * heads * sizeof(double) + (size_t)tok * (dh / 2) * 16;
    const int grid = (n + tok - 1) / tok;
#define RK_SCORE_DH(T, D)                                                                                      \
  launch_pdl(score_dh_kernel<T, D>, dim3(grid), dim3(tok * 2 * heads), smem, s, (const T*)ctx_v, (const T*)cache_v, (const T*)ctx_k,          \
                                                (const T*)cache_kpre, n, heads, rope, base, s_dev, s_key)
    if (elem == 4 && dh == 64) RK_SCORE_DH(float, 64);
    else if (elem == 4) RK_SCORE_DH(float, 128);
    else if (dh == 64) RK_SCORE_DH(__nv_bfloat16, 64);
    else RK_SCORE_DH(__nv_bfloat16, 128);
#undef RK_SCORE_DH
    return;
  }
  int tok = (int)std::min<size_t>(16, std::max<size_t>(1, 40960 / (4 * row)));
  const size_t smem = 4 * row * tok + (size_t)tok * 2 * heads * sizeof(double);
  if (smem > 48 * 1024) {
    static bool attr = false;
    if (!attr) {
      RK_CUDA(cudaFuncSetAttribute(score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
  }
  score_kernel<<<(n + tok - 1) / tok, 256, smem, s>>>(ctx_v, cache_v, ctx_k, cache_kpre, elem, n, kv, heads, dh,
                                                      rope, base, s_dev, s_key, tok);
}

void select_relay(cudaStream_t s, const double* s_dev, const float* influence,
                  const double* infl_mean, int n, double tau_dev, double tau_inf, int suffix_k,
                  int* sel_idx, uint32_t* sel_tags, int* info, double* dinfo, cudaStream_t side,
                  cudaEvent_t fork, cudaEvent_t join) {
  // flags scratch lives after sel_tags (caller sizes sel_tags to 2n)
  if (side) {
    RK_CUDA(cudaEventRecord(fork, s));
    RK_CUDA(cudaStreamWaitEvent(side, fork, 0));
    seq_threshold_report_kernel<<<1, 1024, 0, side>>>(s_dev, n, tau_dev, dinfo);
    RK_CUDA(cudaEventRecord(join, side));
  } else {
    seq_threshold_report_kernel<<<1, 1024, 0, s>>>(s_dev, n, tau_dev, dinfo);
  }
  launch_pdl(select_relay_kernel, dim3(1), dim3(1024), 0, s, s_dev, influence, infl_mean, n, tau_dev, tau_inf, suffix_k, sel_tags + n,
                                         sel_idx, sel_tags, info);
}
void blend_scores(cudaStream_t s, const void* ctx_v, const void* cache_v, size_t elem, int n,
                  int kv, double* score) {
  blend_score_kernel<<<blocks_for(n), kThreads, 0, s>>>(ctx_v, cache_v, elem, n, kv, score);
}
void select_topk(cudaStream_t s, const double* score, int n, int count, int* sel_idx,
                 uint32_t* sel_tags, int* info) {
  topk_radix_kernel<<<1, 1024, 0, s>>>(score, n, count, sel_tags + n, sel_idx, sel_tags, info);
}
void seq_mean(cudaStream_t s, const float* x, int n, double* out) {
  seq_mean_kernel<<<1, 1, 0, s>>>(x, n, out);
}

}  // namespace k
}  // namespace rk

// ---------------------------------------------------------------------------
// layer-major fused agent schedule helpers (runner.cpp agent_fused)
// ---------------------------------------------------------------------------
namespace rk {
namespace {
__global__ void segment_offsets_kernel(k::SegCounts c, int U, int start, int* offs) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int o = start;
  for (int u = 0; u < U; ++u) {
    offs[u] = o;
    o += *c.count[u];
  }
  offs[U] = o;
}
// H[off + r] = src[idx[r]]; pos[off + r] = base + idx[r]
__global__ void gather_rows_to_kernel(float* H, const int* off, const float* src, const int* idx, const int* count,
                                      int d, int* pos, int base) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int rows = *count, o = *off;
  if ((d & 3) == 0) {  // 16-byte vectors, 32-bit index math
    const int d4 = d / 4, total = rows * d4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
      const int r = i / d4, c = i - r * d4, j = idx[r];
      reinterpret_cast<float4*>(H + (size_t)(o + r) * d)[c] = reinterpret_cast<const float4*>(src + (size_t)j * d)[c];
      if (c == 0) pos[o + r] = base + j;
    }
    return;
  }
  const size_t total = (size_t)rows * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / d, c = i % d;
    H[(size_t)(o + r) * d + c] = src[(size_t)idx[r] * d + c];
    if (c == 0) pos[o + r] = base + idx[r];
  }
}
// dst[idx[r]] = H[off + r]; depth[idx[r]] = value
__global__ void scatter_rows_from_kernel(float* dst, const float* H, const int* off, const int* idx, const int* count,
                                         int d, uint64_t* depth, uint64_t value) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int rows = *count, o = *off;
  if ((d & 3) == 0) {
    const int d4 = d / 4, total = rows * d4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
      const int r = i / d4, c = i - r * d4, j = idx[r];
      reinterpret_cast<float4*>(dst + (size_t)j * d)[c] = reinterpret_cast<const float4*>(H + (size_t)(o + r) * d)[c];
      if (c == 0) depth[j] = value;
    }
    return;
  }
  const size_t total = (size_t)rows * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / d, c = i % d;
    dst[(size_t)idx[r] * d + c] = H[(size_t)(o + r) * d + c];
    if (c == 0) depth[idx[r]] = value;
  }
}
}  // namespace

namespace k {
void segment_offsets(cudaStream_t s, const SegCounts& c, int U, int start, int* offs) {
  launch_pdl(segment_offsets_kernel, dim3(1), dim3(32), 0, s, c, U, start, offs);
}
void gather_rows_to(cudaStream_t s, float* H, const int* off, const float* src, const int* idx, const int* count,
                    int rows_max, int d, int* pos, int base) {
  const size_t total = (size_t)rows_max * d / (d % 4 ? 1 : 4);
  launch_pdl(gather_rows_to_kernel, dim3(blocks_for(total) < 4096 ? blocks_for(total) : 4096), dim3(kThreads), 0, s, H, off, src, idx, count, d, pos, base);
}
void scatter_rows_from(cudaStream_t s, float* dst, const float* H, const int* off, const int* idx, const int* count,
                       int rows_max, int d, uint64_t* depth, uint64_t value) {
  const size_t total = (size_t)rows_max * d / (d % 4 ? 1 : 4);
  launch_pdl(scatter_rows_from_kernel, dim3(blocks_for(total) < 4096 ? blocks_for(total) : 4096), dim3(kThreads), 0, s, dst, H, off, idx, count, d, depth, value);
}
}  // namespace k
}  // namespace rk
