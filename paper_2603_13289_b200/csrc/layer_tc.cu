// layer_tc.cu -- RK_FP32_TC: the fp32-accurate tensor-core mode.
//
// Storage, context, caches and every relay kernel are the fp32-exact path's
// (realign, deviation scores, selection, RMSNorm, RoPE/commit); what changes
// is the arithmetic of the two hot ops of run_layer_rows (model.cpp:237-280):
//
//  * matmul (tensor.cpp:66-86) as 3xTF32 on tcgen05: x = hi + lo with hi the
//    tf32 truncation of x and lo = x - hi (exact in fp32), and
//    A.B ~= hi_A.hi_B + hi_A.lo_B + lo_A.hi_B -- the dropped lo_A.lo_B term
//    and the tf32 rounding of lo are ~2^-21 relative, so a product row keeps
//    fp32-level accuracy. The three products are one GEMM over a
//    K-concatenation: A' = [hi_A | hi_A | lo_A] (M x 3K), B' = [hi_B | lo_B |
//    hi_B] (N x 3K), run by the bf16 GEMM kernel's kind::tf32 instantiation
//    (fp32 rows are 128-byte TMA/SW128 rows of 32 elements, exactly the byte
//    layout of 64 bf16, so the pipeline is unchanged). Weights are packed
//    [N x 3K] once at upload; activations are split right before each GEMM.
//  * attend_row (model.cpp:170-204) as an fp32 flash attention on the CUDA
//    cores (online softmax over 64-key blocks, fp32 accumulation).
//
// Results are not bit-identical to the reference (the summation order of the
// tensor core differs); the relative error is ~1e-6 per layer output, far
// below north_star's 1e-4 bound for an fp32-accumulate mode.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "internal.h"
#include "layer_bf16.h"
#include "layer_tc.h"
#include "prof.h"
#include "sm100.cuh"

namespace rk {
namespace {

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

__device__ __forceinline__ int live_rows_tc(const Rows& r) { return r.rows_dev ? *r.rows_dev : r.rows_max; }

// dst row r = [hi(src_r) | hi(src_r) | lo(src_r)]  (A side), rows < rows_max
// (rows past the live count are split too: the GEMM reads them, never stores)
__global__ void split3_rows_kernel(const float* __restrict__ src, int lds, float* __restrict__ dst, int rows,
                                   int K) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int k4 = K / 4;
  const long long n = (long long)rows * k4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / k4), c = (int)(i % k4) * 4;
    const float4 x = *reinterpret_cast<const float4*>(src + (size_t)r * lds + c);
    const float4 h = make_float4(tf32_hi(x.x), tf32_hi(x.y), tf32_hi(x.z), tf32_hi(x.w));
    const float4 l = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
    float* d = dst + (size_t)r * 3 * K + c;
    *reinterpret_cast<float4*>(d) = h;
    *reinterpret_cast<float4*>(d + K) = h;
    *reinterpret_cast<float4*>(d + 2 * K) = l;
  }
}

// Weight packing (B side): src is the reference layout [K x ldsrc] (row k,
// column c0 + n * cs holds W[k][n]); dst row n = [hi(W[:,n]) | lo | hi], 3K wide.
__global__ void pack_b3_kernel(const float* __restrict__ src, int ldsrc, int c0, int cs, float* __restrict__ dst,
                               int K, int N) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && n < N) ? src[(size_t)k * ldsrc + c0 + (size_t)n * cs] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K) {
      const float x = tile[threadIdx.x][i], h = tf32_hi(x);
      float* d = dst + (size_t)n * 3 * K;
      d[k] = h;
      d[K + k] = x - h;
      d[2 * K + k] = h;
    }
  }
}

// act[r][j] = silu(gu[r][2j]) * gu[r][2j+1]  (model.cpp:208, 226; fp32)
__global__ void silu_pair_kernel(const float* __restrict__ gu, float* __restrict__ act, Rows rows, int ff) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  const int M = live_rows_tc(rows);
  const long long n = (long long)M * ff;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / ff, j = i % ff;
    const float2 v = *reinterpret_cast<const float2*>(gu + r * 2 * ff + 2 * j);
    act[i] = v.x / (1.0f + expf(-v.x)) * v.y;
  }
}

// ---------------------------------------------------------------------------
// fp32 flash attention (attend_row semantics: query row r at absolute
// position pos_r sees keys 0..pos_r of its layer, kv head = h / (H/Hkv)).
// CTA = 64 query rows x 1 head, 256 threads; thread (ty, tx): rows 4ty..4ty+3,
// score columns tx + 16j (j < 4) of each 64-key block, output columns
// 4tx..4tx+3 (+64 for d_head 128). Q and K staged transposed in shared
// memory, P transposed, V row-major.
// ---------------------------------------------------------------------------
constexpr int kBR = 64, kBC = 64, kPadT = 68;  // padded row length of the transposed tiles

template <int DH>
__global__ void __launch_bounds__(256) attn_f32_kernel(const float* __restrict__ qkv, int ld, Rows rows, int H,
                                                        int Hkv, const float* __restrict__ ck,
                                                        const float* __restrict__ cv, float* __restrict__ out,
                                                        float scale_log2, int* status) {
  sm100::pdl_trigger();
  sm100::pdl_wait();
  extern __shared__ __align__(16) float sm[];
  float* Qt = sm;                   // [DH][kPadT]
  float* Kt = Qt + DH * kPadT;      // [DH][kPadT]
  float* Vs = Kt + DH * kPadT;      // [kBC][DH]
  float* Pt = Vs + kBC * DH;        // [kBC][kPadT]
  __shared__ int s_kmax;
  const int M = live_rows_tc(rows);
  const int r0 = blockIdx.x * kBR;
  if (r0 >= M) return;
  const int h = blockIdx.y, kvh = h / (H / Hkv), kv = Hkv * DH;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int nr = min(kBR, M - r0);
  if (tid == 0) s_kmax = -1;
  __syncthreads();
  if (tid < nr) atomicMax(&s_kmax, rows.pos[r0 + tid]);
  // Q tile, transposed: Qt[d][row]
  for (int i = tid; i < kBR * (DH / 4); i += 256) {
    const int rr = i % kBR, c = (i / kBR) * 4;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rr < nr) x = *reinterpret_cast<const float4*>(qkv + (size_t)(r0 + rr) * ld + h * DH + c);
    Qt[(c + 0) * kPadT + rr] = x.x;
    Qt[(c + 1) * kPadT + rr] = x.y;
    Qt[(c + 2) * kPadT + rr] = x.z;
    Qt[(c + 3) * kPadT + rr] = x.w;
  }
  __syncthreads();
  const int kmax = s_kmax;
  int pos[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) pos[i] = (4 * ty + i < nr) ? rows.pos[r0 + 4 * ty + i] : -1;
  constexpr int OC = DH / 16;  // output columns per thread
  float o[4][OC];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < OC; ++c) o[i][c] = 0.f;
  float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, l[4] = {0.f, 0.f, 0.f, 0.f};
  const int nblk = kmax / kBC + 1;
  for (int b = 0; b < nblk; ++b) {
    const int j0 = b * kBC;
    __syncthreads();  // previous block's Kt / Vs / Pt fully consumed
    for (int i = tid; i < kBC * (DH / 4); i += 256) {
      const int key = i % kBC, c = (i / kBC) * 4;
      float4 x = make_float4(0.f, 0.f, 0.f, 0.f), y = x;
      if (j0 + key <= kmax) {
        x = *reinterpret_cast<const float4*>(ck + (size_t)(j0 + key) * kv + kvh * DH + c);
        y = *reinterpret_cast<const float4*>(cv + (size_t)(j0 + key) * kv + kvh * DH + c);
      }
      Kt[(c + 0) * kPadT + key] = x.x;
      Kt[(c + 1) * kPadT + key] = x.y;
      Kt[(c + 2) * kPadT + key] = x.z;
      Kt[(c + 3) * kPadT + key] = x.w;
      *reinterpret_cast<float4*>(Vs + key * DH + c) = y;
    }
    __syncthreads();
    float s[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 8
    for (int d = 0; d < DH; ++d) {
      const float4 q4 = *reinterpret_cast<const float4*>(Qt + d * kPadT + 4 * ty);
      const float qa[4] = {q4.x, q4.y, q4.z, q4.w};
      float kk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) kk[j] = Kt[d * kPadT + tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = fmaf(qa[i], kk[j], s[i][j]);
    }
    // online softmax (base 2), rows reduced over the 16 tx lanes
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s[i][j] = (j0 + tx + 16 * j <= pos[i]) ? s[i][j] * scale_log2 : -INFINITY;
        mx = fmaxf(mx, s[i][j]);
      }
#pragma unroll
      for (int w = 1; w < 16; w <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, w));
      const float m_new = fmaxf(m[i], mx);
      const float corr = m_new == -INFINITY ? 1.f : exp2f(m[i] - m_new);
      float ls = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float pj = m_new == -INFINITY ? 0.f : exp2f(s[i][j] - m_new);
        s[i][j] = pj;
        ls += pj;
      }
#pragma unroll
      for (int w = 1; w < 16; w <<= 1) ls += __shfl_xor_sync(0xffffffffu, ls, w);
      l[i] = l[i] * corr + ls;
      m[i] = m_new;
#pragma unroll
      for (int c = 0; c < OC; ++c) o[i][c] *= corr;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(Pt + (tx + 16 * j) * kPadT + 4 * ty) = make_float4(s[0][j], s[1][j], s[2][j], s[3][j]);
    __syncthreads();
#pragma unroll 4
    for (int key = 0; key < kBC; ++key) {
      const float4 p4 = *reinterpret_cast<const float4*>(Pt + key * kPadT + 4 * ty);
      const float pa[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
      for (int c4 = 0; c4 < OC / 4; ++c4) {
        const float4 v4 = *reinterpret_cast<const float4*>(Vs + key * DH + 64 * c4 + 4 * tx);
        const float va[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) o[i][4 * c4 + c] = fmaf(pa[i], va[c], o[i][4 * c4 + c]);
      }
    }
  }
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = 4 * ty + i;
    if (rr >= nr) continue;
    const float inv = 1.f / l[i];
#pragma unroll
    for (int c4 = 0; c4 < OC / 4; ++c4) {
      const float4 v = make_float4(o[i][4 * c4] * inv, o[i][4 * c4 + 1] * inv, o[i][4 * c4 + 2] * inv,
                                   o[i][4 * c4 + 3] * inv);
      bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
      *reinterpret_cast<float4*>(out + (size_t)(r0 + rr) * (H * DH) + h * DH + 64 * c4 + 4 * tx) = v;
    }
  }
  if (bad && status) *reinterpret_cast<volatile int*>(status) = 1;
}

template <typename... KArgs, typename... Args>
void launch_pdl_tc(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
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
  RK_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

int grid_for(rk_engine* e, long long n) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 8LL * e->sm_count));
}

}  // namespace

namespace tc {

void pack_weight(cudaStream_t st, float* dst, const float* src, int ldsrc, int c0, int cs, int K, int N) {
  pack_b3_kernel<<<dim3((K + 31) / 32, (N + 31) / 32), dim3(32, 8), 0, st>>>(src, ldsrc, c0, cs, dst, K, N);
  RK_CUDA(cudaGetLastError());
}

void gemm(rk_engine* e, const float* A, int lda, Rows rows, const float* Wtc, int N, int K, float* out, int ldo,
          bool add) {
  Scratch& S = *e->scratch;
  const size_t need = (size_t)rows.rows_max * 3 * K * 4;
  S.tc_split.ensure(need);
  float* a3 = S.tc_split.as<float>();
  ProfScope ps(e, "tc_split_gemm", 0, 0);
  launch_pdl_tc(split3_rows_kernel, dim3(grid_for(e, (long long)rows.rows_max * K / 4)), dim3(256), 0, e->stream, A,
                lda, a3, rows.rows_max, K);
  e->launches += 1;
  GemmArgs g;
  g.rows_max = rows.rows_max;
  g.rows_dev = rows.rows_dev;
  g.N = N;
  g.K = 2 * 3 * K;  // fp32 [.. x 3K] viewed as bf16 pairs
  g.epi = add ? EPI_ADD : EPI_F32;
  g.out_f32 = out;
  g.ld_out = ldo;
  g.tf32 = 1;
  gemm_bf16(e, reinterpret_cast<const __nv_bfloat16*>(a3), 2 * 3 * K, reinterpret_cast<const __nv_bfloat16*>(Wtc), g,
            rows.rows_dev ? (rows.hint > 0 ? rows.hint : std::max(1, rows.rows_max / 3)) : 0);
}

void silu(rk_engine* e, const float* gu, float* act, Rows rows, int ff) {
  launch_pdl_tc(silu_pair_kernel, dim3(grid_for(e, (long long)rows.rows_max * ff)), dim3(256), 0, e->stream, gu, act,
                rows, ff);
  e->launches += 1;
}

void attention(rk_engine* e, const float* qkv, int ld, Rows rows, int H, int Hkv, int dh, const float* ck,
               const float* cv, float* out) {
  if (rows.rows_max <= 0) return;
  const float scale_log2 = 1.4426950408889634f / std::sqrt((float)dh);
  const dim3 grid((rows.rows_max + kBR - 1) / kBR, H);
  ProfScope ps(e, "attn_tc_f32", 0, 0);
  if (dh == 64) {
    constexpr size_t smem = (2 * 64 * kPadT + kBC * 64 + kBC * kPadT) * 4;
    static bool attr = false;
    if (!attr) {
      RK_CUDA(cudaFuncSetAttribute(attn_f32_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    launch_pdl_tc(attn_f32_kernel<64>, grid, dim3(256), smem, e->stream, qkv, ld, rows, H, Hkv, ck, cv, out,
                  scale_log2, e->status.as<int>());
  } else if (dh == 128) {
    constexpr size_t smem = (2 * 128 * kPadT + kBC * 128 + kBC * kPadT) * 4;
    static bool attr = false;
    if (!attr) {
      RK_CUDA(cudaFuncSetAttribute(attn_f32_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    launch_pdl_tc(attn_f32_kernel<128>, grid, dim3(256), smem, e->stream, qkv, ld, rows, H, Hkv, ck, cv, out,
                  scale_log2, e->status.as<int>());
  } else {
    raise(RK_ERR_INVALID_ARGUMENT, "fp32-tc mode supports d_head 64 or 128");
  }
  e->launches += 1;
}

}  // namespace tc
}  // namespace rk
