// kernels_exact.cu -- the RK_FP32_EXACT layer path.
//
// Each kernel replays the reference's fp32 operation order so the device
// result is bit-identical to the CPU reference (SURVEY.md 8(a) "numerics
// contract"): no FMA anywhere (explicit __fmul_rn/__fadd_rn), per-output
// sequential reductions in the reference's index order, glibc-identical expf,
// RoPE from the host-built double cos/sin table. Parallelism comes from the
// independent outputs (rows x columns, rows x heads), never from reassociating
// a reduction the reference performs sequentially.
#include "glibc_expf.h"
#include "internal.h"

namespace rk {
namespace {

__device__ __forceinline__ int live_rows(const Rows& r) { return r.rows_dev ? *r.rows_dev : r.rows_max; }

// rms_norm (tensor.cpp:109-119): ms sequential over the row, then
// inv = 1/sqrt(ms/n + eps), out = x * inv * gain.
// CTA = 32 rows, 256 threads: the 8 warps stage 64-column chunks of the rows
// into shared memory with coalesced loads (double-buffered), and lane r of
// warp 0 adds its row's squares in column order -- the reference's sequential
// sum, bit for bit, without a strided global load per element.
constexpr int kNormRows = 32, kNormCols = 64;
__global__ void __launch_bounds__(256) rmsnorm_exact_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                                            float eps, float* __restrict__ out, Rows rows, int d) {
  __shared__ float tile[2][kNormRows][kNormCols + 1];
  __shared__ float inv_s[kNormRows];
  const int M = live_rows(rows);
  const int r0 = blockIdx.x * kNormRows;
  if (r0 >= M) return;
  const int nr = min(kNormRows, M - r0);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  auto stage = [&](int buf, int c0) {
    for (int rr = warp; rr < nr; rr += 8)
      for (int c = lane; c < kNormCols; c += 32)
        tile[buf][rr][c] = c0 + c < d ? x[(size_t)(r0 + rr) * d + c0 + c] : 0.0f;
  };
  float ms = 0.0f;
  const int nch = (d + kNormCols - 1) / kNormCols;
  stage(0, 0);
  __syncthreads();
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) stage((ch + 1) & 1, (ch + 1) * kNormCols);  // next chunk lands while warp 0 sums
    if (warp == 0 && lane < nr) {
      const int n = min(kNormCols, d - ch * kNormCols);
      const float* t = tile[ch & 1][lane];
      for (int c = 0; c < n; ++c) ms = __fadd_rn(ms, __fmul_rn(t[c], t[c]));
    }
    __syncthreads();
  }
  if (warp == 0 && lane < nr) {
    ms = __fdiv_rn(ms, (float)d);
    inv_s[lane] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, eps)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nr * d; i += blockDim.x) {
    const int rr = i / d, c = i % d;
    const size_t idx = (size_t)(r0 + rr) * d + c;
    out[idx] = __fmul_rn(__fmul_rn(x[idx], inv_s[rr]), gain[c]);
  }
}

// matmul (tensor.cpp:66-86): C[i][j] = sum_k A[i][k]*B[k][j], k ascending from
// 0.0f, multiply then add. 64x64 tiles, BK = 16, 4x4 outputs per thread.
// K-tail zero padding adds +0 terms, an identity on the running sum (which
// is never -0 since it starts at +0).
// Epilogues: STORE; ADD (hidden += result, model.cpp:217-218, 229-231);
// SILU_PAIR (columns interleaved gate/up: silu(g)*u, model.cpp:208, 226).
template <int EPI>
__global__ void __launch_bounds__(256) gemm_exact_kernel(const float* __restrict__ A,
                                                         const float* __restrict__ B,
                                                         float* __restrict__ C, Rows rows, int N,
                                                         int K, int* status) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ __align__(16) float As[BK][BM];
  __shared__ __align__(16) float Bs[BK][BN];
  const int M = live_rows(rows);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (m0 >= M) return;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  const bool vecA = (K % 4) == 0, vecB = (N % 4) == 0;
  for (int k0 = 0; k0 < K; k0 += BK) {
    {  // A tile: 64 rows x 16 k, transposed into As[k][m]
      const int row = tid / 4, kq = (tid % 4) * 4;
      const int gr = m0 + row, gk = k0 + kq;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (gr < M) {
        if (vecA && gk + 3 < K) {
          const float4 t = *reinterpret_cast<const float4*>(A + (size_t)gr * K + gk);
          v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
          for (int e = 0; e < 4; ++e) if (gk + e < K) v[e] = A[(size_t)gr * K + gk + e];
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) As[kq + e][row] = v[e];
    }
    {  // B tile: 16 k x 64 cols
      const int kk = tid / 16, c = (tid % 16) * 4;
      const int gk = k0 + kk, gc = n0 + c;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (gk < K) {
        if (vecB && gc + 3 < N) {
          const float4 t = *reinterpret_cast<const float4*>(B + (size_t)gk * N + gc);
          v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
          for (int e = 0; e < 4; ++e) if (gc + e < N) v[e] = B[(size_t)gk * N + gc + e];
        }
      }
      *reinterpret_cast<float4*>(&Bs[kk][c]) = make_float4(v[0], v[1], v[2], v[3]);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w};
      const float b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(a[i], b[j]));
    }
    __syncthreads();
  }
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c >= N) continue;
      const float v = acc[i][j];
      if (!isfinite(v)) bad = true;
      if (EPI == k::EPI_STORE) {
        C[(size_t)r * N + c] = v;
      } else if (EPI == k::EPI_ADD) {
        C[(size_t)r * N + c] = __fadd_rn(C[(size_t)r * N + c], v);
      } else if ((j & 1) == 0 && c + 1 < N) {  // SILU_PAIR: (gate, up) at (c, c+1)
        const float g = v, u = acc[i][j + 1];
        if (!isfinite(u)) bad = true;
        const float sg = __fdiv_rn(g, __fadd_rn(1.0f, glibc_expf(-g)));
        C[(size_t)r * (N / 2) + c / 2] = __fmul_rn(sg, u);
      }
    }
  }
  if (bad && status) status[0] = 1;
}

// Q/K rotation (model.cpp:261-265, rope_rotate tensor.cpp:134-142) and the
// K/V commit into the context (model.cpp:266-269). qkv rows are
// [Q (H*dh) | K (Hkv*dh) | V (Hkv*dh)]; K is rotated in place too (the
// pure-query pass reads it as self_k).
__global__ void rope_commit_exact_kernel(float* qkv, Rows rows, int H, int Hkv, int dh,
                                         const double2* __restrict__ rope, float* ctx_k,
                                         float* ctx_v, int commit) {
  const int M = live_rows(rows);
  const int r = blockIdx.x;
  if (r >= M) return;
  const int q = H * dh, kv = Hkv * dh, half = dh / 2;
  const int pos = rows.pos[r];
  float* row = qkv + (size_t)r * (q + 2 * kv);
  const double2* cs = rope + (size_t)pos * half;
  for (int p = threadIdx.x; p < (H + Hkv) * half; p += blockDim.x) {
    const int head = p / half, i = p % half;
    float* x = row + head * dh + 2 * i;  // Q heads then K heads are contiguous
    const double2 c = cs[i];
    const double x0 = x[0], x1 = x[1];
    x[0] = __double2float_rn(__dsub_rn(__dmul_rn(c.x, x0), __dmul_rn(c.y, x1)));
    x[1] = __double2float_rn(__dadd_rn(__dmul_rn(c.y, x0), __dmul_rn(c.x, x1)));
  }
  if (!commit) return;
  __syncthreads();
  for (int i = threadIdx.x; i < kv; i += blockDim.x) {
    ctx_k[(size_t)pos * kv + i] = row[q + i];
    ctx_v[(size_t)pos * kv + i] = row[q + kv + i];
  }
}

// attend_row (model.cpp:170-204) for one (row, head): scores sequential over
// d, scaled by 1/sqrt(dh); softmax_inplace (tensor.cpp:88-98) with a
// sequential sum and a division; out[d] accumulated over j in order.
// self_override: the cell at the row's own position is read from the row's
// fresh (uncommitted) K/V in qkv (row_logits_from_layer, model.cpp:353).
__global__ void __launch_bounds__(128) attn_exact_kernel(const float* __restrict__ qkv, Rows rows,
                                                         int H, int Hkv, int dh,
                                                         const float* __restrict__ ctx_k,
                                                         const float* __restrict__ ctx_v,
                                                         float* __restrict__ out, int self_override,
                                                         float* __restrict__ probs, int key_lo,
                                                         int key_n) {
  extern __shared__ float smem[];
  const int M = live_rows(rows);
  const int r = blockIdx.x, h = blockIdx.y;
  if (r >= M) return;
  const int q = H * dh, kv = Hkv * dh, ld = q + 2 * kv;
  const int kvh = h / (H / Hkv);
  const int pos = rows.pos[r];
  const int ctx_len = pos + 1;
  float* qs = smem;
  float* scores = smem + dh;
  __shared__ float red[32];
  __shared__ float bcast;
  const float* qrow = qkv + (size_t)r * ld;
  for (int i = threadIdx.x; i < dh; i += blockDim.x) qs[i] = qrow[h * dh + i];
  __syncthreads();
  const float inv_sqrt_dh = __fdiv_rn(1.0f, __fsqrt_rn((float)dh));
  const float* self_k = qrow + q + kvh * dh;
  const float* self_v = qrow + q + kv + kvh * dh;
  float mx = -__int_as_float(0x7f800000);
  for (int j = threadIdx.x; j < ctx_len; j += blockDim.x) {
    const float* kj = (self_override && j == pos) ? self_k : ctx_k + (size_t)j * kv + kvh * dh;
    float s = 0.0f;
    for (int d = 0; d < dh; ++d) s = __fadd_rn(s, __fmul_rn(qs[d], kj[d]));
    s = __fmul_rn(s, inv_sqrt_dh);
    scores[j] = s;
    mx = fmaxf(mx, s);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    bcast = m;
  }
  __syncthreads();
  mx = bcast;
  for (int j = threadIdx.x; j < ctx_len; j += blockDim.x) scores[j] = glibc_expf(__fsub_rn(scores[j], mx));
  __syncthreads();
  if (threadIdx.x == 0) {
    float sum = 0.0f;
    for (int j = 0; j < ctx_len; ++j) sum = __fadd_rn(sum, scores[j]);
    bcast = sum;
  }
  __syncthreads();
  const float sum = bcast;
  for (int j = threadIdx.x; j < ctx_len; j += blockDim.x) scores[j] = __fdiv_rn(scores[j], sum);
  __syncthreads();
  if (probs) {  // decode-time capture: attention row over the segment keys
    float* pr = probs + ((size_t)r * gridDim.y + h) * key_n;
    for (int jj = threadIdx.x; jj < key_n; jj += blockDim.x)
      pr[jj] = (key_lo + jj < ctx_len) ? scores[key_lo + jj] : 0.0f;
  }
  for (int d = threadIdx.x; d < dh; d += blockDim.x) {
    float acc = 0.0f;
    for (int j = 0; j < ctx_len; ++j) {
      const float* vj = (self_override && j == pos) ? self_v : ctx_v + (size_t)j * kv + kvh * dh;
      acc = __fadd_rn(acc, __fmul_rn(scores[j], vj[d]));
    }
    out[(size_t)r * q + h * dh + d] = acc;
  }
}

// RelayRecorder::feed influence sums (relay_cache.cpp:108-123): for each
// capture row in order, acc[j] += p[h][key_lo + j] over heads in order, for
// segment keys strictly before the row (or up to it with include_self).
__global__ void influence_accum_kernel(double* acc, const float* probs, Rows rows, int H,
                                       int key_lo, int key_n, int include_self) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= key_n) return;
  const int M = live_rows(rows);
  double a = acc[j];
  for (int r = 0; r < M; ++r) {
    const int t = rows.pos[r] - key_lo;
    if (include_self ? t < j : t <= j) continue;
    for (int h = 0; h < H; ++h) a = __dadd_rn(a, (double)probs[((size_t)r * H + h) * key_n + j]);
  }
  acc[j] = a;
}

}  // namespace

namespace k {

void rmsnorm_exact(cudaStream_t s, const float* x, const float* gain, float eps, float* out,
                   Rows rows, int d) {
  if (rows.rows_max <= 0) return;
  rmsnorm_exact_kernel<<<(rows.rows_max + kNormRows - 1) / kNormRows, 256, 0, s>>>(x, gain, eps, out, rows, d);
}

void gemm_exact(cudaStream_t s, const float* A, const float* B, float* C, Rows rows, int N, int K,
                int epi, int* status) {
  if (rows.rows_max <= 0) return;
  dim3 grid((N + 63) / 64, (rows.rows_max + 63) / 64);
  if (epi == EPI_STORE) gemm_exact_kernel<EPI_STORE><<<grid, 256, 0, s>>>(A, B, C, rows, N, K, status);
  else if (epi == EPI_ADD) gemm_exact_kernel<EPI_ADD><<<grid, 256, 0, s>>>(A, B, C, rows, N, K, status);
  else gemm_exact_kernel<EPI_SILU_PAIR><<<grid, 256, 0, s>>>(A, B, C, rows, N, K, status);
}

void rope_commit_exact(cudaStream_t s, float* qkv, Rows rows, int H, int Hkv, int dh,
                       const double2* rope, float* ctx_k, float* ctx_v, int commit) {
  if (rows.rows_max <= 0) return;
  rope_commit_exact_kernel<<<rows.rows_max, 128, 0, s>>>(qkv, rows, H, Hkv, dh, rope, ctx_k, ctx_v, commit);
}

static int g_attn_smem_set = 0;
void attn_exact(cudaStream_t s, const float* qkv, Rows rows, int H, int Hkv, int dh,
                const float* ctx_k, const float* ctx_v, float* out, int self_override,
                int max_ctx, float* probs, int key_lo, int key_n) {
  if (rows.rows_max <= 0) return;
  const size_t smem = (size_t)(dh + max_ctx + 1) * sizeof(float);
  constexpr size_t kMaxDyn = 220 * 1024;
  if (!g_attn_smem_set) {
    RK_CUDA(cudaFuncSetAttribute(attn_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDyn));
    g_attn_smem_set = 1;
  }
  if (smem > kMaxDyn) raise(RK_ERR_INVALID_ARGUMENT, "fp32-exact attention: context too long for shared memory");
  dim3 grid(rows.rows_max, H);
  attn_exact_kernel<<<grid, 128, smem, s>>>(qkv, rows, H, Hkv, dh, ctx_k, ctx_v, out, self_override,
                                            probs, key_lo, key_n);
}

void influence_accum(cudaStream_t s, double* acc, const float* probs, Rows rows, int H, int key_lo,
                     int key_n, int include_self) {
  if (rows.rows_max <= 0 || key_n <= 0) return;
  influence_accum_kernel<<<(key_n + 127) / 128, 128, 0, s>>>(acc, probs, rows, H, key_lo, key_n, include_self);
}

}  // namespace k
}  // namespace rk
