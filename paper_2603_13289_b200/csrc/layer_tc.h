// layer_tc.h -- RK_FP32_TC building blocks (layer_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

namespace rk {
namespace tc {
// dst [N x 3K] = [hi | lo | hi] of W[k][n] = src[k * ldsrc + c0 + n * cs]
void pack_weight(cudaStream_t st, float* dst, const float* src, int ldsrc, int c0, int cs, int K, int N);
// out[r][0..N) (=|+=) A[r][0..K) . W, W packed by pack_weight; 3xTF32 on tcgen05
void gemm(rk_engine* e, const float* A, int lda, Rows rows, const float* Wtc, int N, int K, float* out, int ldo,
          bool add);
// act[r][j] = silu(gu[r][2j]) * gu[r][2j+1]
void silu(rk_engine* e, const float* gu, float* act, Rows rows, int ff);
// fp32 flash attention of the Q columns of qkv (row stride ld) over the layer's fp32 context
void attention(rk_engine* e, const float* qkv, int ld, Rows rows, int H, int Hkv, int dh, const float* ck,
               const float* cv, float* out);
}  // namespace tc
}  // namespace rk
