// Microbenchmark: MUFU.EX2 / FFMA2 / F2FP throughput per SM on the B200
// (clock64 over a fixed instruction count, warps per SM varied).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int OP>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) a[i] = __fmaf_rn(a[i], 0.999f, 1e-3f);
      if (OP == 2) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i+1)&7])); a[i] = __uint_as_float(r); }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  const char* names[] = {"MUFU.EX2", "FFMA", "F2FP.BF16x2"};
  for (int op = 0; op < 3; ++op)
    for (int warps : {1, 4, 8, 16, 32}) {
      auto fn = op == 0 ? k<0> : op == 1 ? k<1> : k<2>;
      fn<<<148, warps * 32>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      long long c[148]; cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
      double ops = (double)warps * 32 * iters * 8;  // per SM
      printf("%-12s warps/SM=%2d: %.2f thread-ops/clk/SM (%.1f clk per warp-instr per SMSP)\n", names[op], warps,
             ops / c[0], (double)c[0] / ((double)warps * iters * 8 / (warps < 4 ? warps : 4)));
    }
  return 0;
}
