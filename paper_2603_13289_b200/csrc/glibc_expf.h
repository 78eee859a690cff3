// glibc_expf.h -- bit-exact restatement of glibc 2.39's expf for device code.
//
// The reference computes softmax (tensor.cpp:93) and SiLU (model.cpp:208)
// with std::exp on floats, i.e. glibc's expf. On x86-64 with FMA, glibc
// dispatches to __expf_fma: the generic algorithm (sysdeps/ieee754/flt-32/
// e_expf.c: 2^(k/32) table + degree-3 polynomial in double) compiled with
// -mfma, where GCC contracts `r = z - kd` (z = InvLn2N*x) into
// fma(InvLn2N, x, -kd) and the polynomial into FMAs. This restatement
// reproduces that variant; it matched this container's libm expf on all
// 2^32 float inputs (tests/test_expf.py re-checks a sample on every host,
// and the GPU test re-checks the device build against the host's libm).
//
// Usable from host C++ (for the CPU check) and CUDA device code.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define RK_HD __host__ __device__ __forceinline__
#else
#define RK_HD inline
#include <math.h>
#include <string.h>
#endif

namespace rk {

// tab[i] = asuint64(2^(i/32)) - (i << 47): the exp2f_data table, N = 32.
#define RK_EXP2F_TAB {0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL, \
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL, \
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL, \
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL, \
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL, \
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL, \
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL, \
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL}
#ifdef __CUDACC__
__device__ __constant__ static const uint64_t kExp2fTabDev[32] = RK_EXP2F_TAB;
#endif
static const uint64_t kExp2fTabHost[32] = RK_EXP2F_TAB;

#ifdef __CUDACC__
RK_HD uint32_t f2u(float f) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(f);
#else
  uint32_t u; memcpy(&u, &f, 4); return u;
#endif
}
#else
RK_HD uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
#endif

RK_HD uint64_t d2u(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u; memcpy(&u, &d, 8); return u;
#endif
}
RK_HD double u2d(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d; memcpy(&d, &u, 8); return d;
#endif
}

#ifdef __CUDA_ARCH__
#define RK_DMUL(a, b) __dmul_rn(a, b)
#define RK_DADD(a, b) __dadd_rn(a, b)
#define RK_DSUB(a, b) __dsub_rn(a, b)
#define RK_DFMA(a, b, c) __fma_rn(a, b, c)
#define RK_D2F(a) __double2float_rn(a)
#else
#define RK_DMUL(a, b) ((a) * (b))
#define RK_DADD(a, b) ((a) + (b))
#define RK_DSUB(a, b) ((a) - (b))
#define RK_DFMA(a, b, c) fma(a, b, c)
#define RK_D2F(a) ((float)(a))
#endif

// == glibc 2.39 expf (FMA variant), bit for bit.
RK_HD float glibc_expf(float x) {
  const double kInvLn2N = 0x1.71547652b82fep+0 * 32;
  const double kShift = 0x1.8p+52;
  const double kC0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32;
  const double kC1 = 0x1.ebfce50fac4f3p-3 / 32 / 32;
  const double kC2 = 0x1.62e42ff0c52d6p-1 / 32;
  const uint32_t ux = f2u(x);
  const uint32_t abstop = (ux >> 20) & 0x7ff;
  if (abstop >= 0x42bu) {            // |x| >= 88 or nan
    if (ux == 0xff800000u) return 0.0f;  // -inf
    if (abstop >= 0x7f8u) return x + x;  // inf or nan
    if (x > 0x1.62e42ep6f) return __builtin_huge_valf();  // overflow
    if (x < -0x1.9fe368p6f) return 0.0f;                  // underflow
  }
  const double xd = (double)x;
  const double z = RK_DMUL(kInvLn2N, xd);
  double kd = RK_DADD(z, kShift);
  const uint64_t ki = d2u(kd);
  kd = RK_DSUB(kd, kShift);
  const double r = RK_DFMA(kInvLn2N, xd, -kd);
#ifdef __CUDA_ARCH__
  uint64_t t = kExp2fTabDev[ki % 32];
#else
  uint64_t t = kExp2fTabHost[ki % 32];
#endif
  t += ki << 47;
  const double s = u2d(t);
  const double zz = RK_DFMA(kC0, r, kC1);
  const double r2 = RK_DMUL(r, r);
  double y = RK_DFMA(kC2, r, 1.0);
  y = RK_DFMA(zz, r2, y);
  y = RK_DMUL(y, s);
  return RK_D2F(y);
}

}  // namespace rk
