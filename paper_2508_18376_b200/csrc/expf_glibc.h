// glibc-exact expf, usable from host C++ (g++) and device code (nvcc).
// The reference calls std::exp(float) in softmax_inplace (matrix.hpp:74) and
// swish (matrix.hpp:91); bit-exact routing and importance profiles need the
// same float glibc returns — SURVEY.md Appendix A.3.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

namespace dsb {


// ----------------------------------------------------------------------------
// glibc __expf (sysdeps/ieee754/flt-32/e_expf.c, EXP2F_TABLE_BITS = 5) in the
// FMA-contracted form the x86-64 IFUNC selects on FMA hosts.  Table entry i is
// asuint64(2^(i/32)) - (i << 47), generated to correct rounding by
// tools/gen_exp2f_table.py; verified bit-exact against libm expf over every
// float by tools/check_expf.sh (CPU, host build of this same function; sampled in
// tests/test_capi_cpu.py).
// ----------------------------------------------------------------------------
#ifdef __CUDACC__
#define DSB_HD __host__ __device__ __forceinline__
#else
#define DSB_HD inline
#endif

#ifdef __CUDA_ARCH__
__device__ __constant__ uint64_t kExp2fTab[32] = {
#else
static const uint64_t kExp2fTab[32] = {
#endif
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

#ifdef __CUDA_ARCH__
__device__ __forceinline__ double dsb_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double dsb_dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }
__device__ __forceinline__ uint64_t d2u(double d) { return (uint64_t)__double_as_longlong(d); }
__device__ __forceinline__ double u2d(uint64_t u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }
#else
inline double dsb_fma(double a, double b, double c) { return fma(a, b, c); }
inline double dsb_dmul(double a, double b) {
  volatile double r = a * b;  // no contraction into a neighbouring add
  return r;
}
inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
inline uint64_t d2u(double d) { uint64_t u; memcpy(&u, &d, 8); return u; }
inline double u2d(uint64_t u) { double d; memcpy(&d, &u, 8); return d; }
inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
#endif

DSB_HD float glibc_expf(float x) {
  const uint32_t abstop = (f2u(x) >> 20) & 0x7ff;
  if (abstop >= 0x42b) {                          // |x| >= 88 or NaN
    if (f2u(x) == 0xff800000u) return 0.0f;       // -inf
    if (abstop >= 0x7f8) return x + x;            // inf / nan
    if (x > 0x1.62e42ep6f) return u2f(0x7f800000u);   // overflow -> +inf
    if (x < -0x1.9fe368p6f) return 0.0f;          // underflow -> +0
  }
  const double InvLn2N = 0x1.71547652b82fep+5;
  const double SHIFT = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-20, C1 = 0x1.ebfce50fac4f3p-13, C2 = 0x1.62e42ff0c52d6p-6;
  const double xd = (double)x;
  double kd = dsb_fma(InvLn2N, xd, SHIFT);
  const uint64_t ki = d2u(kd);
  kd -= SHIFT;
  const double r = dsb_fma(InvLn2N, xd, -kd);
  const double s = u2d(kExp2fTab[ki % 32] + (ki << 47));
  const double y = dsb_fma(dsb_fma(C0, r, C1), dsb_dmul(r, r), dsb_fma(C2, r, 1.0));
  return (float)dsb_dmul(y, s);
}

}  // namespace dsb
