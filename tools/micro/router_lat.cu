// Latency of the router's building blocks on one warp (clock64), to find the
// dependent chain that makes router_quad_kernel take ~10 us for one block.
#include <cstdio>
#include <cstdint>
#include "../../paper_2508_18376_b200/csrc/common.cuh"
using namespace dsb;
__device__ __forceinline__ float expf_tab(float x, const uint64_t* tab) {
  // glibc's main path, computed unconditionally; its special-case exits
  // (|x| >= 88, inf, nan) become selects, so independent calls carry no
  // branches and the compiler can interleave them (one call alone is ~200
  // cycles of dependent FP64 latency)
  const uint32_t ux = __float_as_uint(x);
  const uint32_t abstop = (ux >> 20) & 0x7ff;
  const double InvLn2N = 0x1.71547652b82fep+5, SHIFT = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-20, C1 = 0x1.ebfce50fac4f3p-13, C2 = 0x1.62e42ff0c52d6p-6;
  const double xd = static_cast<double>(x);
  double kd = __fma_rn(InvLn2N, xd, SHIFT);
  const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
  kd = __dsub_rn(kd, SHIFT);
  const double r = __fma_rn(InvLn2N, xd, -kd);
  const double s = __longlong_as_double(static_cast<long long>(tab[ki % 32] + (ki << 47)));
  const double y = __fma_rn(__fma_rn(C0, r, C1), __dmul_rn(r, r), __fma_rn(C2, r, 1.0));
  float res = static_cast<float>(__dmul_rn(y, s));
  // glibc's exits for abstop >= top12(88): none of these conditions holds
  // below that, so they apply unconditionally (selects, no branch)
  res = x < -0x1.9fe368p6f ? 0.0f : res;
  res = x > 0x1.62e42ep6f ? __uint_as_float(0x7f800000u) : res;
  res = abstop >= 0x7f8 ? x + x : res;
  res = ux == 0xff800000u ? 0.0f : res;
  return res;
}
__global__ void k(const float* in, float* out, long long* cyc) {
  __shared__ uint64_t tab[32];
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2fTab[threadIdx.x];
  __syncthreads();
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = in[threadIdx.x * 16 + i];
  long long t0 = clock64();
  float mx = v[0];
  for (int i = 0; i < 16; ++i) mx = mx < v[i] ? v[i] : mx;
  for (int i = 0; i < 16; ++i) v[i] = expf_tab(__fsub_rn(v[i], mx), tab);
  float s0 = v[0] + v[15]; 
  long long t1 = clock64();
  float sum = 0.f;
  for (int k = 0; k < 4; ++k) {
    for (int i = 0; i < 16; ++i) sum = __fadd_rn(sum, v[i]);
    sum = __shfl_sync(0xffffffffu, sum, k);
  }
  long long t2 = clock64();
  for (int i = 0; i < 16; ++i) v[i] = __fdiv_rn(v[i], sum);
  long long t3 = clock64();
  double ds = 0.0;
  for (int i = 0; i < 8; ++i) ds = __dadd_rn(ds, (double)v[i]);
  double n0 = __ddiv_rn((double)v[0], ds), n1 = __ddiv_rn((double)v[1], ds);
  long long t4 = clock64();
  out[threadIdx.x] = s0 + sum + v[3] + (float)(n0 + n1);
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  float *in, *out; long long* cyc;
  cudaMalloc(&in, 32 * 16 * 4); cudaMalloc(&out, 128); cudaMallocManaged(&cyc, 64);
  float h[512]; for (int i = 0; i < 512; ++i) h[i] = (i % 37) * 0.1f - 1.5f;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(in, out, cyc); cudaDeviceSynchronize(); }
  printf("max+16 expf %lld cyc, 64-add chain %lld, 16 fdiv %lld, dsum+2 ddiv %lld\n", cyc[0], cyc[1], cyc[2], cyc[3]);
  return 0;
}
