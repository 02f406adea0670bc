// FP64 latency vs throughput on one warp (is the router's expf chain bound by DFMA latency or rate?)
#include <cstdio>
__global__ void k(const double* in, double* out, long long* cyc) {
  double a = in[threadIdx.x], b = in[threadIdx.x + 32], c[8];
  for (int i = 0; i < 8; ++i) c[i] = in[threadIdx.x + 64 + i];
  long long t0 = clock64();
  double x = a;
#pragma unroll
  for (int i = 0; i < 64; ++i) x = __fma_rn(x, b, a);
  long long t1 = clock64();
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = __fma_rn(c[i], b, a);
  long long t2 = clock64();
  float f = (float)a, g = (float)b;
#pragma unroll
  for (int i = 0; i < 64; ++i) f = __fmaf_rn(f, g, 1.0f);
  long long t3 = clock64();
  double s = x;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[threadIdx.x] = s + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double *in, *out; long long* cyc;
  cudaMalloc(&in, 1024); cudaMalloc(&out, 512); cudaMallocManaged(&cyc, 64);
  cudaMemset(in, 0, 1024);
  for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(in, out, cyc); cudaDeviceSynchronize(); }
  printf("64 dependent DFMA %lld cyc, 8x8 independent DFMA %lld cyc, 64 dependent FFMA %lld cyc\n", cyc[0], cyc[1], cyc[2]);
  return 0;
}
