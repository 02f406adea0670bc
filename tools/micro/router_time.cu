// Device time of one router_quad_kernel launch (T tokens, E = 64, K = 8) in a
// back-to-back loop, to separate the kernel's own latency from launch overhead.
#include <cstdio>
#include <vector>
#include "../../paper_2508_18376_b200/csrc/router.cu"
using namespace dsb;
__global__ void empty_kernel() {}
int main(int argc, char** argv) {
  const int E = 64, K = 8, P = 2;
  for (int T : {32, 512, 16384}) {
    std::vector<float> h(static_cast<size_t>(T) * E);
    for (size_t i = 0; i < h.size(); ++i) h[i] = float((i * 2654435761u) % 1000) * 0.003f;
    float* lg; cudaMalloc(&lg, h.size() * 4); cudaMemcpy(lg, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    int32_t *idx, *sel_code; float *raw, *sel_raw; double* norm; uint8_t* frac; int* cnt; unsigned long long* ctr;
    cudaMalloc(&idx, T * K * P * 4); cudaMalloc(&raw, T * K * P * 4); cudaMalloc(&norm, T * K * P * 8);
    cudaMalloc(&frac, T * K * P); cudaMalloc(&sel_code, T * K * 4); cudaMalloc(&sel_raw, T * K * 4);
    cudaMalloc(&cnt, (T / 32 + 1) * 2 * E * 4); cudaMalloc(&ctr, 64);
    RouterArgs a{};
    a.logits = lg; a.ld_logits = E; a.nsplit = 1; a.T = T; a.E = E; a.K = K; a.P = P; a.kind = 2;
    a.t_major = 0.07; a.t_minor = 0.09; a.keep_top1 = 1; a.normalize = 1;
    a.idx = idx; a.raw = raw; a.norm = norm; a.frac = frac; a.sel_code = sel_code; a.sel_raw = sel_raw;
    a.cnt_chunk = cnt; a.counters = ctr;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 10; ++i) launch_router(a, 0);
    const int n = 200;
    cudaEventRecord(e0);
    for (int i = 0; i < n; ++i) launch_router(a, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaEventRecord(e0);
    for (int i = 0; i < n; ++i) empty_kernel<<<1, 32>>>();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float me; cudaEventElapsedTime(&me, e0, e1);
    printf("T=%5d router %.2f us/launch (empty kernel %.2f us/launch) err=%s\n", T, 1e3 * ms / n, 1e3 * me / n,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
