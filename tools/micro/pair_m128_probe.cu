// Probe: where does tcgen05.mma.cta_group::2 with M = 128 read A / B rows from
// and where does it put D in the two CTAs' TMEM?  A[r][0] = 128*cta + r,
// A[r][1] = 1; B[n][0] = 1, B[n][1] = 256 * (64*cta + n)  =>  D = a_id + 256 * b_id.
#include <cstdio>
#include <cstdint>
#include "../../paper_2508_18376_b200/csrc/common.cuh"
using namespace dsb;

constexpr int N = 64;
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) probe(float* out, int M) {
  __shared__ __align__(1024) uint8_t sA[128 * 128];  // 128 rows x 64 bf16, SW128
  __shared__ __align__(1024) uint8_t sB[64 * 128];   // 64 rows x 64 bf16, SW128
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int cta = pair_rank(), tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // fill A (128 rows) and B (64 rows) in SWIZZLE_128B K-major layout
  for (int r = tid; r < 128; r += 128) {
    for (int k = 0; k < 64; ++k) {
      float v = k == 0 ? float(128 * cta + r) : (k == 1 ? 1.f : 0.f);
      const int chunk = k >> 3, within = k & 7;
      const int off = r * 128 + ((chunk ^ (r & 7)) << 4) + within * 2;
      *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16(v);
    }
  }
  for (int r = tid; r < 64; r += 128) {
    for (int k = 0; k < 64; ++k) {
      float v = k == 0 ? 1.f : (k == 1 ? float(256 * (64 * cta + r)) : 0.f);
      const int chunk = k >> 3, within = k & 7;
      const int off = r * 128 + ((chunk ^ (r & 7)) << 4) + within * 2;
      *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16(v);
    }
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc_pair(&tslot, 64);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  pair_sync();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (cta == 0 && warp == 0) {
    if (elect_one()) {
      const uint64_t da = sdesc_sw128(smem_u32(sA)), db = sdesc_sw128(smem_u32(sB));
      const uint32_t idesc = idesc_bf16(M, N);
      for (int k = 0; k < 4; ++k) umma_bf16_pair(tmem, da + 2 * k, db + 2 * k, idesc, k != 0);
      umma_commit_pair(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[64];
  tmem_ld64(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
  tmem_ld_wait();
  for (int c = 0; c < N; ++c) out[(cta * 128 + warp * 32 + lane) * N + c] = __uint_as_float(v[c]);
  tc_fence_before();
  pair_sync();
  if (warp == 0) tmem_dealloc_pair(tmem, 64);
}

int main() {
  float* out;
  cudaMallocManaged(&out, 2 * 128 * N * 4);
  for (int M : {256, 128}) {
    for (int i = 0; i < 2 * 128 * N; ++i) out[i] = -1.f;
    probe<<<2, 128>>>(out, M);
    cudaError_t e = cudaDeviceSynchronize();
    printf("M=%d err=%s\n", M, cudaGetErrorString(e));
    for (int cta = 0; cta < 2; ++cta)
      for (int lane = 0; lane < 128; lane += (lane < 8 || (lane >= 60 && lane < 68) || lane >= 124) ? 1 : 8) {
        printf("cta%d lane%3d:", cta, lane);
        for (int c : {0, 1, 2, 31, 32, 33, 63}) {
          float x = out[(cta * 128 + lane) * N + c];
          int iv = int(x);
          printf("  c%d=%s(a%d,b%d)", c, x < 0 ? "-" : "", iv % 256, iv / 256);
        }
        printf("\n");
      }
  }
  return 0;
}
