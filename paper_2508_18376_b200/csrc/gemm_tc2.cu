// K3 / K4 on CTA pairs: the grouped GEMM with tcgen05.mma.cta_group::2.
//
// Same work items and epilogues as gemm_tc.cu (GEMM1 [W1|W3] + SwiGLU -> H,
// GEMM2 W2 x raw score -> Y), but every tile is M = 256 rows computed by a
// 2-CTA cluster on two SMs of one TPC:
//   * each CTA stages its own 128 A rows and HALF of the B rows (N/2) — the
//     pair's UMMA reads A M-split and B N-split across the two SMs' shared
//     memory, so per-SM operand traffic (TMA writes + tensor-core reads) per
//     FLOP is 2/3 of the single-CTA kernel's, which is what bounded it
//     (SMEM bandwidth: 192 B/cycle needed at M=128/N=256 vs 128 B/cycle);
//   * the leader CTA (rank 0) issues the MMAs; both CTAs' TMA loads complete
//     on the leader's full barrier, MMA completion is multicast to both CTAs'
//     empty / accumulator-full barriers, and both CTAs' epilogues release the
//     accumulator on the leader's barrier;
//   * each CTA's TMEM holds its 128 accumulator rows x N columns; the
//     epilogue (8 warps, smem-staged coalesced stores) is per CTA.
// Persistent: 74 clusters walk the tile list in a static round robin.
#include "common.cuh"

namespace dsb {

constexpr int k2Stages = 5;
constexpr int k2ABytes = 128 * kTileK * 2;          // 16 KB: this CTA's 128 A rows
constexpr int k2BBytes = 128 * kTileK * 2;          // 16 KB: this CTA's N/2 (<=128) B rows
constexpr int k2StageBytes = k2ABytes + k2BBytes;   // 32 KB
constexpr int k2OutBytes = 128 * 256;               // epilogue staging
constexpr int k2Threads = 320;                      // producer, MMA, 8 epilogue warps
constexpr int k2Smem = k2Stages * k2StageBytes + k2OutBytes + 1024 + 256;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;         // shared::cluster address -> leader CTA's copy

enum { k2SwiGLU = 1, k2Scale = 2 };

struct Gemm2Args {
  const GemmTile* tiles;  // M = 256 tiles
  const int* num_tiles;
  void* out;
  long long ldo;
  const float* row_scale;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
// TMA load whose completion is signalled on the LEADER CTA's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma2_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// MMA completion -> the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float silu2(float g) { return g / (1.0f + __expf(-g)); }

__device__ __forceinline__ void stage_put2(uint8_t* buf, int r, int col, const uint32_t* pk) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = (col >> 3) + i;
    *reinterpret_cast<uint4*>(buf + r * 256 + ((k ^ (r & 15)) << 4)) =
        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  }
}
__device__ __forceinline__ void epi_sync2() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void copy_out2(const uint8_t* buf, __nv_bfloat16* out, long long ld, int width, int m_valid,
                                          int tid) {
  const int cpr = width >> 3;
  for (int i = tid; i < 128 * cpr; i += 256) {
    const int row = i / cpr, k = i - row * cpr;
    if (row < m_valid)
      *reinterpret_cast<uint4*>(out + row * ld + (k << 3)) =
          *reinterpret_cast<const uint4*>(buf + row * 256 + ((k ^ (row & 15)) << 4));
  }
}

template <int MODE>
__global__ void __launch_bounds__(k2Threads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
                    const __grid_constant__ CUtensorMap mapB, const Gemm2Args args) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* stage_buf = smem + k2Stages * k2StageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_buf + k2OutBytes);
  uint64_t* empty = full + k2Stages;
  uint64_t* tfull = empty + k2Stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int ntiles = *args.num_tiles;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(&full[s], 2);   // leader's expect_tx arrive + the peer's arrive
      mbar_init(&empty[s], 1);  // multicast MMA commit
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 16);  // one arrive per epilogue warp of both CTAs
    }
    fence_mbar_init();
    tma_prefetch(&mapA);
    tma_prefetch(&mapA2);
    tma_prefetch(&mapB);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cl; t < ntiles; t += ncl) {
        const GemmTile tl = args.tiles[t];
        const int a_row = tl.a_row + static_cast<int>(rank) * 128;
        const int b_row = tl.b_row + static_cast<int>(rank) * (tl.n_mma >> 1);
        const void* ma = (tl.m_live & kTileAltA) ? static_cast<const void*>(&mapA2) : static_cast<const void*>(&mapA);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * k2StageBytes;
          if (leader)
            mbar_expect_tx(&full[stage], 2 * k2StageBytes);
          else
            mbar_arrive_cluster_relaxed(&full[stage], 0);
          tma_load_2d_pair(sa, ma, &full[stage], kb * kTileK, a_row);
          tma_load_2d_pair(sa + k2ABytes, &mapB, &full[stage], kb * kTileK, b_row);
          if (++stage == k2Stages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader CTA only)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t sbase = smem_u32(smem);
      for (int t = cl; t < ntiles; t += ncl) {
        const GemmTile tl = args.tiles[t];
        const uint32_t idesc = idesc_bf16(256, tl.n_mma);
        const uint32_t dtmem = tmem_base + acc * 256;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = sbase + stage * k2StageBytes;
          const uint64_t adesc = sdesc_sw128(sa);
          const uint64_t bdesc = sdesc_sw128(sa + k2ABytes);
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k) umma2_bf16(dtmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          umma2_commit_both(&empty[stage]);
          if (++stage == k2Stages) { stage = 0; phase ^= 1; }
        }
        umma2_commit_both(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9 (both CTAs): this CTA's 128 rows
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int etid = threadIdx.x - 64;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cl; t < ntiles; t += ncl) {
      const GemmTile tl = args.tiles[t];
      const int row0 = static_cast<int>(rank) * 128;
      const int m_valid = max(0, min(128, tl.m_valid - row0));
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * 256 + (static_cast<uint32_t>(q * 32) << 16);
      const long long orow0 = static_cast<long long>(tl.out_row) + row0;
      auto release = [&]() {  // accumulator drained: tell the leader's MMA
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
      };
      if constexpr (MODE == k2SwiGLU) {
        const int nc = tl.n_mma >> 1;
        const int live = max(0, min(128, (tl.m_live & 0xFFFFF) - row0));
        for (int grp = half; grp < nc / kGroup; grp += 2) {  // [g | u] groups (w13_row_of)
          const int c = kGroup * grp;
          uint32_t g[32], u[32];
          tmem_ld32(taddr + 2 * c, g);
          tmem_ld32(taddr + 2 * c + kGroup, u);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float h0 = 0.f, h1 = 0.f;
            if (r < live) {
              h0 = silu2(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]);
              h1 = silu2(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]);
            }
            pk[i] = pack_bf16x2(h0, h1);
          }
          stage_put2(stage_buf, r, c, pk);
        }
        release();
        epi_sync2();
        copy_out2(stage_buf, static_cast<__nv_bfloat16*>(args.out) + orow0 * args.ldo + tl.out_col, args.ldo, nc,
                  m_valid, etid);
        epi_sync2();
      } else {
        const float sc = r < m_valid ? args.row_scale[orow0 + r] : 0.f;
        for (int p0 = 0; p0 < tl.n_mma; p0 += 128) {
          const int w = min(128, tl.n_mma - p0);
          for (int c = 32 * half; c < w; c += 64) {
            uint32_t v[32];
            tmem_ld32(taddr + p0 + c, v);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              pk[i] = pack_bf16x2(__uint_as_float(v[2 * i]) * sc, __uint_as_float(v[2 * i + 1]) * sc);
            stage_put2(stage_buf, r, c, pk);
          }
          if (p0 + 128 >= tl.n_mma) release();
          epi_sync2();
          copy_out2(stage_buf, static_cast<__nv_bfloat16*>(args.out) + orow0 * args.ldo + tl.out_col + p0, args.ldo,
                    w, m_valid, etid);
          epi_sync2();
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
}

int launch_gemm_tc2(int mode, const CUtensorMap* mapA, const CUtensorMap* mapA2, const CUtensorMap* mapB,
                    const GemmTile* tiles,
                    const int* num_tiles, int max_tiles, void* out, long long ldo, const float* row_scale, int num_sms,
                    cudaStream_t stream) {
  Gemm2Args a{tiles, num_tiles, out, ldo, row_scale};
  int clusters = num_sms / 2;
  if (max_tiles < clusters) clusters = max_tiles > 0 ? max_tiles : 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(k2Threads);
  cfg.dynamicSmemBytes = k2Smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (mode == k2SwiGLU) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(gemm_tc2_kernel<k2SwiGLU>, cudaFuncAttributeMaxDynamicSharedMemorySize, k2Smem);
      attr_set = true;
    }
    e = cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<k2SwiGLU>, *mapA, *mapA2, *mapB, a);
  } else if (mode == k2Scale) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(gemm_tc2_kernel<k2Scale>, cudaFuncAttributeMaxDynamicSharedMemorySize, k2Smem);
      attr_set = true;
    }
    e = cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<k2Scale>, *mapA, *mapA2, *mapB, a);
  } else {
    return -1;
  }
  return e == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
