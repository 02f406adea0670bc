// K3 / K4 (and K0): persistent grouped GEMM on the 5th-generation tensor cores.
//
// Replaces the per-token scalar loops of accumulate_block
// (/root/reference/proj/include/dsmoe/moe.hpp:213-231) and the gate matmul of
// gate_scores (moe.hpp:174 -> matrix.hpp:47-64) for bf16 layers.
//
// One CTA per SM (448 threads, warp-specialised):
//   warp 0      TMA producer: A (128 x 64) and B (N x 64) bf16 tiles, SWIZZLE_128B,
//               4-stage smem ring guarded by full/empty mbarriers;
//   warps 1..4  row gatherers (GEMM1 with fused gather only): warp g owns ring
//               stage g and fills its A tile straight from the token rows of X
//               (16-byte cp.async, one warp instruction = 4 rows x 128 B, so
//               every request is a whole L2 line), then proxy-fences and
//               arrives on the stage's full barrier — no permuted copy of X;
//   warp 5      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N<=256,
//               K=16 per instruction), fp32 accumulators in TMEM, two
//               accumulator stages (2 x 256 columns) so the epilogue of tile i
//               overlaps the MMAs of tile i+1;
//   warps 6..13 epilogue (two warps per TMEM lane quarter, alternating 32-column
//               chunks): tcgen05.ld 32x32b -> registers -> fused op -> global.
// Work items (GemmTile) are produced on the device by plan_tiles (permute.cu)
// and walked in a static round-robin over the persistent CTAs.
//
// Epilogue modes
//   kEpiF32     fp32 store (gate logits, K0);
//   kEpiSwiGLU  h = swish(g) * u over the [g | u] column halves of the tile,
//               rows >= m_live store zeros (major-only rows of a minor chunk),
//               bf16 store into H (K3);
//   kEpiScale   y = acc * row_scale[row] (the raw gate score, moe.hpp:235-237),
//               bf16 store into Y (K4).
#include <cstdlib>

#include "common.cuh"

namespace dsb {

constexpr int kStages = 4;
constexpr int kABytes = kTileM * kTileK * 2;       // 16 KB
constexpr int kBBytesMax = 256 * kTileK * 2;       // 32 KB
constexpr int kStageBytes = kABytes + kBBytesMax;  // 48 KB
constexpr int kGatherWarp0 = 1;     // warps 1-4: fused row gather, warp 1 + s owns stage s
constexpr int kGatherWarps = kStages;
constexpr int kMmaWarp = 5;         // warp 5: TMEM alloc + tcgen05.mma issue
constexpr int kEpiWarp0 = 6;        // warps 6-13: epilogue
constexpr int kGemmThreads = 448;
constexpr int kEpiThreads = 256;
constexpr int kAccCols = 256;
constexpr int kGemmSmem = kStages * kStageBytes + 128 * 256 /*output stage*/ + 1024 /*align*/ + 256 /*barriers*/;

enum { kEpiF32 = 0, kEpiSwiGLU = 1, kEpiScale = 2 };

struct GemmArgs {
  const GemmTile* tiles;
  const int* num_tiles;
  void* out;
  long long ldo;           // output row stride in elements
  const float* row_scale;  // kEpiScale
  uint32_t b_bytes;        // bytes of one B box (rows * 128)
  const int* row_token;    // gathered A tiles: token of each permuted row
  const void* gather_src;  // gathered A tiles: X (bf16, gather_ld bytes per row)
  long long gather_ld;
  int flags;               // bit 0: B loads evict-first in L2 (fused gather)
};

__device__ __forceinline__ float silu_fast(float g) { return g / (1.0f + __expf(-g)); }

// Output staging for coalesced stores: 128 rows x 256 B (128 bf16) in smem,
// 16-byte chunks XOR-swizzled by row so both the per-row writes (one row per
// thread) and the row-contiguous reads are bank-conflict free.
constexpr int kStageOutBytes = 128 * 256;

__device__ __forceinline__ void stage_put(uint8_t* buf, int r, int col, const uint32_t* pk) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = (col >> 3) + i;
    *reinterpret_cast<uint4*>(buf + r * 256 + ((k ^ (r & 15)) << 4)) =
        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  }
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// rows < m_valid of the staged tile (width bf16 columns) -> out (row stride ld)
__device__ __forceinline__ void copy_out(const uint8_t* buf, __nv_bfloat16* out, long long ld, int width,
                                         int m_valid, int tid) {
  const int cpr = width >> 3;  // 16-byte chunks per row
  for (int i = tid; i < 128 * cpr; i += 256) {
    const int row = i / cpr, k = i - row * cpr;
    if (row < m_valid)
      *reinterpret_cast<uint4*>(out + row * ld + (k << 3)) =
          *reinterpret_cast<const uint4*>(buf + row * 256 + ((k ^ (row & 15)) << 4));
  }
}

template <int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
                   const __grid_constant__ CUtensorMap mapB, const GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* stage_buf = smem + kStages * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_buf + kStageOutBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ntiles = *args.num_tiles;

  const bool fused = MODE == kEpiSwiGLU && args.gather_src != nullptr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], fused ? 2 : 1);  // TMA expect_tx arrive (+ the stage's gather warp)
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiThreads);
    }
    fence_mbar_init();
    tma_prefetch(&mapA);
    tma_prefetch(&mapA2);
    tma_prefetch(&mapB);
  }
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_slot, 2 * kAccCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: B always; A for tiles whose rows are
      // contiguous (explicit X_perm, or X itself for shared experts)
      int stage = 0;
      uint32_t phase = 0;
      // fused gather: weights stream through L2 evict-first so the token rows
      // of X (gathered evict-last, ~48 reads each) stay resident
      uint64_t pol_b;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_b));
      GemmTile nxt = blockIdx.x < static_cast<unsigned>(ntiles) ? args.tiles[blockIdx.x] : GemmTile{};
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const GemmTile tl = nxt;  // descriptor prefetched one tile ahead
        if (t + static_cast<int>(gridDim.x) < ntiles) nxt = args.tiles[t + gridDim.x];
        const bool alt = (tl.m_live & kTileAltA) != 0;
        const bool gather = fused && (tl.m_live & kTileGatherA) != 0;
        const void* ma = alt ? static_cast<const void*>(&mapA2) : static_cast<const void*>(&mapA);
        for (int kb = 0; kb < tl.nkb; ++kb) {
          uint8_t* sa = smem + stage * kStageBytes;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], (gather ? 0u : static_cast<uint32_t>(kABytes)) + args.b_bytes);
          if (!gather) tma_load_2d(sa, ma, &full[stage], kb * kTileK, tl.a_row);
          if (fused && (args.flags & 1))
            tma_load_2d_hint(sa + kABytes, &mapB, &full[stage], kb * kTileK, tl.b_row, pol_b);
          else
            tma_load_2d(sa + kABytes, &mapB, &full[stage], kb * kTileK, tl.b_row);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp < kGatherWarp0 + kGatherWarps) {
    if (fused) {
      // ---------------- row gatherers.  Warp g fills ring stage g, i.e. the
      // k-blocks whose running index (over this CTA's tiles) is g mod 4.
      // Lane l copies 16-byte chunk (l & 7) of row 4i + (l >> 3) in
      // instruction i; the chunk lands at its SWIZZLE_128B position.
      const int gw = warp - kGatherWarp0;
      const int rr = lane >> 3, ch = lane & 7;
      const uint32_t sa = smem_u32(smem + gw * kStageBytes);
      const char* X = static_cast<const char*>(args.gather_src);
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      uint32_t phase = 0;
      int g = 0;  // running k-block index
      // descriptor and row tokens are loaded one tile ahead: the loads of tile
      // i+1 are in flight while tile i's k-blocks are gathered
      auto load_tok = [&](const GemmTile& tl, int* tok) {
        if ((tl.m_live & kTileGatherA) == 0) return;
        const int* rt = args.row_token + tl.a_row;
#pragma unroll
        for (int j = 0; j < 4; ++j) tok[j] = rt[lane + 32 * j < tl.m_valid ? lane + 32 * j : 0];
      };
      const int t0 = blockIdx.x, gs = gridDim.x;
      GemmTile cur = t0 < ntiles ? args.tiles[t0] : GemmTile{};
      GemmTile nxt = t0 + gs < ntiles ? args.tiles[t0 + gs] : GemmTile{};
      int tok[4] = {0, 0, 0, 0};
      if (t0 < ntiles) load_tok(cur, tok);
      for (int t = t0; t < ntiles; t += gs) {
        int tok_n[4] = {0, 0, 0, 0};
        if (t + gs < ntiles) load_tok(nxt, tok_n);
        const GemmTile nxt2 = t + 2 * gs < ntiles ? args.tiles[t + 2 * gs] : GemmTile{};
        const GemmTile& tl = cur;
        const bool gather = (tl.m_live & kTileGatherA) != 0;
        const int first = (gw - g) & (kStages - 1);  // first k-block of this tile owned by this warp
        for (int kb = first; kb < tl.nkb; kb += kStages) {
          mbar_wait(&empty[gw], phase ^ 1);
          if (gather) {
            const char* src = X + kb * 128 + ch * 16;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int row = 4 * i + rr;
              const long long tk = __shfl_sync(0xffffffffu, tok[i >> 3], 4 * (i & 7) + rr);
              const uint32_t dst = sa + row * 128 + ((ch ^ (row & 7)) << 4);
              asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst),
                           "l"(src + tk * args.gather_ld), "l"(pol)
                           : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tcgen05 reads
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[gw]);
          phase ^= 1;
        }
        g += tl.nkb;
        cur = nxt;
        nxt = nxt2;
#pragma unroll
        for (int j = 0; j < 4; ++j) tok[j] = tok_n[j];
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      // ---------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      const uint32_t sbase = smem_u32(smem);
      GemmTile nxt = blockIdx.x < static_cast<unsigned>(ntiles) ? args.tiles[blockIdx.x] : GemmTile{};
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const GemmTile tl = nxt;  // descriptor prefetched one tile ahead
        if (t + static_cast<int>(gridDim.x) < ntiles) nxt = args.tiles[t + gridDim.x];
        const uint32_t idesc = idesc_bf16(kTileM, tl.n_mma);
        const uint32_t dtmem = tmem_base + acc * kAccCols;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < tl.nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = sbase + stage * kStageBytes;
          const uint64_t adesc = sdesc_sw128(sa);
          const uint64_t bdesc = sdesc_sw128(sa + kABytes);
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k) {
            // advance 16 bf16 = 32 B along K inside the 128 B swizzle row
            umma_bf16(dtmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    // ---------------- epilogue warps 2..9: two per TMEM lane quarter, 32-column
    // chunks interleaved between them
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - kEpiWarp0) >> 2;
    const int r = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    GemmTile nxt = blockIdx.x < static_cast<unsigned>(ntiles) ? args.tiles[blockIdx.x] : GemmTile{};
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const GemmTile tl = nxt;  // descriptor prefetched one tile ahead
      if (t + static_cast<int>(gridDim.x) < ntiles) nxt = args.tiles[t + gridDim.x];
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * kAccCols + (static_cast<uint32_t>(q * 32) << 16);
      const bool valid = r < tl.m_valid;
      const long long orow = static_cast<long long>(tl.out_row + r);
      if constexpr (MODE == kEpiSwiGLU) {
        // h = swish(g) * u -> bf16 -> staged in smem -> coalesced row stores
        const int nc = tl.n_mma >> 1;
        const bool live = r < (tl.m_live & 0xFFFFF);
        for (int c = 32 * half; c < nc; c += 64) {
          uint32_t g[32], u[32];
          tmem_ld32(taddr + c, g);
          tmem_ld32(taddr + nc + c, u);
          tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float h0 = 0.f, h1 = 0.f;
            if (live) {
              h0 = silu_fast(__uint_as_float(g[2 * i])) * __uint_as_float(u[2 * i]);
              h1 = silu_fast(__uint_as_float(g[2 * i + 1])) * __uint_as_float(u[2 * i + 1]);
            }
            pk[i] = pack_bf16x2(h0, h1);
          }
          stage_put(stage_buf, r, c, pk);
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);  // accumulator drained: MMA may reuse it
        epi_sync();
        copy_out(stage_buf, static_cast<__nv_bfloat16*>(args.out) + static_cast<long long>(tl.out_row) * args.ldo +
                                tl.out_col, args.ldo, nc, tl.m_valid, threadIdx.x - kEpiWarp0 * 32);
        epi_sync();
      } else if constexpr (MODE == kEpiScale) {
        // y = acc * raw score -> bf16.  All of this thread's columns are read
        // from TMEM first (4 x 32, packed to bf16 in registers) so the
        // accumulator is released to the MMA before any global traffic; then
        // staged 128 columns at a time for coalesced row stores.
        const float sc = valid ? args.row_scale[orow] : 0.f;
        uint32_t pk[4][16];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 32 * half + 64 * j;
          if (c < tl.n_mma) {
            uint32_t v[32];
            tmem_ld32(taddr + c, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i)
              pk[j][i] = pack_bf16x2(__uint_as_float(v[2 * i]) * sc, __uint_as_float(v[2 * i + 1]) * sc);
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int p0 = 128 * p;
          if (p0 >= tl.n_mma) break;
          const int w = min(128, tl.n_mma - p0);
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int c = 32 * half + 64 * jj;  // column inside this 128-wide pass
            if (c < w) stage_put(stage_buf, r, c, pk[2 * p + jj]);
          }
          epi_sync();
          copy_out(stage_buf, static_cast<__nv_bfloat16*>(args.out) + static_cast<long long>(tl.out_row) * args.ldo +
                                  tl.out_col + p0, args.ldo, w, tl.m_valid, threadIdx.x - kEpiWarp0 * 32);
          epi_sync();
        }
      } else {
        float* O = static_cast<float*>(args.out) + orow * args.ldo + tl.out_col;
        for (int c = 32 * half; c < tl.n_mma; c += 64) {
          uint32_t v[32];
          tmem_ld32(taddr + c, v);
          tmem_ld_wait();
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(O + c);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        }
      }
      if constexpr (MODE == kEpiF32) {
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc(tmem_base, 2 * kAccCols);
}

// ------------------------------------------------------------------ launcher
int launch_gemm_tc(int mode, const CUtensorMap* mapA, const CUtensorMap* mapA2,
                   const CUtensorMap* mapB, const GemmTile* tiles, const int* num_tiles,
                   int max_tiles, void* out, long long ldo, const float* row_scale,
                   int b_box_rows, int num_sms, cudaStream_t stream, const int* row_token,
                   const void* gather_src, long long gather_ld) {
  static const int flags = [] {
    const char* v = std::getenv("DSMOE_B200_GEMM_FLAGS");
    return v ? std::atoi(v) : 0;
  }();
  GemmArgs a{tiles, num_tiles, out, ldo, row_scale, static_cast<uint32_t>(b_box_rows * 128), row_token,
             gather_src, gather_ld, flags};
  const int grid = max_tiles < num_sms ? (max_tiles > 0 ? max_tiles : 1) : num_sms;
  cudaError_t err;
  switch (mode) {
#define DSB_LAUNCH(M)                                                                         \
  case M: {                                                                                   \
    static bool attr = false;                                                                 \
    if (!attr) {                                                                              \
      cudaFuncSetAttribute(gemm_tc_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                           kGemmSmem);                                                        \
      attr = true;                                                                            \
    }                                                                                         \
    gemm_tc_kernel<M><<<grid, kGemmThreads, kGemmSmem, stream>>>(*mapA, *mapA2, *mapB, a);    \
    break;                                                                                    \
  }
    DSB_LAUNCH(kEpiF32)
    DSB_LAUNCH(kEpiSwiGLU)
    DSB_LAUNCH(kEpiScale)
#undef DSB_LAUNCH
    default:
      return -1;
  }
  err = cudaGetLastError();
  return err == cudaSuccess ? 0 : static_cast<int>(err);
}

}  // namespace dsb
