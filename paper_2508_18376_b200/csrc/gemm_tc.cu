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
  int flags;               // DSMOE_B200_GEMM_FLAGS: bit 0 B loads evict-first (fused gather), bit 1 no TMA stores
  int tma_store;           // bf16 outputs leave through mapO
};

// swish(g) = g * sigmoid(g) = 0.5 g (1 + tanh(g / 2)): one MUFU op (tanh.approx,
// rel. err ~2^-11, below the bf16 rounding of h that follows).
__device__ __forceinline__ float silu_fast(float g) {
  const float hg = 0.5f * g;
  float th;
  asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(hg));
  return fmaf(hg, th, hg);
}

// Output staging, per epilogue warp: a 4 KB slot = its 32 rows x 64 bf16
// columns as one TMA box (32 rows x 128 B, SWIZZLE_128B: 16-byte chunk k of
// row rr at rr*128 + ((k ^ (rr & 7)) << 4)).  Every warp stores on its own
// (lane 0 issues the TMA store and owns the bulk group), so the epilogue has
// no CTA-wide barriers; rows cut by the segment end are copied out masked.
constexpr int kWarpSlot = 32 * 128;
constexpr int kStageOutBytes = 8 * kWarpSlot;

// columns [col, col + 32) of this lane's row (pk: 16 packed bf16 pairs)
__device__ __forceinline__ void warp_put(uint8_t* slot, int lane, int col, const uint32_t* pk) {
  uint8_t* rowp = slot + lane * 128;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = (col >> 3) + i;
    *reinterpret_cast<uint4*>(rowp + ((k ^ (lane & 7)) << 4)) =
        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  }
}

// wait until this warp's previous TMA store has read the slot
__device__ __forceinline__ void warp_slot_acquire(int lane) {
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
}

// slot -> out rows [row0, row0 + min(32, nvalid)), columns [col0, col0 + 64)
__device__ __forceinline__ void warp_store(const uint8_t* slot, const CUtensorMap* mapO, const GemmArgs& args,
                                           int row0, int col0, int nvalid, bool full, int lane) {
  if (full && args.tma_store) {
    fence_proxy_async();  // generic smem writes -> async-proxy (TMA) reads
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(mapO, smem_u32(slot), col0, row0);
      bulk_commit();
    }
  } else {
    __syncwarp();
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(args.out);
    const int k = lane & 7;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = 4 * i + (lane >> 3);
      if (rr < nvalid)
        *reinterpret_cast<uint4*>(out + static_cast<long long>(row0 + rr) * args.ldo + col0 + 8 * k) =
            *reinterpret_cast<const uint4*>(slot + rr * 128 + ((k ^ (rr & 7)) << 4));
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapO,
                   const GemmArgs args) {
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
    if (args.tma_store) tma_prefetch(&mapO);
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
    // ---------------- MMA issuer: the whole warp walks the loop (warp-uniform
    // control, so descriptors live in uniform registers); one elected lane
    // issues the tcgen05.mma / commit instructions.
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint64_t d0 = sdesc_sw128(smem_u32(smem));  // stage 0 A; + (bytes >> 4) moves the start address
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
        const uint64_t adesc = d0 + static_cast<uint64_t>(stage * (kStageBytes >> 4));
        const uint64_t bdesc = adesc + (kABytes >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k)  // 16 bf16 = 32 B along K inside the 128 B swizzle row
            umma_bf16(dtmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ---------------- epilogue warps 2..9: two per TMEM lane quarter, 32-column
    // chunks interleaved between them
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - kEpiWarp0) >> 2;
    const int r = q * 32 + lane;
    uint8_t* wslot = stage_buf + (warp - kEpiWarp0) * kWarpSlot;  // this warp's staging slot
    int acc = 0;
    uint32_t acc_phase = 0;
    GemmTile nxt = blockIdx.x < static_cast<unsigned>(ntiles) ? args.tiles[blockIdx.x] : GemmTile{};
    float sc_nxt = 0.f;  // kEpiScale: this thread's row score, loaded a tile ahead
    if (MODE == kEpiScale && blockIdx.x < static_cast<unsigned>(ntiles) && r < nxt.m_valid)
      sc_nxt = args.row_scale[nxt.out_row + r];
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const GemmTile tl = nxt;  // descriptor prefetched one tile ahead
      const float sc_cur = sc_nxt;
      if (t + static_cast<int>(gridDim.x) < ntiles) {
        nxt = args.tiles[t + gridDim.x];
        if (MODE == kEpiScale && r < nxt.m_valid) sc_nxt = args.row_scale[nxt.out_row + r];
      }
      (void)sc_cur;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (args.flags & 8) {  // diagnostics only (wrong results): no epilogue, MMA-only timing
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      const uint32_t taddr = tmem_base + acc * kAccCols + (static_cast<uint32_t>(q * 32) << 16);
      const bool valid = r < tl.m_valid;
      const long long orow = static_cast<long long>(tl.out_row + r);
      // this warp's rows [32q, 32q + 32) of the tile: all inside the segment ->
      // one TMA store per 64-column box; cut by the segment end -> masked copy
      const bool rows_full = 32 * q + 32 <= tl.m_valid;
      if constexpr (MODE == kEpiSwiGLU) {
        // h = swish(g) * u over columns [64 half, 64 half + 64) of the nc-wide output
        const int nc = tl.n_mma >> 1;
        const bool live = r < (tl.m_live & 0xFFFFF);
        const int c0 = 64 * half;  // output columns of this warp: groups 2 half, 2 half + 1
        if (c0 < nc) {
          warp_slot_acquire(lane);
#pragma unroll
          for (int gi = 0; gi < 2; ++gi) {
            uint32_t v[64];  // [g of 32 neurons | u of the same 32]
            tmem_ld64(taddr + 2 * c0 + 64 * gi, v);
            tmem_ld_wait();
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              float h0 = 0.f, h1 = 0.f;
              if (live) {
                h0 = silu_fast(__uint_as_float(v[2 * i])) * __uint_as_float(v[32 + 2 * i]);
                h1 = silu_fast(__uint_as_float(v[2 * i + 1])) * __uint_as_float(v[32 + 2 * i + 1]);
              }
              pk[i] = pack_bf16x2(h0, h1);
            }
            warp_put(wslot, lane, 32 * gi, pk);
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[acc]);  // accumulator drained: MMA may reuse it
        if (c0 < nc)
          warp_store(wslot, &mapO, args, tl.out_row + 32 * q, tl.out_col + c0, tl.m_valid - 32 * q, rows_full, lane);
      } else if constexpr (MODE == kEpiScale) {
        // y = acc * raw score -> bf16; pass p = columns [128p + 64 half, +64),
        // one x64 TMEM load each.  The row's score was loaded a tile ahead.
        const float sc = valid ? sc_cur : 0.f;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int c = 128 * p + 64 * half;
          const bool have = c < tl.n_mma;
          uint32_t pk[32];
          if (have) {
            uint32_t v[64];
            tmem_ld64(taddr + c, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i)
              pk[i] = pack_bf16x2(__uint_as_float(v[2 * i]) * sc, __uint_as_float(v[2 * i + 1]) * sc);
          }
          if (p == 1) {
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
          }
          if (have) {
            warp_slot_acquire(lane);
            warp_put(wslot, lane, 0, pk);
            warp_put(wslot, lane, 32, pk + 16);
            warp_store(wslot, &mapO, args, tl.out_row + 32 * q, tl.out_col + c, tl.m_valid - 32 * q, rows_full, lane);
          }
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
      (void)valid; (void)orow;
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  if (warp >= kEpiWarp0 && lane == 0) bulk_wait0();  // this lane's TMA stores still read its staging slot
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc(tmem_base, 2 * kAccCols);
}

// ------------------------------------------------------------------ launcher
int launch_gemm_tc(int mode, const CUtensorMap* mapA, const CUtensorMap* mapA2,
                   const CUtensorMap* mapB, const GemmTile* tiles, const int* num_tiles,
                   int max_tiles, void* out, long long ldo, const float* row_scale,
                   int b_box_rows, int num_sms, cudaStream_t stream, const int* row_token,
                   const void* gather_src, long long gather_ld, const CUtensorMap* mapO) {
  static const int flags = [] {
    const char* v = std::getenv("DSMOE_B200_GEMM_FLAGS");
    return v ? std::atoi(v) : 0;
  }();
  GemmArgs a{tiles, num_tiles, out, ldo, row_scale, static_cast<uint32_t>(b_box_rows * 128), row_token,
             gather_src, gather_ld, flags, mapO != nullptr && mode != kEpiF32 && !(flags & 2) ? 1 : 0};
  const CUtensorMap* mo = mapO ? mapO : mapB;
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
    gemm_tc_kernel<M><<<grid, kGemmThreads, kGemmSmem, stream>>>(*mapA, *mapA2, *mapB, *mo, a);    \
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
