// K3 / K4 (and K0): persistent grouped GEMM on the 5th-generation tensor cores.
//
// Replaces the per-token scalar loops of accumulate_block
// (/root/reference/proj/include/dsmoe/moe.hpp:213-231) and the gate matmul of
// gate_scores (moe.hpp:174 -> matrix.hpp:47-64) for bf16 layers.
//
// One CTA per SM (warp-specialised, 32 x (1 + kAStages + 1 + 8) threads):
//   warp 0      TMA producer: B (N x 64) weight tiles into a kBStages-deep ring,
//               and A (128 x 64) when the rows are contiguous (explicit X_perm,
//               H, or x itself for shared experts) into a kAStages-deep ring;
//               SWIZZLE_128B, full/empty mbarriers per ring;
//   warps 1..   row gatherers (GEMM1 with fused gather only): warp g owns A
//               stage g and fills it straight from the token rows of X
//               (16-byte cp.async, one warp instruction = 4 rows x 128 B, so
//               every request is a whole L2 line), then proxy-fences and
//               arrives — no permuted copy of X in HBM.  The A ring is the
//               deeper one: gather latency is what the MMA waits on;
//   MMA warp    TMEM allocator + warp-uniform loop, an elected lane issues
//               tcgen05.mma (M=128, N<=256, K=16), fp32 accumulators in TMEM,
//               two accumulator stages (2 x 256 columns) so the epilogue of
//               tile i overlaps the MMAs of tile i+1;
//   8 epilogue  two warps per TMEM lane quarter: tcgen05.ld 32x32b.x64 ->
//   warps       registers -> fused op -> bf16 -> per-warp smem slot -> TMA store.
// Work items (GemmTile) are produced on the device by plan_body (permute.cu)
// and walked in a static round-robin over the persistent CTAs.
//
// PAIR = true (GEMM2 by default): a 2-CTA cluster runs one M = 256 tile with
// tcgen05.mma.cta_group::2 issued by the leader; each CTA stages its own 128
// A rows and half of the B rows; TMA bytes of both CTAs are counted by one
// leader arrive.expect_tx, MMA completion is multicast to both CTAs' empty /
// accumulator barriers, epilogue warps release the accumulator with one
// remote arrive each on the leader's barrier.
//
// Epilogue modes
//   kEpiF32     fp32 store (gate logits, K0; kEpiF32Wide for > 64 experts);
//   kEpiSwiGLU  h = swish(g) * u over [32 g | 32 u] column groups of the tile,
//               rows >= m_live store zeros (major-only rows of a minor chunk),
//               bf16 store into H (K3);
//   kEpiScale   y = acc * row_scale[row] (the raw gate score, moe.hpp:235-237),
//               bf16 store into Y (K4).
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace dsb {

// Separate operand rings: A (128 x 64 rows of tokens) is the latency-critical
// one under the fused gather, so it is deeper than the B (weights) ring.
// CTA pair + fused gather: how the peer's gathered A stage is handed to the
// leader's MMA.  1 (default): the gather warp waits for its cp.async group,
// fences generic -> async proxy at CTA scope and arrives on the leader's
// barrier with a plain (release.cta) remote arrive, the MMA warp polls it with
// a plain try_wait — the hand-off CUTLASS's 2-SM UMMA pipelines use
// (umma_arrive_2x1SM_sm0).  0: release.cluster arrive + acquire.cluster wait +
// cluster-scope proxy fence, which costs 45% more GEMM1 cycles (1361 vs 832
// kcyc, profiles/r13_summary.md).
#ifndef DSB_PAIR_RELAXED
#define DSB_PAIR_RELAXED 1
#endif
#ifndef DSB_PA_STAGES  // CTA pairs: A / B ring depths (16 KB slots each)
#define DSB_PA_STAGES 6
#endif
#ifndef DSB_PB_STAGES
#define DSB_PB_STAGES 6
#endif
#ifndef DSB_A_STAGES
#define DSB_A_STAGES 5
#endif
#ifndef DSB_B_STAGES
#define DSB_B_STAGES 4
#endif
// 1: epilogue warps stage 32 x 64 tiles in smem and leave with TMA stores;
// 0: each thread stores its row's 64-byte runs straight from registers (the
//    32 KB of staging go to the operand rings instead)
#ifndef DSB_STAGE_OUT
#define DSB_STAGE_OUT 2
#endif
constexpr int kABytes = kTileM * kTileK * 2;       // 16 KB
constexpr int kBBytesMax = 256 * kTileK * 2;       // 32 KB
constexpr int kEpiThreads = 256;
constexpr int kAccCols = 256;
constexpr bool kStageOut = DSB_STAGE_OUT != 0;
constexpr int kStageSmem = DSB_STAGE_OUT == 1 ? 8 * 32 * 128 : DSB_STAGE_OUT == 2 ? 8 * 32 * 64 : 0;

enum { kEpiF32 = 0, kEpiSwiGLU = 1, kEpiScale = 2, kEpiF32Wide = 3 };

// Per-mode pipeline geometry.  GEMM1/GEMM2: A (tokens) ring DSB_A_STAGES deep,
// B (weights, N <= 256 rows) ring DSB_B_STAGES deep; gather warps only where
// the fused gather runs (GEMM1).  Gate logits (N = Epad <= 64): 8 KB B slots,
// so both rings can be 8 deep — the gate GEMM is a 64 MB stream of x with
// little math, and in-flight bytes are what bound it.
// dynamic tile claims: id ring slots.  No reader ever lags the leader's
// producer by more than a few tiles (the B ring bounds the producer's lead
// over the MMA, the two accumulators the MMA's over the epilogue, and every
// peer walker is paced by the leader's barriers), so a slot is never
// rewritten before all walkers read it and no "slot free" barrier is needed —
// per-tile remote release-arrives from 15 peer warps cost 5-10% of the GEMMs.
constexpr int kSeq = 32;

#ifndef DSB_GEMM_TIMES
#define DSB_GEMM_TIMES 0  // diagnostic builds: per-launch min / max of CTA entry, post-wait and exit times
#endif
__device__ unsigned long long g_gemm_times[4][8];  // [mode][entry min, max, wait min, max, end min, max, count, -]
__device__ __forceinline__ unsigned long long gemm_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int kLook = 3;  // ids claimed ahead of the tile the leader's producer loads (gather warps read 2 ahead)

template <int MODE, bool PAIR = false>
struct Geo {
  static constexpr bool kGate = MODE == kEpiF32;
  // CTA pair: each CTA stages its 128 A rows and HALF of the B rows (<= 128,
  // 16 KB slots), so both rings can be 6 deep in the same shared memory
  static constexpr int NA = PAIR ? DSB_PA_STAGES : kGate ? 8 : DSB_A_STAGES;
  static constexpr int NB = PAIR ? DSB_PB_STAGES : kGate ? 8 : DSB_B_STAGES;
  static constexpr int BSLOT = PAIR ? 128 * kTileK * 2 : kGate ? 64 * kTileK * 2 : kBBytesMax;
  static constexpr int NGW = MODE == kEpiSwiGLU ? NA : 0;  // gather warps, warp 1 + s owns A stage s
  static constexpr int GW0 = 1;
  static constexpr int MMA = GW0 + NGW;  // TMEM alloc + tcgen05.mma issue
  static constexpr int EPI0 = MMA + 1;   // 8 epilogue warps
  static constexpr int THREADS = (EPI0 + 8) * 32;
  static constexpr int RING = NA * kABytes + NB * BSLOT;
  static constexpr int STAGE = (MODE == kEpiF32 || MODE == kEpiF32Wide) ? 0 : kStageSmem;
  static constexpr int SMEM = RING + STAGE + 1024 /*align*/ + 1024 /*barriers, tile-id ring*/;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert((2 * NA + 2 * NB + 4 + kSeq) * 8 + kSeq * 4 + 4 <= 1024, "barrier area");
};

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
  int flags;               // DSMOE_B200_GEMM_FLAGS: bit 0 B loads evict-first (fused gather), bit 1 no TMA stores,
                           // bit 4 / 5: GEMM1 / GEMM2 output stores evict-first
  int tma_store;           // bf16 outputs leave through mapO
  unsigned long long* zero4;  // gate: the router's 4 counters, zeroed here (saves a memset between launches)
  int* sched;              // CTA pairs: [claim counter, done counter], zero between launches ->
                           // tiles are claimed dynamically (atomic counter) instead of t0 + k gs
};

// swish(g) = g * sigmoid(g) = 0.5 g (1 + tanh(g / 2)): one MUFU op (tanh.approx,
// rel. err ~2^-11, below the bf16 rounding of h that follows).
__device__ __forceinline__ float silu_fast(float g) {
  const float hg = 0.5f * g;
  float th;
  asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(hg));
  return fmaf(hg, th, hg);
}

// Output staging, per epilogue warp (DSB_STAGE_OUT 1): a 4 KB slot = its 32
// rows x 64 bf16 columns as one TMA box (rows of 128 B, SWIZZLE_128B: 16-byte
// chunk k of row rr at rr*128 + ((k ^ (rr & 7)) << 4)); DSB_STAGE_OUT 2: a
// 2 KB slot of 32 rows x 32 columns (rows of 64 B, SWIZZLE_64B: chunk k at
// rr*64 + ((k ^ ((rr >> 1) & 3)) << 4)), which leaves 16 KB more for the
// operand rings.  Every warp stores on its own (lane 0 issues the TMA store
// and owns the bulk group), so the epilogue has no CTA-wide barriers; rows cut
// by the segment end are copied out masked.
constexpr int kBoxCols = DSB_STAGE_OUT == 2 ? 32 : 64;
// half-M pair tiles for segment tails (<= 128 rows); needs the 32-column boxes
#ifndef DSB_HALF_M
#define DSB_HALF_M 1
#endif
constexpr bool kHalfM = DSB_HALF_M != 0 && (kBoxCols == 32 || DSB_STAGE_OUT == 0);
constexpr int kRowBytes = kBoxCols * 2;
constexpr int kWarpSlot = 32 * kRowBytes;

__device__ __forceinline__ int swz(int rr, int k) {
  return kBoxCols == 64 ? (k ^ (rr & 7)) : (k ^ ((rr >> 1) & 3));
}

// columns [col, col + 32) of the slot's box for this lane's row (pk: 16 packed bf16 pairs)
__device__ __forceinline__ void warp_put(uint8_t* slot, int lane, int col, const uint32_t* pk) {
  uint8_t* rowp = slot + lane * kRowBytes;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = (col >> 3) + i;
    *reinterpret_cast<uint4*>(rowp + (swz(lane, k) << 4)) =
        make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  }
}

// wait until this warp's previous TMA store has read the slot
__device__ __forceinline__ void warp_slot_acquire(int lane) {
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
}

// slot -> out rows [row0, row0 + min(32, nvalid)), columns [col0, col0 + kBoxCols)
// st_pol != 0: the TMA store carries that L2 policy (DSMOE_B200_GEMM_FLAGS bits 4 / 5)
__device__ __forceinline__ void warp_store(const uint8_t* slot, const CUtensorMap* mapO, const GemmArgs& args,
                                           int row0, int col0, int nvalid, bool full, int lane,
                                           uint64_t st_pol = 0) {
  if (full && args.tma_store) {
    fence_proxy_async();  // generic smem writes -> async-proxy (TMA) reads
    __syncwarp();
    if (lane == 0) {
      if (st_pol)
        tma_store_2d_hint(mapO, smem_u32(slot), col0, row0, st_pol);
      else
        tma_store_2d(mapO, smem_u32(slot), col0, row0);
      bulk_commit();
    }
  } else {
    __syncwarp();
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(args.out);
    constexpr int kChunks = kRowBytes / 16;  // 16-byte chunks per row
    constexpr int kRowsPerPass = 32 / kChunks;
    const int k = lane % kChunks;
#pragma unroll
    for (int i = 0; i < kChunks; ++i) {
      const int rr = kRowsPerPass * i + lane / kChunks;
      if (rr < nvalid)
        *reinterpret_cast<uint4*>(out + static_cast<long long>(row0 + rr) * args.ldo + col0 + 8 * k) =
            *reinterpret_cast<const uint4*>(slot + rr * kRowBytes + (swz(rr, k) << 4));
    }
  }
}

// box columns the TMA-store map must use (host side builds the map)
int gemm_tc_store_box_cols() { return kBoxCols; }

// direct path: columns [col, col + 32) of output row `row` from registers
__device__ __forceinline__ void row_put(const GemmArgs& args, long long row, int col, const uint32_t* pk) {
  uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(args.out) + row * args.ldo + col);
#pragma unroll
  for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
}

template <int MODE, bool PAIR>
__global__ void __launch_bounds__(Geo<MODE, PAIR>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapA2,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapO,
                   const GemmArgs args) {
  using G = Geo<MODE, PAIR>;
  constexpr int kAStages = G::NA, kBStages = G::NB, kBSlot = G::BSLOT;
  constexpr int kGatherWarp0 = G::GW0, kGatherWarps = G::NGW, kMmaWarp = G::MMA, kEpiWarp0 = G::EPI0;
  constexpr int kRingBytes = G::RING;
  constexpr int kStageOutBytes = G::STAGE;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  const unsigned long long t_entry = DSB_GEMM_TIMES ? gemm_now() : 0ull;
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* ringA = smem;                              // kAStages x 16 KB
  uint8_t* ringB = smem + kAStages * kABytes;         // kBStages x kBSlot
  uint8_t* stage_buf = smem + kRingBytes;
  uint64_t* fullA = reinterpret_cast<uint64_t*>(stage_buf + kStageOutBytes);
  uint64_t* emptyA = fullA + kAStages;
  uint64_t* fullB = emptyA + kAStages;
  uint64_t* emptyB = fullB + kBStages;
  uint64_t* tfull = emptyB + kBStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;  // dynamic tile claims: id ring slot written (both CTAs)
  int* sring = reinterpret_cast<int*>(sfull + kSeq);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sring + kSeq);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // CTA pair: tiles are M = 256; this CTA owns rows [128 rank, 128 rank + 128)
  // and the B rows [rank * N/2, (rank + 1) * N/2); the leader issues the MMAs.
  const int rank = PAIR ? static_cast<int>(pair_rank()) : 0;
  const bool leader = rank == 0;
  const int t0 = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int gs = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  // CTA pair, tiles of <= 128 rows (segment tails): tcgen05.mma M = 128
  // (cta_group::2), each CTA contributes 64 A rows; D lands in each CTA's TMEM
  // as 64 rows x N with N columns [0, N/2) in lanes 0-63 and [N/2, N) in lanes
  // 64-127, both at columns [0, N/2) (probed: tools/micro/pair_m128_probe.cu).
  // Half the MMA time of an M = 256 tile that carries the same rows.
  // (N a multiple of 128, so each lane half holds whole 64-column groups)
  auto half_m = [&](const GemmTile& t) { return PAIR && kHalfM && t.m_valid <= 128 && (t.n_mma & 127) == 0; };
  auto row_off_of = [&](const GemmTile& t) { return half_m(t) ? 64 * rank : 128 * rank; };

  const bool fused = MODE == kEpiSwiGLU && kGatherWarps > 0 && args.gather_src != nullptr;
  // Tile schedule.  Static: this CTA (pair) walks tiles t0, t0 + gs, ...
  // Dynamic (CTA pairs with args.sched): the leader's producer thread claims
  // tile ids from a global counter, kLook positions ahead of the tile it loads,
  // and publishes them in a kSeq-slot ring in both CTAs' shared memory; every
  // walker (producers, gather warps, MMA warp, epilogue warps) reads the ids in
  // order and releases each slot on the leader's barrier.  A pair that runs
  // slow (its SM clock, its memory latency, its tiles' costs) claims fewer
  // tiles, so all pairs finish together.
  const bool dyn_ok = PAIR && args.sched != nullptr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kAStages; ++s) {
      // TMA-fed stages: one arrive.expect_tx (pair: the leader's, for both CTAs'
      // bytes; the peer's TMA only completes bytes on it).  Gathered stages:
      // one arrive per CTA's gather warp.
      mbar_init(&fullA[s], (PAIR && fused) ? 2 : 1);
      mbar_init(&emptyA[s], 1);
    }
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], PAIR ? 16 : kEpiThreads);  // pair: one arrive per epilogue warp of both CTAs
    }
    if (dyn_ok)
      for (int s = 0; s < kSeq; ++s) mbar_init(&sfull[s], 1);
    fence_mbar_init();
    tma_prefetch(&mapA);
    tma_prefetch(&mapA2);
    tma_prefetch(&mapB);
    if (args.tma_store) tma_prefetch(&mapO);
  }
  if (warp == kMmaWarp) {
    if constexpr (PAIR)
      tmem_alloc_pair(tmem_slot, 2 * kAccCols);
    else {
      tmem_alloc(tmem_slot, 2 * kAccCols);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if constexpr (PAIR) {
    pair_sync();      // the peer's barriers exist before any remote arrive
    __syncthreads();  // (and a CTA barrier the race checker models for the TMEM slot)
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the predecessor's outputs (tile lists, A rows) are complete from here on
  const unsigned long long t_wait = DSB_GEMM_TIMES ? gemm_now() : 0ull;
  if (MODE == kEpiF32 || MODE == kEpiF32Wide) pdl_trigger();  // gate: the router may launch
  if (MODE == kEpiScale) pdl_trigger_tail();
#ifdef DSB_PDL_TRIGGER_G1  // experiment: GEMM1 -> GEMM2 (GEMM2 CTAs take SMs as GEMM1 CTAs exit)
  if (MODE == kEpiSwiGLU) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  const int ntiles = *args.num_tiles;
  // claims pay off only with many tiles per pair (tail balance); with a few
  // (small batches) claiming ahead would pile several tiles on some pairs
  // while others idle — there the round-robin order is already balanced
  const bool dyn = dyn_ok && ntiles >= 16 * gs;
  if ((MODE == kEpiF32 || MODE == kEpiF32Wide) && args.zero4 && blockIdx.x == 0 && threadIdx.x < 4) args.zero4[threadIdx.x] = 0ull;
  // "operand ready": own barrier (single CTA) / the leader's (pair)
  auto ready_arrive = [&](uint64_t* bar) {
    if constexpr (PAIR)
      pair_arrive_leader(bar);
    else
      mbar_arrive(bar);
  };
  // one CTA's TMA load of `bytes` into `dst`, counted on the (leader's) full barrier
  // peer_arrives: the barrier also counts one arrival from the peer CTA (gathered A ring)
  auto load_op = [&](void* dst, const void* map, uint64_t* bar, int c0, int c1, uint32_t bytes,
                     bool peer_arrives = false) {
    if constexpr (PAIR) {
      if (leader)
        mbar_expect_tx(bar, 2 * bytes);
      else if (peer_arrives)
        DSB_PAIR_RELAXED ? pair_arrive_leader_cta(bar) : pair_arrive_leader(bar);
      tma_load_2d_to_leader(dst, map, bar, c0, c1);
    } else {
      mbar_expect_tx(bar, bytes);
      tma_load_2d(dst, map, bar, c0, c1);
    }
  };

  // the next tile id of this pair's sequence (reader state rd / rend), -1 at
  // the end; warp_wide: the whole warp calls it (lane 0 releases the slot)
  auto next_id = [&](int& rd, bool& rend, bool warp_wide) -> int {
    if (rend) return -1;
    int v;
    if (!dyn) {
      v = t0 + rd * gs;
      if (v >= ntiles) v = -1;
    } else {
      const int s = rd % kSeq;
      const uint32_t ph = static_cast<uint32_t>(rd / kSeq) & 1u;
#ifdef DSB_SCHED_CLUSTER_ACQ  // A/B: plain remote store + cluster-scope acquire on the peer
      if (leader)
        mbar_wait(&sfull[s], ph);
      else
        mbar_wait_cluster(&sfull[s], ph);
#else  // the peer's slot arrives by st.async, tracked on its own barrier
      mbar_wait(&sfull[s], ph);
#endif
      v = *reinterpret_cast<volatile int*>(&sring[s]);
      (void)warp_wide;
    }
    ++rd;
    if (v < 0) rend = true;
    return v;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer: B always; A too unless the gather warps own it
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      uint64_t pol_b;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_b));
      // the leader's claims: sequence positions [0, claimed) are published.
      // The atomic of the next claim is issued one tile before its value is
      // published, so its latency never stalls the loads.
      int claimed = 0, pend = 0;
      bool ended = false, have_pend = false;
      auto publish = [&](int t) {
        const int s = claimed % kSeq;
        if (t >= ntiles) {
          t = -1;
          ended = true;
          // every pair publishes exactly one claim past the end: the last one re-arms the counters
          if (atomicAdd(args.sched + 1, 1) == gs - 1) {
            atomicExch(args.sched, 0);
            atomicExch(args.sched + 1, 0);
          }
        }
        sring[s] = t;
        mbar_arrive(&sfull[s]);
#ifdef DSB_SCHED_CLUSTER_ACQ
        pair_store_arrive_peer(&sring[s], t, &sfull[s], 1);
#else
        pair_store_async_peer(&sring[s], t, &sfull[s], 1);
#endif
        ++claimed;
      };
#ifdef DSB_SCHED_RING_STATIC  // diagnostic: the ring protocol with the static order (t0 + k gs)
      int kstat = 0;
      auto claim1 = [&]() { return t0 + (kstat++) * gs; };
#else
      auto claim1 = [&]() { return atomicAdd(args.sched, 1); };
#endif
      if (dyn && leader) {
#ifdef DSB_SCHED_RING_STATIC
        for (int k = 0; k <= kLook && !ended; ++k) publish(claim1());
#else
        const int base = atomicAdd(args.sched, kLook + 1);  // the first kLook + 1 positions: one atomic
        for (int k = 0; k <= kLook && !ended; ++k) publish(base + k);
#endif
        if (!ended) {
          pend = claim1();
          have_pend = true;
        }
      }
      int rd = 0, j = 0;
      bool rend = false;
      int id = next_id(rd, rend, false);
      GemmTile nxt = id >= 0 ? args.tiles[id] : GemmTile{};
      while (id >= 0) {
        const GemmTile tl = nxt;  // descriptor prefetched one tile ahead
        if (have_pend && claimed <= j + 1 + kLook) {  // keep kLook ids published past this tile
          have_pend = false;
          publish(pend);
          if (!ended) {
            pend = claim1();
            have_pend = true;
          }
        }
        id = next_id(rd, rend, false);
        if (id >= 0) nxt = args.tiles[id];
        ++j;
        const bool alt = (tl.m_live & kTileAltA) != 0;
        const void* ma = alt ? static_cast<const void*>(&mapA2) : static_cast<const void*>(&mapA);
        const int brow = tl.b_row + (PAIR ? rank * (tl.n_mma >> 1) : 0);
        // gate tiles of a split-K launch: K blocks [kb0, kb0 + nkb) (m_live low bits)
        const int kb0 = (MODE == kEpiF32 || MODE == kEpiF32Wide) ? (tl.m_live & 0xFFFFF) : 0;
        for (int kb = 0; kb < tl.nkb; ++kb) {
          if (!fused) {
            mbar_wait(&emptyA[sa], pa ^ 1);
            load_op(ringA + sa * kABytes, ma, &fullA[sa], (kb0 + kb) * kTileK, tl.a_row + row_off_of(tl), kABytes);
            if (++sa == kAStages) { sa = 0; pa ^= 1; }
          }
          mbar_wait(&emptyB[sb], pb ^ 1);
          if (!PAIR && fused && (args.flags & 1)) {
            mbar_expect_tx(&fullB[sb], args.b_bytes);
            tma_load_2d_hint(ringB + sb * kBSlot, &mapB, &fullB[sb], kb * kTileK, brow, pol_b);
          } else {
            load_op(ringB + sb * kBSlot, &mapB, &fullB[sb], (kb0 + kb) * kTileK, brow, args.b_bytes);
          }
          if (++sb == kBStages) { sb = 0; pb ^= 1; }
        }
      }
    }
  } else if (warp < kGatherWarp0 + kGatherWarps) {
    if (fused) {
      // ---------------- row gatherers.  Warp g fills A stage g, i.e. the
      // k-blocks whose running index (over this CTA's tiles) is g mod kAStages.
      // Lane l copies 16-byte chunk (l & 7) of row 4i + (l >> 3) in
      // instruction i; the chunk lands at its SWIZZLE_128B position.  Tiles
      // whose rows are contiguous in X (shared experts) are one TMA load.
      const int gw = warp - kGatherWarp0;
      const int rr = lane >> 3, ch = lane & 7;
      uint8_t* sa_ptr = ringA + gw * kABytes;
      const uint32_t sa = smem_u32(sa_ptr);
      const char* X = static_cast<const char*>(args.gather_src);
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      uint32_t phase = 0;
      int g = 0;  // running k-block index
      // descriptor and row tokens are loaded one tile ahead: the loads of tile
      // i+1 are in flight while tile i's k-blocks are gathered
      auto load_tok = [&](const GemmTile& tl, int* tok) {
        if ((tl.m_live & kTileGatherA) == 0) return;
        const int* rt = args.row_token + tl.a_row;  // this CTA's rows start at row_off_of(tl)
        const int ro = row_off_of(tl);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i = ro + lane + 32 * j;
          tok[j] = rt[i < tl.m_valid ? i : 0];
        }
      };
      int rd = 0;
      bool rend = false;
      int id_cur = next_id(rd, rend, true);
      int id_nxt = next_id(rd, rend, true);
      GemmTile cur = id_cur >= 0 ? args.tiles[id_cur] : GemmTile{};
      GemmTile nxt = id_nxt >= 0 ? args.tiles[id_nxt] : GemmTile{};
      int tok[4] = {0, 0, 0, 0};
      if (id_cur >= 0) load_tok(cur, tok);
      while (id_cur >= 0) {
        int tok_n[4] = {0, 0, 0, 0};
        if (id_nxt >= 0) load_tok(nxt, tok_n);
        const int id_nxt2 = next_id(rd, rend, true);
        const GemmTile nxt2 = id_nxt2 >= 0 ? args.tiles[id_nxt2] : GemmTile{};
        id_cur = id_nxt;
        id_nxt = id_nxt2;
        const GemmTile& tl = cur;
        const bool gather = (tl.m_live & kTileGatherA) != 0;
        const void* ma = (tl.m_live & kTileAltA) ? static_cast<const void*>(&mapA2) : static_cast<const void*>(&mapA);
        int first = (gw - g) % kAStages;  // first k-block of this tile owned by this warp
        if (first < 0) first += kAStages;
        for (int kb = first; kb < tl.nkb; kb += kAStages) {
          mbar_wait(&emptyA[gw], phase ^ 1);
          if (gather) {
            const char* src = X + kb * 128 + ch * 16;
            // rows past the segment end are not loaded: their accumulator rows
            // are never stored, and fetching a placeholder token for each of
            // them would hammer one L2 line (small segments: most of the tile)
            const int nrow = min(tl.m_valid - row_off_of(tl), half_m(tl) ? 64 : 128);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int row = 4 * i + rr;
              const long long tk = __shfl_sync(0xffffffffu, tok[i >> 3], 4 * (i & 7) + rr);
              const uint32_t dst = sa + row * 128 + ((ch ^ (row & 7)) << 4);
              if (row < nrow)
                asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst),
                             "l"(src + tk * args.gather_ld), "l"(pol)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            if constexpr (PAIR && !DSB_PAIR_RELAXED)  // the leader's MMA reads this CTA's smem
              asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
            else
              fence_proxy_async();  // generic writes -> tcgen05 reads
            __syncwarp();
            if (lane == 0) {
              if constexpr (PAIR && DSB_PAIR_RELAXED)
                pair_arrive_leader_cta(&fullA[gw]);
              else
                ready_arrive(&fullA[gw]);
            }
          } else if (lane == 0) {
            load_op(sa_ptr, ma, &fullA[gw], kb * kTileK, tl.a_row + row_off_of(tl), kABytes, true);
          }
          __syncwarp();
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
    int sa = 0, sb = 0;
    uint32_t pa = 0, pb = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint64_t da0 = sdesc_sw128(smem_u32(ringA));  // + (bytes >> 4) moves the start address
    const uint64_t db0 = sdesc_sw128(smem_u32(ringB));
    int rd = 0;
    bool rend = !leader;  // the peer's MMA warp does not walk the tiles
    int id = next_id(rd, rend, true);
    GemmTile nxt = id >= 0 ? args.tiles[id] : GemmTile{};
    while (id >= 0) {
      const GemmTile tl = nxt;  // descriptor prefetched one tile ahead
      id = next_id(rd, rend, true);
      if (id >= 0) nxt = args.tiles[id];
      const uint32_t idesc = idesc_bf16(PAIR ? (half_m(tl) ? kTileM : 2 * kTileM) : kTileM, tl.n_mma);
      const uint32_t dtmem = tmem_base + acc * kAccCols;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < tl.nkb; ++kb) {
        if (PAIR && fused && !DSB_PAIR_RELAXED) {  // the peer's gathered rows are released at cluster scope
          mbar_wait_cluster(&fullA[sa], pa);
          mbar_wait(&fullB[sb], pb);
        } else {
          mbar_wait(&fullA[sa], pa);
          mbar_wait(&fullB[sb], pb);
        }
        tc_fence_after();
        const uint64_t adesc = da0 + static_cast<uint64_t>(sa * (kABytes >> 4));
        const uint64_t bdesc = db0 + static_cast<uint64_t>(sb * (kBSlot >> 4));
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kTileK / 16; ++k) {  // 16 bf16 = 32 B along K inside the 128 B swizzle row
            if constexpr (PAIR)
              umma_bf16_pair(dtmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
            else
              umma_bf16(dtmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          }
          if constexpr (PAIR) {
            umma_commit_pair(&emptyA[sa]);
            umma_commit_pair(&emptyB[sb]);
          } else {
            umma_commit(&emptyA[sa]);
            umma_commit(&emptyB[sb]);
          }
        }
        __syncwarp();
        if (++sa == kAStages) { sa = 0; pa ^= 1; }
        if (++sb == kBStages) { sb = 0; pb ^= 1; }
      }
      if (elect_one()) {
        if constexpr (PAIR)
          umma_commit_pair(&tfull[acc]);
        else
          umma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    // ---------------- epilogue warps 2..9: two per TMEM lane quarter, 32-column
    // chunks interleaved between them
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - kEpiWarp0) >> 2;
    // rows of this warp within its CTA's rows of a tile: M = 256 pair / single
    // tiles: lane quarter q holds rows [32q, 32q + 32); half-M pair tiles: 64
    // rows per CTA, quarters q and q + 2 hold the same rows (other N half)
    auto row_base = [&](const GemmTile& t) { return half_m(t) ? 32 * (q & 1) : 32 * q; };
    uint8_t* wslot = stage_buf + (warp - kEpiWarp0) * kWarpSlot;  // this warp's staging slot
    uint64_t st_pol = 0;  // A/B: output stores evict-first (H / Y must not push x / weights out of L2)
    if ((MODE == kEpiSwiGLU && (args.flags & 16)) || (MODE == kEpiScale && (args.flags & 32)))
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(st_pol));
    int acc = 0;
    uint32_t acc_phase = 0;
    // accumulator drained: MMA may reuse it (pair: one release-arrive per warp
    // on the leader's barrier)
    auto release_acc = [&](int a) {
      tc_fence_before();
      if constexpr (PAIR) {
        __syncwarp();
        if (lane == 0) {
          if constexpr (DSB_PAIR_RELAXED)
            pair_arrive_leader_cta(&tempty[a]);
          else
            pair_arrive_leader(&tempty[a]);
        }
      } else {
        mbar_arrive(&tempty[a]);
      }
    };
    int rd = 0;
    bool rend = false;
    int id = next_id(rd, rend, true);
    GemmTile nxt = id >= 0 ? args.tiles[id] : GemmTile{};
    float sc_nxt = 0.f;  // kEpiScale: this thread's row score, loaded a tile ahead
    auto load_score = [&](const GemmTile& t) {
      const int rr = row_off_of(t) + row_base(t) + lane;
      return rr < t.m_valid ? args.row_scale[t.out_row + rr] : 0.f;
    };
    if (MODE == kEpiScale && id >= 0) sc_nxt = load_score(nxt);
    while (id >= 0) {
      GemmTile tl = nxt;  // descriptor prefetched one tile ahead
      const float sc_cur = sc_nxt;
      id = next_id(rd, rend, true);
      if (id >= 0) {
        nxt = args.tiles[id];
        if (MODE == kEpiScale) sc_nxt = load_score(nxt);
      }
      const bool hm = half_m(tl);
      const int rb = row_base(tl);
      const int r = rb + lane;
      if constexpr (PAIR) {  // this CTA's rows of the pair tile
        const int ro = row_off_of(tl);
        tl.out_row += ro;
        tl.m_valid -= ro;
        const int live = (tl.m_live & 0xFFFFF) - ro;
        tl.m_live = (tl.m_live & ~0xFFFFF) | (live > 0 ? live : 0);
      }
      (void)sc_cur;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      // diagnostics only (wrong results): no epilogue, MMA-only timing of the
      // expert GEMMs (the gate keeps its epilogue so the routing is unchanged)
      if ((args.flags & 8) && MODE != kEpiF32 && MODE != kEpiF32Wide) {
        release_acc(acc);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      const uint32_t taddr = tmem_base + acc * kAccCols + (static_cast<uint32_t>(q * 32) << 16);
      const bool valid = r < tl.m_valid;
      const long long orow = static_cast<long long>(tl.out_row + r);
      // this warp's 32 rows: all inside the segment -> TMA stores; cut by the
      // segment end -> masked copy
      const bool rows_full = rb + 32 <= tl.m_valid;
      if constexpr (MODE == kEpiSwiGLU) {
        // h = swish(g) * u; a 32-neuron group = 64 accumulator columns [g | u].
        // M = 256 / single: groups 2 half, 2 half + 1 at TMEM columns 128 half
        // + 64 gi.  Half-M: lane half q >> 1 holds groups [(q >> 1) G, +G),
        // G = N / 128, at TMEM columns 64 j; this warp takes j = half.
        const int nc = tl.n_mma >> 1;
        const bool live = r < (tl.m_live & 0xFFFFF);
        const int c0 = 64 * half;
        if (kStageOut && kBoxCols == 64 && c0 < nc) warp_slot_acquire(lane);
#pragma unroll
        for (int gi = 0; gi < 2; ++gi) {
          if (hm && gi == 1) break;
          const int tcol = hm ? 64 * half : 2 * c0 + 64 * gi;
          const int ocol = hm ? (64 * half < (tl.n_mma >> 1) ? 32 * ((q >> 1) * (tl.n_mma >> 7) + half) : nc)
                              : c0 + 32 * gi;
          if (ocol >= nc) continue;
          if (kStageOut && kBoxCols == 32) warp_slot_acquire(lane);
          uint32_t v[64];  // [g of 32 neurons | u of the same 32]
          tmem_ld64(taddr + tcol, v);
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
          if (kStageOut && kBoxCols == 32) {
            warp_put(wslot, lane, 0, pk);
            warp_store(wslot, &mapO, args, tl.out_row + rb, tl.out_col + ocol, tl.m_valid - rb, rows_full, lane, st_pol);
          } else if (kStageOut)
            warp_put(wslot, lane, 32 * gi, pk);
          else if (valid)
            row_put(args, orow, tl.out_col + ocol, pk);
        }
        release_acc(acc);
        if (kStageOut && kBoxCols == 64 && c0 < nc)
          warp_store(wslot, &mapO, args, tl.out_row + rb, tl.out_col + c0, tl.m_valid - rb, rows_full, lane, st_pol);
      } else if constexpr (MODE == kEpiScale) {
        // y = acc * raw score -> bf16, 64 output columns per x64 TMEM load.
        // M = 256 / single: columns 128 p + 64 half (p = 0, 1) at the same
        // TMEM column.  Half-M: column (q >> 1) N/2 + 64 half at TMEM column
        // 64 half (when 64 half < N/2).  The row's score was loaded a tile ahead.
        const float sc = valid ? sc_cur : 0.f;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const bool last = hm || p == 1;
          const int c = hm ? (q >> 1) * (tl.n_mma >> 1) + 64 * half : 128 * p + 64 * half;
          const int tcol = hm ? 64 * half : c;
          const bool have = hm ? 64 * half < (tl.n_mma >> 1) : c < tl.n_mma;
          uint32_t pk[32];
          if (have) {
            uint32_t v[64];
            tmem_ld64(taddr + tcol, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i)
              pk[i] = pack_bf16x2(__uint_as_float(v[2 * i]) * sc, __uint_as_float(v[2 * i + 1]) * sc);
          }
          if (last) release_acc(acc);
          if (have && kStageOut && kBoxCols == 64) {
            warp_slot_acquire(lane);
            warp_put(wslot, lane, 0, pk);
            warp_put(wslot, lane, 32, pk + 16);
            warp_store(wslot, &mapO, args, tl.out_row + rb, tl.out_col + c, tl.m_valid - rb, rows_full, lane, st_pol);
          } else if (have && kStageOut) {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              warp_slot_acquire(lane);
              warp_put(wslot, lane, 0, pk + 16 * hh);
              warp_store(wslot, &mapO, args, tl.out_row + rb, tl.out_col + c + 32 * hh, tl.m_valid - rb, rows_full,
                         lane, st_pol);
            }
          } else if (have && valid) {
            row_put(args, orow, tl.out_col + c, pk);
            row_put(args, orow, tl.out_col + c + 32, pk + 16);
          }
          if (last) break;
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
      if constexpr (MODE == kEpiF32 || MODE == kEpiF32Wide) release_acc(acc);
      (void)valid; (void)orow;
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  if (warp >= kEpiWarp0 && lane == 0) bulk_wait0();  // this lane's TMA stores still read its staging slot
  if (DSB_GEMM_TIMES && PAIR && threadIdx.x == 0 && MODE >= 1 && MODE <= 2) {
    unsigned long long* g = g_gemm_times[MODE];
    const unsigned long long t_end = gemm_now();
    atomicMin(&g[0], t_entry); atomicMax(&g[1], t_entry);
    atomicMin(&g[2], t_wait); atomicMax(&g[3], t_wait);
    atomicMin(&g[4], t_end); atomicMax(&g[5], t_end);
    __threadfence();
    if (atomicAdd(&g[6], 1ull) == gridDim.x - 1) {
      __threadfence();
      const unsigned long long e0 = atomicAdd(&g[0], 0ull);
      if (e0 != 0ull)
        printf("gemm%d: entry spread %llu, wait at +%llu..+%llu, end at +%llu..+%llu ns (from first entry) abs %llu %llu\n",
               MODE, atomicAdd(&g[1], 0ull) - e0, atomicAdd(&g[2], 0ull) - e0, atomicAdd(&g[3], 0ull) - e0,
               atomicAdd(&g[4], 0ull) - e0, atomicAdd(&g[5], 0ull) - e0, e0, atomicAdd(&g[5], 0ull));
      g[0] = g[2] = g[4] = ~0ull;
      g[1] = g[3] = g[5] = 0ull;
      g[6] = 0ull;
    }
  }
  tc_fence_before();
  if constexpr (PAIR) {
    pair_sync();  // the leader's MMAs read the peer's smem until its last commit
    if (warp == kMmaWarp) tmem_dealloc_pair(tmem_base, 2 * kAccCols);
  } else {
    __syncthreads();
    if (warp == kMmaWarp) tmem_dealloc(tmem_base, 2 * kAccCols);
  }
}

// ------------------------------------------------------------------ launcher
int launch_gemm_tc(int mode, const CUtensorMap* mapA, const CUtensorMap* mapA2,
                   const CUtensorMap* mapB, const GemmTile* tiles, const int* num_tiles,
                   int max_tiles, void* out, long long ldo, const float* row_scale,
                   int b_box_rows, int num_sms, cudaStream_t stream, const int* row_token,
                   const void* gather_src, long long gather_ld, const CUtensorMap* mapO, int pair,
                   unsigned long long* zero4, int* sched) {
  static const int flags = [] {
    const char* v = std::getenv("DSMOE_B200_GEMM_FLAGS");
    return v ? std::atoi(v) : 0;
  }();
  GemmArgs a{tiles, num_tiles, out, ldo, row_scale, static_cast<uint32_t>(b_box_rows * 128), row_token,
             gather_src, gather_ld, flags, mapO != nullptr && mode != kEpiF32 && mode != kEpiF32Wide && !(flags & 2) ? 1 : 0,
             zero4, pair ? sched : nullptr};
  // gate logits with more than 64 output columns need the wide B slots
  if (mode == kEpiF32 && b_box_rows > 64) mode = kEpiF32Wide;
  const CUtensorMap* mo = mapO ? mapO : mapB;
  const int grid = max_tiles < num_sms ? (max_tiles > 0 ? max_tiles : 1) : num_sms;
  cudaError_t err;
  if (pair) {  // 2-CTA clusters, one M = 256 tile per pair
    if (mode != kEpiSwiGLU && mode != kEpiScale) return -1;
    int clusters = num_sms / 2;
    if (max_tiles < clusters) clusters = max_tiles > 0 ? max_tiles : 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * clusters);
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
#define DSB_LAUNCH_PAIR(M)                                                                         \
  {                                                                                                \
    set_max_dyn_smem(gemm_tc_kernel<M, true>, Geo<M, true>::SMEM);                                 \
    cfg.blockDim = dim3(Geo<M, true>::THREADS);                                                    \
    cfg.dynamicSmemBytes = Geo<M, true>::SMEM;                                                     \
    err = cudaLaunchKernelEx(&cfg, gemm_tc_kernel<M, true>, *mapA, *mapA2, *mapB, *mo, a);         \
  }
    if (mode == kEpiSwiGLU)
      DSB_LAUNCH_PAIR(kEpiSwiGLU)
    else
      DSB_LAUNCH_PAIR(kEpiScale)
#undef DSB_LAUNCH_PAIR
    if (err != cudaSuccess) return static_cast<int>(err);
    err = cudaGetLastError();
    return err == cudaSuccess ? 0 : static_cast<int>(err);
  }
  switch (mode) {
#define DSB_LAUNCH(M)                                                                         \
  case M: {                                                                                   \
    set_max_dyn_smem(gemm_tc_kernel<M, false>, Geo<M>::SMEM);                                 \
    err = launch_pdl(gemm_tc_kernel<M, false>, dim3(grid), dim3(Geo<M>::THREADS), Geo<M>::SMEM, stream, *mapA, \
                     *mapA2, *mapB, *mo, a);                                                  \
    if (err != cudaSuccess) return static_cast<int>(err);                                      \
    break;                                                                                    \
  }
    DSB_LAUNCH(kEpiF32)
    DSB_LAUNCH(kEpiF32Wide)
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
