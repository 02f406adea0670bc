// K2 (scan + scatter + gather), the device-side tile planner, and K5 (combine).
//
// The reference has no token permutation: moe_forward walks tokens and their
// kept selections one at a time (/root/reference/proj/include/dsmoe/moe.hpp:253-269).
// On B200 the kept (token, selection) pairs are grouped per expert unit so the
// expert FFN runs as a grouped GEMM.  Canonical row order:
// units ascending; inside a unit the rows evaluated on every sub-block ("full")
// first, then the major-only rows; each list in ascending (token, slot) order.
// The order is a pure function of the routing (deterministic), checked
// bit-for-bit against a CPU counting sort in tests/.
//
//   router / import  -> per 128-token chunk histograms of (unit, level)
//   scan_plan        -> one block: exclusive scan of every code over chunks,
//                       unit segments, and the GEMM1 / GEMM2 work lists
//   scatter          -> one block per chunk: rank of each kept slot inside its
//                       chunk (warp __match_any + per-warp prefix), final row
//   gather           -> X_perm[row] = X[token(row)], 16-byte vectors
#include <cooperative_groups.h>
#include <cstdio>

#include "kernels.h"

namespace dsb {

#ifndef DSB_PERMUTE_PHASES
#define DSB_PERMUTE_PHASES 0  // 1: blocks 0, 73, last print the phase durations (diagnostic builds only)
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__shared__ unsigned long long s_tq[3];  // diagnostic builds: plan sub-phase timestamps
__device__ inline bool phase_block() {
  return DSB_PERMUTE_PHASES && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 73 || blockIdx.x == gridDim.x - 1);
}

__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

// Block-wide exclusive scan of v[0..n) in shared memory, in place; returns
// the total.  Every thread of the block must call it.
__device__ int block_excl_scan(int* v, int n) {
  __shared__ int wsum[32];
  __shared__ int s_tot, s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int x = i < n ? v[i] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int ws = lane < nw ? wsum[lane] : 0;
      int wi = ws;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < nw) wsum[lane] = wi - ws;
      if (lane == 31) s_tot = wi;
    }
    __syncthreads();
    if (i < n) v[i] = s_carry + wsum[warp] + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) s_carry += s_tot;
    __syncthreads();
  }
  const int total = s_carry;
  __syncthreads();  // every thread has read s_carry before a next call resets it
  return total;
}

// --------------------------------------------------------------------------
// scan + plan (one block of 1024 threads)
// --------------------------------------------------------------------------
constexpr int kPlanMaxUnits = 2048;

// Work lists.  GEMM1 tiles of a unit: m-tile major; for m-tiles holding full
// rows every sub-block's chunks, afterwards only sub-block 0's.  GEMM2 tiles:
// m-tile major, then d_model tiles.  Minor sub-blocks get tiles only for the
// full rows, so FLOPs fall with the drop rate (no masks).
// su: room for the units' descriptors in shared memory (staged here), or
// null; su_ready: the caller staged them already (before its griddepcontrol.wait)
// pcta / npcta: this block's index among the npcta blocks that build the
// lists (default: every block of the grid)
__device__ void plan_body(const PlanArgs& a, const UnitSeg* seg, int* off1, int* off2, UnitInfo* su = nullptr,
                          bool su_ready = false, int pcta = -1, int npcta = 0) {
  if (npcta <= 0) {
    pcta = blockIdx.x;
    npcta = gridDim.x;
  }
  const int nu = a.num_routed + a.num_shared;
  const int tm = a.tile_m ? a.tile_m : kTileM;     // GEMM1 rows per tile: 128 (single CTA) or 256 (CTA pair)
  const int tm2 = a.tile_m2 ? a.tile_m2 : tm;      // GEMM2 rows per tile
  const int ntd = cdiv(a.d, kTileN2);
  const bool unified = tm2 <= tm && tm % tm2 == 0;
  auto unit_of = [&](int u) { return u < a.num_routed ? (a.seg_unit ? a.seg_unit[u] : u) : a.shared_unit0 + (u - a.num_routed); };
  auto seg_of = [&](int u) {
    if (u < a.num_routed) return seg[u];
    const int s = u - a.num_routed;
    return UnitSeg{a.shared_row0 + s * a.T, a.T, a.T, 0};
  };
  auto unit_info = [&](int u) -> const UnitInfo& { return su ? su[u] : a.units[unit_of(u)]; };
  // tiles of one unit in each work list
  auto unit_tiles = [&](const UnitInfo& ui, const UnitSeg& sg, int& c1, int& c2) {
    const int mt_all = cdiv(sg.n_tot, tm), mt_full = cdiv(sg.n_full, tm);
    c1 = 0;
    for (int p = 0; p < ui.nsub; ++p) c1 += cdiv(ui.sub_wpad[p], kChunk) * (p == 0 ? mt_all : mt_full);
    // GEMM2 (unified, tm2 <= tm): tiles over all rows; a tile holding any
    // full row runs K = full width — its major-only rows read minor-sub-block H
    // that GEMM1's straddling minor tile wrote as zeros (rows in [live,
    // m_valid) of a GEMM1 tile store 0, and GEMM1 tiles of tm rows contain the
    // GEMM2 tile).  Otherwise the full rows and the major-only rows tile
    // separately (two tails per unit instead of one).
    c2 = (unified ? cdiv(sg.n_tot, tm2) : cdiv(sg.n_full, tm2) + cdiv(sg.n_tot - sg.n_full, tm2)) * ntd;
  };
  if (nu <= 64) {
    // one warp: descriptors staged (when there is room), tile counts and both
    // exclusive scans in registers — no block-wide scan barriers
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      int c1[2] = {0, 0}, c2[2] = {0, 0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = lane + 32 * h;
        if (u < nu) {
          const UnitInfo ui = su_ready ? su[u] : a.units[unit_of(u)];
          if (su && !su_ready) su[u] = ui;
          unit_tiles(ui, seg_of(u), c1[h], c2[h]);
        }
      }
      int i1[2] = {c1[0], c1[1]}, i2[2] = {c2[0], c2[1]};
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int y1 = __shfl_up_sync(0xffffffffu, i1[h], o), y2 = __shfl_up_sync(0xffffffffu, i2[h], o);
          if (lane >= o) {
            i1[h] += y1;
            i2[h] += y2;
          }
        }
      }
      const int a1 = __shfl_sync(0xffffffffu, i1[0], 31), a2 = __shfl_sync(0xffffffffu, i2[0], 31);
      const int b1 = __shfl_sync(0xffffffffu, i1[1], 31), b2 = __shfl_sync(0xffffffffu, i2[1], 31);
      if (lane < nu) {
        off1[lane] = i1[0] - c1[0];
        off2[lane] = i2[0] - c2[0];
      }
      if (lane + 32 < nu) {
        off1[lane + 32] = a1 + i1[1] - c1[1];
        off2[lane + 32] = a2 + i2[1] - c2[1];
      }
      if (lane == 0) {
        off1[nu] = a1 + b1;
        off2[nu] = a2 + b2;
        if (a.n1 && pcta == 0) *a.n1 = a1 + b1;
        if (a.n2 && pcta == 0) *a.n2 = a2 + b2;
      }
    }
    __syncthreads();
  } else {
    // the units' descriptors staged in shared memory when the caller provides
    // room: the tile builders below read them many times in dependent order
    if (su && !su_ready) {
      for (int u = threadIdx.x; u < nu; u += blockDim.x) su[u] = a.units[unit_of(u)];
      __syncthreads();
    }
    // tile counts per unit, then block-wide exclusive scans
    for (int u = threadIdx.x; u < nu; u += blockDim.x) unit_tiles(unit_info(u), seg_of(u), off1[u], off2[u]);
    __syncthreads();
    const int tot1 = block_excl_scan(off1, nu);
    const int tot2 = block_excl_scan(off2, nu);
    if (threadIdx.x == 0) {
      off1[nu] = tot1;
      off2[nu] = tot2;
      if (a.n1 && pcta == 0) *a.n1 = tot1;
      if (a.n2 && pcta == 0) *a.n2 = tot2;
    }
    __syncthreads();
  }
  unsigned long long tq0 = 0, tq1 = 0, tq2 = 0;
  if (DSB_PERMUTE_PHASES) tq0 = gtimer();
  auto find = [&](const int* off, int i) {  // largest u with off[u] <= i
    int lo = 0, hi = nu - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (off[mid] <= i) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  // tiles interleaved over the blocks (tile i -> block i % grid) so every
  // block builds a few instead of the first ones building them all
  const int gtid = threadIdx.x * npcta + pcta, gstride = npcta * blockDim.x;
  for (int i = gtid; i < off1[nu]; i += gstride) {
    const int u = find(off1, i);
    const UnitInfo& ui = unit_info(u);
    const UnitSeg sg = seg_of(u);
    const bool sh = ui.shared != 0;
    const int mt_full = cdiv(sg.n_full, tm);
    int ch_all = 0;
    for (int p = 0; p < ui.nsub; ++p) ch_all += cdiv(ui.sub_wpad[p], kChunk);
    const int ch0 = cdiv(ui.sub_wpad[0], kChunk);
    int li = i - off1[u], mt, r;
    if (li < mt_full * ch_all) {
      mt = li / ch_all;
      r = li - mt * ch_all;
    } else {
      li -= mt_full * ch_all;
      mt = mt_full + li / ch0;
      r = li - (mt - mt_full) * ch0;
    }
    int p = 0, wrow = ui.w13_row, hcol = 0;
    while (r >= cdiv(ui.sub_wpad[p], kChunk)) {
      r -= cdiv(ui.sub_wpad[p], kChunk);
      wrow += 2 * ui.sub_wpad[p];
      hcol += ui.sub_wpad[p];
      ++p;
    }
    const int c = r;
    const int nc = min(kChunk, ui.sub_wpad[p] - c * kChunk);
    const int m_valid = min(tm, sg.n_tot - mt * tm);
    const int live = p == 0 ? m_valid : max(0, min(tm, sg.n_full - mt * tm));
    GemmTile tl;
    tl.a_row = sh ? mt * tm : sg.start + mt * tm;
    tl.b_row = wrow + 2 * kChunk * c;
    tl.out_row = sg.start + mt * tm;
    tl.out_col = hcol + kChunk * c;
    tl.nkb = a.d / kTileK;
    tl.n_mma = 2 * nc;
    tl.m_valid = m_valid;
    tl.m_live = live | (sh ? kTileAltA : (a.gather ? kTileGatherA : 0));
    a.tiles1[i] = tl;
  }
  if (DSB_PERMUTE_PHASES) tq1 = gtimer();
  // GEMM2 tiles start on the other half of the block's warps: both lists are
  // built concurrently (each list has ~1 tile per thread of a few warps)
  const int gtid2 = ((threadIdx.x + (blockDim.x >> 1)) % blockDim.x) * npcta + pcta;
  for (int i = gtid2; i < off2[nu]; i += gstride) {
    const int u = find(off2, i);
    const UnitInfo& ui = unit_info(u);
    const UnitSeg sg = seg_of(u);
    const int li = i - off2[u];
    const int mt = li / ntd, nt = li - mt * ntd;
    const int mt_f = cdiv(sg.n_full, tm2);
    const bool full = mt < mt_f;
    const int row0 = (full || unified) ? mt * tm2 : sg.n_full + (mt - mt_f) * tm2;
    const int m_valid = min(tm2, ((full && !unified) ? sg.n_full : sg.n_tot) - row0);
    GemmTile tl;
    tl.a_row = sg.start + row0;
    tl.b_row = ui.w2t_row + nt * kTileN2;
    tl.out_row = sg.start + row0;
    tl.out_col = nt * kTileN2;
    tl.nkb = (full ? ui.hwidth : ui.sub_wpad[0]) / kTileK;
    tl.n_mma = min(kTileN2, a.d - nt * kTileN2);
    tl.m_valid = m_valid;
    tl.m_live = m_valid;
    a.tiles2[i] = tl;
  }
  if (DSB_PERMUTE_PHASES && threadIdx.x == 0) {
    tq2 = gtimer();
    s_tq[0] = tq0;
    s_tq[1] = tq1;
    s_tq[2] = tq2;
  }
}

// codes: c = unit * 2 + (level == 2 ? 0 : 1).  chunk_off[chunk][c] = rows of
// code c in earlier chunks.  One block per code: every chunk count loaded in
// parallel, block-wide exclusive scan, total per code.
__global__ void __launch_bounds__(512) scan_codes_kernel(const int* __restrict__ cnt_chunk, int nchunks, int ncode,
                                                         int* __restrict__ chunk_off, int* __restrict__ code_tot) {
  __shared__ int warp_sum[16];
  __shared__ int carry;
  const int c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int ch0 = 0; ch0 < nchunks; ch0 += blockDim.x) {
    const int ch = ch0 + threadIdx.x;
    const int v = ch < nchunks ? cnt_chunk[static_cast<long long>(ch) * ncode + c] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) warp_sum[warp] = incl;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < warp; ++w) before += warp_sum[w];
    if (ch < nchunks) chunk_off[static_cast<long long>(ch) * ncode + c] = before + incl - v;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < nwarps; ++w) t += warp_sum[w];
      carry += t;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) code_tot[c] = carry;
}

// Unit segments from the per-code totals (every block, in shared memory;
// block 0 publishes them), then optionally the GEMM work lists.
__global__ void __launch_bounds__(1024) seg_plan_kernel(const int* __restrict__ code_tot, int E,
                                                        UnitSeg* __restrict__ seg, int* __restrict__ code_base,
                                                        int* __restrict__ r_total, const PlanArgs a, int do_plan) {
  __shared__ int off1[kPlanMaxUnits + 1], off2[kPlanMaxUnits + 1];
  __shared__ UnitSeg s_seg[256];
  __shared__ int s_rows[256];
  // unit segments: rows of unit u start after all rows of units < u
  for (int u = threadIdx.x; u < E; u += blockDim.x) s_rows[u] = code_tot[2 * u] + code_tot[2 * u + 1];
  __syncthreads();
  const int rtot = block_excl_scan(s_rows, E);
  for (int u = threadIdx.x; u < E; u += blockDim.x) {
    const int nf = code_tot[2 * u], nm = code_tot[2 * u + 1];
    s_seg[u] = UnitSeg{s_rows[u], nf, nf + nm, 0};
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *r_total = rtot;
  __syncthreads();
  if (blockIdx.x == 0)
    for (int u = threadIdx.x; u < E; u += blockDim.x) {
      seg[u] = s_seg[u];
      code_base[2 * u] = s_seg[u].start;
      code_base[2 * u + 1] = s_seg[u].start + s_seg[u].n_full;
    }
  if (do_plan) plan_body(a, s_seg, off1, off2);
}

int launch_scan_plan(const int* cnt_chunk, int nchunks, int E, int* chunk_off, int* code_base, UnitSeg* seg,
                     int* r_total, int* code_tot, const PlanArgs* plan, int num_sms, cudaStream_t stream) {
  if (E > 256) return -1;
  PlanArgs a{};
  if (plan) a = *plan;
  scan_codes_kernel<<<2 * E, 512, 0, stream>>>(cnt_chunk, nchunks, 2 * E, chunk_off, code_tot);
  seg_plan_kernel<<<plan ? num_sms : 1, 1024, 0, stream>>>(code_tot, E, seg, code_base, r_total, a, plan != nullptr);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// plan only, over caller segments (expert-parallel receive side)
__global__ void __launch_bounds__(1024) plan_kernel(const PlanArgs a) {
  __shared__ int off1[kPlanMaxUnits + 1], off2[kPlanMaxUnits + 1];
  plan_body(a, a.seg_routed, off1, off2);
}

int launch_plan(const PlanArgs& a, int num_sms, cudaStream_t stream) {
  if (a.num_routed + a.num_shared > kPlanMaxUnits) return -1;
  plan_kernel<<<num_sms, 1024, 0, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// scatter: one block per 128-token chunk, slots processed in passes of
// blockDim in slot order; rank = chunk offset + earlier passes + earlier warps
// + earlier lanes with the same code.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) scatter_kernel(const int32_t* __restrict__ sel_code,
                                                       const float* __restrict__ sel_raw, int T, int K, int E,
                                                       const int* __restrict__ chunk_off,
                                                       const int* __restrict__ code_base,
                                                       int32_t* __restrict__ row_token, float* __restrict__ row_scale,
                                                       int32_t* __restrict__ slot_pos) {
  extern __shared__ int sm[];
  const int ncode = 2 * E;
  const int nwarps = blockDim.x >> 5;
  int* carry = sm;                 // ncode: rows placed by earlier passes
  int* wcnt = sm + ncode;          // nwarps x ncode
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int chunk = blockIdx.x;
  for (int c = threadIdx.x; c < ncode; c += blockDim.x)
    carry[c] = chunk_off[static_cast<long long>(chunk) * ncode + c] + code_base[c];
  const long long s0 = static_cast<long long>(chunk) * kRouterChunk * K;
  const long long s1 = min(static_cast<long long>(T) * K, s0 + static_cast<long long>(kRouterChunk) * K);
  for (long long p0 = s0; p0 < s1; p0 += blockDim.x) {
    for (int i = threadIdx.x; i < nwarps * ncode; i += blockDim.x) wcnt[i] = 0;
    __syncthreads();
    const long long i = p0 + threadIdx.x;
    const int code = i < s1 ? sel_code[i] : -1;
    const int c = code < 0 ? -1 : (code >> 2) * 2 + ((code & 3) == 2 ? 0 : 1);
    const unsigned grp = __match_any_sync(0xffffffffu, c);
    const int rank_w = __popc(grp & ((1u << lane) - 1u));
    if (c >= 0 && rank_w == 0) wcnt[warp * ncode + c] = __popc(grp);
    __syncthreads();
    // exclusive prefix over warps, per code (in place), then advance carry
    for (int cc = threadIdx.x; cc < ncode; cc += blockDim.x) {
      int run = carry[cc];
      for (int w = 0; w < nwarps; ++w) {
        const int v = wcnt[w * ncode + cc];
        wcnt[w * ncode + cc] = run;
        run += v;
      }
      carry[cc] = run;
    }
    __syncthreads();
    if (i < s1) {
      if (c >= 0) {
        const int pos = wcnt[warp * ncode + c] + rank_w;
        row_token[pos] = static_cast<int32_t>(i / K);
        row_scale[pos] = sel_raw[i];
        slot_pos[i] = pos;
      } else {
        slot_pos[i] = -1;
      }
    }
    __syncthreads();
  }
}

int launch_scatter(const int32_t* sel_code, const float* sel_raw, int T, int K, int E, const int* chunk_off,
                   const int* code_base, int32_t* row_token, float* row_scale, int32_t* slot_pos, cudaStream_t stream) {
  const int nchunks = (T + kRouterChunk - 1) / kRouterChunk;
  const int threads = 1024;
  const size_t smem = static_cast<size_t>(2 * E) * (1 + threads / 32) * sizeof(int);
  if (set_max_dyn_smem(scatter_kernel, smem) != cudaSuccess) return -2;
  if (nchunks > 0)
    scatter_kernel<<<nchunks, threads, smem, stream>>>(sel_code, sel_raw, T, K, E, chunk_off, code_base, row_token,
                                                       row_scale, slot_pos);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// Fused permutation: scan_codes + seg_plan + scatter in ONE cooperative launch
// (one CTA per SM, grid-wide barrier between the phases):
//   A  exclusive scan of every (unit, level) code over the 32-token chunks
//      -> chunk offsets + per-code totals;
//   -- grid sync --
//   B  every CTA derives the unit segments from the totals in shared memory
//      (CTA 0 publishes them), scatters its share of the chunks (ordered
//      ranks, the scatter_kernel algorithm) and builds its share of the GEMM
//      work lists (plan_body).
// Saves two launches and the kernel boundaries between three latency-bound
// kernels; results are identical to the three-kernel path.
// --------------------------------------------------------------------------
struct PermuteArgs {
  const int* cnt_chunk;
  int nchunks, E;
  int* chunk_off;
  int* code_tot;
  int* code_base;
  UnitSeg* seg;
  int* r_total;
  const int32_t* sel_code;
  const float* sel_raw;
  int T, K;
  int32_t* row_token;
  float* row_scale;
  int32_t* slot_pos;
  PlanArgs plan;
  int do_plan;
  const int* sc;                          // superchunk histograms (gate_route), or null: phase A
  int sc_chunks;
  const unsigned long long* sc_epoch;
};

// dynamic shared memory of permute_fused_kernel, in ints: [2E bases | 4 x (2E
// carry | 8 x 2E warp counts)], then the units' descriptors (plan), then the
// superchunk prefixes (sc path, kScCap x kScCodes)
constexpr int kScLd = kScCodes + 1;  // shared-memory row stride of the superchunk prefixes
constexpr int kPlanCtasMin = 8;      // permute_sc: blocks without chunks that take the work lists alone
static_assert(kScCodes == 128, "superchunk rows are indexed with shifts");
__host__ __device__ inline int permute_smem_ints(int E) { return (2 * E * (1 + 4 * (1 + 8)) + 3) & ~3; }
__host__ __device__ inline int permute_units_ints(int nu) {
  return ((nu * static_cast<int>(sizeof(UnitInfo)) + 15) & ~15) / 4;
}


__global__ void __launch_bounds__(1024) permute_fused_kernel(const PermuteArgs a) {
  unsigned long long tp[6];
  if (DSB_PERMUTE_PHASES) tp[0] = gtimer();
  namespace cg = cooperative_groups;
  extern __shared__ int dsm[];  // [2E bases | 4 x (2E carry | 8 x 2E warp counts)]
  __shared__ int off1[kPlanMaxUnits + 1], off2[kPlanMaxUnits + 1];
  __shared__ UnitSeg s_seg[256];
  __shared__ int s_rows[256];
  __shared__ int warp_sum[32];
  __shared__ int s_carry;
  const int ncode = 2 * a.E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  pdl_wait();
  pdl_trigger();
  if (DSB_PERMUTE_PHASES) tp[1] = gtimer();
  // ---- phase A: per-code exclusive scans over chunks (scan_codes_kernel)
  for (int c = blockIdx.x; c < ncode; c += gridDim.x) {
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int ch0 = 0; ch0 < a.nchunks; ch0 += blockDim.x) {
      const int ch = ch0 + threadIdx.x;
      const int v = ch < a.nchunks ? a.cnt_chunk[static_cast<long long>(ch) * ncode + c] : 0;
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) warp_sum[warp] = incl;
      __syncthreads();
      int before = s_carry;
      for (int w = 0; w < warp; ++w) before += warp_sum[w];
      if (ch < a.nchunks) a.chunk_off[static_cast<long long>(ch) * ncode + c] = before + incl - v;
      __syncthreads();
      if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < nwarps; ++w) t += warp_sum[w];
        s_carry += t;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) a.code_tot[c] = s_carry;
    __syncthreads();
  }
  if (DSB_PERMUTE_PHASES) tp[2] = gtimer();
  cg::this_grid().sync();
  if (DSB_PERMUTE_PHASES) tp[3] = gtimer();
  // ---- phase B1: unit segments (every CTA, in shared memory)
  for (int u = threadIdx.x; u < a.E; u += blockDim.x) s_rows[u] = a.code_tot[2 * u] + a.code_tot[2 * u + 1];
  __syncthreads();
  const int rtot = block_excl_scan(s_rows, a.E);
  int* base = dsm;
  int* carry = dsm + ncode;
  for (int u = threadIdx.x; u < a.E; u += blockDim.x) {
    const int nf = a.code_tot[2 * u], nm = a.code_tot[2 * u + 1];
    s_seg[u] = UnitSeg{s_rows[u], nf, nf + nm, 0};
    base[2 * u] = s_rows[u];
    base[2 * u + 1] = s_rows[u] + nf;
    if (blockIdx.x == 0) {
      a.seg[u] = s_seg[u];
      a.code_base[2 * u] = s_rows[u];
      a.code_base[2 * u + 1] = s_rows[u] + nf;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *a.r_total = rtot;
  __syncthreads();
  // ---- phase B2: ordered scatter (scatter_kernel's algorithm); the CTA's
  // 1024 threads work on kGroups chunks at once, 256 threads (8 warps) each
  {
    constexpr int kGroups = 4, kGW = 8;  // chunks in flight per CTA, warps per chunk
    const int grp = warp / kGW, gwarp = warp % kGW, gtid = threadIdx.x % (kGW * 32);
    int* gcarry = carry + grp * (ncode + kGW * ncode);
    int* gwcnt = gcarry + ncode;
    const long long slots_per_chunk = static_cast<long long>(kRouterChunk) * a.K;
    const int passes = static_cast<int>((slots_per_chunk + kGW * 32 - 1) / (kGW * 32));
    for (int c0 = blockIdx.x * kGroups; c0 < a.nchunks; c0 += gridDim.x * kGroups) {
      const int chunk = c0 + grp;
      const bool have = chunk < a.nchunks;
      for (int c = gtid; c < ncode; c += kGW * 32)
        gcarry[c] = have ? a.chunk_off[static_cast<long long>(chunk) * ncode + c] + base[c] : 0;
      const long long s0 = static_cast<long long>(chunk) * slots_per_chunk;
      const long long s1 = have ? min(static_cast<long long>(a.T) * a.K, s0 + slots_per_chunk) : s0;
      for (int ps = 0; ps < passes; ++ps) {
        const long long p0 = s0 + static_cast<long long>(ps) * kGW * 32;
        for (int i = gtid; i < kGW * ncode; i += kGW * 32) gwcnt[i] = 0;
        __syncthreads();
        const long long i = p0 + gtid;
        const int code = i < s1 ? a.sel_code[i] : -1;
        const int c = code < 0 ? -1 : (code >> 2) * 2 + ((code & 3) == 2 ? 0 : 1);
        const unsigned mg = __match_any_sync(0xffffffffu, c);
        const int rank_w = __popc(mg & ((1u << lane) - 1u));
        if (c >= 0 && rank_w == 0) gwcnt[gwarp * ncode + c] = __popc(mg);
        __syncthreads();
        for (int cc = gtid; cc < ncode; cc += kGW * 32) {
          int run = gcarry[cc];
          for (int w = 0; w < kGW; ++w) {
            const int v = gwcnt[w * ncode + cc];
            gwcnt[w * ncode + cc] = run;
            run += v;
          }
          gcarry[cc] = run;
        }
        __syncthreads();
        if (i < s1) {
          if (c >= 0) {
            const int pos = gwcnt[gwarp * ncode + c] + rank_w;
            a.row_token[pos] = static_cast<int32_t>(i / a.K);
            a.row_scale[pos] = a.sel_raw[i];
            a.slot_pos[i] = pos;
          } else {
            a.slot_pos[i] = -1;
          }
        }
        __syncthreads();
      }
    }
  }
  if (DSB_PERMUTE_PHASES) tp[4] = gtimer();
  // ---- phase B3: this CTA's share of the GEMM work lists
  if (a.do_plan) {
    // after the scatter's dynamic region: room for the units' descriptors
    UnitInfo* su = reinterpret_cast<UnitInfo*>(dsm + permute_smem_ints(a.E));
    plan_body(a.plan, s_seg, off1, off2, su);
  }
  if (DSB_PERMUTE_PHASES) {
    tp[5] = gtimer();
    if (phase_block())
      printf("permute block %d: wait %llu  A %llu  sync/A' %llu  B12 %llu  B3 %llu (prologue %llu tiles1 %llu tiles2 %llu) ns\n",
             blockIdx.x, tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4],
             a.do_plan ? s_tq[0] - tp[4] : 0ull, a.do_plan ? s_tq[1] - s_tq[0] : 0ull, a.do_plan ? s_tq[2] - s_tq[1] : 0ull);
  }
}

// --------------------------------------------------------------------------
// Superchunk permutation (after the fused gate + router, E <= 64): that kernel
// added every 64-token tile's histogram into its superchunk (sc_chunks chunks)
// of the buffer the device epoch selects.  Every CTA scans the <= kScCap
// superchunks itself — exclusive prefix per code and per-code totals — so the
// chunk scan and the grid-wide barrier of permute_fused_kernel disappear; a
// chunk's offset is its superchunk prefix plus the chunk rows before it in
// that superchunk.  Loads are issued early: the units' descriptors before
// griddepcontrol.wait (layer constants), the epoch, the chunk rows and the
// first scatter pass's selections together after it.  Results are identical
// to permute_fused_kernel.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) permute_sc_kernel(const PermuteArgs a) {
  unsigned long long tp[6];
  if (DSB_PERMUTE_PHASES) tp[0] = gtimer();
  extern __shared__ int dsm[];
  __shared__ int off1[kPlanMaxUnits + 1], off2[kPlanMaxUnits + 1];
  __shared__ UnitSeg s_seg[64];
  __shared__ int s_ctot[kScCodes];
  constexpr int kGroups = 4, kGW = 8;  // chunks in flight per CTA, warps per chunk
  const int ncode = 2 * a.E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int nu_plan = a.do_plan ? a.plan.num_routed + a.plan.num_shared : 0;
  UnitInfo* su = reinterpret_cast<UnitInfo*>(dsm + permute_smem_ints(a.E));
  int* scp = dsm + permute_smem_ints(a.E) + permute_units_ints(nu_plan);  // 2 x kScLd superchunk prefixes
  int* base = dsm;
  int* carry = dsm + ncode;
  // layer constants: staged while the router kernel still runs
  if (a.do_plan)
    for (int u = threadIdx.x; u < nu_plan; u += blockDim.x)
      su[u] = a.plan.units[u < a.plan.num_routed ? (a.plan.seg_unit ? a.plan.seg_unit[u] : u)
                                                  : a.plan.shared_unit0 + (u - a.plan.num_routed)];
  const int grp = warp / kGW, gwarp = warp % kGW, gtid = threadIdx.x % (kGW * 32);
  const long long slots_per_chunk = static_cast<long long>(kRouterChunk) * a.K;
  const int passes = static_cast<int>((slots_per_chunk + kGW * 32 - 1) / (kGW * 32));
  pdl_wait();
  pdl_trigger();
  if (DSB_PERMUTE_PHASES) tp[1] = gtimer();
  // ---- loads that depend only on the router's outputs, all in flight at once
  const unsigned long long ep = *reinterpret_cast<const volatile unsigned long long*>(a.sc_epoch);
  const int chunk0 = blockIdx.x * kGroups + grp;     // this group's first chunk
  const int cc = gtid & (kScCodes - 1), ch_half = gtid >> 7;
  int pre = 0;  // rows of code cc in this superchunk's chunks before chunk0 (this thread's half)
  if (chunk0 < a.nchunks && cc < ncode)
    for (int ch = (chunk0 / a.sc_chunks) * a.sc_chunks + ch_half; ch < chunk0; ch += 16) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (ch + 2 * j < chunk0) pre += a.cnt_chunk[static_cast<long long>(ch + 2 * j) * ncode + cc];
    }
  const long long i_pre = static_cast<long long>(chunk0) * slots_per_chunk + gtid;  // first pass's selection
  const long long s1_pre = min(static_cast<long long>(a.T) * a.K, static_cast<long long>(chunk0 + 1) * slots_per_chunk);
  const bool pre_ok = chunk0 < a.nchunks && i_pre < s1_pre;
  const int code_pre = pre_ok ? a.sel_code[i_pre] : -1;
  const float raw_pre = pre_ok && code_pre >= 0 ? a.sel_raw[i_pre] : 0.f;
  // ---- per-code totals over all superchunks and the prefix before this CTA's
  // superchunk (threads 0..ncode-1, one code each, every load in flight);
  // threads [512, 512 + ncode): the prefix before the superchunk of the CTA's
  // last group when its chunks straddle a superchunk boundary
  const int* buf = a.sc + static_cast<long long>((ep + 1ull) & 1ull) * kScCap * kScCodes;  // = (ep - 1) & 1
  const int nsc = cdiv(a.nchunks, a.sc_chunks);
  const int sc_first = min(blockIdx.x * kGroups, a.nchunks - 1) / a.sc_chunks;
  const int sc_last = min(blockIdx.x * kGroups + kGroups - 1, a.nchunks - 1) / a.sc_chunks;
  {
    const int c = threadIdx.x & 511;
    const int upto = threadIdx.x < 512 ? sc_first : sc_last;
    if (c < ncode && (threadIdx.x < 512 || sc_last != sc_first)) {
      int tot = 0, pfx = 0;
      for (int s0 = 0; s0 < nsc; s0 += 16) {
        int v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = s0 + j < nsc ? buf[(s0 + j) * kScCodes + c] : 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          tot += v[j];
          if (s0 + j < upto) pfx += v[j];
        }
      }
      if (threadIdx.x < 512) {
        s_ctot[c] = tot;
        scp[c] = pfx;
      } else {
        scp[kScLd + c] = pfx;
      }
    }
  }
  __syncthreads();
  if (DSB_PERMUTE_PHASES) tp[2] = tp[3] = gtimer();
  // ---- unit segments (one warp, 2 units per lane)
  if (warp == 0) {
    const int r0 = lane < a.E ? s_ctot[2 * lane] + s_ctot[2 * lane + 1] : 0;
    const int r1 = lane + 32 < a.E ? s_ctot[2 * lane + 64] + s_ctot[2 * lane + 65] : 0;
    int i0 = r0, i1 = r1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y0 = __shfl_up_sync(0xffffffffu, i0, o), y1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) {
        i0 += y0;
        i1 += y1;
      }
    }
    const int t0 = __shfl_sync(0xffffffffu, i0, 31), t1 = __shfl_sync(0xffffffffu, i1, 31);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = lane + 32 * h;
      if (u < a.E) {
        const int start = h ? t0 + i1 - r1 : i0 - r0;
        const int nf = s_ctot[2 * u], nm = s_ctot[2 * u + 1];
        s_seg[u] = UnitSeg{start, nf, nf + nm, 0};
        base[2 * u] = start;
        base[2 * u + 1] = start + nf;
        if (blockIdx.x == 0) {
          a.seg[u] = s_seg[u];
          a.code_base[2 * u] = start;
          a.code_base[2 * u + 1] = start + nf;
        }
      }
    }
    if (lane == 0 && blockIdx.x == 0) *a.r_total = t0 + t1;
  }
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < ncode; c += blockDim.x) a.code_tot[c] = s_ctot[c];
  __syncthreads();
  // ---- ordered scatter (permute_fused_kernel phase B2), chunk offsets from the prefixes
  {
    int* gcarry = carry + grp * (ncode + kGW * ncode);
    int* gwcnt = gcarry + ncode;
    bool first = true;
    for (int c0 = blockIdx.x * kGroups; c0 < a.nchunks; c0 += gridDim.x * kGroups) {
      const int chunk = c0 + grp;
      const bool have = chunk < a.nchunks;
      const int sc0 = have ? chunk / a.sc_chunks : 0;
      int v = pre;
      if (!first && have && cc < ncode) {  // later rounds (T > gridDim x kGroups chunks)
        v = 0;
        for (int ch = sc0 * a.sc_chunks + ch_half; ch < chunk; ch += 2)
          v += a.cnt_chunk[static_cast<long long>(ch) * ncode + cc];
        if (ch_half == 0)
          for (int q = 0; q < sc0; ++q) v += buf[q * kScCodes + cc];
      }
      if (ch_half == 1 && cc < ncode) gwcnt[cc] = v;  // gwcnt is free until the first pass below
      __syncthreads();
      if (ch_half == 0 && cc < ncode)
        gcarry[cc] = have ? (first ? scp[(sc0 == sc_first ? 0 : kScLd) + cc] : 0) + base[cc] + v + gwcnt[cc] : 0;
      const long long s0 = static_cast<long long>(chunk) * slots_per_chunk;
      const long long s1 = have ? min(static_cast<long long>(a.T) * a.K, s0 + slots_per_chunk) : s0;
      for (int ps = 0; ps < passes; ++ps) {
        const long long p0 = s0 + static_cast<long long>(ps) * kGW * 32;
        __syncthreads();  // gcarry written / the previous pass's gwcnt readers done
        for (int i = gtid; i < kGW * ncode; i += kGW * 32) gwcnt[i] = 0;
        __syncthreads();
        const long long i = p0 + gtid;
        const bool use_pre = first && ps == 0;
        const int code = use_pre ? code_pre : (i < s1 ? a.sel_code[i] : -1);
        const int c = code < 0 ? -1 : (code >> 2) * 2 + ((code & 3) == 2 ? 0 : 1);
        const unsigned mg = __match_any_sync(0xffffffffu, c);
        const int rank_w = __popc(mg & ((1u << lane) - 1u));
        if (c >= 0 && rank_w == 0) gwcnt[gwarp * ncode + c] = __popc(mg);
        __syncthreads();
        for (int q = gtid; q < ncode; q += kGW * 32) {
          int run = gcarry[q];
#pragma unroll
          for (int w = 0; w < kGW; ++w) {
            const int x = gwcnt[w * ncode + q];
            gwcnt[w * ncode + q] = run;
            run += x;
          }
          gcarry[q] = run;
        }
        __syncthreads();
        if (i < s1) {
          if (c >= 0) {
            const int pos = gwcnt[gwarp * ncode + c] + rank_w;
            a.row_token[pos] = static_cast<int32_t>(i / a.K);
            a.row_scale[pos] = use_pre ? raw_pre : a.sel_raw[i];
            a.slot_pos[i] = pos;
          } else {
            a.slot_pos[i] = -1;
          }
        }
      }
      first = false;
      __syncthreads();
    }
  }
  if (DSB_PERMUTE_PHASES) tp[4] = gtimer();
  // ---- GEMM work lists (descriptors already staged).  When enough blocks
  // have no chunk to scatter (T <= 18944 at 148 SMs: 20+ idle blocks at
  // T = 16384) they build the lists while the others scatter; otherwise every
  // block builds its share after its scatter.
  if (a.do_plan) {
    const int scatter_ctas = min(static_cast<int>(gridDim.x), cdiv(a.nchunks, kGroups));
    const int idle = static_cast<int>(gridDim.x) - scatter_ctas;
    if (idle >= kPlanCtasMin) {
      if (static_cast<int>(blockIdx.x) >= scatter_ctas)
        plan_body(a.plan, s_seg, off1, off2, su, true, blockIdx.x - scatter_ctas, idle);
    } else {
      plan_body(a.plan, s_seg, off1, off2, su, true);
    }
  }
  if (DSB_PERMUTE_PHASES) {
    tp[5] = gtimer();
    if (phase_block())
      printf("permute_sc block %d: wait %llu  A' %llu  B12 %llu  B3 %llu (prologue %llu tiles1 %llu tiles2 %llu) ns"
             " abs %llu %llu %llu\n",
             blockIdx.x, tp[1] - tp[0], tp[2] - tp[1], tp[4] - tp[3], tp[5] - tp[4],
             a.do_plan ? s_tq[0] - tp[4] : 0ull, a.do_plan ? s_tq[1] - s_tq[0] : 0ull,
             a.do_plan ? s_tq[2] - s_tq[1] : 0ull, tp[0], tp[1], tp[5]);
  }
}

int launch_permute_fused(const int* cnt_chunk, int nchunks, int E, int* chunk_off, int* code_base, UnitSeg* seg,
                         int* r_total, int* code_tot, const int32_t* sel_code, const float* sel_raw, int T, int K,
                         int32_t* row_token, float* row_scale, int32_t* slot_pos, const PlanArgs* plan, int num_sms,
                         cudaStream_t stream, const int* sc, const unsigned long long* sc_epoch) {
  if (E > 256) return -1;
  if (sc && (E > 64 || !sc_epoch || (nchunks + gate_route_sc_chunks(T) - 1) / gate_route_sc_chunks(T) > kScCap))
    return -1;
  PermuteArgs a{cnt_chunk, nchunks, E, chunk_off, code_tot, code_base, seg, r_total, sel_code, sel_raw, T, K,
                row_token, row_scale, slot_pos, plan ? *plan : PlanArgs{}, plan != nullptr,
                sc, sc ? gate_route_sc_chunks(T) : 0, sc_epoch};
  const int threads = 1024;
  const size_t smem =
      static_cast<size_t>(permute_smem_ints(E) + (plan ? permute_units_ints(plan->num_routed + plan->num_shared) : 0) +
                          (sc ? 2 * kScLd : 0)) *
      sizeof(int);
  auto* kern = sc ? permute_sc_kernel : permute_fused_kernel;
  if (set_max_dyn_smem(kern, smem) != cudaSuccess) return -2;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) return -3;
  const int grid = num_sms;  // one CTA per SM: every CTA is co-resident (cooperative launch checks it)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = sc ? 0 : 1;  // the superchunk path has no grid-wide barrier
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  return e == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// gather: X_perm[p] = X[row_token[p]] for p < *r_total; one warp per row,
// 16-byte vectors, streaming loads.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gather_rows_kernel(const uint4* __restrict__ x,
                                                          uint4* __restrict__ xp,
                                                          const int32_t* __restrict__ row_token,
                                                          const int* __restrict__ r_total,
                                                          int vec_per_row) {
  const int R = *r_total;
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < R; r += gridDim.x * wpb) {
    const uint4* src = x + static_cast<long long>(row_token[r]) * vec_per_row;
    uint4* dst = xp + static_cast<long long>(r) * vec_per_row;
    int i = lane;
    for (; i + 7 * 32 < vec_per_row; i += 8 * 32) {  // 8 loads in flight per lane, then 8 stores
      uint4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(src + i + 32 * j);
#pragma unroll
      for (int j = 0; j < 8; ++j) __stcs(dst + i + 32 * j, v[j]);
    }
    for (; i < vec_per_row; i += 32) __stcs(dst + i, __ldg(src + i));
  }
}

int launch_gather(const void* x, void* xp, const int32_t* row_token, const int* r_total,
                  int row_bytes, int num_sms, cudaStream_t stream) {
  gather_rows_kernel<<<num_sms * 8, 256, 0, stream>>>(static_cast<const uint4*>(x),
                                                      static_cast<uint4*>(xp), row_token, r_total,
                                                      row_bytes / 16);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// combine: out[t] = sum over kept selections s (slot order) of Y[slot_pos] +
// sum over shared experts of Y[shared_row0 + s*T + t].  Deterministic (no
// atomics).  Y rows already carry the raw-score weight (K4 epilogue).
// --------------------------------------------------------------------------
template <typename TY, typename TO>
__global__ void __launch_bounds__(256) combine_kernel(const TY* __restrict__ y, const TY* __restrict__ ysh,
                                                      const int32_t* __restrict__ slot_pos,
                                                      TO* __restrict__ out, int T, int d, int K,
                                                      int S, int shared_row0, const TY* __restrict__ resid) {
  constexpr int V = 16 / sizeof(TY);  // elements per 16-byte vector
  const int nvec = d / V;
  pdl_wait();
  pdl_trigger_tail();
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      float acc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = 0.f;
      if (resid) {  // residual stream x_{l+1} = x_l + moe(x_l) (dropping.hpp:271), fused
        const uint4 q = *(reinterpret_cast<const uint4*>(resid + static_cast<long long>(t) * d) + v);
        const TY* e = reinterpret_cast<const TY*>(&q);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = static_cast<float>(e[i]);
      }
      auto add_vec = [&](const uint4& q) {
        if constexpr (sizeof(TY) == 2) {
          // bf16 pairs -> float2 (exact: a bf16 is the top half of an fp32),
          // packed fp32x2 adds (same per-element IEEE rounding as scalar adds)
          const uint32_t* w = reinterpret_cast<const uint32_t*>(&q);
#pragma unroll
          for (int i = 0; i < V / 2; ++i) {
            const float2 f = make_float2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
            const float2 r = __fadd2_rn(make_float2(acc[2 * i], acc[2 * i + 1]), f);
            acc[2 * i] = r.x;
            acc[2 * i + 1] = r.y;
          }
        } else {
          const TY* e = reinterpret_cast<const TY*>(&q);
#pragma unroll
          for (int i = 0; i < V; ++i) acc[i] += static_cast<float>(e[i]);
        }
      };
      // every kept row's vector is requested before the first add (memory-level
      // parallelism), then summed in slot order (deterministic)
      const int32_t* sp = slot_pos + static_cast<long long>(t) * K;
      for (int s0 = 0; s0 < K; s0 += 8) {
        uint4 q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int p = s0 + j < K ? sp[s0 + j] : -1;
          q[j] = p >= 0 ? __ldcs(reinterpret_cast<const uint4*>(y + static_cast<long long>(p) * d) + v)
                        : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (s0 + j < K && sp[s0 + j] >= 0) add_vec(q[j]);
      }
      for (int s = 0; s < S; ++s)
        add_vec(__ldcs(reinterpret_cast<const uint4*>(
                           ysh + (static_cast<long long>(shared_row0) + static_cast<long long>(s) * T + t) * d) +
                       v));
      TO* o = out + static_cast<long long>(t) * d + static_cast<long long>(v) * V;
      if constexpr (sizeof(TO) == 2) {
        uint32_t pk[V / 2];
#pragma unroll
        for (int i = 0; i < V / 2; ++i) pk[i] = pack_bf16x2(acc[2 * i], acc[2 * i + 1]);
        *reinterpret_cast<uint4*>(o) = *reinterpret_cast<const uint4*>(pk);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) o[i] = static_cast<TO>(acc[i]);
      }
    }
  }
}

// y: routed rows (slot_pos); ysh: buffer holding the shared-expert rows
int launch_combine2(const void* y, const void* ysh, int y_bf16, const int32_t* slot_pos, void* out, int T, int d,
                    int K, int S, int shared_row0, int num_sms, cudaStream_t stream, const void* resid) {
  const int grid = T < num_sms * 16 ? (T > 0 ? T : 1) : num_sms * 16;
  if (y_bf16)
    launch_pdl(combine_kernel<__nv_bfloat16, __nv_bfloat16>, dim3(grid), dim3(256), 0, stream,
               static_cast<const __nv_bfloat16*>(y), static_cast<const __nv_bfloat16*>(ysh), slot_pos,
               static_cast<__nv_bfloat16*>(out), T, d, K, S, shared_row0, static_cast<const __nv_bfloat16*>(resid));
  else
    launch_pdl(combine_kernel<float, float>, dim3(grid), dim3(256), 0, stream, static_cast<const float*>(y),
               static_cast<const float*>(ysh), slot_pos, static_cast<float*>(out), T, d, K, S, shared_row0,
               static_cast<const float*>(resid));
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int launch_combine(const void* y, int y_bf16, const int32_t* slot_pos, void* out, int T, int d, int K,
                   int S, int shared_row0, int num_sms, cudaStream_t stream, const void* resid) {
  return launch_combine2(y, y, y_bf16, slot_pos, out, T, d, K, S, shared_row0, num_sms, stream, resid);
}

__global__ void fill_f32_kernel(float* p, float v, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    p[i] = v;
}

int launch_fill_f32(float* p, float v, long long n, cudaStream_t stream) {
  if (n <= 0) return 0;
  const long long b = (n + 255) / 256;
  fill_f32_kernel<<<static_cast<int>(b < 4096 ? b : 4096), 256, 0, stream>>>(p, v, n);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
