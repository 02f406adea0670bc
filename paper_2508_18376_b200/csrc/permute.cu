// K2 (permute + gather), the device-side tile planner, and K5 (combine).
//
// The reference has no token permutation: moe_forward walks tokens and their
// kept selections one at a time (/root/reference/proj/include/dsmoe/moe.hpp:253-269).
// On B200 the kept (token, selection) pairs are grouped per expert unit so the
// expert FFN runs as a grouped GEMM.  Canonical row order:
// units ascending; inside a unit the rows evaluated on every sub-block ("full")
// first, then the major-only rows; each list in ascending (token, slot) order.
// The order is a pure function of the routing, so it is deterministic and is
// checked bit-for-bit against a CPU counting sort in tests/.
#include "kernels.h"

namespace dsb {

// --------------------------------------------------------------------------
// permute: grid (num_units, 2).  Block (u, 0) places the full rows of unit u,
// block (u, 1) its major-only rows.  Ordered compaction with warp ballots.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) permute_kernel(const int32_t* __restrict__ sel_code,
                                                       const float* __restrict__ sel_raw,
                                                       const int* __restrict__ cnt, int TK, int K,
                                                       int num_units, int32_t* __restrict__ row_token,
                                                       float* __restrict__ row_scale,
                                                       int32_t* __restrict__ slot_pos,
                                                       UnitSeg* __restrict__ seg, int* __restrict__ r_total) {
  const int u = blockIdx.x;
  const int lvl = blockIdx.y == 0 ? 2 : 1;
  __shared__ int s_warp[32];
  __shared__ int s_start;
  // start of unit u = sum of the counts of units < u
  int part = 0;
  for (int i = threadIdx.x; i < u; i += blockDim.x) part += cnt[2 * i] + cnt[2 * i + 1];
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (lane == 0) s_warp[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < nwarps; ++w) s += s_warp[w];
    s_start = s;
  }
  __syncthreads();
  const int start = s_start;
  const int n_full = cnt[2 * u], n_maj = cnt[2 * u + 1];
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    seg[u] = UnitSeg{start, n_full, n_full + n_maj, 0};
    if (u == num_units - 1) *r_total = start + n_full + n_maj;
  }
  const int base = start + (lvl == 2 ? 0 : n_full);
  const int target = u * 4 + lvl;
  int running = 0;
  for (int i0 = 0; i0 < TK; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const bool m = i < TK && sel_code[i] == target;
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    __syncthreads();  // s_warp reuse
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    int woff = 0, tot = 0;
    for (int w = 0; w < nwarps; ++w) {
      const int c = s_warp[w];
      woff += w < warp ? c : 0;
      tot += c;
    }
    if (m) {
      const int pos = base + running + woff + __popc(bal & ((1u << lane) - 1u));
      row_token[pos] = i / K;
      row_scale[pos] = sel_raw[i];
      slot_pos[i] = pos;
    }
    running += tot;
  }
}

int launch_permute(const int32_t* sel_code, const float* sel_raw, const int* cnt, int T, int K,
                   int num_units, int32_t* row_token, float* row_scale, int32_t* slot_pos,
                   UnitSeg* seg, int* r_total, cudaStream_t stream) {
  dim3 grid(num_units, 2);
  permute_kernel<<<grid, 1024, 0, stream>>>(sel_code, sel_raw, cnt, T * K, K, num_units, row_token,
                                            row_scale, slot_pos, seg, r_total);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// plan_tiles: one block turns the unit segments into the GEMM1 ([W1|W3] +
// SwiGLU) and GEMM2 (W2 + raw-score scale) work lists.  Minor sub-blocks get
// tiles only for the full rows, so FLOPs fall with the drop rate (no masks).
// --------------------------------------------------------------------------
__device__ __forceinline__ UnitSeg plan_seg(const PlanArgs& a, int u) {
  if (u < a.num_routed) return a.seg_routed[u];
  const int s = u - a.num_routed;
  return UnitSeg{a.shared_row0 + s * a.T, a.T, a.T, 0};
}

__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

__global__ void __launch_bounds__(1024) plan_tiles_kernel(const PlanArgs a) {
  __shared__ int s1[1024], s2[1024];
  __shared__ int carry1, carry2;
  if (threadIdx.x == 0) { carry1 = 0; carry2 = 0; }
  const int nu = a.num_routed + a.num_shared;
  const int ntd = cdiv(a.d, kTileN2);
  for (int u0 = 0; u0 < nu; u0 += blockDim.x) {
    const int u = u0 + threadIdx.x;
    int c1 = 0, c2 = 0;
    UnitSeg sg{0, 0, 0, 0};
    UnitInfo ui{};
    if (u < nu) {
      ui = a.units[u];
      sg = plan_seg(a, u);
      const int mt_all = cdiv(sg.n_tot, kTileM), mt_full = cdiv(sg.n_full, kTileM);
      for (int p = 0; p < ui.nsub; ++p) c1 += cdiv(ui.sub_wpad[p], kChunk) * (p == 0 ? mt_all : mt_full);
      c2 = mt_all * ntd;
    }
    __syncthreads();
    s1[threadIdx.x] = c1;
    s2[threadIdx.x] = c2;
    __syncthreads();
    // inclusive Hillis-Steele scan
    for (int o = 1; o < blockDim.x; o <<= 1) {
      const int v1 = threadIdx.x >= o ? s1[threadIdx.x - o] : 0;
      const int v2 = threadIdx.x >= o ? s2[threadIdx.x - o] : 0;
      __syncthreads();
      s1[threadIdx.x] += v1;
      s2[threadIdx.x] += v2;
      __syncthreads();
    }
    const int off1 = carry1 + s1[threadIdx.x] - c1;
    const int off2 = carry2 + s2[threadIdx.x] - c2;
    if (u < nu) {
      const bool sh = ui.shared != 0;
      const int mt_all = cdiv(sg.n_tot, kTileM), mt_full = cdiv(sg.n_full, kTileM);
      int k1 = off1;
      for (int mt = 0; mt < mt_all; ++mt) {
        const int m_valid = min(kTileM, sg.n_tot - mt * kTileM);
        int wrow = ui.w13_row, hcol = 0;
        for (int p = 0; p < ui.nsub; ++p) {
          const int wp = ui.sub_wpad[p];
          if (p == 0 || mt < mt_full) {
            const int live = p == 0 ? m_valid : max(0, min(kTileM, sg.n_full - mt * kTileM));
            for (int c = 0; c < cdiv(wp, kChunk); ++c) {
              const int nc = min(kChunk, wp - c * kChunk);
              GemmTile tl;
              tl.a_row = sh ? mt * kTileM : sg.start + mt * kTileM;
              tl.b_row = wrow + 2 * kChunk * c;
              tl.out_row = sg.start + mt * kTileM;
              tl.out_col = hcol + kChunk * c;
              tl.nkb = a.d / kTileK;
              tl.n_mma = 2 * nc;
              tl.m_valid = m_valid;
              tl.m_live = live | (sh ? kTileAltA : 0);
              a.tiles1[k1++] = tl;
            }
          }
          wrow += 2 * wp;
          hcol += wp;
        }
      }
      int k2 = off2;
      for (int mt = 0; mt < mt_all; ++mt) {
        const int m_valid = min(kTileM, sg.n_tot - mt * kTileM);
        const int kw = (mt * kTileM < sg.n_full) ? ui.hwidth : ui.sub_wpad[0];
        for (int nt = 0; nt < ntd; ++nt) {
          GemmTile tl;
          tl.a_row = sg.start + mt * kTileM;
          tl.b_row = ui.w2t_row + nt * kTileN2;
          tl.out_row = sg.start + mt * kTileM;
          tl.out_col = nt * kTileN2;
          tl.nkb = kw / kTileK;
          tl.n_mma = min(kTileN2, a.d - nt * kTileN2);
          tl.m_valid = m_valid;
          tl.m_live = m_valid;
          a.tiles2[k2++] = tl;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry1 += s1[threadIdx.x];
      carry2 += s2[threadIdx.x];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *a.n1 = carry1;
    *a.n2 = carry2;
  }
}

int launch_plan(const PlanArgs& a, cudaStream_t stream) {
  plan_tiles_kernel<<<1, 1024, 0, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
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
    for (int i = lane; i < vec_per_row; i += 32) dst[i] = __ldcs(src + i);
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
__global__ void __launch_bounds__(256) combine_kernel(const TY* __restrict__ y,
                                                      const int32_t* __restrict__ slot_pos,
                                                      TO* __restrict__ out, int T, int d, int K,
                                                      int S, int shared_row0) {
  constexpr int V = 16 / sizeof(TY);  // elements per 16-byte vector
  const int nvec = d / V;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      float acc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = 0.f;
      auto add_row = [&](long long row) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(y + row * d) + v);
        const TY* e = reinterpret_cast<const TY*>(&q);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += static_cast<float>(e[i]);
      };
      for (int s = 0; s < K; ++s) {
        const int p = slot_pos[static_cast<long long>(t) * K + s];
        if (p >= 0) add_row(p);
      }
      for (int s = 0; s < S; ++s) add_row(static_cast<long long>(shared_row0) + static_cast<long long>(s) * T + t);
      TO* o = out + static_cast<long long>(t) * d + static_cast<long long>(v) * V;
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = static_cast<TO>(acc[i]);
    }
  }
}

int launch_combine(const void* y, int y_bf16, const int32_t* slot_pos, void* out, int T, int d, int K,
                   int S, int shared_row0, int num_sms, cudaStream_t stream) {
  const int grid = T < num_sms * 16 ? (T > 0 ? T : 1) : num_sms * 16;
  if (y_bf16)
    combine_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(y), slot_pos, static_cast<__nv_bfloat16*>(out), T, d, K, S,
        shared_row0);
  else
    combine_kernel<float, float><<<grid, 256, 0, stream>>>(static_cast<const float*>(y), slot_pos,
                                                           static_cast<float*>(out), T, d, K, S,
                                                           shared_row0);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
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
