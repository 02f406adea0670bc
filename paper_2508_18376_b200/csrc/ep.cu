// Expert-parallel token exchange with one row per (token, destination rank).
//
// The reference only models EP (simulate_step, /root/reference/proj/include/
// dsmoe/ep_sim.hpp:110-160).  Moving one row per kept SELECTION (the first EP
// path) ships a token to a rank once per expert it selected there; with
// top-8 of 64 experts that is 1.5x (8 ranks) to 4x (2 ranks) more rows than
// there are (token, rank) pairs.  Here a token goes to each rank once:
//
//   ep_pack (sender, one cooperative launch)
//     phase 1  per 256-token chunk: destination mask of every token (ranks
//              owning a kept selection) and per-destination counts of
//              unique rows and of selection records;
//     phase 2  per destination: exclusive scan over chunks;
//     phase 3  ordered placement: send_token[] (destination-major, tokens
//              ascending), pos_td[t][d] (send slot of (t, d) or -1), and the
//              selection records (unit*4+level, row within the destination's
//              list, raw score) in (token, slot) order.
//   ep_local_routing (receiver): records -> the dense per-row routing codes
//              (rows x K, -1 = empty) and the 32-row chunk histograms the
//              permutation kernels consume, so the received rows run through
//              the regular forward (permute, grouped GEMMs with fused row
//              gather, combine) and come back as ONE row per (token, rank);
//   ep_final_combine (sender): out[t] = sum over destinations (ascending) of
//              the returned rows + the local shared experts.
#include <cooperative_groups.h>

#include "kernels.h"

namespace dsb {

constexpr int kPackChunk = 256;  // tokens per chunk (one thread each)
constexpr int kMaxDest = 32;

struct PackArgs {
  const int32_t* sel_code;  // T x K: unit * 4 + level, -1 dropped
  const float* sel_raw;     // T x K
  const uint32_t* dest;     // 2 x unit: destination-rank masks of a full / a major-only selection
                            // (the holders of all the unit's blocks / of its block 0)
  int T, K, N, nchunks;
  int* cnt_u;               // nchunks x N  (in place -> exclusive offsets)
  int* cnt_s;               // nchunks x N
  int* tot;                 // [N unique rows | N records | base_u N | base_s N]
  int32_t* send_token;      // U_total
  int32_t* pos_td;          // T x N
  int32_t* rec_code;        // S_total records, element stride rec_stride
  int32_t* rec_row;
  float* rec_raw;
  int* r_total;             // U_total (device scalar for the row gather)
  int rec_stride;           // 1: three separate arrays; 3: one interleaved {code, row, raw} array
  long long* counts_out;    // optional: N x {rows, records} as int64 (device), for a sync-free exchange
};

__global__ void __launch_bounds__(kPackChunk) ep_pack_kernel(const PackArgs a) {
  namespace cg = cooperative_groups;
  __shared__ int s_u[kMaxDest], s_s[kMaxDest];
  __shared__ int w_u[kPackChunk / 32][kMaxDest], w_s[kPackChunk / 32][kMaxDest];
  __shared__ int base_u[kMaxDest], base_s[kMaxDest];
  const int N = a.N, K = a.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto dest_of = [&](int c) { return a.dest[2 * (c >> 2) + ((c & 3) == 2 ? 0 : 1)]; };
  auto token_info = [&](int t, uint32_t& mask, int* cnt) {  // destinations of t, records per destination
    mask = 0u;
    for (int d = 0; d < N; ++d) cnt[d] = 0;
    if (t >= a.T) return;
    for (int s = 0; s < K; ++s) {
      const int c = a.sel_code[static_cast<long long>(t) * K + s];
      if (c < 0) continue;
      const uint32_t m = dest_of(c);
      mask |= m;
      for (int d = 0; d < N; ++d) cnt[d] += (m >> d) & 1u;
    }
  };
  // ---- phase 1: per-chunk counts
  for (int ch = blockIdx.x; ch < a.nchunks; ch += gridDim.x) {
    if (threadIdx.x < N) { s_u[threadIdx.x] = 0; s_s[threadIdx.x] = 0; }
    __syncthreads();
    uint32_t mask;
    int cnt[kMaxDest];
    token_info(ch * kPackChunk + threadIdx.x, mask, cnt);
    for (int d = 0; d < N; ++d) {
      const int u = __popc(__ballot_sync(0xffffffffu, (mask >> d) & 1u));
      int sc = cnt[d];
      for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
      if (lane == 0 && (u | sc)) { atomicAdd(&s_u[d], u); atomicAdd(&s_s[d], sc); }
    }
    __syncthreads();
    if (threadIdx.x < N) {
      a.cnt_u[ch * N + threadIdx.x] = s_u[threadIdx.x];
      a.cnt_s[ch * N + threadIdx.x] = s_s[threadIdx.x];
    }
    __syncthreads();
  }
  cg::this_grid().sync();
  // ---- phase 2: per-destination exclusive scans over chunks (one thread per
  // destination; nchunks is small: T / 256)
  if (blockIdx.x == 0 && threadIdx.x < N) {
    const int d = threadIdx.x;
    int ru = 0, rs = 0;
    for (int ch = 0; ch < a.nchunks; ++ch) {
      const int u = a.cnt_u[ch * N + d], s = a.cnt_s[ch * N + d];
      a.cnt_u[ch * N + d] = ru;
      a.cnt_s[ch * N + d] = rs;
      ru += u;
      rs += s;
    }
    a.tot[d] = ru;
    a.tot[N + d] = rs;
    if (a.counts_out) {
      a.counts_out[2 * d] = ru;
      a.counts_out[2 * d + 1] = rs;
    }
  }
  cg::this_grid().sync();
  if (threadIdx.x == 0) {
    int bu = 0, bs = 0;
    for (int d = 0; d < N; ++d) {
      base_u[d] = bu;
      base_s[d] = bs;
      bu += a.tot[d];
      bs += a.tot[N + d];
    }
    if (blockIdx.x == 0) {
      for (int d = 0; d < N; ++d) { a.tot[2 * N + d] = base_u[d]; a.tot[3 * N + d] = base_s[d]; }
      *a.r_total = bu;
    }
  }
  __syncthreads();
  // ---- phase 3: ordered placement
  for (int ch = blockIdx.x; ch < a.nchunks; ch += gridDim.x) {
    const int t = ch * kPackChunk + threadIdx.x;
    uint32_t mask;
    int cnt[kMaxDest];
    token_info(t, mask, cnt);
    int pu[kMaxDest], ps[kMaxDest];  // this token's rank among earlier tokens of the warp
    for (int d = 0; d < N; ++d) {
      const uint32_t b = __ballot_sync(0xffffffffu, (mask >> d) & 1u);
      pu[d] = __popc(b & ((1u << lane) - 1u));
      int inc = cnt[d];
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      ps[d] = inc - cnt[d];
      if (lane == 31) { w_u[warp][d] = __popc(b); w_s[warp][d] = inc; }
    }
    __syncthreads();
    if (threadIdx.x < N) {  // exclusive prefix over warps, per destination
      const int d = threadIdx.x;
      int ru = 0, rs = 0;
      for (int w = 0; w < kPackChunk / 32; ++w) {
        const int u = w_u[w][d], s = w_s[w][d];
        w_u[w][d] = ru;
        w_s[w][d] = rs;
        ru += u;
        rs += s;
      }
    }
    __syncthreads();
    if (t < a.T) {
      int rec_next[kMaxDest];
      for (int d = 0; d < N; ++d) {
        const long long q = static_cast<long long>(t) * N + d;
        if ((mask >> d) & 1u) {
          const int pos = base_u[d] + a.cnt_u[ch * N + d] + w_u[warp][d] + pu[d];
          a.send_token[pos] = t;
          a.pos_td[q] = pos;
          rec_next[d] = base_s[d] + a.cnt_s[ch * N + d] + w_s[warp][d] + ps[d];
        } else {
          a.pos_td[q] = -1;
        }
      }
      for (int s = 0; s < K; ++s) {  // records in slot order, one per destination holding a needed block
        const long long i = static_cast<long long>(t) * K + s;
        const int c = a.sel_code[i];
        if (c < 0) continue;
        for (uint32_t m = dest_of(c); m; m &= m - 1u) {
          const int d = __ffs(m) - 1;
          const long long r = static_cast<long long>(rec_next[d]++) * a.rec_stride;
          a.rec_code[r] = c;
          a.rec_row[r] = a.pos_td[static_cast<long long>(t) * N + d] - base_u[d];
          a.rec_raw[r] = a.sel_raw[i];
        }
      }
    }
    __syncthreads();
  }
}

int launch_ep_pack(const int32_t* sel_code, const float* sel_raw, const uint32_t* dest, int T, int K, int N,
                   int* cnt_u, int* cnt_s, int* tot, int32_t* send_token, int32_t* pos_td, int32_t* rec_code,
                   int32_t* rec_row, float* rec_raw, int* r_total, int num_sms, cudaStream_t stream, int rec_stride,
                   long long* counts_out) {
  if (N < 1 || N > kMaxDest || K > 16) return -1;
  PackArgs a{sel_code, sel_raw, dest, T, K, N, (T + kPackChunk - 1) / kPackChunk, cnt_u, cnt_s, tot, send_token,
             pos_td, rec_code, rec_row, rec_raw, r_total, rec_stride, counts_out};
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ep_pack_kernel, kPackChunk, 0);
  if (per_sm < 1) return -3;
  int grid = num_sms * per_sm;
  if (grid > a.nchunks) grid = a.nchunks > 0 ? a.nchunks : 1;
  void* args[] = {&a};
  const cudaError_t e =
      cudaLaunchCooperativeKernel(reinterpret_cast<void*>(ep_pack_kernel), dim3(grid), dim3(kPackChunk), args, 0,
                                  stream);
  return e == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// Receiver: records -> dense routing codes (rows x K) + 32-row chunk
// histograms.  Records of one source arrive in (row, slot) order, so a
// record's slot is the number of earlier records of the same row.
// --------------------------------------------------------------------------
__global__ void ep_local_routing_kernel(const int32_t* __restrict__ rec_code, const int32_t* __restrict__ rec_row,
                                        const float* __restrict__ rec_raw, long long S, int stride,
                                        const long long* __restrict__ src_rec_base,
                                        const long long* __restrict__ src_row_base, int N, int K, int E,
                                        const unsigned char* __restrict__ hold, int32_t* __restrict__ sel_code,
                                        float* __restrict__ sel_raw, int* __restrict__ cnt_chunk,
                                        unsigned long long* __restrict__ flags) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < S;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    int src = 0;
    while (src + 1 < N && src_rec_base[src + 1] <= i) ++src;
    const long long lo = src_rec_base[src];
    const int row_local = rec_row[i * stride];
    int j = 0;
    while (i - 1 - j >= lo && rec_row[(i - 1 - j) * stride] == row_local) ++j;
    const long long row = src_row_base[src] + row_local;
    const int c = rec_code[i * stride];
    const int unit = c >> 2, level = c & 3;
    // an expert block this rank does not hold: a full selection needs any of
    // the unit's blocks here, a major-only one its block 0
    const bool ok = unit >= 0 && unit < E && j < K && (!hold || (hold[unit] & (level == 2 ? 1 : 2)));
    if (!ok) {
      atomicOr(&flags[2], 4ull);
      atomicOr(&flags[4], 4ull);
      continue;
    }
    sel_code[row * K + j] = c;
    sel_raw[row * K + j] = rec_raw[i * stride];
    atomicAdd(&cnt_chunk[(row / kRouterChunk) * 2 * E + 2 * unit + (level == 2 ? 0 : 1)], 1);
  }
}

int launch_ep_local_routing(const int32_t* rec_code, const int32_t* rec_row, const float* rec_raw, long long S,
                            int stride, const long long* src_rec_base, const long long* src_row_base, int N, int K,
                            int E, const unsigned char* hold, int32_t* sel_code, float* sel_raw, int* cnt_chunk,
                            unsigned long long* flags, int num_sms, cudaStream_t stream) {
  if (S <= 0) return 0;
  const long long b = (S + 255) / 256;
  ep_local_routing_kernel<<<static_cast<int>(b < num_sms * 8 ? b : num_sms * 8), 256, 0, stream>>>(
      rec_code, rec_row, rec_raw, S, stride, src_rec_base, src_row_base, N, K, E, hold, sel_code, sel_raw, cnt_chunk,
      flags);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// Per-expert selection counts of the last routing, from the router's 32-token
// chunk histograms (full + major-only kept selections): the integers the EP
// step all-reduces (device_loads of the whole batch, ep_sim.hpp:59-72).
// --------------------------------------------------------------------------
__global__ void ep_counts_kernel(const int* __restrict__ cnt_chunk, int nchunks, int E, long long* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    long long full = 0, major = 0;
    for (int ch = 0; ch < nchunks; ++ch) {
      full += cnt_chunk[static_cast<long long>(ch) * 2 * E + 2 * e];
      major += cnt_chunk[static_cast<long long>(ch) * 2 * E + 2 * e + 1];
    }
    out[2 * e] = full;   // selections kept on every sub-block
    out[2 * e + 1] = major;  // major-only selections
  }
}

int launch_ep_counts(const int* cnt_chunk, int nchunks, int E, long long* out, cudaStream_t stream) {
  ep_counts_kernel<<<(E + 127) / 128, 128, 0, stream>>>(cnt_chunk, nchunks, E, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// Device-side load-aware thresholds, right after the count all-reduce:
// device_loads (ep_sim.hpp:59-72) of the no-drop routing — each selection
// adds 1/P to the device of each of its P blocks, so device d's load is
// copies_d additions of 1/P — then load_aware_thresholds (:76-89) and the
// owner table t_unit[e] = threshold of the device of block e*P (:139-141).
// Same IEEE double operations, same order as the host functions.  One block.
// --------------------------------------------------------------------------
__global__ void ep_thresholds_kernel(const long long* __restrict__ counts, int E, int P, int D,
                                     const int32_t* __restrict__ device_of, double t_max, int load_aware,
                                     double* __restrict__ t_unit, double* __restrict__ loads_out) {
  extern __shared__ unsigned char smem_raw[];
  long long* copies = reinterpret_cast<long long*>(smem_raw);
  double* loads = reinterpret_cast<double*>(copies + D);
  double* th = loads + D;
  for (int d = threadIdx.x; d < D; d += blockDim.x) copies[d] = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < E * P; b += blockDim.x)  // no-drop counts: every selection keeps all P copies
    atomicAdd(reinterpret_cast<unsigned long long*>(&copies[device_of[b]]),
              static_cast<unsigned long long>(counts[2 * (b / P)] + counts[2 * (b / P) + 1]));
  __syncthreads();
  const double w = __ddiv_rn(1.0, static_cast<double>(P));
  const bool pow2 = (P & (P - 1)) == 0;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double l = 0.0;
    if (pow2) {
      l = __dmul_rn(static_cast<double>(copies[d]), w);  // every partial sum exact
    } else {
      for (long long i = 0; i < copies[d]; ++i) l = __dadd_rn(l, w);
    }
    loads[d] = l;
    if (loads_out) loads_out[d] = l;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double total = 0.0;
    for (int d = 0; d < D; ++d) total = __dadd_rn(total, loads[d]);
    const double ideal = __ddiv_rn(total, static_cast<double>(D));
    for (int d = 0; d < D; ++d) {
      if (!load_aware) {
        th[d] = t_max;
      } else {
        const double ratio = __ddiv_rn(loads[d], ideal);
        th[d] = ratio >= 1.0 ? t_max : __dmul_rn(t_max, ratio);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) t_unit[e] = th[device_of[e * P]];
}

int launch_ep_thresholds(const long long* counts, int E, int P, int D, const int32_t* device_of, double t_max,
                         int load_aware, double* t_unit, double* loads_out, cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(D) * (8 + 8 + 8);
  if (smem > 48 * 1024) return -1;
  ep_thresholds_kernel<<<1, 256, smem, stream>>>(counts, E, P, D, device_of, t_max, load_aware, t_unit, loads_out);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// --------------------------------------------------------------------------
// Sender: out[t] = sum over destinations d (ascending) of ret[pos_td[t][d]]
// + the local shared-expert rows.
// --------------------------------------------------------------------------
template <typename TY>
__global__ void __launch_bounds__(256) ep_final_combine_kernel(const TY* __restrict__ ret,
                                                               const int32_t* __restrict__ pos_td, int N,
                                                               const TY* __restrict__ ysh, int S, int shared_row0,
                                                               TY* __restrict__ out, int T, int d) {
  constexpr int V = 16 / sizeof(TY);
  const int nvec = d / V;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      float acc[V];
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = 0.f;
      auto add = [&](const TY* base, long long row) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(base + row * d) + v);
        const TY* e = reinterpret_cast<const TY*>(&q);
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += static_cast<float>(e[i]);
      };
      for (int dd = 0; dd < N; ++dd) {
        const int p = pos_td[static_cast<long long>(t) * N + dd];
        if (p >= 0) add(ret, p);
      }
      for (int s = 0; s < S; ++s) add(ysh, static_cast<long long>(shared_row0) + static_cast<long long>(s) * T + t);
      TY* o = out + static_cast<long long>(t) * d + static_cast<long long>(v) * V;
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = static_cast<TY>(acc[i]);
    }
  }
}

int launch_ep_final_combine(const void* ret, int y_bf16, const int32_t* pos_td, int N, const void* ysh, int S,
                            int shared_row0, void* out, int T, int d, int num_sms, cudaStream_t stream) {
  if (T <= 0) return 0;
  const int grid = T < num_sms * 16 ? T : num_sms * 16;
  if (y_bf16)
    ep_final_combine_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(ret), pos_td, N, static_cast<const __nv_bfloat16*>(ysh), S, shared_row0,
        static_cast<__nv_bfloat16*>(out), T, d);
  else
    ep_final_combine_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(ret), pos_td, N,
                                                             static_cast<const float*>(ysh), S, shared_row0,
                                                             static_cast<float*>(out), T, d);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
