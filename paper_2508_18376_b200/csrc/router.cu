// K0 (exact mode) and K1: gate logits and the fused router.
//
// K1 restates, per token and bit for bit, the routing half of route_and_drop
// (/root/reference/proj/include/dsmoe/dropping.hpp:248-258):
//   softmax_inplace      matrix.hpp:68-78   (sequential max, glibc expf, sequential
//                                            float sum in ascending e, IEEE divide)
//   topk_route           moe.hpp:181-206    (K argmax rounds, strict >, lower index wins)
//   replay_routing       moe.hpp:277-309    (copy-major slots p*K+s, index e*P+p)
//   normalize_topk       dropping.hpp:60-72 (double sum over base_k in slot order)
//   apply_bands_fn       dropping.hpp:93-122 (1T/2T bands, keep-top-1 guard)
//   + per-owner-device thresholds of simulate_step (ep_sim.hpp:139-149) for EP.
// It also emits the forward metadata the permute kernel consumes: per original
// selection (t, s) the expert unit and its level (2 = every sub-block, 1 =
// major sub-block only, 0 = dropped), per-unit row counts, and the retained
// copy counters drop_stats (dropping.hpp:171-195) is computed from.
//
// This translation unit is compiled with -fmad=false: every float / double
// operation rounds exactly where the reference's (-ffp-contract=off) does.
#include "kernels.h"

namespace dsb {

constexpr int kMaxK = 16;  // Top-K selections per token supported on device

__global__ void __launch_bounds__(128) router_kernel(const RouterArgs a) {
  extern __shared__ float sm[];
  const int E = a.E, K = a.K, P = a.P;
  const int ld = E + 1;
  const int t0 = blockIdx.x * blockDim.x;
  const int nt = min(static_cast<int>(blockDim.x), a.T - t0);
  // coalesced stage of this block's logits rows
  for (int i = threadIdx.x; i < nt * E; i += blockDim.x) {
    const int r = i / E, c = i - r * E;
    sm[r * ld + c] = a.logits[static_cast<long long>(t0 + r) * a.ld_logits + c];
  }
  __shared__ unsigned long long s_n1, s_nh;
  if (threadIdx.x == 0) { s_n1 = 0; s_nh = 0; }
  __syncthreads();
  unsigned long long n1 = 0, nh = 0;
  const int tl = threadIdx.x;
  if (tl < nt) {
    const int t = t0 + tl;
    float* v = sm + tl * ld;
    // softmax_inplace: mx = std::max(mx, x) over the row
    float mx = v[0];
    for (int e = 0; e < E; ++e) mx = (mx < v[e]) ? v[e] : mx;
    float sum = 0.0f;
    for (int e = 0; e < E; ++e) {
      const float ex = glibc_expf(__fsub_rn(v[e], mx));
      v[e] = ex;
      sum = __fadd_rn(sum, ex);
    }
    for (int e = 0; e < E; ++e) v[e] = __fdiv_rn(v[e], sum);
    // topk_route
    int sel[kMaxK];
    float sraw[kMaxK];
    unsigned long long taken[4] = {0, 0, 0, 0};
    for (int j = 0; j < K; ++j) {
      int best = -1;
      float bv = 0.f;
      for (int e = 0; e < E; ++e) {
        if ((taken[e >> 6] >> (e & 63)) & 1ull) continue;
        if (best < 0 || v[e] > bv) { best = e; bv = v[e]; }
      }
      taken[best >> 6] |= 1ull << (best & 63);
      sel[j] = best;
      sraw[j] = bv;
    }
    // ensure_normalized / normalize_topk
    double dsum = 0.0;
    if (a.normalize) {
      for (int j = 0; j < K; ++j) dsum = __dadd_rn(dsum, static_cast<double>(sraw[j]));
      if (!(dsum > 0.0)) atomicOr(&a.counters[2], 1ull);
    }
    double ns[kMaxK];
    for (int j = 0; j < K; ++j)
      ns[j] = a.normalize ? __ddiv_rn(static_cast<double>(sraw[j]), dsum) : static_cast<double>(sraw[j]);
    // apply_bands_fn: level 2 = keep all copies, 1 = major part, 0 = drop
    int level[kMaxK];
    int top_slot = 0;
    for (int s = 0; s < K; ++s) {
      if (ns[s] > ns[top_slot]) top_slot = s;
      if (a.kind == 0) { level[s] = 2; continue; }
      double tmaj = a.t_major, tmin = a.t_minor;
      if (a.t_unit) {
        const double own = a.t_unit[sel[s]];
        tmaj = __dadd_rn(own, a.maj_off);
        tmin = __dadd_rn(own, a.min_off);
      }
      level[s] = ns[s] >= tmin ? 2 : (ns[s] >= tmaj ? 1 : 0);
    }
    if (a.kind != 0 && a.keep_top1) level[top_slot] = 2;
    // outputs
    const long long kp = static_cast<long long>(K) * P;
    for (int s = 0; s < K; ++s) {
      const int lv = level[s];
      for (int cp = 0; cp < P; ++cp) {
        // fraction code of copy cp: P == 1 -> {0, 0.5, 1}; P > 1 -> copy 0 kept
        // unless dropped, copies >= 1 kept only in the full band.
        uint8_t fc;
        if (P == 1) fc = static_cast<uint8_t>(lv);  // 2 -> 1.0, 1 -> 0.5
        else fc = (cp == 0) ? (lv > 0 ? 2 : 0) : (lv == 2 ? 2 : 0);
        n1 += fc == 2;
        nh += fc == 1;
        const long long f = t * kp + static_cast<long long>(cp) * K + s;
        if (a.idx) a.idx[f] = sel[s] * P + cp;
        if (a.raw) a.raw[f] = sraw[s];
        if (a.norm) a.norm[f] = ns[s];
        if (a.frac) a.frac[f] = fc;
      }
      const long long g = static_cast<long long>(t) * K + s;
      a.sel_code[g] = lv > 0 ? sel[s] * 4 + lv : -1;
      a.sel_raw[g] = sraw[s];
      a.slot_pos[g] = -1;
      if (lv > 0) atomicAdd(&a.cnt[2 * sel[s] + (lv == 2 ? 0 : 1)], 1);
    }
  }
  // block-reduce the retained-copy counters
  for (int o = 16; o > 0; o >>= 1) {
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    nh += __shfl_xor_sync(0xffffffffu, nh, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_n1, n1);
    atomicAdd(&s_nh, nh);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&a.counters[0], s_n1);
    atomicAdd(&a.counters[1], s_nh);
  }
}

int launch_router(const RouterArgs& a, cudaStream_t stream) {
  if (a.K > kMaxK || a.E > 256 || a.K < 1 || a.K > a.E) return -1;
  const int threads = 128;
  const int blocks = (a.T + threads - 1) / threads;
  const size_t smem = static_cast<size_t>(threads) * (a.E + 1) * sizeof(float);
  if (smem > 48 * 1024) cudaFuncSetAttribute(router_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (blocks > 0) router_kernel<<<blocks, threads, smem, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ---------------------------------------------------------------------------
// Caller-supplied RoutingDecision -> forward metadata (moe_forward with an
// explicit routing, moe.hpp:239).  Accepts the canonical layouts route_tokens /
// replay_routing / apply_bands produce: copy cp of selection s at slot cp*K+s
// with index (e/P)*P+cp, copies >= 1 sharing one fraction, copy 0 kept whenever
// any copy is, equal raw scores across copies; P == 1 allows fraction 0.5.
// Anything else sets error bit 2 (the host reports invalid_state).
// ---------------------------------------------------------------------------
__global__ void import_routing_kernel(const ImportArgs a) {
  const long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= static_cast<long long>(a.T) * a.K) return;
  const int t = static_cast<int>(g / a.K), s = static_cast<int>(g - static_cast<long long>(t) * a.K);
  const long long kp = static_cast<long long>(a.K) * a.P;
  const long long f0 = t * kp + s;
  const int e0 = a.idx[f0];
  const double fr0 = a.frac[f0];
  const double r0 = a.raw[f0];
  bool ok = e0 >= 0 && e0 < a.nphys && (e0 % a.P) == 0;
  int lv = 0;
  if (a.P == 1) {
    ok = ok && (fr0 == 0.0 || fr0 == 0.5 || fr0 == 1.0);
    lv = fr0 == 1.0 ? 2 : (fr0 == 0.5 ? 1 : 0);
  } else {
    const double fr1 = a.frac[f0 + a.K];
    ok = ok && (fr0 == 0.0 || fr0 == 1.0) && (fr1 == 0.0 || fr1 == 1.0) && !(fr0 == 0.0 && fr1 != 0.0);
    for (int cp = 1; cp < a.P; ++cp) {
      const long long f = f0 + static_cast<long long>(cp) * a.K;
      ok = ok && a.idx[f] == e0 + cp && a.frac[f] == fr1 && a.raw[f] == r0;
    }
    lv = fr0 == 0.0 ? 0 : (fr1 == 1.0 ? 2 : 1);
  }
  if (!ok) {
    atomicOr(&a.counters[2], 4ull);
    lv = 0;
  }
  const int unit = e0 / a.P;
  a.sel_code[g] = lv > 0 ? unit * 4 + lv : -1;
  a.sel_raw[g] = static_cast<float>(r0);
  a.slot_pos[g] = -1;
  if (lv > 0) atomicAdd(&a.cnt[2 * unit + (lv == 2 ? 0 : 1)], 1);
}

int launch_import_routing(const ImportArgs& a, cudaStream_t stream) {
  const long long n = static_cast<long long>(a.T) * a.K;
  if (n > 0) import_routing_kernel<<<static_cast<int>((n + 255) / 256), 256, 0, stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ---------------------------------------------------------------------------
// K0, exact-order mode: logits[t][e] = sum_k x[t][k] * gate[k][e] accumulated
// from +0 in ascending k with one rounding per multiply and per add — the
// i-k-j matmul of matrix.hpp:47-64 under -ffp-contract=off.  For bf16 inputs
// every product is exact in fp32, so this reproduces the oracle's logits on
// the bf16-rounded operands bit for bit.
// ---------------------------------------------------------------------------
template <typename TX>
__global__ void __launch_bounds__(256) gate_logits_exact_kernel(const TX* __restrict__ x,
                                                                const float* __restrict__ gate,
                                                                float* __restrict__ out, int T,
                                                                int d, int E) {
  __shared__ float xs[64][33];
  __shared__ float gs[32][65];
  const int tb = blockIdx.x * 64, eb = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  for (int k0 = 0; k0 < d; k0 += 32) {
    for (int i = threadIdx.x; i < 64 * 32; i += 256) {
      const int r = i >> 5, c = i & 31;
      const int t = tb + r, k = k0 + c;
      xs[r][c] = (t < T && k < d) ? static_cast<float>(x[static_cast<long long>(t) * d + k]) : 0.0f;
    }
    for (int i = threadIdx.x; i < 32 * 64; i += 256) {
      const int r = i >> 6, c = i & 63;
      const int k = k0 + r, e = eb + c;
      gs[r][c] = (k < d && e < E) ? gate[static_cast<long long>(k) * E + e] : 0.0f;
    }
    __syncthreads();
    const int kn = min(32, d - k0);
    for (int k = 0; k < kn; ++k) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float xv = xs[ty + 16 * i][k];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(xv, gs[k][tx + 16 * j]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int t = tb + ty + 16 * i, e = eb + tx + 16 * j;
      if (t < T && e < E) out[static_cast<long long>(t) * E + e] = acc[i][j];
    }
}

int launch_gate_logits_exact(const void* x, int x_bf16, const float* gate, float* out, int T, int d,
                             int E, cudaStream_t stream) {
  dim3 grid((T + 63) / 64, (E + 63) / 64);
  if (T <= 0) return 0;
  if (x_bf16)
    gate_logits_exact_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(x), gate, out, T, d, E);
  else
    gate_logits_exact_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(x), gate, out,
                                                               T, d, E);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
