// K0 (exact mode) and K1: gate logits and the fused router.
//
// K1 restates, per token and bit for bit, the routing half of route_and_drop
// (/root/reference/proj/include/dsmoe/dropping.hpp:248-258):
//   softmax_inplace      matrix.hpp:68-78   (max, glibc expf, float sum in
//                                            ascending e, IEEE divide)
//   topk_route           moe.hpp:181-206    (K argmax rounds, strict >, lower index wins)
//   replay_routing       moe.hpp:277-309    (copy-major slots p*K+s, index e*P+p)
//   normalize_topk       dropping.hpp:60-72 (double sum over base_k in slot order)
//   apply_bands_fn       dropping.hpp:93-122 (1T/2T bands, keep-top-1 guard)
//   + per-owner-device thresholds of simulate_step (ep_sim.hpp:139-149) for EP.
// One warp per token: lanes hold experts e = lane + 32 j.  The max and the
// arg-max rounds are order-independent, so they run as warp shuffles; the
// softmax denominator is order-dependent, so lane 0 adds the exponentials in
// ascending e exactly like the reference loop.
//
// It also emits the forward metadata the scatter kernel consumes: per original
// selection (t, s) the expert unit and its level (2 = every sub-block, 1 =
// major sub-block only, 0 = dropped), per-chunk (128 tokens) histograms of
// (unit, level), and the retained-copy counters drop_stats
// (dropping.hpp:171-195) is computed from.
//
// This translation unit is compiled with -fmad=false: every float / double
// operation rounds exactly where the reference's (-ffp-contract=off) does.
#include <cooperative_groups.h>

#include <cstdio>

#include "kernels.h"

namespace dsb {

constexpr int kMaxK = 32;     // Top-K selections per token supported on device (one lane each)
constexpr int kMaxEPL = 8;    // experts per lane (E <= 256)

// glibc expf (expf_glibc.h) with the 2^(i/32) table staged in shared memory:
// lanes index it divergently, which serialises in the constant cache.
__device__ __forceinline__ float expf_tab(float x, const uint64_t* tab) {
  // glibc's main path, computed unconditionally; its special-case exits
  // (|x| >= 88, inf, nan) become selects, so independent calls carry no
  // branches and the compiler can interleave them (one call alone is ~200
  // cycles of dependent FP64 latency)
  const uint32_t ux = __float_as_uint(x);
  const uint32_t abstop = (ux >> 20) & 0x7ff;
  const double InvLn2N = 0x1.71547652b82fep+5, SHIFT = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-20, C1 = 0x1.ebfce50fac4f3p-13, C2 = 0x1.62e42ff0c52d6p-6;
  const double xd = static_cast<double>(x);
  double kd = __fma_rn(InvLn2N, xd, SHIFT);
  const uint64_t ki = static_cast<uint64_t>(__double_as_longlong(kd));
  kd = __dsub_rn(kd, SHIFT);
  const double r = __fma_rn(InvLn2N, xd, -kd);
  const double s = __longlong_as_double(static_cast<long long>(tab[ki % 32] + (ki << 47)));
  const double y = __fma_rn(__fma_rn(C0, r, C1), __dmul_rn(r, r), __fma_rn(C2, r, 1.0));
  float res = static_cast<float>(__dmul_rn(y, s));
  // glibc's exits for abstop >= top12(88): none of these conditions holds
  // below that, so they apply unconditionally (selects, no branch)
  res = x < -0x1.9fe368p6f ? 0.0f : res;
  res = x > 0x1.62e42ep6f ? __uint_as_float(0x7f800000u) : res;
  res = abstop >= 0x7f8 ? x + x : res;
  res = ux == 0xff800000u ? 0.0f : res;
  return res;
}

template <int EPL>  // experts per lane, E <= 32 * EPL
__global__ void __launch_bounds__(kRouterChunk * 32) router_kernel(const RouterArgs a) {
  extern __shared__ int s_hist[];  // 2E codes: [unit*2 + (level==2 ? 0 : 1)]
  __shared__ uint64_t tab[32];
  __shared__ unsigned long long s_n1, s_nh;
  const int E = a.E, K = a.K, P = a.P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) s_hist[i] = 0;
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2fTab[threadIdx.x];
  if (threadIdx.x == 0) { s_n1 = 0; s_nh = 0; }
  __syncthreads();
  pdl_wait();
  constexpr int epl = EPL;
  unsigned long long n1 = 0, nh = 0;
  const int t = blockIdx.x * kRouterChunk + warp;  // one token per warp
  if (t < a.T) {
    const float* row = a.logits + static_cast<long long>(t) * a.ld_logits;
    float v[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = lane + 32 * j;
      v[j] = (j < epl && e < E) ? row[e] : -INFINITY;
    }
    // softmax_inplace: max (order-free), exp, ordered float sum, divide
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < EPL; ++j) mx = (mx < v[j]) ? v[j] : mx;
    for (int o = 16; o > 0; o >>= 1) {
      const float other = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = (mx < other) ? other : mx;
    }
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (j < epl) v[j] = (lane + 32 * j < E) ? expf_tab(__fsub_rn(v[j], mx), tab) : 0.0f;
    float sum = 0.0f;  // ascending e, identical on every lane
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      if (j >= epl) break;
      const int lim = min(32, E - 32 * j);
#pragma unroll 8
      for (int l = 0; l < 32; ++l) {
        const float ex = __shfl_sync(0xffffffffu, v[j], l);
        if (l < lim) sum = __fadd_rn(sum, ex);
      }
    }
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (j < epl) v[j] = __fdiv_rn(v[j], sum);
    // topk_route: strict >, lower index first (moe.hpp:193-205) is the
    // descending order of key = (probability bits << 32) | ~expert — the
    // probabilities are non-negative floats, so their bit patterns order like
    // their values.  A warp bitonic sort of the 32*EPL keys (element i =
    // expert i, held by lane i % 32, slot i / 32) leaves the rank-s key in
    // slot 0 of lane s.  Padding experts get key 0 and sort last.
    unsigned long long key[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = lane + 32 * j;
      key[j] = e < E ? (static_cast<unsigned long long>(__float_as_uint(v[j])) << 32) |
                           static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<unsigned>(e))
                     : 0ull;
    }
#pragma unroll
    for (int k = 2; k <= 32 * EPL; k <<= 1) {
#pragma unroll
      for (int dist = k >> 1; dist > 0; dist >>= 1) {
        if (dist >= 32) {  // partner in this lane
#pragma unroll
          for (int j = 0; j < EPL; ++j) {
            const int pj = j ^ (dist >> 5);
            if (pj > j) {
              const bool desc = (((j * 32 + lane) & k) == 0);
              const unsigned long long a = key[j], b = key[pj];
              const unsigned long long hi = a > b ? a : b, lo = a > b ? b : a;
              key[j] = desc ? hi : lo;
              key[pj] = desc ? lo : hi;
            }
          }
        } else {  // partner in lane ^ dist
#pragma unroll
          for (int j = 0; j < EPL; ++j) {
            const int i = j * 32 + lane;
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, key[j], dist);
            const bool take_max = ((i & dist) == 0) == ((i & k) == 0);
            key[j] = take_max ? (key[j] > o ? key[j] : o) : (key[j] > o ? o : key[j]);
          }
        }
      }
    }
    const int my_e = static_cast<int>(0xFFFFFFFFu - static_cast<unsigned>(key[0] & 0xFFFFFFFFull));
    const float my_raw = __uint_as_float(static_cast<unsigned>(key[0] >> 32));
    // normalize_topk: ordered double sum over the K selections, then divide
    const bool active = lane < K;
    double dsum = 0.0;
    if (a.normalize) {
      for (int s = 0; s < K; ++s) dsum = __dadd_rn(dsum, static_cast<double>(__shfl_sync(0xffffffffu, my_raw, s)));
      if (!(dsum > 0.0) && lane == 0) { atomicOr(&a.counters[2], 1ull); atomicOr(&a.counters[4], 1ull); }
    }
    const double ns = active ? (a.normalize ? __ddiv_rn(static_cast<double>(my_raw), dsum) : static_cast<double>(my_raw))
                             : -1.0;
    // top_slot = first maximum of ns (strict >, dropping.hpp:99)
    double tv = ns;
    int ts = active ? lane : 1 << 30;
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, tv, o);
      const int os = __shfl_xor_sync(0xffffffffu, ts, o);
      if (ov > tv || (ov == tv && os < ts)) { tv = ov; ts = os; }
    }
    // apply_bands_fn on this lane's selection
    int lv = 0;
    if (active) {
      if (a.kind == 0) {
        lv = 2;
      } else {
        double tmaj = a.t_major, tmin = a.t_minor;
        if (a.t_unit) {
          const double own = a.t_unit[my_e];
          tmaj = __dadd_rn(own, a.maj_off);
          tmin = __dadd_rn(own, a.min_off);
        }
        lv = ns >= tmin ? 2 : (ns >= tmaj ? 1 : 0);
        if (a.keep_top1 && lane == ts) lv = 2;
      }
      for (int cp = 0; cp < P; ++cp) {
        const uint8_t fc = P == 1 ? static_cast<uint8_t>(lv) : (cp == 0 ? (lv > 0 ? 2 : 0) : (lv == 2 ? 2 : 0));
        n1 += fc == 2;
        nh += fc == 1;
        const long long g = static_cast<long long>(t) * K * P + static_cast<long long>(cp) * K + lane;
        if (a.idx) a.idx[g] = my_e * P + cp;
        if (a.raw) a.raw[g] = my_raw;
        if (a.norm) a.norm[g] = ns;
        if (a.frac) a.frac[g] = fc;
      }
      const long long q = static_cast<long long>(t) * K + lane;
      a.sel_code[q] = lv > 0 ? my_e * 4 + lv : -1;
      a.sel_raw[q] = my_raw;
      if (lv > 0) atomicAdd(&s_hist[2 * my_e + (lv == 2 ? 0 : 1)], 1);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    nh += __shfl_xor_sync(0xffffffffu, nh, o);
  }
  if (lane == 0 && (n1 | nh)) {
    atomicAdd(&s_n1, n1);
    atomicAdd(&s_nh, nh);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x)
    a.cnt_chunk[static_cast<long long>(blockIdx.x) * 2 * E + i] = s_hist[i];
  if (threadIdx.x == 0) {
    atomicAdd(&a.counters[0], s_n1);
    atomicAdd(&a.counters[1], s_nh);
  }
}

// Quad-per-token variant for E <= 4 * EPT (64): lane q of a token's quad
// holds experts [q*EPT, (q+1)*EPT) in registers.  The softmax denominator is
// one ascending-e chain of float adds handed from lane to lane (the
// reference's summation order).  topk_route's K arg-max rounds (strict >,
// lower index wins) are the descending order of the keys (probability bits
// << 32) | ~expert (router_kernel): each lane sorts its keys with a register
// bitonic network, then two bitonic merges with the partner lanes (xor 1,
// xor 2) leave the quad's top KK keys, sorted, on every lane — a few dozen
// dependent steps instead of K serial scan + shuffle rounds.  Each lane then
// finishes the slots j = q mod 4.  One block = 32 tokens = one scatter chunk
// (kRouterChunk).
template <int N>
__device__ __forceinline__ void sort_desc(unsigned long long (&k)[N]) {
#pragma unroll
  for (int w = 2; w <= N; w <<= 1) {
#pragma unroll
    for (int j = w >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long a = k[i], b = k[l];
          const bool sw = ((i & w) == 0) ? (a < b) : (a > b);
          k[i] = sw ? b : a;
          k[l] = sw ? a : b;
        }
      }
    }
  }
}

// One token on a group of LPT lanes (lane q holds experts [q*EPT, (q+1)*EPT)
// of its logits in v): softmax, top-K, replay, normalize, bands, and the
// token's outputs (RoutingDecision slots, forward codes, s_hist counts).
// Returns true when the token's top-K scores sum to <= 0 (normalize_topk
// throws, dropping.hpp:67).  Shared by the standalone router and the fused
// gate + router kernel, so both are the same arithmetic.
// Descending 8-key sort with the 19-comparator, depth-6 network (Batcher /
// Knuth's optimum for 8 inputs; checked with the 0-1 principle) instead of the
// 24-comparator bitonic network.
__device__ __forceinline__ void cex_desc(unsigned long long& a, unsigned long long& b) {
  const unsigned long long x = a, y = b;
  const bool sw = x < y;
  a = sw ? y : x;
  b = sw ? x : y;
}
__device__ __forceinline__ void sort8_desc(unsigned long long* k) {
  cex_desc(k[0], k[2]); cex_desc(k[1], k[3]); cex_desc(k[4], k[6]); cex_desc(k[5], k[7]);
  cex_desc(k[0], k[4]); cex_desc(k[1], k[5]); cex_desc(k[2], k[6]); cex_desc(k[3], k[7]);
  cex_desc(k[0], k[1]); cex_desc(k[2], k[3]); cex_desc(k[4], k[5]); cex_desc(k[6], k[7]);
  cex_desc(k[2], k[4]); cex_desc(k[3], k[5]);
  cex_desc(k[1], k[4]); cex_desc(k[3], k[6]);
  cex_desc(k[1], k[2]); cex_desc(k[3], k[4]); cex_desc(k[5], k[6]);
}
// the lane's top KK keys, descending, in key[0..KK).  EPT = 2 KK = 16: sort
// both halves (2 x 19 comparators), keep max(a[i], b[KK-1-i]) (a bitonic
// sequence holding the top KK of the union) and merge it (12) — 50
// comparators + 8 maxima instead of the 80 of a 16-key bitonic sort.
template <int NS, int EPT, int KK>
__device__ __forceinline__ void lane_topk(unsigned long long (&key)[NS]) {
  if constexpr (EPT == 16 && KK == 8 && NS == 16) {
    sort8_desc(key);
    sort8_desc(key + 8);
#pragma unroll
    for (int i = 0; i < 8; ++i) key[i] = key[i] > key[15 - i] ? key[i] : key[15 - i];
#pragma unroll
    for (int j = 4; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int l = i ^ j;
        if (l > i) cex_desc(key[i], key[l]);
      }
    }
  } else {
    sort_desc<NS>(key);
  }
}

template <int EPT, int LPT, int KK>
__device__ __forceinline__ bool quad_route(const RouterArgs& a, int t, bool tok_ok, float (&v)[EPT], int lane,
                                           const uint64_t* tab, int* s_hist, unsigned long long& n1,
                                           unsigned long long& nh) {
  constexpr int NS = KK > EPT ? KK : EPT;  // keys sorted per lane (padded with 0 = "no expert")
  const int E = a.E, K = a.K, P = a.P;
  const int q = lane % LPT, qbase = lane - q;
  const int e0 = q * EPT;
  bool bad = false;
  // softmax_inplace (matrix.hpp:68-78): max (order-free), expf, ascending-e sum, divide
  float mx = v[0];
#pragma unroll
  for (int i = 0; i < EPT; ++i) mx = (mx < v[i]) ? v[i] : mx;
#pragma unroll
  for (int o = 1; o < LPT; o <<= 1) {
    const float other = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = (mx < other) ? other : mx;
  }
#pragma unroll
  for (int i = 0; i < EPT; ++i) v[i] = e0 + i < E ? expf_tab(__fsub_rn(v[i], mx), tab) : 0.0f;
  float sum = 0.0f;
#pragma unroll
  for (int k = 0; k < LPT; ++k) {
    if (q == k) {
#pragma unroll
      for (int i = 0; i < EPT; ++i)
        if (e0 + i < E) sum = __fadd_rn(sum, v[i]);
    }
    sum = __shfl_sync(0xffffffffu, sum, qbase | k);
  }
#pragma unroll
  for (int i = 0; i < EPT; ++i) v[i] = __fdiv_rn(v[i], sum);
  // topk_route (moe.hpp:193-205) as a key sort
  unsigned long long key[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const int e = e0 + i;
    key[i] = (i < EPT && e < E) ? (static_cast<unsigned long long>(__float_as_uint(v[i < EPT ? i : 0])) << 32) |
                                      static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<unsigned>(e))
                                : 0ull;
  }
  lane_topk<NS, EPT, KK>(key);
#pragma unroll
  for (int m = 1; m < LPT; m <<= 1) {
    // top KK of (mine U partner's): max(mine[i], theirs[KK-1-i]) is bitonic
    unsigned long long c[KK];
#pragma unroll
    for (int i = 0; i < KK; ++i) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, key[KK - 1 - i], m);
      c[i] = key[i] > o ? key[i] : o;
    }
#pragma unroll
    for (int j = KK >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < KK; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const unsigned long long x = c[i], y = c[l];
          c[i] = x > y ? x : y;
          c[l] = x > y ? y : x;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < KK; ++i) key[i] = c[i];
  }
  float sraw[KK];
  int sel[KK];
#pragma unroll
  for (int j = 0; j < KK; ++j) {
    sel[j] = static_cast<int>(0xFFFFFFFFu - static_cast<unsigned>(key[j] & 0xFFFFFFFFull));
    sraw[j] = __uint_as_float(static_cast<unsigned>(key[j] >> 32));
  }
  // normalize_topk (dropping.hpp:60-72)
  double dsum = 0.0;
  if (a.normalize) {
#pragma unroll
    for (int j = 0; j < KK; ++j)
      if (j < K) dsum = __dadd_rn(dsum, static_cast<double>(sraw[j]));
    bad = tok_ok && q == 0 && !(dsum > 0.0);
  }
  // this lane's slots j = q, q+LPT, ...; top_slot = first maximum of ns (dropping.hpp:99)
  constexpr int kSl = KK / LPT;
  double nsj[kSl];
  float rsj[kSl];
  int esj[kSl];
  double tv = -1.0;
  int ts = 1 << 30;
#pragma unroll
  for (int m = 0; m < kSl; ++m) {
    const int j = q + LPT * m;
    float rj = 0.0f;
    int ej = 0;
#pragma unroll
    for (int jj = LPT * m; jj < LPT * (m + 1); ++jj)
      if (jj == j) { rj = sraw[jj]; ej = sel[jj]; }
    rsj[m] = rj;
    esj[m] = ej;
    nsj[m] = 0.0;
    if (j < K) {
      nsj[m] = a.normalize ? __ddiv_rn(static_cast<double>(rj), dsum) : static_cast<double>(rj);
      if (ts == (1 << 30) || nsj[m] > tv) { tv = nsj[m]; ts = j; }
    }
  }
#pragma unroll
  for (int o = 1; o < LPT; o <<= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, tv, o);
    const int os = __shfl_xor_sync(0xffffffffu, ts, o);
    if (os != (1 << 30) && (ts == (1 << 30) || ov > tv || (ov == tv && os < ts))) { tv = ov; ts = os; }
  }
  // apply_bands_fn (dropping.hpp:93-122) on this lane's slots
  if (tok_ok) {
#pragma unroll
    for (int m = 0; m < kSl; ++m) {
      const int j = q + LPT * m;
      if (j >= K) break;
      const int my_e = esj[m];
      const double ns = nsj[m];
      int lv = 2;
      if (a.kind != 0) {
        double tmaj = a.t_major, tmin = a.t_minor;
        if (a.t_unit) {
          const double own = a.t_unit[my_e];
          tmaj = __dadd_rn(own, a.maj_off);
          tmin = __dadd_rn(own, a.min_off);
        }
        lv = ns >= tmin ? 2 : (ns >= tmaj ? 1 : 0);
        if (a.keep_top1 && j == ts) lv = 2;
      }
      for (int cp = 0; cp < P; ++cp) {
        const uint8_t fc = P == 1 ? static_cast<uint8_t>(lv) : (cp == 0 ? (lv > 0 ? 2 : 0) : (lv == 2 ? 2 : 0));
        n1 += fc == 2;
        nh += fc == 1;
        const long long g = static_cast<long long>(t) * K * P + static_cast<long long>(cp) * K + j;
        if (a.idx) a.idx[g] = my_e * P + cp;
        if (a.raw) a.raw[g] = rsj[m];
        if (a.norm) a.norm[g] = ns;
        if (a.frac) a.frac[g] = fc;
      }
      const long long qi = static_cast<long long>(t) * K + j;
      a.sel_code[qi] = lv > 0 ? my_e * 4 + lv : -1;
      a.sel_raw[qi] = rsj[m];
      if (lv > 0) atomicAdd(&s_hist[2 * my_e + (lv == 2 ? 0 : 1)], 1);
    }
  }
  return bad;
}

template <int EPT, int LPT, int KK>
__global__ void __launch_bounds__(kRouterChunk * LPT) router_quad_kernel(const RouterArgs a) {
  extern __shared__ int s_hist[];  // 2E
  __shared__ uint64_t tab[32];
  __shared__ unsigned long long s_n1, s_nh;
  static_assert(KK <= 16 && EPT <= 16, "quad router: at most 16 keys per lane");
  const int E = a.E;
  const int lane = threadIdx.x & 31, q = lane % LPT;
  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) s_hist[i] = 0;
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2fTab[threadIdx.x];
  if (threadIdx.x == 0) { s_n1 = 0; s_nh = 0; }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  unsigned long long n1 = 0, nh = 0;
  const int t = blockIdx.x * kRouterChunk + threadIdx.x / LPT;
  const bool tok_ok = t < a.T;  // uniform across the quad
  const int e0 = q * EPT;
  const float* row = a.logits + static_cast<long long>(tok_ok ? t : 0) * a.ld_logits;
  float v[EPT];
#pragma unroll
  for (int i = 0; i < EPT; ++i) v[i] = (tok_ok && e0 + i < E) ? row[e0 + i] : -INFINITY;
  if (a.nsplit > 1) {  // split-K gate: partial planes summed in ascending order, written back
    for (int sp0 = 1; sp0 < a.nsplit; sp0 += 4) {  // 4 planes' loads in flight, then the ordered adds
      float w[4][EPT];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float* rs = row + (sp0 + j) * a.split_stride;
#pragma unroll
        for (int i = 0; i < EPT; ++i) w[j][i] = (sp0 + j < a.nsplit && tok_ok && e0 + i < E) ? rs[e0 + i] : 0.0f;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (sp0 + j < a.nsplit) {
#pragma unroll
          for (int i = 0; i < EPT; ++i)
            if (e0 + i < E) v[i] = __fadd_rn(v[i], w[j][i]);
        }
    }
    if (tok_ok) {
      float* w = a.logits_sum + static_cast<long long>(t) * a.ld_logits;
#pragma unroll
      for (int i = 0; i < EPT; ++i)
        if (e0 + i < E) w[e0 + i] = v[i];
    }
  }
  if (quad_route<EPT, LPT, KK>(a, t, tok_ok, v, lane, tab, s_hist, n1, nh)) {
    atomicOr(&a.counters[2], 1ull);
    atomicOr(&a.counters[4], 1ull);
  }
  for (int o = 16; o > 0; o >>= 1) {
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    nh += __shfl_xor_sync(0xffffffffu, nh, o);
  }
  if (lane == 0 && (n1 | nh)) {
    atomicAdd(&s_n1, n1);
    atomicAdd(&s_nh, nh);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x)
    a.cnt_chunk[static_cast<long long>(blockIdx.x) * 2 * E + i] = s_hist[i];
  if (threadIdx.x == 0) {
    atomicAdd(&a.counters[0], s_n1);
    atomicAdd(&a.counters[1], s_nh);
  }
}

int launch_router(const RouterArgs& a, cudaStream_t stream) {
  if (a.K > kMaxK || a.E > 32 * kMaxEPL || a.K < 1 || a.K > a.E) return -1;
  const int blocks = (a.T + kRouterChunk - 1) / kRouterChunk;
  const size_t smem = static_cast<size_t>(2 * a.E) * sizeof(int);
  if (blocks <= 0) return 0;
  if (a.nsplit > 1 && !(a.E <= 64 && a.K <= 16)) return -1;  // split planes: quad router only
  // DSMOE_B200_ROUTER_LPT=8: eight lanes per token (8 experts each) for E <= 64,
  // K <= 8 — shorter per-lane chains, more tokens resident per SM (A/B knob)
  static const int lpt_env = [] {
    const char* v = getenv("DSMOE_B200_ROUTER_LPT");
    return v ? atoi(v) : 4;
  }();
  if (lpt_env == 8 && a.E <= 64 && a.K <= 8 && a.nsplit <= 1) {
    launch_pdl(router_quad_kernel<8, 8, 8>, dim3(blocks), dim3(kRouterChunk * 8), smem, stream, a);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
  }
  if (a.E <= 64 && a.K <= 16) {
    if (a.E <= 32 && a.K <= 8)
      launch_pdl(router_quad_kernel<8, 4, 8>, dim3(blocks), dim3(kRouterChunk * 4), smem, stream, a);
    else if (a.E <= 32)
      launch_pdl(router_quad_kernel<8, 4, 16>, dim3(blocks), dim3(kRouterChunk * 4), smem, stream, a);
    else if (a.K <= 8)
      launch_pdl(router_quad_kernel<16, 4, 8>, dim3(blocks), dim3(kRouterChunk * 4), smem, stream, a);
    else
      launch_pdl(router_quad_kernel<16, 4, 16>, dim3(blocks), dim3(kRouterChunk * 4), smem, stream, a);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
  }
  const int epl = (a.E + 31) / 32;
  if (epl <= 1)
    launch_pdl(router_kernel<1>, dim3(blocks), dim3(kRouterChunk * 32), smem, stream, a);
  else if (epl <= 2)
    launch_pdl(router_kernel<2>, dim3(blocks), dim3(kRouterChunk * 32), smem, stream, a);
  else if (epl <= 4)
    launch_pdl(router_kernel<4>, dim3(blocks), dim3(kRouterChunk * 32), smem, stream, a);
  else
    launch_pdl(router_kernel<8>, dim3(blocks), dim3(kRouterChunk * 32), smem, stream, a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ---------------------------------------------------------------------------
// K0 + K1 fused (bf16 layers on the tensor-mode gate, E <= 64, K <= 16): the
// gate GEMM of a 64-token tile accumulates in TMEM and the same CTA routes
// the tile — the logits never make a round trip through HBM, and the router's
// launch, ramp and tail disappear into the gate kernel.
//   warp 0       TMA producer: x rows (64 x 64 boxes) and gate rows (Epad x
//                64) into a kGrStages-deep ring, one full/empty barrier pair
//                per stage;
//   warp 1       TMEM allocator + tcgen05.mma issuer (M = 128 over a stage
//                whose upper 64 rows are left over from earlier stages: those
//                accumulator rows are never read; N = Epad), two accumulator
//                stages;
//   warps 2..17  two router groups of 8 warps; group g owns accumulator g and
//                the CTA's tiles j = g, g + 2, ...: 4 (Epad 64) / 2 (Epad 32)
//                of its warps drain the accumulator (tcgen05.ld 32x32b.x32,
//                TMEM lanes 0-63) into the group's shared-memory logits tile
//                (and the fp32 logits buffer that LOGITS_REUSE and the logits
//                read-back use), then the 8 warps route 8 tokens each, four
//                lanes per token — quad_route, the arithmetic of
//                router_quad_kernel — and publish the tile's two 32-token
//                chunk histograms (+ their sum into the tile's superchunk).
// 64-token tiles put a CTA on every SM at T = 16384 (256 tiles) and let one
// group route tile j while the producer / MMA already stream tile j + 1 into
// the other accumulator: the routing of all but each CTA's last tile hides
// under the gate's HBM stream.
// The per-call counters (copies kept whole / half, error flags) are reduced
// per CTA, accumulated in acc[0..2], and the last CTA to finish (acc[3]
// counts them) moves them into counters[0..3] and re-zeroes acc: no memset and
// no zeroing race with the atomics of other CTAs.
// ---------------------------------------------------------------------------
#ifndef DSB_GR_TIMES
#define DSB_GR_TIMES 0  // diagnostic builds: CTAs 0, 100, last print their tile timeline (globaltimer, ns)
#endif
__device__ __forceinline__ unsigned long long gr_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int kGrStages = 7;
constexpr int kGrRows = 64;                 // tokens per tile
constexpr int kGrGroupWarps = 8;            // router warps per group (64 tokens x 4 lanes)
constexpr int kGrThreads = (2 + 2 * kGrGroupWarps) * 32;
constexpr int kGrASlot = 128 * 64 * 2;      // the M = 128 MMA reads a whole 128-row slot
constexpr int kGrBSlot = 64 * 64 * 2;
constexpr int kGrChunks = kGrRows / kRouterChunk;

template <int EPAD>
struct GrGeo {
  static constexpr int LGS = EPAD + 4;  // logits tile row stride (floats; 16-byte rows)
  static constexpr int RING = kGrStages * (kGrASlot + kGrBSlot);
  static constexpr int LG = 2 * kGrRows * LGS * 4;          // one logits tile per group
  static constexpr int HIST = 2 * kGrChunks * 128 * 4;      // per group: its tile's chunk histograms (2E <= 128)
  static constexpr int SMEM = 1024 + RING + LG + HIST + 32 * 8 + (2 * kGrStages + 4) * 8 + 64;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
};

struct GateRouteArgs {
  RouterArgs r;
  float* logits_out;         // T x Epad fp32 (row stride Epad), or null
  int epad, nkb, ntiles;
  unsigned long long* acc;   // [n1, nh, err, done] (zero between launches), [4] superchunk epoch
  int* sc;                   // 2 x kScCap x 128 superchunk histograms (buffer = epoch parity), or null
  int sc_chunks;             // 32-token chunks per superchunk (even: a tile never straddles two)
};

__device__ __forceinline__ void group_bar_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kGrGroupWarps * 32) : "memory");
}

template <int EPAD, int EPT, int KK>
__global__ void __launch_bounds__(kGrThreads, 1)
    gate_route_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      const GateRouteArgs g) {
  using G = GrGeo<EPAD>;
  constexpr int NS = kGrStages, LGS = G::LGS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* ringA = smem;
  uint8_t* ringB = smem + NS * kGrASlot;
  float* lg_all = reinterpret_cast<float*>(smem + G::RING);
  int* hist_all = reinterpret_cast<int*>(smem + G::RING + G::LG);
  uint64_t* tab = reinterpret_cast<uint64_t*>(smem + G::RING + G::LG + G::HIST);
  uint64_t* full = tab + 32;
  uint64_t* empty = full + NS;
  uint64_t* tfull = empty + NS;
  uint64_t* tempty = tfull + 2;
  unsigned long long* red = reinterpret_cast<unsigned long long*>(tempty + 2);  // n1, nh, err
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red + 3);
  const RouterArgs& a = g.r;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kLoaders = 2 * (EPAD / 32);  // router warps draining TMEM lanes 0-63, 32 columns each
  const uint32_t tx_bytes = static_cast<uint32_t>(kGrRows * 128 + g.epad * 128);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kLoaders * 32);
    }
    red[0] = red[1] = red[2] = 0ull;
    fence_mbar_init();
    tma_prefetch(&mapA);
    tma_prefetch(&mapB);
  }
  for (int i = threadIdx.x; i < 2 * kGrChunks * 128; i += blockDim.x) hist_all[i] = 0;
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2fTab[threadIdx.x];
  if (warp == 1) {
    tmem_alloc(tmem_slot, 2 * EPAD);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  __shared__ unsigned long long s_gt[8];  // diagnostic timeline: start, [acc ready, routed] x 2 tiles, end
  pdl_wait();     // x / the previous forward's readers of the routing buffers are done
  pdl_trigger();  // the permutation may launch (it waits for this grid to complete)
  if (DSB_GR_TIMES && threadIdx.x == 0) s_gt[0] = gr_now();
  // superchunk epoch: constant for the whole launch (the last CTA advances it
  // only after every CTA has arrived)
  const unsigned long long epoch = g.sc ? *reinterpret_cast<volatile unsigned long long*>(&g.acc[4]) : 0ull;
  if (g.sc) {
    // clear the other superchunk buffer for the next launch, a slice per CTA:
    // its readers (the previous forward's permutation) finished before this
    // grid's griddepcontrol.wait returned
    int4* o = reinterpret_cast<int4*>(g.sc + static_cast<long long>((epoch + 1ull) & 1ull) * kScCap * kScCodes);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kScCap * kScCodes / 4; i += gridDim.x * blockDim.x)
      o[i] = make_int4(0, 0, 0, 0);
  }
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x)
        for (int kb = 0; kb < g.nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
#ifdef DSB_GR_DIAG_NO_B  // diagnostic builds only: gate rows not streamed (wrong logits; timing of the x stream)
          mbar_expect_tx(&full[s], kGrRows * 128);
          tma_load_2d(ringA + s * kGrASlot, &mapA, &full[s], kb * 64, tile * kGrRows);
#else
          mbar_expect_tx(&full[s], tx_bytes);
          tma_load_2d(ringA + s * kGrASlot, &mapA, &full[s], kb * 64, tile * kGrRows);
          tma_load_2d(ringB + s * kGrBSlot, &mapB, &full[s], kb * 64, 0);
#endif
          if (++s == NS) { s = 0; ph ^= 1; }
        }
    }
  } else if (warp == 1) {
    int s = 0, acc = 0;
    uint32_t ph = 0, acc_phase = 0;
    const uint64_t da0 = sdesc_sw128(smem_u32(ringA));
    const uint64_t db0 = sdesc_sw128(smem_u32(ringB));
    const uint32_t idesc = idesc_bf16(128, g.epad);
    for (int tile = blockIdx.x; tile < g.ntiles; tile += gridDim.x) {
      const uint32_t dtmem = tmem_base + acc * EPAD;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < g.nkb; ++kb) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t adesc = da0 + static_cast<uint64_t>(s * (kGrASlot >> 4));
        const uint64_t bdesc = db0 + static_cast<uint64_t>(s * (kGrBSlot >> 4));
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) umma_bf16(dtmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == NS) { s = 0; ph ^= 1; }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else {
    const int rw = warp - 2;                   // router warp 0..15
    const int grp = rw / kGrGroupWarps;        // accumulator / tile parity this warp serves
    const int gw = rw % kGrGroupWarps;         // warp within the group: tokens [8 gw, 8 gw + 8)
    const int quarter = warp & 3;              // TMEM lane quarter this warp may access
    const int cb = gw >> 2;                    // loader: accumulator columns [32 cb, 32 cb + 32)
    const bool loader = quarter < 2 && cb < EPAD / 32;
    const int ncode = 2 * a.E;
    const int nchunks = (a.T + kRouterChunk - 1) / kRouterChunk;
    float* lg = lg_all + grp * kGrRows * LGS;
    int* hist = hist_all + grp * kGrChunks * 128;
    const int gtid = threadIdx.x - 64 - grp * kGrGroupWarps * 32;
    uint32_t acc_phase = 0;
    unsigned long long n1 = 0, nh = 0;
    bool bad = false;
    for (int tile = blockIdx.x + grp * gridDim.x; tile < g.ntiles; tile += 2 * gridDim.x) {
      if (loader) {
        mbar_wait(&tfull[grp], acc_phase);
        tc_fence_after();
        uint32_t v[32];
        tmem_ld32(tmem_base + grp * EPAD + (static_cast<uint32_t>(quarter * 32) << 16) + 32 * cb, v);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&tempty[grp]);
        const int row = quarter * 32 + lane;
        float4* dst = reinterpret_cast<float4*>(lg + row * LGS + 32 * cb);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                               __uint_as_float(v[4 * i + 3]));
        const long long t = static_cast<long long>(tile) * kGrRows + row;
        if (g.logits_out && t < a.T && 32 * cb < g.epad) {
          uint4* o = reinterpret_cast<uint4*>(g.logits_out + t * g.epad + 32 * cb);
#pragma unroll
          for (int i = 0; i < 8; ++i) o[i] = make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
      acc_phase ^= 1;
      group_bar_sync(grp);  // the tile's logits are in shared memory
      const int lt = (tile - blockIdx.x) / gridDim.x;  // this CTA's tile index (diagnostics)
      if (DSB_GR_TIMES && gtid == 0 && lt < 3) s_gt[1 + 2 * lt] = gr_now();
      {
        const int tk = gw * 8 + (lane >> 2);
        const int t = tile * kGrRows + tk;
        const bool tok_ok = t < a.T;
        const int e0 = (lane & 3) * EPT;
        float v[EPT];
        const float* src = lg + tk * LGS + e0;
#pragma unroll
        for (int i = 0; i < EPT; ++i) v[i] = (tok_ok && e0 + i < a.E) ? src[i] : -INFINITY;
#ifndef DSB_GR_DIAG_NO_ROUTE  // diagnostic builds only: the gate phase alone
        bad |= quad_route<EPT, 4, KK>(a, t, tok_ok, v, lane, tab, hist + (gw >> 2) * ncode, n1, nh);
#else
        if (v[0] == 12345.f) bad = true;
        if (tok_ok && (lane & 3) == 0)
          for (int j = 0; j < a.K; ++j) a.sel_code[static_cast<long long>(t) * a.K + j] = -1;
#endif
      }
      group_bar_sync(grp);  // the tile's histograms are complete (and the logits tile is free)
      if (DSB_GR_TIMES && gtid == 0 && lt < 3) s_gt[2 + 2 * lt] = gr_now();
      // per-chunk histograms, and their sum added into the tile's superchunk
      // (the permutation scans superchunks instead of every chunk: no grid-wide
      // barrier there)
      int* scb = g.sc ? g.sc + (static_cast<long long>(epoch & 1ull) * kScCap +
                                (tile * kGrChunks) / g.sc_chunks) * kScCodes
                      : nullptr;
      for (int code = gtid; code < ncode; code += kGrGroupWarps * 32) {
        int sum = 0;
#pragma unroll
        for (int c = 0; c < kGrChunks; ++c) {
          const int chunk = tile * kGrChunks + c;
          const int v = hist[c * ncode + code];
          if (chunk < nchunks) a.cnt_chunk[static_cast<long long>(chunk) * ncode + code] = v;
          sum += v;
          hist[c * ncode + code] = 0;  // the group's next tile counts after its first group_bar_sync
        }
        if (scb && sum) atomicAdd(scb + code, sum);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      n1 += __shfl_xor_sync(0xffffffffu, n1, o);
      nh += __shfl_xor_sync(0xffffffffu, nh, o);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
      if (n1) atomicAdd(&red[0], n1);
      if (nh) atomicAdd(&red[1], nh);
      if (bad) atomicOr(&red[2], 1ull);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (DSB_GR_TIMES && threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 100 || blockIdx.x == gridDim.x - 1)) {
    const unsigned long long t0 = s_gt[0], te = gr_now();
    printf("gate_route cta %d: tile0 acc %llu routed %llu | tile1 acc %llu routed %llu | end %llu ns abs %llu\n",
           blockIdx.x, s_gt[1] - t0, s_gt[2] - t0, s_gt[3] > t0 ? s_gt[3] - t0 : 0ull, s_gt[4] > t0 ? s_gt[4] - t0 : 0ull,
           te - t0, t0);
  }
  if (warp == 1) tmem_dealloc(tmem_base, 2 * EPAD);
  if (threadIdx.x == 0) {
    if (red[0]) atomicAdd(&g.acc[0], red[0]);
    if (red[1]) atomicAdd(&g.acc[1], red[1]);
    if (red[2]) atomicOr(&g.acc[2], red[2]);
    __threadfence();
    if (atomicAdd(&g.acc[3], 1ull) == gridDim.x - 1) {  // last CTA: publish and re-arm
      __threadfence();
      const unsigned long long t1 = atomicExch(&g.acc[0], 0ull);
      const unsigned long long th = atomicExch(&g.acc[1], 0ull);
      const unsigned long long te = atomicExch(&g.acc[2], 0ull);
      a.counters[0] = t1;
      a.counters[1] = th;
      a.counters[2] = te;
      a.counters[3] = 0ull;
      if (te) atomicOr(&a.counters[4], te);
      atomicExch(&g.acc[3], 0ull);
      // every CTA has read the epoch and cleared its slice: advance it
      if (g.sc) *reinterpret_cast<volatile unsigned long long*>(&g.acc[4]) = epoch + 1ull;
    }
  }
}

int gate_route_tile_rows() { return kGrRows; }

int gate_route_sc_chunks(int T) {
  const int nchunks = (T + kRouterChunk - 1) / kRouterChunk;
  // at most kScCap superchunks; >= 16 chunks (512 tokens) each; even
  const int per = (nchunks + kScCap - 1) / kScCap;
  return per <= 16 ? 16 : per + (per & 1);
}

int launch_gate_route(const CUtensorMap* mapA, const CUtensorMap* mapB, const RouterArgs& r, int epad, int nkb,
                      float* logits_out, unsigned long long* acc, int num_sms, cudaStream_t stream, int* sc) {
  if (r.E > 64 || r.K > 16 || r.K < 1 || r.K > r.E || r.nsplit > 1 || (epad != 32 && epad != 64)) return -1;
  const int ntiles = (r.T + kGrRows - 1) / kGrRows;
  if (ntiles <= 0) return 0;
  static_assert(kGrChunks == 2, "superchunks hold whole tiles");
  GateRouteArgs g{r, logits_out, epad, nkb, ntiles, acc, sc, gate_route_sc_chunks(r.T)};
  const int grid = ntiles < num_sms ? ntiles : num_sms;
  cudaError_t err;
#define DSB_GR(EP, EPT, KK)                                                                                  \
  {                                                                                                          \
    set_max_dyn_smem(gate_route_kernel<EP, EPT, KK>, GrGeo<EP>::SMEM);                                       \
    err = launch_pdl(gate_route_kernel<EP, EPT, KK>, dim3(grid), dim3(kGrThreads), GrGeo<EP>::SMEM, stream, \
                     *mapA, *mapB, g);                                                                       \
  }
  if (epad == 32) {
    if (r.K <= 8)
      DSB_GR(32, 8, 8)
    else
      DSB_GR(32, 8, 16)
  } else {
    if (r.K <= 8)
      DSB_GR(64, 16, 8)
    else
      DSB_GR(64, 16, 16)
  }
#undef DSB_GR
  if (err != cudaSuccess) return -2;
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ---------------------------------------------------------------------------
// Caller-supplied RoutingDecision -> forward metadata (moe_forward with an
// explicit routing, moe.hpp:239).  Accepts the canonical layouts route_tokens /
// replay_routing / apply_bands produce: copy cp of selection s at slot cp*K+s
// with index (e/P)*P+cp, copies >= 1 sharing one fraction, copy 0 kept whenever
// any copy is, equal raw scores across copies; P == 1 allows fraction 0.5.
// Anything else sets error bit 2 (the host reports invalid_state).
// One block per 128-token chunk, one thread per token.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRouterChunk) import_routing_kernel(const ImportArgs a) {
  extern __shared__ int s_hist[];
  for (int i = threadIdx.x; i < 2 * a.nunits; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const int t = blockIdx.x * kRouterChunk + threadIdx.x;
  if (t < a.T) {
    const long long kp = static_cast<long long>(a.K) * a.P;
    for (int s = 0; s < a.K; ++s) {
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
        atomicOr(&a.counters[4], 4ull);
        lv = 0;
      }
      const int unit = ok ? e0 / a.P : 0;
      const long long g = static_cast<long long>(t) * a.K + s;
      a.sel_code[g] = lv > 0 ? unit * 4 + lv : -1;
      a.sel_raw[g] = static_cast<float>(r0);
      if (lv > 0) atomicAdd(&s_hist[2 * unit + (lv == 2 ? 0 : 1)], 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * a.nunits; i += blockDim.x)
    a.cnt_chunk[static_cast<long long>(blockIdx.x) * 2 * a.nunits + i] = s_hist[i];
}

int launch_import_routing(const ImportArgs& a, cudaStream_t stream) {
  const int blocks = (a.T + kRouterChunk - 1) / kRouterChunk;
  if (blocks > 0)
    import_routing_kernel<<<blocks, kRouterChunk, static_cast<size_t>(2 * a.nunits) * sizeof(int), stream>>>(a);
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

namespace dsb {

// ---------------------------------------------------------------------------
// analyze_gating (dropping.hpp:207-228) histograms on the device: per
// original selection (copy 0 of the replayed routing) the selected expert
// count, and uniform-bin histograms of the raw and the normalized scores,
// bin = clamp(int(v * bins), 0, bins - 1) with the product in double.
// ---------------------------------------------------------------------------
__global__ void gating_hist_kernel(const int32_t* __restrict__ idx, const float* __restrict__ raw,
                                   const double* __restrict__ norm, int T, int K, int P, int E, int bins,
                                   unsigned long long* __restrict__ counts, unsigned long long* __restrict__ rh,
                                   unsigned long long* __restrict__ nh) {
  extern __shared__ unsigned int sh[];  // E + 2 * bins
  unsigned int* sc = sh;
  unsigned int* sr = sh + E;
  unsigned int* sn = sr + bins;
  for (int i = threadIdx.x; i < E + 2 * bins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const long long n = static_cast<long long>(T) * K;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long t = i / K, s = i - t * K;
    const long long f = t * K * P + s;
    atomicAdd(&sc[idx[f] / P], 1u);
    const int br = static_cast<int>(__dmul_rn(static_cast<double>(raw[f]), static_cast<double>(bins)));
    const int bn = static_cast<int>(__dmul_rn(norm[f], static_cast<double>(bins)));
    atomicAdd(&sr[min(max(br, 0), bins - 1)], 1u);
    atomicAdd(&sn[min(max(bn, 0), bins - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x)
    if (sc[i]) atomicAdd(&counts[i], static_cast<unsigned long long>(sc[i]));
  for (int i = threadIdx.x; i < bins; i += blockDim.x) {
    if (sr[i]) atomicAdd(&rh[i], static_cast<unsigned long long>(sr[i]));
    if (sn[i]) atomicAdd(&nh[i], static_cast<unsigned long long>(sn[i]));
  }
}

int launch_gating_hist(const int32_t* idx, const float* raw, const double* norm, int T, int K, int P, int E,
                       int bins, unsigned long long* counts, unsigned long long* rh, unsigned long long* nh,
                       int num_sms, cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(E + 2 * bins) * sizeof(unsigned int);
  if (smem > 48 * 1024) return -1;
  gating_hist_kernel<<<num_sms, 256, smem, stream>>>(idx, raw, norm, T, K, P, E, bins, counts, rh, nh);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ---------------------------------------------------------------------------
// Rate-targeted drop on the device (north star item 2, "rate-based drop
// mask"; the reference has thresholds only, and its tests reach a rate by
// bisecting the threshold, acceptance.cpp:342-352).  Input: the normalized
// scores ns of a no-drop routing (copy 0 of every selection, T x K) — the
// band decision of drop_1t / drop_2t depends on nothing else
// (dropping.hpp:93-122).  The kernel replays the host bisection exactly:
//   t = 0.5 (lo + hi); rate = drop_stats(...).drop_rate under one_t(t) /
//   two_t_from(t) (2T band t -/+ 0.01 in double); keep the closest; stop
//   when |rate - target| <= tol; rate < target ? lo = t : hi = t.
// The drop rate of a candidate t is exact: retained copies are integer
// counts (P a power of two; stats_from_counts' arithmetic).  Every thread
// holds one selection's ns in a register across iterations; per iteration
// the grid counts kept copies and one grid barrier separates the rounds
// (iteration-indexed counters, so nothing is reset).  Output: t and its rate,
// and t_unit[e] = t for every expert — the threshold table the router applies
// in its second pass without a host round trip.
// ---------------------------------------------------------------------------
struct RateArgs {
  const double* norm;   // T x (K*P), copy-major: slot s of copy 0 at [t*K*P + s]
  int T, K, P, S;
  int two_t, keep_top1;
  double target, tol;
  int iters;
  unsigned long long* cnt;  // iters x 2 (copies kept at fraction 1, at 0.5); zeroed by the host
  double* t_unit;           // E
  int E;
  double* result;           // [t, rate]
};

__global__ void __launch_bounds__(1024) rate_calibrate_kernel(const RateArgs a) {
  namespace cg = cooperative_groups;
  __shared__ unsigned long long s1, sh;
  __shared__ double s_lo, s_hi, s_best_t, s_best_r;
  __shared__ int s_done;
  const long long n = static_cast<long long>(a.T) * a.K;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long g0 = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  constexpr int kPer = 4;  // selections per thread held in registers (T*K <= 4 x grid threads)
  double ns[kPer];
  bool top[kPer], live[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const long long g = g0 + i * stride;
    live[i] = g < n;
    ns[i] = 0.0;
    top[i] = false;
    if (live[i]) {
      const long long t = g / a.K;
      const int s = static_cast<int>(g - t * a.K);
      const double* row = a.norm + t * a.K * a.P;
      ns[i] = row[s];
      bool first_max = true;  // top_slot: the first strict maximum of ns (dropping.hpp:99)
      for (int j = 0; j < a.K; ++j) {
        if (j < s && !(ns[i] > row[j])) first_max = false;
        if (j > s && row[j] > ns[i]) first_max = false;
      }
      top[i] = first_max;
    }
  }
  const long long ncopies = n * a.P;
  const double w = 1.0 / a.P;
  const double total = __dmul_rn(static_cast<double>(ncopies), w);
  const double denom = __dadd_rn(total, static_cast<double>(a.S) * a.T);
  if (threadIdx.x == 0) {
    s_lo = 0.0;
    s_hi = 1.0;
    s_best_t = 0.0;
    s_best_r = -1.0;
    s_done = 0;
  }
  __syncthreads();
  for (int it = 0; it < a.iters; ++it) {
    const double t = __dmul_rn(0.5, __dadd_rn(s_lo, s_hi));
    const double tmaj = a.two_t ? __dsub_rn(t, 0.01) : t;
    const double tmin = a.two_t ? __dadd_rn(t, 0.01) : t;
    unsigned long long c1 = 0, ch = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      if (!live[i]) continue;
      int lv = ns[i] >= tmin ? 2 : (ns[i] >= tmaj ? 1 : 0);
      if (a.keep_top1 && top[i]) lv = 2;
      if (a.P == 1) {
        c1 += lv == 2;
        ch += lv == 1;
      } else {  // full: every copy at fraction 1; major-only: copy 0 at fraction 1
        c1 += lv == 2 ? a.P : (lv == 1 ? 1 : 0);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      ch += __shfl_xor_sync(0xffffffffu, ch, o);
    }
    if (threadIdx.x == 0) {
      s1 = 0;
      sh = 0;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && (c1 | ch)) {
      atomicAdd(&s1, c1);
      atomicAdd(&sh, ch);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(&a.cnt[2 * it], s1);
      atomicAdd(&a.cnt[2 * it + 1], sh);
    }
    cg::this_grid().sync();
    if (threadIdx.x == 0) {  // every block derives the same next step from the same totals
      const unsigned long long n1 = atomicAdd(&a.cnt[2 * it], 0ull), nh = atomicAdd(&a.cnt[2 * it + 1], 0ull);
      const double retained = __dmul_rn(static_cast<double>(2 * n1 + nh), __dmul_rn(0.5, w));
      const double dropped = __dsub_rn(total, retained);
      const double rate = denom > 0.0 ? __ddiv_rn(dropped, denom) : 0.0;
      const double err = fabs(__dsub_rn(rate, a.target));
      if (s_best_r < 0.0 || err < fabs(__dsub_rn(s_best_r, a.target))) {
        s_best_t = t;
        s_best_r = rate;
      }
      if (err <= a.tol) {
        s_done = 1;
      } else if (rate < a.target) {
        s_lo = t;
      } else {
        s_hi = t;
      }
    }
    __syncthreads();
    if (s_done) break;
  }
  if (blockIdx.x == 0) {
    for (int e = threadIdx.x; e < a.E; e += blockDim.x) a.t_unit[e] = s_best_t;
    if (threadIdx.x == 0) {
      a.result[0] = s_best_t;
      a.result[1] = s_best_r;
    }
  }
}

int launch_rate_calibrate(const double* norm, int T, int K, int P, int S, int two_t, int keep_top1, double target,
                          double tol, int iters, unsigned long long* cnt, double* t_unit, int E, double* result,
                          int num_sms, cudaStream_t stream) {
  if (P < 1 || (P & (P - 1)) != 0 || iters < 1) return -1;
  RateArgs a{norm, T, K, P, S, two_t, keep_top1, target, tol, iters, cnt, t_unit, E, result};
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rate_calibrate_kernel, 1024, 0);
  if (per_sm < 1) return -3;
  const long long n = static_cast<long long>(T) * K;
  const long long need = (n + 4 * 1024 - 1) / (4 * 1024);
  if (need > static_cast<long long>(num_sms) * per_sm) return -1;  // > 4 selections per thread
  const int grid = static_cast<int>(need < 1 ? 1 : need);
  void* args[] = {&a};
  const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(rate_calibrate_kernel), dim3(grid),
                                                    dim3(1024), args, 0, stream);
  return e == cudaSuccess ? 0 : -2;
}

}  // namespace dsb
