// Micro-benchmark: where the latency of one quad_route call goes (E = 64,
// K = 8, P = 2, 2T): 8 warps route 64 tokens from shared memory, like one
// router group of gate_route_kernel; clock64 stamps between the phases of an
// instrumented copy of quad_route (warp 0's view), plus the same with 1 warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false tools/micro/route_phases.cu -o tools/micro/route_phases
#include <cstdio>
#include <vector>
#include "../../paper_2508_18376_b200/csrc/router.cu"
using namespace dsb;
namespace dsb {
cudaError_t set_max_dyn_smem(const void* func, size_t bytes) {  // (the library's per-device version lives in capi.cpp)
  return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}
template <int EPT, int LPT, int KK>
__device__ __forceinline__ bool quad_route_timed(const RouterArgs& a, int t, bool tok_ok, float (&v)[EPT], int lane,
                                           const uint64_t* tab, int* s_hist, unsigned long long& n1,
                                           unsigned long long& nh, long long* tstamp) {
  constexpr int NS = KK > EPT ? KK : EPT;  // keys sorted per lane (padded with 0 = "no expert")
  const int E = a.E, K = a.K, P = a.P;
  const int q = lane % LPT, qbase = lane - q;
  const int e0 = q * EPT;
  bool bad = false;
  if (tstamp) { __syncwarp(); tstamp[0] = clock64(); }
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
  if (tstamp) { __syncwarp(); tstamp[1] = clock64(); }
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
  if (tstamp) { __syncwarp(); tstamp[2] = clock64(); }
  for (int i = 0; i < EPT; ++i) v[i] = __fdiv_rn(v[i], sum);
  if (tstamp) { __syncwarp(); tstamp[3] = clock64(); }
  // topk_route (moe.hpp:193-205) as a key sort
  unsigned long long key[NS];
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    const int e = e0 + i;
    key[i] = (i < EPT && e < E) ? (static_cast<unsigned long long>(__float_as_uint(v[i < EPT ? i : 0])) << 32) |
                                      static_cast<unsigned long long>(0xFFFFFFFFu - static_cast<unsigned>(e))
                                : 0ull;
  }
  if (tstamp) { __syncwarp(); tstamp[4] = clock64(); }
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
  if (tstamp) { __syncwarp(); tstamp[5] = clock64(); }
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
  if (tstamp) { __syncwarp(); tstamp[6] = clock64(); }
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
  if (tstamp) { __syncwarp(); tstamp[7] = clock64(); }
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
  if (tstamp) { __syncwarp(); tstamp[8] = clock64(); }
  return bad;
}

}  // namespace dsb

template <int NW>
__global__ void phases_kernel(const float* lg, RouterArgs a, long long* out) {
  __shared__ uint64_t tab[32];
  __shared__ int hist[256];
  __shared__ float s_lg[64 * 68];
  if (threadIdx.x < 32) tab[threadIdx.x] = kExp2fTab[threadIdx.x];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) s_lg[(i / 64) * 68 + i % 64] = lg[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long ts[9];
  unsigned long long n1 = 0, nh = 0;
  bool bad = false;
  const long long t0 = clock64();
  for (int rep = 0; rep < 8 / NW; ++rep) {  // NW warps cover the 64 tokens
    const int tk = (rep * NW + warp) * 8 + (lane >> 2);
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = s_lg[tk * 68 + (lane & 3) * 16 + i];
    bad |= quad_route_timed<16, 4, 8>(a, tk, true, v, lane, tab, hist, n1, nh, warp == 0 && rep == 0 ? ts : nullptr);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 9; ++i) out[i] = ts[i] - t0;
    out[9] = t1 - t0;
    out[10] = bad + n1 + nh;
  }
}

int main() {
  const int T = 64, E = 64, K = 8, P = 2;
  std::vector<float> h(T * E);
  for (size_t i = 0; i < h.size(); ++i) h[i] = float((i * 2654435761u) % 1000) * 0.004f - 2.f;
  float* lg; cudaMalloc(&lg, h.size() * 4); cudaMemcpy(lg, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  int32_t* sel_code; float* sel_raw; cudaMalloc(&sel_code, T * K * 4); cudaMalloc(&sel_raw, T * K * 4);
  long long* out; cudaMalloc(&out, 16 * 8);
  RouterArgs a{};
  a.T = T; a.E = E; a.K = K; a.P = P; a.kind = 2; a.t_major = 0.07; a.t_minor = 0.09; a.keep_top1 = 1; a.normalize = 1;
  a.sel_code = sel_code; a.sel_raw = sel_raw;
  const char* names[9] = {"start", "max", "expf", "div", "keys", "lane sort", "merges", "normalize", "bands+writes"};
  for (int nw : {8, 1}) {
    for (int it = 0; it < 3; ++it) {
      if (nw == 8) phases_kernel<8><<<1, 256>>>(lg, a, out); else phases_kernel<1><<<1, 32>>>(lg, a, out);
      cudaDeviceSynchronize();
    }
    long long o[11];
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("%d warp(s) (%s):", nw, cudaGetErrorString(cudaGetLastError()));
    for (int i = 1; i < 9; ++i) printf("  %s %lld", names[i], o[i] - o[i - 1]);
    printf("  | warp 0 call %lld cycles, all 64 tokens %lld cycles\n", o[8] - o[0], o[9]);
  }
  return 0;
}
