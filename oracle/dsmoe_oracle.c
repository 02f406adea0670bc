/* TEST INFRASTRUCTURE ONLY — see dsmoe_oracle.h.  Each function cites the
 * reference file:line (under /root/reference/proj) whose arithmetic it
 * restates.  Compiled with -ffp-contract=off and without fast-math so every
 * float/double operation rounds exactly where the reference's does. */
#include "dsmoe_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { ST_OK = 0, ST_INVALID_ARGUMENT = 1, ST_SHAPE = 2, ST_INVALID_STATE = 3, ST_INTERNAL = 8 };

/* ---------------------------------------------------------------- rng.hpp */

typedef struct { uint64_t s[4]; } xoshiro;

static uint64_t splitmix_next(uint64_t* state) { /* rng.hpp:19-24 */
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_splitmix_nth(uint64_t seed, int n) { /* io.cpp:358-364: layer seeds */
  uint64_t st = seed, v = 0;
  for (int i = 0; i <= n; ++i) v = splitmix_next(&st);
  return v;
}

static void xo_seed(xoshiro* x, uint64_t seed) { /* rng.hpp:32-35 */
  uint64_t st = seed;
  for (int i = 0; i < 4; ++i) x->s[i] = splitmix_next(&st);
}

static inline uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static inline uint64_t xo_next(xoshiro* x) { /* rng.hpp:37-47 */
  uint64_t* s = x->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

static inline double xo_gauss(xoshiro* x) { /* rng.hpp:50-57: Irwin-Hall */
  double acc = 0.0;
  for (int i = 0; i < 12; ++i) acc += (double)(xo_next(x) >> 11) * 0x1.0p-53;
  return acc - 6.0;
}

int orc_generate_layer(int d, int ffn, int E, int S, uint64_t seed, double scale, float* flat) {
  /* generate_synthetic, io.cpp:330-356 */
  if (d < 1 || ffn < 2 || E < 1 || S < 0) return ST_INVALID_ARGUMENT;
  xoshiro rng;
  xo_seed(&rng, seed);
  const double sd = scale / sqrt((double)d);
  const size_t n = (size_t)d * E + (size_t)(E + S) * 3 * (size_t)d * ffn;
  for (size_t i = 0; i < n; ++i) flat[i] = (float)(xo_gauss(&rng) * sd);
  return ST_OK;
}

int orc_generate_tokens(int64_t rows, int cols, uint64_t seed, double scale, float* out) {
  /* generate_tokens, io.cpp:368-374 */
  if (rows < 1 || cols < 1) return ST_INVALID_ARGUMENT;
  xoshiro rng;
  xo_seed(&rng, seed);
  for (size_t i = 0; i < (size_t)rows * cols; ++i) out[i] = (float)(xo_gauss(&rng) * scale);
  return ST_OK;
}

/* ------------------------------------------------------------- matrix.hpp */

void orc_gate_logits(const float* x, const float* gate, int T, int d, int E, float* logits) {
  /* matmul i-k-j, matrix.hpp:47-64: out starts at +0, += a_ik * b_kj for
   * ascending k (FMUL then FADD; contraction is off). */
  for (int t = 0; t < T; ++t) {
    float* o = logits + (size_t)t * E;
    for (int e = 0; e < E; ++e) o[e] = 0.0f;
    const float* xr = x + (size_t)t * d;
    for (int k = 0; k < d; ++k) {
      const float a = xr[k];
      const float* g = gate + (size_t)k * E;
      for (int e = 0; e < E; ++e) o[e] += a * g[e];
    }
  }
}

static void softmax_row(float* v, int E) { /* matrix.hpp:68-78 */
  float mx = v[0];
  for (int e = 0; e < E; ++e) mx = (mx < v[e]) ? v[e] : mx; /* std::max(mx, x) */
  float sum = 0.0f;
  for (int e = 0; e < E; ++e) {
    v[e] = expf(v[e] - mx);
    sum += v[e];
  }
  for (int e = 0; e < E; ++e) v[e] /= sum;
}

void orc_softmax_rows(float* s, int T, int E) {
  for (int t = 0; t < T; ++t) softmax_row(s + (size_t)t * E, E);
}

static inline float swishf(float x) { return x / (1.0f + expf(-x)); } /* matrix.hpp:88-92 */

/* ------------------------------------------------------- moe.hpp / dropping */

/* topk_route, moe.hpp:181-206: K argmax rounds, strict >, lower index wins
 * ties; raw = (double)score.  scores is one row of E floats. */
static void topk_row(const float* row, int E, int K, char* taken, int32_t* sel, double* sraw) {
  memset(taken, 0, (size_t)E);
  for (int j = 0; j < K; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e)
      if (!taken[e] && (best < 0 || row[e] > row[best])) best = e;
    taken[best] = 1;
    sel[j] = best;
    sraw[j] = (double)row[best];
  }
}

int orc_topk(const float* scores, int T, int E, int K, int32_t* idx, double* raw) {
  if (K < 1 || K > E) return ST_INVALID_ARGUMENT; /* moe.hpp:182-184 */
  char* taken = (char*)malloc((size_t)E);
  for (int t = 0; t < T; ++t)
    topk_row(scores + (size_t)t * E, E, K, taken, idx + (size_t)t * K, raw + (size_t)t * K);
  free(taken);
  return ST_OK;
}

/* normalize_topk, dropping.hpp:60-72: per token, sum of the first base_k raw
 * scores in slot order (double), then raw/sum for all K*P slots. */
int orc_normalize(const double* raw, int T, int K, int P, double* norm) {
  const int k = K * P;
  for (int t = 0; t < T; ++t) {
    const double* r = raw + (size_t)t * k;
    double sum = 0.0;
    for (int j = 0; j < K; ++j) sum += r[j];
    if (!(sum > 0.0)) return ST_INVALID_ARGUMENT;
    for (int j = 0; j < k; ++j) norm[(size_t)t * k + j] = r[j] / sum;
  }
  return ST_OK;
}

/* apply_bands_fn, dropping.hpp:93-122, on copy-major T x K*P normalized
 * scores.  Thresholds per original selection when the *_slot arrays are
 * given (ep_sim.hpp:139-149), else the scalars. */
void orc_apply_bands(const double* norm, int T, int K, int P, double t_major, double t_minor,
                     const double* t_major_slot, const double* t_minor_slot, int keep_top1,
                     double* frac) {
  const int k = K * P;
  for (int t = 0; t < T; ++t) {
    const size_t base = (size_t)t * k;
    int top_slot = 0;
    for (int s = 0; s < K; ++s) {
      const double ns = norm[base + s];
      if (ns > norm[base + top_slot]) top_slot = s;
      const double tmin = t_minor_slot ? t_minor_slot[(size_t)t * K + s] : t_minor;
      const double tmaj = t_major_slot ? t_major_slot[(size_t)t * K + s] : t_major;
      if (ns >= tmin) {
        for (int cp = 0; cp < P; ++cp) frac[base + (size_t)cp * K + s] = 1.0;
      } else if (ns >= tmaj) {
        if (P == 1) {
          frac[base + s] = 0.5;
        } else {
          frac[base + s] = 1.0;
          for (int cp = 1; cp < P; ++cp) frac[base + (size_t)cp * K + s] = 0.0;
        }
      } else {
        for (int cp = 0; cp < P; ++cp) frac[base + (size_t)cp * K + s] = 0.0;
      }
    }
    if (keep_top1)
      for (int cp = 0; cp < P; ++cp) frac[base + (size_t)cp * K + top_slot] = 1.0;
  }
}

/* Routing on caller logits = the routing half of route_and_drop
 * (dropping.hpp:248-258): softmax_inplace per row, topk_route, replay_routing
 * (moe.hpp:277-309, copy-major cp*K+s, index e*P+cp), ensure_normalized,
 * drop_1t / drop_2t. */
int orc_route_from_logits(const float* logits, int T, int E, int K, int P, int kind, double t_drop,
                          double t_major, double t_minor, int keep_top1, int normalize,
                          const double* t_major_slot, const double* t_minor_slot, int32_t* idx,
                          double* raw, double* norm, double* frac, double* pre_frac) {
  if (K < 1 || K > E) return ST_INVALID_ARGUMENT; /* moe.hpp:182-184 */
  if (P < 1) return ST_INVALID_ARGUMENT;
  if (kind == ORC_2T) {
    if (!(t_major <= t_minor)) return ST_INVALID_ARGUMENT; /* dropping.hpp:145-146 */
    if (P != 2) return ST_INVALID_STATE;                   /* dropping.hpp:147-148 */
  }
  if (kind == ORC_1T) t_major = t_minor = t_drop; /* drop_1t, dropping.hpp:136 */
  const int k = K * P;
  float* row = (float*)malloc(sizeof(float) * (size_t)E);
  char* taken = (char*)malloc((size_t)E);
  int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * (size_t)K);
  double* sraw = (double*)malloc(sizeof(double) * (size_t)K);
  for (int t = 0; t < T; ++t) {
    memcpy(row, logits + (size_t)t * E, sizeof(float) * (size_t)E);
    softmax_row(row, E);
    topk_row(row, E, K, taken, sel, sraw);
    const size_t base = (size_t)t * k;
    for (int cp = 0; cp < P; ++cp)
      for (int s = 0; s < K; ++s) {
        const size_t f = base + (size_t)cp * K + s;
        idx[f] = sel[s] * P + cp;
        raw[f] = sraw[s];
        frac[f] = 1.0;
        if (pre_frac) pre_frac[f] = 1.0;
      }
  }
  free(row);
  free(taken);
  free(sel);
  free(sraw);
  int st = ST_OK;
  if (normalize) {
    st = orc_normalize(raw, T, K, P, norm);
  } else {
    memcpy(norm, raw, sizeof(double) * (size_t)T * k);
  }
  if (st != ST_OK || kind == ORC_NONE) return st;
  orc_apply_bands(norm, T, K, P, t_major, t_minor, t_major_slot, t_minor_slot, keep_top1, frac);
  return ST_OK;
}

void orc_drop_stats(const double* pre_frac, const double* post_frac, int64_t n, int P, int S,
                    int64_t T, int d, int ffn, double* out7) {
  /* dropping.hpp:176-194 */
  const double w = 1.0 / P;
  double total = 0.0, retained = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    total += pre_frac[i] * w;
    retained += post_frac[i] * w;
  }
  const double dropped = total - retained;
  const double shared = (double)S * (double)T;
  const double denom = total + shared;
  const double unit = 6.0 * d * ffn;
  out7[0] = total;
  out7[1] = dropped;
  out7[2] = shared;
  out7[3] = denom > 0.0 ? dropped / denom : 0.0;
  out7[4] = denom * unit;
  out7[5] = dropped * unit;
  out7[6] = out7[4] - out7[5];
}

/* accumulate_block, moe.hpp:213-231.  g_n and u_n are each a serial float
 * sum over ascending kk; iterating kk outer / n inner performs exactly the
 * same additions per n (in the same order) while keeping rows contiguous. */
static void accumulate_block(const float* xr, int d, const float* w1, const float* w3,
                             const float* w2, int width, float weight, int active, float* g,
                             float* u, float* out_row) {
  for (int n = 0; n < active; ++n) g[n] = u[n] = 0.0f;
  for (int kk = 0; kk < d; ++kk) {
    const float xv = xr[kk];
    const float* r1 = w1 + (size_t)kk * width;
    const float* r3 = w3 + (size_t)kk * width;
    for (int n = 0; n < active; ++n) {
      g[n] += xv * r1[n];
      u[n] += xv * r3[n];
    }
  }
  for (int n = 0; n < active; ++n) {
    const float hn = (swishf(g[n]) * u[n]) * weight;
    const float* r2 = w2 + (size_t)n * d;
    for (int j = 0; j < d; ++j) out_row[j] += hn * r2[j];
  }
}

int orc_moe_forward(const float* x, int T, int d, int nblocks, int kslots,
                    const float* const* w1, const float* const* w3, const float* const* w2,
                    const int32_t* widths, int S, const float* const* sw1,
                    const float* const* sw3, const float* const* sw2, const int32_t* swidths,
                    const int32_t* idx, const double* raw, const double* frac, float* out) {
  /* moe_forward, moe.hpp:239-271 */
  int wmax = 1;
  for (int b = 0; b < nblocks; ++b) wmax = widths[b] > wmax ? widths[b] : wmax;
  for (int s = 0; s < S; ++s) wmax = swidths[s] > wmax ? swidths[s] : wmax;
  float* g = (float*)malloc(sizeof(float) * (size_t)wmax);
  float* u = (float*)malloc(sizeof(float) * (size_t)wmax);
  int st = ST_OK;
  for (int t = 0; t < T && st == ST_OK; ++t) {
    const float* xr = x + (size_t)t * d;
    float* orow = out + (size_t)t * d;
    for (int j = 0; j < d; ++j) orow[j] = 0.0f;
    for (int j = 0; j < kslots; ++j) {
      const size_t f = (size_t)t * kslots + j;
      const double fr = frac[f];
      if (fr == 0.0) continue;
      const int e = idx[f];
      if (e < 0 || e >= nblocks) { st = ST_INVALID_STATE; break; }
      const int w = widths[e];
      const int active = fr == 0.5 ? (w + 1) / 2 : w;
      accumulate_block(xr, d, w1[e], w3[e], w2[e], w, (float)raw[f], active, g, u, orow);
    }
    for (int s = 0; s < S && st == ST_OK; ++s)
      accumulate_block(xr, d, sw1[s], sw3[s], sw2[s], swidths[s], 1.0f, swidths[s], g, u, orow);
  }
  free(g);
  free(u);
  return st;
}

/* ---------------------------------------------------------- reconstruct.hpp */

int orc_profile_importance(const float* x, int T, int d, int E, int ffn, int K,
                           const float* const* w1, const float* const* w3, const int32_t* idx,
                           int metric, double* values) {
  /* reconstruct.hpp:99-149 */
  if (T < 1) return ST_INVALID_ARGUMENT;
  if (metric < 0 || metric > 3) return ST_INVALID_ARGUMENT;
  const int need_u = metric >= 2;
  float* g = (float*)malloc(sizeof(float) * (size_t)ffn);
  float* u = (float*)malloc(sizeof(float) * (size_t)ffn);
  memset(values, 0, sizeof(double) * (size_t)E * ffn);
  int st = ST_OK;
  for (int t = 0; t < T && st == ST_OK; ++t) {
    const float* xr = x + (size_t)t * d;
    for (int j = 0; j < K; ++j) {
      const int e = idx[(size_t)t * K + j];
      if (e < 0 || e >= E) { st = ST_INVALID_STATE; break; }
      for (int n = 0; n < ffn; ++n) g[n] = u[n] = 0.0f;
      for (int kk = 0; kk < d; ++kk) {
        const float xv = xr[kk];
        const float* r1 = w1[e] + (size_t)kk * ffn;
        for (int n = 0; n < ffn; ++n) g[n] += xv * r1[n];
        if (need_u) {
          const float* r3 = w3[e] + (size_t)kk * ffn;
          for (int n = 0; n < ffn; ++n) u[n] += xv * r3[n];
        }
      }
      double* acc = values + (size_t)e * ffn;
      for (int n = 0; n < ffn; ++n) {
        const double sg = (double)swishf(g[n]);
        double v = 0.0;
        switch (metric) {
          case 0: v = sg; break;
          case 1: v = fabs(sg); break;
          case 2: v = sg * (double)u[n]; break;
          case 3: v = fabs(sg * (double)u[n]); break;
        }
        acc[n] += v;
      }
    }
  }
  free(g);
  free(u);
  return st;
}

void orc_reconstruction_order(const double* values, int E, int ffn, int32_t* order) {
  /* build_reconstruction_map, reconstruct.hpp:151-168: std::stable_sort of
   * iota by imp[a] > imp[b].  Bottom-up merge sort: takes from the right run
   * only when strictly greater, so equal keys keep ascending index order. */
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)ffn);
  for (int e = 0; e < E; ++e) {
    const double* imp = values + (size_t)e * ffn;
    int32_t* a = order + (size_t)e * ffn;
    for (int n = 0; n < ffn; ++n) a[n] = n;
    for (int width = 1; width < ffn; width *= 2) {
      for (int lo = 0; lo < ffn; lo += 2 * width) {
        int mid = lo + width < ffn ? lo + width : ffn;
        int hi = lo + 2 * width < ffn ? lo + 2 * width : ffn;
        int i = lo, j = mid, o = lo;
        while (i < mid && j < hi) tmp[o++] = (imp[a[j]] > imp[a[i]]) ? a[j++] : a[i++];
        while (i < mid) tmp[o++] = a[i++];
        while (j < hi) tmp[o++] = a[j++];
      }
      memcpy(a, tmp, sizeof(int32_t) * (size_t)ffn);
    }
  }
  free(tmp);
}

/* ------------------------------------------------------------------ ep_sim */

int orc_place_experts(int num_experts, int devices, int round_robin, int32_t* device_of) {
  /* ep_sim.hpp:38-54 */
  if (!(devices >= 1 && num_experts >= devices)) return ST_INVALID_ARGUMENT;
  if (round_robin) {
    for (int e = 0; e < num_experts; ++e) device_of[e] = e % devices;
  } else {
    if (num_experts % devices != 0) return ST_INVALID_ARGUMENT;
    const int chunk = num_experts / devices;
    for (int e = 0; e < num_experts; ++e) device_of[e] = e / chunk;
  }
  return ST_OK;
}

void orc_device_loads(const int32_t* idx, const double* frac, int64_t n, int P,
                      const int32_t* device_of, int D, double* loads) {
  /* ep_sim.hpp:59-72 */
  const double w = 1.0 / P;
  for (int d = 0; d < D; ++d) loads[d] = 0.0;
  for (int64_t i = 0; i < n; ++i) loads[device_of[idx[i]]] += frac[i] * w;
}

int orc_load_aware_thresholds(const double* loads, int D, double t_max, double* out) {
  /* ep_sim.hpp:76-89 */
  if (!(t_max > 0.0 && t_max <= 1.0)) return ST_INVALID_ARGUMENT;
  double total = 0.0;
  for (int d = 0; d < D; ++d) total += loads[d];
  if (!(total > 0.0)) return ST_INVALID_ARGUMENT;
  const double ideal = total / (double)D;
  for (int d = 0; d < D; ++d) {
    const double ratio = loads[d] / ideal;
    out[d] = ratio >= 1.0 ? t_max : t_max * ratio;
  }
  return ST_OK;
}

int orc_simulate_step(const float* logits, int T, int E, int K, int P, int S, int d, int ffn,
                      int devices, int round_robin, int kind, double t_drop, double t_major,
                      double t_minor, int keep_top1, int normalize, int load_aware,
                      double* pre_loads, double* post_loads, double* thresholds, double* rep5,
                      int32_t* idx, double* frac) {
  /* ep_sim.hpp:110-160 */
  if (kind == ORC_2T && P != 2) return ST_INVALID_STATE;
  const int nphys = E * P, k = K * P;
  const size_t n = (size_t)T * k;
  int32_t* dev = (int32_t*)malloc(sizeof(int32_t) * (size_t)nphys);
  double* raw = (double*)malloc(sizeof(double) * n);
  double* norm = (double*)malloc(sizeof(double) * n);
  double* pre = (double*)malloc(sizeof(double) * n);
  double* tmaj = (double*)malloc(sizeof(double) * (size_t)T * K);
  double* tmin = (double*)malloc(sizeof(double) * (size_t)T * K);
  int st = orc_place_experts(nphys, devices, round_robin, dev);
  if (st == ST_OK)
    st = orc_route_from_logits(logits, T, E, K, P, ORC_NONE, 0, 0, 0, 0, normalize, NULL, NULL,
                               idx, raw, norm, pre, NULL);
  if (st == ST_OK) {
    orc_device_loads(idx, pre, (int64_t)n, P, dev, devices, pre_loads);
    double total = 0.0;
    for (int i = 0; i < devices; ++i) total += pre_loads[i];
    rep5[0] = total / devices;
    if (kind == ORC_NONE) {
      for (int i = 0; i < devices; ++i) thresholds[i] = 0.0;
      memcpy(frac, pre, sizeof(double) * n);
    } else {
      if (load_aware) {
        st = orc_load_aware_thresholds(pre_loads, devices, t_drop, thresholds);
      } else {
        for (int i = 0; i < devices; ++i) thresholds[i] = t_drop;
      }
      const double maj_off = kind == ORC_2T ? t_major - t_drop : 0.0;
      const double min_off = kind == ORC_2T ? t_minor - t_drop : 0.0;
      for (int t = 0; t < T && st == ST_OK; ++t)
        for (int s = 0; s < K; ++s) {
          const double own = thresholds[dev[idx[(size_t)t * k + s]]];
          tmaj[(size_t)t * K + s] = own + maj_off;
          tmin[(size_t)t * K + s] = own + min_off;
        }
      if (st == ST_OK) {
        /* apply_bands_fn on the normalized pre routing; 2T offsets are
         * already folded into the per-slot thresholds.  Route as 1T so the
         * P==2 check of drop_2t does not fire twice. */
        st = orc_route_from_logits(logits, T, E, K, P, ORC_1T, 0, 0, 0, keep_top1, normalize,
                                   tmaj, tmin, idx, raw, norm, frac, NULL);
      }
    }
  }
  if (st == ST_OK) {
    orc_device_loads(idx, frac, (int64_t)n, P, dev, devices, post_loads);
    double st7[7];
    orc_drop_stats(pre, frac, (int64_t)n, P, S, T, d, ffn, st7);
    rep5[1] = st7[3];
    rep5[3] = st7[0];
    rep5[4] = st7[1];
    double mpre = pre_loads[0], mpost = post_loads[0];
    for (int i = 1; i < devices; ++i) {
      mpre = pre_loads[i] > mpre ? pre_loads[i] : mpre; /* std::max_element */
      mpost = post_loads[i] > mpost ? post_loads[i] : mpost;
    }
    rep5[2] = mpost > 0.0 ? mpre / mpost : (mpre > 0.0 ? INFINITY : 1.0);
  }
  free(dev);
  free(raw);
  free(norm);
  free(pre);
  free(tmaj);
  free(tmin);
  return st;
}
