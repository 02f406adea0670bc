// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" shim over the reference's own header-only hot path
// (/root/reference/proj/include/dsmoe/*.hpp), compiled from the sources where
// they lie by oracle/Makefile into oracle/_ref/libdsmoe_refshim.so.  Nothing
// here re-implements reference arithmetic: every entry point builds the
// reference's own C++ types from plain arrays and calls the reference's
// templates, so tests can pin oracle/dsmoe_oracle.c (the C restatement) and
// the CUDA path against the real thing, and bench.py's reference arm can time
// the reference's CPU path (route_and_drop + moe_forward) on host threads.
//
// Reference entry points wrapped (all file:line into /root/reference/proj):
//   generate_synthetic       src/io.cpp:330      generate_tokens   src/io.cpp:368
//   softmax_inplace          include/dsmoe/matrix.hpp:68
//   topk_route / replay      include/dsmoe/moe.hpp:181 / :277
//   ensure_normalized        include/dsmoe/dropping.hpp:75
//   drop_1t / drop_2t        include/dsmoe/dropping.hpp:133 / :141
//   route_and_drop           include/dsmoe/dropping.hpp:248
//   drop_stats               include/dsmoe/dropping.hpp:171
//   moe_forward              include/dsmoe/moe.hpp:239
//   profile_importance       include/dsmoe/reconstruct.hpp:99
//   reconstruct_experts      include/dsmoe/reconstruct.hpp:196
//   partial/complete         include/dsmoe/transform.hpp:100 / :66
//   load_aware_thresholds    include/dsmoe/ep_sim.hpp:76
//   simulate_step            include/dsmoe/ep_sim.hpp:110
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "dsmoe/dropping.hpp"
#include "dsmoe/ep_sim.hpp"
#include "dsmoe/io.hpp"
#include "dsmoe/reconstruct.hpp"
#include "dsmoe/transform.hpp"

using namespace dsmoe;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 8;
  }
}

struct Layer {
  MoeLayer<float> l;
};

DropPolicy make_policy(int kind, double t_drop, double t_major, double t_minor, int keep_top1,
                       int normalize) {
  DropPolicy p;
  if (kind == 1) p = DropPolicy::one_t(t_drop);
  if (kind == 2) p = DropPolicy::two_t(t_drop, t_major, t_minor);
  p.keep_top1 = keep_top1 != 0;
  p.normalize = normalize != 0;
  return p;
}

void export_routing(const RoutingDecision& r, int32_t* idx, double* raw, double* norm, double* frac) {
  const size_t n = r.indices.size();
  for (size_t i = 0; i < n; ++i) {
    if (idx) idx[i] = r.indices[i];
    if (raw) raw[i] = r.raw[i];
    if (norm) norm[i] = r.has_normalized() ? r.normalized[i] : 0.0;
    if (frac) frac[i] = r.fraction[i];
  }
}

Matrix<float> rows_of(const float* x, int T, int d) {
  Matrix<float> m(T, d);
  std::memcpy(m.data.data(), x, sizeof(float) * static_cast<size_t>(T) * d);
  return m;
}

}  // namespace

extern "C" {

const char* refshim_last_error(void) { return g_err.c_str(); }

// ---- layer construction ----------------------------------------------------

// Layer from flat arrays in the reference's own generation order
// (src/io.cpp:330-355): gate d x E, then per block w1 (d x w), w3 (d x w),
// w2 (w x d), then shared experts the same way.  widths has E*P entries.
int refshim_layer_create(int d, int ffn, int E, int K, int S, int prenorm, int P, int lineage,
                         const int32_t* widths, const int32_t* shared_widths, const float* flat,
                         const int32_t* neuron_order, void** out) {
  return guard([&] {
    auto* L = new Layer;
    MoeLayer<float>& l = L->l;
    l.config.d_model = d;
    l.config.d_ffn = ffn;
    l.config.num_experts = E;
    l.config.top_k = K;
    l.config.num_shared_experts = S;
    l.config.gate_prenormalized = prenorm != 0;
    l.replay_factor = P;
    l.lineage = static_cast<Lineage>(lineage);
    const float* p = flat;
    auto take = [&](int r, int c) {
      Matrix<float> m(r, c);
      std::memcpy(m.data.data(), p, sizeof(float) * static_cast<size_t>(r) * c);
      p += static_cast<size_t>(r) * c;
      return m;
    };
    l.gate = take(d, E);
    for (int b = 0; b < E * P; ++b) {
      Expert<float> e;
      e.w1 = take(d, widths[b]);
      e.w3 = take(d, widths[b]);
      e.w2 = take(widths[b], d);
      l.experts.push_back(std::move(e));
    }
    for (int s = 0; s < S; ++s) {
      Expert<float> e;
      e.w1 = take(d, shared_widths[s]);
      e.w3 = take(d, shared_widths[s]);
      e.w2 = take(shared_widths[s], d);
      l.shared_experts.push_back(std::move(e));
    }
    if (neuron_order) {
      l.neuron_order.assign(static_cast<size_t>(E), std::vector<int>(static_cast<size_t>(ffn)));
      for (int e = 0; e < E; ++e)
        for (int n = 0; n < ffn; ++n) l.neuron_order[e][n] = neuron_order[e * ffn + n];
    }
    l.validate();
    *out = L;
  });
}

void refshim_layer_free(void* h) { delete static_cast<Layer*>(h); }

// Reference generator (src/io.cpp:330): fresh layer handle.
int refshim_generate_layer(int d, int ffn, int E, int K, int S, int prenorm, uint64_t seed,
                           double scale, void** out) {
  return guard([&] {
    MoeConfig c;
    c.d_model = d;
    c.d_ffn = ffn;
    c.num_experts = E;
    c.top_k = K;
    c.num_shared_experts = S;
    c.gate_prenormalized = prenorm != 0;
    auto* L = new Layer;
    L->l = generate_synthetic<float>(c, seed, scale);
    *out = L;
  });
}

int refshim_generate_tokens(int64_t rows, int cols, uint64_t seed, double scale, float* out) {
  return guard([&] {
    Matrix<float> m = generate_tokens<float>(rows, cols, seed, scale);
    std::memcpy(out, m.data.data(), sizeof(float) * m.data.size());
  });
}

// Layer shape queries + flat export in generation order (the inverse of
// refshim_layer_create).
int refshim_layer_info(void* h, int64_t* info /* d,ffn,E,K,S,P,lineage,n_floats */) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    size_t n = l.gate.size();
    for (const auto& e : l.experts) n += e.w1.size() + e.w3.size() + e.w2.size();
    for (const auto& e : l.shared_experts) n += e.w1.size() + e.w3.size() + e.w2.size();
    info[0] = l.config.d_model;
    info[1] = l.config.d_ffn;
    info[2] = l.config.num_experts;
    info[3] = l.config.top_k;
    info[4] = l.config.num_shared_experts;
    info[5] = l.replay_factor;
    info[6] = static_cast<int>(l.lineage);
    info[7] = static_cast<int64_t>(n);
  });
}

int refshim_layer_export(void* h, float* flat, int32_t* widths, int32_t* shared_widths,
                         int32_t* neuron_order /* may be null */) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    float* p = flat;
    auto put = [&](const Matrix<float>& m) {
      std::memcpy(p, m.data.data(), sizeof(float) * m.size());
      p += m.size();
    };
    put(l.gate);
    for (size_t b = 0; b < l.experts.size(); ++b) {
      widths[b] = l.experts[b].width();
      put(l.experts[b].w1);
      put(l.experts[b].w3);
      put(l.experts[b].w2);
    }
    for (size_t s = 0; s < l.shared_experts.size(); ++s) {
      shared_widths[s] = l.shared_experts[s].width();
      put(l.shared_experts[s].w1);
      put(l.shared_experts[s].w3);
      put(l.shared_experts[s].w2);
    }
    if (neuron_order && !l.neuron_order.empty())
      for (size_t e = 0; e < l.neuron_order.size(); ++e)
        for (size_t n = 0; n < l.neuron_order[e].size(); ++n)
          neuron_order[e * l.config.d_ffn + n] = l.neuron_order[e][n];
  });
}

// ---- routing -----------------------------------------------------------------

// Gate logits exactly as gate_scores computes them before the softmax
// (moe.hpp:174 -> matrix.hpp:47 matmul).
int refshim_gate_logits(void* h, const float* x, int T, float* logits) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    Matrix<float> s = matmul(rows_of(x, T, l.config.d_model), l.gate);
    std::memcpy(logits, s.data.data(), sizeof(float) * s.size());
  });
}

// The routing half of route_and_drop on caller-supplied fp32 logits:
// softmax_inplace per row, topk_route, replay_routing, ensure_normalized,
// drop_1t/drop_2t.  pre_frac receives the pre-drop fractions.
int refshim_route_from_logits(const float* logits, int T, int E, int K, int P, int kind,
                              double t_drop, double t_major, double t_minor, int keep_top1,
                              int normalize, int32_t* idx, double* raw, double* norm, double* frac,
                              double* pre_frac) {
  return guard([&] {
    Matrix<float> s(T, E);
    std::memcpy(s.data.data(), logits, sizeof(float) * s.size());
    for (int t = 0; t < T; ++t) softmax_inplace(s.row(t));
    RoutingDecision r = topk_route(s, K);
    if (P > 1) r = replay_routing(r, K, P);
    const DropPolicy pol = make_policy(kind, t_drop, t_major, t_minor, keep_top1, normalize);
    r = ensure_normalized(r, pol);
    if (pre_frac) export_routing(r, nullptr, nullptr, nullptr, pre_frac);
    RoutingDecision post = r;
    if (kind == 1) post = drop_1t(r, pol);
    if (kind == 2) post = detail::apply_bands(r, pol.t_major, pol.t_minor, pol.keep_top1);
    export_routing(post, idx, raw, norm, frac);
  });
}

// Full route_and_drop on a layer (dropping.hpp:248).
int refshim_route_and_drop(void* h, const float* x, int T, int kind, double t_drop, double t_major,
                           double t_minor, int keep_top1, int normalize, int32_t* idx, double* raw,
                           double* norm, double* frac, double* pre_frac) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    const DropPolicy pol = make_policy(kind, t_drop, t_major, t_minor, keep_top1, normalize);
    RoutingDecision pre;
    RoutingDecision post = route_and_drop(l, rows_of(x, T, l.config.d_model), pol, &pre);
    export_routing(post, idx, raw, norm, frac);
    if (pre_frac) export_routing(pre, nullptr, nullptr, nullptr, pre_frac);
  });
}

// drop_stats (dropping.hpp:171): out = {total_routed_units, dropped_units,
// shared_units, drop_rate, total_flops, saved_flops, retained_flops}.
int refshim_drop_stats(void* h, int T, const double* pre_frac, const double* post_frac,
                       double* out) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    const int P = l.replay_factor, K = l.config.top_k;
    RoutingDecision a, b;
    a.num_tokens = b.num_tokens = T;
    a.base_k = b.base_k = K;
    a.replay_factor = b.replay_factor = P;
    a.k = b.k = K * P;
    const size_t n = static_cast<size_t>(T) * K * P;
    a.indices.assign(n, 0);
    b.indices.assign(n, 0);
    a.raw.assign(n, 0.0);
    b.raw.assign(n, 0.0);
    a.fraction.assign(pre_frac, pre_frac + n);
    b.fraction.assign(post_frac, post_frac + n);
    DropStats st = drop_stats(a, b, l.config);
    out[0] = st.total_routed_units;
    out[1] = st.dropped_units;
    out[2] = st.shared_units;
    out[3] = st.drop_rate;
    out[4] = st.total_flops;
    out[5] = st.saved_flops;
    out[6] = st.retained_flops;
  });
}

// ---- forward -----------------------------------------------------------------

// moe_forward (moe.hpp:239) over token rows, sharded into `threads` contiguous
// row blocks (one std::thread each).  The forward is per-token separable
// (moe.hpp:253-269), so the result is bit-identical to one call.
int refshim_moe_forward(void* h, const float* x, int T, const int32_t* idx, const double* raw,
                        const double* frac, float* out, int threads) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    const int d = l.config.d_model, K = l.config.top_k, P = l.replay_factor, k = K * P;
    if (threads < 1) threads = 1;
    if (threads > T) threads = T > 0 ? T : 1;
    std::vector<std::thread> pool;
    std::vector<std::string> errs(static_cast<size_t>(threads));
    for (int w = 0; w < threads; ++w) {
      const int t0 = static_cast<int>(static_cast<long>(T) * w / threads);
      const int t1 = static_cast<int>(static_cast<long>(T) * (w + 1) / threads);
      pool.emplace_back([&, w, t0, t1] {
        try {
          if (t1 <= t0) return;
          const int n = t1 - t0;
          RoutingDecision r;
          r.num_tokens = n;
          r.base_k = K;
          r.replay_factor = P;
          r.k = k;
          const size_t off = static_cast<size_t>(t0) * k, cnt = static_cast<size_t>(n) * k;
          r.indices.assign(idx + off, idx + off + cnt);
          r.raw.assign(raw + off, raw + off + cnt);
          r.fraction.assign(frac + off, frac + off + cnt);
          Matrix<float> y = moe_forward(l, rows_of(x + static_cast<size_t>(t0) * d, n, d), r);
          std::memcpy(out + static_cast<size_t>(t0) * d, y.data.data(), sizeof(float) * y.size());
        } catch (const std::exception& e) {
          errs[static_cast<size_t>(w)] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (!e.empty()) fail(Status::internal, e);
  });
}

// ---- reconstruction ------------------------------------------------------------

int refshim_profile_importance(void* h, const float* x, int T, const int32_t* idx, int metric,
                               double* values /* E x ffn */) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    RoutingDecision r;
    r.num_tokens = T;
    r.k = r.base_k = l.config.top_k;
    r.replay_factor = 1;
    const size_t n = static_cast<size_t>(T) * r.k;
    r.indices.assign(idx, idx + n);
    r.raw.assign(n, 0.0);
    r.fraction.assign(n, 1.0);
    ImportanceProfile p =
        profile_importance(l, rows_of(x, T, l.config.d_model), r, static_cast<Metric>(metric));
    for (int e = 0; e < p.num_experts; ++e)
      std::memcpy(values + static_cast<size_t>(e) * p.d_ffn, p.values[e].data(),
                  sizeof(double) * p.d_ffn);
  });
}

// reconstruct_experts (reconstruct.hpp:196) from a profile; returns a new
// layer handle (replay 2, lineage reconstructed) and the order.
int refshim_reconstruct(void* h, const double* values, int metric, void** out, int32_t* order) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    ImportanceProfile p;
    p.metric = static_cast<Metric>(metric);
    p.num_experts = l.config.num_experts;
    p.d_ffn = l.config.d_ffn;
    p.token_count = 1;
    p.values.assign(static_cast<size_t>(p.num_experts), std::vector<double>(p.d_ffn));
    for (int e = 0; e < p.num_experts; ++e)
      std::memcpy(p.values[e].data(), values + static_cast<size_t>(e) * p.d_ffn,
                  sizeof(double) * p.d_ffn);
    auto [rl, spec, map] = reconstruct_experts(l, p);
    (void)spec;
    for (int e = 0; e < map.num_experts; ++e)
      for (int n = 0; n < map.d_ffn; ++n) order[e * map.d_ffn + n] = map.order[e][n];
    auto* L = new Layer;
    L->l = std::move(rl);
    *out = L;
  });
}

int refshim_transform(void* h, int complete, int p, void** out) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    auto* L = new Layer;
    if (complete)
      L->l = complete_transform(l, p);
    else
      L->l = partial_transform(l, p).first;
    *out = L;
  });
}

// ---- expert parallelism ------------------------------------------------------------

int refshim_load_aware_thresholds(const double* loads, int D, double t_max, double* out) {
  return guard([&] {
    std::vector<double> t = load_aware_thresholds(std::vector<double>(loads, loads + D), t_max);
    std::memcpy(out, t.data(), sizeof(double) * D);
  });
}

// simulate_step (ep_sim.hpp:110).  rep = {ideal_load, drop_rate, speedup,
// total_routed_units, dropped_units}; loads/thresholds are D-long.
int refshim_simulate_step(void* h, const float* x, int T, int devices, int round_robin, int kind,
                          double t_drop, double t_major, double t_minor, int keep_top1,
                          int normalize, int load_aware, double* pre_loads, double* post_loads,
                          double* thresholds, double* rep, int32_t* idx, double* frac) {
  return guard([&] {
    const MoeLayer<float>& l = static_cast<Layer*>(h)->l;
    Placement plc = place_experts(l.num_physical_experts(), devices,
                                  round_robin ? Placement::Strategy::round_robin
                                              : Placement::Strategy::contiguous);
    const DropPolicy pol = make_policy(kind, t_drop, t_major, t_minor, keep_top1, normalize);
    auto [r, post] = simulate_step(l, rows_of(x, T, l.config.d_model), plc, pol, load_aware != 0);
    std::memcpy(pre_loads, r.pre_loads.data(), sizeof(double) * devices);
    std::memcpy(post_loads, r.post_loads.data(), sizeof(double) * devices);
    std::memcpy(thresholds, r.thresholds.data(), sizeof(double) * devices);
    rep[0] = r.ideal_load;
    rep[1] = r.drop_rate;
    rep[2] = r.speedup;
    rep[3] = r.stats.total_routed_units;
    rep[4] = r.stats.dropped_units;
    export_routing(post, idx, nullptr, nullptr, frac);
  });
}

}  // extern "C"
