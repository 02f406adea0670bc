// dsmoe_b200.hpp — C++ drop-in for the reference's forward path, over the
// C ABI of libdsmoe_b200.so (dsmoe_b200.h).
//
// Include AFTER the reference's own headers are on the include path
// (/root/reference/proj/include): the functions below take and return the
// reference's types — dsmoe::MoeLayer<T>, dsmoe::Matrix<T>, dsmoe::DropPolicy,
// dsmoe::RoutingDecision, dsmoe::DropStats — and throw dsmoe::Error with the
// reference's Status codes (error.hpp:10-50), so a caller of
//
//   route_and_drop(layer, x, policy, &pre)      (dropping.hpp:248)
//   moe_forward(layer, x, routing)              (moe.hpp:239)
//   drop_stats(pre, post, config)               (dropping.hpp:171)
//   complete_transform(layer, p)                (transform.hpp:66)
//   partial_transform(layer, p)                 (transform.hpp:100)
//   profile_importance(layer, calib, r, m, l)   (reconstruct.hpp:99)
//   reconstruct_experts(layer, profile)         (reconstruct.hpp:196)
//   simulate_step(layer, x, placement, pol, la) (ep_sim.hpp:110)
//   load_aware_thresholds(loads, t_max)         (ep_sim.hpp:76)
//
// switches to dsmoe::b200::route_and_drop(ctx, dev_layer, x, policy, &pre)
// etc. with the same argument meaning: a b200::Context first, a
// b200::DeviceLayer where the function evaluates a layer.  Host Matrix in,
// host Matrix out; the device-resident entry points of dsmoe_b200.h are the
// fast path.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "dsmoe/dropping.hpp"
#include "dsmoe/ep_sim.hpp"
#include "dsmoe/reconstruct.hpp"
#include "dsmoe/transform.hpp"
#include "dsmoe_b200.h"

namespace dsmoe::b200 {

inline void check(int rc) {
  if (rc != DSMOE_OK) throw Error(static_cast<Status>(rc), dsmoe_b200_last_error());
}
inline void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw Error(Status::internal, std::string("CUDA: ") + cudaGetErrorString(e));
}

// device buffer (RAII)
struct Buf {
  void* p = nullptr;
  explicit Buf(size_t n) { cuda(cudaMalloc(&p, n ? n : 1)); }
  ~Buf() { cudaFree(p); }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};

class Context {
 public:
  explicit Context(cudaStream_t s = nullptr) : stream_(s) { check(dsmoe_b200_ctx_create(s, &h_)); }
  ~Context() { dsmoe_b200_ctx_free(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  dsmoe_b200_ctx* get() const { return h_; }
  cudaStream_t stream() const { return stream_; }

 private:
  dsmoe_b200_ctx* h_ = nullptr;
  cudaStream_t stream_;
};

// A reference MoeLayer<T> uploaded and packed for the device.  Storage /
// compute type: fp32 (bit-faithful weights) or bf16 (round to nearest even).
template <std::floating_point T>
class DeviceLayer {
  // The device path computes in fp32 (or bf16).  A 64-bit layer — the
  // reference's verification mode, whose gate matmul and softmax run in
  // double — would be narrowed silently and could route differently on
  // near-ties, so it is rejected at compile time.
  static_assert(std::is_same_v<T, float>, "dsmoe::b200::DeviceLayer: the device path computes fp32/bf16; "
                                          "64-bit (scalar_width 8) layers are not supported");

 public:
  DeviceLayer(const MoeLayer<T>& layer, bool bf16 = false, cudaStream_t s = nullptr)
      : config(layer.config), replay_factor(layer.replay_factor), bf16_(bf16) {
    layer.validate();
    std::vector<int32_t> widths, swidths;
    for (const auto& e : layer.experts) widths.push_back(e.width());
    for (const auto& e : layer.shared_experts) swidths.push_back(e.width());
    dsmoe_b200_layer_config cfg{config.d_model, config.d_ffn, config.num_experts, config.top_k,
                                config.num_shared_experts, config.gate_prenormalized ? 1 : 0,
                                layer.replay_factor, bf16 ? DSMOE_B200_BF16 : DSMOE_B200_F32,
                                widths.data(), swidths.empty() ? nullptr : swidths.data()};
    check(dsmoe_b200_layer_create(&cfg, &h_));
    try {
      check(dsmoe_b200_layer_set_gate(h_, f32(layer.gate).data(), DSMOE_B200_F32, 0, s));
      for (size_t b = 0; b < layer.experts.size(); ++b) {
        const auto& e = layer.experts[b];
        check(dsmoe_b200_layer_set_block(h_, static_cast<int>(b), f32(e.w1).data(), f32(e.w3).data(),
                                         f32(e.w2).data(), DSMOE_B200_F32, 0, s));
      }
      for (size_t i = 0; i < layer.shared_experts.size(); ++i) {
        const auto& e = layer.shared_experts[i];
        check(dsmoe_b200_layer_set_shared(h_, static_cast<int>(i), f32(e.w1).data(), f32(e.w3).data(),
                                          f32(e.w2).data(), DSMOE_B200_F32, 0, s));
      }
    } catch (...) {
      dsmoe_b200_layer_free(h_);
      throw;
    }
  }
  // adopt a layer the library created (transform / reconstruct)
  DeviceLayer(dsmoe_b200_layer* h, bool bf16) : h_(h), bf16_(bf16) {
    int32_t info[8];
    check(dsmoe_b200_layer_info(h_, info));
    config.d_model = info[0];
    config.d_ffn = info[1];
    config.num_experts = info[2];
    config.top_k = info[3];
    config.num_shared_experts = info[4];
    config.gate_prenormalized = info[7] != 0;
    replay_factor = info[5];
  }
  ~DeviceLayer() { dsmoe_b200_layer_free(h_); }
  DeviceLayer(const DeviceLayer&) = delete;
  DeviceLayer& operator=(const DeviceLayer&) = delete;

  // the device weights in the reference layout (moe.hpp:73-120); lineage and
  // neuron_order are the caller's to set
  MoeLayer<T> to_host(Context& ctx) const {
    MoeLayer<T> L;
    L.config = config;
    L.replay_factor = replay_factor;
    const int d = config.d_model, nb = config.num_experts * replay_factor, ns = config.num_shared_experts;
    std::vector<int32_t> bw(static_cast<size_t>(nb)), sw(static_cast<size_t>(ns > 0 ? ns : 1));
    check(dsmoe_b200_layer_widths(h_, bw.data(), sw.data()));
    std::vector<unsigned char> g(static_cast<size_t>(d) * config.num_experts * elem());
    check(dsmoe_b200_layer_get_gate(ctx.get(), h_, g.data(), 0));
    L.gate = decode(g, d, config.num_experts);
    auto get = [&](bool shared, int i, int w) {
      std::vector<unsigned char> a(static_cast<size_t>(d) * w * elem()), b(a.size()), c(a.size());
      if (shared)
        check(dsmoe_b200_layer_get_shared(ctx.get(), h_, i, a.data(), b.data(), c.data(), 0));
      else
        check(dsmoe_b200_layer_get_block(ctx.get(), h_, i, a.data(), b.data(), c.data(), 0));
      Expert<T> e;
      e.w1 = decode(a, d, w);
      e.w3 = decode(b, d, w);
      e.w2 = decode(c, w, d);
      return e;
    };
    for (int b = 0; b < nb; ++b) L.experts.push_back(get(false, b, bw[static_cast<size_t>(b)]));
    for (int i = 0; i < ns; ++i) L.shared_experts.push_back(get(true, i, sw[static_cast<size_t>(i)]));
    return L;
  }

  const dsmoe_b200_layer* get() const { return h_; }
  bool bf16() const { return bf16_; }
  size_t elem() const { return bf16_ ? 2 : 4; }

  MoeConfig config;
  int replay_factor;

  // tokens in the layer's storage type
  std::vector<unsigned char> encode(const Matrix<T>& x) const {
    std::vector<unsigned char> out(x.data.size() * elem());
    for (size_t i = 0; i < x.data.size(); ++i) {
      const float v = static_cast<float>(x.data[i]);
      if (bf16_) {
        const __nv_bfloat16 b = __float2bfloat16_rn(v);
        std::memcpy(out.data() + 2 * i, &b, 2);
      } else {
        std::memcpy(out.data() + 4 * i, &v, 4);
      }
    }
    return out;
  }
  Matrix<T> decode(const std::vector<unsigned char>& raw, int rows, int cols) const {
    Matrix<T> m(rows, cols);
    for (size_t i = 0; i < m.data.size(); ++i) {
      float v;
      if (bf16_) {
        __nv_bfloat16 b;
        std::memcpy(&b, raw.data() + 2 * i, 2);
        v = __bfloat162float(b);
      } else {
        std::memcpy(&v, raw.data() + 4 * i, 4);
      }
      m.data[i] = static_cast<T>(v);
    }
    return m;
  }

 private:
  static std::vector<float> f32(const Matrix<T>& m) { return std::vector<float>(m.data.begin(), m.data.end()); }
  dsmoe_b200_layer* h_ = nullptr;
  bool bf16_;
};

inline dsmoe_b200_policy to_c(const DropPolicy& p) {
  return dsmoe_b200_policy{static_cast<int>(p.kind), p.t_drop, p.t_major, p.t_minor, p.keep_top1 ? 1 : 0,
                           p.normalize ? 1 : 0, nullptr};
}

// route_and_drop (dropping.hpp:248).  `pre` receives the normalized pre-drop
// routing.  Logits in exact serial-k order by default (bit-equal to the
// reference's gate matmul), so the routing is the reference's bit for bit.
template <std::floating_point T>
RoutingDecision route_and_drop(Context& ctx, const DeviceLayer<T>& layer, const Matrix<T>& x,
                               const DropPolicy& policy, RoutingDecision* pre = nullptr,
                               int logits_mode = DSMOE_B200_LOGITS_EXACT) {
  require(x.cols == layer.config.d_model, Status::shape_mismatch, "route_and_drop: token width mismatch");
  const int T_ = x.rows, K = layer.config.top_k, P = layer.replay_factor, k = K * P;
  const size_t n = static_cast<size_t>(T_) * k;
  const auto xh = layer.encode(x);
  Buf dx(xh.size()), di(n * 4), dr(n * 4), dn(n * 8), df(n);
  cuda(cudaMemcpyAsync(dx.p, xh.data(), xh.size(), cudaMemcpyHostToDevice, ctx.stream()));
  dsmoe_b200_routing out{static_cast<int32_t*>(di.p), static_cast<float*>(dr.p), static_cast<double*>(dn.p),
                         static_cast<uint8_t*>(df.p)};
  const dsmoe_b200_policy pol = to_c(policy);
  check(dsmoe_b200_route(ctx.get(), layer.get(), dx.p, T_, &pol, logits_mode, nullptr, nullptr, &out, nullptr));
  std::vector<int32_t> idx(n);
  std::vector<float> raw(n);
  std::vector<double> norm(n);
  std::vector<uint8_t> fr(n);
  cuda(cudaMemcpyAsync(idx.data(), di.p, n * 4, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaMemcpyAsync(raw.data(), dr.p, n * 4, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaMemcpyAsync(norm.data(), dn.p, n * 8, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaMemcpyAsync(fr.data(), df.p, n, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaStreamSynchronize(ctx.stream()));
  RoutingDecision r;
  r.num_tokens = T_;
  r.k = k;
  r.base_k = K;
  r.replay_factor = P;
  r.indices.assign(idx.begin(), idx.end());
  r.raw.assign(raw.begin(), raw.end());
  r.normalized = norm;
  r.fraction.resize(n);
  for (size_t i = 0; i < n; ++i) r.fraction[i] = fr[i] == 2 ? 1.0 : (fr[i] == 1 ? 0.5 : 0.0);
  if (pre) {
    *pre = r;
    pre->fraction.assign(n, 1.0);
  }
  return r;
}

// moe_forward (moe.hpp:239) on the device for an explicit routing.
template <std::floating_point T>
Matrix<T> moe_forward(Context& ctx, const DeviceLayer<T>& layer, const Matrix<T>& x, const RoutingDecision& routing) {
  routing.validate();
  require(routing.num_tokens == x.rows, Status::invalid_argument, "moe_forward: routing/batch size mismatch");
  require(x.cols == layer.config.d_model, Status::shape_mismatch, "moe_forward: token width does not match d_model");
  require(routing.replay_factor == layer.replay_factor, Status::invalid_state,
          "moe_forward: routing replay factor does not match layer");
  const int T_ = x.rows;
  const size_t n = routing.indices.size();
  const auto xh = layer.encode(x);
  Buf dx(xh.size()), di(n * 4), dr(n * 8), df(n * 8), dy(xh.size());
  std::vector<int32_t> idx(routing.indices.begin(), routing.indices.end());
  cuda(cudaMemcpyAsync(dx.p, xh.data(), xh.size(), cudaMemcpyHostToDevice, ctx.stream()));
  cuda(cudaMemcpyAsync(di.p, idx.data(), n * 4, cudaMemcpyHostToDevice, ctx.stream()));
  cuda(cudaMemcpyAsync(dr.p, routing.raw.data(), n * 8, cudaMemcpyHostToDevice, ctx.stream()));
  cuda(cudaMemcpyAsync(df.p, routing.fraction.data(), n * 8, cudaMemcpyHostToDevice, ctx.stream()));
  check(dsmoe_b200_moe_forward(ctx.get(), layer.get(), dx.p, T_, static_cast<int32_t*>(di.p),
                               static_cast<double*>(dr.p), static_cast<double*>(df.p), dy.p));
  std::vector<unsigned char> yh(xh.size());
  cuda(cudaMemcpyAsync(yh.data(), dy.p, yh.size(), cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaStreamSynchronize(ctx.stream()));
  return layer.decode(yh, T_, x.cols);
}

// drop_stats (dropping.hpp:171) through the C ABI (same double arithmetic).
inline DropStats drop_stats(const RoutingDecision& before, const RoutingDecision& after, const MoeConfig& config) {
  require(before.num_tokens == after.num_tokens && before.k == after.k &&
              before.replay_factor == after.replay_factor,
          Status::invalid_argument, "drop_stats: routing shapes differ");
  dsmoe_b200_drop_stats_t s{};
  check(dsmoe_b200_drop_stats(before.fraction.data(), after.fraction.data(), static_cast<long>(before.fraction.size()),
                              before.replay_factor, config.num_shared_experts, before.num_tokens, config.d_model,
                              config.d_ffn, &s));
  DropStats st;
  st.num_tokens = s.num_tokens;
  st.total_routed_units = s.total_routed_units;
  st.dropped_units = s.dropped_units;
  st.shared_units = s.shared_units;
  st.drop_rate = s.drop_rate;
  st.total_flops = s.total_flops;
  st.saved_flops = s.saved_flops;
  st.retained_flops = s.retained_flops;
  return st;
}

// load_aware_thresholds (ep_sim.hpp:76).
inline std::vector<double> load_aware_thresholds(const std::vector<double>& loads, double t_max) {
  std::vector<double> out(loads.size());
  check(dsmoe_b200_load_aware_thresholds(loads.data(), static_cast<int>(loads.size()), t_max, out.data()));
  return out;
}

// ---------------------------------------------------------- partition API
// complete_transform (transform.hpp:66-95), re-grouped on the device.
inline MoeLayer<float> complete_transform(Context& ctx, const MoeLayer<float>& layer, int p) {
  layer.validate();
  require(layer.replay_factor == 1, Status::invalid_state,
          "complete_transform: layer already carries a partial transformation");
  DeviceLayer<float> src(layer);
  dsmoe_b200_layer* h = nullptr;
  check(dsmoe_b200_transform(ctx.get(), src.get(), DSMOE_B200_TRANSFORM_COMPLETE, p, &h));
  DeviceLayer<float> dst(h, false);
  MoeLayer<float> out = dst.to_host(ctx);
  out.lineage = Lineage::complete;
  out.validate();
  return out;
}

// partial_transform (transform.hpp:100-131), re-grouped on the device.
inline std::pair<MoeLayer<float>, PartitionSpec> partial_transform(Context& ctx, const MoeLayer<float>& layer, int p) {
  layer.validate();
  require(layer.replay_factor == 1, Status::invalid_state,
          "partial_transform: layer already carries a partial transformation");
  DeviceLayer<float> src(layer);
  dsmoe_b200_layer* h = nullptr;
  check(dsmoe_b200_transform(ctx.get(), src.get(), DSMOE_B200_TRANSFORM_PARTIAL, p, &h));
  DeviceLayer<float> dst(h, false);
  MoeLayer<float> out = dst.to_host(ctx);
  out.lineage = Lineage::partial;
  out.validate();
  PartitionSpec spec;
  spec.factor = p;
  spec.mode = PartitionSpec::Mode::partial;
  spec.num_experts = layer.config.num_experts;
  spec.d_ffn = layer.config.d_ffn;
  spec.chunk_cols = layer.config.d_ffn / p;
  return {std::move(out), spec};
}

// profile_importance (reconstruct.hpp:99-149) on the device: bit-equal
// double accumulators (token-major, then slot, as the reference sums).
inline ImportanceProfile profile_importance(Context& ctx, const DeviceLayer<float>& layer, const Matrix<float>& calib,
                                            const RoutingDecision& routing, Metric metric, int layer_index = 0) {
  routing.validate();
  require(layer.replay_factor == 1, Status::invalid_state,
          "profile_importance: profile the original layer, not a partitioned one");
  require(calib.rows >= 1, Status::invalid_argument, "profile_importance: empty calibration set");
  require(routing.num_tokens == calib.rows, Status::invalid_argument,
          "profile_importance: routing does not match calibration batch");
  require(calib.cols == layer.config.d_model, Status::shape_mismatch,
          "profile_importance: token width does not match d_model");
  const int E = layer.config.num_experts, F = layer.config.d_ffn;
  const auto xh = layer.encode(calib);
  std::vector<int32_t> idx(routing.indices.begin(), routing.indices.end());
  Buf dx(xh.size()), di(idx.size() * 4), dv(static_cast<size_t>(E) * F * 8);
  cuda(cudaMemcpyAsync(dx.p, xh.data(), xh.size(), cudaMemcpyHostToDevice, ctx.stream()));
  cuda(cudaMemcpyAsync(di.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice, ctx.stream()));
  check(dsmoe_b200_profile_importance(ctx.get(), layer.get(), dx.p, calib.rows, static_cast<int32_t*>(di.p),
                                      static_cast<int>(metric), static_cast<double*>(dv.p)));
  std::vector<double> v(static_cast<size_t>(E) * F);
  cuda(cudaMemcpy(v.data(), dv.p, v.size() * 8, cudaMemcpyDeviceToHost));
  ImportanceProfile prof;
  prof.metric = metric;
  prof.num_experts = E;
  prof.d_ffn = F;
  prof.token_count = calib.rows;
  prof.layer_index = layer_index;
  for (int e = 0; e < E; ++e)
    prof.values.emplace_back(v.begin() + static_cast<long>(e) * F, v.begin() + static_cast<long>(e + 1) * F);
  return prof;
}

// reconstruct_experts (reconstruct.hpp:196-230): the stable descending order
// (build_reconstruction_map :151-168) and the permuted, sliced layer, on the
// device.
inline std::tuple<MoeLayer<float>, PartitionSpec, ReconstructionMap> reconstruct_experts(
    Context& ctx, const MoeLayer<float>& layer, const ImportanceProfile& profile) {
  layer.validate();
  profile.validate();
  require(layer.replay_factor == 1, Status::invalid_state, "reconstruct_experts: layer already partitioned");
  require(profile.num_experts == layer.config.num_experts && profile.d_ffn == layer.config.d_ffn,
          Status::invalid_argument, "reconstruct_experts: profile does not match layer shape");
  const int E = layer.config.num_experts, F = layer.config.d_ffn;
  DeviceLayer<float> src(layer);
  std::vector<double> v;
  for (const auto& row : profile.values) v.insert(v.end(), row.begin(), row.end());
  Buf dv(v.size() * 8), dord(static_cast<size_t>(E) * F * 4);
  cuda(cudaMemcpyAsync(dv.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice, ctx.stream()));
  dsmoe_b200_layer* h = nullptr;
  check(dsmoe_b200_reconstruct(ctx.get(), src.get(), static_cast<double*>(dv.p), static_cast<int32_t*>(dord.p), &h));
  DeviceLayer<float> dst(h, false);
  std::vector<int32_t> ord(static_cast<size_t>(E) * F);
  cuda(cudaMemcpy(ord.data(), dord.p, ord.size() * 4, cudaMemcpyDeviceToHost));
  ReconstructionMap map;
  map.num_experts = E;
  map.d_ffn = F;
  map.major_size = (F + 1) / 2;
  for (int e = 0; e < E; ++e)
    map.order.emplace_back(ord.begin() + static_cast<long>(e) * F, ord.begin() + static_cast<long>(e + 1) * F);
  MoeLayer<float> out = dst.to_host(ctx);
  out.lineage = Lineage::reconstructed;
  out.neuron_order = map.order;
  out.validate();
  PartitionSpec spec;
  spec.factor = 2;
  spec.mode = PartitionSpec::Mode::partial;
  spec.num_experts = E;
  spec.d_ffn = F;
  spec.chunk_cols = map.major_size;
  return {std::move(out), spec, std::move(map)};
}

// simulate_step (ep_sim.hpp:110-160) on the device: returns the report and
// the dropped routing, as the reference does.
template <std::floating_point T>
std::pair<EpReport, RoutingDecision> simulate_step(Context& ctx, const DeviceLayer<T>& layer, const Matrix<T>& tokens,
                                                   const Placement& placement, const DropPolicy& policy,
                                                   bool load_aware) {
  placement.validate();
  require(static_cast<int>(placement.device_of.size()) == layer.config.num_experts * layer.replay_factor,
          Status::invalid_argument, "simulate_step: placement does not cover this layer's experts");
  const int T_ = tokens.rows, D = placement.devices, k = layer.config.top_k * layer.replay_factor;
  const size_t n = static_cast<size_t>(T_) * k;
  const auto xh = layer.encode(tokens);
  Buf dx(xh.size()), di(n * 4), dr(n * 4), dn(n * 8), df(n);
  cuda(cudaMemcpyAsync(dx.p, xh.data(), xh.size(), cudaMemcpyHostToDevice, ctx.stream()));
  std::vector<int32_t> dv(placement.device_of.begin(), placement.device_of.end());
  EpReport rep;
  rep.devices = D;
  rep.load_aware = load_aware;
  rep.policy_kind = policy.kind_name();
  rep.pre_loads.assign(static_cast<size_t>(D), 0.0);
  rep.post_loads.assign(static_cast<size_t>(D), 0.0);
  rep.thresholds.assign(static_cast<size_t>(D), 0.0);
  double sc[3];
  dsmoe_b200_drop_stats_t st{};
  dsmoe_b200_routing out{static_cast<int32_t*>(di.p), static_cast<float*>(dr.p), static_cast<double*>(dn.p),
                         static_cast<uint8_t*>(df.p)};
  const dsmoe_b200_policy pol = to_c(policy);
  check(dsmoe_b200_simulate_step(ctx.get(), layer.get(), dx.p, T_, D, dv.data(), &pol, load_aware ? 1 : 0,
                                 DSMOE_B200_LOGITS_EXACT, rep.pre_loads.data(), rep.post_loads.data(),
                                 rep.thresholds.data(), sc, &st, &out, nullptr, 0));
  rep.ideal_load = sc[0];
  rep.drop_rate = sc[1];
  rep.speedup = sc[2];
  rep.stats.num_tokens = st.num_tokens;
  rep.stats.total_routed_units = st.total_routed_units;
  rep.stats.dropped_units = st.dropped_units;
  rep.stats.shared_units = st.shared_units;
  rep.stats.drop_rate = st.drop_rate;
  rep.stats.total_flops = st.total_flops;
  rep.stats.saved_flops = st.saved_flops;
  rep.stats.retained_flops = st.retained_flops;
  std::vector<int32_t> idx(n);
  std::vector<float> raw(n);
  std::vector<double> norm(n);
  std::vector<uint8_t> fr(n);
  cuda(cudaMemcpyAsync(idx.data(), di.p, n * 4, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaMemcpyAsync(raw.data(), dr.p, n * 4, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaMemcpyAsync(norm.data(), dn.p, n * 8, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaMemcpyAsync(fr.data(), df.p, n, cudaMemcpyDeviceToHost, ctx.stream()));
  cuda(cudaStreamSynchronize(ctx.stream()));
  RoutingDecision r;
  r.num_tokens = T_;
  r.k = k;
  r.base_k = layer.config.top_k;
  r.replay_factor = layer.replay_factor;
  r.indices.assign(idx.begin(), idx.end());
  r.raw.assign(raw.begin(), raw.end());
  if (policy.normalize) r.normalized = norm;
  r.fraction.resize(n);
  for (size_t i = 0; i < n; ++i) r.fraction[i] = fr[i] == 2 ? 1.0 : (fr[i] == 1 ? 0.5 : 0.0);
  return {std::move(rep), std::move(r)};
}

}  // namespace dsmoe::b200
