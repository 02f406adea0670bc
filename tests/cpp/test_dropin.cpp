// Drop-in test: the reference's own C++ types and generators
// (/root/reference/proj, linked from oracle/_ref/core.a) on one side, the
// B200 path through include/dsmoe_b200.hpp on the other, read like the
// reference's own tests (proj/tests/test_dropping.cpp, test_moe_model.cpp).
// Built by __graft_entry__.build() into build/test_dropin when the reference
// sources are present; run on the GPU by tests/test_gpu_dropin.py.
#include <cmath>
#include <cstdio>

#include "dsmoe/ep_sim.hpp"
#include "dsmoe/io.hpp"
#include "dsmoe_b200.hpp"

using namespace dsmoe;

static int failures = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::printf("[FAIL] %s:%d %s\n", __FILE__, __LINE__, #cond);   \
      ++failures;                                                    \
    }                                                                \
  } while (0)

static double scaled_residual(const Matrix<float>& a, const Matrix<float>& b) {
  double num = 0, ma = 0, mb = 0;
  for (size_t i = 0; i < a.data.size(); ++i) {
    num = std::max(num, std::fabs(double(a.data[i]) - b.data[i]));
    ma = std::max(ma, std::fabs(double(a.data[i])));
    mb = std::max(mb, std::fabs(double(b.data[i])));
  }
  return num / std::max(ma, mb);
}

int main() {
  MoeConfig c;
  c.d_model = 512;
  c.d_ffn = 1024;
  c.num_experts = 8;
  c.top_k = 2;
  MoeLayer<float> base = generate_synthetic<float>(c, 1234, 1.0);   // io.cpp:330
  Matrix<float> x = generate_tokens<float>(256, 512, 99, 1.0);       // io.cpp:368
  // reference offline partition on the CPU
  ImportanceProfile prof = profile_importance(base, x, route_tokens(base, x), Metric::abs_gate);
  auto [rec, spec, map] = reconstruct_experts(base, prof);

  b200::Context ctx;
  b200::DeviceLayer<float> dev(rec);
  for (double t : {0.30, 0.40, 0.45}) {
    const DropPolicy pol = DropPolicy::two_t_from(t);
    RoutingDecision pre_ref, pre_dev;
    RoutingDecision want = route_and_drop(rec, x, pol, &pre_ref);
    RoutingDecision got = b200::route_and_drop(ctx, dev, x, pol, &pre_dev);
    CHECK(got.indices == want.indices);
    CHECK(got.raw == want.raw);
    CHECK(got.normalized == want.normalized);
    CHECK(got.fraction == want.fraction);
    CHECK(pre_dev.fraction == pre_ref.fraction);
    const DropStats a = drop_stats(pre_ref, want, rec.config);
    const DropStats b = b200::drop_stats(pre_dev, got, rec.config);
    CHECK(a.drop_rate == b.drop_rate && a.retained_flops == b.retained_flops);
    Matrix<float> y_ref = moe_forward(rec, x, want);
    Matrix<float> y_dev = b200::moe_forward(ctx, dev, x, got);
    const double err = scaled_residual(y_dev, y_ref);
    std::printf("t=%.2f drop_rate=%.6f rel_err=%.3g\n", t, b.drop_rate, err);
    CHECK(err < 1e-5);
  }
  // 1T on the unsplit layer, keep_top1 off
  {
    b200::DeviceLayer<float> dbase(base);
    const DropPolicy pol = DropPolicy::one_t(0.45, false);
    RoutingDecision want = route_and_drop(base, x, pol);
    RoutingDecision got = b200::route_and_drop(ctx, dbase, x, pol);
    CHECK(got.fraction == want.fraction && got.indices == want.indices);
    CHECK(scaled_residual(b200::moe_forward(ctx, dbase, x, got), moe_forward(base, x, want)) < 1e-5);
    // same error class as the reference: 2T needs a P=2 layer (dropping.hpp:147)
    Status ref_code = Status::ok, dev_code = Status::ok;
    try { route_and_drop(base, x, DropPolicy::two_t_from(0.3)); } catch (const Error& e) { ref_code = e.code(); }
    try { b200::route_and_drop(ctx, dbase, x, DropPolicy::two_t_from(0.3)); } catch (const Error& e) { dev_code = e.code(); }
    CHECK(ref_code == Status::invalid_state && dev_code == ref_code);
  }
  // partition API on the device vs the reference's transforms (transform.hpp:66-131)
  {
    auto same_layer = [](const MoeLayer<float>& a, const MoeLayer<float>& b) {
      if (!(a.config == b.config) || a.replay_factor != b.replay_factor || a.lineage != b.lineage) return false;
      if (a.gate.data != b.gate.data || a.experts.size() != b.experts.size()) return false;
      for (size_t i = 0; i < a.experts.size(); ++i)
        if (a.experts[i].w1.data != b.experts[i].w1.data || a.experts[i].w3.data != b.experts[i].w3.data ||
            a.experts[i].w2.data != b.experts[i].w2.data)
          return false;
      return a.neuron_order == b.neuron_order;
    };
    CHECK(same_layer(b200::complete_transform(ctx, base, 4), complete_transform(base, 4)));
    CHECK(same_layer(b200::partial_transform(ctx, base, 2).first, partial_transform(base, 2).first));
    CHECK(b200::partial_transform(ctx, base, 4).second.chunk_cols == partial_transform(base, 4).second.chunk_cols);
    Status ref_code = Status::ok, dev_code = Status::ok;
    try { complete_transform(base, 3); } catch (const Error& e) { ref_code = e.code(); }
    try { b200::complete_transform(ctx, base, 3); } catch (const Error& e) { dev_code = e.code(); }
    CHECK(ref_code == Status::invalid_argument && dev_code == ref_code);
    // profile_importance + reconstruct_experts (reconstruct.hpp:99-230)
    b200::DeviceLayer<float> dbase(base);
    const RoutingDecision r0 = route_tokens(base, x);
    for (Metric m : {Metric::gate, Metric::abs_gate, Metric::gate_up, Metric::abs_gate_up}) {
      const ImportanceProfile pr = profile_importance(base, x, r0, m, 3);
      const ImportanceProfile pd = b200::profile_importance(ctx, dbase, x, r0, m, 3);
      CHECK(pd.values == pr.values && pd.layer_index == 3 && pd.token_count == pr.token_count);
    }
    auto [drec, dspec, dmap] = b200::reconstruct_experts(ctx, base, prof);
    CHECK(same_layer(drec, rec));
    CHECK(dmap.order == map.order && dspec.chunk_cols == spec.chunk_cols);
  }
  // simulate_step (ep_sim.hpp:110-160): report and dropped routing
  for (auto strat : {Placement::Strategy::contiguous, Placement::Strategy::round_robin})
    for (bool la : {false, true}) {
      const Placement pl = place_experts(rec.num_physical_experts(), 4, strat);
      const DropPolicy pol = DropPolicy::two_t_from(0.4);
      auto [want, wr] = simulate_step(rec, x, pl, pol, la);
      auto [got, gr] = b200::simulate_step(ctx, dev, x, pl, pol, la);
      CHECK(got.pre_loads == want.pre_loads && got.post_loads == want.post_loads);
      CHECK(got.thresholds == want.thresholds && got.ideal_load == want.ideal_load);
      CHECK(got.speedup == want.speedup && got.drop_rate == want.drop_rate);
      CHECK(got.stats.retained_flops == want.stats.retained_flops);
      CHECK(gr.indices == wr.indices && gr.fraction == wr.fraction && gr.normalized == wr.normalized);
      std::printf("simulate_step %s load_aware=%d speedup=%.6f\n", strategy_name(strat), int(la), got.speedup);
    }
  // load-aware thresholds (test_ep_sim.cpp:71-91)
  CHECK(b200::load_aware_thresholds({120.0, 80.0, 100.0, 100.0}, 0.12) ==
        load_aware_thresholds({120.0, 80.0, 100.0, 100.0}, 0.12));
  std::printf(failures ? "[FAIL] %d checks\n" : "[PASS] drop-in parity\n", failures);
  return failures ? 1 : 0;
}
