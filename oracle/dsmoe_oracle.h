/* TEST INFRASTRUCTURE ONLY.  C restatement of the reference's hot path
 * (/root/reference/proj), used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER — never by the product path.
 *
 * Parity pinned: every function is checked (tests/test_oracle.py) against the
 * reference's own golden vectors (proj/tests/test_*.cpp) and against the
 * reference itself compiled from its sources into oracle/_ref/ by
 * oracle/Makefile; fixtures generated that way live in tests/golden/.
 *
 * Arithmetic contract: same IEEE operation sequence as the reference
 * (-ffp-contract=off, serial sums in reference order, glibc expf).
 * Status codes equal the reference's dsmoe::Status (error.hpp:10-20). */
#ifndef DSMOE_ORACLE_H
#define DSMOE_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* policy kinds (dropping.hpp:13) */
#define ORC_NONE 0
#define ORC_1T 1
#define ORC_2T 2

/* SplitMix64 / xoshiro256++ generator (rng.hpp:15-61) and the synthetic data
 * of io.cpp:330-374.  Layer buffer layout = generation order: gate (d x E),
 * per expert w1 (d x ffn), w3 (d x ffn), w2 (ffn x d), then shared experts. */
uint64_t orc_splitmix_nth(uint64_t seed, int n);
int orc_generate_layer(int d, int ffn, int E, int S, uint64_t seed, double scale, float* flat);
int orc_generate_tokens(int64_t rows, int cols, uint64_t seed, double scale, float* out);

/* gate logits = matmul(x, gate): single accumulator, ascending k, no FMA
 * (moe.hpp:174, matrix.hpp:47-64). */
void orc_gate_logits(const float* x, const float* gate, int T, int d, int E, float* logits);

/* softmax_inplace (matrix.hpp:68-78) on each row of s. */
void orc_softmax_rows(float* s, int T, int E);

/* topk_route (moe.hpp:181-206) on T x E scores -> T x K. */
int orc_topk(const float* scores, int T, int E, int K, int32_t* idx, double* raw);
/* normalize_topk (dropping.hpp:60-72) on copy-major T x K*P raw scores. */
int orc_normalize(const double* raw, int T, int K, int P, double* norm);
/* apply_bands_fn (dropping.hpp:93-122) on copy-major T x K*P normalized scores. */
void orc_apply_bands(const double* norm, int T, int K, int P, double t_major, double t_minor,
                     const double* t_major_slot, const double* t_minor_slot, int keep_top1,
                     double* frac);

/* Routing on caller logits: softmax, topk_route (moe.hpp:181), replay_routing
 * (moe.hpp:277), ensure_normalized (dropping.hpp:75), drop_1t/drop_2t
 * (dropping.hpp:133/141).  Arrays are T*K*P in copy-major slot order.
 * t_major_slot / t_minor_slot (nullable, T*K) override the policy band per
 * original selection — the per-device thresholds of ep_sim.hpp:139-149. */
int orc_route_from_logits(const float* logits, int T, int E, int K, int P, int kind, double t_drop,
                          double t_major, double t_minor, int keep_top1, int normalize,
                          const double* t_major_slot, const double* t_minor_slot, int32_t* idx,
                          double* raw, double* norm, double* frac, double* pre_frac);

/* drop_stats (dropping.hpp:171-195).  out7 = total_routed_units,
 * dropped_units, shared_units, drop_rate, total_flops, saved_flops,
 * retained_flops. */
void orc_drop_stats(const double* pre_frac, const double* post_frac, int64_t n, int P, int S,
                    int64_t T, int d, int ffn, double* out7);

/* moe_forward (moe.hpp:239-271) with accumulate_block (moe.hpp:213-231):
 * bit-identical float arithmetic, neuron loop vectorised in the same
 * per-element order.  w1[b]/w3[b] are d x widths[b], w2[b] widths[b] x d. */
int orc_moe_forward(const float* x, int T, int d, int nblocks, int kslots,
                    const float* const* w1, const float* const* w3, const float* const* w2,
                    const int32_t* widths, int S, const float* const* sw1,
                    const float* const* sw3, const float* const* sw2, const int32_t* swidths,
                    const int32_t* idx, const double* raw, const double* frac, float* out);

/* profile_importance (reconstruct.hpp:99-149); values is E x ffn doubles,
 * metric: 0 gate, 1 abs_gate, 2 gate_up, 3 abs_gate_up. */
int orc_profile_importance(const float* x, int T, int d, int E, int ffn, int K,
                           const float* const* w1, const float* const* w3, const int32_t* idx,
                           int metric, double* values);

/* build_reconstruction_map (reconstruct.hpp:151-168): per expert, stable
 * descending order of importance. */
void orc_reconstruction_order(const double* values, int E, int ffn, int32_t* order);

/* place_experts / device_loads / load_aware_thresholds (ep_sim.hpp:38-89). */
int orc_place_experts(int num_experts, int devices, int round_robin, int32_t* device_of);
void orc_device_loads(const int32_t* idx, const double* frac, int64_t n, int P,
                      const int32_t* device_of, int D, double* loads);
int orc_load_aware_thresholds(const double* loads, int D, double t_max, double* out);

/* simulate_step (ep_sim.hpp:110-160) on caller logits.  rep5 = ideal_load,
 * drop_rate, speedup, total_routed_units, dropped_units. */
int orc_simulate_step(const float* logits, int T, int E, int K, int P, int S, int d, int ffn,
                      int devices, int round_robin, int kind, double t_drop, double t_major,
                      double t_minor, int keep_top1, int normalize, int load_aware,
                      double* pre_loads, double* post_loads, double* thresholds, double* rep5,
                      int32_t* idx, double* frac);

#ifdef __cplusplus
}
#endif
#endif
