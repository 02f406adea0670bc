/* dsmoe_b200 — B200 (sm_100a) device path for the DualSparse-MoE MoE-module
 * forward.  C ABI: plain pointers, sizes and status codes; no C++ or torch
 * types cross it.  Status codes and the thread-local last-error convention are
 * the reference's (/root/reference/proj/include/dsmoe.h:16-24, capi.cpp:35-58):
 * every entry point returns DSMOE_OK (0) or a DSMOE_E_* code and never lets an
 * exception escape.
 *
 * Pointers documented "device" are CUDA global-memory addresses; "host"
 * pointers are ordinary memory.  `stream` is a cudaStream_t passed as void*
 * (NULL = the legacy default stream).  Layers are immutable after their
 * weights are set; calls on distinct contexts may run concurrently.
 *
 * Reference interfaces replaced (file:line under /root/reference/proj):
 *   dsmoe_b200_layer_*          MoeLayer<T> (include/dsmoe/moe.hpp:73-120)
 *   dsmoe_b200_route            route_and_drop (include/dsmoe/dropping.hpp:248),
 *                               i.e. gate_scores moe.hpp:170, topk_route :181,
 *                               replay_routing :277, ensure_normalized
 *                               dropping.hpp:75, drop_1t :133 / drop_2t :141
 *   dsmoe_b200_moe_forward      moe_forward (include/dsmoe/moe.hpp:239)
 *   dsmoe_b200_forward          route_and_drop + drop_stats + moe_forward, the
 *                               per-layer body of model_forward_dropped
 *                               (dropping.hpp:263-274) and of dsmoe_infer
 *                               (include/dsmoe.h:67, src/capi.cpp:328)
 *   dsmoe_b200_drop_stats       drop_stats (include/dsmoe/dropping.hpp:171)
 *   dsmoe_b200_profile_importance  profile_importance (reconstruct.hpp:99)
 *   dsmoe_b200_reconstruct      build_reconstruction_map + reconstruct_experts
 *                               (reconstruct.hpp:151, :196)
 *   dsmoe_b200_load_aware_thresholds  load_aware_thresholds (ep_sim.hpp:76)
 *   dsmoe_b200_transform        complete_transform / partial_transform /
 *                               reverse_partial (transform.hpp:66, :100, :136)
 */
#ifndef DSMOE_B200_H
#define DSMOE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef DSMOE_OK
#define DSMOE_OK 0
#define DSMOE_E_INVALID_ARGUMENT 1
#define DSMOE_E_SHAPE_MISMATCH 2
#define DSMOE_E_INVALID_STATE 3
#define DSMOE_E_IO 4
#define DSMOE_E_BAD_MAGIC 5
#define DSMOE_E_TRUNCATED 6
#define DSMOE_E_SCHEMA 7
#define DSMOE_E_INTERNAL 8
#endif

#define DSMOE_B200_F32 0  /* element types */
#define DSMOE_B200_BF16 1

#define DSMOE_B200_DROP_NONE 0 /* DropPolicy::Kind (dropping.hpp:13) */
#define DSMOE_B200_DROP_1T 1
#define DSMOE_B200_DROP_2T 2

#define DSMOE_B200_LOGITS_TENSOR 0 /* gate logits on tcgen05 (bf16 layers) */
#define DSMOE_B200_LOGITS_EXACT 1  /* serial-k fp32, bit-equal to matmul (matrix.hpp:47) */
#define DSMOE_B200_LOGITS_REUSE 2  /* the logits of the previous call on this context (same layer, same T):
                                      re-route a batch under new thresholds without the gate GEMM */

#define DSMOE_B200_METRIC_GATE 0 /* Metric (reconstruct.hpp:13) */
#define DSMOE_B200_METRIC_ABS_GATE 1
#define DSMOE_B200_METRIC_GATE_UP 2
#define DSMOE_B200_METRIC_ABS_GATE_UP 3

typedef struct dsmoe_b200_layer dsmoe_b200_layer;
typedef struct dsmoe_b200_ctx dsmoe_b200_ctx;

/* MoeConfig (moe.hpp:17-36) + the layer state that shapes the blocks:
 * replay_factor P (moe.hpp:79), block widths (E*P entries, block e*P+p is
 * slice p of expert e) and shared-expert widths (S entries). */
typedef struct {
  int d_model;
  int d_ffn;
  int num_experts;
  int top_k;
  int num_shared_experts;
  int gate_prenormalized;
  int replay_factor;
  int dtype; /* DSMOE_B200_F32 | DSMOE_B200_BF16: storage + compute type */
  const int32_t* block_widths;  /* host, E*P entries; NULL -> d_ffn / P each */
  const int32_t* shared_widths; /* host, S entries; NULL -> d_ffn each */
} dsmoe_b200_layer_config;

/* DropPolicy (dropping.hpp:12-56) as the policy JSON of capi.cpp:96-112 maps
 * it: for 2T the caller supplies t_major/t_minor (default t_drop -/+ 0.01).
 * normalize < 0 selects the default (!gate_prenormalized).
 * t_unit (device, optional, num_experts doubles) overrides the threshold per
 * original expert: t_major = t_unit[e] + (t_major - t_drop), t_minor =
 * t_unit[e] + (t_minor - t_drop) — the owner-device thresholds of
 * simulate_step (ep_sim.hpp:133-149). */
typedef struct {
  int kind;
  double t_drop;
  double t_major;
  double t_minor;
  int keep_top1;
  int normalize;
  const double* t_unit;
} dsmoe_b200_policy;

/* RoutingDecision (moe.hpp:142-167) on the device, T x (K*P) slots in the
 * reference's copy-major order.  Any field may be NULL. */
typedef struct {
  int32_t* indices;
  float* raw;        /* raw score; the reference's double raw is exactly this float */
  double* normalized;
  uint8_t* fraction; /* 0 -> 0.0, 1 -> 0.5, 2 -> 1.0 */
} dsmoe_b200_routing;

/* DropStats (dropping.hpp:156-166), same fields and arithmetic. */
typedef struct {
  long num_tokens;
  double total_routed_units;
  double dropped_units;
  double shared_units;
  double drop_rate;
  double total_flops;
  double saved_flops;
  double retained_flops;
} dsmoe_b200_drop_stats_t;

const char* dsmoe_b200_version(void);
const char* dsmoe_b200_last_error(void);
/* number of kernels the last dsmoe_b200_forward / _moe_forward launched */
int dsmoe_b200_last_launch_count(void);
/* every kernel this library has launched in this process (all entry points) */
long long dsmoe_b200_total_launch_count(void);

/* ---- layers ------------------------------------------------------------ */
int dsmoe_b200_layer_create(const dsmoe_b200_layer_config* cfg, dsmoe_b200_layer** out);
void dsmoe_b200_layer_free(dsmoe_b200_layer* layer);
/* gate: d_model x num_experts row-major (moe.hpp:75).  src_dtype is the
 * element type of the source; src_on_device says where it lives. */
int dsmoe_b200_layer_set_gate(dsmoe_b200_layer* layer, const void* gate, int src_dtype,
                              int src_on_device, void* stream);
/* physical block b (Expert<T>, moe.hpp:39-45): w1, w3 d x width; w2 width x d. */
int dsmoe_b200_layer_set_block(dsmoe_b200_layer* layer, int block, const void* w1, const void* w3,
                               const void* w2, int src_dtype, int src_on_device, void* stream);
int dsmoe_b200_layer_set_shared(dsmoe_b200_layer* layer, int s, const void* w1, const void* w3,
                                const void* w2, int src_dtype, int src_on_device, void* stream);
/* shape query: out8 = d, ffn, E, K, S, P, dtype, prenorm */
int dsmoe_b200_layer_info(const dsmoe_b200_layer* layer, int32_t* out8);

/* ---- execution contexts (stream + workspace) ---------------------------- */
int dsmoe_b200_ctx_create(void* stream, dsmoe_b200_ctx** out);
void dsmoe_b200_ctx_free(dsmoe_b200_ctx* ctx);
/* synchronise the context's stream and report any device-side error flag
 * raised since the last check (zero-sum normalisation, non-canonical routing) */
int dsmoe_b200_ctx_check(dsmoe_b200_ctx* ctx);

/* Per-stage device timing for dsmoe_b200_forward (CUDA events on the
 * context's stream, recorded without synchronising — a ring of event sets is
 * resolved when the profile is read, so it can run inside a timed loop).  Stages: 0 gate logits,
 * 1 router, 2 permute + tile plan, 3 gather, 4 grouped GEMM1 ([W1|W3] +
 * SwiGLU), 5 grouped GEMM2 (W2 + score), 6 combine.  ms receives the summed
 * milliseconds per stage since profiling was (re)enabled. */
int dsmoe_b200_ctx_set_profiling(dsmoe_b200_ctx* ctx, int on);  /* on = N > 1: every N-th forward */
int dsmoe_b200_ctx_profile(dsmoe_b200_ctx* ctx, double* ms, int n, long* calls);

/* The token permutation of the last forward on this context (host copies,
 * any pointer may be NULL): row_token[r] = token of permuted row r (r <
 * *r_total), slot_pos[t*K+s] = row of selection (t, s) or -1 when dropped,
 * seg[3e..3e+2] = start, full rows, total rows of expert unit e.  Canonical
 * order: units ascending, full rows then major-only rows, (t, s) ascending. */
int dsmoe_b200_ctx_permutation(dsmoe_b200_ctx* ctx, int T, int K, int E, int32_t* row_token,
                               int32_t* slot_pos, int32_t* seg, int* r_total);

/* ---- the forward path --------------------------------------------------- */
/* route_and_drop on device x (T x d_model, layer dtype).  `logits_in`
 * (device, T x E fp32, optional) bypasses the gate matmul.  `logits_out`
 * (device, optional) receives the logits used.  stats (host, optional)
 * forces a stream sync and is filled like drop_stats(pre, post, config). */
int dsmoe_b200_route(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                     const dsmoe_b200_policy* policy, int logits_mode, const float* logits_in,
                     float* logits_out, const dsmoe_b200_routing* out,
                     dsmoe_b200_drop_stats_t* stats);
/* moe_forward with a caller routing (device arrays, T x K*P): out (device,
 * T x d_model, layer dtype) = sum over kept slots of raw * block(x) + shared.
 * Any valid RoutingDecision (moe.hpp:142-167) is accepted: the canonical
 * replayed layout runs on the fused path, anything else (any physical block
 * and fraction per slot) on the layer's block view.  Index out of range or a
 * fraction outside {0, 0.5, 1}: DSMOE_E_INVALID_STATE (moe.hpp:258-262). */
int dsmoe_b200_moe_forward(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x,
                           int T, const int32_t* indices, const double* raw,
                           const double* fraction, void* out);
/* route + drop + forward in one launch sequence (no host sync unless stats
 * is non-NULL).  The timed hot path. */
int dsmoe_b200_forward(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                       const dsmoe_b200_policy* policy, int logits_mode, void* out,
                       dsmoe_b200_drop_stats_t* stats);

/* ---- expert parallelism data path (north-star item 6; ep.py drives NCCL) --
 * Source side: route + drop (policy->t_unit carries the owner-device
 * thresholds of simulate_step, ep_sim.hpp:133-149), permute, and gather the
 * kept token rows in the canonical order — experts ascending, so under
 * contiguous placement (ep_sim.hpp:48-52) the rows for each destination rank
 * are one contiguous run.  rows_out (device, >= T*K x d_model, layer dtype)
 * and scale_out (device, >= T*K fp32 raw scores) may be NULL (count only);
 * seg_out (host, E x 3) = start, full rows, total rows per expert.  Shared
 * experts are evaluated locally here.  Synchronises the stream. */
int dsmoe_b200_dispatch(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                        const dsmoe_b200_policy* policy, int logits_mode, void* rows_out,
                        float* scale_out, int32_t* seg_out, int* r_total,
                        dsmoe_b200_drop_stats_t* stats);
/* Expert side: grouped SwiGLU FFN (K3 + K4) over caller segments of `rows`
 * (device, nrows x d_model): segment i = rows [seg_start[i], +seg_ntot[i]) of
 * expert seg_unit[i], its first seg_nfull[i] rows evaluated on every
 * sub-block, the rest on the major sub-block only; y_out (device, nrows x
 * d_model) = row_scale[r] * expert(row r).  Segment arrays are host. */
int dsmoe_b200_expert_ffn(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* rows,
                          const float* row_scale, long nrows, int nseg, const int32_t* seg_unit,
                          const int32_t* seg_start, const int32_t* seg_nfull,
                          const int32_t* seg_ntot, void* y_out);
/* out (device, T x d_model) = sum over the last dispatch's kept selections of
 * y_rows (device, dispatch row order) + the local shared experts (K5). */
int dsmoe_b200_combine(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* y_rows, int T,
                       void* out);

/* EP with one row per (token, destination rank) instead of one per kept
 * selection.  Sender: after dsmoe_b200_dispatch (rows_out may be NULL) routed
 * the batch on this context, ep_pack places every token once per rank that
 * owns one of its kept selections: send_rows (device, >= T*min(nranks,K)
 * rows, layer dtype) destination-major with tokens ascending; one record per
 * kept selection (rec_code = expert*4 + level, rec_row = row within the
 * destination's block, rec_raw = raw score; device, >= T*K) destination-major;
 * counts (host, 2*nranks) = rows then records per destination.  owner (host,
 * E) = rank of each expert.  Synchronises the stream. */
int dsmoe_b200_ep_pack(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T, int nranks,
                       const int32_t* owner, void* send_rows, int32_t* rec_code, int32_t* rec_row, float* rec_raw,
                       int64_t* counts);
/* Receiver: U rows and S records gathered from nranks sources (source s owns
 * rows [src_row_base[s], src_row_base[s+1]) and records [src_rec_base[s],
 * src_rec_base[s+1]); host arrays of nranks+1).  out (device, U x d_model) =
 * per row the sum over its records of raw * expert(row) — the routed experts
 * only, one row back per (token, rank). */
int dsmoe_b200_ep_expert(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* rows, long U,
                         const int32_t* rec_code, const int32_t* rec_row, const float* rec_raw, long S,
                         const int64_t* src_row_base, const int64_t* src_rec_base, int nranks, void* out);
/* Sender: out (device, T x d_model) = sum over destinations (ascending) of the
 * rows returned in send order (ret_rows, same layout as send_rows) + the local
 * shared experts of the last dispatch. */
int dsmoe_b200_ep_combine(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* ret_rows, int T,
                          void* out);

/* EP with one host synchronisation per step (ep.py, ExpertParallelMoE):
 *   ep_route_counts   route the batch without drop (normalisation per the
 *                     policy) and write the per-expert selection counts
 *                     (device, E x {full, major-only} int64) — the integers
 *                     all-reduced across ranks;
 *   ep_last_counts    the same counts of the last routing on the context
 *                     (after ep_dispatch: the kept selections, for post loads);
 *   ep_thresholds     from the all-reduced counts (device): device_loads of the
 *                     placement device_of (device, E*P int32) over `devices`,
 *                     load-aware or uniform thresholds, and the owner table
 *                     t_unit (device, E doubles) simulate_step applies
 *                     (ep_sim.hpp:59-89, :139-141); loads (device, optional);
 *   ep_dispatch       re-route under policy->t_unit (logits_mode
 *                     DSMOE_B200_LOGITS_REUSE reuses the logits of
 *                     ep_route_counts on the same context; `logits` (device,
 *                     row stride logits_ld, optional) routes a token chunk
 *                     from another context's logits), pack one row per (token, destination)
 *                     into send_rows and one 3 x int32 record {expert*4+level,
 *                     row, raw-score bits} per kept selection into records,
 *                     counts (device, nranks x {rows, records} int64), and
 *                     evaluate the local shared experts; dest (device, 2E
 *                     uint32): destination-rank bit masks of a full and of a
 *                     major-only selection of each expert — the ranks holding
 *                     its blocks / its block 0, so an expert's sub-blocks may
 *                     live on different ranks (S-ETP placement);
 *   ep_expert_packed  dsmoe_b200_ep_expert with the interleaved records.
 * None of them synchronises the host. */
int dsmoe_b200_ep_route_counts(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                               const dsmoe_b200_policy* policy, int logits_mode, int64_t* counts);
int dsmoe_b200_ep_last_counts(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, int T, int64_t* counts);
int dsmoe_b200_ep_thresholds(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const int64_t* counts, int devices,
                             const int32_t* device_of, double t_max, int load_aware, double* t_unit, double* loads);
int dsmoe_b200_ep_dispatch(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                           const dsmoe_b200_policy* policy, int logits_mode, const float* logits, int logits_ld,
                           int nranks, const uint32_t* dest, void* send_rows, int32_t* records, int64_t* counts);
/* The gate logits of the last routing on ctx (device, T rows, row stride ld
 * floats; valid until the next routing there): token chunks of one batch
 * re-route from them on other contexts (ep_dispatch's logits / logits_ld:
 * pass logits + c0 * ld for the chunk starting at token c0). */
int dsmoe_b200_ctx_logits(dsmoe_b200_ctx* ctx, const float** logits, int* ld, int* T);
int dsmoe_b200_ep_expert_packed(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* rows, long U,
                                const int32_t* records, long S, const int64_t* src_row_base,
                                const int64_t* src_rec_base, int nranks, void* out);
/* An expert shard of `layer` for expert parallelism: the same gate, shared
 * experts and shapes, but only routed experts [unit_lo, unit_hi) hold
 * weights (contiguous placement puts each rank's experts in one range,
 * ep_sim.hpp:48-52).  A shard routes, dispatches and runs ep_expert for its
 * own experts; whole-layer entry points (forward, moe_forward, profile,
 * reconstruct, transform) reject it with DSMOE_E_INVALID_STATE. */
int dsmoe_b200_layer_shard(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, int unit_lo, int unit_hi,
                           dsmoe_b200_layer** out);
/* The general shard: held (host, E*P flags) marks the physical blocks this
 * rank stores — e.g. Placement::device_of == rank for any placement
 * (ep_sim.hpp:38-54), including S-ETP placements that put the sub-blocks
 * of one expert on different ranks.  A unit's sub-blocks are its held
 * blocks in order; a full selection evaluates them all, a major-only one
 * block 0 (dsmoe_b200_ep_dispatch's dest masks send it only where block 0
 * lives). */
int dsmoe_b200_layer_shard_blocks(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const uint8_t* held,
                                  dsmoe_b200_layer** out);

/* dsmoe_b200_forward with flags.  DSMOE_B200_RESIDUAL: out = x + moe(x), the
 * residual step of model_forward_dropped (dropping.hpp:271) fused into the
 * combine kernel (out may not alias x). */
#define DSMOE_B200_RESIDUAL 1
int dsmoe_b200_forward_ex(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                          const dsmoe_b200_policy* policy, int logits_mode, int flags, void* out,
                          dsmoe_b200_drop_stats_t* stats);

/* Rate-targeted drop (north star item 2).  The reference reaches a drop
 * rate by bisecting the threshold (acceptance.cpp:342-352); here the
 * bisection runs on the device in one kernel over the batch's normalized
 * scores: t = (lo + hi) / 2, the exact drop_stats rate of one_t(t) /
 * two_t_from(t) (policy->kind 1T / 2T, keep_top1, normalize as in the
 * policy; its thresholds are ignored), the closest t so far kept, stop at
 * |rate - target| <= tol or after `iters` rounds — the same t, bit for bit,
 * as that host loop.  calibrate_rate returns t and its rate on the host
 * (synchronises); forward_rate routes the batch under that t and runs the
 * forward without a host round trip (t_rate: device, optional, receives
 * [t, rate]; stats: host, optional, synchronises). */
int dsmoe_b200_calibrate_rate(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                              const dsmoe_b200_policy* policy, double target, double tol, int iters, int logits_mode,
                              double* t_out, double* rate_out);
int dsmoe_b200_forward_rate(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                            const dsmoe_b200_policy* policy, double target, double tol, int iters, int logits_mode,
                            int flags, void* out, double* t_rate, dsmoe_b200_drop_stats_t* stats);

/* analyze_gating (dropping.hpp:207-228) on the device: Top-K (no drop, always
 * normalized) of the layer's own gate; host outputs selection_counts[E],
 * raw_hist[bins], norm_hist[bins] with bin = clamp(int(v * bins), 0, bins-1). */
int dsmoe_b200_analyze_gating(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T,
                              int bins, int logits_mode, long long* selection_counts, long long* raw_hist,
                              long long* norm_hist);

/* drop_stats from host fraction arrays (n = T*K*P doubles each). */
int dsmoe_b200_drop_stats(const double* pre_fraction, const double* post_fraction, long n,
                          int replay_factor, int num_shared, long num_tokens, int d_model,
                          int d_ffn, dsmoe_b200_drop_stats_t* out);

/* ---- offline partition + reconstruction (north-star item 1) ------------- */
/* profile_importance: x (device, T x d, layer dtype), indices (device, T x K,
 * an unsplit layer's routing); values (device, E x d_ffn doubles). */
int dsmoe_b200_profile_importance(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x,
                                  int T, const int32_t* indices, int metric, double* values);
/* reconstruct_experts: stable descending order of each expert's importance
 * (order: device, E x d_ffn int32, optional), then a new layer with P = 2
 * (major = first ceil(d_ffn/2) neurons of the order). */
int dsmoe_b200_reconstruct(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const double* values,
                           int32_t* order, dsmoe_b200_layer** out);

/* ---- partition API on the device (transform.hpp) ----------------------- */
#define DSMOE_B200_TRANSFORM_COMPLETE 0 /* complete_transform (transform.hpp:66-95) */
#define DSMOE_B200_TRANSFORM_PARTIAL 1  /* partial_transform (transform.hpp:100-131) */
#define DSMOE_B200_TRANSFORM_REVERSE 2  /* reverse_partial (transform.hpp:136-170) */
/* A new device layer re-grouped from `layer` without leaving the device:
 * complete -> E*p experts of width d_ffn/p, gate columns repeated (copies of
 * e at e*p..e*p+p-1), W2 scaled by p, top-K*p; partial -> replay_factor p,
 * unscaled chunks, gate unchanged; reverse -> the sub-blocks concatenated
 * back into P = 1 experts.  Errors as the reference (p >= 2, p | d_ffn,
 * layer not already partitioned). */
int dsmoe_b200_transform(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, int mode, int p,
                         dsmoe_b200_layer** out);
/* block widths (E*P entries) and shared-expert widths (S entries), host */
int dsmoe_b200_layer_widths(const dsmoe_b200_layer* layer, int32_t* block_widths, int32_t* shared_widths);
/* Read-back in the reference layout (moe.hpp:39-45, :75), layer dtype:
 * gate d x E; block b: w1, w3 d x width, w2 width x d.  dst_on_device says
 * whether the destinations are device or host pointers. */
int dsmoe_b200_layer_get_gate(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, void* gate, int dst_on_device);
int dsmoe_b200_layer_get_block(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, int block, void* w1, void* w3,
                               void* w2, int dst_on_device);
int dsmoe_b200_layer_get_shared(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, int s, void* w1, void* w3,
                                void* w2, int dst_on_device);

/* ---- expert parallelism policy (ep_sim.hpp) ----------------------------- */
/* host arrays; same arithmetic as load_aware_thresholds (ep_sim.hpp:76-89) */
int dsmoe_b200_load_aware_thresholds(const double* loads, int devices, double t_max, double* out);
/* simulate_step (ep_sim.hpp:110-160) for one layer on the device: the batch x
 * (device, T x d) routed without drop, device_loads of the placement
 * device_of (host, E*P block devices over `devices`), uniform or load-aware
 * thresholds, the batch re-routed under each selection's owner-device
 * threshold (2T keeping the policy's band offsets).  Host outputs:
 * pre_loads / post_loads / thresholds (`devices` each), scalars3 = {ideal
 * load, drop rate, speed-up max(pre)/max(post)}, stats (optional).  Optional
 * device outputs: post (the dropped RoutingDecision) and y = moe_forward(x,
 * post) (+ x with DSMOE_B200_RESIDUAL in flags) — simulate_step followed by
 * the forward of dsmoe_sim_ep (capi.cpp:421-429).  The loads are exact: each
 * device's load is its number of kept copies times 1/P, summed as the
 * reference's slot loop sums them. */
int dsmoe_b200_simulate_step(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T, int devices,
                             const int32_t* device_of, const dsmoe_b200_policy* policy, int load_aware,
                             int logits_mode, double* pre_loads, double* post_loads, double* thresholds,
                             double* scalars3, dsmoe_b200_drop_stats_t* stats, const dsmoe_b200_routing* post,
                             void* y, int flags);

#ifdef __cplusplus
}
#endif
#endif /* DSMOE_B200_H */
