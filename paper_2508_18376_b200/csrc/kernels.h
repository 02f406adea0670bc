// Host-side declarations of the kernel launchers (one per .cu file).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace dsb {

// router.cu
struct RouterArgs {
  const float* logits;
  int ld_logits;
  int nsplit;               // > 1: logits = sum of nsplit partial planes (split-K gate), ascending
  long long split_stride;   // elements between planes
  float* logits_sum;        // nsplit > 1: the summed logits are written back here (plane 0)
  int T, E, K, P;
  int kind;
  double t_major, t_minor;
  int keep_top1, normalize;
  const double* t_unit;
  double maj_off, min_off;
  int32_t* idx;
  float* raw;
  double* norm;
  uint8_t* frac;
  int32_t* sel_code;   // T x K : unit * 4 + level, -1 when dropped
  float* sel_raw;      // T x K
  int* cnt_chunk;      // ceil(T/128) x 2E histograms of (unit, level)
  unsigned long long* counters;  // [0] copies with fraction 1, [1] fraction 0.5, [2] error flags of this call,
                                 // [4] sticky error flags (cleared only when reported, dsmoe_b200_ctx_check)
};
struct ImportArgs {
  const int32_t* idx;
  const double* raw;
  const double* frac;
  int T, K, P, nphys, nunits;
  int32_t* sel_code;
  float* sel_raw;
  int* cnt_chunk;
  unsigned long long* counters;
};
constexpr int kRouterChunk = 32;  // tokens per router block (one warp each) / scatter chunk
int launch_router(const RouterArgs& a, cudaStream_t stream);
// K0 + K1 fused (bf16, E <= 64, K <= 16, no split): mapA = x (gate_route_tile_rows()-row boxes),
// mapB = the layer's gate rows (Epad-row boxes); acc = 4 zeroed u64 per context
// sc (optional): 2 x kScCap x kScCodes ints, zero at allocation — the launch adds
// every tile's histogram into its superchunk (gate_route_sc_chunks(T) chunks) of
// buffer acc[4] & 1, clears the other buffer and advances acc[4]; the
// permutation then needs no chunk scan (launch_permute_fused with sc)
constexpr int kScCap = 64, kScCodes = 128;
int launch_gate_route(const CUtensorMap* mapA, const CUtensorMap* mapB, const RouterArgs& r, int epad, int nkb,
                      float* logits_out, unsigned long long* acc, int num_sms, cudaStream_t stream,
                      int* sc = nullptr);
int gate_route_tile_rows();
int gate_route_sc_chunks(int T);
int launch_rate_calibrate(const double* norm, int T, int K, int P, int S, int two_t, int keep_top1, double target,
                          double tol, int iters, unsigned long long* cnt, double* t_unit, int E, double* result,
                          int num_sms, cudaStream_t stream);
int launch_import_routing(const ImportArgs& a, cudaStream_t stream);
int launch_gate_logits_exact(const void* x, int x_bf16, const float* gate, float* out, int T, int d,
                             int E, cudaStream_t stream);

// permute.cu
struct PlanArgs {
  const UnitInfo* units;
  const UnitSeg* seg_routed;   // num_routed segments
  const int* seg_unit;         // optional: unit (index into units) of each segment; identity if null
  int shared_unit0;            // index of the first shared unit in units
  int num_routed, num_shared;
  int T, d;
  int shared_row0;
  GemmTile* tiles1;
  int* n1;
  GemmTile* tiles2;
  int* n2;
  int gather;                  // GEMM1 routed tiles gather A rows from X through row_token
  int tile_m;                  // GEMM1 rows per tile: 128 (single CTA) or 256 (CTA pair); 0 -> 128
  int tile_m2;                 // GEMM2 rows per tile; 0 -> tile_m
};
int launch_scan_plan(const int* cnt_chunk, int nchunks, int E, int* chunk_off, int* code_base, UnitSeg* seg,
                     int* r_total, int* code_tot, const PlanArgs* plan, int num_sms, cudaStream_t stream);
int launch_plan(const PlanArgs& a, int num_sms, cudaStream_t stream);
// scan + segments + ordered scatter (+ work lists) in one cooperative launch
// sc / sc_epoch (E <= 64, after launch_gate_route with sc): chunk offsets from
// the superchunk histograms — no chunk scan, no grid-wide barrier
int launch_permute_fused(const int* cnt_chunk, int nchunks, int E, int* chunk_off, int* code_base, UnitSeg* seg,
                         int* r_total, int* code_tot, const int32_t* sel_code, const float* sel_raw, int T, int K,
                         int32_t* row_token, float* row_scale, int32_t* slot_pos, const PlanArgs* plan, int num_sms,
                         cudaStream_t stream, const int* sc = nullptr, const unsigned long long* sc_epoch = nullptr);
int launch_scatter(const int32_t* sel_code, const float* sel_raw, int T, int K, int E, const int* chunk_off,
                   const int* code_base, int32_t* row_token, float* row_scale, int32_t* slot_pos, cudaStream_t stream);
int launch_gather(const void* x, void* xp, const int32_t* row_token, const int* r_total,
                  int row_bytes, int num_sms, cudaStream_t stream);
int launch_combine(const void* y, int y_bf16, const int32_t* slot_pos, void* out, int T, int d, int K,
                   int S, int shared_row0, int num_sms, cudaStream_t stream, const void* resid = nullptr);
int launch_combine2(const void* y, const void* ysh, int y_bf16, const int32_t* slot_pos, void* out, int T, int d,
                    int K, int S, int shared_row0, int num_sms, cudaStream_t stream, const void* resid = nullptr);
int launch_fill_f32(float* p, float v, long long n, cudaStream_t stream);

// gemm_tc.cu
int launch_gemm_tc(int mode, const CUtensorMap* mapA, const CUtensorMap* mapA2,
                   const CUtensorMap* mapB, const GemmTile* tiles, const int* num_tiles,
                   int max_tiles, void* out, long long ldo, const float* row_scale,
                   int b_box_rows, int num_sms, cudaStream_t stream, const int* row_token = nullptr,
                   const void* gather_src = nullptr, long long gather_ld = 0,
                   const CUtensorMap* mapO = nullptr, int pair = 0, unsigned long long* zero4 = nullptr,
                   int* sched = nullptr);  // CTA pairs: 2 zeroed ints -> tiles claimed dynamically

int gemm_tc_store_box_cols();  // TMA-store box width the gemm_tc build expects (64: SW128, 32: SW64)

// ep.cu (EP with one row per (token, destination rank))
int launch_ep_pack(const int32_t* sel_code, const float* sel_raw, const uint32_t* dest, int T, int K, int N,
                   int* cnt_u, int* cnt_s, int* tot, int32_t* send_token, int32_t* pos_td, int32_t* rec_code,
                   int32_t* rec_row, float* rec_raw, int* r_total, int num_sms, cudaStream_t stream,
                   int rec_stride = 1, long long* counts_out = nullptr);
int launch_ep_local_routing(const int32_t* rec_code, const int32_t* rec_row, const float* rec_raw, long long S,
                            int stride, const long long* src_rec_base, const long long* src_row_base, int N, int K,
                            int E, const unsigned char* hold, int32_t* sel_code, float* sel_raw, int* cnt_chunk,
                            unsigned long long* flags, int num_sms, cudaStream_t stream);
int launch_ep_counts(const int* cnt_chunk, int nchunks, int E, long long* out, cudaStream_t stream);
int launch_ep_thresholds(const long long* counts, int E, int P, int D, const int32_t* device_of, double t_max,
                         int load_aware, double* t_unit, double* loads_out, cudaStream_t stream);
int launch_ep_final_combine(const void* ret, int y_bf16, const int32_t* pos_td, int N, const void* ysh, int S,
                            int shared_row0, void* out, int T, int d, int num_sms, cudaStream_t stream);

// gemm_simt.cu
struct SimtArgs {
  const float* A;
  const float* A2;
  long long lda;
  long long a_rows, a2_rows;
  const float* B;
  long long ldb;
  const GemmTile* tiles;
  const int* num_tiles;
  float* out;
  long long ldo;
  const float* row_scale;
};
int launch_gemm_simt(int mode, const SimtArgs& a, int max_tiles, int num_sms, cudaStream_t stream);

// reconstruct.cu
struct ImpUnitC {
  long long base0, base1;
  int h0, wpad0, wpad1;
};
int launch_importance_tiles(int bf16, const void* x, const int32_t* row_token, int seg_start, int nrows,
                            const void* w13, const ImpUnitC& u, int d, int ffn, int metric, double* v,
                            cudaStream_t s);
int launch_importance_reduce(const double* v, const UnitSeg* seg, int E, int ffn, double* values, cudaStream_t s);
int launch_order_sort(const double* values, int E, int ffn, int32_t* order, cudaStream_t s);
int launch_gather_unit(int bf16, const void* w13_src, void* w13_dst, const void* w2t_src, void* w2t_dst,
                       const int32_t* order, const ImpUnitC& u, int ffn, int d, long long w2t_row0,
                       long long hstride, cudaStream_t s);

// pack.cu
int launch_pack_w13(int src_dt, int dst_dt, const void* w1, const void* w3, int d, int ld, const int* order,
                    int col0, int ncols, void* dst, long long base, int wpad, cudaStream_t s);
int launch_pack_w2t(int src_dt, int dst_dt, const void* w2, int d, const int* order, int row0, int nrows,
                    void* dst, long long drow, int hcol0, long long hstride, cudaStream_t s);
int launch_pack_gate(int src_dt, int dst_dt, const void* gate, int d, int E, void* gateT, float* gate_exact,
                     cudaStream_t s);

// transform.cu (re-grouping of the packed layout, read-back)
struct ColUnit {
  long long dst_row0, src_row0;
  int map_off, ncols;
  float scale;
  int pad;
};
int launch_row_gather(const void* src, void* dst, const long long* dst_row, const long long* src_row, long long n,
                      long long row_bytes, int num_sms, cudaStream_t s);
int launch_col_gather(int bf16, const void* src, void* dst, const ColUnit* units, int nunits, const int* colmap,
                      int rows, long long src_ld, long long dst_ld, cudaStream_t s);
int launch_transpose(int bf16, const void* src, long long src_ld, const long long* rows, long long row0,
                     long long col0, int R, int Ccount, void* out, cudaStream_t s);
int launch_compare_rows(int bf16, const void* a, const void* b, int T, int d, double* out, cudaStream_t s);

}  // namespace dsb

namespace dsb {
int launch_gating_hist(const int32_t* idx, const float* raw, const double* norm, int T, int K, int P, int E,
                       int bins, unsigned long long* counts, unsigned long long* rh, unsigned long long* nh,
                       int num_sms, cudaStream_t stream);
}  // namespace dsb
