// C ABI of libdsmoe_b200.so (include/dsmoe_b200.h) and the C++ host runtime
// behind it: layer packing, workspace management, tensor-map encoding and the
// launch sequence of the MoE-module forward.  Error convention follows the
// reference C ABI (/root/reference/proj/src/capi.cpp:35-58): status codes,
// thread-local message, nothing thrown across the boundary.
#include "../../include/dsmoe_b200.h"

#include <atomic>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.h"

namespace {

using namespace dsb;

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg) { throw Error(code, msg); }
void require(bool ok, int code, const std::string& msg) {
  if (!ok) fail(code, msg);
}
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(DSMOE_E_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}
void launch_check(int rc, const char* what) {
  if (rc == -1) fail(DSMOE_E_INVALID_ARGUMENT, std::string(what) + ": unsupported shape");
  if (rc != 0) {
    const cudaError_t e = cudaGetLastError();
    fail(DSMOE_E_INTERNAL, std::string(what) + ": launch failed: " + cudaGetErrorString(e));
  }
}

thread_local std::string g_last_error;
thread_local int g_launches = 0;
std::atomic<long long> g_launches_total{0};  // every kernel this library launched, process-wide
inline void count_launch(int n) {
  g_launches += n;
  g_launches_total.fetch_add(n, std::memory_order_relaxed);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return DSMOE_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of memory";
    return DSMOE_E_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return DSMOE_E_INTERNAL;
  }
}

// --------------------------------------------------------------- helpers
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  // grow-only allocation; contents are not preserved
  void ensure(size_t n) {
    if (n <= bytes) return;
    release();
    cuda_check(cudaMalloc(&p, n), "cudaMalloc");
    bytes = n;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

int round_up(int v, int m) { return (v + m - 1) / m * m; }
int esize(int dt) { return dt == DSMOE_B200_BF16 ? 2 : 4; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  require(fn != nullptr, DSMOE_E_INTERNAL, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2-D bf16 tensor map: `rows` x `cols` (row stride `ld` elements), box
// 64 columns x box_rows rows, 128-byte swizzle (the UMMA descriptor layout).
CUtensorMap make_map(const void* base, long long rows, long long cols, long long ld, int box_rows,
                     int box_cols = 64) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                 strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, DSMOE_E_INTERNAL,
          "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}

// Rows allocated past the last permuted row: a 256-row tile may overrun.
constexpr long long kRowSlack = 256;

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
  }
  return n;
}

}  // namespace

// ==================================================================== layer
struct dsmoe_b200_layer;
int pair_mask(const dsmoe_b200_layer* L);

struct dsmoe_b200_layer {
  int d = 0, ffn = 0, E = 0, K = 0, S = 0, P = 1, prenorm = 0, dtype = DSMOE_B200_BF16;
  std::vector<int> widths, swidths;
  std::vector<UnitInfo> units;  // E routed units then S shared units
  int hstride = 0;
  long long w13_rows = 0;
  int Epad = 0;  // gate rows padded to 32 (UMMA N of the gate GEMM)
  int max_chunks = 0;
  DevBuf w13, w2t, gateT, gate_exact, d_units;
  CUtensorMap map_w13{}, map_w2t{}, map_gate{};
  CUtensorMap map_w13_h{}, map_w2t_h{};  // 128-row boxes: half-N B tiles of the CTA-pair GEMM
  std::vector<char> block_set, shared_set;
  bool gate_set = false;
  // lazily built "block view" of a P > 1 layer: every physical block its own
  // unit, so a RoutingDecision outside the canonical replayed layout (any
  // block, any fraction per slot, moe.hpp:239-271) runs on the same kernels
  mutable dsmoe_b200_layer* bview = nullptr;
  mutable std::mutex bview_mu;
  // expert shard (expert parallelism): held[b] marks the physical blocks this
  // layer stores (empty = all).  A routed unit's sub-blocks are its held
  // blocks in order, so the blocks of one expert may live on different ranks
  // (S-ETP placement); the gate and the shared experts are whole.
  std::vector<char> held;
  DevBuf d_hold;  // per routed unit: bit 0 any block held, bit 1 block 0 held
  ~dsmoe_b200_layer();

  int nunits() const { return E + S; }
  bool held_block(int b) const { return held.empty() || held[static_cast<size_t>(b)]; }
  bool sharded() const {
    for (char h : held)
      if (!h) return true;
    return false;
  }
  bool holds(int unit) const {
    if (unit >= E || held.empty()) return true;
    for (int p = 0; p < P; ++p)
      if (held[static_cast<size_t>(unit * P + p)]) return true;
    return false;
  }
  // index of block (e, p) among unit e's stored sub-blocks
  int local_sub(int b) const {
    int q = 0;
    for (int i = (b / P) * P; i < b; ++i) q += held_block(i) ? 1 : 0;
    return q;
  }
  // sub-block p of routed unit e <- block (e, p) columns [col0, col0 + n)
  void check_ready() const {
    require(gate_set, DSMOE_E_INVALID_STATE, "layer: gate weights not set");
    for (size_t b = 0; b < block_set.size(); ++b)
      require(block_set[b], DSMOE_E_INVALID_STATE, "layer: expert block " + std::to_string(b) + " not set");
    for (size_t s = 0; s < shared_set.size(); ++s)
      require(shared_set[s], DSMOE_E_INVALID_STATE, "layer: shared expert " + std::to_string(s) + " not set");
  }
};

dsmoe_b200_layer::~dsmoe_b200_layer() { delete bview; }

int pair_mask(const dsmoe_b200_layer* L) {
  // Which grouped GEMMs run on CTA pairs (tcgen05 cta_group::2, M = 256
  // tiles): bit 0 GEMM1, bit 1 GEMM2.  Default: both — GEMM2 15% and GEMM1
  // (fused gather, CTA-scope stage hand-off) 11% fewer cycles than
  // single-CTA tiles (profiles/r12_summary.md, r13_summary.md).
  // DSMOE_B200_CTA_PAIR: digits '1' / '2' select GEMM1 / GEMM2, "0" none.
  static const int mask = [] {
    const char* v = std::getenv("DSMOE_B200_CTA_PAIR");
    if (!v) return 3;
    const std::string sv(v);
    return (sv.find('1') != std::string::npos ? 1 : 0) | (sv.find('2') != std::string::npos ? 2 : 0);
  }();
  return L->dtype == DSMOE_B200_BF16 ? mask : 0;
}

namespace {

void layer_build(dsmoe_b200_layer* L, const dsmoe_b200_layer_config& c, bool ragged = false,
                 const char* held = nullptr) {
  require(c.d_model >= 1, DSMOE_E_INVALID_ARGUMENT, "config: d_model must be >= 1");
  require(c.d_ffn >= 2, DSMOE_E_INVALID_ARGUMENT, "config: d_ffn must be >= 2");
  require(c.num_experts >= 1, DSMOE_E_INVALID_ARGUMENT, "config: num_experts must be >= 1");
  require(c.top_k >= 1 && c.top_k <= c.num_experts, DSMOE_E_INVALID_ARGUMENT,
          "config: top_k must satisfy 1 <= K <= E");
  require(c.num_shared_experts >= 0, DSMOE_E_INVALID_ARGUMENT, "config: num_shared_experts must be >= 0");
  require(c.replay_factor >= 1 && c.replay_factor <= kMaxSub, DSMOE_E_INVALID_STATE,
          "layer: replay_factor must be in [1, 8]");
  require(c.dtype == DSMOE_B200_F32 || c.dtype == DSMOE_B200_BF16, DSMOE_E_INVALID_ARGUMENT,
          "layer: dtype must be f32 or bf16");
  require(c.d_model % 64 == 0, DSMOE_E_SHAPE_MISMATCH, "layer: d_model must be a multiple of 64 on device");
  require(c.num_experts <= 256, DSMOE_E_INVALID_ARGUMENT, "layer: at most 256 experts on device");
  require(c.top_k <= 16, DSMOE_E_INVALID_ARGUMENT, "layer: top_k must be <= 16 on device");
  L->d = c.d_model;
  L->ffn = c.d_ffn;
  L->E = c.num_experts;
  L->K = c.top_k;
  L->S = c.num_shared_experts;
  L->P = c.replay_factor;
  L->prenorm = c.gate_prenormalized != 0;
  L->dtype = c.dtype;
  const int P = L->P;
  if (held) L->held.assign(held, held + static_cast<size_t>(c.num_experts) * c.replay_factor);
  for (int b = 0; b < L->E * P; ++b) L->widths.push_back(c.block_widths ? c.block_widths[b] : c.d_ffn / P);
  for (int s = 0; s < L->S; ++s) L->swidths.push_back(c.shared_widths ? c.shared_widths[s] : c.d_ffn);
  for (int e = 0; e < L->E; ++e) {
    int tot = 0;
    for (int p = 0; p < P; ++p) {
      require(L->widths[e * P + p] >= 1, DSMOE_E_SHAPE_MISMATCH, "layer: block widths must be >= 1");
      tot += L->widths[e * P + p];
    }
    require(ragged || tot == L->ffn, DSMOE_E_INVALID_STATE,
            "layer: block widths of expert " + std::to_string(e) + " sum to " + std::to_string(tot) +
                ", expected " + std::to_string(L->ffn));
  }
  long long row = 0;
  int hmax = 0, chmax = 0, w2t_units = 0;
  for (int e = 0; e < L->E + L->S; ++e) {
    UnitInfo u{};
    const bool sh = e >= L->E;
    std::vector<int> w;
    if (sh) {
      w = {L->swidths[e - L->E]};
    } else if (P == 1) {
      // virtual split at ceil(w/2): fraction 0.5 evaluates the first half
      // (moe.hpp:264), i.e. sub-block 0; the routed layer needs no copy.
      if (L->held_block(e)) {
        const int wd = L->widths[e], h0 = (wd + 1) / 2;
        w = {h0};
        if (wd - h0 > 0) w.push_back(wd - h0);
      }
    } else {
      for (int p = 0; p < P; ++p)
        if (L->held_block(e * P + p)) w.push_back(L->widths[e * P + p]);
    }
    u.nsub = static_cast<int>(w.size());
    u.hwidth = 0;
    int chunks = 0;
    for (int p = 0; p < u.nsub; ++p) {
      u.sub_w[p] = w[p];
      u.sub_wpad[p] = round_up(w[p], 64);
      u.hwidth += u.sub_wpad[p];
      chunks += (u.sub_wpad[p] + kChunk - 1) / kChunk;
    }
    u.shared = sh ? 1 : 0;
    if (!w.empty()) {  // units without held blocks (expert shards) have no storage
      u.w13_row = static_cast<int>(row);
      u.w2t_row = w2t_units++ * L->d;
      row += 2LL * u.hwidth;
    }
    hmax = std::max(hmax, u.hwidth);
    chmax = std::max(chmax, chunks);
    L->units.push_back(u);
  }
  require(row < (1LL << 31) && static_cast<long long>(w2t_units) * L->d < (1LL << 31),
          DSMOE_E_INVALID_ARGUMENT, "layer: packed weights exceed 2^31 rows");
  L->w13_rows = row;
  L->hstride = hmax;
  L->max_chunks = chmax;
  L->Epad = round_up(L->E, 32);
  const int es = esize(L->dtype);
  L->w13.ensure(static_cast<size_t>(row) * L->d * es);
  L->w2t.ensure(static_cast<size_t>(w2t_units) * L->d * L->hstride * es);
  L->gateT.ensure(static_cast<size_t>(L->Epad) * L->d * es);
  L->gate_exact.ensure(static_cast<size_t>(L->d) * L->E * 4);
  cuda_check(cudaMemset(L->w13.p, 0, L->w13.bytes), "memset");
  cuda_check(cudaMemset(L->w2t.p, 0, L->w2t.bytes), "memset");
  cuda_check(cudaMemset(L->gateT.p, 0, L->gateT.bytes), "memset");
  L->d_units.ensure(sizeof(UnitInfo) * L->units.size());
  cuda_check(cudaMemcpy(L->d_units.p, L->units.data(), sizeof(UnitInfo) * L->units.size(),
                        cudaMemcpyHostToDevice),
             "upload units");
  if (L->dtype == DSMOE_B200_BF16) {
    L->map_w13 = make_map(L->w13.p, row, L->d, L->d, 256);
    L->map_w2t = make_map(L->w2t.p, static_cast<long long>(w2t_units) * L->d, L->hstride, L->hstride, 256);
    L->map_w13_h = make_map(L->w13.p, row, L->d, L->d, 128);
    L->map_w2t_h = make_map(L->w2t.p, static_cast<long long>(w2t_units) * L->d, L->hstride, L->hstride, 128);
    L->map_gate = make_map(L->gateT.p, L->Epad, L->d, L->d, L->Epad);
  }
  L->block_set.assign(static_cast<size_t>(L->E * P), 0);
  for (int b = 0; b < L->E * P; ++b)
    if (!L->held_block(b)) L->block_set[static_cast<size_t>(b)] = 1;  // not part of this shard
  if (L->sharded()) {
    std::vector<unsigned char> hold(static_cast<size_t>(L->E));
    for (int e = 0; e < L->E; ++e)
      hold[static_cast<size_t>(e)] = (L->holds(e) ? 1 : 0) | (L->held_block(e * P) ? 2 : 0);
    L->d_hold.ensure(hold.size());
    cuda_check(cudaMemcpy(L->d_hold.p, hold.data(), hold.size(), cudaMemcpyHostToDevice), "upload shard");
  }
  L->shared_set.assign(static_cast<size_t>(L->S), 0);
}

// Source staging: host sources are copied to a temporary device buffer.
struct Staged {
  DevBuf buf;
  const void* p = nullptr;
  Staged(const void* src, size_t bytes, int on_device, cudaStream_t s) {
    if (on_device) {
      p = src;
    } else {
      buf.ensure(bytes);
      cuda_check(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, s), "stage H2D");
      p = buf.p;
    }
  }
};

// Pack sub-block p of unit u from a source block (w1/w3: d x ld, w2: ld x d);
// neurons [col0, col0 + n) of the source, optionally through `order`.
void pack_sub(dsmoe_b200_layer* L, int u, int p, const void* w1, const void* w3, const void* w2, int ld,
              const int* order, int col0, int src_dt, cudaStream_t s) {
  const UnitInfo& ui = L->units[u];
  long long base = ui.w13_row;
  int hcol = 0;
  for (int q = 0; q < p; ++q) {
    base += 2LL * ui.sub_wpad[q];
    hcol += ui.sub_wpad[q];
  }
  launch_check(launch_pack_w13(src_dt, L->dtype, w1, w3, L->d, ld, order, col0, ui.sub_w[p], L->w13.p, base,
                               ui.sub_wpad[p], s),
               "pack_w13");
  launch_check(launch_pack_w2t(src_dt, L->dtype, w2, L->d, order, col0, ui.sub_w[p], L->w2t.p,
                               ui.w2t_row, hcol, L->hstride, s),
               "pack_w2t");
}

// ------------------------------------------------ re-grouping (transform.cu)
// Neuron n of a unit, counted over the concatenated true widths of its
// sub-blocks -> (sub-block, index inside it).
struct NeuronLoc {
  int sub, i;
};
NeuronLoc neuron_loc(const UnitInfo& u, int n) {
  for (int p = 0; p < u.nsub; ++p) {
    if (n < u.sub_w[p]) return {p, n};
    n -= u.sub_w[p];
  }
  fail(DSMOE_E_INTERNAL, "neuron_loc: neuron outside the unit");
}
long long sub_w13_base(const UnitInfo& u, int p) {
  long long b = u.w13_row;
  for (int q = 0; q < p; ++q) b += 2LL * u.sub_wpad[q];
  return b;
}
int sub_hcol(const UnitInfo& u, int p) {
  int h = 0;
  for (int q = 0; q < p; ++q) h += u.sub_wpad[q];
  return h;
}

template <class T>
struct Staging {  // host vector -> device copy (freed after the stream syncs)
  DevBuf buf;
  T* put(const std::vector<T>& v, cudaStream_t s) {
    buf.ensure(sizeof(T) * std::max<size_t>(1, v.size()));
    if (!v.empty()) cuda_check(cudaMemcpyAsync(buf.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, s), "H2D");
    return buf.as<T>();
  }
};

// Fill the packed weights of R from L: dst unit u' takes its neurons from src
// unit src_unit[u'] through nmap(u', n') -> n (concatenated true-width
// indices), W2 scaled by scale[u'].  gmap[e'] = src gate column of dst gate
// column e' (the gate is re-grouped too: complete_transform repeats columns).
template <class NMap>
void regroup(const dsmoe_b200_layer* L, dsmoe_b200_layer* R, const std::vector<int>& src_unit,
             const std::vector<float>& scale, NMap nmap, const std::vector<int>& gmap, cudaStream_t s) {
  const int es = esize(L->dtype);
  std::vector<long long> drow, srow;
  std::vector<int> colmap(static_cast<size_t>(R->nunits()) * R->hstride, -1);
  std::vector<ColUnit> cu;
  for (int v = 0; v < R->nunits(); ++v) {
    if (!R->holds(v)) continue;
    const UnitInfo& du = R->units[v];
    const UnitInfo& su = L->units[src_unit[v]];
    require(L->holds(src_unit[v]), DSMOE_E_INVALID_STATE, "regroup: source unit not held by this expert shard");
    int off = 0;
    for (int p = 0; p < du.nsub; ++p) {
      const long long db = sub_w13_base(du, p);
      const int dh = sub_hcol(du, p);
      for (int i = 0; i < du.sub_wpad[p]; ++i) {
        long long s1 = -1, s3 = -1;
        if (i < du.sub_w[p]) {
          const NeuronLoc sl = neuron_loc(su, nmap(v, off + i));
          const long long sb = sub_w13_base(su, sl.sub);
          s1 = w13_row_of(sb, sl.i, 0);
          s3 = w13_row_of(sb, sl.i, 1);
          colmap[static_cast<size_t>(v) * R->hstride + dh + i] = sub_hcol(su, sl.sub) + sl.i;
        }
        drow.push_back(w13_row_of(db, i, 0));
        srow.push_back(s1);
        drow.push_back(w13_row_of(db, i, 1));
        srow.push_back(s3);
      }
      off += du.sub_w[p];
    }
    cu.push_back(ColUnit{du.w2t_row, su.w2t_row, v * R->hstride, R->hstride, scale[v], 0});
  }
  Staging<long long> sd, ss;
  Staging<int> sc, sg;
  Staging<ColUnit> su;
  launch_check(launch_row_gather(L->w13.p, R->w13.p, sd.put(drow, s), ss.put(srow, s), static_cast<long long>(drow.size()),
                                 static_cast<long long>(L->d) * es, num_sms(), s),
               "regroup W13");
  launch_check(launch_col_gather(L->dtype == DSMOE_B200_BF16, L->w2t.p, R->w2t.p, su.put(cu, s),
                                 static_cast<int>(cu.size()), sc.put(colmap, s), L->d, L->hstride, R->hstride, s),
               "regroup W2T");
  // gate: gateT rows (Epad x d, layer dtype) and the exact-mode d x E fp32 copy
  std::vector<long long> gd, gs;
  for (int e = 0; e < R->Epad; ++e) {
    gd.push_back(e);
    gs.push_back(e < R->E ? gmap[e] : -1);
  }
  Staging<long long> sgd, sgs;
  launch_check(launch_row_gather(L->gateT.p, R->gateT.p, sgd.put(gd, s), sgs.put(gs, s), R->Epad,
                                 static_cast<long long>(L->d) * es, num_sms(), s),
               "regroup gate");
  std::vector<ColUnit> gu{ColUnit{0, 0, 0, R->E, 1.0f, 0}};
  Staging<ColUnit> sgu;
  launch_check(launch_col_gather(0, L->gate_exact.p, R->gate_exact.p, sgu.put(gu, s), 1, sg.put(gmap, s), L->d, L->E,
                                 R->E, s),
               "regroup exact gate");
  count_launch(4);
  cuda_check(cudaStreamSynchronize(s), "sync");
  R->gate_set = L->gate_set;
  std::fill(R->block_set.begin(), R->block_set.end(), 1);
  std::fill(R->shared_set.begin(), R->shared_set.end(), 1);
}

constexpr int kModeComplete = 0, kModePartial = 1, kModeReverse = 2, kModeBlocks = 3;

// complete_transform / partial_transform / reverse_partial (transform.hpp:66-170)
// or the block view of a device layer, as a new device layer.
dsmoe_b200_layer* transform_layer(const dsmoe_b200_layer* L, int mode, int p, cudaStream_t s) {
  require(!L->sharded(), DSMOE_E_INVALID_STATE, "transform: layer is an expert shard");
  std::vector<int32_t> widths, swidths(L->swidths.begin(), L->swidths.end());
  dsmoe_b200_layer_config cfg{L->d, L->ffn, L->E, L->K, L->S, L->prenorm, 1, L->dtype, nullptr, nullptr};
  std::vector<int> src_unit, gmap;
  std::vector<float> scale;
  std::function<int(int, int)> nmap;
  if (mode == kModeComplete || mode == kModePartial) {
    const char* who = mode == kModeComplete ? "complete_transform" : "partial_transform";
    require(L->P == 1, DSMOE_E_INVALID_STATE, std::string(who) + ": layer already carries a partial transformation");
    require(p >= 2, DSMOE_E_INVALID_ARGUMENT, std::string(who) + ": p must be >= 2");
    require(L->ffn % p == 0, DSMOE_E_INVALID_ARGUMENT,
            std::string(who) + ": d_ffn " + std::to_string(L->ffn) + " not divisible by p " + std::to_string(p));
  }
  const int c = (mode == kModeComplete || mode == kModePartial) ? L->ffn / p : 0;
  if (mode == kModeComplete) {
    cfg.d_ffn = c;
    cfg.num_experts = L->E * p;
    cfg.top_k = L->K * p;
    for (int e = 0; e < L->E * p; ++e) widths.push_back(c);
    for (int e = 0; e < L->E; ++e)
      for (int q = 0; q < p; ++q) {
        src_unit.push_back(e);
        scale.push_back(static_cast<float>(p));
        gmap.push_back(e);
      }
    nmap = [c, p](int v, int n) { return (v % p) * c + n; };
  } else if (mode == kModePartial) {
    cfg.replay_factor = p;
    for (int e = 0; e < L->E * p; ++e) widths.push_back(c);
    for (int e = 0; e < L->E; ++e) {
      src_unit.push_back(e);
      scale.push_back(1.0f);
      gmap.push_back(e);
    }
    nmap = [](int, int n) { return n; };
  } else if (mode == kModeReverse) {
    require(L->P > 1, DSMOE_E_INVALID_STATE, "reverse: layer does not carry a partial transformation");
    for (int e = 0; e < L->E; ++e) {
      widths.push_back(L->ffn);
      src_unit.push_back(e);
      scale.push_back(1.0f);
      gmap.push_back(e);
    }
    nmap = [](int, int n) { return n; };
  } else {  // block view: unit b = e*P + q <- sub-block q of unit e
    const int P = L->P;
    cfg.num_experts = L->E * P;
    cfg.top_k = L->K * P;
    cfg.d_ffn = *std::max_element(L->widths.begin(), L->widths.end());
    for (int b = 0; b < L->E * P; ++b) {
      widths.push_back(L->widths[b]);
      src_unit.push_back(b / P);
      scale.push_back(1.0f);
      gmap.push_back(std::min(b / P, L->E - 1));
    }
    nmap = [L, P](int v, int n) {
      const UnitInfo& u = L->units[v / P];
      int off = 0;
      for (int q = 0; q < v % P; ++q) off += u.sub_w[q];
      return off + n;
    };
  }
  for (int si = 0; si < L->S; ++si) {
    src_unit.push_back(L->E + si);
    scale.push_back(1.0f);
  }
  require(cfg.num_experts <= 256 && cfg.top_k <= 16, DSMOE_E_INVALID_ARGUMENT,
          "transform: the result exceeds the device limits (256 experts, top_k 16)");
  cfg.block_widths = widths.data();
  cfg.shared_widths = swidths.empty() ? nullptr : swidths.data();
  auto* R = new dsmoe_b200_layer;
  try {
    // block view: block widths need not sum to a common d_ffn (major / minor halves)
    layer_build(R, cfg, /*ragged=*/mode == kModeBlocks);
    const int nE = R->E;
    auto full = [&](int v, int n) { return v < nE ? nmap(v, n) : n; };
    regroup(L, R, src_unit, scale, full, gmap, s);
  } catch (...) {
    delete R;
    throw;
  }
  return R;
}

}  // namespace

// ====================================================================== ctx
struct dsmoe_b200_ctx {
  cudaStream_t stream = nullptr;
  DevBuf logits, sel_code, sel_raw, slot_pos, cnt_chunk, chunk_off, code_base, counters, row_token, row_scale, seg,
      scalars;
  DevBuf tiles1, tiles2, tiles_gate, xperm, H, Y, frac_ws, vseg, vseg_unit;
  DevBuf rate_norm, rate_cnt, rate_tunit, rate_result;  // rate-targeted drop (dsmoe_b200_forward_rate)
  // superchunk histograms of the fused gate + router (2 x kScCap x kScCodes,
  // zero at allocation, double-buffered by counters[12]); sc_T = token count of
  // the last routing that filled them, -1 when cnt_chunk came from elsewhere
  DevBuf sc_hist;
  int sc_T = -1;
  // dynamic tile claims of the CTA-pair GEMMs: [GEMM1 claim, done, GEMM2 claim, done], zero between launches
  DevBuf gsched;
  // EP with one row per (token, rank): last ep_pack's layout on this context
  DevBuf ep_pos_td, ep_send_token, ep_cnt, ep_tot, ep_owner, ep_base;
  int ep_N = 0, ep_T = -1;
  int gate_tiles_T = -1, gate_tiles_Epad = -1, gate_tiles_d = -1, gate_tiles_S = -1;
  // logits left in `logits` by the last routing on this context (LOGITS_REUSE)
  const void* logits_layer = nullptr;
  int logits_T = -1, logits_ld = 0;
  int routed_T = -1;  // token count of the last routing (any logits source)
  long long scale_fill_key = -1;
  unsigned long long last_err_flags = 0;
  // optional per-stage CUDA-event timing (bench.py): 0 gate, 1 router,
  // 2 permute+plan, 3 gather, 4 gemm1, 5 gemm2, 6 combine.  Non-blocking: each
  // forward records into its own event set from a ring; the sets are resolved
  // (synchronised and summed) only when the profile is read or the ring is
  // full, so timing can run inside a back-to-back timed loop.
  static constexpr int kStages = 7;
  static constexpr int kRing = 256;
  struct EvSet {
    cudaEvent_t ev[kStages + 1] = {};
    bool hit[kStages + 1] = {};
  };
  bool profiling = false;
  int prof_period = 1;    // profile every prof_period-th forward (the others run unmarked)
  long prof_seen = 0;
  std::vector<EvSet> ring;
  int ring_head = 0, ring_pending = 0;
  EvSet* cur = nullptr;
  double prof_ms[kStages] = {};
  long prof_calls = 0;
  void mark(int i) {
    if (!profiling || !cur) return;
    cuda_check(cudaEventRecord(cur->ev[i], stream), "event");
    cur->hit[i] = true;
  }
  void prof_begin() {
    cur = nullptr;
    if (!profiling || (prof_seen++ % prof_period) != 0) return;
    if (ring.empty()) {
      ring.resize(kRing);
      for (auto& es : ring)
        for (auto& e : es.ev) cuda_check(cudaEventCreate(&e), "event create");
    }
    if (ring_pending == kRing) resolve();
    cur = &ring[(ring_head + ring_pending) % kRing];
    for (auto& h : cur->hit) h = false;
  }
  void prof_end() {
    if (!profiling || !cur) return;
    mark(kStages);
    cur = nullptr;
    ++ring_pending;
  }
  void resolve() {
    for (; ring_pending > 0; --ring_pending, ring_head = (ring_head + 1) % kRing) {
      EvSet& es = ring[ring_head];
      cuda_check(cudaEventSynchronize(es.ev[kStages]), "event sync");
      int prev = -1;
      for (int i = 0; i <= kStages; ++i) {
        if (!es.hit[i]) continue;
        if (prev >= 0) {
          float ms = 0.f;
          cuda_check(cudaEventElapsedTime(&ms, es.ev[prev], es.ev[i]), "elapsed");
          prof_ms[prev] += ms;
        }
        prev = i;
      }
      ++prof_calls;
    }
  }
  ~dsmoe_b200_ctx() {
    for (auto& es : ring)
      for (auto& e : es.ev)
        if (e) cudaEventDestroy(e);
  }

  // workspace for T tokens on layer L
  void ensure(const dsmoe_b200_layer* L, int T) {
    const int es = esize(L->dtype);
    const long long TK = static_cast<long long>(T) * L->K;
    const long long Rcap = TK;
    const long long rows = Rcap + static_cast<long long>(L->S) * T + kRowSlack;
    logits.ensure(static_cast<size_t>(T) * L->Epad * 4 + 16);
    sel_code.ensure(static_cast<size_t>(TK) * 4 + 16);
    sel_raw.ensure(static_cast<size_t>(TK) * 4 + 16);
    slot_pos.ensure(static_cast<size_t>(TK) * 4 + 16);
    const size_t nchunks = static_cast<size_t>((T + kRouterChunk - 1) / kRouterChunk);
    cnt_chunk.ensure(nchunks * 2 * L->E * 4 + 16);
    chunk_off.ensure(nchunks * 2 * L->E * 4 + 16);
    code_base.ensure(static_cast<size_t>(4 * L->E) * 4);  // [2E bases | 2E totals]
    if (!counters.p) {  // [0..3] per call (zeroed by each routing), [4] sticky error flags,
                        // [8..11] the fused gate + router's accumulators (zero between launches)
      counters.ensure(16 * sizeof(unsigned long long));
      cuda_check(cudaMemsetAsync(counters.p, 0, counters.bytes, stream), "memset");
    }
    if (!gsched.p) {
      gsched.ensure(4 * sizeof(int));
      cuda_check(cudaMemsetAsync(gsched.p, 0, gsched.bytes, stream), "memset");
    }
    if (!sc_hist.p) {
      sc_hist.ensure(2ull * kScCap * kScCodes * sizeof(int));
      cuda_check(cudaMemsetAsync(sc_hist.p, 0, sc_hist.bytes, stream), "memset");
    }
    row_token.ensure(static_cast<size_t>(Rcap + kRowSlack) * 4);
    seg.ensure(sizeof(UnitSeg) * L->E);
    scalars.ensure(4 * sizeof(int));  // r_total, n1, n2, ngate
    const long long mt = (Rcap + kTileM - 1) / kTileM + 2LL * L->E;  // + per-unit ceil and full/major split
    const long long mts = static_cast<long long>(L->S) * ((T + kTileM - 1) / kTileM);
    const long long t1 = (mt + mts) * L->max_chunks;
    const long long t2 = (mt + mts) * ((L->d + kTileN2 - 1) / kTileN2);
    tiles1.ensure(static_cast<size_t>(t1 + 1) * sizeof(GemmTile));
    tiles2.ensure(static_cast<size_t>(t2 + 1) * sizeof(GemmTile));
    xperm.ensure(static_cast<size_t>(Rcap + kRowSlack) * L->d * es);
    H.ensure(static_cast<size_t>(rows) * L->hstride * es);
    Y.ensure(static_cast<size_t>(rows) * L->d * es);
    const size_t rs_bytes = static_cast<size_t>(rows) * 4;
    if (row_scale.bytes < rs_bytes) {
      row_scale.ensure(rs_bytes);
      scale_fill_key = -1;
    }
    // shared-expert rows are weighted 1 (moe.hpp:267-268)
    const long long key = (Rcap << 20) ^ (static_cast<long long>(L->S) * T);
    if (L->S > 0 && scale_fill_key != key) {
      launch_check(launch_fill_f32(row_scale.as<float>() + Rcap, 1.0f, static_cast<long long>(L->S) * T, stream),
                   "fill");
      count_launch(1);
      scale_fill_key = key;
    }
  }
  long long max_tiles1(const dsmoe_b200_layer* L, int T) const {
    const long long Rcap = static_cast<long long>(T) * L->K;
    const long long mt = (Rcap + kTileM - 1) / kTileM + 2LL * L->E;
    const long long mts = static_cast<long long>(L->S) * ((T + kTileM - 1) / kTileM);
    return (mt + mts) * L->max_chunks;
  }
  long long max_tiles2(const dsmoe_b200_layer* L, int T) const {
    const long long Rcap = static_cast<long long>(T) * L->K;
    const long long mt = (Rcap + kTileM - 1) / kTileM + 2LL * L->E;
    const long long mts = static_cast<long long>(L->S) * ((T + kTileM - 1) / kTileM);
    return (mt + mts) * ((L->d + kTileN2 - 1) / kTileN2);
  }
};

namespace {

struct PolicyResolved {
  int kind = 0;
  double t_drop = 0, t_major = 0, t_minor = 0;
  int keep_top1 = 1, normalize = 1;
  const double* t_unit = nullptr;
  double maj_off = 0, min_off = 0;
};

PolicyResolved resolve_policy(const dsmoe_b200_layer* L, const dsmoe_b200_policy* p) {
  PolicyResolved r;
  r.normalize = !L->prenorm;
  if (!p) return r;
  require(p->kind >= 0 && p->kind <= 2, DSMOE_E_INVALID_ARGUMENT, "policy: kind must be none, 1t or 2t");
  r.kind = p->kind;
  r.t_drop = p->t_drop;
  r.keep_top1 = p->keep_top1 != 0;
  if (p->normalize >= 0) r.normalize = p->normalize != 0;
  if (r.kind == DSMOE_B200_DROP_1T) {
    r.t_major = r.t_minor = p->t_drop;  // drop_1t (dropping.hpp:133-138)
  } else if (r.kind == DSMOE_B200_DROP_2T) {
    require(p->t_major <= p->t_minor, DSMOE_E_INVALID_ARGUMENT, "drop policy: t_major must be <= t_minor");
    // drop_2t (dropping.hpp:147-148) / map_from_layer (:233-234)
    require(L->P == 2, DSMOE_E_INVALID_STATE, "drop_2t: routing must be replayed with P=2");
    r.t_major = p->t_major;
    r.t_minor = p->t_minor;
  }
  r.t_unit = p->t_unit;
  if (r.kind == DSMOE_B200_DROP_2T) {  // ep_sim.hpp:139-142
    r.maj_off = p->t_major - p->t_drop;
    r.min_off = p->t_minor - p->t_drop;
  }
  return r;
}

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

// drop_stats (dropping.hpp:171-195) from retained-copy counts.  With P a
// power of two every partial sum of fraction/P is exact, so the counts give
// the reference's sequential sums bit for bit.
void stats_from_counts(const dsmoe_b200_layer* L, int T, unsigned long long n1, unsigned long long nh,
                       const uint8_t* frac_host, dsmoe_b200_drop_stats_t* st) {
  const long long n = static_cast<long long>(T) * L->K * L->P;
  const double w = 1.0 / L->P;
  double total = 0.0, retained = 0.0;
  if (is_pow2(L->P)) {
    total = static_cast<double>(n) * w;
    retained = static_cast<double>(2 * n1 + nh) * (0.5 * w);
  } else {
    for (long long i = 0; i < n; ++i) {
      total += 1.0 * w;
      const double f = frac_host[i] == 2 ? 1.0 : (frac_host[i] == 1 ? 0.5 : 0.0);
      retained += f * w;
    }
  }
  st->num_tokens = T;
  st->total_routed_units = total;
  st->dropped_units = total - retained;
  st->shared_units = static_cast<double>(L->S) * T;
  const double denom = st->total_routed_units + st->shared_units;
  st->drop_rate = denom > 0.0 ? st->dropped_units / denom : 0.0;
  const double unit = 6.0 * L->d * L->ffn;
  st->total_flops = denom * unit;
  st->saved_flops = st->dropped_units * unit;
  st->retained_flops = st->total_flops - st->saved_flops;
}

// Error flags raised on the device.  counters[2] belongs to the last call;
// counters[4] is sticky: a forward launched without stats (no host sync)
// still reports its degenerate-normalisation error (normalize_topk throws,
// dropping.hpp:67) at the next synchronising call on the context.
void raise_flags(unsigned long long f) {
  if (f & 1ull) fail(DSMOE_E_INVALID_ARGUMENT, "normalize_topk: degenerate zero-sum scores");
  if (f & 4ull)
    fail(DSMOE_E_INVALID_STATE,
         "moe_forward: routing has an expert index out of range or a compute fraction outside {0, 0.5, 1}");
}

// read counters[0..4] after the work queued so far (synchronises the stream);
// sticky flags are cleared once reported
void read_counters(dsmoe_b200_ctx* C, unsigned long long* h5) {
  cuda_check(cudaMemcpyAsync(h5, C->counters.p, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, C->stream),
             "D2H counters");
  cuda_check(cudaStreamSynchronize(C->stream), "sync");
  const unsigned long long f = h5[2] | h5[4] | C->last_err_flags;
  C->last_err_flags = 0;
  if (h5[2] | h5[4]) {  // report once: the next check on this context starts clean
    cuda_check(cudaMemsetAsync(C->counters.as<unsigned long long>() + 2, 0, 8, C->stream), "memset");
    cuda_check(cudaMemsetAsync(C->counters.as<unsigned long long>() + 4, 0, 8, C->stream), "memset");
  }
  raise_flags(f);
}

void check_flags(dsmoe_b200_ctx* C) {
  unsigned long long h[5];
  read_counters(C, h);
}

// -------------------------------------------------- stage: gate logits + K1
void stage_route(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                 const PolicyResolved& pol, int logits_mode, const float* logits_in, float* logits_out,
                 const dsmoe_b200_routing* out, uint8_t* frac_ws, int logits_in_ld = 0) {
  cudaStream_t s = C->stream;
  bool counters_zeroed = false;  // the tensor-core gate kernel zeroes them in its prologue
  bool fused = false;            // gate + router in one launch (tensor-mode logits)
  const float* lg = logits_in;
  int ld = logits_in_ld > 0 ? logits_in_ld : L->E;
  C->routed_T = T;
  int nsplit = 1;               // split-K gate: partial logit planes the router sums
  long long split_stride = 0;
  C->mark(0);
  if (!lg && logits_mode == DSMOE_B200_LOGITS_REUSE) {
    require(C->logits_layer == L && C->logits_T == T, DSMOE_E_INVALID_STATE,
            "logits reuse: the previous routing on this context was for another layer or batch");
    lg = C->logits.as<float>();
    ld = C->logits_ld;
  }
  if (!lg) {
    const bool tc = logits_mode == DSMOE_B200_LOGITS_TENSOR && L->dtype == DSMOE_B200_BF16;
    // K0 + K1 in one kernel (gate_route_kernel, router.cu) unless a split gate
    // is asked for; DSMOE_B200_GATE_ROUTE=0 keeps the two-kernel chain (A/B)
    static const bool fuse_env = [] {
      const char* v = std::getenv("DSMOE_B200_GATE_ROUTE");
      return !v || std::atoi(v) != 0;
    }();
    static const bool split_req = [] {
      const char* v = std::getenv("DSMOE_B200_GATE_SPLIT");
      return v && std::atoi(v) > 1;
    }();
    fused = tc && fuse_env && !split_req && L->E <= 64 && L->K <= 16;
    if (fused) {
      C->logits.ensure(static_cast<size_t>(T) * L->Epad * 4 + 16);
      ld = L->Epad;
    } else if (tc) {
      // K may be split into S pieces over S CTAs per 128-token tile (partial
      // fp32 logit planes the router sums in ascending order and writes
      // back).  S depends on the layer only, never on T, so a token's logits
      // — and its top-K / drop band on near-ties — do not change with the
      // batch it rides in (EP ranks with different shard sizes route
      // identical tokens identically).  Default S = 1: a second
      // plane cost +10 us of gate + router at T = 16384 (r2 bench).
      // DSMOE_B200_GATE_SPLIT=S selects a split (small-batch latency).
      const int nt = (T + kTileM - 1) / kTileM;
      const int nkb = L->d / kTileK;
      static const int split_env = [] {
        const char* v = std::getenv("DSMOE_B200_GATE_SPLIT");
        return v ? std::max(1, std::atoi(v)) : 1;
      }();
      int S = (L->E <= 64 && L->K <= 16) ? std::min(split_env, std::max(1, nkb / 2)) : 1;
      if (S < 2) S = 1;
      const long long Tp = static_cast<long long>(nt) * kTileM;
      if (C->gate_tiles_T != T || C->gate_tiles_Epad != L->Epad || C->gate_tiles_d != L->d ||
          C->gate_tiles_S != S) {
        std::vector<GemmTile> tl;
        for (int sp = 0; sp < S; ++sp) {
          const int kb0 = sp * nkb / S, kb1 = (sp + 1) * nkb / S;
          for (int m = 0; m < nt; ++m)
            tl.push_back(GemmTile{m * kTileM, 0, static_cast<int>(sp * Tp) + m * kTileM, 0, kb1 - kb0, L->Epad,
                                  std::min(kTileM, T - m * kTileM), kb0});
        }
        const int ntiles = static_cast<int>(tl.size());
        C->tiles_gate.ensure(sizeof(GemmTile) * (ntiles + 1) + 16);
        cuda_check(cudaMemcpyAsync(C->tiles_gate.p, tl.data(), sizeof(GemmTile) * ntiles, cudaMemcpyHostToDevice, s),
                   "H2D");
        int* ng = C->scalars.as<int>() + 3;
        cuda_check(cudaMemcpyAsync(ng, &ntiles, sizeof(int), cudaMemcpyHostToDevice, s), "H2D");
        cuda_check(cudaStreamSynchronize(s), "sync");
        C->gate_tiles_T = T;
        C->gate_tiles_Epad = L->Epad;
        C->gate_tiles_d = L->d;
        C->gate_tiles_S = S;
      }
      C->logits.ensure(static_cast<size_t>(S * Tp) * L->Epad * 4 + 16);
      if (S > 1) {
        nsplit = S;
        split_stride = Tp * L->Epad;
      }
      const CUtensorMap mx = make_map(x, T, L->d, L->d, kTileM);
      launch_check(launch_gemm_tc(0, &mx, &mx, &L->map_gate, C->tiles_gate.as<GemmTile>(),
                                  C->scalars.as<int>() + 3, S * nt, C->logits.p, L->Epad,
                                  nullptr, L->Epad, num_sms(), s, nullptr, nullptr, 0, nullptr, 0,
                                  C->counters.as<unsigned long long>()),
                   "gate gemm");
      counters_zeroed = true;
      ld = L->Epad;
    } else {
      launch_check(launch_gate_logits_exact(x, L->dtype == DSMOE_B200_BF16, L->gate_exact.as<float>(),
                                            C->logits.as<float>(), T, L->d, L->E, s),
                   "gate logits");
    }
    if (!fused) count_launch(1);
    lg = C->logits.as<float>();
    C->logits_layer = L;
    C->logits_T = T;
    C->logits_ld = ld;
  }
  if (!counters_zeroed && !fused)  // the fused kernel publishes counters[0..3] itself
    cuda_check(cudaMemsetAsync(C->counters.p, 0, 4 * sizeof(unsigned long long), s), "memset");
  if (!fused) C->mark(1);  // fused: the one kernel is timed as stage 0 (gate)
  RouterArgs a{};
  a.logits = lg;
  a.ld_logits = ld;
  a.T = T;
  a.E = L->E;
  a.K = L->K;
  a.P = L->P;
  a.kind = pol.kind;
  a.t_major = pol.t_major;
  a.t_minor = pol.t_minor;
  a.keep_top1 = pol.keep_top1;
  a.normalize = pol.normalize;
  a.t_unit = pol.t_unit;
  a.maj_off = pol.maj_off;
  a.min_off = pol.min_off;
  if (out) {
    a.idx = out->indices;
    a.raw = out->raw;
    a.norm = out->normalized;
    a.frac = out->fraction;
  }
  if (!a.frac && frac_ws) a.frac = frac_ws;
  a.sel_code = C->sel_code.as<int32_t>();
  a.sel_raw = C->sel_raw.as<float>();
  a.cnt_chunk = C->cnt_chunk.as<int>();
  a.counters = C->counters.as<unsigned long long>();
  a.nsplit = nsplit;
  a.split_stride = split_stride;
  a.logits_sum = nsplit > 1 ? C->logits.as<float>() : nullptr;
  if (fused) {
    const CUtensorMap mx = make_map(x, T, L->d, L->d, gate_route_tile_rows());
    static const bool sc_env = [] {  // DSMOE_B200_PERMUTE_SC=0: the permutation scans every chunk itself
      const char* v = std::getenv("DSMOE_B200_PERMUTE_SC");
      return !(v && std::atoi(v) == 0);
    }();
    launch_check(launch_gate_route(&mx, &L->map_gate, a, L->Epad, L->d / kTileK, C->logits.as<float>(),
                                   C->counters.as<unsigned long long>() + 8, num_sms(), s,
                                   sc_env ? C->sc_hist.as<int>() : nullptr),
                 "gate + router");
    C->sc_T = sc_env ? T : -1;
  } else {
    launch_check(launch_router(a, s), "router");
    C->sc_T = -1;
  }
  count_launch(1);
  // after the router: with a split-K gate the summed logits exist only now
  if (logits_out && logits_out != lg) {
    cuda_check(cudaMemcpy2DAsync(logits_out, L->E * 4, lg, ld * 4, L->E * 4, T, cudaMemcpyDeviceToDevice, s),
               "logits copy");
  }
}

// K2a: chunk scan + unit segments (+ GEMM work lists) + ordered scatter
void stage_permute(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, int T, bool plan, bool gather = false,
                   int tile_m = kTileM, int tile_m2 = kTileM, bool routed_only = false) {
  cudaStream_t s = C->stream;
  const long long Rcap = static_cast<long long>(T) * L->K;
  int* r_total = C->scalars.as<int>();
  PlanArgs pa{};
  pa.units = L->d_units.as<UnitInfo>();
  pa.seg_routed = C->seg.as<UnitSeg>();
  pa.seg_unit = nullptr;
  pa.shared_unit0 = L->E;
  pa.num_routed = L->E;
  pa.num_shared = routed_only ? 0 : L->S;
  pa.T = T;
  pa.d = L->d;
  pa.shared_row0 = static_cast<int>(Rcap);
  pa.tiles1 = C->tiles1.as<GemmTile>();
  pa.n1 = r_total + 1;
  pa.tiles2 = C->tiles2.as<GemmTile>();
  pa.n2 = r_total + 2;
  pa.gather = gather ? 1 : 0;
  pa.tile_m = tile_m;
  pa.tile_m2 = tile_m2;
  const int nchunks = (T + kRouterChunk - 1) / kRouterChunk;
  // one cooperative launch by default; DSMOE_B200_PERMUTE=split runs the
  // three-kernel path (scan_codes, seg_plan, scatter) — identical results
  static const bool split = [] {
    const char* v = std::getenv("DSMOE_B200_PERMUTE");
    return v && std::string(v) == "split";
  }();
  if (!split) {
    // after the fused gate + router: chunk offsets from its superchunk sums
    const bool sc = C->sc_T == T && L->E <= 64;
    launch_check(launch_permute_fused(C->cnt_chunk.as<int>(), nchunks, L->E, C->chunk_off.as<int>(),
                                      C->code_base.as<int>(), C->seg.as<UnitSeg>(), r_total,
                                      C->code_base.as<int>() + 2 * L->E, C->sel_code.as<int32_t>(),
                                      C->sel_raw.as<float>(), T, L->K, C->row_token.as<int32_t>(),
                                      C->row_scale.as<float>(), C->slot_pos.as<int32_t>(), plan ? &pa : nullptr,
                                      num_sms(), s, sc ? C->sc_hist.as<int>() : nullptr,
                                      sc ? C->counters.as<unsigned long long>() + 12 : nullptr),
                 "permute");
    count_launch(1);
    return;
  }
  launch_check(launch_scan_plan(C->cnt_chunk.as<int>(), nchunks, L->E, C->chunk_off.as<int>(), C->code_base.as<int>(),
                                C->seg.as<UnitSeg>(), r_total, C->code_base.as<int>() + 2 * L->E, plan ? &pa : nullptr, num_sms(), s),
               "scan/plan");
  launch_check(launch_scatter(C->sel_code.as<int32_t>(), C->sel_raw.as<float>(), T, L->K, L->E, C->chunk_off.as<int>(),
                              C->code_base.as<int>(), C->row_token.as<int32_t>(), C->row_scale.as<float>(),
                              C->slot_pos.as<int32_t>(), s),
               "scatter");
  count_launch(3);
}

// K3 + K4 over the work lists at n1/n2: A = `rows` (permuted tokens, a_rows
// allocated), alt A = x (shared experts), H in the context, Y = y (ld d).
void run_gemms(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* rows, long long a_rows, const void* x,
               int T, const int* n1, const int* n2, long long max1, long long max2, long long h_rows, void* y,
               const float* row_scale, const int* row_token = nullptr, int pair = 0, long long y_rows = -1) {
  if (y_rows < 0) y_rows = h_rows;
  cudaStream_t s = C->stream;
  const int mt1 = static_cast<int>(std::min<long long>(max1, 1 << 30));
  const int mt2 = static_cast<int>(std::min<long long>(max2, 1 << 30));
  if (L->dtype == DSMOE_B200_BF16) {
    // pair & 1 / pair & 2: GEMM1 / GEMM2 on CTA pairs (M = 256 tiles, B split
    // in two 128-row halves, one per CTA)
    const bool p1 = (pair & 1) != 0, p2 = (pair & 2) != 0;
    const CUtensorMap mx = make_map(x ? x : rows, x ? T : a_rows, L->d, L->d, kTileM);
    const CUtensorMap mxp = make_map(rows, a_rows, L->d, L->d, kTileM);
    const CUtensorMap mh = make_map(C->H.p, h_rows, L->hstride, L->hstride, kTileM);
    // TMA-store targets: 32-row boxes (one per epilogue warp)
    const CUtensorMap my = make_map(y, y_rows, L->d, L->d, 32, gemm_tc_store_box_cols());
    const CUtensorMap mh32 = make_map(C->H.p, h_rows, L->hstride, L->hstride, 32, gemm_tc_store_box_cols());
    // The CTA pairs walk their tiles in a fixed round-robin.  DSMOE_B200_SCHED=dyn
    // makes GEMM1 claim them dynamically (dyn2: both GEMMs): fewer SM cycles
    // under ncu's serialised replay, but 8 us slower per step in the
    // back-to-back loop (tools/gemm_span.sh, profiles/r4_ab_front.txt)
    static const bool dyn_env = [] {
      const char* v = std::getenv("DSMOE_B200_SCHED");
      return v && (std::string(v) == "dyn" || std::string(v) == "dyn2");
    }();
    static const bool dyn2_env = [] {  // GEMM2 claims too (DSMOE_B200_SCHED=dyn2)
      const char* v = std::getenv("DSMOE_B200_SCHED");
      return v && std::string(v) == "dyn2";
    }();
    int* gs = dyn_env ? C->gsched.as<int>() : nullptr;
    C->mark(4);
    launch_check(launch_gemm_tc(1, &mxp, &mx, p1 ? &L->map_w13_h : &L->map_w13, C->tiles1.as<GemmTile>(), n1, mt1,
                                C->H.p, L->hstride, nullptr, p1 ? 128 : 256, num_sms(), s, row_token,
                                row_token ? x : nullptr, static_cast<long long>(L->d) * 2, &mh32, p1 ? 1 : 0,
                                nullptr, gs),
                 "gemm1");
    C->mark(5);
    launch_check(launch_gemm_tc(2, &mh, &mh, p2 ? &L->map_w2t_h : &L->map_w2t, C->tiles2.as<GemmTile>(), n2, mt2, y,
                                L->d, row_scale, p2 ? 128 : 256, num_sms(), s, nullptr, nullptr, 0, &my, p2 ? 1 : 0,
                                nullptr, (gs && dyn2_env) ? gs + 2 : nullptr),
                 "gemm2");
  } else {
    SimtArgs g1{};
    g1.A = static_cast<const float*>(rows);
    g1.A2 = static_cast<const float*>(x ? x : rows);
    g1.lda = L->d;
    g1.a_rows = a_rows;
    g1.a2_rows = x ? T : a_rows;
    g1.B = L->w13.as<float>();
    g1.ldb = L->d;
    g1.tiles = C->tiles1.as<GemmTile>();
    g1.num_tiles = n1;
    g1.out = C->H.as<float>();
    g1.ldo = L->hstride;
    C->mark(4);
    launch_check(launch_gemm_simt(1, g1, mt1, num_sms(), s), "gemm1 simt");
    SimtArgs g2{};
    g2.A = C->H.as<float>();
    g2.A2 = C->H.as<float>();
    g2.lda = L->hstride;
    g2.a_rows = g2.a2_rows = h_rows;
    g2.B = L->w2t.as<float>();
    g2.ldb = L->hstride;
    g2.tiles = C->tiles2.as<GemmTile>();
    g2.num_tiles = n2;
    g2.out = static_cast<float*>(y);
    g2.ldo = L->d;
    g2.row_scale = row_scale;
    C->mark(5);
    launch_check(launch_gemm_simt(2, g2, mt2, num_sms(), s), "gemm2 simt");
  }
  count_launch(2);
}

// ------------------------------------- stage: K2 permute/gather, K3, K4, K5
// routed_only: the expert side of EP (received rows): no shared experts
void stage_ffn(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T, void* out,
               const void* resid = nullptr, bool routed_only = false) {
  cudaStream_t s = C->stream;
  const int es = esize(L->dtype);
  const long long Rcap = static_cast<long long>(T) * L->K;
  int* r_total = C->scalars.as<int>();
  int* n1 = r_total + 1;
  int* n2 = r_total + 2;
  // GEMM1's gather warps read the token rows of X straight into the swizzled
  // A tiles (gemm_tc.cu, warp-per-stage cp.async) by default;
  // DSMOE_B200_GATHER=explicit materialises X_perm with the 16-byte-vector
  // gather kernel first (bit-identical results).
  static const bool fused_env = [] {
    const char* v = std::getenv("DSMOE_B200_GATHER");
    return !(v && std::string(v) == "explicit");
  }();
  const bool fused_gather = fused_env && L->dtype == DSMOE_B200_BF16;
  const int pair = pair_mask(L);
  C->mark(2);
  stage_permute(C, L, T, true, fused_gather, (pair & 1) ? 256 : kTileM, (pair & 2) ? 256 : kTileM, routed_only);
  C->mark(3);
  if (!fused_gather) {
    launch_check(launch_gather(x, C->xperm.p, C->row_token.as<int32_t>(), r_total, L->d * es, num_sms(), s), "gather");
    count_launch(1);
  }
  const long long rows = Rcap + static_cast<long long>(L->S) * T + kRowSlack;
  run_gemms(C, L, fused_gather ? x : C->xperm.p, fused_gather ? T : Rcap + kRowSlack, x, T, n1, n2, C->max_tiles1(L, T),
            C->max_tiles2(L, T), rows, C->Y.p,
            C->row_scale.as<float>(), fused_gather ? C->row_token.as<int>() : nullptr, pair);
  C->mark(6);
  launch_check(launch_combine(C->Y.p, L->dtype == DSMOE_B200_BF16, C->slot_pos.as<int32_t>(), out, T, L->d, L->K,
                              routed_only ? 0 : L->S, static_cast<int>(Rcap), num_sms(), s, resid),
               "combine");
  count_launch(1);
}

void require_layer(const dsmoe_b200_layer* L) {
  require(L != nullptr, DSMOE_E_INVALID_ARGUMENT, "null layer");
  L->check_ready();
}
// entry points that evaluate arbitrary experts need every expert's weights
void require_whole(const dsmoe_b200_layer* L) {
  require_layer(L);
  require(!L->sharded(), DSMOE_E_INVALID_STATE,
          "layer is an expert shard (expert parallelism): it evaluates only its own experts");
}

}  // namespace

// ================================================================= C ABI
extern "C" {

const char* dsmoe_b200_version(void) { return "dsmoe_b200 0.1 (sm_100a)"; }
const char* dsmoe_b200_last_error(void) { return g_last_error.c_str(); }
int dsmoe_b200_last_launch_count(void) { return g_launches; }
long long dsmoe_b200_total_launch_count(void) { return g_launches_total.load(std::memory_order_relaxed); }

int dsmoe_b200_layer_create(const dsmoe_b200_layer_config* cfg, dsmoe_b200_layer** out) {
  return guarded([&] {
    require(cfg && out, DSMOE_E_INVALID_ARGUMENT, "null argument");
    auto* L = new dsmoe_b200_layer;
    try {
      layer_build(L, *cfg);
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
  });
}

void dsmoe_b200_layer_free(dsmoe_b200_layer* layer) { delete layer; }

int dsmoe_b200_layer_info(const dsmoe_b200_layer* L, int32_t* o) {
  return guarded([&] {
    require(L && o, DSMOE_E_INVALID_ARGUMENT, "null argument");
    const int32_t v[8] = {L->d, L->ffn, L->E, L->K, L->S, L->P, L->dtype, L->prenorm};
    std::memcpy(o, v, sizeof(v));
  });
}

int dsmoe_b200_layer_set_gate(dsmoe_b200_layer* L, const void* gate, int src_dtype, int src_on_device,
                              void* stream) {
  return guarded([&] {
    require(L && gate, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(src_dtype == 0 || src_dtype == 1, DSMOE_E_INVALID_ARGUMENT, "bad source dtype");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Staged g(gate, static_cast<size_t>(L->d) * L->E * esize(src_dtype), src_on_device, s);
    launch_check(launch_pack_gate(src_dtype, L->dtype, g.p, L->d, L->E, L->gateT.p, L->gate_exact.as<float>(), s),
                 "pack gate");
    cuda_check(cudaStreamSynchronize(s), "sync");
    L->gate_set = true;
  });
}

int dsmoe_b200_layer_set_block(dsmoe_b200_layer* L, int b, const void* w1, const void* w3, const void* w2,
                               int src_dtype, int src_on_device, void* stream) {
  return guarded([&] {
    require(L && w1 && w3 && w2, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(b >= 0 && b < L->E * L->P, DSMOE_E_INVALID_ARGUMENT, "block index out of range");
    require(L->held_block(b), DSMOE_E_INVALID_ARGUMENT, "block is not part of this expert shard");
    require(src_dtype == 0 || src_dtype == 1, DSMOE_E_INVALID_ARGUMENT, "bad source dtype");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int wd = L->widths[b];
    const size_t nb = static_cast<size_t>(L->d) * wd * esize(src_dtype);
    Staged a1(w1, nb, src_on_device, s), a3(w3, nb, src_on_device, s), a2(w2, nb, src_on_device, s);
    const int e = b / L->P, p = b % L->P;
    if (L->P == 1) {
      const UnitInfo& u = L->units[e];
      pack_sub(L, e, 0, a1.p, a3.p, a2.p, wd, nullptr, 0, src_dtype, s);
      if (u.nsub > 1) pack_sub(L, e, 1, a1.p, a3.p, a2.p, wd, nullptr, u.sub_w[0], src_dtype, s);
    } else {
      pack_sub(L, e, L->local_sub(b), a1.p, a3.p, a2.p, wd, nullptr, 0, src_dtype, s);
    }
    cuda_check(cudaStreamSynchronize(s), "sync");
    L->block_set[b] = 1;
  });
}

int dsmoe_b200_layer_set_shared(dsmoe_b200_layer* L, int si, const void* w1, const void* w3, const void* w2,
                                int src_dtype, int src_on_device, void* stream) {
  return guarded([&] {
    require(L && w1 && w3 && w2, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(si >= 0 && si < L->S, DSMOE_E_INVALID_ARGUMENT, "shared expert index out of range");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int wd = L->swidths[si];
    const size_t nb = static_cast<size_t>(L->d) * wd * esize(src_dtype);
    Staged a1(w1, nb, src_on_device, s), a3(w3, nb, src_on_device, s), a2(w2, nb, src_on_device, s);
    pack_sub(L, L->E + si, 0, a1.p, a3.p, a2.p, wd, nullptr, 0, src_dtype, s);
    cuda_check(cudaStreamSynchronize(s), "sync");
    L->shared_set[si] = 1;
  });
}

int dsmoe_b200_ctx_create(void* stream, dsmoe_b200_ctx** out) {
  return guarded([&] {
    require(out != nullptr, DSMOE_E_INVALID_ARGUMENT, "null argument");
    auto* C = new dsmoe_b200_ctx;
    C->stream = static_cast<cudaStream_t>(stream);
    *out = C;
  });
}

void dsmoe_b200_ctx_free(dsmoe_b200_ctx* C) {
  if (C) cudaStreamSynchronize(C->stream);
  delete C;
}

int dsmoe_b200_ctx_check(dsmoe_b200_ctx* C) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    if (!C->counters.p) return;
    check_flags(C);
  });
}

int dsmoe_b200_ctx_set_profiling(dsmoe_b200_ctx* C, int on) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require(on >= 0, DSMOE_E_INVALID_ARGUMENT, "profiling period must be >= 0");
    C->resolve();
    C->profiling = on != 0;
    C->prof_period = on > 1 ? on : 1;
    C->prof_seen = 0;
    for (double& v : C->prof_ms) v = 0.0;
    C->prof_calls = 0;
  });
}

int dsmoe_b200_ctx_profile(dsmoe_b200_ctx* C, double* ms, int n, long* calls) {
  return guarded([&] {
    require(C && ms, DSMOE_E_INVALID_ARGUMENT, "null argument");
    C->resolve();
    for (int i = 0; i < n && i < dsmoe_b200_ctx::kStages; ++i) ms[i] = C->prof_ms[i];
    if (calls) *calls = C->prof_calls;
  });
}

int dsmoe_b200_ctx_permutation(dsmoe_b200_ctx* C, int T, int K, int E, int32_t* row_token, int32_t* slot_pos,
                               int32_t* seg, int* r_total) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require(C->row_token.p && C->slot_pos.bytes >= static_cast<size_t>(T) * K * 4 &&
                C->seg.bytes >= sizeof(UnitSeg) * E,
            DSMOE_E_INVALID_STATE, "no permutation recorded for this shape");
    int R = 0;
    cuda_check(cudaStreamSynchronize(C->stream), "sync");
    cuda_check(cudaMemcpy(&R, C->scalars.p, sizeof(int), cudaMemcpyDeviceToHost), "D2H");
    if (r_total) *r_total = R;
    if (row_token) cuda_check(cudaMemcpy(row_token, C->row_token.p, sizeof(int32_t) * R, cudaMemcpyDeviceToHost), "D2H");
    if (slot_pos)
      cuda_check(cudaMemcpy(slot_pos, C->slot_pos.p, sizeof(int32_t) * T * K, cudaMemcpyDeviceToHost), "D2H");
    if (seg) {
      std::vector<UnitSeg> h(static_cast<size_t>(E));
      cuda_check(cudaMemcpy(h.data(), C->seg.p, sizeof(UnitSeg) * E, cudaMemcpyDeviceToHost), "D2H");
      for (int e = 0; e < E; ++e) {
        seg[3 * e] = h[e].start;
        seg[3 * e + 1] = h[e].n_full;
        seg[3 * e + 2] = h[e].n_tot;
      }
    }
  });
}

int dsmoe_b200_route(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                     const dsmoe_b200_policy* policy, int logits_mode, const float* logits_in,
                     float* logits_out, const dsmoe_b200_routing* out, dsmoe_b200_drop_stats_t* stats) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(T >= 0, DSMOE_E_INVALID_ARGUMENT, "negative token count");
    require(x || logits_in || T == 0, DSMOE_E_INVALID_ARGUMENT, "null input");
    g_launches = 0;
    const PolicyResolved pol = resolve_policy(L, policy);
    if (T == 0) {
      if (stats) stats_from_counts(L, 0, 0, 0, nullptr, stats);
      return;
    }
    C->ensure(L, T);
    const bool need_frac = stats && !is_pow2(L->P) && !(out && out->fraction);
    if (need_frac) C->frac_ws.ensure(static_cast<size_t>(T) * L->K * L->P);
    stage_route(C, L, x, T, pol, logits_mode, logits_in, logits_out, out, need_frac ? C->frac_ws.as<uint8_t>() : nullptr);
    if (stats) {
      unsigned long long h[5];
      read_counters(C, h);
      std::vector<uint8_t> fh;
      if (!is_pow2(L->P)) {
        fh.resize(static_cast<size_t>(T) * L->K * L->P);
        const void* src = (out && out->fraction) ? static_cast<const void*>(out->fraction) : C->frac_ws.p;
        cuda_check(cudaMemcpy(fh.data(), src, fh.size(), cudaMemcpyDeviceToHost), "D2H");
      }
      stats_from_counts(L, T, h[0], h[1], fh.data(), stats);
    }
  });
}

int dsmoe_b200_moe_forward(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                           const int32_t* indices, const double* raw, const double* fraction, void* out) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_whole(L);
    require(T >= 0, DSMOE_E_INVALID_ARGUMENT, "negative token count");
    g_launches = 0;
    if (T == 0) return;
    require(x && indices && raw && fraction && out, DSMOE_E_INVALID_ARGUMENT, "null argument");
    C->ensure(L, T);
    cudaStream_t s = C->stream;
    cuda_check(cudaMemsetAsync(C->counters.p, 0, 4 * sizeof(unsigned long long), s), "memset");
    ImportArgs a{};
    a.idx = indices;
    a.raw = raw;
    a.frac = fraction;
    a.T = T;
    a.K = L->K;
    a.P = L->P;
    a.nphys = L->E * L->P;
    a.nunits = L->E;
    a.sel_code = C->sel_code.as<int32_t>();
    a.sel_raw = C->sel_raw.as<float>();
    a.cnt_chunk = C->cnt_chunk.as<int>();
    a.counters = C->counters.as<unsigned long long>();
    C->sc_T = -1;
    launch_check(launch_import_routing(a, s), "import routing");
    count_launch(1);
    unsigned long long h[5];
    cuda_check(cudaMemcpyAsync(h, C->counters.p, sizeof(h), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    if (!(h[2] & 4ull) || L->P == 1) {
      stage_ffn(C, L, x, T, out);
      check_flags(C);
      return;
    }
    // Not the canonical replayed layout (e.g. copies of one selection with
    // different raw scores, a kept copy 1 without copy 0, fraction 0.5 on a
    // split layer, duplicate blocks): evaluate every slot on its own physical
    // block through the layer's block view — moe_forward's per-slot semantics
    // (moe.hpp:253-266): block indices[f], its first ceil(w/2) neurons when
    // fraction 0.5, weighted by raw.
    const dsmoe_b200_layer* B = nullptr;
    {
      std::lock_guard<std::mutex> lock(L->bview_mu);
      if (!L->bview) L->bview = transform_layer(L, kModeBlocks, 0, s);
      B = L->bview;
    }
    C->ensure(B, T);
    cuda_check(cudaMemsetAsync(C->counters.p, 0, 5 * sizeof(unsigned long long), s), "memset");
    ImportArgs b = a;
    b.K = B->K;
    b.P = 1;
    b.nphys = B->E;
    b.nunits = B->E;
    b.sel_code = C->sel_code.as<int32_t>();
    b.sel_raw = C->sel_raw.as<float>();
    b.cnt_chunk = C->cnt_chunk.as<int>();
    C->sc_T = -1;
    launch_check(launch_import_routing(b, s), "import routing (block view)");
    count_launch(1);
    stage_ffn(C, B, x, T, out);
    check_flags(C);
  });
}

int dsmoe_b200_forward(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                       const dsmoe_b200_policy* policy, int logits_mode, void* out,
                       dsmoe_b200_drop_stats_t* stats) {
  return dsmoe_b200_forward_ex(C, L, x, T, policy, logits_mode, 0, out, stats);
}

int dsmoe_b200_forward_ex(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                          const dsmoe_b200_policy* policy, int logits_mode, int flags, void* out,
                          dsmoe_b200_drop_stats_t* stats) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_whole(L);
    require(T >= 0, DSMOE_E_INVALID_ARGUMENT, "negative token count");
    g_launches = 0;
    const PolicyResolved pol = resolve_policy(L, policy);
    if (T == 0) {
      if (stats) stats_from_counts(L, 0, 0, 0, nullptr, stats);
      return;
    }
    require(x && out, DSMOE_E_INVALID_ARGUMENT, "null argument");
    C->ensure(L, T);
    const bool need_frac = stats && !is_pow2(L->P);
    if (need_frac) C->frac_ws.ensure(static_cast<size_t>(T) * L->K * L->P);
    C->prof_begin();
    stage_route(C, L, x, T, pol, logits_mode, nullptr, nullptr, nullptr, need_frac ? C->frac_ws.as<uint8_t>() : nullptr);
    stage_ffn(C, L, x, T, out, (flags & DSMOE_B200_RESIDUAL) ? x : nullptr);
    C->prof_end();
    if (stats) {
      unsigned long long h[5];
      read_counters(C, h);
      std::vector<uint8_t> fh;
      if (need_frac) {
        fh.resize(static_cast<size_t>(T) * L->K * L->P);
        cuda_check(cudaMemcpy(fh.data(), C->frac_ws.p, fh.size(), cudaMemcpyDeviceToHost), "D2H");
      }
      stats_from_counts(L, T, h[0], h[1], fh.data(), stats);
    }
  });
}

int dsmoe_b200_dispatch(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                        const dsmoe_b200_policy* policy, int logits_mode, void* rows_out, float* scale_out,
                        int32_t* seg_out, int* r_total_out, dsmoe_b200_drop_stats_t* stats) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(T >= 1 && x, DSMOE_E_INVALID_ARGUMENT, "dispatch: empty batch");
    g_launches = 0;
    const PolicyResolved pol = resolve_policy(L, policy);
    C->ensure(L, T);
    cudaStream_t s = C->stream;
    const bool need_frac = stats && !is_pow2(L->P);
    if (need_frac) C->frac_ws.ensure(static_cast<size_t>(T) * L->K * L->P);
    stage_route(C, L, x, T, pol, logits_mode, nullptr, nullptr, nullptr, need_frac ? C->frac_ws.as<uint8_t>() : nullptr);
    stage_permute(C, L, T, false);
    int* r_total = C->scalars.as<int>();
    if (rows_out) {
      launch_check(launch_gather(x, rows_out, C->row_token.as<int32_t>(), r_total, L->d * esize(L->dtype), num_sms(), s),
                   "gather");
      count_launch(1);
    }
    if (scale_out)
      cuda_check(cudaMemcpyAsync(scale_out, C->row_scale.p, sizeof(float) * static_cast<size_t>(T) * L->K,
                                 cudaMemcpyDeviceToDevice, s),
                 "scale copy");
    // shared experts run locally on this rank's tokens (moe.hpp:267-268)
    if (L->S > 0) {
      const long long Rcap = static_cast<long long>(T) * L->K;
      PlanArgs pa{};
      pa.units = L->d_units.as<UnitInfo>();
      pa.seg_routed = C->seg.as<UnitSeg>();
      pa.shared_unit0 = L->E;
      pa.num_routed = 0;
      pa.num_shared = L->S;
      pa.T = T;
      pa.d = L->d;
      pa.shared_row0 = static_cast<int>(Rcap);
      pa.tiles1 = C->tiles1.as<GemmTile>();
      pa.n1 = r_total + 1;
      pa.tiles2 = C->tiles2.as<GemmTile>();
      pa.n2 = r_total + 2;
      launch_check(launch_plan(pa, num_sms(), s), "plan shared");
      count_launch(1);
      const long long rows = Rcap + static_cast<long long>(L->S) * T + kTileM;
      run_gemms(C, L, x, T, x, T, r_total + 1, r_total + 2, C->max_tiles1(L, T), C->max_tiles2(L, T), rows, C->Y.p,
                C->row_scale.as<float>());
    }
    std::vector<UnitSeg> h(static_cast<size_t>(L->E));
    unsigned long long cnt[5];
    cuda_check(cudaMemcpyAsync(h.data(), C->seg.p, sizeof(UnitSeg) * L->E, cudaMemcpyDeviceToHost, s), "D2H");
    read_counters(C, cnt);
    int R = 0;
    for (int e = 0; e < L->E; ++e) {
      if (seg_out) {
        seg_out[3 * e] = h[e].start;
        seg_out[3 * e + 1] = h[e].n_full;
        seg_out[3 * e + 2] = h[e].n_tot;
      }
      R += h[e].n_tot;
    }
    if (r_total_out) *r_total_out = R;
    if (stats) {
      std::vector<uint8_t> fh;
      if (need_frac) {
        fh.resize(static_cast<size_t>(T) * L->K * L->P);
        cuda_check(cudaMemcpy(fh.data(), C->frac_ws.p, fh.size(), cudaMemcpyDeviceToHost), "D2H");
      }
      stats_from_counts(L, T, cnt[0], cnt[1], fh.data(), stats);
    }
  });
}

int dsmoe_b200_expert_ffn(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* rows, const float* row_scale,
                          long nrows, int nseg, const int32_t* seg_unit, const int32_t* seg_start,
                          const int32_t* seg_nfull, const int32_t* seg_ntot, void* y_out) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_whole(L);
    require(nseg >= 0 && nseg <= 2048, DSMOE_E_INVALID_ARGUMENT, "expert_ffn: at most 2048 segments");
    require(nseg == 0 || (seg_unit && seg_start && seg_nfull && seg_ntot), DSMOE_E_INVALID_ARGUMENT, "null segments");
    g_launches = 0;
    if (nseg == 0 || nrows == 0) return;
    require(rows && row_scale && y_out, DSMOE_E_INVALID_ARGUMENT, "null argument");
    cudaStream_t s = C->stream;
    std::vector<UnitSeg> sg(static_cast<size_t>(nseg));
    long long mt = 0;
    for (int i = 0; i < nseg; ++i) {
      require(seg_unit[i] >= 0 && seg_unit[i] < L->E, DSMOE_E_INVALID_ARGUMENT, "expert_ffn: unit out of range");
      require(seg_start[i] >= 0 && seg_nfull[i] >= 0 && seg_nfull[i] <= seg_ntot[i] &&
                  static_cast<long long>(seg_start[i]) + seg_ntot[i] <= nrows,
              DSMOE_E_INVALID_ARGUMENT, "expert_ffn: segment outside the row buffer");
      sg[i] = UnitSeg{seg_start[i], seg_nfull[i], seg_ntot[i], 0};
      mt += (seg_ntot[i] + kTileM - 1) / kTileM + 1;  // + the full / major-only split of GEMM2
    }
    C->vseg.ensure(sizeof(UnitSeg) * nseg);
    C->vseg_unit.ensure(sizeof(int) * nseg);
    C->scalars.ensure(4 * sizeof(int));
    cuda_check(cudaMemcpyAsync(C->vseg.p, sg.data(), sizeof(UnitSeg) * nseg, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(C->vseg_unit.p, seg_unit, sizeof(int) * nseg, cudaMemcpyHostToDevice, s), "H2D");
    const long long max1 = mt * L->max_chunks, max2 = mt * ((L->d + kTileN2 - 1) / kTileN2);
    C->tiles1.ensure(static_cast<size_t>(max1 + 1) * sizeof(GemmTile));
    C->tiles2.ensure(static_cast<size_t>(max2 + 1) * sizeof(GemmTile));
    const long long h_rows = nrows + kRowSlack;
    const int pair = pair_mask(L);
    C->H.ensure(static_cast<size_t>(h_rows) * L->hstride * esize(L->dtype));
    int* nn = C->scalars.as<int>();
    PlanArgs pa{};
    pa.units = L->d_units.as<UnitInfo>();
    pa.seg_routed = C->vseg.as<UnitSeg>();
    pa.seg_unit = C->vseg_unit.as<int>();
    pa.shared_unit0 = L->E;
    pa.num_routed = nseg;
    pa.num_shared = 0;
    pa.T = 0;
    pa.d = L->d;
    pa.tiles1 = C->tiles1.as<GemmTile>();
    pa.n1 = nn + 1;
    pa.tiles2 = C->tiles2.as<GemmTile>();
    pa.n2 = nn + 2;
    pa.tile_m = (pair & 1) ? 256 : kTileM;
    pa.tile_m2 = (pair & 2) ? 256 : kTileM;
    launch_check(launch_plan(pa, num_sms(), s), "plan");
    count_launch(1);
    run_gemms(C, L, rows, nrows, nullptr, 0, nn + 1, nn + 2, max1, max2, h_rows, y_out, row_scale, nullptr, pair, nrows);
    // no host sync: the segment tables were staged by cudaMemcpyAsync from
    // pageable memory (copied before the call returns); rows / y_out are the
    // caller's device buffers, ordered on the context stream
  });
}

int dsmoe_b200_combine(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* y_rows, int T, void* out) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(T >= 0 && (T == 0 || (y_rows && out)), DSMOE_E_INVALID_ARGUMENT, "null argument");
    g_launches = 0;
    if (T == 0) return;
    require(C->slot_pos.bytes >= static_cast<size_t>(T) * L->K * 4, DSMOE_E_INVALID_STATE,
            "combine: no dispatch recorded for this batch");
    const long long Rcap = static_cast<long long>(T) * L->K;
    // routed rows come from the caller (returned expert outputs); shared rows
    // from the dispatch's local shared-expert GEMMs (context Y)
    launch_check(launch_combine2(y_rows, C->Y.p, L->dtype == DSMOE_B200_BF16, C->slot_pos.as<int32_t>(), out, T, L->d,
                                 L->K, L->S, static_cast<int>(Rcap), num_sms(), C->stream),
                 "combine");
    count_launch(1);
  });
}

int dsmoe_b200_ep_pack(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T, int nranks,
                       const int32_t* owner, void* send_rows, int32_t* rec_code, int32_t* rec_row, float* rec_raw,
                       int64_t* counts) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(nranks >= 1 && nranks <= 32, DSMOE_E_INVALID_ARGUMENT, "ep_pack: 1 <= nranks <= 32");
    require(T >= 1 && x && owner && send_rows && rec_code && rec_row && rec_raw && counts, DSMOE_E_INVALID_ARGUMENT,
            "null argument");
    require(C->sel_code.bytes >= static_cast<size_t>(T) * L->K * 4 && C->logits_T == T, DSMOE_E_INVALID_STATE,
            "ep_pack: no routing recorded on this context for this batch (dispatch first)");
    for (int e = 0; e < L->E; ++e)
      require(owner[e] >= 0 && owner[e] < nranks, DSMOE_E_INVALID_ARGUMENT, "ep_pack: owner rank out of range");
    g_launches = 0;
    cudaStream_t s = C->stream;
    const int nchunks = (T + 255) / 256;
    C->ep_pos_td.ensure(static_cast<size_t>(T) * nranks * 4);
    C->ep_send_token.ensure(static_cast<size_t>(T) * std::min(nranks, L->K) * 4 + 16);
    C->ep_cnt.ensure(static_cast<size_t>(2) * nchunks * nranks * 4);
    C->ep_tot.ensure(static_cast<size_t>(4) * nranks * 4 + 16);
    // expert-aligned placement: a selection of expert e goes to owner[e] whatever its level
    std::vector<uint32_t> dest(static_cast<size_t>(2) * L->E);
    for (int e = 0; e < L->E; ++e) dest[2 * e] = dest[2 * e + 1] = 1u << owner[e];
    C->ep_owner.ensure(dest.size() * 4);
    cuda_check(cudaMemcpyAsync(C->ep_owner.p, dest.data(), dest.size() * 4, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaStreamSynchronize(s), "sync");
    int* cnt = C->ep_cnt.as<int>();
    int* r_total = C->ep_tot.as<int>() + 4 * nranks;
    launch_check(launch_ep_pack(C->sel_code.as<int32_t>(), C->sel_raw.as<float>(), C->ep_owner.as<uint32_t>(), T, L->K,
                                nranks, cnt, cnt + nchunks * nranks, C->ep_tot.as<int>(), C->ep_send_token.as<int32_t>(),
                                C->ep_pos_td.as<int32_t>(), rec_code, rec_row, rec_raw, r_total, num_sms(), s),
                 "ep_pack");
    count_launch(1);
    launch_check(launch_gather(x, send_rows, C->ep_send_token.as<int32_t>(), r_total, L->d * esize(L->dtype),
                               num_sms(), s),
                 "ep gather");
    count_launch(2);
    std::vector<int> tot(static_cast<size_t>(2 * nranks));
    cuda_check(cudaMemcpyAsync(tot.data(), C->ep_tot.p, tot.size() * 4, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    for (int i = 0; i < 2 * nranks; ++i) counts[i] = tot[i];
    C->ep_N = nranks;
    C->ep_T = T;
  });
}

}  // extern "C"

namespace {
void ep_expert_impl(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* rows, long U, const int32_t* rec_code,
                    const int32_t* rec_row, const float* rec_raw, int rec_stride, long S, const int64_t* src_row_base,
                    const int64_t* src_rec_base, int nranks, void* out);
}  // namespace

extern "C" {

int dsmoe_b200_ep_expert(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* rows, long U,
                         const int32_t* rec_code, const int32_t* rec_row, const float* rec_raw, long S,
                         const int64_t* src_row_base, const int64_t* src_rec_base, int nranks, void* out) {
  return guarded([&] {
    ep_expert_impl(C, L, rows, U, rec_code, rec_row, rec_raw, 1, S, src_row_base, src_rec_base, nranks, out);
  });
}

int dsmoe_b200_ep_expert_packed(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* rows, long U,
                                const int32_t* records, long S, const int64_t* src_row_base,
                                const int64_t* src_rec_base, int nranks, void* out) {
  return guarded([&] {
    require(S == 0 || records != nullptr, DSMOE_E_INVALID_ARGUMENT, "null records");
    ep_expert_impl(C, L, rows, U, records, records ? records + 1 : nullptr,
                   records ? reinterpret_cast<const float*>(records + 2) : nullptr, 3, S, src_row_base, src_rec_base,
                   nranks, out);
  });
}

}  // extern "C"

namespace {
void ep_expert_impl(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* rows, long U, const int32_t* rec_code,
                    const int32_t* rec_row, const float* rec_raw, int rec_stride, long S, const int64_t* src_row_base,
                    const int64_t* src_rec_base, int nranks, void* out) {
  {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(nranks >= 1 && nranks <= 32 && src_row_base && src_rec_base, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(U >= 0 && S >= 0 && U <= (1L << 30), DSMOE_E_INVALID_ARGUMENT, "ep_expert: bad sizes");
    require(src_row_base[nranks] == U && src_rec_base[nranks] == S, DSMOE_E_INVALID_ARGUMENT,
            "ep_expert: source bases do not cover the received rows / records");
    g_launches = 0;
    if (U == 0) return;
    require(rows && rec_code && rec_row && rec_raw && out, DSMOE_E_INVALID_ARGUMENT, "null argument");
    const int Ti = static_cast<int>(U);
    C->ensure(L, Ti);
    cudaStream_t s = C->stream;
    C->ep_base.ensure(static_cast<size_t>(2) * (nranks + 1) * 8);
    cuda_check(cudaMemcpyAsync(C->ep_base.p, src_rec_base, static_cast<size_t>(nranks + 1) * 8,
                               cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemcpyAsync(C->ep_base.as<char>() + (nranks + 1) * 8, src_row_base,
                               static_cast<size_t>(nranks + 1) * 8, cudaMemcpyHostToDevice, s), "H2D");
    const int nchunks = (Ti + kRouterChunk - 1) / kRouterChunk;
    cuda_check(cudaMemsetAsync(C->sel_code.p, 0xFF, static_cast<size_t>(Ti) * L->K * 4, s), "memset");
    C->sc_T = -1;
    cuda_check(cudaMemsetAsync(C->cnt_chunk.p, 0, static_cast<size_t>(nchunks) * 2 * L->E * 4, s), "memset");
    const long long* b = C->ep_base.as<long long>();
    launch_check(launch_ep_local_routing(rec_code, rec_row, rec_raw, S, rec_stride, b, b + nranks + 1, nranks, L->K,
                                         L->E, L->sharded() ? L->d_hold.as<unsigned char>() : nullptr,
                                         C->sel_code.as<int32_t>(),
                                         C->sel_raw.as<float>(), C->cnt_chunk.as<int>(),
                                         C->counters.as<unsigned long long>(), num_sms(), s),
                 "ep local routing");
    count_launch(1);
    count_launch(1);
    C->logits_T = -1;  // the routing codes on this context are no longer a gate routing
    stage_ffn(C, L, rows, Ti, out, nullptr, /*routed_only=*/true);
  }
}
}  // namespace

extern "C" {

int dsmoe_b200_ep_combine(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* ret_rows, int T, void* out) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(T >= 1 && ret_rows && out, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(C->ep_T == T && C->ep_N >= 1, DSMOE_E_INVALID_STATE, "ep_combine: no ep_pack recorded for this batch");
    g_launches = 0;
    const long long Rcap = static_cast<long long>(T) * L->K;
    launch_check(launch_ep_final_combine(ret_rows, L->dtype == DSMOE_B200_BF16, C->ep_pos_td.as<int32_t>(), C->ep_N,
                                         C->Y.p, L->S, static_cast<int>(Rcap), out, T, L->d, num_sms(), C->stream),
                 "ep combine");
    count_launch(1);
  });
}

int dsmoe_b200_ep_route_counts(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                               const dsmoe_b200_policy* policy, int logits_mode, int64_t* counts) {
  return guarded([&] {
    require(C != nullptr && counts != nullptr, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require_layer(L);
    require(T >= 1 && x, DSMOE_E_INVALID_ARGUMENT, "ep_route_counts: empty batch");
    g_launches = 0;
    PolicyResolved pol = resolve_policy(L, nullptr);
    if (policy && policy->normalize >= 0) pol.normalize = policy->normalize != 0;  // ensure_normalized only
    C->ensure(L, T);
    stage_route(C, L, x, T, pol, logits_mode, nullptr, nullptr, nullptr, nullptr);
    launch_check(launch_ep_counts(C->cnt_chunk.as<int>(), (T + kRouterChunk - 1) / kRouterChunk, L->E,
                                  reinterpret_cast<long long*>(counts), C->stream),
                 "ep counts");
    count_launch(1);
  });
}

int dsmoe_b200_ep_last_counts(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, int T, int64_t* counts) {
  return guarded([&] {
    require(C != nullptr && L != nullptr && counts != nullptr, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(C->routed_T == T && T >= 1, DSMOE_E_INVALID_STATE,
            "ep_last_counts: no routing of this batch on the context");
    launch_check(launch_ep_counts(C->cnt_chunk.as<int>(), (T + kRouterChunk - 1) / kRouterChunk, L->E,
                                  reinterpret_cast<long long*>(counts), C->stream),
                 "ep counts");
    count_launch(1);
  });
}

int dsmoe_b200_ep_thresholds(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const int64_t* counts, int devices,
                             const int32_t* device_of, double t_max, int load_aware, double* t_unit, double* loads) {
  return guarded([&] {
    require(C && L && counts && device_of && t_unit, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(devices >= 1 && devices <= 2048, DSMOE_E_INVALID_ARGUMENT, "ep_thresholds: bad device count");
    require(t_max > 0.0 && t_max <= 1.0, DSMOE_E_INVALID_ARGUMENT, "load_aware_thresholds: t_max must be in (0, 1]");
    g_launches = 0;
    launch_check(launch_ep_thresholds(reinterpret_cast<const long long*>(counts), L->E, L->P, devices, device_of, t_max,
                                      load_aware, t_unit, loads, C->stream),
                 "ep thresholds");
    count_launch(1);
  });
}

}  // extern "C"

namespace {
// The rate-targeted threshold on the device: a no-drop routing writes the
// normalized scores, the bisection kernel (router.cu) picks t exactly as the
// host bisection over drop_stats would and fills the per-expert threshold
// table.  Returns the device pointer of [t, rate].
double* stage_rate(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T, const PolicyResolved& pol,
                   double target, double tol, int iters, int logits_mode) {
  require(pol.kind == DSMOE_B200_DROP_1T || pol.kind == DSMOE_B200_DROP_2T, DSMOE_E_INVALID_ARGUMENT,
          "rate-targeted drop: the policy kind must be 1t or 2t");
  require(target >= 0.0 && target <= 1.0 && tol >= 0.0 && iters >= 1 && iters <= 64, DSMOE_E_INVALID_ARGUMENT,
          "rate-targeted drop: target in [0, 1], tol >= 0, 1 <= iters <= 64");
  require(is_pow2(L->P), DSMOE_E_INVALID_STATE, "rate-targeted drop: replay factor must be a power of two");
  cudaStream_t s = C->stream;
  const size_t n = static_cast<size_t>(T) * L->K * L->P;
  C->rate_norm.ensure(n * 8 + 16);
  C->rate_cnt.ensure(static_cast<size_t>(64) * 2 * 8);
  C->rate_tunit.ensure(static_cast<size_t>(L->E) * 8 + 16);
  C->rate_result.ensure(2 * 8);
  PolicyResolved none = pol;
  none.kind = DSMOE_B200_DROP_NONE;
  none.t_unit = nullptr;
  dsmoe_b200_routing r{nullptr, nullptr, C->rate_norm.as<double>(), nullptr};
  stage_route(C, L, x, T, none, logits_mode, nullptr, nullptr, &r, nullptr);
  cuda_check(cudaMemsetAsync(C->rate_cnt.p, 0, static_cast<size_t>(iters) * 2 * 8, s), "memset");
  launch_check(launch_rate_calibrate(C->rate_norm.as<double>(), T, L->K, L->P, L->S, pol.kind == DSMOE_B200_DROP_2T,
                                     pol.keep_top1, target, tol, iters, C->rate_cnt.as<unsigned long long>(),
                                     C->rate_tunit.as<double>(), L->E, C->rate_result.as<double>(), num_sms(), s),
               "rate calibration");
  count_launch(1);
  return C->rate_result.as<double>();
}

// the policy the router's second pass applies: one_t(t) / two_t_from(t) with t
// per expert from the device table (t_major = t + (-0.01) == t - 0.01 exactly)
PolicyResolved rate_policy(const PolicyResolved& pol, const double* t_unit) {
  PolicyResolved p = pol;
  p.t_drop = 0.0;
  p.t_unit = t_unit;
  p.maj_off = pol.kind == DSMOE_B200_DROP_2T ? -0.01 : 0.0;
  p.min_off = pol.kind == DSMOE_B200_DROP_2T ? 0.01 : 0.0;
  p.t_major = p.maj_off;
  p.t_minor = p.min_off;
  return p;
}
}  // namespace

extern "C" {

int dsmoe_b200_calibrate_rate(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                              const dsmoe_b200_policy* policy, double target, double tol, int iters, int logits_mode,
                              double* t_out, double* rate_out) {
  return guarded([&] {
    require(C != nullptr && policy != nullptr, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require_layer(L);
    require(T >= 1 && x, DSMOE_E_INVALID_ARGUMENT, "calibrate_rate: empty batch");
    g_launches = 0;
    dsmoe_b200_policy pc = *policy;
    if (pc.kind == DSMOE_B200_DROP_2T) pc.t_major = pc.t_minor = 0.0;  // the band comes from t
    const PolicyResolved pol = resolve_policy(L, &pc);
    C->ensure(L, T);
    const double* res = stage_rate(C, L, x, T, pol, target, tol, iters, logits_mode);
    double h[2];
    cuda_check(cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, C->stream), "D2H");
    unsigned long long cnt[5];
    read_counters(C, cnt);
    if (t_out) *t_out = h[0];
    if (rate_out) *rate_out = h[1];
  });
}

int dsmoe_b200_forward_rate(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                            const dsmoe_b200_policy* policy, double target, double tol, int iters, int logits_mode,
                            int flags, void* out, double* t_rate, dsmoe_b200_drop_stats_t* stats) {
  return guarded([&] {
    require(C != nullptr && policy != nullptr, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require_whole(L);
    require(T >= 1 && x && out, DSMOE_E_INVALID_ARGUMENT, "forward_rate: empty batch");
    g_launches = 0;
    dsmoe_b200_policy pc = *policy;
    if (pc.kind == DSMOE_B200_DROP_2T) pc.t_major = pc.t_minor = 0.0;
    const PolicyResolved pol = resolve_policy(L, &pc);
    C->ensure(L, T);
    C->prof_begin();
    const double* res = stage_rate(C, L, x, T, pol, target, tol, iters, logits_mode);
    stage_route(C, L, x, T, rate_policy(pol, C->rate_tunit.as<double>()), DSMOE_B200_LOGITS_REUSE, nullptr, nullptr,
                nullptr, nullptr);
    stage_ffn(C, L, x, T, out, (flags & DSMOE_B200_RESIDUAL) ? x : nullptr);
    C->prof_end();
    if (t_rate)
      cuda_check(cudaMemcpyAsync(t_rate, res, 2 * sizeof(double), cudaMemcpyDeviceToDevice, C->stream), "copy t");
    if (stats) {
      unsigned long long h[5];
      read_counters(C, h);
      stats_from_counts(L, T, h[0], h[1], nullptr, stats);
    }
  });
}

int dsmoe_b200_ctx_logits(dsmoe_b200_ctx* C, const float** logits, int* ld, int* T) {
  return guarded([&] {
    require(C && logits && ld && T, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(C->logits_T >= 0 && C->logits.p, DSMOE_E_INVALID_STATE, "ctx_logits: no gate logits on this context");
    *logits = C->logits.as<float>();
    *ld = C->logits_ld;
    *T = C->logits_T;
  });
}

int dsmoe_b200_ep_dispatch(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                           const dsmoe_b200_policy* policy, int logits_mode, const float* logits, int logits_ld,
                           int nranks, const uint32_t* dest, void* send_rows, int32_t* records, int64_t* counts) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(nranks >= 1 && nranks <= 32, DSMOE_E_INVALID_ARGUMENT, "ep_dispatch: 1 <= nranks <= 32");
    require(T >= 1 && x && dest && send_rows && records && counts, DSMOE_E_INVALID_ARGUMENT, "null argument");
    g_launches = 0;
    const PolicyResolved pol = resolve_policy(L, policy);
    C->ensure(L, T);
    cudaStream_t s = C->stream;
    stage_route(C, L, x, T, pol, logits_mode, logits, nullptr, nullptr, nullptr, logits_ld);
    const int nchunks = (T + 255) / 256;
    C->ep_pos_td.ensure(static_cast<size_t>(T) * nranks * 4);
    C->ep_send_token.ensure(static_cast<size_t>(T) * std::min(nranks, L->K) * 4 + 16);
    C->ep_cnt.ensure(static_cast<size_t>(2) * nchunks * nranks * 4);
    C->ep_tot.ensure(static_cast<size_t>(4) * nranks * 4 + 16);
    int* cnt = C->ep_cnt.as<int>();
    int* r_total = C->ep_tot.as<int>() + 4 * nranks;
    launch_check(launch_ep_pack(C->sel_code.as<int32_t>(), C->sel_raw.as<float>(), dest, T, L->K, nranks, cnt,
                                cnt + nchunks * nranks, C->ep_tot.as<int>(), C->ep_send_token.as<int32_t>(),
                                C->ep_pos_td.as<int32_t>(), records, records + 1, reinterpret_cast<float*>(records + 2),
                                r_total, num_sms(), s, 3, reinterpret_cast<long long*>(counts)),
                 "ep_pack");
    launch_check(launch_gather(x, send_rows, C->ep_send_token.as<int32_t>(), r_total, L->d * esize(L->dtype),
                               num_sms(), s),
                 "ep gather");
    count_launch(2);
    // the local shared experts (moe.hpp:267-268) into the context's Y rows
    if (L->S > 0) {
      const long long Rcap = static_cast<long long>(T) * L->K;
      int* sc = C->scalars.as<int>();
      PlanArgs pa{};
      pa.units = L->d_units.as<UnitInfo>();
      pa.seg_routed = C->seg.as<UnitSeg>();
      pa.shared_unit0 = L->E;
      pa.num_routed = 0;
      pa.num_shared = L->S;
      pa.T = T;
      pa.d = L->d;
      pa.shared_row0 = static_cast<int>(Rcap);
      pa.tiles1 = C->tiles1.as<GemmTile>();
      pa.n1 = sc + 1;
      pa.tiles2 = C->tiles2.as<GemmTile>();
      pa.n2 = sc + 2;
      launch_check(launch_plan(pa, num_sms(), s), "plan shared");
      count_launch(1);
      const long long rows = Rcap + static_cast<long long>(L->S) * T + kTileM;
      run_gemms(C, L, x, T, x, T, sc + 1, sc + 2, C->max_tiles1(L, T), C->max_tiles2(L, T), rows, C->Y.p,
                C->row_scale.as<float>());
    }
    C->ep_N = nranks;
    C->ep_T = T;
  });
}

int dsmoe_b200_layer_shard_blocks(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const uint8_t* held,
                                  dsmoe_b200_layer** out) {
  return guarded([&] {
    require(C && out && held, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require_whole(L);
    const int P = L->P;
    std::vector<char> h(static_cast<size_t>(L->E) * P);
    bool any = false;
    for (size_t b = 0; b < h.size(); ++b) any |= (h[b] = held[b] ? 1 : 0) != 0;
    require(any, DSMOE_E_INVALID_ARGUMENT, "layer_shard: the shard holds no expert block");
    std::vector<int32_t> widths(L->widths.begin(), L->widths.end()), swidths(L->swidths.begin(), L->swidths.end());
    dsmoe_b200_layer_config cfg{L->d, L->ffn, L->E, L->K, L->S, L->prenorm, P, L->dtype, widths.data(),
                                swidths.empty() ? nullptr : swidths.data()};
    auto* R = new dsmoe_b200_layer;
    try {
      layer_build(R, cfg, false, h.data());
      std::vector<int> src_unit(static_cast<size_t>(L->nunits())), gmap(static_cast<size_t>(L->E));
      for (int v = 0; v < L->nunits(); ++v) src_unit[static_cast<size_t>(v)] = v;
      for (int e = 0; e < L->E; ++e) gmap[static_cast<size_t>(e)] = e;
      std::vector<float> scale(static_cast<size_t>(L->nunits()), 1.0f);
      // dst neuron n of unit v (over its held blocks) -> src neuron (over all blocks)
      auto nmap = [L, R, P](int v, int n) {
        if (v >= L->E || P == 1) return n;
        int off = 0;
        for (int p = 0; p < P; ++p) {
          const int w = L->widths[static_cast<size_t>(v * P + p)];
          if (R->held_block(v * P + p)) {
            if (n < w) return off + n;
            n -= w;
          }
          off += w;
        }
        return off;  // unreachable for n inside the unit
      };
      regroup(L, R, src_unit, scale, nmap, gmap, C->stream);
    } catch (...) {
      delete R;
      throw;
    }
    *out = R;
  });
}

int dsmoe_b200_layer_shard(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, int unit_lo, int unit_hi,
                           dsmoe_b200_layer** out) {
  return guarded([&] {
    require(L != nullptr, DSMOE_E_INVALID_ARGUMENT, "null layer");
    require(unit_lo >= 0 && unit_lo < unit_hi && unit_hi <= L->E, DSMOE_E_INVALID_ARGUMENT,
            "layer_shard: need 0 <= lo < hi <= num_experts");
    std::vector<uint8_t> held(static_cast<size_t>(L->E) * L->P, 0);
    for (int b = unit_lo * L->P; b < unit_hi * L->P; ++b) held[static_cast<size_t>(b)] = 1;
    const int rc = dsmoe_b200_layer_shard_blocks(C, L, held.data(), out);
    if (rc != DSMOE_OK) fail(rc, g_last_error);
  });
}

int dsmoe_b200_analyze_gating(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T, int bins,
                              int logits_mode, long long* selection_counts, long long* raw_hist,
                              long long* norm_hist) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_layer(L);
    require(bins >= 2, DSMOE_E_INVALID_ARGUMENT, "analyze_gating: bins must be >= 2");
    require(T >= 1 && x, DSMOE_E_INVALID_ARGUMENT, "analyze_gating: empty token set");
    require(selection_counts && raw_hist && norm_hist, DSMOE_E_INVALID_ARGUMENT, "null argument");
    g_launches = 0;
    C->ensure(L, T);
    cudaStream_t s = C->stream;
    const size_t n = static_cast<size_t>(T) * L->K * L->P;
    DevBuf di, dr, dn, acc;
    di.ensure(n * 4);
    dr.ensure(n * 4);
    dn.ensure(n * 8);
    acc.ensure(sizeof(unsigned long long) * (L->E + 2 * bins));
    cuda_check(cudaMemsetAsync(acc.p, 0, acc.bytes, s), "memset");
    PolicyResolved pol;
    pol.normalize = 1;  // analyze_gating always applies normalize_topk (dropping.hpp:211)
    dsmoe_b200_routing out{di.as<int32_t>(), dr.as<float>(), dn.as<double>(), nullptr};
    stage_route(C, L, x, T, pol, logits_mode, nullptr, nullptr, &out, nullptr);
    auto* a = acc.as<unsigned long long>();
    launch_check(launch_gating_hist(di.as<int32_t>(), dr.as<float>(), dn.as<double>(), T, L->K, L->P, L->E, bins, a,
                                    a + L->E, a + L->E + bins, num_sms(), s),
                 "gating histogram");
    count_launch(1);
    std::vector<unsigned long long> h(static_cast<size_t>(L->E + 2 * bins));
    cuda_check(cudaMemcpyAsync(h.data(), acc.p, acc.bytes, cudaMemcpyDeviceToHost, s), "D2H");
    unsigned long long cnt[5];
    read_counters(C, cnt);  // normalize_topk on a zero-sum row throws (dropping.hpp:67)
    for (int e = 0; e < L->E; ++e) selection_counts[e] = static_cast<long long>(h[e]);
    for (int b = 0; b < bins; ++b) {
      raw_hist[b] = static_cast<long long>(h[L->E + b]);
      norm_hist[b] = static_cast<long long>(h[L->E + bins + b]);
    }
  });
}

int dsmoe_b200_drop_stats(const double* pre, const double* post, long n, int P, int S, long T, int d, int ffn,
                          dsmoe_b200_drop_stats_t* st) {
  return guarded([&] {
    require(pre && post && st && P >= 1, DSMOE_E_INVALID_ARGUMENT, "null argument");
    const double w = 1.0 / P;
    double total = 0.0, retained = 0.0;
    for (long i = 0; i < n; ++i) {
      total += pre[i] * w;
      retained += post[i] * w;
    }
    st->num_tokens = T;
    st->total_routed_units = total;
    st->dropped_units = total - retained;
    st->shared_units = static_cast<double>(S) * T;
    const double denom = st->total_routed_units + st->shared_units;
    st->drop_rate = denom > 0.0 ? st->dropped_units / denom : 0.0;
    const double unit = 6.0 * d * ffn;
    st->total_flops = denom * unit;
    st->saved_flops = st->dropped_units * unit;
    st->retained_flops = st->total_flops - st->saved_flops;
  });
}

int dsmoe_b200_transform(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, int mode, int p, dsmoe_b200_layer** out) {
  return guarded([&] {
    require(C != nullptr && out != nullptr, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require_layer(L);
    require(mode == kModeComplete || mode == kModePartial || mode == kModeReverse, DSMOE_E_INVALID_ARGUMENT,
            "transform: mode must be complete, partial or reverse");
    g_launches = 0;
    *out = transform_layer(L, mode, p, C->stream);
  });
}

int dsmoe_b200_layer_widths(const dsmoe_b200_layer* L, int32_t* block_widths, int32_t* shared_widths) {
  return guarded([&] {
    require(L != nullptr, DSMOE_E_INVALID_ARGUMENT, "null layer");
    if (block_widths) std::copy(L->widths.begin(), L->widths.end(), block_widths);
    if (shared_widths) std::copy(L->swidths.begin(), L->swidths.end(), shared_widths);
  });
}

namespace {
// host or device destination of a read-back
struct Sink {
  void* dst;
  int on_device;
  DevBuf tmp;
  void* dev(size_t bytes) {
    if (on_device) return dst;
    tmp.ensure(bytes);
    return tmp.p;
  }
  void finish(size_t bytes, cudaStream_t s) {
    if (!on_device) cuda_check(cudaMemcpyAsync(dst, tmp.p, bytes, cudaMemcpyDeviceToHost, s), "D2H");
  }
};

// unit u (sub-blocks [p0, p1)) -> reference-layout w1, w3 (d x w), w2 (w x d)
void read_unit(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, int u, int p0, int p1, void* w1, void* w3, void* w2,
               int on_device) {
  cudaStream_t s = C->stream;
  const UnitInfo& ui = L->units[u];
  const int es = esize(L->dtype), bf = L->dtype == DSMOE_B200_BF16;
  std::vector<long long> r1, r3;
  for (int p = p0; p < p1; ++p) {
    const long long b = sub_w13_base(ui, p);
    for (int i = 0; i < ui.sub_w[p]; ++i) {
      r1.push_back(w13_row_of(b, i, 0));
      r3.push_back(w13_row_of(b, i, 1));
    }
  }
  const int w = static_cast<int>(r1.size());
  const size_t nb = static_cast<size_t>(w) * L->d * es;
  Sink k1{w1, on_device}, k3{w3, on_device}, k2{w2, on_device};
  Staging<long long> s1, s3;
  launch_check(launch_transpose(bf, L->w13.p, L->d, s1.put(r1, s), 0, 0, w, L->d, k1.dev(nb), s), "read w1");
  launch_check(launch_transpose(bf, L->w13.p, L->d, s3.put(r3, s), 0, 0, w, L->d, k3.dev(nb), s), "read w3");
  char* o2 = static_cast<char*>(k2.dev(nb));
  for (int p = p0; p < p1; ++p) {  // W2T columns of each sub-block -> w2 rows
    launch_check(launch_transpose(bf, L->w2t.p, L->hstride, nullptr, ui.w2t_row, sub_hcol(ui, p), L->d, ui.sub_w[p],
                                  o2, s),
                 "read w2");
    o2 += static_cast<size_t>(ui.sub_w[p]) * L->d * es;
  }
  count_launch(2 + (p1 - p0));
  k1.finish(nb, s);
  k3.finish(nb, s);
  k2.finish(nb, s);
  cuda_check(cudaStreamSynchronize(s), "sync");
}
}  // namespace

int dsmoe_b200_layer_get_gate(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, void* gate, int dst_on_device) {
  return guarded([&] {
    require(C && L && gate, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(L->gate_set, DSMOE_E_INVALID_STATE, "layer: gate weights not set");
    const size_t nb = static_cast<size_t>(L->d) * L->E * esize(L->dtype);
    Sink k{gate, dst_on_device};
    launch_check(launch_transpose(L->dtype == DSMOE_B200_BF16, L->gateT.p, L->d, nullptr, 0, 0, L->E, L->d,
                                  k.dev(nb), C->stream),
                 "read gate");
    count_launch(1);
    k.finish(nb, C->stream);
    cuda_check(cudaStreamSynchronize(C->stream), "sync");
  });
}

int dsmoe_b200_layer_get_block(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, int b, void* w1, void* w3, void* w2,
                               int dst_on_device) {
  return guarded([&] {
    require(C && L && w1 && w3 && w2, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(b >= 0 && b < L->E * L->P, DSMOE_E_INVALID_ARGUMENT, "block index out of range");
    require(L->block_set[b], DSMOE_E_INVALID_STATE, "layer: expert block not set");
    const int e = b / L->P;
    if (L->P == 1)
      read_unit(C, L, e, 0, L->units[e].nsub, w1, w3, w2, dst_on_device);  // both virtual halves
    else
      read_unit(C, L, e, b % L->P, b % L->P + 1, w1, w3, w2, dst_on_device);
  });
}

int dsmoe_b200_layer_get_shared(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, int si, void* w1, void* w3, void* w2,
                                int dst_on_device) {
  return guarded([&] {
    require(C && L && w1 && w3 && w2, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(si >= 0 && si < L->S, DSMOE_E_INVALID_ARGUMENT, "shared expert index out of range");
    read_unit(C, L, L->E + si, 0, 1, w1, w3, w2, dst_on_device);
  });
}

int dsmoe_b200_load_aware_thresholds(const double* loads, int D, double t_max, double* out) {
  return guarded([&] {
    require(loads && out && D >= 1, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require(t_max > 0.0 && t_max <= 1.0, DSMOE_E_INVALID_ARGUMENT, "load_aware_thresholds: t_max must be in (0, 1]");
    double total = 0.0;
    for (int i = 0; i < D; ++i) total += loads[i];
    require(total > 0.0, DSMOE_E_INVALID_ARGUMENT, "load_aware_thresholds: zero total load");
    const double ideal = total / static_cast<double>(D);
    for (int i = 0; i < D; ++i) {
      const double ratio = loads[i] / ideal;
      out[i] = ratio >= 1.0 ? t_max : t_max * ratio;
    }
  });
}

static ImpUnitC imp_unit(const dsmoe_b200_layer* L, int e) {
  const UnitInfo& u = L->units[e];
  ImpUnitC c{};
  c.base0 = u.w13_row;
  c.base1 = u.w13_row + 2LL * u.sub_wpad[0];
  c.h0 = u.sub_w[0];
  c.wpad0 = u.sub_wpad[0];
  c.wpad1 = u.nsub > 1 ? u.sub_wpad[1] : 0;
  return c;
}

int dsmoe_b200_profile_importance(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const void* x, int T,
                                  const int32_t* indices, int metric, double* values) {
  return guarded([&] {
    require(C != nullptr, DSMOE_E_INVALID_ARGUMENT, "null ctx");
    require_whole(L);
    require(L->P == 1, DSMOE_E_INVALID_STATE,
            "profile_importance: profile the original layer, not a partitioned one");
    require(T >= 1, DSMOE_E_INVALID_ARGUMENT, "profile_importance: empty calibration set");
    require(metric >= 0 && metric <= 3, DSMOE_E_INVALID_ARGUMENT, "unknown importance metric");
    require(x && indices && values, DSMOE_E_INVALID_ARGUMENT, "null argument");
    g_launches = 0;
    C->ensure(L, T);
    cudaStream_t s = C->stream;
    const long long n = static_cast<long long>(T) * L->K;
    // every selection counts, regardless of fraction (reconstruct.hpp:121-125)
    std::vector<double> ones(static_cast<size_t>(n), 1.0);
    DevBuf dfrac;
    dfrac.ensure(sizeof(double) * n);
    cuda_check(cudaMemcpyAsync(dfrac.p, ones.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaMemsetAsync(C->counters.p, 0, 4 * sizeof(unsigned long long), s), "memset");
    ImportArgs a{};
    a.idx = indices;
    a.raw = dfrac.as<double>();
    a.frac = dfrac.as<double>();
    a.T = T;
    a.K = L->K;
    a.P = 1;
    a.nphys = L->E;
    a.nunits = L->E;
    a.sel_code = C->sel_code.as<int32_t>();
    a.sel_raw = C->sel_raw.as<float>();
    a.cnt_chunk = C->cnt_chunk.as<int>();
    a.counters = C->counters.as<unsigned long long>();
    C->sc_T = -1;
    launch_check(launch_import_routing(a, s), "import routing");
    stage_permute(C, L, T, false);
    unsigned long long flags[5];
    cuda_check(cudaMemcpyAsync(flags, C->counters.p, sizeof(flags), cudaMemcpyDeviceToHost, s), "D2H");
    std::vector<UnitSeg> seg(static_cast<size_t>(L->E));
    cuda_check(cudaMemcpyAsync(seg.data(), C->seg.p, sizeof(UnitSeg) * L->E, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "sync");
    if (flags[4] & 4ull) cuda_check(cudaMemsetAsync(C->counters.as<unsigned long long>() + 4, 0, 8, s), "memset");
    require(!(flags[2] & 4ull), DSMOE_E_INVALID_STATE, "profile_importance: expert index out of range");
    DevBuf v;
    v.ensure(sizeof(double) * static_cast<size_t>(n) * L->ffn + 8);
    for (int e = 0; e < L->E; ++e)
      launch_check(launch_importance_tiles(L->dtype == DSMOE_B200_BF16, x, C->row_token.as<int32_t>(), seg[e].start,
                                           seg[e].n_tot, L->w13.p, imp_unit(L, e), L->d, L->ffn, metric, v.as<double>(),
                                           s),
                   "importance");
      count_launch(1);
    launch_check(launch_importance_reduce(v.as<double>(), C->seg.as<UnitSeg>(), L->E, L->ffn, values, s), "reduce");
    count_launch(1);
    cuda_check(cudaStreamSynchronize(s), "sync");
  });
}

int dsmoe_b200_reconstruct(dsmoe_b200_ctx* C, const dsmoe_b200_layer* L, const double* values, int32_t* order_out,
                           dsmoe_b200_layer** out) {
  return guarded([&] {
    require(C != nullptr && out != nullptr && values != nullptr, DSMOE_E_INVALID_ARGUMENT, "null argument");
    require_whole(L);
    require(L->P == 1, DSMOE_E_INVALID_STATE, "reconstruct_experts: layer already partitioned");
    cudaStream_t s = C->stream;
    DevBuf ord;
    int32_t* order = order_out;
    if (!order) {
      ord.ensure(sizeof(int32_t) * static_cast<size_t>(L->E) * L->ffn);
      order = ord.as<int32_t>();
    }
    launch_check(launch_order_sort(values, L->E, L->ffn, order, s), "order sort");
    const int major = (L->ffn + 1) / 2;  // ReconstructionMap::major_size (reconstruct.hpp:157)
    std::vector<int32_t> widths;
    for (int e = 0; e < L->E; ++e) {
      widths.push_back(major);
      widths.push_back(L->ffn - major);
    }
    dsmoe_b200_layer_config cfg{L->d, L->ffn, L->E, L->K, L->S, L->prenorm, 2, L->dtype, widths.data(),
                                L->swidths.data()};
    auto* R = new dsmoe_b200_layer;
    try {
      layer_build(R, cfg);
      require(R->w13_rows == L->w13_rows && R->hstride == L->hstride, DSMOE_E_INTERNAL,
              "reconstruct: packed geometry mismatch");
      for (int e = 0; e < L->E; ++e)
        launch_check(launch_gather_unit(L->dtype == DSMOE_B200_BF16, L->w13.p, R->w13.p, L->w2t.p, R->w2t.p,
                                        order + static_cast<size_t>(e) * L->ffn, imp_unit(L, e), L->ffn, L->d,
                                        static_cast<long long>(e) * L->d, L->hstride, s),
                     "gather unit");
      const int es = esize(L->dtype);
      if (L->S > 0) {
        const size_t r0 = static_cast<size_t>(L->units[L->E].w13_row);
        cuda_check(cudaMemcpyAsync(R->w13.as<char>() + r0 * L->d * es, L->w13.as<char>() + r0 * L->d * es,
                                   L->w13.bytes - r0 * L->d * es, cudaMemcpyDeviceToDevice, s),
                   "copy shared");
        const size_t q0 = static_cast<size_t>(L->E) * L->d * L->hstride * es;
        cuda_check(cudaMemcpyAsync(R->w2t.as<char>() + q0, L->w2t.as<char>() + q0, L->w2t.bytes - q0,
                                   cudaMemcpyDeviceToDevice, s),
                   "copy shared");
      }
      cuda_check(cudaMemcpyAsync(R->gateT.p, L->gateT.p, L->gateT.bytes, cudaMemcpyDeviceToDevice, s), "copy gate");
      cuda_check(cudaMemcpyAsync(R->gate_exact.p, L->gate_exact.p, L->gate_exact.bytes, cudaMemcpyDeviceToDevice, s),
                 "copy gate");
      cuda_check(cudaStreamSynchronize(s), "sync");
      R->gate_set = true;
      std::fill(R->block_set.begin(), R->block_set.end(), 1);
      std::fill(R->shared_set.begin(), R->shared_set.end(), 1);
    } catch (...) {
      delete R;
      throw;
    }
    *out = R;
  });
}

}  // extern "C"
