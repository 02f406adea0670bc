// The reference's own C ABI (include/dsmoe_abi.h: the dsmoe_* entry points of
// /root/reference/proj/include/dsmoe.h) implemented over the B200 device
// path.  Same symbols, status codes, thread-local last error, JSON
// documents, token files passed by path, DSMOE1 containers, `new char[]`
// output strings freed by dsmoe_string_free (capi.cpp:29-68).  Every compute
// entry point — infer, reconstruct, transform, reverse_partial, sweep,
// analyze_gating, sim_ep, verify_equivalence — runs on the GPU through the
// device C ABI (dsmoe_b200.h): fp32 layers, serial-k exact gate logits, so
// routing, drop masks, drop rates and importance orders are the reference's
// bit for bit and outputs agree to fp32 rounding.  Host code here only
// parses, generates, loads and saves (the reference's io.cpp / capi.cpp
// host side) and formats reports.
//
// 64-bit models (scalar_width 8, the reference's verification precision)
// load, save, describe and generate, but the device compute entry points
// reject them with DSMOE_E_INVALID_ARGUMENT: the device computes in fp32.
// dsmoe_sim_comm / dsmoe_sim_comm_sweep (the alpha-beta communication model,
// comm_sim.cpp) are outside the device path and return DSMOE_E_INVALID_STATE.
#include "../../include/dsmoe_abi.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dsmoe_b200.h"
#include "kernels.h"
#include "minijson.h"

using minijson::Value;

namespace {

// ------------------------------------------------------------------ errors
struct AbiError : std::runtime_error {
  int code;
  AbiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& m) { throw AbiError(code, m); }
void require(bool ok, int code, const std::string& m) {
  if (!ok) fail(code, m);
}
void check_arg(bool ok, const char* m) { require(ok, DSMOE_E_INVALID_ARGUMENT, m); }
// a device C ABI call: its status and message become ours
void dev(int rc) {
  if (rc != DSMOE_OK) fail(rc, dsmoe_b200_last_error());
}
void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(DSMOE_E_INTERNAL, std::string(what) + ": " + cudaGetErrorString(e));
}

thread_local std::string t_last_error;

template <class F>
int guarded(F&& f) noexcept {
  try {
    f();
    t_last_error.clear();
    return DSMOE_OK;
  } catch (const AbiError& e) {
    t_last_error = e.what();
    return e.code;
  } catch (const minijson::Error& e) {  // caller documents (capi.cpp:47-51)
    t_last_error = e.what();
    return DSMOE_E_INVALID_ARGUMENT;
  } catch (const std::bad_alloc&) {
    t_last_error = "out of memory";
    return DSMOE_E_INTERNAL;
  } catch (const std::exception& e) {
    t_last_error = e.what();
    return DSMOE_E_INTERNAL;
  } catch (...) {
    t_last_error = "unknown error";
    return DSMOE_E_INTERNAL;
  }
}

void set_out(char** slot, const std::string& s) {
  if (!slot) return;
  char* p = new char[s.size() + 1];
  std::memcpy(p, s.c_str(), s.size() + 1);
  *slot = p;
}

Value parse_doc(const char* text, const char* what) {
  check_arg(text != nullptr, "missing JSON argument");
  try {
    return minijson::parse(text);
  } catch (const minijson::Error& e) {
    fail(DSMOE_E_INVALID_ARGUMENT, std::string(what) + ": invalid JSON: " + e.what());
  }
}

// ------------------------------------------------------------ host model
struct Config {  // MoeConfig (moe.hpp:17-36)
  int d_model = 0, d_ffn = 0, num_experts = 0, top_k = 0, num_shared_experts = 0;
  bool gate_prenormalized = false;
  void validate() const {
    check_arg(d_model >= 1, "config: d_model must be >= 1");
    check_arg(d_ffn >= 2, "config: d_ffn must be >= 2");
    check_arg(num_experts >= 1, "config: num_experts must be >= 1");
    check_arg(top_k >= 1 && top_k <= num_experts, "config: top_k must satisfy 1 <= K <= E");
    check_arg(num_shared_experts >= 0, "config: num_shared_experts must be >= 0");
  }
  Value json() const {
    Value v = Value::object();
    v["d_model"] = d_model;
    v["d_ffn"] = d_ffn;
    v["num_experts"] = num_experts;
    v["top_k"] = top_k;
    v["num_shared_experts"] = num_shared_experts;
    v["gate_prenormalized"] = gate_prenormalized;
    return v;
  }
};

const char* kLineage[] = {"base", "complete", "partial", "reconstructed"};
int lineage_of(const std::string& s) {
  for (int i = 0; i < 4; ++i)
    if (s == kLineage[i]) return i;
  fail(DSMOE_E_SCHEMA, "unknown lineage tag: " + s);
}

template <class T>
struct Mat {  // row-major rows x cols
  int rows = 0, cols = 0;
  std::vector<T> v;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), v(static_cast<size_t>(r) * c) {}
};

template <class T>
struct Block {  // Expert<T> (moe.hpp:39-45): w1, w3 d x width; w2 width x d
  Mat<T> w1, w3, w2;
  int width() const { return w1.cols; }
};

template <class T>
struct Layer {  // MoeLayer<T> (moe.hpp:73-120)
  Config cfg;
  Mat<T> gate;
  std::vector<Block<T>> experts, shared;
  int replay = 1;
  int lineage = 0;
  std::vector<std::vector<int>> order;  // neuron_order

  void validate() const {
    cfg.validate();
    require(replay >= 1, DSMOE_E_INVALID_STATE, "layer: replay_factor must be >= 1");
    require(gate.rows == cfg.d_model && gate.cols == cfg.num_experts, DSMOE_E_SHAPE_MISMATCH,
            "layer: gate shape " + std::to_string(gate.rows) + "x" + std::to_string(gate.cols) + " expected " +
                std::to_string(cfg.d_model) + "x" + std::to_string(cfg.num_experts));
    require(static_cast<int>(experts.size()) == cfg.num_experts * replay, DSMOE_E_INVALID_STATE,
            "layer: expected " + std::to_string(cfg.num_experts * replay) + " expert blocks, have " +
                std::to_string(experts.size()));
    for (int e = 0; e < cfg.num_experts; ++e) {
      int tot = 0;
      for (int p = 0; p < replay; ++p) {
        const Block<T>& b = experts[static_cast<size_t>(e) * replay + p];
        require(b.w1.rows == cfg.d_model && b.w3.rows == cfg.d_model && b.w1.cols == b.w3.cols &&
                    b.w2.rows == b.w1.cols && b.w2.cols == cfg.d_model,
                DSMOE_E_SHAPE_MISMATCH, "layer: inconsistent block shapes for expert " + std::to_string(e));
        tot += b.width();
      }
      require(tot == cfg.d_ffn, DSMOE_E_INVALID_STATE,
              "layer: block widths of expert " + std::to_string(e) + " sum to " + std::to_string(tot) +
                  ", expected " + std::to_string(cfg.d_ffn));
    }
    for (const Block<T>& s : shared)
      require(s.w1.rows == cfg.d_model && s.w1.cols == s.w3.cols && s.w3.rows == cfg.d_model &&
                  s.w2.rows == s.w1.cols && s.w2.cols == cfg.d_model,
              DSMOE_E_SHAPE_MISMATCH, "layer: inconsistent shared expert shapes");
    require(static_cast<int>(shared.size()) == cfg.num_shared_experts, DSMOE_E_INVALID_STATE,
            "layer: shared expert count mismatch");
    if (!order.empty())
      require(static_cast<int>(order.size()) == cfg.num_experts, DSMOE_E_INVALID_STATE,
              "layer: neuron_order must cover every original expert");
  }
};

template <class T>
void validate_model(const std::vector<Layer<T>>& layers) {
  require(!layers.empty(), DSMOE_E_INVALID_STATE, "model has no layers");
  for (const auto& l : layers) l.validate();
}

}  // namespace

struct dsmoe_model {
  int width = 4;
  std::vector<Layer<float>> f;
  std::vector<Layer<double>> d;
  // device copies of the fp32 layers, built on first use per CUDA device (the
  // model is immutable, so the cache never goes stale); dev_id = the device
  // the `dev` copies live on
  mutable std::mutex mu;
  mutable std::vector<dsmoe_b200_layer*> dev;
  mutable int dev_id = -1;
  mutable std::vector<std::pair<int, std::vector<dsmoe_b200_layer*>>> other;  // copies on other devices
  ~dsmoe_model() {
    for (auto* L : dev)
      if (L) dsmoe_b200_layer_free(L);
    for (auto& o : other)
      for (auto* L : o.second)
        if (L) dsmoe_b200_layer_free(L);
  }
  int num_layers() const { return width == 4 ? static_cast<int>(f.size()) : static_cast<int>(d.size()); }
};

namespace {

const dsmoe_model& model_ref(const dsmoe_model* m) {
  check_arg(m != nullptr, "model handle is null");
  return *m;
}

const std::vector<Layer<float>>& fp32_layers(const dsmoe_model& m) {
  require(m.width == 4, DSMOE_E_INVALID_ARGUMENT,
          "the B200 device path computes in fp32/bf16: scalar_width 8 models are not supported by this entry "
          "point (convert the model to scalar_width 4)");
  validate_model(m.f);
  return m.f;
}

// ------------------------------------------------ generators (rng.hpp, io.cpp)
struct SplitMix64 {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
};
struct Xoshiro {  // xoshiro256++ seeded through SplitMix64
  uint64_t st[4];
  explicit Xoshiro(uint64_t seed) {
    SplitMix64 sm{seed};
    for (auto& v : st) v = sm.next();
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(st[0] + st[3], 23) + st[0];
    const uint64_t t = st[1] << 17;
    st[2] ^= st[0];
    st[3] ^= st[1];
    st[1] ^= st[2];
    st[0] ^= st[3];
    st[2] ^= t;
    st[3] = rotl(st[3], 45);
    return r;
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double gaussian() {  // Irwin-Hall: 12 uniforms - 6
    double a = 0.0;
    for (int i = 0; i < 12; ++i) a += unit();
    return a - 6.0;
  }
};

template <class T>
Layer<T> generate_layer(const Config& c, uint64_t seed, double scale) {
  c.validate();
  Xoshiro rng(seed);
  const double sd = scale / std::sqrt(static_cast<double>(c.d_model));
  auto fill = [&](Mat<T>& m) {
    for (T& v : m.v) v = static_cast<T>(rng.gaussian() * sd);
  };
  Layer<T> L;
  L.cfg = c;
  L.gate = Mat<T>(c.d_model, c.num_experts);
  fill(L.gate);
  auto expert = [&] {
    Block<T> b;
    b.w1 = Mat<T>(c.d_model, c.d_ffn);
    b.w3 = Mat<T>(c.d_model, c.d_ffn);
    b.w2 = Mat<T>(c.d_ffn, c.d_model);
    fill(b.w1);
    fill(b.w3);
    fill(b.w2);
    return b;
  };
  for (int e = 0; e < c.num_experts; ++e) L.experts.push_back(expert());
  for (int s = 0; s < c.num_shared_experts; ++s) L.shared.push_back(expert());
  return L;
}

// ----------------------------------------------------------- file I/O
void write_atomic(const std::string& path, const std::string& content) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream f(tmp, std::ios::binary | std::ios::trunc);
    require(f.good(), DSMOE_E_IO, "cannot open for writing: " + tmp);
    f.write(content.data(), static_cast<std::streamsize>(content.size()));
    f.flush();
    require(f.good(), DSMOE_E_IO, "write failed: " + tmp);
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    fail(DSMOE_E_IO, "cannot move temporary file into place: " + path);
  }
}

std::string read_all(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  require(f.good(), DSMOE_E_IO, "cannot open for reading: " + path);
  std::string data((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  require(!f.bad(), DSMOE_E_IO, "read failed: " + path);
  return data;
}

void put_u64(std::string& out, uint64_t v) {
  for (int i = 0; i < 8; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xff));
}
uint64_t get_u64(const char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(static_cast<unsigned char>(p[i])) << (8 * i);
  return v;
}

// token file: u64 rows, u64 cols, fp32 row-major payload (io.cpp token format)
struct Tokens {
  int rows = 0, cols = 0;
  std::vector<float> v;
};
Tokens load_tokens(const char* path) {
  const std::string raw = read_all(path);
  require(raw.size() >= 16, DSMOE_E_TRUNCATED, "token file: missing header");
  const uint64_t rows = get_u64(raw.data()), cols = get_u64(raw.data() + 8);
  require(rows <= (1u << 24) && cols <= (1u << 20), DSMOE_E_SCHEMA, "token file: implausible dimensions");
  require(raw.size() >= 16 + rows * cols * 4, DSMOE_E_TRUNCATED, "token file: payload truncated");
  Tokens t;
  t.rows = static_cast<int>(rows);
  t.cols = static_cast<int>(cols);
  t.v.resize(rows * cols);
  std::memcpy(t.v.data(), raw.data() + 16, rows * cols * 4);
  return t;
}

// --------------------------------------------------- DSMOE1 container
constexpr char kMagic[8] = {'D', 'S', 'M', 'O', 'E', '1', '\0', '\0'};
constexpr size_t kAlign = 64;
size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <class T>
void save_container(const std::vector<Layer<T>>& layers, const std::string& path) {
  validate_model(layers);
  struct Ref {
    std::string name;
    int rows, cols;
    const void* data;
    size_t bytes;
  };
  std::vector<Ref> refs;
  auto add = [&](std::string n, const Mat<T>& m) {
    refs.push_back({std::move(n), m.rows, m.cols, m.v.data(), m.v.size() * sizeof(T)});
  };
  Value jl = Value::array();
  for (size_t l = 0; l < layers.size(); ++l) {
    const Layer<T>& L = layers[l];
    const std::string b = "layers/" + std::to_string(l) + "/";
    add(b + "gate", L.gate);
    for (size_t e = 0; e < L.experts.size(); ++e) {
      const std::string eb = b + "experts/" + std::to_string(e) + "/";
      add(eb + "w1", L.experts[e].w1);
      add(eb + "w3", L.experts[e].w3);
      add(eb + "w2", L.experts[e].w2);
    }
    for (size_t s = 0; s < L.shared.size(); ++s) {
      const std::string sb = b + "shared/" + std::to_string(s) + "/";
      add(sb + "w1", L.shared[s].w1);
      add(sb + "w3", L.shared[s].w3);
      add(sb + "w2", L.shared[s].w2);
    }
    Value one = Value::object();
    one["config"] = L.cfg.json();
    one["lineage"] = kLineage[L.lineage];
    one["replay_factor"] = L.replay;
    Value ord = Value::array();
    for (const auto& o : L.order) ord.push_back(Value(o));
    one["neuron_order"] = ord;
    jl.push_back(one);
  }
  Value manifest = Value::object();
  manifest["format"] = "dsmoe-container";
  manifest["version"] = 1;
  manifest["scalar_width"] = static_cast<int>(sizeof(T));
  manifest["num_layers"] = static_cast<int>(layers.size());
  manifest["layers"] = jl;
  // the tensor table holds absolute offsets, which depend on the manifest's
  // length: size it with zero offsets plus a fixed allowance per tensor, then
  // render the real offsets and pad with spaces to that length
  auto render = [&](bool zero, size_t base, std::vector<size_t>* offs) {
    Value table = Value::array();
    size_t off = base;
    for (const Ref& r : refs) {
      off = align_up(off, kAlign);
      Value e = Value::object();
      e["name"] = r.name;
      e["shape"] = Value(std::vector<int>{r.rows, r.cols});
      e["width"] = static_cast<int>(sizeof(T));
      e["offset"] = static_cast<long long>(zero ? 0 : off);
      table.push_back(e);
      if (offs) offs->push_back(off);
      off += r.bytes;
    }
    Value m = manifest;
    m["tensors"] = table;
    return m.dump();
  };
  const size_t mlen = render(true, 0, nullptr).size() + refs.size() * 24;
  const size_t base = align_up(16 + mlen, kAlign);
  std::vector<size_t> offs;
  std::string body = render(false, base, &offs);
  require(body.size() <= mlen, DSMOE_E_INTERNAL, "manifest length estimate too small");
  body.resize(mlen, ' ');
  std::string out;
  out.reserve(base + (refs.empty() ? 0 : offs.back() + refs.back().bytes));
  out.append(kMagic, 8);
  put_u64(out, mlen);
  out += body;
  for (size_t i = 0; i < refs.size(); ++i) {
    out.resize(offs[i], '\0');
    out.append(static_cast<const char*>(refs[i].data), refs[i].bytes);
  }
  write_atomic(path, out);
}

Config config_from_manifest(const Value& j) {
  Config c;
  c.d_model = static_cast<int>(j.at("d_model").as_int());
  c.d_ffn = static_cast<int>(j.at("d_ffn").as_int());
  c.num_experts = static_cast<int>(j.at("num_experts").as_int());
  c.top_k = static_cast<int>(j.at("top_k").as_int());
  c.num_shared_experts = static_cast<int>(j.at("num_shared_experts").as_int());
  c.gate_prenormalized = j.at("gate_prenormalized").as_bool();
  return c;
}

template <class T>
std::vector<Layer<T>> layers_from_container(const Value& man, const std::string& raw) {
  const int nl = static_cast<int>(man.at("num_layers").as_int());
  require(nl >= 1, DSMOE_E_SCHEMA, "container: num_layers must be >= 1");
  const Value& jls = man.at("layers");
  require(jls.is_array() && static_cast<int>(jls.size()) == nl, DSMOE_E_SCHEMA,
          "container: layer list does not match num_layers");
  const Value& jt = man.at("tensors");
  require(jt.is_array(), DSMOE_E_SCHEMA, "container: tensor table missing");
  struct Entry {
    std::string name;
    int rows, cols;
    size_t offset, bytes;
  };
  std::vector<Entry> ents;
  size_t prev_end = 0;
  for (const Value& e : jt.items()) {
    Entry en;
    en.name = e.at("name").as_string();
    const Value& sh = e.at("shape");
    require(sh.is_array() && sh.size() == 2, DSMOE_E_SCHEMA, "container: tensor shape must be [rows, cols]");
    en.rows = static_cast<int>(sh[0].as_int());
    en.cols = static_cast<int>(sh[1].as_int());
    require(en.rows >= 0 && en.cols >= 0, DSMOE_E_SCHEMA, "container: negative tensor shape");
    require(e.at("width").as_int() == static_cast<long long>(sizeof(T)), DSMOE_E_SCHEMA,
            "container: tensor width disagrees with scalar_width");
    const long long off = e.at("offset").as_int();
    require(off >= 0, DSMOE_E_SCHEMA, "container: negative tensor offset");
    en.offset = static_cast<size_t>(off);
    en.bytes = static_cast<size_t>(en.rows) * static_cast<size_t>(en.cols) * sizeof(T);
    require(en.offset % kAlign == 0, DSMOE_E_SCHEMA, "container: tensor offset not 64-byte aligned: " + en.name);
    require(en.offset >= prev_end, DSMOE_E_SCHEMA, "container: overlapping or out-of-order tensor offsets at " + en.name);
    prev_end = en.offset + en.bytes;
    require(prev_end <= raw.size(), DSMOE_E_TRUNCATED, "container: payload truncated at " + en.name);
    ents.push_back(std::move(en));
  }
  size_t next = 0;
  auto take = [&](const std::string& name) {
    require(next < ents.size() && ents[next].name == name, DSMOE_E_SCHEMA, "container: expected tensor " + name);
    const Entry& en = ents[next++];
    Mat<T> m(en.rows, en.cols);
    std::memcpy(m.v.data(), raw.data() + en.offset, en.bytes);
    return m;
  };
  std::vector<Layer<T>> layers;
  for (int l = 0; l < nl; ++l) {
    const Value& jl = jls[static_cast<size_t>(l)];
    Layer<T> L;
    L.cfg = config_from_manifest(jl.at("config"));
    L.lineage = lineage_of(jl.at("lineage").as_string());
    L.replay = static_cast<int>(jl.at("replay_factor").as_int());
    for (const Value& o : jl.at("neuron_order").items()) {
      std::vector<int> row;
      for (const Value& v : o.items()) row.push_back(static_cast<int>(v.as_int()));
      L.order.push_back(std::move(row));
    }
    const std::string b = "layers/" + std::to_string(l) + "/";
    L.gate = take(b + "gate");
    const int blocks = L.cfg.num_experts * L.replay;
    for (int e = 0; e < blocks; ++e) {
      const std::string eb = b + "experts/" + std::to_string(e) + "/";
      Block<T> bl;
      bl.w1 = take(eb + "w1");
      bl.w3 = take(eb + "w3");
      bl.w2 = take(eb + "w2");
      L.experts.push_back(std::move(bl));
    }
    for (int s = 0; s < L.cfg.num_shared_experts; ++s) {
      const std::string sb = b + "shared/" + std::to_string(s) + "/";
      Block<T> bl;
      bl.w1 = take(sb + "w1");
      bl.w3 = take(sb + "w3");
      bl.w2 = take(sb + "w2");
      L.shared.push_back(std::move(bl));
    }
    layers.push_back(std::move(L));
  }
  require(next == ents.size(), DSMOE_E_SCHEMA, "container: unused tensors in table");
  try {
    validate_model(layers);
  } catch (const AbiError& e) {
    fail(DSMOE_E_SCHEMA, std::string("container: inconsistent model: ") + e.what());
  }
  return layers;
}

dsmoe_model* load_container(const char* path) {
  const std::string raw = read_all(path);
  require(raw.size() >= 16, DSMOE_E_TRUNCATED, "container: file shorter than header");
  require(std::memcmp(raw.data(), kMagic, 8) == 0, DSMOE_E_BAD_MAGIC, "container: bad magic");
  const uint64_t mlen = get_u64(raw.data() + 8);
  require(16 + mlen <= raw.size(), DSMOE_E_TRUNCATED, "container: manifest truncated");
  Value man;
  try {
    man = minijson::parse(raw.substr(16, static_cast<size_t>(mlen)));
  } catch (const minijson::Error& e) {
    fail(DSMOE_E_SCHEMA, std::string("container: manifest is not valid JSON: ") + e.what());
  }
  try {
    require(man.at("format").as_string() == "dsmoe-container", DSMOE_E_SCHEMA, "container: unknown format tag");
    require(man.at("version").as_int() == 1, DSMOE_E_SCHEMA, "container: unsupported version");
    const long long w = man.at("scalar_width").as_int();
    auto m = std::make_unique<dsmoe_model>();
    if (w == 4) {
      m->width = 4;
      m->f = layers_from_container<float>(man, raw);
    } else if (w == 8) {
      m->width = 8;
      m->d = layers_from_container<double>(man, raw);
    } else {
      fail(DSMOE_E_SCHEMA, "container: scalar_width must be 4 or 8");
    }
    return m.release();
  } catch (const minijson::Error& e) {
    fail(DSMOE_E_SCHEMA, std::string("container: manifest field error: ") + e.what());
  }
}

// ------------------------------------------------------- policy document
struct Policy {  // DropPolicy (dropping.hpp:12-56) as policy_from builds it (capi.cpp:96-112)
  int kind = DSMOE_B200_DROP_NONE;
  double t_drop = 0.0, t_major = 0.0, t_minor = 0.0;
  bool keep_top1 = true, normalize = true;
  const char* kind_name() const { return kind == 0 ? "none" : (kind == 1 ? "1t" : "2t"); }
  dsmoe_b200_policy c(const double* t_unit = nullptr) const {
    return dsmoe_b200_policy{kind, t_drop, t_major, t_minor, keep_top1 ? 1 : 0, normalize ? 1 : 0, t_unit};
  }
  Value json() const {
    Value v = Value::object();
    v["kind"] = kind_name();
    v["t_drop"] = t_drop;
    v["t_major"] = t_major;
    v["t_minor"] = t_minor;
    v["keep_top1"] = keep_top1;
    v["normalize"] = normalize;
    return v;
  }
};

Policy policy_from(const Value& j, bool prenorm) {
  const std::string kind = j.get("kind", "none");
  Policy p;
  if (kind == "none") {
  } else if (kind == "1t") {
    p.kind = DSMOE_B200_DROP_1T;
    p.t_drop = j.at("t_drop").as_double();
  } else if (kind == "2t") {
    p.kind = DSMOE_B200_DROP_2T;
    p.t_drop = j.at("t_drop").as_double();
    p.t_major = j.get("t_major", p.t_drop - 0.01);
    p.t_minor = j.get("t_minor", p.t_drop + 0.01);
    check_arg(p.t_major <= p.t_minor, "drop policy: t_major must be <= t_minor");
  } else {
    fail(DSMOE_E_INVALID_ARGUMENT, "policy: unknown kind: " + kind);
  }
  p.keep_top1 = j.get("keep_top1", true);
  p.normalize = j.get("normalize", !prenorm);
  return p;
}

Value stats_json(const dsmoe_b200_drop_stats_t& s) {
  Value v = Value::object();
  v["num_tokens"] = static_cast<long long>(s.num_tokens);
  v["total_routed_units"] = s.total_routed_units;
  v["dropped_units"] = s.dropped_units;
  v["shared_units"] = s.shared_units;
  v["drop_rate"] = s.drop_rate;
  v["total_flops"] = s.total_flops;
  v["saved_flops"] = s.saved_flops;
  v["retained_flops"] = s.retained_flops;
  return v;
}

std::string fmt_double(double v) {  // reports.cpp fmt_double: %.17g, named non-finite values
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// ---------------------------------------------------------- device side
// One stream + device context per call (calls on distinct or const handles
// may run concurrently, SPEC "Concurrency Model").
struct Device {
  cudaStream_t s = nullptr;
  dsmoe_b200_ctx* ctx = nullptr;
  Device() {
    cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    dev(dsmoe_b200_ctx_create(s, &ctx));
  }
  ~Device() {
    dsmoe_b200_ctx_free(ctx);
    cudaStreamDestroy(s);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
};

struct Buf {
  void* p = nullptr;
  size_t n = 0;
  Buf() = default;
  explicit Buf(size_t bytes) { alloc(bytes); }
  void alloc(size_t bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    n = bytes;
    cuda(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc");
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

dsmoe_b200_layer* upload_layer(const Layer<float>& L, cudaStream_t s) {
  std::vector<int32_t> w, sw;
  for (const auto& b : L.experts) w.push_back(b.width());
  for (const auto& b : L.shared) sw.push_back(b.width());
  dsmoe_b200_layer_config cfg{L.cfg.d_model, L.cfg.d_ffn, L.cfg.num_experts, L.cfg.top_k, L.cfg.num_shared_experts,
                              L.cfg.gate_prenormalized ? 1 : 0, L.replay, DSMOE_B200_F32, w.data(),
                              sw.empty() ? nullptr : sw.data()};
  dsmoe_b200_layer* D = nullptr;
  dev(dsmoe_b200_layer_create(&cfg, &D));
  try {
    dev(dsmoe_b200_layer_set_gate(D, L.gate.v.data(), DSMOE_B200_F32, 0, s));
    for (size_t b = 0; b < L.experts.size(); ++b)
      dev(dsmoe_b200_layer_set_block(D, static_cast<int>(b), L.experts[b].w1.v.data(), L.experts[b].w3.v.data(),
                                     L.experts[b].w2.v.data(), DSMOE_B200_F32, 0, s));
    for (size_t i = 0; i < L.shared.size(); ++i)
      dev(dsmoe_b200_layer_set_shared(D, static_cast<int>(i), L.shared[i].w1.v.data(), L.shared[i].w3.v.data(),
                                      L.shared[i].w2.v.data(), DSMOE_B200_F32, 0, s));
  } catch (...) {
    dsmoe_b200_layer_free(D);
    throw;
  }
  return D;
}

// device copy of layer l of an fp32 model (cached on the handle)
const dsmoe_b200_layer* device_layer(const dsmoe_model& m, int l, cudaStream_t s) {
  int cur = 0;
  cuda(cudaGetDevice(&cur), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(m.mu);
  if (m.dev_id < 0) m.dev_id = cur;
  std::vector<dsmoe_b200_layer*>* cache = &m.dev;
  if (cur != m.dev_id) {  // the handle is used from another GPU: a separate set of copies there
    cache = nullptr;
    for (auto& o : m.other)
      if (o.first == cur) cache = &o.second;
    if (!cache) {
      m.other.emplace_back(cur, std::vector<dsmoe_b200_layer*>{});
      cache = &m.other.back().second;
    }
  }
  if (cache->size() != m.f.size()) cache->assign(m.f.size(), nullptr);
  auto& slot = (*cache)[static_cast<size_t>(l)];
  if (!slot) slot = upload_layer(m.f[static_cast<size_t>(l)], s);
  return slot;
}

// device fp32 layer -> host Layer<float> (weights in the reference layout)
Layer<float> download_layer(const dsmoe_b200_layer* D, Device& g) {
  int32_t info[8];
  dev(dsmoe_b200_layer_info(D, info));
  Layer<float> L;
  L.cfg.d_model = info[0];
  L.cfg.d_ffn = info[1];
  L.cfg.num_experts = info[2];
  L.cfg.top_k = info[3];
  L.cfg.num_shared_experts = info[4];
  L.replay = info[5];
  L.cfg.gate_prenormalized = info[7] != 0;
  std::vector<int32_t> bw(static_cast<size_t>(info[2]) * info[5]), sw(static_cast<size_t>(std::max(1, info[4])));
  dev(dsmoe_b200_layer_widths(D, bw.data(), sw.data()));
  const int d = info[0];
  L.gate = Mat<float>(d, info[2]);
  dev(dsmoe_b200_layer_get_gate(g.ctx, D, L.gate.v.data(), 0));
  auto get = [&](bool shared, int i, int w) {
    Block<float> b;
    b.w1 = Mat<float>(d, w);
    b.w3 = Mat<float>(d, w);
    b.w2 = Mat<float>(w, d);
    if (shared)
      dev(dsmoe_b200_layer_get_shared(g.ctx, D, i, b.w1.v.data(), b.w3.v.data(), b.w2.v.data(), 0));
    else
      dev(dsmoe_b200_layer_get_block(g.ctx, D, i, b.w1.v.data(), b.w3.v.data(), b.w2.v.data(), 0));
    return b;
  };
  for (size_t b = 0; b < bw.size(); ++b) L.experts.push_back(get(false, static_cast<int>(b), bw[b]));
  for (int i = 0; i < info[4]; ++i) L.shared.push_back(get(true, i, sw[static_cast<size_t>(i)]));
  return L;
}

Buf upload_tokens(const Tokens& t, int d_model, cudaStream_t s) {
  require(t.cols == d_model, DSMOE_E_SHAPE_MISMATCH,
          "gate_scores: token width " + std::to_string(t.cols) + " does not match d_model " + std::to_string(d_model));
  Buf b(t.v.size() * 4);
  cuda(cudaMemcpyAsync(b.p, t.v.data(), t.v.size() * 4, cudaMemcpyHostToDevice, s), "H2D tokens");
  return b;
}

// The residual chain x_{l+1} = x_l + moe_l(x_l) on the device (model_forward
// moe.hpp:328 with policy none, model_forward_dropped dropping.hpp:263-274
// otherwise), exact fp32 logits; returns the buffer holding the output.
Buf chain(const dsmoe_model& m, const Tokens& tok, Device& g, const Policy* policy,
          std::vector<dsmoe_b200_drop_stats_t>* stats) {
  const auto& layers = fp32_layers(m);
  Buf a = upload_tokens(tok, layers[0].cfg.d_model, g.s);
  Buf b(a.n);
  for (size_t l = 0; l < layers.size(); ++l) {
    const dsmoe_b200_layer* D = device_layer(m, static_cast<int>(l), g.s);
    Policy none;
    none.normalize = false;  // full_forward routes without renormalising (moe.hpp:320-323)
    const dsmoe_b200_policy pc = (policy ? *policy : none).c();
    dsmoe_b200_drop_stats_t st{};
    dev(dsmoe_b200_forward_ex(g.ctx, D, a.p, tok.rows, &pc, DSMOE_B200_LOGITS_EXACT, DSMOE_B200_RESIDUAL, b.p,
                              stats ? &st : nullptr));
    if (stats) stats->push_back(st);
    std::swap(a.p, b.p);
  }
  dev(dsmoe_b200_ctx_check(g.ctx));
  return a;
}

// per-token comparison of two device outputs (compare_rows_kernel)
std::vector<double> compare(const Buf& y, const Buf& base, int T, int d, Device& g) {
  Buf o(static_cast<size_t>(T) * 5 * 8);
  if (dsb::launch_compare_rows(0, y.p, base.p, T, d, o.as<double>(), g.s) != 0) fail(DSMOE_E_INTERNAL, "compare rows");
  std::vector<double> h(static_cast<size_t>(T) * 5);
  cuda(cudaMemcpyAsync(h.data(), o.p, h.size() * 8, cudaMemcpyDeviceToHost, g.s), "D2H");
  cuda(cudaStreamSynchronize(g.s), "sync");
  return h;
}

// mean_relative_error (dropping.hpp:278-293): mean over tokens of
// ||a_t - b_t|| / ||b_t||, b the baseline
double mean_rel_error(const std::vector<double>& cmp, int T) {
  double acc = 0.0;
  for (int t = 0; t < T; ++t) {
    const double d2 = cmp[5 * t], b2 = cmp[5 * t + 1];
    acc += b2 > 0.0 ? std::sqrt(d2) / std::sqrt(b2) : std::sqrt(d2);
  }
  return T > 0 ? acc / T : 0.0;
}

int metric_code(const std::string& s) {  // metric_from_name (reconstruct.hpp:25-31)
  if (s == "gate") return DSMOE_B200_METRIC_GATE;
  if (s == "abs_gate" || s == "abs-gate") return DSMOE_B200_METRIC_ABS_GATE;
  if (s == "gate_up" || s == "gate-up") return DSMOE_B200_METRIC_GATE_UP;
  if (s == "abs_gate_up" || s == "abs-gate-up") return DSMOE_B200_METRIC_ABS_GATE_UP;
  fail(DSMOE_E_INVALID_ARGUMENT, "unknown importance metric: " + s);
}
const char* kMetricName[] = {"gate", "abs_gate", "gate_up", "abs_gate_up"};

// Placement::device_of of place_experts (ep_sim.hpp:38-54)
std::vector<int32_t> place(int n, int devices, const std::string& strategy) {
  bool rr;
  if (strategy == "round_robin" || strategy == "round-robin")
    rr = true;
  else if (strategy == "contiguous")
    rr = false;
  else
    fail(DSMOE_E_INVALID_ARGUMENT, "unknown placement strategy: " + strategy);
  check_arg(devices >= 1 && n >= devices, "place_experts: need num_experts >= devices >= 1");
  std::vector<int32_t> dv(static_cast<size_t>(n));
  if (rr) {
    for (int e = 0; e < n; ++e) dv[static_cast<size_t>(e)] = e % devices;
  } else {
    check_arg(n % devices == 0, "place_experts: contiguous placement needs num_experts divisible by devices");
    for (int e = 0; e < n; ++e) dv[static_cast<size_t>(e)] = e / (n / devices);
  }
  return dv;
}

// sum of n additions of w, in order (the reference's device_loads adds
// fraction / P slot by slot, ep_sim.hpp:66-70; every kept copy adds the same
// w, so a device's load depends only on how many copies it received)
double repeated_sum(double w, long long n) {
  if (n == 0) return 0.0;
  double f;
  int e;
  f = std::frexp(w, &e);
  if (f == 0.5) return static_cast<double>(n) * w;  // w a power of two: every partial sum is exact
  double s = 0.0;
  for (long long i = 0; i < n; ++i) s += w;
  return s;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

int dsmoe_b200_simulate_step(dsmoe_b200_ctx* ctx, const dsmoe_b200_layer* layer, const void* x, int T, int devices,
                             const int32_t* device_of, const dsmoe_b200_policy* policy, int load_aware,
                             int logits_mode, double* pre_loads, double* post_loads, double* thresholds,
                             double* scalars3, dsmoe_b200_drop_stats_t* stats, const dsmoe_b200_routing* post,
                             void* y, int flags) {
  return guarded([&] {
    check_arg(ctx && layer && device_of && policy && pre_loads && post_loads && thresholds && scalars3,
              "null argument");
    check_arg(T >= 1 && x, "simulate_step: empty batch");
    check_arg(devices >= 1, "placement: need at least one device");
    int32_t info[8];
    dev(dsmoe_b200_layer_info(layer, info));
    const int E = info[2], P = info[5];
    for (int b = 0; b < E * P; ++b)
      require(device_of[b] >= 0 && device_of[b] < devices, DSMOE_E_INVALID_STATE, "placement: device id out of range");
    if (policy->kind == DSMOE_B200_DROP_2T)
      require(P == 2, DSMOE_E_INVALID_STATE, "simulate_step: 2T policy needs a layer split into major/minor halves");
    // 1. pre-drop routing (ensure_normalized as the policy says): per-expert selection counts
    dsmoe_b200_policy none = *policy;
    none.kind = DSMOE_B200_DROP_NONE;
    none.t_unit = nullptr;
    std::vector<int32_t> seg(static_cast<size_t>(3) * E);
    int R = 0;
    dev(dsmoe_b200_dispatch(ctx, layer, x, T, &none, logits_mode, nullptr, nullptr, seg.data(), &R, nullptr));
    const double w = 1.0 / P;
    std::vector<long long> copies(static_cast<size_t>(devices), 0);
    for (int e = 0; e < E; ++e)
      for (int p = 0; p < P; ++p) copies[static_cast<size_t>(device_of[e * P + p])] += seg[3 * e + 2];
    double total = 0.0;
    for (int dv = 0; dv < devices; ++dv) {
      pre_loads[dv] = repeated_sum(w, copies[static_cast<size_t>(dv)]);
      total += pre_loads[dv];
    }
    const double ideal = total / devices;
    // 2. per-device thresholds (load_aware_thresholds, ep_sim.hpp:76-89) and the
    //    owner table: a selection uses its copy-0 block's device (ep_sim.hpp:139-141)
    if (policy->kind == DSMOE_B200_DROP_NONE) {
      for (int dv = 0; dv < devices; ++dv) thresholds[dv] = 0.0;
    } else if (load_aware) {
      dev(dsmoe_b200_load_aware_thresholds(pre_loads, devices, policy->t_drop, thresholds));
    } else {
      for (int dv = 0; dv < devices; ++dv) thresholds[dv] = policy->t_drop;
    }
    std::vector<double> tu(static_cast<size_t>(E));
    for (int e = 0; e < E; ++e) tu[static_cast<size_t>(e)] = thresholds[device_of[e * P]];
    Buf d_tu(tu.size() * 8);
    cuda(cudaMemcpy(d_tu.p, tu.data(), tu.size() * 8, cudaMemcpyHostToDevice), "H2D thresholds");
    dsmoe_b200_policy pol = *policy;
    pol.t_unit = policy->kind == DSMOE_B200_DROP_NONE ? nullptr : d_tu.as<double>();
    // 3. the dropped routing (from the same logits), its forward and its loads
    dsmoe_b200_drop_stats_t st{};
    if (y) {
      dev(dsmoe_b200_forward_ex(ctx, layer, x, T, &pol, DSMOE_B200_LOGITS_REUSE, flags, y, &st));
      std::vector<int32_t> sg(static_cast<size_t>(3) * E);
      int rt = 0;
      dev(dsmoe_b200_ctx_permutation(ctx, T, info[3], E, nullptr, nullptr, sg.data(), &rt));
      seg = sg;
    } else {
      dev(dsmoe_b200_dispatch(ctx, layer, x, T, &pol, DSMOE_B200_LOGITS_REUSE, nullptr, nullptr, seg.data(), &R, &st));
    }
    if (post) dev(dsmoe_b200_route(ctx, layer, x, T, &pol, DSMOE_B200_LOGITS_REUSE, nullptr, nullptr, post, nullptr));
    dev(dsmoe_b200_ctx_check(ctx));  // the threshold table is read until here
    std::fill(copies.begin(), copies.end(), 0);
    std::vector<double> halves(static_cast<size_t>(devices), 0.0);
    for (int e = 0; e < E; ++e) {
      const long long nf = seg[3 * e + 1], nm = seg[3 * e + 2] - seg[3 * e + 1];
      if (P == 1) {  // fraction 1 (full) or 0.5 (first half): sums of 1 and 0.5, exact in any order
        halves[static_cast<size_t>(device_of[e])] += static_cast<double>(nf) + 0.5 * static_cast<double>(nm);
      } else {  // copy 0 kept by full and major-only selections, copies >= 1 by full ones (fraction 1)
        copies[static_cast<size_t>(device_of[e * P])] += nf + nm;
        for (int p = 1; p < P; ++p) copies[static_cast<size_t>(device_of[e * P + p])] += nf;
      }
    }
    for (int dv = 0; dv < devices; ++dv)
      post_loads[dv] = P == 1 ? halves[static_cast<size_t>(dv)] : repeated_sum(w, copies[static_cast<size_t>(dv)]);
    const double mx_pre = *std::max_element(pre_loads, pre_loads + devices);
    const double mx_post = *std::max_element(post_loads, post_loads + devices);
    scalars3[0] = ideal;
    scalars3[1] = st.drop_rate;
    scalars3[2] = mx_post > 0.0 ? mx_pre / mx_post : (mx_pre > 0.0 ? std::numeric_limits<double>::infinity() : 1.0);
    if (stats) *stats = st;
  });
}

const char* dsmoe_version(void) { return "1.0.0"; }

const char* dsmoe_status_name(int code) {
  static const char* names[] = {"ok",      "invalid_argument", "shape_mismatch", "invalid_state", "io_error",
                                "bad_magic", "truncated",      "schema_error",   "internal"};
  return code >= 0 && code <= 8 ? names[code] : "unknown";
}

const char* dsmoe_last_error(void) { return t_last_error.c_str(); }

void dsmoe_string_free(char* s) { delete[] s; }

void dsmoe_model_free(dsmoe_model* m) { delete m; }

int dsmoe_generate_model(const char* config_json, uint64_t seed, double scale, int scalar_width, dsmoe_model** out) {
  return guarded([&] {
    check_arg(out != nullptr, "output pointer is null");
    const Value j = parse_doc(config_json, "config");
    Config c;
    c.d_model = static_cast<int>(j.at("d_model").as_int());
    c.d_ffn = static_cast<int>(j.at("d_ffn").as_int());
    c.num_experts = static_cast<int>(j.at("num_experts").as_int());
    c.top_k = static_cast<int>(j.at("top_k").as_int());
    c.num_shared_experts = j.get("num_shared_experts", 0);
    c.gate_prenormalized = j.get("gate_prenormalized", false);
    c.validate();
    const int nl = j.get("num_layers", 1);
    check_arg(scalar_width == 4 || scalar_width == 8, "scalar_width must be 4 or 8");
    check_arg(nl >= 1, "generate_model: num_layers must be >= 1");
    auto m = std::make_unique<dsmoe_model>();
    m->width = scalar_width;
    SplitMix64 mix{seed};  // layer l: the l-th SplitMix64 output (io.cpp generate_model)
    for (int l = 0; l < nl; ++l) {
      const uint64_t ls = mix.next();
      if (scalar_width == 4)
        m->f.push_back(generate_layer<float>(c, ls, scale));
      else
        m->d.push_back(generate_layer<double>(c, ls, scale));
    }
    *out = m.release();
  });
}

int dsmoe_generate_tokens(int64_t rows, int64_t cols, uint64_t seed, double scale, const char* path) {
  return guarded([&] {
    check_arg(path != nullptr, "path is null");
    check_arg(rows >= 1 && cols >= 1, "generate_tokens: bad shape");
    Xoshiro rng(seed);
    std::string out;
    put_u64(out, static_cast<uint64_t>(rows));
    put_u64(out, static_cast<uint64_t>(cols));
    out.reserve(16 + static_cast<size_t>(rows * cols) * 4);
    for (int64_t i = 0; i < rows * cols; ++i) {
      const float f = static_cast<float>(rng.gaussian() * scale);
      char b[4];
      std::memcpy(b, &f, 4);
      out.append(b, 4);
    }
    write_atomic(path, out);
  });
}

int dsmoe_model_load(const char* path, dsmoe_model** out) {
  return guarded([&] {
    check_arg(path != nullptr && out != nullptr, "path or output pointer is null");
    *out = load_container(path);
  });
}

int dsmoe_model_save(const dsmoe_model* m, const char* path) {
  return guarded([&] {
    check_arg(path != nullptr, "path is null");
    const dsmoe_model& M = model_ref(m);
    if (M.width == 4)
      save_container(M.f, path);
    else
      save_container(M.d, path);
  });
}

int dsmoe_model_info(const dsmoe_model* m, char** json_out) {
  return guarded([&] {
    check_arg(json_out != nullptr, "output pointer is null");
    const dsmoe_model& M = model_ref(m);
    Value layers = Value::array();
    Config c;
    auto describe = [&](const auto& ls) {
      validate_model(ls);
      c = ls[0].cfg;
      for (const auto& L : ls) {
        Value v = Value::object();
        v["lineage"] = kLineage[L.lineage];
        v["replay_factor"] = L.replay;
        v["physical_experts"] = L.cfg.num_experts * L.replay;
        v["block_width"] = L.experts.empty() ? 0 : L.experts[0].width();
        v["reconstructed"] = !L.order.empty();
        layers.push_back(v);
      }
    };
    if (M.width == 4)
      describe(M.f);
    else
      describe(M.d);
    Value info = Value::object();
    info["scalar_width"] = M.width;
    info["num_layers"] = M.num_layers();
    info["config"] = c.json();
    info["layers"] = layers;
    set_out(json_out, info.dump(2) + "\n");
  });
}

int dsmoe_transform(const dsmoe_model* m, const char* mode, int p, dsmoe_model** out) {
  return guarded([&] {
    check_arg(mode != nullptr && out != nullptr, "mode or output pointer is null");
    const std::string ms = mode;
    check_arg(ms == "complete" || ms == "partial", "mode must be complete or partial");
    const auto& layers = fp32_layers(model_ref(m));
    Device g;
    auto res = std::make_unique<dsmoe_model>();
    cuda(cudaGetDevice(&res->dev_id), "cudaGetDevice");  // seeded with this device's copies
    res->width = 4;
    for (size_t l = 0; l < layers.size(); ++l) {
      const dsmoe_b200_layer* D = device_layer(*m, static_cast<int>(l), g.s);
      dsmoe_b200_layer* R = nullptr;
      dev(dsmoe_b200_transform(g.ctx, D, ms == "complete" ? DSMOE_B200_TRANSFORM_COMPLETE : DSMOE_B200_TRANSFORM_PARTIAL,
                               p, &R));
      std::unique_ptr<dsmoe_b200_layer, void (*)(dsmoe_b200_layer*)> keep(R, dsmoe_b200_layer_free);
      Layer<float> L = download_layer(R, g);
      L.lineage = ms == "complete" ? 1 : 2;
      res->f.push_back(std::move(L));
      res->dev.push_back(keep.release());
    }
    validate_model(res->f);
    *out = res.release();
  });
}

int dsmoe_reverse_partial(const dsmoe_model* m, dsmoe_model** out) {
  return guarded([&] {
    check_arg(out != nullptr, "output pointer is null");
    const auto& layers = fp32_layers(model_ref(m));
    Device g;
    auto res = std::make_unique<dsmoe_model>();
    cuda(cudaGetDevice(&res->dev_id), "cudaGetDevice");  // seeded with this device's copies
    for (size_t l = 0; l < layers.size(); ++l) {
      const Layer<float>& S = layers[l];
      require(S.replay > 1, DSMOE_E_INVALID_STATE, "reverse: model does not carry a partial transformation");
      dsmoe_b200_layer* R = nullptr;
      dev(dsmoe_b200_transform(g.ctx, device_layer(*m, static_cast<int>(l), g.s), DSMOE_B200_TRANSFORM_REVERSE, 0, &R));
      std::unique_ptr<dsmoe_b200_layer, void (*)(dsmoe_b200_layer*)> keep(R, dsmoe_b200_layer_free);
      Layer<float> L = download_layer(R, g);
      L.lineage = 0;  // base, natural order (transform.hpp:148-150)
      res->f.push_back(std::move(L));
      res->dev.push_back(keep.release());
    }
    *out = res.release();
  });
}

int dsmoe_reconstruct(const dsmoe_model* m, const char* tokens_path, const char* metric, dsmoe_model** out,
                      char** profiles_json_out) {
  return guarded([&] {
    check_arg(tokens_path != nullptr && metric != nullptr && out != nullptr,
              "tokens_path, metric, or output pointer is null");
    const int mt = metric_code(metric);
    const auto& layers = fp32_layers(model_ref(m));
    const Tokens calib = load_tokens(tokens_path);
    Device g;
    Buf cur = upload_tokens(calib, layers[0].cfg.d_model, g.s);
    Buf nxt(cur.n);
    const int T = calib.rows;
    auto res = std::make_unique<dsmoe_model>();
    cuda(cudaGetDevice(&res->dev_id), "cudaGetDevice");  // seeded with this device's copies
    Value profiles = Value::array();
    for (size_t l = 0; l < layers.size(); ++l) {
      const Layer<float>& S = layers[l];
      const dsmoe_b200_layer* D = device_layer(*m, static_cast<int>(l), g.s);
      const int E = S.cfg.num_experts, K = S.cfg.top_k, ffn = S.cfg.d_ffn;
      require(S.replay == 1, DSMOE_E_INVALID_STATE,
              "profile_importance: profile the original layer, not a partitioned one");
      check_arg(T >= 1, "profile_importance: empty calibration set");
      // route_tokens (no drop, no renormalisation) -> profile_importance ->
      // reconstruct_experts (capi.cpp:294-305), all on the device
      Buf idx(static_cast<size_t>(T) * K * 4), vals(static_cast<size_t>(E) * ffn * 8),
          ord(static_cast<size_t>(E) * ffn * 4);
      dsmoe_b200_routing r{idx.as<int32_t>(), nullptr, nullptr, nullptr};
      Policy none;
      none.normalize = false;
      const dsmoe_b200_policy pc = none.c();
      dev(dsmoe_b200_route(g.ctx, D, cur.p, T, &pc, DSMOE_B200_LOGITS_EXACT, nullptr, nullptr, &r, nullptr));
      dev(dsmoe_b200_profile_importance(g.ctx, D, cur.p, T, idx.as<int32_t>(), mt, vals.as<double>()));
      dsmoe_b200_layer* R = nullptr;
      dev(dsmoe_b200_reconstruct(g.ctx, D, vals.as<double>(), ord.as<int32_t>(), &R));
      std::unique_ptr<dsmoe_b200_layer, void (*)(dsmoe_b200_layer*)> keep(R, dsmoe_b200_layer_free);
      std::vector<double> hv(static_cast<size_t>(E) * ffn);
      std::vector<int32_t> ho(static_cast<size_t>(E) * ffn);
      cuda(cudaMemcpy(hv.data(), vals.p, hv.size() * 8, cudaMemcpyDeviceToHost), "D2H values");
      cuda(cudaMemcpy(ho.data(), ord.p, ho.size() * 4, cudaMemcpyDeviceToHost), "D2H order");
      Layer<float> L = download_layer(R, g);
      L.lineage = 3;
      L.cfg = S.cfg;
      for (int e = 0; e < E; ++e)
        L.order.emplace_back(ho.begin() + static_cast<long>(e) * ffn, ho.begin() + static_cast<long>(e + 1) * ffn);
      res->f.push_back(std::move(L));
      res->dev.push_back(keep.release());
      Value pv = Value::object();
      pv["metric"] = kMetricName[mt];
      pv["num_experts"] = E;
      pv["d_ffn"] = ffn;
      pv["token_count"] = T;
      pv["layer_index"] = static_cast<int>(l);
      Value rows = Value::array();
      for (int e = 0; e < E; ++e)
        rows.push_back(Value(std::vector<double>(hv.begin() + static_cast<long>(e) * ffn,
                                                 hv.begin() + static_cast<long>(e + 1) * ffn)));
      pv["values"] = rows;
      profiles.push_back(pv);
      // advance the calibration activations through the original layer
      dev(dsmoe_b200_forward_ex(g.ctx, D, cur.p, T, &pc, DSMOE_B200_LOGITS_EXACT, DSMOE_B200_RESIDUAL, nxt.p, nullptr));
      std::swap(cur.p, nxt.p);
    }
    dev(dsmoe_b200_ctx_check(g.ctx));
    validate_model(res->f);
    Value doc = Value::object();
    doc["profiles"] = profiles;
    set_out(profiles_json_out, doc.dump(2) + "\n");
    *out = res.release();
  });
}

int dsmoe_verify_equivalence(const dsmoe_model* a, const dsmoe_model* b, const char* tokens_path, double tol,
                             char** json_out) {
  return guarded([&] {
    check_arg(b != nullptr && tokens_path != nullptr, "model or tokens_path is null");
    const dsmoe_model& A = model_ref(a);
    require(A.width == b->width, DSMOE_E_INVALID_ARGUMENT, "verify: models have different scalar widths");
    fp32_layers(A);
    fp32_layers(*b);
    const Tokens tok = load_tokens(tokens_path);
    Device g;
    Buf ya = chain(A, tok, g, nullptr, nullptr);
    Buf yb = chain(*b, tok, g, nullptr, nullptr);
    const std::vector<double> c = compare(ya, yb, tok.rows, tok.cols, g);
    double mad = 0.0, scale = 0.0;
    for (int t = 0; t < tok.rows; ++t) {
      mad = std::max(mad, c[5 * t + 2]);
      scale = std::max({scale, c[5 * t + 3], c[5 * t + 4]});
    }
    Value v = Value::object();
    v["max_abs_diff"] = mad;
    v["max_rel_diff"] = scale > 0.0 ? mad / scale : mad;
    v["tol"] = tol;
    v["pass"] = (scale > 0.0 ? mad / scale : mad) <= tol;
    set_out(json_out, v.dump(2) + "\n");
  });
}

int dsmoe_infer(const dsmoe_model* m, const char* tokens_path, const char* policy_json, char** json_out) {
  return guarded([&] {
    check_arg(tokens_path != nullptr && json_out != nullptr, "tokens_path or output pointer is null");
    const auto& layers = fp32_layers(model_ref(m));
    const Policy pol = policy_from(parse_doc(policy_json, "policy"), layers[0].cfg.gate_prenormalized);
    const Tokens tok = load_tokens(tokens_path);
    Device g;
    Buf base = chain(*m, tok, g, nullptr, nullptr);
    std::vector<dsmoe_b200_drop_stats_t> st;
    Buf y = chain(*m, tok, g, &pol, &st);
    double dropped = 0.0, denom = 0.0, flops = 0.0, saved = 0.0;
    Value per = Value::array();
    for (const auto& s : st) {
      dropped += s.dropped_units;
      denom += s.total_routed_units + s.shared_units;
      flops += s.total_flops;
      saved += s.saved_flops;
      per.push_back(stats_json(s));
    }
    Value v = Value::object();
    v["policy"] = pol.json();
    v["drop_rate"] = denom > 0.0 ? dropped / denom : 0.0;
    v["dropped_units"] = dropped;
    v["total_units"] = denom;
    v["total_flops"] = flops;
    v["saved_flops"] = saved;
    v["rel_error"] = mean_rel_error(compare(y, base, tok.rows, tok.cols, g), tok.rows);
    v["per_layer"] = per;
    set_out(json_out, v.dump(2) + "\n");
  });
}

int dsmoe_sweep(const dsmoe_model* m, const char* tokens_path, const char* policy_kind, const double* thresholds,
                size_t n, int keep_top1, char** json_out, char** csv_out) {
  return guarded([&] {
    check_arg(tokens_path != nullptr && policy_kind != nullptr, "tokens_path or policy_kind is null");
    check_arg(thresholds != nullptr && n > 0, "threshold list is empty");
    const std::string kind = policy_kind;
    check_arg(kind == "1t" || kind == "2t", "policy_kind must be 1t or 2t");
    model_ref(m);
    const Tokens tok = load_tokens(tokens_path);
    check_arg(std::is_sorted(thresholds, thresholds + n), "threshold_sweep: thresholds must be sorted ascending");
    const auto& layers = fp32_layers(*m);
    Device g;
    Buf base = chain(*m, tok, g, nullptr, nullptr);
    Value rows = Value::array();
    std::string csv = "threshold,drop_rate,rel_error";
    for (size_t l = 0; l < layers.size(); ++l) csv += ",drop_rate_layer" + std::to_string(l);
    csv += "\n";
    for (size_t i = 0; i < n; ++i) {
      const double t = thresholds[i];
      Policy pol;  // one_t(t, keep) / two_t_from(t, keep) (dropping.hpp:326-328)
      pol.kind = kind == "1t" ? DSMOE_B200_DROP_1T : DSMOE_B200_DROP_2T;
      pol.t_drop = t;
      if (pol.kind == DSMOE_B200_DROP_2T) {
        pol.t_major = t - 0.01;
        pol.t_minor = t + 0.01;
      }
      pol.keep_top1 = keep_top1 != 0;
      pol.normalize = !layers[0].cfg.gate_prenormalized;
      std::vector<dsmoe_b200_drop_stats_t> st;
      Buf y = chain(*m, tok, g, &pol, &st);
      double dropped = 0.0, denom = 0.0;
      std::vector<double> rates;
      for (const auto& s : st) {
        dropped += s.dropped_units;
        denom += s.total_routed_units + s.shared_units;
        rates.push_back(s.drop_rate);
      }
      const double rate = denom > 0.0 ? dropped / denom : 0.0;
      const double err = mean_rel_error(compare(y, base, tok.rows, tok.cols, g), tok.rows);
      Value r = Value::object();
      r["threshold"] = t;
      r["drop_rate"] = rate;
      r["per_layer_rates"] = Value(rates);
      r["mean_rel_error"] = err;
      rows.push_back(r);
      csv += fmt_double(t) + "," + fmt_double(rate) + "," + fmt_double(err);
      for (double v : rates) csv += "," + fmt_double(v);
      csv += "\n";
    }
    Value doc = Value::object();
    doc["policy_kind"] = kind;
    doc["rows"] = rows;
    set_out(json_out, doc.dump(2) + "\n");
    set_out(csv_out, csv);
  });
}

int dsmoe_analyze_gating(const dsmoe_model* m, const char* tokens_path, int bins, char** json_out, char** csv_out) {
  return guarded([&] {
    check_arg(tokens_path != nullptr, "tokens_path is null");
    const auto& layers = fp32_layers(model_ref(m));
    const Tokens tok = load_tokens(tokens_path);
    check_arg(bins >= 2, "analyze_gating: bins must be >= 2");
    check_arg(tok.rows >= 1, "analyze_gating: empty token set");
    Device g;
    Buf x = upload_tokens(tok, layers[0].cfg.d_model, g.s);
    const int E = layers[0].cfg.num_experts;
    std::vector<long long> sel(static_cast<size_t>(E)), rh(static_cast<size_t>(bins)), nh(static_cast<size_t>(bins));
    dev(dsmoe_b200_analyze_gating(g.ctx, device_layer(*m, 0, g.s), x.p, tok.rows, bins, DSMOE_B200_LOGITS_EXACT,
                                  sel.data(), rh.data(), nh.data()));
    Value v = Value::object();
    v["bins"] = bins;
    v["num_tokens"] = tok.rows;
    v["top_k"] = layers[0].cfg.top_k;
    v["selection_counts"] = Value(sel);
    v["raw_hist"] = Value(rh);
    v["norm_hist"] = Value(nh);
    set_out(json_out, v.dump(2) + "\n");
    std::string csv = "series,index,bin_low,bin_high,count\n";
    for (int e = 0; e < E; ++e)
      csv += "selection," + std::to_string(e) + ",,," + std::to_string(sel[static_cast<size_t>(e)]) + "\n";
    auto hist = [&](const char* series, const std::vector<long long>& h) {
      for (int b = 0; b < bins; ++b)
        csv += std::string(series) + "," + std::to_string(b) + "," + fmt_double(static_cast<double>(b) / bins) + "," +
               fmt_double(static_cast<double>(b + 1) / bins) + "," + std::to_string(h[static_cast<size_t>(b)]) + "\n";
    };
    hist("raw", rh);
    hist("normalized", nh);
    set_out(csv_out, csv);
  });
}

int dsmoe_sim_ep(const dsmoe_model* m, const char* tokens_path, int devices, const char* strategy,
                 const char* policy_json, int load_aware, char** json_out) {
  return guarded([&] {
    check_arg(tokens_path != nullptr && strategy != nullptr && json_out != nullptr,
              "tokens_path, strategy, or output pointer is null");
    const auto& layers = fp32_layers(model_ref(m));
    const Policy pol = policy_from(parse_doc(policy_json, "policy"), layers[0].cfg.gate_prenormalized);
    const Tokens tok = load_tokens(tokens_path);
    const std::vector<int32_t> dv = place(layers[0].cfg.num_experts * layers[0].replay, devices, strategy);
    Device g;
    Buf cur = upload_tokens(tok, layers[0].cfg.d_model, g.s);
    Buf nxt(cur.n);
    Value out_layers = Value::array();
    for (size_t l = 0; l < layers.size(); ++l) {
      const Layer<float>& S = layers[l];
      check_arg(static_cast<int>(dv.size()) == S.cfg.num_experts * S.replay,
                "simulate_step: placement does not cover this layer's experts");
      std::vector<double> pre(static_cast<size_t>(devices)), post(static_cast<size_t>(devices)),
          th(static_cast<size_t>(devices));
      double sc[3];
      dsmoe_b200_drop_stats_t st{};
      const dsmoe_b200_policy pc = pol.c();
      dev(dsmoe_b200_simulate_step(g.ctx, device_layer(*m, static_cast<int>(l), g.s), cur.p, tok.rows, devices,
                                   dv.data(), &pc, load_aware, DSMOE_B200_LOGITS_EXACT, pre.data(), post.data(),
                                   th.data(), sc, &st, nullptr, nxt.p, DSMOE_B200_RESIDUAL));
      std::swap(cur.p, nxt.p);
      Value r = Value::object();
      r["devices"] = devices;
      r["load_aware"] = load_aware != 0;
      r["policy_kind"] = pol.kind_name();
      r["pre_loads"] = Value(pre);
      r["post_loads"] = Value(post);
      r["thresholds"] = Value(th);
      r["ideal_load"] = sc[0];
      r["drop_rate"] = sc[1];
      r["speedup"] = std::isfinite(sc[2]) ? Value(sc[2]) : Value(fmt_double(sc[2]));  // reports.cpp num()
      r["stats"] = stats_json(st);
      out_layers.push_back(r);
    }
    dev(dsmoe_b200_ctx_check(g.ctx));
    Value v = Value::object();
    v["devices"] = devices;
    v["strategy"] = strategy;
    v["load_aware"] = load_aware != 0;
    v["layers"] = out_layers;
    set_out(json_out, v.dump(2) + "\n");
  });
}

int dsmoe_sim_comm(const char* scenario_json, char** json_out) {
  (void)scenario_json;
  (void)json_out;
  return guarded([&] {
    fail(DSMOE_E_INVALID_STATE,
         "sim_comm: the alpha-beta communication model (comm_sim.cpp) is not part of the B200 device library; "
         "expert-parallel traffic is measured over NCCL instead (paper_2508_18376_b200/ep.py)");
  });
}

int dsmoe_sim_comm_sweep(const char* scenario_json, const int64_t* sizes, size_t n, char** json_out, char** csv_out) {
  (void)scenario_json;
  (void)sizes;
  (void)n;
  (void)json_out;
  (void)csv_out;
  return dsmoe_sim_comm(nullptr, nullptr);
}

}  // extern "C"
