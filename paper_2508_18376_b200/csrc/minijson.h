// Minimal JSON value / parser / printer for the reference-compatible C ABI
// (dsmoe_abi.cpp): policy and config documents in, reports and container
// manifests out.  Objects keep their keys sorted (std::map), the order the
// reference's documents are printed in (nlohmann::json's default object
// type), so `dump()` of a manifest reproduces the reference's container
// bytes.  Numbers: integers stay 64-bit integers, everything else a double
// printed with the fewest digits that read back to the same bits.
#pragma once

#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace minijson {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Value {
 public:
  enum class Type { Null, Bool, Int, Double, String, Array, Object };

  Value() = default;
  Value(std::nullptr_t) {}
  Value(bool b) : t_(Type::Bool), b_(b) {}
  Value(int v) : t_(Type::Int), i_(v) {}
  Value(long v) : t_(Type::Int), i_(v) {}
  Value(long long v) : t_(Type::Int), i_(v) {}
  Value(unsigned long v) : t_(Type::Int), i_(static_cast<long long>(v)) {}
  Value(unsigned long long v) : t_(Type::Int), i_(static_cast<long long>(v)) {}
  Value(double v) : t_(Type::Double), d_(v) {}
  Value(const char* s) : t_(Type::String), s_(s) {}
  Value(std::string s) : t_(Type::String), s_(std::move(s)) {}
  template <class T>
  Value(const std::vector<T>& v) : t_(Type::Array) {
    for (const auto& x : v) a_.emplace_back(x);
  }

  static Value array() {
    Value v;
    v.t_ = Type::Array;
    return v;
  }
  static Value object() {
    Value v;
    v.t_ = Type::Object;
    return v;
  }

  Type type() const { return t_; }
  bool is_null() const { return t_ == Type::Null; }
  bool is_number() const { return t_ == Type::Int || t_ == Type::Double; }
  bool is_array() const { return t_ == Type::Array; }
  bool is_object() const { return t_ == Type::Object; }
  bool is_string() const { return t_ == Type::String; }

  // ---- access (throws Error on a type mismatch, like json::at / get<T>)
  const Value& at(const std::string& k) const {
    need(Type::Object, "object");
    auto it = o_.find(k);
    if (it == o_.end()) throw Error("key '" + k + "' not found");
    return it->second;
  }
  bool contains(const std::string& k) const { return t_ == Type::Object && o_.count(k) > 0; }
  const Value& operator[](size_t i) const {
    need(Type::Array, "array");
    if (i >= a_.size()) throw Error("array index out of range");
    return a_[i];
  }
  Value& operator[](const std::string& k) {
    if (t_ == Type::Null) t_ = Type::Object;
    need(Type::Object, "object");
    return o_[k];
  }
  size_t size() const { return t_ == Type::Array ? a_.size() : (t_ == Type::Object ? o_.size() : 0); }
  const std::vector<Value>& items() const {
    need(Type::Array, "array");
    return a_;
  }
  const std::map<std::string, Value>& members() const {
    need(Type::Object, "object");
    return o_;
  }
  void push_back(Value v) {
    if (t_ == Type::Null) t_ = Type::Array;
    need(Type::Array, "array");
    a_.push_back(std::move(v));
  }

  double as_double() const {
    if (t_ == Type::Int) return static_cast<double>(i_);
    need(Type::Double, "number");
    return d_;
  }
  long long as_int() const {
    if (t_ == Type::Double) {
      if (d_ != std::floor(d_)) throw Error("number is not an integer");
      return static_cast<long long>(d_);
    }
    need(Type::Int, "integer");
    return i_;
  }
  bool as_bool() const {
    need(Type::Bool, "boolean");
    return b_;
  }
  const std::string& as_string() const {
    need(Type::String, "string");
    return s_;
  }
  // value(key, default) as nlohmann's json::value
  double get(const std::string& k, double def) const { return contains(k) ? at(k).as_double() : def; }
  long long get(const std::string& k, long long def) const { return contains(k) ? at(k).as_int() : def; }
  int get(const std::string& k, int def) const { return contains(k) ? static_cast<int>(at(k).as_int()) : def; }
  bool get(const std::string& k, bool def) const { return contains(k) ? at(k).as_bool() : def; }
  std::string get(const std::string& k, const char* def) const { return contains(k) ? at(k).as_string() : def; }

  // ---- output
  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

  static std::string number(double v) {
    if (!std::isfinite(v)) return "null";
    char buf[40];
    for (int prec = 1; prec <= 17; ++prec) {  // fewest digits that round-trip
      std::snprintf(buf, sizeof buf, "%.*g", prec, v);
      if (std::strtod(buf, nullptr) == v) break;
    }
    std::string s = buf;
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // keep it a floating-point literal
    return s;
  }

 private:
  void need(Type t, const char* what) const {
    if (t_ != t) throw Error(std::string("type must be ") + what);
  }
  static void escape(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\n': out += "\\n"; break;
        case '\r': out += "\\r"; break;
        case '\t': out += "\\t"; break;
        case '\b': out += "\\b"; break;
        case '\f': out += "\\f"; break;
        default:
          if (c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", c);
            out += b;
          } else {
            out += static_cast<char>(c);
          }
      }
    }
    out += '"';
  }
  void write(std::string& out, int indent, int level) const {
    const bool pretty = indent >= 0;
    auto nl = [&](int lv) {
      if (!pretty) return;
      out += '\n';
      out.append(static_cast<size_t>(indent) * lv, ' ');
    };
    switch (t_) {
      case Type::Null: out += "null"; break;
      case Type::Bool: out += b_ ? "true" : "false"; break;
      case Type::Int: out += std::to_string(i_); break;
      case Type::Double: out += number(d_); break;
      case Type::String: escape(out, s_); break;
      case Type::Array:
        if (a_.empty()) {
          out += "[]";
          break;
        }
        out += '[';
        for (size_t i = 0; i < a_.size(); ++i) {
          if (i) out += ',';
          nl(level + 1);
          a_[i].write(out, indent, level + 1);
        }
        nl(level);
        out += ']';
        break;
      case Type::Object:
        if (o_.empty()) {
          out += "{}";
          break;
        }
        out += '{';
        {
          bool first = true;
          for (const auto& kv : o_) {
            if (!first) out += ',';
            first = false;
            nl(level + 1);
            escape(out, kv.first);
            out += pretty ? ": " : ":";
            kv.second.write(out, indent, level + 1);
          }
        }
        nl(level);
        out += '}';
        break;
    }
  }

  Type t_ = Type::Null;
  bool b_ = false;
  long long i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> a_;
  std::map<std::string, Value> o_;
  friend class Parser;
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (p_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& m) const {
    throw Error("parse error at byte " + std::to_string(p_) + ": " + m);
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\r' || s_[p_] == '\t')) ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (p_ >= s_.size()) fail("unexpected end of input");
    const char c = s_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value(string());
    if (lit("true")) return Value(true);
    if (lit("false")) return Value(false);
    if (lit("null")) return Value();
    return number();
  }
  Value object() {
    Value v = Value::object();
    ++p_;
    ws();
    if (p_ < s_.size() && s_[p_] == '}') {
      ++p_;
      return v;
    }
    for (;;) {
      ws();
      if (p_ >= s_.size() || s_[p_] != '"') fail("expected a key");
      std::string k = string();
      ws();
      if (p_ >= s_.size() || s_[p_] != ':') fail("expected ':'");
      ++p_;
      v.o_[k] = value();
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < s_.size() && s_[p_] == '}') {
        ++p_;
        return v;
      }
      fail("expected ',' or '}'");
    }
  }
  Value array() {
    Value v = Value::array();
    ++p_;
    ws();
    if (p_ < s_.size() && s_[p_] == ']') {
      ++p_;
      return v;
    }
    for (;;) {
      v.a_.push_back(value());
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < s_.size() && s_[p_] == ']') {
        ++p_;
        return v;
      }
      fail("expected ',' or ']'");
    }
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (p_ + 4 > s_.size()) fail("bad \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = s_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= c - '0';
      else if (c >= 'a' && c <= 'f') v |= c - 'a' + 10;
      else if (c >= 'A' && c <= 'F') v |= c - 'A' + 10;
      else fail("bad \\u escape");
    }
    return v;
  }
  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < s_.size()) {
      const char c = s_[p_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= s_.size()) break;
      const char e = s_[p_++];
      switch (e) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && p_ + 6 <= s_.size() && s_[p_] == '\\' && s_[p_ + 1] == 'u') {
            p_ += 2;
            const unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    fail("unterminated string");
  }
  Value number() {
    const size_t b = p_;
    if (p_ < s_.size() && s_[p_] == '-') ++p_;
    bool is_int = true;
    if (p_ >= s_.size() || !(s_[p_] >= '0' && s_[p_] <= '9')) fail("invalid literal");
    while (p_ < s_.size()) {
      const char c = s_[p_];
      if (c >= '0' && c <= '9') {
        ++p_;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') {
        is_int = false;
        ++p_;
      } else {
        break;
      }
    }
    const std::string tok = s_.substr(b, p_ - b);
    char* end = nullptr;
    if (is_int) {
      errno = 0;
      const long long v = std::strtoll(tok.c_str(), &end, 10);
      if (errno == 0 && end && *end == '\0') return Value(v);
    }
    const double d = std::strtod(tok.c_str(), &end);
    if (!end || *end != '\0') fail("invalid number");
    return Value(d);
  }

  const std::string& s_;
  size_t p_ = 0;
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

}  // namespace minijson
