// JSON parse / dump for the scenario and report wire formats (see json.hpp).
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "microslice/json.hpp"

namespace microslice {

namespace {

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}

  json document() {
    json v = value();
    skip_ws();
    if (pos_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* what) const {
    throw ValidationError("json", std::string(what) + " at offset " + std::to_string(pos_));
  }
  void skip_ws() {
    while (pos_ < s_.size() &&
           (s_[pos_] == ' ' || s_[pos_] == '\n' || s_[pos_] == '\r' || s_[pos_] == '\t'))
      ++pos_;
  }
  bool eat(char c) {
    skip_ws();
    if (pos_ < s_.size() && s_[pos_] == c) {
      ++pos_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail((std::string("expected '") + c + "'").c_str());
  }
  bool literal(const char* word) {
    const std::size_t n = std::char_traits<char>::length(word);
    if (s_.compare(pos_, n, word) != 0) return false;
    pos_ += n;
    return true;
  }

  json value() {
    skip_ws();
    if (pos_ >= s_.size()) fail("unexpected end of input");
    const char c = s_[pos_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return json(string());
    if (literal("true")) return json(true);
    if (literal("false")) return json(false);
    if (literal("null")) return json(nullptr);
    return number();
  }

  json object() {
    expect('{');
    json obj = json::object();
    if (eat('}')) return obj;
    do {
      skip_ws();
      if (pos_ >= s_.size() || s_[pos_] != '"') fail("expected object key");
      std::string key = string();
      expect(':');
      obj[key] = value();
    } while (eat(','));
    expect('}');
    return obj;
  }

  json array() {
    expect('[');
    json arr = json::array();
    if (eat(']')) return arr;
    do arr.push_back(value());
    while (eat(','));
    expect(']');
    return arr;
  }

  static void put_utf8(std::string& out, unsigned cp) {
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
    if (pos_ + 4 > s_.size()) fail("bad \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      const char h = s_[pos_++];
      v <<= 4;
      if (h >= '0' && h <= '9') v |= static_cast<unsigned>(h - '0');
      else if (h >= 'a' && h <= 'f') v |= static_cast<unsigned>(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') v |= static_cast<unsigned>(h - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }

  std::string string() {
    ++pos_;  // opening quote
    std::string out;
    while (true) {
      if (pos_ >= s_.size()) fail("unterminated string");
      const char c = s_[pos_++];
      if (c == '"') break;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (pos_ >= s_.size()) fail("unterminated escape");
      const char e = s_[pos_++];
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
          if (cp >= 0xD800 && cp < 0xDC00 && pos_ + 6 <= s_.size() && s_[pos_] == '\\' &&
              s_[pos_ + 1] == 'u') {
            pos_ += 2;
            const unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }

  json number() {
    const std::size_t start = pos_;
    if (pos_ < s_.size() && s_[pos_] == '-') ++pos_;
    bool is_float = false;
    while (pos_ < s_.size()) {
      const char c = s_[pos_];
      if (c >= '0' && c <= '9') { ++pos_; continue; }
      if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') { is_float = true; ++pos_; continue; }
      break;
    }
    if (pos_ == start) fail("unexpected character");
    const std::string tok = s_.substr(start, pos_ - start);
    if (!is_float) {
      if (tok[0] == '-') {
        std::int64_t v = 0;
        auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
        if (r.ec == std::errc()) return json(static_cast<long long>(v));
      } else {
        std::uint64_t v = 0;
        auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
        if (r.ec == std::errc()) return json(static_cast<unsigned long long>(v));
      }
    }
    char* end = nullptr;
    const double d = std::strtod(tok.c_str(), &end);
    if (end != tok.c_str() + tok.size()) fail("malformed number");
    return json(d);
  }

  const std::string& s_;
  std::size_t pos_ = 0;
};

void escape_into(std::string& out, const std::string& s) {
  out += '"';
  for (const char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", static_cast<unsigned char>(c));
          out += buf;
        } else {
          out += c;
        }
    }
  }
  out += '"';
}

}  // namespace

json json::parse(const std::string& text) { return Parser(text).document(); }

std::size_t json::size() const {
  if (type_ == Type::Array) return a_->size();
  if (type_ == Type::Object) return o_->size();
  return type_ == Type::Null ? 0 : 1;
}

bool json::contains(const std::string& key) const {
  return type_ == Type::Object && o_->count(key) > 0;
}

const json& json::at(const std::string& key) const {
  if (type_ != Type::Object) throw ValidationError("json", "at('" + key + "') on a non-object");
  auto it = o_->find(key);
  if (it == o_->end()) throw ValidationError("json", "key '" + key + "' not found");
  return it->second;
}

const json& json::at(std::size_t i) const {
  if (type_ != Type::Array || i >= a_->size())
    throw ValidationError("json", "array index " + std::to_string(i) + " out of range");
  return (*a_)[i];
}

json& json::operator[](const std::string& key) {
  if (type_ == Type::Null) *this = object();
  if (type_ != Type::Object) throw ValidationError("json", "operator[] on a non-object");
  return (*o_)[key];
}

void json::push_back(json v) {
  if (type_ == Type::Null) *this = array();
  if (type_ != Type::Array) throw ValidationError("json", "push_back on a non-array");
  a_->push_back(std::move(v));
}

const json::array_t& json::items() const {
  static const array_t kEmpty;
  if (type_ == Type::Array) return *a_;
  if (type_ == Type::Null) return kEmpty;
  throw ValidationError("json", "not an array");
}

const json::object_t& json::fields() const {
  static const object_t kEmpty;
  if (type_ == Type::Object) return *o_;
  if (type_ == Type::Null) return kEmpty;
  throw ValidationError("json", "not an object");
}

bool json::as_bool() const {
  if (type_ != Type::Boolean) throw ValidationError("json", "value is not a boolean");
  return b_;
}

std::string json::as_string() const {
  if (type_ != Type::String) throw ValidationError("json", "value is not a string");
  return s_;
}

double json::as_double() const {
  switch (type_) {
    case Type::Integer: return static_cast<double>(i_);
    case Type::Unsigned: return static_cast<double>(u_);
    case Type::Float: return d_;
    default: throw ValidationError("json", "value is not a number");
  }
}

std::int64_t json::as_i64() const {
  switch (type_) {
    case Type::Integer: return i_;
    case Type::Unsigned: return static_cast<std::int64_t>(u_);
    case Type::Float: return static_cast<std::int64_t>(d_);
    case Type::Boolean: return b_ ? 1 : 0;
    default: throw ValidationError("json", "value is not a number");
  }
}

std::uint64_t json::as_u64() const {
  switch (type_) {
    case Type::Integer: return static_cast<std::uint64_t>(i_);
    case Type::Unsigned: return u_;
    case Type::Float: return static_cast<std::uint64_t>(d_);
    case Type::Boolean: return b_ ? 1 : 0;
    default: throw ValidationError("json", "value is not a number");
  }
}

void json::dump_to(std::string& out, int indent, int depth) const {
  const auto newline = [&](int d) {
    if (indent < 0) return;
    out += '\n';
    out.append(static_cast<std::size_t>(indent * d), ' ');
  };
  switch (type_) {
    case Type::Null: out += "null"; return;
    case Type::Boolean: out += b_ ? "true" : "false"; return;
    case Type::Integer: out += std::to_string(i_); return;
    case Type::Unsigned: out += std::to_string(u_); return;
    case Type::Float: {
      if (!std::isfinite(d_)) { out += "null"; return; }
      char buf[64];
      auto r = std::to_chars(buf, buf + sizeof buf, d_);
      std::string t(buf, r.ptr);
      if (t.find_first_of(".eE") == std::string::npos) t += ".0";
      out += t;
      return;
    }
    case Type::String: escape_into(out, s_); return;
    case Type::Array: {
      out += '[';
      if (a_->empty()) { out += ']'; return; }
      for (std::size_t i = 0; i < a_->size(); ++i) {
        if (i) out += ',';
        newline(depth + 1);
        (*a_)[i].dump_to(out, indent, depth + 1);
      }
      newline(depth);
      out += ']';
      return;
    }
    case Type::Object: {
      out += '{';
      if (o_->empty()) { out += '}'; return; }
      bool first = true;
      for (const auto& [k, v] : *o_) {
        if (!first) out += ',';
        first = false;
        newline(depth + 1);
        escape_into(out, k);
        out += indent < 0 ? ":" : ": ";
        v.dump_to(out, indent, depth + 1);
      }
      newline(depth);
      out += '}';
      return;
    }
  }
}

std::string json::dump(int indent) const {
  std::string out;
  dump_to(out, indent, 0);
  return out;
}

bool json::operator==(const json& o) const {
  if (is_number() && o.is_number()) {
    if (type_ == Type::Float || o.type_ == Type::Float) return as_double() == o.as_double();
    return as_i64() == o.as_i64();
  }
  if (type_ != o.type_) return false;
  switch (type_) {
    case Type::Null: return true;
    case Type::Boolean: return b_ == o.b_;
    case Type::String: return s_ == o.s_;
    case Type::Array: return *a_ == *o.a_;
    case Type::Object: return *o_ == *o.o_;
    default: return false;
  }
}

}  // namespace microslice
