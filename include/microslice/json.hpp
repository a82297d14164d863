// Minimal JSON document type for the scenario / report wire formats.
// The reference uses nlohmann/json 3.11.3 (an un-vendored third-party header, see
// SURVEY.md §8c); this build carries its own small DOM with the subset of that API the
// microslice formats use (at / contains / value / get<T> / operator[] / dump), so the
// drop-in has no third-party dependency.  Objects keep keys sorted (nlohmann default).
#pragma once

#include <cstdint>
#include <initializer_list>
#include <map>
#include <memory>
#include <string>
#include <type_traits>
#include <vector>

#include "microslice/common.hpp"

namespace microslice {

class json {
 public:
  enum class Type { Null, Boolean, Integer, Unsigned, Float, String, Array, Object };
  using array_t = std::vector<json>;
  using object_t = std::map<std::string, json>;

  json() = default;
  json(const json& o) { *this = o; }
  json(json&&) noexcept = default;
  json& operator=(json&&) noexcept = default;
  json& operator=(const json& o) {  // value semantics: containers are deep-copied
    if (this == &o) return *this;
    type_ = o.type_; b_ = o.b_; i_ = o.i_; u_ = o.u_; d_ = o.d_; s_ = o.s_;
    a_ = o.a_ ? std::make_shared<array_t>(*o.a_) : nullptr;
    o_ = o.o_ ? std::make_shared<object_t>(*o.o_) : nullptr;
    return *this;
  }
  json(std::nullptr_t) {}
  json(bool b) : type_(Type::Boolean), b_(b) {}
  json(int v) : type_(Type::Integer), i_(v) {}
  json(long v) : type_(Type::Integer), i_(v) {}
  json(long long v) : type_(Type::Integer), i_(v) {}
  json(unsigned v) : type_(Type::Unsigned), u_(v) {}
  json(unsigned long v) : type_(Type::Unsigned), u_(v) {}
  json(unsigned long long v) : type_(Type::Unsigned), u_(v) {}
  json(double v) : type_(Type::Float), d_(v) {}
  json(const char* s) : type_(Type::String), s_(s) {}
  json(std::string s) : type_(Type::String), s_(std::move(s)) {}
  template <typename T>
  json(const std::vector<T>& v) : type_(Type::Array), a_(std::make_shared<array_t>()) {
    for (const T& x : v) a_->push_back(json(x));
  }

  static json array() { json j; j.type_ = Type::Array; j.a_ = std::make_shared<array_t>(); return j; }
  static json object() { json j; j.type_ = Type::Object; j.o_ = std::make_shared<object_t>(); return j; }
  static json parse(const std::string& text);

  Type type() const { return type_; }
  bool is_null() const { return type_ == Type::Null; }
  bool is_object() const { return type_ == Type::Object; }
  bool is_array() const { return type_ == Type::Array; }
  bool is_string() const { return type_ == Type::String; }
  bool is_number() const {
    return type_ == Type::Integer || type_ == Type::Unsigned || type_ == Type::Float;
  }
  bool is_boolean() const { return type_ == Type::Boolean; }

  std::size_t size() const;
  bool contains(const std::string& key) const;
  const json& at(const std::string& key) const;
  const json& at(std::size_t i) const;
  json& operator[](const std::string& key);  // promotes null to object
  void push_back(json v);                     // promotes null to array
  const array_t& items() const;               // array elements
  const object_t& fields() const;             // object members
  array_t::const_iterator begin() const { return items().begin(); }
  array_t::const_iterator end() const { return items().end(); }

  template <typename T>
  T get() const {
    if constexpr (std::is_same_v<T, bool>) return as_bool();
    else if constexpr (std::is_same_v<T, std::string>) return as_string();
    else if constexpr (std::is_floating_point_v<T>) return static_cast<T>(as_double());
    else if constexpr (std::is_unsigned_v<T>) return static_cast<T>(as_u64());
    else return static_cast<T>(as_i64());
  }
  template <typename T>
  T value(const std::string& key, T fallback) const {
    return contains(key) ? at(key).get<T>() : fallback;
  }
  std::string value(const std::string& key, const char* fallback) const {
    return contains(key) ? at(key).get<std::string>() : std::string(fallback);
  }

  std::string dump(int indent = -1) const;
  bool operator==(const json& o) const;

 private:
  bool as_bool() const;
  std::string as_string() const;
  double as_double() const;
  std::int64_t as_i64() const;
  std::uint64_t as_u64() const;
  void dump_to(std::string& out, int indent, int depth) const;

  Type type_ = Type::Null;
  bool b_ = false;
  std::int64_t i_ = 0;
  std::uint64_t u_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::shared_ptr<array_t> a_;
  std::shared_ptr<object_t> o_;
};

}  // namespace microslice
