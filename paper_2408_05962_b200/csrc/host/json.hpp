// Minimal JSON value, parser and pretty printer for the plan persistence
// formats (hiercoll-program-v1 / -plan-v1 / -pipelined-v1 / -machine-v1).
//
// The printer reproduces the byte layout the reference produces when it
// is built in this image (nlohmann::ordered_json::dump(2) as vendored by
// cudnn_frontend 3.11.3, whose one local change prints arrays whose first
// element is an integer on one line: "[1,2]"). Keys keep insertion order.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace hiccl::json {

struct Value {
  enum class Type { null, boolean, integer, number, string, array, object };
  Type type = Type::null;
  bool b = false;
  int64_t i = 0;
  double d = 0;
  std::string s;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  Value() = default;
  static Value Int(int64_t v) { Value x; x.type = Type::integer; x.i = v; return x; }
  static Value Num(double v) { Value x; x.type = Type::number; x.d = v; return x; }
  static Value Bool(bool v) { Value x; x.type = Type::boolean; x.b = v; return x; }
  static Value Str(std::string v) { Value x; x.type = Type::string; x.s = std::move(v); return x; }
  static Value Arr() { Value x; x.type = Type::array; return x; }
  static Value Obj() { Value x; x.type = Type::object; return x; }
  template <class T>
  static Value IntArr(const std::vector<T>& v) {
    Value x = Arr();
    for (auto e : v) x.arr.push_back(Int((int64_t)e));
    return x;
  }

  Value& set(const std::string& key, Value v);  // insert or replace
  Value& push(Value v) { arr.push_back(std::move(v)); return arr.back(); }
  bool has(const std::string& key) const;
  const Value& at(const std::string& key) const;  // throws ParseError
  void erase(const std::string& key);

  int64_t as_int() const;
  double as_num() const;
  bool as_bool() const;
  const std::string& as_str() const;
  template <class T>
  std::vector<T> as_int_vec() const {
    std::vector<T> out;
    for (const auto& e : arr) out.push_back((T)e.as_int());
    return out;
  }
  // value-or-default accessors
  int64_t int_or(const std::string& key, int64_t dflt) const;
  bool bool_or(const std::string& key, bool dflt) const;
  std::string str_or(const std::string& key, const std::string& dflt) const;
};

std::string dump(const Value& v);  // indent 2, trailing newline NOT added
Value parse(const std::string& text);  // throws hiccl::Error(ParseError)

}  // namespace hiccl::json
