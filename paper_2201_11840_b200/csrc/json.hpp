// Minimal JSON DOM for the GC3-IR loader.
//
// The reference parses IR files with nlohmann/json (ir.hpp:14, 226-233). This runtime parses
// the fixed IR schema itself but reproduces the nlohmann behaviours the schema
// checks depend on:
//   * numbers: non-negative integer literals are "unsigned", negative ones "integer", anything
//     with a fraction/exponent (or an integer that overflows 64 bits) is "float";
//   * objects keep keys sorted (std::map) and a repeated key keeps its last value;
//   * strict RFC 8259 syntax: no comments, no trailing commas, no leading zeros.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace gc3 {
namespace json {

enum class Kind { null, boolean, integer, unsigned_integer, floating, string, array, object };

struct Value {
  Kind kind = Kind::null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> a;
  std::map<std::string, Value> o;

  bool is_object() const { return kind == Kind::object; }
  bool is_array() const { return kind == Kind::array; }
  bool is_string() const { return kind == Kind::string; }
  bool is_bool() const { return kind == Kind::boolean; }
  bool is_int() const { return kind == Kind::integer || kind == Kind::unsigned_integer; }
  bool is_unsigned() const { return kind == Kind::unsigned_integer; }
  bool contains(const std::string& k) const { return kind == Kind::object && o.count(k) != 0; }
  const Value& at(const std::string& k) const { return o.at(k); }
  // nlohmann get<int64_t>() / get<int>() semantics: plain static_cast of the stored integer
  int64_t as_i64() const { return kind == Kind::unsigned_integer ? static_cast<int64_t>(u) : i; }
  uint64_t as_u64() const { return kind == Kind::unsigned_integer ? u : static_cast<uint64_t>(i); }
};

// Parses `text`; on failure returns false and fills `error` with a one-line description
// (line/column and what was expected).
bool parse(const std::string& text, Value& out, std::string& error);

// Canonical writer with nlohmann `dump(2)` layout: 2-space indent, sorted keys, "key": value,
// empty containers as [] / {}, nlohmann string escaping.
std::string dump(const Value& v, int indent = 2);

}  // namespace json
}  // namespace gc3
