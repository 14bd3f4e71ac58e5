#include "json.hpp"

#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace gc3 {
namespace json {
namespace {

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}

  bool run(Value& out, std::string& err) {
    skip_ws();
    if (!value(out, 0)) {
      err = err_;
      return false;
    }
    skip_ws();
    if (p_ != t_.size()) {
      fail("unexpected trailing characters");
      err = err_;
      return false;
    }
    return true;
  }

 private:
  const std::string& t_;
  size_t p_ = 0;
  std::string err_;

  bool fail(const char* what) {
    if (err_.empty()) {
      size_t line = 1, col = 1;
      for (size_t k = 0; k < p_ && k < t_.size(); ++k) {
        if (t_[k] == '\n') { ++line; col = 1; } else { ++col; }
      }
      err_ = "parse error at line " + std::to_string(line) + ", column " + std::to_string(col) + ": " + what;
    }
    return false;
  }
  void skip_ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool literal(const char* word) {
    const size_t n = std::strlen(word);
    if (t_.compare(p_, n, word) != 0) return fail("invalid literal");
    p_ += n;
    return true;
  }

  bool value(Value& v, int depth) {
    if (depth > 512) return fail("nesting too deep");
    if (p_ >= t_.size()) return fail("unexpected end of input");
    const char c = t_[p_];
    switch (c) {
      case '{': return object(v, depth);
      case '[': return array(v, depth);
      case '"': v.kind = Kind::string; return string(v.s);
      case 't': v.kind = Kind::boolean; v.b = true; return literal("true");
      case 'f': v.kind = Kind::boolean; v.b = false; return literal("false");
      case 'n': v.kind = Kind::null; return literal("null");
      default:
        if (c == '-' || (c >= '0' && c <= '9')) return number(v);
        return fail("invalid literal");
    }
  }

  bool object(Value& v, int depth) {
    v.kind = Kind::object;
    ++p_;
    skip_ws();
    if (p_ < t_.size() && t_[p_] == '}') { ++p_; return true; }
    for (;;) {
      skip_ws();
      if (p_ >= t_.size() || t_[p_] != '"') return fail("expected string literal (object key)");
      std::string key;
      if (!string(key)) return false;
      skip_ws();
      if (p_ >= t_.size() || t_[p_] != ':') return fail("expected ':'");
      ++p_;
      skip_ws();
      Value child;
      if (!value(child, depth + 1)) return false;
      v.o[key] = std::move(child);  // repeated key: last one wins (nlohmann behaviour)
      skip_ws();
      if (p_ < t_.size() && t_[p_] == ',') { ++p_; continue; }
      if (p_ < t_.size() && t_[p_] == '}') { ++p_; return true; }
      return fail("expected ',' or '}'");
    }
  }

  bool array(Value& v, int depth) {
    v.kind = Kind::array;
    ++p_;
    skip_ws();
    if (p_ < t_.size() && t_[p_] == ']') { ++p_; return true; }
    for (;;) {
      skip_ws();
      Value child;
      if (!value(child, depth + 1)) return false;
      v.a.push_back(std::move(child));
      skip_ws();
      if (p_ < t_.size() && t_[p_] == ',') { ++p_; continue; }
      if (p_ < t_.size() && t_[p_] == ']') { ++p_; return true; }
      return fail("expected ',' or ']'");
    }
  }

  static void put_utf8(std::string& s, uint32_t cp) {
    if (cp < 0x80) s += static_cast<char>(cp);
    else if (cp < 0x800) { s += static_cast<char>(0xC0 | (cp >> 6)); s += static_cast<char>(0x80 | (cp & 0x3F)); }
    else if (cp < 0x10000) {
      s += static_cast<char>(0xE0 | (cp >> 12));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      s += static_cast<char>(0xF0 | (cp >> 18));
      s += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  bool hex4(uint32_t& out) {
    if (p_ + 4 > t_.size()) return fail("incomplete \\u escape");
    out = 0;
    for (int k = 0; k < 4; ++k) {
      const char h = t_[p_++];
      out <<= 4;
      if (h >= '0' && h <= '9') out |= h - '0';
      else if (h >= 'a' && h <= 'f') out |= h - 'a' + 10;
      else if (h >= 'A' && h <= 'F') out |= h - 'A' + 10;
      else return fail("invalid \\u escape");
    }
    return true;
  }
  bool string(std::string& s) {
    ++p_;  // opening quote
    s.clear();
    for (;;) {
      if (p_ >= t_.size()) return fail("missing closing quote");
      const unsigned char c = static_cast<unsigned char>(t_[p_++]);
      if (c == '"') return true;
      if (c < 0x20) return fail("control character in string");
      if (c != '\\') { s += static_cast<char>(c); continue; }
      if (p_ >= t_.size()) return fail("incomplete escape");
      const char e = t_[p_++];
      switch (e) {
        case '"': s += '"'; break;
        case '\\': s += '\\'; break;
        case '/': s += '/'; break;
        case 'b': s += '\b'; break;
        case 'f': s += '\f'; break;
        case 'n': s += '\n'; break;
        case 'r': s += '\r'; break;
        case 't': s += '\t'; break;
        case 'u': {
          uint32_t cp;
          if (!hex4(cp)) return false;
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            uint32_t lo;
            if (p_ + 2 > t_.size() || t_[p_] != '\\' || t_[p_ + 1] != 'u') return fail("unpaired surrogate");
            p_ += 2;
            if (!hex4(lo)) return false;
            if (lo < 0xDC00 || lo > 0xDFFF) return fail("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            return fail("unpaired surrogate");
          }
          put_utf8(s, cp);
          break;
        }
        default: return fail("invalid escape");
      }
    }
  }

  bool number(Value& v) {
    const size_t start = p_;
    bool neg = false, is_float = false;
    if (t_[p_] == '-') { neg = true; ++p_; }
    if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) return fail("invalid number");
    if (t_[p_] == '0') {
      ++p_;
      if (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') return fail("invalid number: leading zero");
    } else {
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    if (p_ < t_.size() && t_[p_] == '.') {
      is_float = true;
      ++p_;
      if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) return fail("invalid number");
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      is_float = true;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) return fail("invalid number");
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    const std::string lit = t_.substr(start, p_ - start);
    if (!is_float) {
      errno = 0;
      char* end = nullptr;
      if (neg) {
        const long long x = std::strtoll(lit.c_str(), &end, 10);
        if (errno == 0) { v.kind = Kind::integer; v.i = x; return true; }
      } else {
        const unsigned long long x = std::strtoull(lit.c_str(), &end, 10);
        if (errno == 0) { v.kind = Kind::unsigned_integer; v.u = x; return true; }
      }
    }
    v.kind = Kind::floating;  // fractions, exponents and 64-bit overflow become floats
    v.d = std::strtod(lit.c_str(), nullptr);
    return true;
  }
};

void dump_string(const std::string& s, std::string& out) {
  out += '"';
  for (const unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          out += buf;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

void dump_value(const Value& v, int indent, int level, std::string& out) {
  const std::string pad(static_cast<size_t>(indent) * (level + 1), ' ');
  const std::string close_pad(static_cast<size_t>(indent) * level, ' ');
  switch (v.kind) {
    case Kind::null: out += "null"; break;
    case Kind::boolean: out += v.b ? "true" : "false"; break;
    case Kind::integer: out += std::to_string(v.i); break;
    case Kind::unsigned_integer: out += std::to_string(v.u); break;
    case Kind::floating: {
      char buf[64];
      std::snprintf(buf, sizeof(buf), "%.17g", v.d);
      out += buf;
      break;
    }
    case Kind::string: dump_string(v.s, out); break;
    case Kind::array:
      if (v.a.empty()) { out += "[]"; break; }
      out += "[\n";
      for (size_t k = 0; k < v.a.size(); ++k) {
        out += pad;
        dump_value(v.a[k], indent, level + 1, out);
        out += k + 1 < v.a.size() ? ",\n" : "\n";
      }
      out += close_pad + "]";
      break;
    case Kind::object: {
      if (v.o.empty()) { out += "{}"; break; }
      out += "{\n";
      size_t k = 0;
      for (const auto& [key, child] : v.o) {
        out += pad;
        dump_string(key, out);
        out += ": ";
        dump_value(child, indent, level + 1, out);
        out += ++k < v.o.size() ? ",\n" : "\n";
      }
      out += close_pad + "}";
      break;
    }
  }
}

}  // namespace

bool parse(const std::string& text, Value& out, std::string& error) {
  Parser p(text);
  out = Value();
  return p.run(out, error);
}

std::string dump(const Value& v, int indent) {
  std::string out;
  dump_value(v, indent, 0, out);
  return out;
}

}  // namespace json
}  // namespace gc3
