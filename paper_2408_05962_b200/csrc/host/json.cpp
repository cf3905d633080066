#include "json.hpp"

#include <charconv>
#include <cstdio>

#include "hiccl/types.hpp"

namespace hiccl::json {

Value& Value::set(const std::string& key, Value v) {
  for (auto& kv : obj)
    if (kv.first == key) {
      kv.second = std::move(v);
      return kv.second;
    }
  obj.emplace_back(key, std::move(v));
  return obj.back().second;
}

bool Value::has(const std::string& key) const {
  for (const auto& kv : obj)
    if (kv.first == key) return true;
  return false;
}

const Value& Value::at(const std::string& key) const {
  for (const auto& kv : obj)
    if (kv.first == key) return kv.second;
  throw Error(ErrorCode::ParseError, "missing key '" + key + "'");
}

void Value::erase(const std::string& key) {
  for (auto it = obj.begin(); it != obj.end(); ++it)
    if (it->first == key) {
      obj.erase(it);
      return;
    }
}

int64_t Value::as_int() const {
  if (type == Type::integer) return i;
  if (type == Type::number) return (int64_t)d;
  throw Error(ErrorCode::ParseError, "expected integer");
}
double Value::as_num() const {
  if (type == Type::number) return d;
  if (type == Type::integer) return (double)i;
  throw Error(ErrorCode::ParseError, "expected number");
}
bool Value::as_bool() const {
  if (type != Type::boolean) throw Error(ErrorCode::ParseError, "expected boolean");
  return b;
}
const std::string& Value::as_str() const {
  if (type != Type::string) throw Error(ErrorCode::ParseError, "expected string");
  return s;
}
int64_t Value::int_or(const std::string& key, int64_t dflt) const {
  return has(key) ? at(key).as_int() : dflt;
}
bool Value::bool_or(const std::string& key, bool dflt) const {
  return has(key) ? at(key).as_bool() : dflt;
}
std::string Value::str_or(const std::string& key, const std::string& dflt) const {
  return has(key) ? at(key).as_str() : dflt;
}

namespace {

void escape_into(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof buf, "\\u%04x", c);
          out += buf;
        } else {
          out += (char)c;
        }
    }
  }
  out += '"';
}

void number_into(std::string& out, double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  // nlohmann writes two-digit negative exponents as e-06
  auto e = s.find("e-");
  if (e != std::string::npos && s.size() - (e + 2) == 1) s.insert(e + 2, "0");
  auto ep = s.find("e+");
  if (ep != std::string::npos) {
    s.erase(ep + 1, 1);
    if (s.size() - (ep + 1) == 1) s.insert(ep + 1, "0");
  }
  out += s;
}

void dump_into(std::string& out, const Value& v, int indent) {
  using T = Value::Type;
  switch (v.type) {
    case T::null: out += "null"; return;
    case T::boolean: out += v.b ? "true" : "false"; return;
    case T::integer: out += std::to_string(v.i); return;
    case T::number: number_into(out, v.d); return;
    case T::string: escape_into(out, v.s); return;
    case T::array: {
      if (v.arr.empty()) {
        out += "[]";
        return;
      }
      if (v.arr.front().type == T::integer) {
        out += '[';
        for (size_t k = 0; k < v.arr.size(); ++k) {
          if (k) out += ',';
          dump_into(out, v.arr[k], indent);
        }
        out += ']';
        return;
      }
      out += "[\n";
      for (size_t k = 0; k < v.arr.size(); ++k) {
        out.append(indent + 2, ' ');
        dump_into(out, v.arr[k], indent + 2);
        out += k + 1 < v.arr.size() ? ",\n" : "\n";
      }
      out.append(indent, ' ');
      out += ']';
      return;
    }
    case T::object: {
      if (v.obj.empty()) {
        out += "{}";
        return;
      }
      out += "{\n";
      for (size_t k = 0; k < v.obj.size(); ++k) {
        out.append(indent + 2, ' ');
        escape_into(out, v.obj[k].first);
        out += ": ";
        dump_into(out, v.obj[k].second, indent + 2);
        out += k + 1 < v.obj.size() ? ",\n" : "\n";
      }
      out.append(indent, ' ');
      out += '}';
      return;
    }
  }
}

struct Parser {
  const std::string& t;
  size_t pos = 0;

  [[noreturn]] void fail(const std::string& what) {
    throw Error(ErrorCode::ParseError,
                what + " at offset " + std::to_string(pos));
  }
  void ws() {
    while (pos < t.size() && (t[pos] == ' ' || t[pos] == '\n' ||
                              t[pos] == '\t' || t[pos] == '\r'))
      ++pos;
  }
  bool eat(char c) {
    ws();
    if (pos < t.size() && t[pos] == c) {
      ++pos;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  std::string str() {
    ws();
    if (pos >= t.size() || t[pos] != '"') fail("expected string");
    ++pos;
    std::string s;
    while (pos < t.size() && t[pos] != '"') {
      char c = t[pos++];
      if (c == '\\') {
        if (pos >= t.size()) fail("bad escape");
        char e = t[pos++];
        switch (e) {
          case 'n': s += '\n'; break;
          case 't': s += '\t'; break;
          case 'r': s += '\r'; break;
          case 'b': s += '\b'; break;
          case 'f': s += '\f'; break;
          case 'u': {
            if (pos + 4 > t.size()) fail("bad \\u escape");
            unsigned cp = std::stoul(t.substr(pos, 4), nullptr, 16);
            pos += 4;
            if (cp < 0x80) s += (char)cp;
            else if (cp < 0x800) { s += (char)(0xC0 | (cp >> 6)); s += (char)(0x80 | (cp & 0x3F)); }
            else { s += (char)(0xE0 | (cp >> 12)); s += (char)(0x80 | ((cp >> 6) & 0x3F)); s += (char)(0x80 | (cp & 0x3F)); }
            break;
          }
          default: s += e;
        }
      } else {
        s += c;
      }
    }
    if (pos >= t.size()) fail("unterminated string");
    ++pos;
    return s;
  }
  Value value() {
    ws();
    if (pos >= t.size()) fail("unexpected end");
    char c = t[pos];
    if (c == '{') {
      ++pos;
      Value o = Value::Obj();
      if (eat('}')) return o;
      do {
        std::string k = str();
        expect(':');
        o.obj.emplace_back(std::move(k), value());
      } while (eat(','));
      expect('}');
      return o;
    }
    if (c == '[') {
      ++pos;
      Value a = Value::Arr();
      if (eat(']')) return a;
      do a.arr.push_back(value());
      while (eat(','));
      expect(']');
      return a;
    }
    if (c == '"') return Value::Str(str());
    if (t.compare(pos, 4, "true") == 0) { pos += 4; return Value::Bool(true); }
    if (t.compare(pos, 5, "false") == 0) { pos += 5; return Value::Bool(false); }
    if (t.compare(pos, 4, "null") == 0) { pos += 4; return Value(); }
    size_t start = pos;
    bool is_float = false;
    if (t[pos] == '-' || t[pos] == '+') ++pos;
    while (pos < t.size()) {
      char d = t[pos];
      if (d >= '0' && d <= '9') { ++pos; continue; }
      if (d == '.' || d == 'e' || d == 'E' || d == '-' || d == '+') { is_float = true; ++pos; continue; }
      break;
    }
    if (start == pos) fail("unexpected character");
    std::string num = t.substr(start, pos - start);
    try {
      if (!is_float) return Value::Int(std::stoll(num));
      return Value::Num(std::stod(num));
    } catch (...) {
      fail("bad number '" + num + "'");
    }
  }
};

}  // namespace

std::string dump(const Value& v) {
  std::string out;
  dump_into(out, v, 0);
  return out;
}

Value parse(const std::string& text) {
  Parser p{text};
  Value v = p.value();
  p.ws();
  if (p.pos != text.size()) p.fail("trailing characters");
  return v;
}

}  // namespace hiccl::json
