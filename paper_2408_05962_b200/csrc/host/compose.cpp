// CollectiveProgram: registration, validation and the hiercoll-program-v1
// text (reference behaviour: proj/src/composition.cpp:87-441).
//
// Registration keeps, per (rank, buffer), the disjoint spans the open
// step already writes, so the eager write-write check is one binary
// search. validate() re-derives everything from the registered steps: it
// turns each step into read/write accesses, sorts the writes of every
// (rank, buffer) by offset and sweeps them once for write-write overlap,
// answers read-write overlap from the same sorted lists, and keeps a
// union of everything written by earlier steps to catch reads of data
// nobody produced.
#include <algorithm>
#include <cstdio>

#include "hiccl/program.hpp"
#include "planning.hpp"

namespace hiccl {

// ---------------------------------------------------------------- vocabulary

std::string to_string(ReduceOp op) { return op == ReduceOp::max ? "max" : "sum"; }

ReduceOp reduce_op_from_string(const std::string& s) {
  if (s == "sum" || s == "max") return s == "sum" ? ReduceOp::sum : ReduceOp::max;
  throw Error(ErrorCode::ParseError, "reduce op must be sum or max, got '" + s + "'");
}

std::string to_string(PrimitiveKind k) {
  return k == PrimitiveKind::reduction ? "reduction" : "multicast";
}

std::string to_string(ErrorCode code) {
  // the reference's names in the reference's order (types.hpp:50-64),
  // then the two the device path adds
  static const std::vector<std::string> names = {
      "EmptyLeafSet", "RankOutOfRange", "EmptyStep", "WriteWriteRace", "ReadWriteRace",
      "BadBufferRef", "UnsupportedFormulation", "InvalidMachine", "InvalidConfig",
      "UninitializedRead", "DependencyViolation", "NoInterNodeBound", "ParseError",
      "CudaError", "Timeout"};
  const size_t i = (size_t)code;
  return i < names.size() ? names[i] : "UnknownError";
}

// The reference hashes with offset basis 1469598103934665603, one digit
// short of FNV's published 14695981039346656037 (composition.cpp:433,
// factorize.cpp:37); program ids and staging-buffer names depend on it.
uint64_t fnv1a64(const std::string& s) {
  constexpr uint64_t kBasis = 1469598103934665603ULL, kPrime = 1099511628211ULL;
  uint64_t h = kBasis;
  for (const char c : s) {
    h ^= (unsigned char)c;
    h *= kPrime;
  }
  return h;
}

std::string hex16(uint64_t v) {
  static const char digits[] = "0123456789abcdef";
  std::string s(16, '0');
  for (int i = 15; i >= 0; --i, v >>= 4) s[i] = digits[v & 15];
  return s;
}

// ---------------------------------------------------------------- accesses

std::vector<RankRange> primitive_writes(const Primitive& p) {
  if (p.kind == PrimitiveKind::reduction) return {{p.root, p.recv}};
  std::vector<RankRange> out;
  out.reserve(p.leaves.size() + 1);
  for (Rank r : p.leaves) out.push_back({r, p.recv});
  if (p.root_participates) out.push_back({p.root, p.recv});
  return out;
}

std::vector<RankRange> primitive_reads(const Primitive& p) {
  if (p.kind == PrimitiveKind::multicast) return {{p.root, p.send}};
  std::vector<RankRange> out;
  out.reserve(p.leaves.size() + 1);
  for (Rank r : p.leaves) out.push_back({r, p.send});
  if (p.root_participates) out.push_back({p.root, p.send});
  return out;
}

namespace {

std::string span_text(const BufferRef& r) {
  return "'" + r.buffer + "'[" + std::to_string(r.offset) + ", " + std::to_string(r.end()) + ")";
}

// Why `r` does not name a valid range of a declared buffer ("" if it does).
std::string range_problem(const std::map<std::string, BufferDecl>& decls, const BufferRef& r) {
  const auto it = decls.find(r.buffer);
  if (it == decls.end()) return "buffer '" + r.buffer + "' was never declared";
  if (r.offset < 0 || r.count <= 0 || r.end() > it->second.length)
    return span_text(r) + " is not inside a buffer of " + std::to_string(it->second.length) +
           " elements";
  return "";
}

// Union of half-open spans, kept merged and sorted.
class SpanUnion {
 public:
  void insert(int64_t lo, int64_t hi) {
    auto first = std::lower_bound(spans_.begin(), spans_.end(), lo,
                                  [](const auto& s, int64_t x) { return s.second < x; });
    auto last = first;
    while (last != spans_.end() && last->first <= hi) {
      lo = std::min(lo, last->first);
      hi = std::max(hi, last->second);
      ++last;
    }
    first = spans_.erase(first, last);
    spans_.insert(first, {lo, hi});
  }
  bool contains(int64_t lo, int64_t hi) const {
    auto it = std::upper_bound(spans_.begin(), spans_.end(), lo,
                               [](int64_t x, const auto& s) { return x < s.first; });
    return it != spans_.begin() && std::prev(it)->second >= hi;
  }

 private:
  std::vector<std::pair<int64_t, int64_t>> spans_;
};

struct Touch {
  RankRange at;
  int prim;
};

}  // namespace

// ---------------------------------------------------------------- registration

CollectiveProgram::CollectiveProgram(int world_size) : world_size_(world_size) {
  if (world_size < 1)
    throw Error(ErrorCode::RankOutOfRange, "a program needs at least one rank, got " +
                                               std::to_string(world_size));
  steps_.resize(1);
}

CollectiveProgram& CollectiveProgram::declare_buffer(const std::string& id, int64_t length,
                                                     bool input, bool internal) {
  if (length < 1)
    throw Error(ErrorCode::BadBufferRef, "buffer '" + id + "' declared with " +
                                             std::to_string(length) + " elements");
  buffers_[id] = BufferDecl{length, input, internal};
  return *this;
}

void CollectiveProgram::admit(Primitive prim) {
  for (const BufferRef* r : {&prim.send, &prim.recv}) {
    const std::string why = range_problem(buffers_, *r);
    if (!why.empty()) throw Error(ErrorCode::BadBufferRef, why);
  }
  if (prim.send.count != prim.recv.count)
    throw Error(ErrorCode::BadBufferRef, "send " + span_text(prim.send) + " and recv " +
                                             span_text(prim.recv) + " differ in length");
  auto in_world = [&](Rank r) { return r >= 0 && r < world_size_; };
  if (!in_world(prim.root))
    throw Error(ErrorCode::RankOutOfRange, "root rank " + std::to_string(prim.root) +
                                               " outside a world of " +
                                               std::to_string(world_size_));
  for (Rank r : prim.leaves)
    if (!in_world(r))
      throw Error(ErrorCode::RankOutOfRange, "leaf rank " + std::to_string(r) +
                                                 " outside a world of " +
                                                 std::to_string(world_size_));

  // normalize: sorted unique leaves; a root among them participates
  std::sort(prim.leaves.begin(), prim.leaves.end());
  prim.leaves.erase(std::unique(prim.leaves.begin(), prim.leaves.end()), prim.leaves.end());
  const auto self = std::lower_bound(prim.leaves.begin(), prim.leaves.end(), prim.root);
  if (self != prim.leaves.end() && *self == prim.root) {
    prim.root_participates = true;
    prim.leaves.erase(self);
  }

  const auto writes = primitive_writes(prim);
  auto first_after = [](const std::vector<std::pair<int64_t, int64_t>>& v, int64_t lo) {
    return std::upper_bound(v.begin(), v.end(), lo,
                            [](int64_t x, const auto& s) { return x < s.second; });
  };
  for (const RankRange& w : writes) {
    const auto it = claimed_.find({w.rank, w.range.buffer});
    if (it == claimed_.end()) continue;
    const auto hit = first_after(it->second, w.range.offset);  // first span ending past lo
    if (hit != it->second.end() && hit->first < w.range.end())
      throw Error(ErrorCode::WriteWriteRace,
                  "rank " + std::to_string(w.rank) + " " + span_text(w.range) +
                      " is already written in this step");
  }
  for (const RankRange& w : writes) {
    auto& spans = claimed_[{w.rank, w.range.buffer}];
    spans.insert(first_after(spans, w.range.offset), {w.range.offset, w.range.end()});
  }
  steps_.back().push_back(std::move(prim));
}

CollectiveProgram& CollectiveProgram::append_primitive(Primitive prim) {
  admit(std::move(prim));
  return *this;
}

CollectiveProgram& CollectiveProgram::add_multicast(const BufferRef& send, const BufferRef& recv,
                                                    Rank root, std::vector<Rank> leaves) {
  if (leaves.empty()) throw Error(ErrorCode::EmptyLeafSet, "a multicast needs receivers");
  Primitive p;
  p.kind = PrimitiveKind::multicast;
  p.root = root;
  p.leaves = std::move(leaves);
  p.send = send;
  p.recv = recv;
  return append_primitive(std::move(p));
}

CollectiveProgram& CollectiveProgram::add_reduction(const BufferRef& send, const BufferRef& recv,
                                                    std::vector<Rank> leaves, Rank root,
                                                    ReduceOp op) {
  if (leaves.empty()) throw Error(ErrorCode::EmptyLeafSet, "a reduction needs contributors");
  Primitive p;
  p.kind = PrimitiveKind::reduction;
  p.root = root;
  p.leaves = std::move(leaves);
  p.send = send;
  p.recv = recv;
  p.op = op;
  return append_primitive(std::move(p));
}

CollectiveProgram& CollectiveProgram::add_fence() {
  if (steps_.back().empty())
    throw Error(ErrorCode::EmptyStep, "nothing registered since the previous fence");
  steps_.emplace_back();
  claimed_.clear();
  return *this;
}

size_t CollectiveProgram::primitive_count() const {
  size_t n = 0;
  for (const auto& step : steps_) n += step.size();
  return n;
}

// ---------------------------------------------------------------- validation

std::vector<Violation> CollectiveProgram::validate() const {
  std::vector<Violation> found;
  auto note = [&found](ErrorCode code, int step, int prim, Rank rank, const BufferRef& at,
                       std::string why) {
    Violation v;
    v.code = code;
    v.message = std::move(why);
    v.step = step;
    v.primitive = prim;
    v.rank = rank;
    v.buffer = at.buffer;
    v.lo = at.offset;
    v.hi = at.end();
    found.push_back(std::move(v));
  };

  const int last = (int)steps_.size() - 1;
  if (last > 0 && steps_[last].empty())
    note(ErrorCode::EmptyStep, last, -1, -1, BufferRef{}, "the program ends with a fence");

  std::map<std::pair<Rank, std::string>, SpanUnion> produced;  // by earlier steps
  for (int si = 0; si <= last; ++si) {
    std::vector<Touch> reads;
    // (rank, buffer) -> the step's writes, sorted by offset below
    std::map<std::pair<Rank, std::string>, std::vector<Touch>> writes;
    for (int pi = 0; pi < (int)steps_[si].size(); ++pi) {
      const Primitive& p = steps_[si][pi];
      const size_t before = found.size();
      std::vector<Rank> ranks{p.root};
      ranks.insert(ranks.end(), p.leaves.begin(), p.leaves.end());
      for (Rank r : ranks)
        if (r < 0 || r >= world_size_)
          note(ErrorCode::RankOutOfRange, si, pi, r, p.recv,
               "rank " + std::to_string(r) + " outside the world");
      for (const BufferRef* ref : {&p.send, &p.recv}) {
        const std::string why = range_problem(buffers_, *ref);
        if (!why.empty()) note(ErrorCode::BadBufferRef, si, pi, p.root, *ref, why);
      }
      if (found.size() != before) continue;  // nothing sound to sweep
      for (const RankRange& a : primitive_writes(p))
        writes[{a.rank, a.range.buffer}].push_back({a, pi});
      for (const RankRange& a : primitive_reads(p)) reads.push_back({a, pi});
    }

    for (auto& [where, list] : writes) {
      std::stable_sort(list.begin(), list.end(), [](const Touch& a, const Touch& b) {
        return a.at.range.offset < b.at.range.offset;
      });
      const Touch* widest = nullptr;  // the write reaching furthest so far
      for (const Touch& w : list) {
        if (widest && widest->prim != w.prim && widest->at.range.end() > w.at.range.offset)
          note(ErrorCode::WriteWriteRace, si, widest->prim, widest->at.rank, widest->at.range,
               "also written by primitive " + std::to_string(w.prim) + " of the same step");
        if (!widest || w.at.range.end() > widest->at.range.end()) widest = &w;
      }
    }
    for (const Touch& r : reads) {
      const auto it = writes.find({r.at.rank, r.at.range.buffer});
      if (it == writes.end()) continue;
      for (const Touch& w : it->second) {
        if (w.at.range.offset >= r.at.range.end()) break;
        if (w.prim == r.prim || !w.at.range.overlaps(r.at.range)) continue;
        note(ErrorCode::ReadWriteRace, si, r.prim, r.at.rank, r.at.range,
             "read while primitive " + std::to_string(w.prim) + " of the same step writes it");
        break;
      }
    }
    for (const Touch& r : reads) {
      if (buffers_.at(r.at.range.buffer).input) continue;
      const auto it = produced.find({r.at.rank, r.at.range.buffer});
      if (it == produced.end() || !it->second.contains(r.at.range.offset, r.at.range.end()))
        note(ErrorCode::UninitializedRead, si, r.prim, r.at.rank, r.at.range,
             "no earlier step writes all of " + span_text(r.at.range));
    }
    for (const auto& [where, list] : writes)
      for (const Touch& w : list) produced[where].insert(w.at.range.offset, w.at.range.end());
  }
  return found;
}

// ---------------------------------------------------------------- persistence

namespace {

json::Value range_to_json(const BufferRef& r) {
  json::Value v = json::Value::Obj();
  v.set("buffer", json::Value::Str(r.buffer));
  v.set("offset", json::Value::Int(r.offset));
  v.set("count", json::Value::Int(r.count));
  return v;
}

BufferRef range_from_json(const json::Value& v) {
  BufferRef r;
  r.buffer = v.at("buffer").as_str();
  r.offset = v.at("offset").as_int();
  r.count = v.at("count").as_int();
  return r;
}

}  // namespace

json::Value buffers_to_json(const std::map<std::string, BufferDecl>& decls) {
  json::Value arr = json::Value::Arr();
  for (const auto& [name, d] : decls) {
    json::Value b = json::Value::Obj();
    b.set("id", json::Value::Str(name));
    b.set("length", json::Value::Int(d.length));
    b.set("input", json::Value::Bool(d.input));
    b.set("internal", json::Value::Bool(d.internal));
    arr.push(std::move(b));
  }
  return arr;
}

std::string CollectiveProgram::serialize() const {
  // key order is part of the format (composition.cpp:363-394)
  json::Value doc = json::Value::Obj();
  doc.set("format", json::Value::Str("hiercoll-program-v1"));
  doc.set("world_size", json::Value::Int(world_size_));
  doc.set("buffers", buffers_to_json(buffers_));
  json::Value steps = json::Value::Arr();
  for (const auto& step : steps_) {
    json::Value prims = json::Value::Arr();
    for (const Primitive& p : step) {
      json::Value o = json::Value::Obj();
      o.set("kind", json::Value::Str(to_string(p.kind)));
      o.set("root", json::Value::Int(p.root));
      o.set("leaves", json::Value::IntArr(p.leaves));
      o.set("root_participates", json::Value::Bool(p.root_participates));
      o.set("send", range_to_json(p.send));
      o.set("recv", range_to_json(p.recv));
      if (p.kind == PrimitiveKind::reduction) o.set("op", json::Value::Str(to_string(p.op)));
      if (p.stripe) o.set("stripe", json::Value::Int(p.stripe));
      prims.push(std::move(o));
    }
    steps.push(std::move(prims));
  }
  doc.set("steps", std::move(steps));
  return json::dump(doc) + "\n";
}

CollectiveProgram CollectiveProgram::deserialize(const std::string& text) {
  const json::Value doc = json::parse(text);
  if (doc.type != json::Value::Type::object ||
      doc.str_or("format", "") != "hiercoll-program-v1")
    throw Error(ErrorCode::ParseError, "expected a hiercoll-program-v1 document");
  CollectiveProgram prog((int)doc.at("world_size").as_int());
  for (const auto& b : doc.at("buffers").arr)
    prog.declare_buffer(b.at("id").as_str(), b.at("length").as_int(),
                        b.bool_or("input", false), b.bool_or("internal", false));
  const auto& steps = doc.at("steps").arr;
  for (size_t si = 0; si < steps.size(); ++si) {
    if (si > 0) prog.add_fence();
    for (const auto& o : steps[si].arr) {
      Primitive p;
      p.kind = o.at("kind").as_str() == "reduction" ? PrimitiveKind::reduction
                                                    : PrimitiveKind::multicast;
      p.root = (Rank)o.at("root").as_int();
      p.leaves = o.at("leaves").as_int_vec<Rank>();
      p.root_participates = o.bool_or("root_participates", false);
      p.send = range_from_json(o.at("send"));
      p.recv = range_from_json(o.at("recv"));
      if (o.has("op")) p.op = reduce_op_from_string(o.at("op").as_str());
      p.stripe = (int)o.int_or("stripe", 0);
      prog.append_primitive(std::move(p));
    }
  }
  return prog;
}

std::string CollectiveProgram::id() const { return hex16(fnv1a64(serialize())); }

}  // namespace hiccl
