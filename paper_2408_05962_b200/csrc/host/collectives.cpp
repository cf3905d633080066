// The eight MPI collectives as compositions (Table 2 of the paper).
//
// Each (collective, formulation) is a small recipe: the buffers it
// declares and a list of lines, each line registering one primitive per
// value of its loop variables, '|' lines being fences. A tiny interpreter
// turns a recipe into a CollectiveProgram. The recipes register the same
// primitives in the same order as the reference's builder
// (proj/src/presets.cpp:89-229) — registration order fixes the primitive
// order inside a step, hence the staging-buffer names and the plan.
#include <vector>

#include "hiccl/presets.hpp"

namespace hiccl {

namespace {

// Ranges, with d the per-rank chunk and p the world size.
enum class Extent : uint8_t {
  all,      // [0, p*d)
  head,     // [0, d)
  chunk_a,  // [a*d, (a+1)*d)
  chunk_b,  // [b*d, (b+1)*d)
};
enum class Who : uint8_t { root, a, b, zero };
enum class Whom : uint8_t { all, all_but_a, all_but_zero, root, b, zero };

struct Slot {
  char buffer;  // 's' sendbuf, 'r' recvbuf, 't' __tmp
  Extent extent;
};

struct Line {
  char what;  // 'M' multicast, 'R' reduction, '|' fence
  int loops;  // 0: once, 1: for a, 2: for a { for b }
  Slot send, recv;
  Who root;
  Whom leaves;
};

constexpr Line kFence{'|', 0, {}, {}, Who::zero, Whom::all};

struct Recipe {
  bool small_send;  // sendbuf holds one chunk (else p chunks)
  bool small_recv;  // recvbuf holds one chunk
  int tmp_chunks;   // internal __tmp: 0 (none), 1 or p (-1) chunks
  std::vector<Line> lines;
};

const Recipe& recipe(CollectiveKind kind, Formulation form) {
  using K = CollectiveKind;
  using F = Formulation;
  static const Recipe scatter{false, true, 0, {
      {'R', 1, {'s', Extent::chunk_a}, {'r', Extent::head}, Who::a, Whom::root}}};
  static const Recipe bcast_single{false, false, 0, {
      {'M', 0, {'s', Extent::all}, {'r', Extent::all}, Who::root, Whom::all}}};
  static const Recipe bcast_multi{false, false, 0, {  // scatter, then all-gather in place
      {'R', 1, {'s', Extent::chunk_a}, {'r', Extent::chunk_a}, Who::a, Whom::root},
      kFence,
      {'M', 1, {'r', Extent::chunk_a}, {'r', Extent::chunk_a}, Who::a, Whom::all_but_a}}};
  static const Recipe gather{true, false, 0, {
      {'M', 1, {'s', Extent::head}, {'r', Extent::chunk_a}, Who::a, Whom::root}}};
  static const Recipe reduce_single{false, false, 0, {
      {'R', 0, {'s', Extent::all}, {'r', Extent::all}, Who::root, Whom::all}}};
  static const Recipe reduce_multi{false, false, 1, {  // reduce-scatter to __tmp, gather
      {'R', 1, {'s', Extent::chunk_a}, {'t', Extent::head}, Who::a, Whom::all},
      kFence,
      {'M', 1, {'t', Extent::head}, {'r', Extent::chunk_a}, Who::a, Whom::root}}};
  static const Recipe all_to_all{false, false, 0, {
      {'M', 2, {'s', Extent::chunk_b}, {'r', Extent::chunk_a}, Who::a, Whom::b}}};
  static const Recipe ag_single{true, false, 0, {
      {'M', 1, {'s', Extent::head}, {'r', Extent::chunk_a}, Who::a, Whom::all}}};
  static const Recipe ag_multi{true, false, 0, {  // gather to 0, broadcast in place
      {'M', 1, {'s', Extent::head}, {'r', Extent::chunk_a}, Who::a, Whom::zero},
      kFence,
      {'M', 0, {'r', Extent::all}, {'r', Extent::all}, Who::zero, Whom::all_but_zero}}};
  static const Recipe rs_single{false, false, 0, {
      {'R', 1, {'s', Extent::chunk_a}, {'r', Extent::chunk_a}, Who::a, Whom::all}}};
  static const Recipe rs_multi{false, false, -1, {  // reduce to 0 in __tmp, scatter
      {'R', 0, {'s', Extent::all}, {'t', Extent::all}, Who::zero, Whom::all},
      kFence,
      {'R', 1, {'t', Extent::chunk_a}, {'r', Extent::chunk_a}, Who::a, Whom::zero}}};
  static const Recipe ar_single{false, false, 0, {
      {'R', 1, {'s', Extent::all}, {'r', Extent::all}, Who::a, Whom::all}}};
  static const Recipe ar_multi{false, false, 0, {  // reduce-scatter, all-gather in place
      {'R', 1, {'s', Extent::chunk_a}, {'r', Extent::chunk_a}, Who::a, Whom::all},
      kFence,
      {'M', 1, {'r', Extent::chunk_a}, {'r', Extent::chunk_a}, Who::a, Whom::all_but_a}}};
  static const Recipe ar_multi_alt{false, false, 0, {  // reduce to 0, broadcast in place
      {'R', 0, {'s', Extent::all}, {'r', Extent::all}, Who::zero, Whom::all},
      kFence,
      {'M', 0, {'r', Extent::all}, {'r', Extent::all}, Who::zero, Whom::all_but_zero}}};

  const bool one = form == F::single;
  switch (kind) {
    case K::scatter: return scatter;
    case K::broadcast: return one ? bcast_single : bcast_multi;
    case K::gather: return gather;
    case K::reduce: return one ? reduce_single : reduce_multi;
    case K::all_to_all: return all_to_all;
    case K::all_gather: return one ? ag_single : ag_multi;
    case K::reduce_scatter: return one ? rs_single : rs_multi;
    case K::all_reduce: return one ? ar_single : form == F::multi ? ar_multi : ar_multi_alt;
  }
  throw Error(ErrorCode::UnsupportedFormulation, "unknown collective");
}

const char* kKindNames[] = {"scatter",    "broadcast",  "gather",         "reduce",
                            "all_to_all", "all_gather", "reduce_scatter", "all_reduce"};

}  // namespace

std::string to_string(CollectiveKind k) { return kKindNames[(int)k]; }

CollectiveKind collective_from_string(const std::string& s) {
  for (int k = 0; k < 8; ++k)
    if (s == kKindNames[k]) return (CollectiveKind)k;
  throw Error(ErrorCode::ParseError, "no collective called '" + s + "'");
}

std::string to_string(Formulation f) {
  static const char* names[] = {"single", "multi", "multi_alt"};
  return names[(int)f];
}

Formulation formulation_from_string(const std::string& s) {
  for (int f = 0; f < 3; ++f)
    if (s == to_string((Formulation)f)) return (Formulation)f;
  throw Error(ErrorCode::ParseError, "no formulation called '" + s + "'");
}

bool is_rooted(CollectiveKind k) { return (int)k <= (int)CollectiveKind::reduce; }

int64_t preset_send_length(const CollectiveSpec& spec, int p) {
  return recipe(spec.kind, Formulation::single).small_send ? spec.count : p * spec.count;
}

int64_t preset_recv_length(const CollectiveSpec& spec, int p) {
  return recipe(spec.kind, Formulation::single).small_recv ? spec.count : p * spec.count;
}

CollectiveProgram build(const CollectiveSpec& spec, int p) {
  if (p < 1) throw Error(ErrorCode::RankOutOfRange, "a collective needs at least one rank");
  if (spec.count < 1) throw Error(ErrorCode::BadBufferRef, "the chunk must hold an element");
  const Rank root = is_rooted(spec.kind) ? spec.root : 0;
  if (root < 0 || root >= p)
    throw Error(ErrorCode::RankOutOfRange, "root " + std::to_string(root) + " outside 0.." +
                                               std::to_string(p - 1));
  Formulation form = spec.formulation;
  if (form == Formulation::multi_alt && spec.kind != CollectiveKind::all_reduce)
    throw Error(ErrorCode::UnsupportedFormulation, "multi_alt composes all_reduce only");
  const bool one_step_only = spec.kind == CollectiveKind::scatter ||
                             spec.kind == CollectiveKind::gather ||
                             spec.kind == CollectiveKind::all_to_all;
  if (form != Formulation::single && one_step_only)
    throw Error(ErrorCode::UnsupportedFormulation,
                to_string(spec.kind) + " has a single-step composition only");
  if (p == 1) form = Formulation::single;  // one rank: no fence to place

  const Recipe& r = recipe(spec.kind, form);
  const int64_t d = spec.count, pd = (int64_t)p * d;
  CollectiveProgram prog(p);
  prog.declare_buffer("sendbuf", r.small_send ? d : pd, true);
  prog.declare_buffer("recvbuf", r.small_recv ? d : pd);
  if (r.tmp_chunks) prog.declare_buffer("__tmp", r.tmp_chunks > 0 ? d : pd, false, true);

  auto range = [&](const Slot& s, Rank a, Rank b) {
    const char* name = s.buffer == 's' ? "sendbuf" : s.buffer == 'r' ? "recvbuf" : "__tmp";
    switch (s.extent) {
      case Extent::all: return BufferRef{name, 0, pd};
      case Extent::head: return BufferRef{name, 0, d};
      case Extent::chunk_a: return BufferRef{name, a * d, d};
      case Extent::chunk_b: return BufferRef{name, b * d, d};
    }
    return BufferRef{};
  };
  auto rank = [&](Who w, Rank a, Rank b) {
    return w == Who::root ? root : w == Who::a ? a : w == Who::b ? b : 0;
  };
  auto ranks = [&](Whom w, Rank a, Rank b) {
    std::vector<Rank> out;
    for (Rank x = 0; x < p; ++x) {
      const bool in = w == Whom::all || (w == Whom::all_but_a && x != a) ||
                      (w == Whom::all_but_zero && x != 0) || (w == Whom::root && x == root) ||
                      (w == Whom::b && x == b) || (w == Whom::zero && x == 0);
      if (in) out.push_back(x);
    }
    return out;
  };
  for (const Line& line : r.lines) {
    if (line.what == '|') {
      prog.add_fence();
      continue;
    }
    const int na = line.loops >= 1 ? p : 1, nb = line.loops >= 2 ? p : 1;
    for (Rank a = 0; a < na; ++a)
      for (Rank b = 0; b < nb; ++b) {
        const BufferRef send = range(line.send, a, b), recv = range(line.recv, a, b);
        if (line.what == 'M')
          prog.add_multicast(send, recv, rank(line.root, a, b), ranks(line.leaves, a, b));
        else
          prog.add_reduction(send, recv, ranks(line.leaves, a, b), rank(line.root, a, b),
                             spec.op);
      }
  }
  return prog;
}

}  // namespace hiccl
