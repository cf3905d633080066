// Canonical order, def-use dependencies and the pipelining transform.
//
// Ordering sorts by an integer key per transfer: buffer names enter as
// their rank among the plan's sorted names, so the key order is the
// reference's tuple order (factorize.cpp:360-365, pipeline.cpp:30-35).
// Dependencies are answered from an interval index per (rank, buffer):
// the writes sorted by start with a running maximum of their ends, so a
// query jumps by binary search to the first write that can still reach
// the queried range instead of scanning from the buffer's start.
#include <algorithm>
#include <array>
#include <map>
#include <numeric>
#include <unordered_map>

#include "planning.hpp"

namespace hiccl {

namespace {

// Sorted distinct buffer names of a transfer list -> ordinal.
class NameOrder {
 public:
  explicit NameOrder(const std::vector<P2PTransfer>& ts) {
    for (const auto& t : ts) {
      names_.push_back(t.src_buffer);
      names_.push_back(t.dst_buffer);
    }
    std::sort(names_.begin(), names_.end());
    names_.erase(std::unique(names_.begin(), names_.end()), names_.end());
    for (size_t i = 0; i < names_.size(); ++i) ordinal_.emplace(names_[i], (int)i);
  }
  int operator()(const std::string& n) const { return ordinal_.at(n); }
  int size() const { return (int)names_.size(); }

 private:
  std::vector<std::string> names_;
  std::unordered_map<std::string, int> ordinal_;
};

using Key = std::array<int64_t, 11>;

Key key_of(const P2PTransfer& t, Clock clock, const NameOrder& name) {
  const int64_t time = clock == Clock::stage ? t.stage : t.slot;
  Key k{time, t.reduce, t.src, t.dst, name(t.dst_buffer), t.dst_offset, name(t.src_buffer),
        t.src_offset, t.count, t.stripe, t.channel};
  if (clock == Clock::slot) k = {time, t.reduce, t.src, t.dst, name(t.dst_buffer), t.dst_offset,
                                 name(t.src_buffer), t.src_offset, t.channel, t.count, t.stripe};
  return k;
}

}  // namespace

void sort_canonical(std::vector<P2PTransfer>& ts, Clock clock) {
  const NameOrder name(ts);
  std::vector<Key> keys(ts.size());
  for (size_t i = 0; i < ts.size(); ++i) keys[i] = key_of(ts[i], clock, name);
  std::vector<size_t> order(ts.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return keys[a] < keys[b]; });
  std::vector<P2PTransfer> sorted;
  sorted.reserve(ts.size());
  for (size_t i : order) sorted.push_back(std::move(ts[i]));
  for (size_t i = 0; i < sorted.size(); ++i) sorted[i].id = (int)i;
  ts = std::move(sorted);
}

void link_dependencies(std::vector<P2PTransfer>& ts, Clock clock,
                       std::vector<FenceBoundary>* fences) {
  struct Write {
    int64_t lo, hi;
    int time, id;
  };
  struct Bucket {
    std::vector<Write> writes;  // by lo
    std::vector<int64_t> reach;  // reach[k] = max hi of writes[0..k]
  };
  const NameOrder name(ts);
  const int nb = std::max(1, name.size());
  auto time_of = [clock](const P2PTransfer& t) { return clock == Clock::stage ? t.stage : t.slot; };
  std::unordered_map<int64_t, Bucket> index;
  auto bucket_id = [nb](Rank r, int buf) { return (int64_t)r * nb + buf; };
  for (const auto& t : ts)
    index[bucket_id(t.dst, name(t.dst_buffer))].writes.push_back(
        {t.dst_offset, t.dst_offset + t.count, time_of(t), t.id});
  for (auto& [id, b] : index) {
    std::stable_sort(b.writes.begin(), b.writes.end(),
                     [](const Write& x, const Write& y) { return x.lo < y.lo; });
    b.reach.resize(b.writes.size());
    int64_t far = INT64_MIN;
    for (size_t k = 0; k < b.writes.size(); ++k) b.reach[k] = far = std::max(far, b.writes[k].hi);
  }

  std::vector<int> deps;
  for (auto& t : ts) {
    deps.clear();
    const int now = time_of(t);
    auto gather = [&](Rank r, const std::string& buf, int64_t lo, int64_t hi) {
      const auto it = index.find(bucket_id(r, name(buf)));
      if (it == index.end()) return;
      const Bucket& b = it->second;
      // first write whose running reach passes lo: nothing before it overlaps
      size_t k = std::upper_bound(b.reach.begin(), b.reach.end(), lo) - b.reach.begin();
      for (; k < b.writes.size() && b.writes[k].lo < hi; ++k) {
        const Write& w = b.writes[k];
        if (w.hi <= lo || w.time >= now || w.id == t.id) continue;
        deps.push_back(w.id);
        if (fences && (w.lo != lo || w.hi != hi))
          for (auto& f : *fences)
            if (f.stage > w.time && f.stage <= now) f.aligned = false;
      }
    };
    gather(t.src, t.src_buffer, t.src_offset, t.src_offset + t.count);
    if (t.reduce) gather(t.dst, t.dst_buffer, t.dst_offset, t.dst_offset + t.count);
    std::sort(deps.begin(), deps.end());
    deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
    t.deps = deps;
  }
}

// The reference's def-use edges are read-after-write only (factorize.cpp:
// 377-414), so a fence is "aligned" — and pipelining overlaps the steps on
// either side — even when a later step overwrites, without reading, a range
// an earlier step writes or reads through different extents. A channel of
// the later step can then land before a channel of the earlier one, and
// the reference's own symbolic oracle rejects the plan (found by
// tests/test_random_programs.py; the presets never compose this). hiccl
// refuses such pipelined plans, as it refuses ring blocks that drop
// members, instead of executing a reordered write.
static void refuse_reordered_writes(const std::vector<P2PTransfer>& ts) {
  struct Access {
    int64_t lo, hi;
    int step, slot, id;
  };
  std::map<std::pair<Rank, std::string>, std::vector<Access>> touched;  // reads and writes
  for (const auto& t : ts) {
    touched[{t.src, t.src_buffer}].push_back(
        {t.src_offset, t.src_offset + t.count, t.step, t.slot, t.id});
    touched[{t.dst, t.dst_buffer}].push_back(
        {t.dst_offset, t.dst_offset + t.count, t.step, t.slot, t.id});
  }
  for (auto& [key, v] : touched)
    std::sort(v.begin(), v.end(), [](const Access& a, const Access& b) { return a.lo < b.lo; });
  for (const auto& t : ts) {
    if (t.reduce) continue;  // reads its destination: a def-use edge orders it
    const auto it = touched.find({t.dst, t.dst_buffer});
    const int64_t lo = t.dst_offset, hi = t.dst_offset + t.count;
    for (const Access& a : it->second) {
      if (a.lo >= hi) break;
      // executed in (slot, id) order (engine.cpp:288-293): a hazard only
      // when the later step's write comes first
      if (a.hi <= lo || a.step >= t.step || a.slot < t.slot || (a.slot == t.slot && a.id < t.id))
        continue;
      throw Error(ErrorCode::InvalidConfig,
                  "pipelining would reorder a write of step " + std::to_string(t.step) +
                      " before an access of step " + std::to_string(a.step) + " to rank " +
                      std::to_string(t.dst) + " '" + t.dst_buffer +
                      "' (the reference orders read-after-write only)");
    }
  }
}

// Pipelining (reference pipeline.cpp:76-132): every transfer is split into
// m balanced channels, channel c running at slot stage + c, so consecutive
// stages overlap. A misaligned fence (a dependency across it between
// different ranges) cannot overlap: it drains, pushing every later stage
// back by m - 1.
PipelinedPlan pipeline(const StagedPlan& plan, int depth) {
  if (depth < 1)
    throw Error(ErrorCode::InvalidConfig, "pipeline depth " + std::to_string(depth) + " < 1");
  PipelinedPlan out;
  out.depth = depth;
  if (depth == 1) {
    out.base = plan;
    for (auto& t : out.base.transfers) {
      t.channel = 0;
      t.slot = t.stage;
    }
    out.slots = plan.num_stages;
    return out;
  }
  std::vector<int> drains;
  for (const auto& f : plan.fences)
    if (!f.aligned) drains.push_back(f.stage);
  std::sort(drains.begin(), drains.end());
  auto delayed = [&](int stage) {
    const int64_t crossed = std::upper_bound(drains.begin(), drains.end(), stage) - drains.begin();
    return stage + (int)crossed * (depth - 1);
  };

  out.base.world_size = plan.world_size;
  out.base.element_size = plan.element_size;
  out.base.stripe = plan.stripe;
  out.base.ring = plan.ring;
  out.base.source_program_id = plan.source_program_id;
  out.base.buffers = plan.buffers;
  out.base.transfers.reserve(plan.transfers.size() * depth);
  for (const auto& t : plan.transfers) {
    const int stage = delayed(t.stage);
    for (int c = 0; c < depth; ++c) {
      const SplitRange part = balanced_split(t.count, depth, c);
      if (part.count == 0) continue;
      P2PTransfer ch = t;
      ch.deps.clear();
      ch.src_offset += part.offset;
      ch.dst_offset += part.offset;
      ch.count = part.count;
      ch.stage = stage;
      ch.channel = c;
      ch.slot = stage + c;
      out.base.transfers.push_back(std::move(ch));
    }
  }
  sort_canonical(out.base.transfers, Clock::slot);
  refuse_reordered_writes(out.base.transfers);
  link_dependencies(out.base.transfers, Clock::slot, nullptr);
  out.base.num_stages = delayed(plan.num_stages - 1) + 1;
  for (const auto& f : plan.fences) out.base.fences.push_back({delayed(f.stage), f.aligned});
  out.slots = out.base.num_stages + depth - 1;
  return out;
}

std::vector<std::vector<int64_t>> comm_matrix(const PipelinedPlan& plan, int slot) {
  if (slot < 0) throw Error(ErrorCode::InvalidConfig, "negative slot " + std::to_string(slot));
  const int p = plan.base.world_size;
  std::vector<std::vector<int64_t>> bytes(p, std::vector<int64_t>(p, 0));
  for (const auto& t : plan.base.transfers)
    if (t.slot == slot) bytes[t.src][t.dst] += t.count * plan.base.element_size;
  return bytes;
}

int64_t StagedPlan::total_bytes() const {
  int64_t n = 0;
  for (const auto& t : transfers) n += t.count;
  return n * element_size;
}

int64_t inter_node_bytes(const StagedPlan& plan, int node_size) {
  int64_t n = 0;
  for (const auto& t : plan.transfers)
    if (t.src / node_size != t.dst / node_size) n += t.count;
  return n * plan.element_size;
}

}  // namespace hiccl
