// Plan -> executor schedule (see schedule.hpp for the rules).
#include "schedule.hpp"

#include <algorithm>
#include <map>
#include <numeric>
#include <random>
#include <set>
#include <tuple>
#include <unordered_map>

namespace hiccl {

namespace {

struct Xfer {
  int id, slot;
  Loc src, dst;
  int64_t count;
  bool reduce;
  ReduceOp op;
};

struct Access {
  int64_t lo, hi;
  int step;
  int exec;
  int item;
  bool write;
};

using Key = std::pair<int, int>;  // (rank, buffer)

int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

bool overlaps(int64_t a, int64_t na, int64_t b, int64_t nb) { return a < b + nb && b < a + na; }

// Deferred accumulator init (push schedules). The reference initializes an
// accumulator with a plain copy and folds into it in a later slot
// (factorize.cpp:323-335 picks the copy; the reduce-into reads the live
// destination). When nothing else touches that range in between, and the
// copy's source is not rewritten meanwhile, the later fold can start from
// the copy's source instead: fold(src, x, ...) is the same sequence of
// folds, with one store instead of a store, a reload and a store — and the
// accumulator is then written once, so it can live where it is read
// (place_internal_buffers).
void fuse_deferred_init(Schedule& S) {
  const int n = (int)S.items.size();
  std::map<Key, std::vector<int>> touch;
  for (int k = 0; k < n; ++k) {
    const WorkItem& w = S.items[k];
    touch[{w.dst.rank, w.dst.buffer}].push_back(k);
    for (const Loc& l : w.srcs) touch[{l.rank, l.buffer}].push_back(k);
  }
  auto reads = [&](const WorkItem& w, const Loc& at, int64_t cnt) {
    for (const Loc& l : w.srcs)
      if (l.rank == at.rank && l.buffer == at.buffer && overlaps(l.offset, w.count, at.offset, cnt)) return true;
    return false;
  };
  auto writes = [&](const WorkItem& w, const Loc& at, int64_t cnt) {
    return w.dst.rank == at.rank && w.dst.buffer == at.buffer && overlaps(w.dst.offset, w.count, at.offset, cnt);
  };
  std::vector<char> dead(n, 0);
  for (int k2 = 0; k2 < n; ++k2) {
    WorkItem& g2 = S.items[k2];
    if (!g2.reads_dst || g2.staging) continue;
    const Loc d = g2.dst;
    int k1 = -1;
    for (int k : touch[{d.rank, d.buffer}]) {  // latest earlier writer of the range
      const WorkItem& w = S.items[k];
      if (k == k2 || dead[k] || w.step >= g2.step || !writes(w, d, g2.count)) continue;
      if (k1 < 0 || w.step > S.items[k1].step) k1 = k;
    }
    if (k1 < 0) continue;
    const WorkItem& g1 = S.items[k1];
    if (g1.reads_dst || g1.srcs.size() != 1 || g1.staging || g1.exec != g2.exec ||
        g1.dst.offset != d.offset || g1.count != g2.count)
      continue;
    bool ok = true;
    for (int k : touch[{d.rank, d.buffer}]) {  // nothing else touches it in between
      const WorkItem& w = S.items[k];
      if (k == k1 || k == k2 || dead[k] || w.step < g1.step || w.step > g2.step) continue;
      if (writes(w, d, g2.count) || reads(w, d, g2.count)) ok = false;
    }
    const Loc src = g1.srcs[0];
    if (src.rank == d.rank && src.buffer == d.buffer) ok = false;
    for (size_t q = 1; q < g2.srcs.size(); ++q)  // g2 must not read the accumulator otherwise
      if (g2.srcs[q].rank == d.rank && g2.srcs[q].buffer == d.buffer &&
          overlaps(g2.srcs[q].offset, g2.count, d.offset, g2.count))
        ok = false;
    for (int k : touch[{src.rank, src.buffer}]) {  // the copy's source unchanged until g2 reads it
      const WorkItem& w = S.items[k];
      if (k == k1 || dead[k] || w.step < g1.step || w.step > g2.step) continue;
      if (writes(w, src, g2.count)) ok = false;
    }
    if (!ok) continue;
    g2.srcs[0] = src;
    g2.reads_dst = false;
    // g2 now reads the copy's source: later candidates must see that access
    touch[{src.rank, src.buffer}].push_back(k2);
    g2.transfer_ids.insert(g2.transfer_ids.begin(), g1.transfer_ids.begin(), g1.transfer_ids.end());
    dead[k1] = 1;
  }
  std::vector<WorkItem> keep;
  for (int k = 0; k < n; ++k)
    if (!dead[k]) keep.push_back(std::move(S.items[k]));
  S.items = std::move(keep);
}

// Copy forwarding (push schedules). An internal range written once (item
// A) and read once, by a plain copy of the same executor at a later step
// (item B: reduce-scatter into __tmp, then gather it to the root), is
// never needed by itself: A stores straight into B's destination and B
// disappears — when nothing touches that destination in between. The
// values and the fold order are A's; the store lands one hop earlier.
void fuse_forward_copy(Schedule& S) {
  const int n = (int)S.items.size();
  std::map<Key, std::vector<int>> touch;
  for (int k = 0; k < n; ++k) {
    const WorkItem& w = S.items[k];
    touch[{w.dst.rank, w.dst.buffer}].push_back(k);
    for (const Loc& l : w.srcs) touch[{l.rank, l.buffer}].push_back(k);
  }
  auto hits = [&](const WorkItem& w, const Loc& at, int64_t cnt, bool& rd, bool& wr) {
    rd = wr = false;
    wr = w.dst.rank == at.rank && w.dst.buffer == at.buffer && overlaps(w.dst.offset, w.count, at.offset, cnt);
    for (const Loc& l : w.srcs)
      rd |= l.rank == at.rank && l.buffer == at.buffer && overlaps(l.offset, w.count, at.offset, cnt);
  };
  std::vector<char> dead(n, 0);
  for (int kb = 0; kb < n; ++kb) {
    const WorkItem& b = S.items[kb];
    if (dead[kb] || b.reads_dst || b.srcs.size() != 1 || b.staging) continue;
    const Loc d = b.srcs[0];
    if (!S.buffer_decls[d.buffer].internal || d.buffer == S.staging_buffer) continue;
    int ka = -1;
    bool ok = true;
    for (int k : touch[{d.rank, d.buffer}]) {  // exactly one writer (A) and one reader (B)
      if (k == kb || dead[k]) continue;
      bool rd, wr;
      hits(S.items[k], d, b.count, rd, wr);
      if (rd || (wr && ka >= 0)) ok = false;
      if (wr) ka = k;
    }
    if (!ok || ka < 0) continue;
    WorkItem& a = S.items[ka];
    if (a.reads_dst || a.staging || a.exec != b.exec || a.step >= b.step || a.dst.offset != d.offset ||
        a.count != b.count)
      continue;
    const Loc e = b.dst;
    for (int k : touch[{e.rank, e.buffer}]) {  // B's destination quiet from A to B
      if (k == kb || dead[k]) continue;
      const WorkItem& w = S.items[k];
      if (w.step < a.step || w.step > b.step) continue;
      bool rd, wr;
      hits(w, e, b.count, rd, wr);
      if (rd || wr) ok = false;
    }
    for (const Loc& l : a.srcs)  // A must not read what it would now write
      if (l.rank == e.rank && l.buffer == e.buffer && overlaps(l.offset, a.count, e.offset, b.count)) ok = false;
    if (!ok) continue;
    a.dst = e;
    // A now writes B's destination: later candidates must see that access
    touch[{e.rank, e.buffer}].push_back(ka);
    a.transfer_ids.insert(a.transfer_ids.end(), b.transfer_ids.begin(), b.transfer_ids.end());
    dead[kb] = 1;
  }
  std::vector<WorkItem> keep;
  for (int k = 0; k < n; ++k)
    if (!dead[k]) keep.push_back(std::move(S.items[k]));
  S.items = std::move(keep);
}

// Internal buffers (accumulators, staging of the reference's plan) are
// declared per rank but live wherever the executor chooses. A buffer whose
// every reader runs on one other executor may move into that executor's
// arena: its readers then load locally and its writers push (remote
// stores) instead of the readers pulling. Whether that pays depends on the
// step it moves the traffic into, so each candidate is kept only if it
// lowers the schedule's link time, sum over steps of the busiest executor
// direction, with pulls at 650 and pushes at 691 GB/s (B200Model). A
// pipelined reduce chain becomes pure push; a reduce-scatter whose
// accumulators are filled by pull-reduces keeps pulling.
void place_internal_buffers(Schedule& S, int element_size) {
  const int E = S.num_execs;
  const int nsteps = (int)S.step_slot.size();
  const double pull_bw = 650e9, push_bw = 691e9;
  auto home_of = [&](const Loc& l) { return S.home[l.rank][l.buffer]; };
  auto link_time = [&]() {
    std::vector<double> eg((size_t)nsteps * E, 0.0), in((size_t)nsteps * E, 0.0);
    for (const WorkItem& w : S.items) {
      const double b = (double)w.count * element_size;
      const size_t row = (size_t)w.step * E;
      for (const Loc& l : w.srcs) {
        const int h = home_of(l);
        if (h == w.exec) continue;
        in[row + w.exec] += b / pull_bw;
        eg[row + h] += b / pull_bw;
      }
      const int hd = home_of(w.dst);
      if (hd != w.exec) {
        eg[row + w.exec] += b / push_bw;
        in[row + hd] += b / push_bw;
      }
    }
    double t = 0;
    for (int s = 0; s < nsteps; ++s) {
      double m = 0;
      for (int e = 0; e < E; ++e) m = std::max({m, eg[(size_t)s * E + e], in[(size_t)s * E + e]});
      t += m;
    }
    return t;
  };
  std::map<Key, std::set<int>> readers;
  for (const WorkItem& w : S.items)
    for (const Loc& l : w.srcs) readers[{l.rank, l.buffer}].insert(w.exec);
  double best = link_time();
  for (const auto& [key, ex] : readers) {
    const auto [r, b] = key;
    if (!S.buffer_decls[b].internal || b == S.staging_buffer || ex.size() != 1) continue;
    const int x = *ex.begin(), was = S.home[r][b];
    if (x == was) continue;
    S.home[r][b] = x;
    const double t = link_time();
    if (t < best * (1 - 1e-9)) best = t;
    else S.home[r][b] = was;
  }
}

}  // namespace

Schedule build_schedule(const PipelinedPlan& plan, const std::vector<int>& rank_to_exec,
                        int num_execs, int element_size, CopyMode copy_mode) {
  const StagedPlan& base = plan.base;
  Schedule S;
  S.world_size = base.world_size;
  S.num_execs = num_execs;
  S.rank_to_exec = rank_to_exec;
  if ((int)rank_to_exec.size() != base.world_size)
    throw Error(ErrorCode::InvalidConfig, "rank_to_exec must name an executor for every rank");
  for (int e : rank_to_exec)
    if (e < 0 || e >= num_execs) throw Error(ErrorCode::InvalidConfig, "executor index out of range");
  if (element_size < 1) throw Error(ErrorCode::InvalidConfig, "element size < 1");

  std::map<std::string, int> buf_id;
  for (const auto& [name, d] : base.buffers) {
    buf_id[name] = (int)S.buffer_names.size();
    S.buffer_names.push_back(name);
    S.buffer_decls.push_back(d);
  }
  const int nbuf = (int)S.buffer_names.size();

  // Transfers in (slot, id) order — the reference's execution order
  // (engine.cpp:288-293).
  std::vector<Xfer> xs;
  xs.reserve(base.transfers.size());
  for (const auto& t : base.transfers) {
    // a copy of a range onto itself changes nothing in the sequential
    // execution (engine.cpp:309-326), but as a write group member it would
    // hide the earlier folds of its slot: drop it
    if (!t.reduce && t.src == t.dst && t.src_buffer == t.dst_buffer && t.src_offset == t.dst_offset)
      continue;
    xs.push_back(Xfer{t.id, t.slot, Loc{t.src, buf_id.at(t.src_buffer), t.src_offset},
                      Loc{t.dst, buf_id.at(t.dst_buffer), t.dst_offset}, t.count, t.reduce,
                      t.op});
  }
  std::stable_sort(xs.begin(), xs.end(), [](const Xfer& a, const Xfer& b) {
    return std::tie(a.slot, a.id) < std::tie(b.slot, b.id);
  });

  // Arena extents (elements) of internal buffers per rank.
  S.extent.assign(S.world_size, std::vector<int64_t>(nbuf, 0));
  for (const auto& x : xs) {
    for (const Loc* l : {&x.src, &x.dst}) {
      if (l->rank < 0 || l->rank >= S.world_size)
        throw Error(ErrorCode::RankOutOfRange, "transfer rank out of range");
      int64_t& e = S.extent[l->rank][l->buffer];
      e = std::max(e, l->offset + x.count);
    }
  }

  // ---- write groups per slot ----
  struct SlotItem {
    WorkItem w;
    std::vector<int> contrib;  // indices into xs (effective contributors)
  };
  std::map<int, std::vector<SlotItem>> slot_items;
  size_t i = 0;
  while (i < xs.size()) {
    size_t j = i;
    while (j < xs.size() && xs[j].slot == xs[i].slot) ++j;
    const int slot = xs[i].slot;
    std::map<Key, std::vector<size_t>> by_dst;
    for (size_t k = i; k < j; ++k) by_dst[{xs[k].dst.rank, xs[k].dst.buffer}].push_back(k);
    for (auto& [key, list] : by_dst) {
      std::vector<int64_t> cuts;
      for (size_t k : list) {
        cuts.push_back(xs[k].dst.offset);
        cuts.push_back(xs[k].dst.offset + xs[k].count);
      }
      std::sort(cuts.begin(), cuts.end());
      cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
      const size_t nseg = cuts.size() - 1;
      std::vector<std::vector<size_t>> cover(nseg);
      for (size_t k : list) {  // list is in id order
        auto a = std::lower_bound(cuts.begin(), cuts.end(), xs[k].dst.offset) - cuts.begin();
        auto b = std::lower_bound(cuts.begin(), cuts.end(), xs[k].dst.offset + xs[k].count) -
                 cuts.begin();
        for (auto s = a; s < b; ++s) cover[s].push_back(k);
      }
      size_t s = 0;
      while (s < nseg) {
        if (cover[s].empty()) {
          ++s;
          continue;
        }
        size_t e = s + 1;
        while (e < nseg && cover[e] == cover[s]) ++e;  // maximal segment
        const int64_t lo = cuts[s], hi = cuts[e];
        const auto& c = cover[s];
        size_t first = 0;
        bool has_copy = false;
        for (size_t q = 0; q < c.size(); ++q)
          if (!xs[c[q]].reduce) {
            first = q;
            has_copy = true;
          }
        SlotItem it;
        it.w.dst = Loc{key.first, key.second, lo};
        it.w.count = hi - lo;
        it.w.reads_dst = !has_copy;
        if (!has_copy) it.w.srcs.push_back(it.w.dst);
        bool op_set = false;
        for (size_t q = has_copy ? first : 0; q < c.size(); ++q) {
          const Xfer& x = xs[c[q]];
          // a fold of the range into itself reads what the group's earlier
          // members wrote: one register pass cannot express it
          if (x.src.rank == x.dst.rank && x.src.buffer == x.dst.buffer &&
              x.src.offset == x.dst.offset && !it.w.srcs.empty() &&
              !(it.w.reads_dst && it.w.srcs.size() == 1))
            throw Error(ErrorCode::ReadWriteRace,
                        "a transfer folds a range into itself after other writes to it in the same slot");
          it.w.srcs.push_back(Loc{x.src.rank, x.src.buffer, x.src.offset + (lo - x.dst.offset)});
          it.contrib.push_back((int)c[q]);
          if (x.reduce) {
            if (op_set && x.op != it.w.op)
              throw Error(ErrorCode::DependencyViolation,
                          "mixed reduce operators fold into one range in one slot");
            it.w.op = x.op;
            op_set = true;
          }
        }
        for (size_t q = 0; q < c.size(); ++q) it.w.transfer_ids.push_back(xs[c[q]].id);
        // A source that partially overlaps its own destination would be
        // read while it is being written (the sequential element loop of
        // engine.cpp:309-326 "smears" such ranges); identical ranges are
        // harmless self-updates.
        for (const Loc& l : it.w.srcs)
          if (l.rank == it.w.dst.rank && l.buffer == it.w.dst.buffer && l.offset != lo &&
              l.offset < hi && lo < l.offset + (hi - lo))
            throw Error(ErrorCode::ReadWriteRace,
                        "a transfer reads a range it partially overwrites");
        slot_items[slot].push_back(std::move(it));
        s = e;
      }
    }
    i = j;
  }

  // ---- phases inside a slot (RAW / WAR between different items) ----
  std::vector<std::pair<int, int>> steps;  // (slot, phase)
  std::map<std::pair<int, int>, int> step_index;
  for (auto& [slot, items] : slot_items) {
    const size_t n = items.size();
    std::vector<int> phase(n, 0);
    // writer index per (rank, buffer)
    std::map<Key, std::vector<size_t>> writers;
    for (size_t a = 0; a < n; ++a) writers[{items[a].w.dst.rank, items[a].w.dst.buffer}].push_back(a);
    std::vector<std::vector<size_t>> after(n);  // a -> items that must follow a
    std::vector<int> indeg(n, 0);
    for (size_t b = 0; b < n; ++b) {
      const auto& wb = items[b].w;
      for (size_t q = wb.reads_dst ? 1 : 0; q < wb.srcs.size(); ++q) {
        const Loc& src = wb.srcs[q];
        auto it = writers.find({src.rank, src.buffer});
        if (it == writers.end()) continue;
        const int reader_id = xs[items[b].contrib[q - (wb.reads_dst ? 1 : 0)]].id;
        for (size_t a : it->second) {
          if (a == b) continue;
          const auto& wa = items[a].w;
          if (wa.dst.offset >= src.offset + wb.count || src.offset >= wa.dst.offset + wa.count)
            continue;
          // every transfer of the segment counts, the ones a later copy
          // overwrites too: the read sees (or not) their writes
          bool before = true, later = true;
          for (int id : wa.transfer_ids) {
            before &= id < reader_id;
            later &= id > reader_id;
          }
          if (!before && !later)
            throw Error(ErrorCode::DependencyViolation,
                        "slot " + std::to_string(slot) +
                            " interleaves a read and the writes of another range");
          size_t from = before ? a : b, to = before ? b : a;
          after[from].push_back(to);
          ++indeg[to];
        }
      }
    }
    // Kahn layering
    std::vector<size_t> frontier;
    for (size_t a = 0; a < n; ++a)
      if (indeg[a] == 0) frontier.push_back(a);
    size_t seen = 0;
    while (!frontier.empty()) {
      std::vector<size_t> next;
      for (size_t a : frontier) {
        ++seen;
        for (size_t b : after[a]) {
          phase[b] = std::max(phase[b], phase[a] + 1);
          if (--indeg[b] == 0) next.push_back(b);
        }
      }
      frontier = std::move(next);
    }
    if (seen != n)
      throw Error(ErrorCode::DependencyViolation,
                  "cyclic read/write order inside slot " + std::to_string(slot));
    for (size_t a = 0; a < n; ++a) {
      items[a].w.step = phase[a];  // temporarily the phase
      S.max_phases = std::max(S.max_phases, phase[a] + 1);
      steps.emplace_back(slot, phase[a]);
    }
  }
  // ---- staged push: remote reduction sources become pushes into staging ----
  // (ll: every remote source, copies included, lands in staging as 16-byte
  // lines {w0, tag, w1, tag} carrying 8 payload bytes and the launch's tag)
  const bool ll = copy_mode == CopyMode::ll;
  auto landing_elems = [&](int64_t count) {
    if (!ll) return count;
    const int64_t lines = (count * element_size + 7) / 8;
    return lines * 16 / element_size;
  };
  if (copy_mode == CopyMode::staged || ll) {
    const int stage_buf = (int)S.buffer_names.size();
    S.staging_buffer = stage_buf;
    S.buffer_names.push_back("__hiccl.staging");
    S.buffer_decls.push_back(BufferDecl{0, false, true});
    for (auto& row : S.extent) row.push_back(0);
    std::vector<int64_t> cursor(S.world_size, 0);
    steps.clear();
    for (auto& [slot, items] : slot_items) {
      std::vector<SlotItem> added;
      for (auto& it : items) {
        WorkItem& w = it.w;
        const int phase = w.step;
        w.step = 2 * phase + 1;  // keeps the original order, room for staging before
        const bool reduction = w.reads_dst || w.srcs.size() > 1;
        if (!reduction && !ll) {
          steps.emplace_back(slot, w.step);
          continue;
        }
        const int dst_exec = rank_to_exec[w.dst.rank];
        for (size_t q = w.reads_dst ? 1 : 0; q < w.srcs.size(); ++q) {
          if (rank_to_exec[w.srcs[q].rank] == dst_exec) continue;
          const Loc land{w.dst.rank, stage_buf, cursor[w.dst.rank]};
          cursor[w.dst.rank] += align_up(landing_elems(w.count), std::max(1, 16 / element_size));
          SlotItem c;
          c.w.step = 2 * phase;
          c.w.dst = land;
          c.w.count = w.count;
          c.w.op = w.op;
          c.w.srcs = {w.srcs[q]};
          c.w.tile_key = w.dst.offset;
          c.w.staging = true;
          w.srcs[q] = land;
          steps.emplace_back(slot, c.w.step);
          added.push_back(std::move(c));
        }
        steps.emplace_back(slot, w.step);
      }
      for (auto& c : added) items.push_back(std::move(c));
    }
    for (int r = 0; r < S.world_size; ++r) S.extent[r][stage_buf] = cursor[r];
    int64_t longest = 1;
    for (int64_t c : cursor) longest = std::max(longest, c);
    S.buffer_decls[stage_buf].length = longest;
  }
  std::sort(steps.begin(), steps.end());
  steps.erase(std::unique(steps.begin(), steps.end()), steps.end());
  for (size_t k = 0; k < steps.size(); ++k) {
    step_index[steps[k]] = (int)k;
    S.step_slot.push_back(steps[k].first);
    S.step_phase.push_back(steps[k].second);
  }
  const int nsteps = (int)steps.size();

  // ---- executor assignment ----
  for (auto& [slot, items] : slot_items) {
    for (auto& it : items) {
      WorkItem w = std::move(it.w);
      w.step = step_index.at({slot, w.step});
      const bool pure_copy = !w.reads_dst && w.srcs.size() == 1;
      const int owner =
          (pure_copy && copy_mode != CopyMode::pull) ? w.srcs[0].rank : w.dst.rank;
      w.exec = rank_to_exec[owner];
      S.max_sources = std::max(S.max_sources, (int)w.srcs.size());
      S.items.push_back(std::move(w));
    }
  }

  const int nbuf_all = (int)S.buffer_names.size();
  S.home.assign(S.world_size, std::vector<int>(nbuf_all, 0));
  for (int r = 0; r < S.world_size; ++r)
    for (int b = 0; b < nbuf_all; ++b) S.home[r][b] = rank_to_exec[r];
  if (copy_mode == CopyMode::push) {
    fuse_deferred_init(S);
    fuse_forward_copy(S);
    place_internal_buffers(S, element_size);
  }

  // ---- internal-buffer arena: only the ranges each rank touches ----
  S.ll = ll;
  S.arena_offset.assign(S.world_size, std::vector<int64_t>(nbuf_all, -1));
  S.arena_bytes.assign(num_execs, 0);
  for (int r = 0; r < S.world_size; ++r) {
    for (int b = 0; b < nbuf_all; ++b) {
      if (!S.buffer_decls[b].internal || S.extent[r][b] == 0) continue;
      const int e = S.home[r][b];
      S.arena_offset[r][b] = S.arena_bytes[e];
      S.arena_bytes[e] = align_up(S.arena_bytes[e] + S.extent[r][b] * element_size, 256);
    }
  }
  if (ll) {
    // Two copies of every arena, alternating by launch parity, so a
    // producer may fill epoch e's staging while its consumer still reads
    // epoch e-1's; the copy distance is the same on every executor.
    for (int64_t b : S.arena_bytes) S.ll_half = std::max(S.ll_half, b);
    S.ll_half = align_up(std::max<int64_t>(S.ll_half, 256), 256);
    for (int64_t& b : S.arena_bytes) b = 2 * S.ll_half;
  }

  // ---- cross-step hazards -> waits ----
  std::map<Key, std::vector<Access>> acc;
  for (int k = 0; k < (int)S.items.size(); ++k) {
    const WorkItem& w = S.items[k];
    acc[{w.dst.rank, w.dst.buffer}].push_back(
        Access{w.dst.offset, w.dst.offset + w.count, w.step, w.exec, k, true});
    for (size_t q = w.reads_dst ? 1 : 0; q < w.srcs.size(); ++q)
      acc[{w.srcs[q].rank, w.srcs[q].buffer}].push_back(
          Access{w.srcs[q].offset, w.srcs[q].offset + w.count, w.step, w.exec, k, false});
  }
  for (auto& [key, v] : acc)
    std::sort(v.begin(), v.end(), [](const Access& a, const Access& b) { return a.lo < b.lo; });

  S.execs.assign(num_execs, ExecProgram{});
  for (auto& ep : S.execs) {
    ep.items_by_step.assign(nsteps, {});
    ep.waits.assign(nsteps, {});
    ep.publish.assign(nsteps, false);
  }
  // need[exec][step][peer] = latest peer step that must be finished
  std::vector<std::vector<std::vector<int>>> need(
      num_execs, std::vector<std::vector<int>>(nsteps, std::vector<int>(num_execs, -1)));
  for (int k = 0; k < (int)S.items.size(); ++k) {
    const WorkItem& w = S.items[k];
    S.execs[w.exec].items_by_step[w.step].push_back(k);
    auto scan = [&](const Loc& l, bool is_write) {
      const auto& v = acc.at({l.rank, l.buffer});
      const int64_t lo = l.offset, hi = l.offset + w.count;
      for (const Access& a : v) {
        if (a.lo >= hi) break;
        if (a.hi <= lo || a.step >= w.step) continue;
        if (!is_write && !a.write) continue;  // read-read is no hazard
        int& n = need[w.exec][w.step][a.exec];
        n = std::max(n, a.step);
      }
    };
    scan(w.dst, true);
    for (size_t q = w.reads_dst ? 1 : 0; q < w.srcs.size(); ++q) scan(w.srcs[q], false);
  }
  for (int e = 0; e < num_execs; ++e)
    for (int s = 0; s < nsteps; ++s)
      for (int x = 0; x < num_execs; ++x)
        if (need[e][s][x] >= 0) {
          S.execs[e].waits[s].push_back(StepWait{x, need[e][s][x]});
          S.execs[x].publish[need[e][s][x]] = true;
        }
  return S;
}

// Segment-compressed replay. Every (rank, buffer) is cut at both ends of
// every range a transfer or an item touches, and the cuts are closed under
// the shifts the transfers and items apply (a cut inside a destination range
// is a cut at the same position of each source range, and back), so all
// elements of a segment go through the same sequence of operations and one
// value stands for them. The replay is then exact at a cost set by the
// plan's structure, not its byte counts: 1 GiB plans verify as fast as
// 1 KiB ones.
bool replay_schedule(const PipelinedPlan& plan, const Schedule& S, int64_t max_segments) {
  std::map<std::string, int> bid;
  for (size_t b = 0; b < S.buffer_names.size(); ++b) bid[S.buffer_names[b]] = (int)b;
  const int nb = (int)S.buffer_names.size();
  const int p = S.world_size;
  auto key = [nb](int r, int b) { return (size_t)r * nb + b; };

  // shift maps: [a, a + n) on one side is [b, b + n) on the other
  struct Shift {
    size_t ka, kb;
    int64_t a, b, n;
  };
  std::vector<Shift> shifts;
  for (const auto& t : plan.base.transfers)
    shifts.push_back({key(t.src, bid.at(t.src_buffer)), key(t.dst, bid.at(t.dst_buffer)),
                      t.src_offset, t.dst_offset, t.count});
  for (const auto& w : S.items)
    for (const auto& l : w.srcs)
      shifts.push_back({key(l.rank, l.buffer), key(w.dst.rank, w.dst.buffer), l.offset,
                        w.dst.offset, w.count});
  std::vector<std::set<int64_t>> cuts((size_t)p * nb);
  std::vector<std::vector<std::pair<int, bool>>> on(cuts.size());  // shifts ending on a key
  for (int r = 0; r < p; ++r)
    for (int b = 0; b < nb; ++b) cuts[key(r, b)] = {0, S.buffer_decls[b].length};
  std::vector<std::pair<size_t, int64_t>> work;
  int64_t total = 0;
  auto add = [&](size_t k, int64_t x) {
    if (cuts[k].insert(x).second) {
      work.push_back({k, x});
      ++total;
    }
  };
  for (size_t i = 0; i < shifts.size(); ++i) {
    const Shift& m = shifts[i];
    on[m.ka].push_back({(int)i, true});
    on[m.kb].push_back({(int)i, false});
    add(m.ka, m.a), add(m.ka, m.a + m.n), add(m.kb, m.b), add(m.kb, m.b + m.n);
  }
  while (!work.empty()) {
    if (total > max_segments) return false;
    const auto [k, x] = work.back();
    work.pop_back();
    for (const auto& [i, side_a] : on[k]) {
      const Shift& m = shifts[i];
      const int64_t lo = side_a ? m.a : m.b;
      if (x <= lo || x >= lo + m.n) continue;
      if (side_a) add(m.kb, m.b + (x - m.a));
      else add(m.ka, m.a + (x - m.b));
    }
  }

  // one value per segment; a range maps to consecutive segments
  std::vector<std::vector<int64_t>> starts(cuts.size());
  for (size_t k = 0; k < cuts.size(); ++k) starts[k].assign(cuts[k].begin(), cuts[k].end());
  auto first_seg = [&](size_t k, int64_t off) {
    const auto& v = starts[k];
    const auto it = std::lower_bound(v.begin(), v.end(), off);
    if (it == v.end() || *it != off) throw Error(ErrorCode::DependencyViolation, "replay: a range ends off a cut");
    return (size_t)(it - v.begin());
  };
  using State = std::vector<std::vector<uint64_t>>;
  auto init = [&]() {
    State st(cuts.size());
    for (int r = 0; r < p; ++r)
      for (int b = 0; b < nb; ++b) {
        const size_t k = key(r, b);
        st[k].assign(starts[k].size() - 1, 0);
        if (S.buffer_decls[b].input)
          for (size_t g = 0; g + 1 < starts[k].size(); ++g)
            st[k][g] = 0x9E3779B97F4A7C15ULL * (uint64_t)(r * 1000003 + b * 7919 + starts[k][g] + 1);
      }
    return st;
  };
  auto fold = [](uint64_t a, uint64_t b) { return a * 0x100000001B3ULL + (b ^ (b >> 29)); };
  // segments of [off, off + n) on key k: (first index, count)
  auto span = [&](size_t k, int64_t off, int64_t n) {
    const size_t g0 = first_seg(k, off), g1 = first_seg(k, off + n);
    return std::make_pair(g0, g1 - g0);
  };

  State seq = init();
  std::vector<const P2PTransfer*> order;
  for (const auto& t : plan.base.transfers) order.push_back(&t);
  std::stable_sort(order.begin(), order.end(), [](const P2PTransfer* a, const P2PTransfer* b) {
    return std::tie(a->slot, a->id) < std::tie(b->slot, b->id);
  });
  for (const P2PTransfer* t : order) {
    const size_t ks = key(t->src, bid.at(t->src_buffer)), kd = key(t->dst, bid.at(t->dst_buffer));
    const auto [s0, n] = span(ks, t->src_offset, t->count);
    const size_t d0 = span(kd, t->dst_offset, t->count).first;
    // element by element in the reference; segment by segment here, in the
    // same order (an in-place shifted copy is refused upstream)
    for (size_t g = 0; g < n; ++g) {
      const uint64_t v = seq[ks][s0 + g];
      uint64_t& c = seq[kd][d0 + g];
      c = t->reduce ? fold(c, v) : v;
    }
  }
  State par = init();
  const int nsteps = (int)S.step_slot.size();
  std::vector<std::vector<int>> by_step(nsteps);
  for (int k = 0; k < (int)S.items.size(); ++k) by_step[S.items[k].step].push_back(k);
  std::mt19937 rng(12345);
  for (int s = 0; s < nsteps; ++s) {
    const State snap = par;
    auto ids = by_step[s];
    std::shuffle(ids.begin(), ids.end(), rng);
    for (int k : ids) {
      const WorkItem& w = S.items[k];
      const size_t kd = key(w.dst.rank, w.dst.buffer);
      const auto [d0, n] = span(kd, w.dst.offset, w.count);
      std::vector<size_t> ks, s0;
      for (const auto& l : w.srcs) {
        ks.push_back(key(l.rank, l.buffer));
        s0.push_back(span(ks.back(), l.offset, w.count).first);
      }
      for (size_t g = 0; g < n; ++g) {
        uint64_t a = snap[ks[0]][s0[0] + g];
        for (size_t q = 1; q < ks.size(); ++q) a = fold(a, snap[ks[q]][s0[q] + g]);
        par[kd][d0 + g] = a;
      }
    }
  }
  for (int r = 0; r < p; ++r)
    for (int b = 0; b < nb; ++b)
      // internal buffers are scratch: push schedules may fold or forward
      // past them (fuse_deferred_init, fuse_forward_copy); what they feed
      // is compared in the user buffers
      if (!S.buffer_decls[b].internal && seq[key(r, b)] != par[key(r, b)])
        throw Error(ErrorCode::DependencyViolation,
                    "schedule replay differs from sequential execution at rank " +
                        std::to_string(r) + " buffer " + S.buffer_names[b]);
  return true;
}

void verify_schedule(const PipelinedPlan& plan, const Schedule& S) {
  // 1) every transfer contributes to some item; contributors cover the
  //    item's range.
  std::vector<int> seen(plan.base.transfers.size(), 0);
  for (const auto& w : S.items)
    for (int id : w.transfer_ids) seen.at(id) = 1;
  for (const auto& t : plan.base.transfers)
    if (!t.reduce && t.src == t.dst && t.src_buffer == t.dst_buffer && t.src_offset == t.dst_offset)
      seen.at(t.id) = 1;  // identity copy, dropped by build_schedule
  for (size_t k = 0; k < seen.size(); ++k)
    if (!seen[k])
      throw Error(ErrorCode::DependencyViolation, "transfer " + std::to_string(k) + " lost");

  // 2) numeric replay with an order-sensitive, non-commutative fold
  if (!replay_schedule(plan, S, 1LL << 26))
    throw Error(ErrorCode::InvalidConfig, "schedule too fragmented to replay");

  // 3) every cross-step hazard has a wait edge (independent O(n^2) scan).
  auto overlap = [](const Loc& a, int64_t na, const Loc& b, int64_t nb2) {
    return a.rank == b.rank && a.buffer == b.buffer && a.offset < b.offset + nb2 &&
           b.offset < a.offset + na;
  };
  for (size_t x = 0; x < S.items.size(); ++x)
    for (size_t y = 0; y < S.items.size(); ++y) {
      const WorkItem& early = S.items[x];
      const WorkItem& late = S.items[y];
      if (early.step >= late.step) continue;
      bool hazard = overlap(early.dst, early.count, late.dst, late.count);
      for (const auto& s2 : late.srcs) hazard |= overlap(early.dst, early.count, s2, late.count);
      for (const auto& s1 : early.srcs) hazard |= overlap(s1, early.count, late.dst, late.count);
      if (!hazard) continue;
      bool ok = false;
      for (const auto& wt : S.execs[late.exec].waits[late.step])
        ok |= wt.exec == early.exec && wt.step >= early.step;
      if (!ok)
        throw Error(ErrorCode::DependencyViolation,
                    "hazard between steps " + std::to_string(early.step) + " and " +
                        std::to_string(late.step) + " has no wait edge");
    }
}

}  // namespace hiccl
