// Device layout and tile-granular synchronization (see layout.hpp).
#include "layout.hpp"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <tuple>

#include "hiccl.h"

namespace hiccl {

namespace {

int first_rank_of(const Schedule& s, int exec) {
  for (int r = 0; r < s.world_size; ++r)
    if (s.rank_to_exec[r] == exec) return r;
  return 0;
}

bool nvls_reduce_ok(int dtype, ReduceOp op) {
  switch (dtype) {
    case HC_F32: case HC_BF16: case HC_F16: return op == ReduceOp::sum;
    case HC_I32: return true;
    default: return false;
  }
}

// Tile -> CTA placement of one item whose last partial rotation has
// `rem` tiles (whole rotations load every CTA alike). The natural base is
// the destination range's position on the tile grid: a range produced in
// one step and consumed in a later one then sits on the same CTA, and the
// consumer waits for that one CTA. When earlier items of the step already
// crowd that window — several ranks' copies of one range: virtual ranks
// sharing a GPU, the copies of a multicast — the item takes the rotation
// whose busiest CTA is least loaded instead (sliding-window maximum over
// the circular load vector); the wait analysis follows any placement.
uint32_t place_item(std::vector<uint32_t>& load, uint32_t natural, uint32_t rem) {
  const uint32_t G = (uint32_t)load.size();
  static const bool natural_only = std::getenv("HICCL_NATURAL_PLACEMENT") != nullptr;  // A/B
  if (rem == 0 || natural_only) return natural;
  // peak[b] = max(load[b .. b+rem-1]) (circular), by a monotone deque
  std::vector<uint32_t> peak(G);
  std::vector<uint32_t> dq;  // indices into the doubled array, loads decreasing
  size_t head = 0;
  for (uint32_t i = 0; i < G + rem - 1; ++i) {
    const uint32_t v = load[i % G];
    while (dq.size() > head && load[dq.back() % G] <= v) dq.pop_back();
    dq.push_back(i);
    if (i + 1 >= rem) {
      const uint32_t b = i + 1 - rem;
      while (dq[head] < b) ++head;
      peak[b] = load[dq[head] % G];
    }
  }
  uint32_t best = natural;
  for (uint32_t b = 0; b < G; ++b)
    if (peak[b] < peak[best]) best = b;
  for (uint32_t k = 0; k < rem; ++k) ++load[(best + k) % G];
  return best;
}

}  // namespace

int auto_ctas(const Schedule& s, int esize, int threads, int sms) {
  if (s.ll) {
    // Tagged lines: one warp per tile, and a single SM drains only
    // ~20 GB/s of peer stores, so spread the busiest step's tiles over as
    // many SMs as it has tiles.
    int64_t max_tiles = 1;
    for (const auto& ep : s.execs)
      for (const auto& items : ep.items_by_step) {
        int64_t t = 0;
        for (int k : items) t += (s.items[k].count * esize + kLLTileBytes - 1) / kLLTileBytes;
        max_tiles = std::max(max_tiles, t);
      }
    return (int)std::min<int64_t>(sms, max_tiles);
  }
  int64_t max_step = 0;
  for (const auto& ep : s.execs)
    for (const auto& items : ep.items_by_step) {
      int64_t b = 0;
      for (int k : items) b += s.items[k].count * esize;
      max_step = std::max(max_step, b);
    }
  const int64_t min_tile = (int64_t)threads * 16 * 2;
  return (int)std::max<int64_t>(1, std::min<int64_t>(sms, (max_step + min_tile - 1) / min_tile));
}

bool want_alt_halves(const Schedule& s, int esize) {
  if (s.ll) return false;
  int busy = 0;
  int64_t max_step = 0;
  for (size_t st = 0; st < s.step_slot.size(); ++st) {
    int64_t top = 0;
    for (const auto& ep : s.execs) {
      int64_t b = 0;
      for (int k : ep.items_by_step[st]) b += s.items[k].count * esize;
      top = std::max(top, b);
    }
    busy += top > 0;
    max_step = std::max(max_step, top);
  }
  return busy >= 4 && max_step <= (int64_t)8 << 20;
}

ExecLayout build_layout(const Schedule& s, int exec, const LayoutParams& lp) {
  ExecLayout out;
  const int P = s.world_size;
  const int me = first_rank_of(s, exec);
  const int esz = lp.esize;
  bool nvls = false;
  for (bool b : lp.multicast) nvls |= b;
  nvls &= !s.ll;  // ll keeps every cross-GPU byte in tagged lines
  if (nvls) {  // one rank per executor
    nvls = s.num_execs == P;
    std::vector<int> seen(s.num_execs, 0);
    for (int r = 0; r < P && nvls; ++r) nvls &= !seen[s.rank_to_exec[r]]++;
  }
  auto mc_ok = [&](int buf) { return buf < (int)lp.multicast.size() && lp.multicast[buf]; };
  auto vec_ok = [&](int64_t off) { return (off * esz) % 16 == 0; };

  const int nsteps = (int)s.step_slot.size();
  out.steps.resize(nsteps);
  for (int st = 0; st < nsteps; ++st) {
    std::vector<int> order = s.execs[exec].items_by_step[st];
    // Peer rotation: start on the peer `distance` ranks ahead so executors
    // do not all converge on rank 0 at the start of a step.
    // Items with no remote side (several ranks on this GPU) group by their
    // first source instead, so copies of one range run back to back (L2 reuse).
    auto peer_of = [&](const WorkItem& w) {
      if (s.rank_to_exec[w.dst.rank] != exec) return w.dst.rank;
      for (const Loc& l : w.srcs)
        if (s.rank_to_exec[l.rank] != exec) return l.rank;
      return w.srcs.empty() ? w.dst.rank : w.srcs[0].rank;
    };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return (peer_of(s.items[a]) - me + P) % P < (peer_of(s.items[b]) - me + P) % P;
    });

    StepLayout& L = out.steps[st];
    const bool alt = lp.alt_halves && !s.ll && lp.ctas >= 2 && lp.ctas % 2 == 0;
    L.cta_n = alt ? lp.ctas / 2 : lp.ctas;
    L.cta_lo = alt ? (st % 2) * L.cta_n : 0;
    std::vector<bool> used(order.size(), false);
    for (size_t i = 0; i < order.size(); ++i) {
      if (used[i]) continue;
      const WorkItem& w = s.items[order[i]];
      const bool whole = (w.count * esz) % 16 == 0;
      // every-rank fold of one (buffer, offset) -> multimem.ld_reduce
      if (nvls && whole && !w.reads_dst && (int)w.srcs.size() == P &&
          nvls_reduce_ok(lp.dtype, w.op) && mc_ok(w.srcs[0].buffer)) {
        bool all = vec_ok(w.srcs[0].offset) && vec_ok(w.dst.offset);
        std::vector<int> hit(P, 0);
        for (const Loc& l : w.srcs) {
          all &= l.buffer == w.srcs[0].buffer && l.offset == w.srcs[0].offset;
          hit[l.rank]++;
        }
        for (int r = 0; r < P; ++r) all &= hit[r] == 1;
        if (all) {
          AbsItem it;
          it.dst = AbsRef{w.dst.rank, w.dst.buffer, w.dst.offset, false};
          it.srcs = {AbsRef{-1, w.srcs[0].buffer, w.srcs[0].offset, true}};
          it.count = w.count;
          it.op = w.op;
          it.kind = ItemKind::mc_reduce;
          it.tile_key = w.dst.offset;
          L.items.push_back(std::move(it));
          used[i] = true;
          continue;
        }
      }
      // one source range to the same range of every rank -> multimem.st
      const bool copy = !w.reads_dst && w.srcs.size() == 1;
      if (nvls && whole && copy && s.rank_to_exec[w.srcs[0].rank] == exec && mc_ok(w.dst.buffer) &&
          vec_ok(w.dst.offset) && vec_ok(w.srcs[0].offset)) {
        const Loc& s0 = w.srcs[0];
        std::vector<size_t> group;
        std::vector<int> hit(P, 0);
        for (size_t j = i; j < order.size(); ++j) {
          if (used[j]) continue;
          const WorkItem& x = s.items[order[j]];
          if (x.reads_dst || x.srcs.size() != 1 || x.count != w.count) continue;
          const Loc& sx = x.srcs[0];
          if (sx.rank != s0.rank || sx.buffer != s0.buffer || sx.offset != s0.offset) continue;
          if (x.dst.buffer != w.dst.buffer || x.dst.offset != w.dst.offset) continue;
          group.push_back(j);
          hit[x.dst.rank] = 1;
        }
        // the multicast also writes the source rank's own copy of the range
        bool all = hit[s0.rank] || (s0.buffer == w.dst.buffer && s0.offset == w.dst.offset);
        for (int r = 0; r < P; ++r) all &= hit[r] || r == s0.rank;
        if (all) {
          for (size_t j : group) used[j] = true;
          AbsItem it;
          it.dst = AbsRef{-1, w.dst.buffer, w.dst.offset, true};
          it.srcs = {AbsRef{s0.rank, s0.buffer, s0.offset, false}};
          it.count = w.count;
          it.op = w.op;
          it.kind = ItemKind::mc_store;
          it.tile_key = w.dst.offset;
          L.items.push_back(std::move(it));
          continue;
        }
      }
      AbsItem it;
      auto is_ll = [&](const Loc& l) { return s.ll && l.buffer == s.staging_buffer; };
      it.dst = AbsRef{w.dst.rank, w.dst.buffer, w.dst.offset, false, is_ll(w.dst)};
      for (const Loc& l : w.srcs)
        it.srcs.push_back(AbsRef{l.rank, l.buffer, l.offset, false, is_ll(l)});
      it.count = w.count;
      it.op = w.op;
      it.tile_key = w.tile_key >= 0 ? w.tile_key : w.dst.offset;
      L.items.push_back(std::move(it));
      used[i] = true;
    }

    // Tile size: the largest threads * {8,4,2,1} vectors that still gives
    // every CTA a tile.
    int kv = lp.max_tile_vec;
    for (; kv > 1; kv /= 2) {
      const int64_t te = (int64_t)lp.threads * kv * 16 / esz;
      int64_t nt = 0;
      for (const AbsItem& it : L.items) nt += (it.count + te - 1) / te;
      if (nt >= L.cta_n) break;
    }
    L.tile_elems = lp.threads * kv * 16 / esz;
    // tagged-line schedules: one warp per tile; 2 lines of 8 payload bytes
    // per lane (one batch of polls per tile, kernels.cuh run_tile_ll) while
    // the step has warps to spare, larger tiles once it has more tiles than
    // the grid has warps (per-tile overhead then dominates)
    if (s.ll) {
      const int64_t warps = (int64_t)lp.ctas * std::max(1, lp.threads / 32);
      int64_t tb = kLLTileBytes;
      auto tiles = [&](int64_t bytes) {
        int64_t nt = 0;
        for (const AbsItem& it : L.items) nt += (it.count * esz + bytes - 1) / bytes;
        return nt;
      };
      while (tb < 8 * kLLTileBytes && tiles(tb) > warps) tb *= 2;
      L.tile_elems = (int)(tb / esz);
    }
    uint32_t tiles = 0;
    std::vector<uint32_t> load(L.cta_n, 0);  // partial-rotation tiles per CTA so far
    for (AbsItem& it : L.items) {
      it.n_tiles = (uint32_t)((it.count + L.tile_elems - 1) / L.tile_elems);
      it.base_cta = place_item(load, (uint32_t)((it.tile_key / L.tile_elems) % L.cta_n),
                               it.n_tiles % (uint32_t)L.cta_n);
      tiles += it.n_tiles;
    }
    L.n_tiles = tiles;
  }
  return out;
}

int fuse_nvls(const Schedule& s, std::vector<ExecLayout>& layouts) {
  const int W = s.world_size;
  struct Acc {
    int64_t lo, hi;
    int step, exec, item;
  };
  // item-level accesses per (rank, buffer); multicast references touch the
  // range on every rank
  std::map<std::pair<int, int>, std::vector<Acc>> acc;
  auto add = [&](const AbsRef& r, int64_t n, int st, int e, int i) {
    if (r.ll) return;
    if (r.multicast) {
      for (int k = 0; k < W; ++k) acc[{k, r.buffer}].push_back(Acc{r.offset, r.offset + n, st, e, i});
    } else {
      acc[{r.rank, r.buffer}].push_back(Acc{r.offset, r.offset + n, st, e, i});
    }
  };
  for (int e = 0; e < (int)layouts.size(); ++e)
    for (int st = 0; st < (int)layouts[e].steps.size(); ++st) {
      const auto& items = layouts[e].steps[st].items;
      for (int i = 0; i < (int)items.size(); ++i) {
        add(items[i].dst, items[i].count, st, e, i);
        for (const AbsRef& r : items[i].srcs) add(r, items[i].count, st, e, i);
      }
    }
  // is [lo, hi) of `buffer` on every rank untouched in steps [s1, s2), the
  // reduction (e, s1, i1) aside?
  auto quiet = [&](int buffer, int64_t lo, int64_t hi, int s1, int s2, int e, int i1) {
    for (int k = 0; k < W; ++k) {
      auto it = acc.find({k, buffer});
      if (it == acc.end()) continue;
      for (const Acc& a : it->second) {
        if (a.step < s1 || a.step >= s2 || a.hi <= lo || a.lo >= hi) continue;
        if (a.exec == e && a.step == s1 && a.item == i1) continue;
        return false;
      }
    }
    return true;
  };
  int fused = 0;
  for (int e = 0; e < (int)layouts.size(); ++e) {
    auto& steps = layouts[e].steps;
    std::vector<std::vector<int>> drop(steps.size());
    for (int s2 = 0; s2 < (int)steps.size(); ++s2)
      for (int i2 = 0; i2 < (int)steps[s2].items.size(); ++i2) {
        const AbsItem& m = steps[s2].items[i2];
        if (m.kind != ItemKind::mc_store) continue;
        const AbsRef& src = m.srcs[0];
        // in-place multicast only: the reduction's own local result is
        // part of what the fused store writes
        if (src.multicast || src.buffer != m.dst.buffer || src.offset != m.dst.offset) continue;
        // the latest earlier reduction of this executor producing exactly it
        int s1 = -1, i1 = -1;
        for (int st = s2 - 1; st >= 0 && s1 < 0; --st)
          for (int i = 0; i < (int)steps[st].items.size(); ++i) {
            const AbsItem& r = steps[st].items[i];
            if (r.kind == ItemKind::mc_reduce && !r.dst.multicast && r.dst.rank == src.rank &&
                r.dst.buffer == src.buffer && r.dst.offset == src.offset && r.count == m.count) {
              s1 = st;
              i1 = i;
              break;
            }
          }
        if (s1 < 0 || !quiet(src.buffer, src.offset, src.offset + m.count, s1, s2, e, i1)) continue;
        AbsItem& r = steps[s1].items[i1];
        r.kind = ItemKind::mc_reduce_store;
        r.dst = AbsRef{-1, src.buffer, src.offset, true};
        add(r.dst, r.count, s1, e, i1);  // later candidates see the new writes
        drop[s2].push_back(i2);
        ++fused;
      }
    for (int st = 0; st < (int)steps.size(); ++st) {
      if (drop[st].empty()) continue;
      std::sort(drop[st].rbegin(), drop[st].rend());
      for (int i : drop[st]) steps[st].items.erase(steps[st].items.begin() + i);
      uint32_t tiles = 0;
      for (const AbsItem& it : steps[st].items) tiles += it.n_tiles;
      steps[st].n_tiles = tiles;
    }
  }
  return fused;
}

std::vector<std::vector<uint32_t>> tile_ordinals(const StepLayout& L) {
  // the device loop (kernels.cuh): for round, for j: item (j + b) % n,
  // tile first(item) + round * G if it exists — per CTA b, a running count
  const uint32_t G = (uint32_t)L.cta_n, n = (uint32_t)L.items.size();
  std::vector<std::vector<uint32_t>> ord(n);
  uint32_t rounds = 0;
  for (uint32_t i = 0; i < n; ++i) {
    ord[i].assign(L.items[i].n_tiles, 0);
    rounds = std::max(rounds, (L.items[i].n_tiles + G - 1) / G);
  }
  std::vector<uint32_t> next(G, 0);  // per CTA, tiles enumerated so far
  for (uint32_t round = 0; round < rounds; ++round)
    for (uint32_t b = 0; b < G; ++b)
      for (uint32_t j = 0; j < n; ++j) {
        const uint32_t i = (j + b) % n;
        const uint32_t local = (b + G - L.items[i].base_cta % G) % G + round * G;
        if (local < L.items[i].n_tiles) ord[i][local] = next[b]++;
      }
  return ord;
}

namespace {

struct Rec {
  int64_t lo, hi;
  int exec, step, cta;
  bool write;
  int ord;  // the tile's ordinal on its CTA within the step
};

// Expand a reference into the (rank, buffer, [lo, hi)) ranges it touches.
// Tagged-line staging is left out: a consumer polls the tags of exactly the
// lines it reads, and each landing range has one writer and one reader.
template <class F>
void touches(const AbsRef& r, int64_t lo, int64_t hi, int world, F&& f) {
  if (r.ll) return;
  if (r.multicast) {
    for (int k = 0; k < world; ++k) f(k, r.buffer, r.offset + lo, r.offset + hi);
  } else {
    f(r.rank, r.buffer, r.offset + lo, r.offset + hi);
  }
}

template <class F>
void for_each_tile_access(const Schedule& s, const ExecLayout& L, int exec, int G, F&& f) {
  (void)G;
  for (int st = 0; st < (int)L.steps.size(); ++st) {
    const StepLayout& S = L.steps[st];
    const auto ord = tile_ordinals(S);
    for (size_t i = 0; i < S.items.size(); ++i) {
      const AbsItem& it = S.items[i];
      for (uint32_t local = 0; local < it.n_tiles; ++local) {
        const int64_t lo = (int64_t)local * S.tile_elems;
        const int64_t hi = std::min<int64_t>(lo + S.tile_elems, it.count);
        const int cta = tile_cta(it, local, S);
        const int o = (int)ord[i][local];
        touches(it.dst, lo, hi, s.world_size, [&](int r, int b, int64_t a, int64_t z) {
          f(exec, st, cta, r, b, a, z, true, o);
        });
        for (const AbsRef& src : it.srcs)
          touches(src, lo, hi, s.world_size, [&](int r, int b, int64_t a, int64_t z) {
            f(exec, st, cta, r, b, a, z, false, o);
          });
      }
    }
  }
}

struct Index {
  std::map<std::pair<int, int>, std::vector<Rec>> by_key;
  std::map<std::pair<int, int>, int64_t> max_len;
  void add(int r, int b, const Rec& rec) {
    by_key[{r, b}].push_back(rec);
    int64_t& m = max_len[{r, b}];
    m = std::max(m, rec.hi - rec.lo);
  }
  void finish() {
    for (auto& [k, v] : by_key)
      std::sort(v.begin(), v.end(), [](const Rec& a, const Rec& b) { return a.lo < b.lo; });
  }
  template <class F>
  void query(int r, int b, int64_t lo, int64_t hi, F&& f) const {
    auto it = by_key.find({r, b});
    if (it == by_key.end()) return;
    const auto& v = it->second;
    const int64_t from = lo - max_len.at({r, b});
    auto p = std::lower_bound(v.begin(), v.end(), from,
                              [](const Rec& a, int64_t x) { return a.lo < x; });
    for (; p != v.end() && p->lo < hi; ++p)
      if (p->hi > lo) f(*p);
  }
};

// Tile-granular waits: for every consumer tile, the producer tiles of
// earlier steps it conflicts with (RAW, WAR, WAW), as progress values
// step * T + ordinal + 1 of the producer CTA. Per (consumer step, CTA,
// producer CTA) only the waits that raise the running maximum along the
// consumer's tile order are kept; those before its first tile go to
// `waits` (checked at step start), later ones to `tile_waits`. A CTA's own
// earlier steps and producers spread over most of an executor keep
// step-level waits.
void analyze_tile_sync(const Schedule& s, const std::vector<ExecLayout>& layouts, const Index& idx,
                       int G, int T, std::vector<ExecSync>& out) {
  const int E = (int)layouts.size();
  for (int f = 0; f < E; ++f) {
    // (step, cta) -> (exec, producer cta) -> [(consumer ordinal, value)]
    std::map<std::pair<int, int>, std::map<std::pair<int, int>, std::vector<std::pair<int, int64_t>>>>
        need;
    for_each_tile_access(s, layouts[f], f, G,
                         [&](int, int st, int cta, int r, int b, int64_t lo, int64_t hi, bool w,
                             int o) {
                           auto& n = need[{st, cta}];
                           idx.query(r, b, lo, hi, [&](const Rec& p) {
                             if (p.step >= st || (!w && !p.write)) return;
                             n[{p.exec, p.cta}].push_back({o, (int64_t)p.step * T + p.ord + 1});
                           });
                         });
    for (auto& [key, deps] : need) {
      const int st = key.first, cta = key.second;
      auto& at0 = out[f].waits[st][cta];
      auto& later = out[f].tile_waits[st][cta];
      std::map<int, int> producers;  // exec -> distinct producer CTAs
      for (auto& [pk, list] : deps) ++producers[pk.first];
      std::map<int, int64_t> whole;  // exec -> max value (step-level whole waits)
      for (auto& [pk, list] : deps) {
        out[f].required[st][cta].push_back(CtaWait{pk.first, pk.second, 0, -1, 0});
        int64_t top = 0;
        for (auto& x : list) top = std::max(top, x.second);
        out[f].required[st][cta].back().step = (int)((top - 1) / T);
        if (producers[pk.first] * 2 > G) {
          int64_t& m = whole[pk.first];
          m = std::max(m, top);
          continue;
        }
        if (pk.first == f && pk.second == cta) {  // own earlier steps: step level
          at0.push_back(CtaWait{pk.first, pk.second, (int)((top - 1) / T), -1, 0});
          ++out[f].paired;
          continue;
        }
        std::sort(list.begin(), list.end());
        int64_t run = 0;
        for (auto& [o, v] : list) {
          if (v <= run) continue;
          run = v;
          CtaWait w{pk.first, pk.second, (int)((v - 1) / T), v, o};
          if (v == (int64_t)(w.step + 1) * T) w.value = -1;
          if (o == 0) {
            if (!at0.empty() && at0.back().exec == w.exec && at0.back().cta == w.cta)
              at0.back() = w;  // a later value at the same ordinal supersedes
            else
              at0.push_back(w);
          } else if (!later.empty() && later.back().exec == w.exec && later.back().cta == w.cta &&
                     later.back().at == o) {
            later.back() = w;
          } else {
            later.push_back(w);
          }
          ++out[f].paired;
        }
      }
      for (auto& [e, v] : whole) {
        at0.push_back(CtaWait{e, -1, (int)((v - 1) / T), -1, 0});
        ++out[f].whole;
      }
      std::stable_sort(later.begin(), later.end(),
                       [](const CtaWait& a, const CtaWait& b) { return a.at < b.at; });
    }
  }
  for (int f = 0; f < E; ++f)
    for (const auto* table : {&out[f].waits, &out[f].tile_waits})
      for (const auto& per_step : *table)
        for (const auto& per_cta : per_step)
          for (const CtaWait& w : per_cta) {
            uint8_t& p = out[w.exec].publish[w.step];
            p = std::max<uint8_t>(p, w.exec == f ? 1 : 2);
            if (w.value >= 0) out[w.exec].tile_publish[w.step] = 1;
          }
  for (int e = 0; e < E; ++e)
    for (int st = 0; st < (int)layouts[e].steps.size(); ++st) {
      uint8_t& p = out[e].publish[st];
      if (p != 1) continue;
      for (const AbsItem& it : layouts[e].steps[st].items)
        if (!it.dst.ll && (it.dst.multicast || s.home[it.dst.rank][it.dst.buffer] != e)) p = 2;
    }
}

}  // namespace

std::vector<ExecSync> analyze_sync(const Schedule& s, const std::vector<ExecLayout>& layouts,
                                   const LayoutParams& lp) {
  const int E = (int)layouts.size();
  const int G = lp.ctas;
  Index idx;
  for (int e = 0; e < E; ++e)
    for_each_tile_access(s, layouts[e], e, G,
                         [&](int ex, int st, int cta, int r, int b, int64_t lo, int64_t hi, bool w,
                             int o) { idx.add(r, b, Rec{lo, hi, ex, st, cta, w, o}); });
  idx.finish();

  // Tile-granular progress needs every CTA's tiles of a step below the
  // stride T; tagged-line schedules keep their own protocol.
  const bool tiles = lp.tile_sync && !s.ll;
  int T = 1;
  if (tiles)
    for (const auto& L : layouts)
      for (const auto& S : L.steps) {
        std::vector<int> per(G, 0);
        for (const AbsItem& it : S.items)
          for (uint32_t l = 0; l < it.n_tiles; ++l) ++per[tile_cta(it, l, S)];
        for (int c : per) T = std::max(T, c + 1);
      }

  std::vector<ExecSync> out(E);
  for (int f = 0; f < E; ++f) {
    const int nsteps = (int)layouts[f].steps.size();
    out[f].waits.assign(nsteps, std::vector<std::vector<CtaWait>>(G));
    out[f].publish.assign(nsteps, 0);
    out[f].barrier.assign(nsteps, 0);
    out[f].required.assign(nsteps, std::vector<std::vector<CtaWait>>(G));
    out[f].tile_waits.assign(nsteps, std::vector<std::vector<CtaWait>>(G));
    out[f].tile_publish.assign(nsteps, 0);
    out[f].tile_stride = T;
  }
  if (tiles) {
    analyze_tile_sync(s, layouts, idx, G, T, out);
    return out;
  }
  for (int f = 0; f < E; ++f) {
    // need[(step, cta)][(exec, producer cta)] = latest producer step
    std::map<std::pair<int, int>, std::map<std::pair<int, int>, int>> need;
    for_each_tile_access(s, layouts[f], f, G,
                         [&](int, int st, int cta, int r, int b, int64_t lo, int64_t hi, bool w,
                             int) {
                           auto& n = need[{st, cta}];
                           idx.query(r, b, lo, hi, [&](const Rec& p) {
                             if (p.step >= st || (!w && !p.write)) return;
                             // (a CTA's own earlier step counts too: its
                             // publish is the barrier + fence that makes
                             // other threads' writes visible)
                             int& v = n[{p.exec, p.cta}];
                             v = std::max(v, p.step + 1) ;
                           });
                         });
    for (auto& [key, deps] : need) {
      const int st = key.first, cta = key.second;
      std::map<int, std::vector<std::pair<int, int>>> per_exec;  // exec -> (cta, step)
      for (auto& [pk, step1] : deps) {
        if (s.ll && pk.first == f && pk.second == cta) {
          out[f].barrier[st] = 1;  // own earlier tile: a CTA barrier orders it
          continue;
        }
        per_exec[pk.first].push_back({pk.second, step1 - 1});
        out[f].required[st][cta].push_back(CtaWait{pk.first, pk.second, step1 - 1});
      }
      auto& list = out[f].waits[st][cta];
      for (auto& [e, v] : per_exec) {
        if ((int)v.size() * 2 > G) {
          int m = 0;
          for (auto& cs : v) m = std::max(m, cs.second);
          list.push_back(CtaWait{e, -1, m});
          ++out[f].whole;
        } else {
          for (auto& cs : v) {
            list.push_back(CtaWait{e, cs.first, cs.second});
            ++out[f].paired;
          }
        }
      }
    }
  }
  for (int f = 0; f < E; ++f)
    for (const auto& per_step : out[f].waits)
      for (const auto& per_cta : per_step)
        for (const CtaWait& w : per_cta) {
          uint8_t& p = out[w.exec].publish[w.step];
          p = std::max<uint8_t>(p, w.exec == f ? 1 : 2);
        }
  // A local waiter of a step that stored into peer memory (not tagged
  // lines) needs those stores ordered system-wide too.
  for (int e = 0; e < E; ++e)
    for (int st = 0; st < (int)layouts[e].steps.size(); ++st) {
      uint8_t& p = out[e].publish[st];
      if (p != 1) continue;
      for (const AbsItem& it : layouts[e].steps[st].items)
        if (!it.dst.ll && (it.dst.multicast || s.home[it.dst.rank][it.dst.buffer] != e)) p = 2;
    }
  if (s.ll)
    for (int f = 0; f < E; ++f)
      for (const auto& per_step : out[f].waits)
        for (const auto& per_cta : per_step)
          for (const CtaWait& w : per_cta)
            if (w.exec != f)
              throw Error(ErrorCode::DependencyViolation,
                          "ll schedule left a cross-executor edge outside the staging lines");
  return out;
}

void verify_sync(const Schedule& s, const std::vector<ExecLayout>& layouts,
                 const std::vector<ExecSync>& sync, const LayoutParams& lp) {
  // Every pair of conflicting tile accesses at different steps must be
  // ordered: same CTA (program order), or the later CTA waits for the
  // earlier one (explicitly or as part of a whole-executor wait) at a step
  // no earlier than the producer's.
  const int E = (int)layouts.size();
  const int G = lp.ctas;
  std::vector<std::tuple<int, int, int, int, int, int64_t, int64_t, bool, int>> acc;
  for (int e = 0; e < E; ++e)
    for_each_tile_access(s, layouts[e], e, G,
                         [&](int ex, int st, int cta, int r, int b, int64_t lo, int64_t hi, bool w,
                             int o) { acc.emplace_back(ex, st, cta, r, b, lo, hi, w, o); });
  for (const auto& x : acc)
    for (const auto& y : acc) {
      const auto& [ex, sx, cx, rx, bx, lx, hx, wx, ox] = x;
      const auto& [ey, sy, cy, ry, by, ly, hy, wy, oy] = y;
      if (sx >= sy || rx != ry || bx != by || lx >= hy || ly >= hx || (!wx && !wy)) continue;
      bool ok = ex == ey && cx == cy && sync[ey].barrier[sy];
      const int T = sync[ey].tile_stride;
      // the producer tile's progress value (step-level when T == 1)
      const int64_t need = T > 1 ? (int64_t)sx * T + ox + 1 : (int64_t)sx + 1;
      for (const CtaWait& w : sync[ey].waits[sy][cy])
        ok |= w.exec == ex && (w.cta == -1 || w.cta == cx) && w.target(T) >= need;
      if (!sync[ey].tile_waits.empty())
        for (const CtaWait& w : sync[ey].tile_waits[sy][cy])
          ok |= w.exec == ex && w.cta == cx && w.at <= oy && w.target(T) >= need;
      if (!ok)
        throw Error(ErrorCode::DependencyViolation,
                    "tile hazard executor " + std::to_string(ex) + " step " + std::to_string(sx) +
                        " cta " + std::to_string(cx) + " -> executor " + std::to_string(ey) +
                        " step " + std::to_string(sy) + " cta " + std::to_string(cy) +
                        " has no wait");
    }
}

}  // namespace hiccl
