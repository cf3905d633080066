// Factorizer: composed primitives -> point-to-point transfers for a
// machine hierarchy. The rules are the reference's (proj/src/factorize.cpp:
// 62-662, restated in SURVEY.md Appendix A) because the plan fixes the
// fold order the executor reproduces bit for bit; the construction here
// is organised around one object, the hierarchical spanning tree.
//
// Spanning tree. From an anchor rank and a sorted member set, at depth d
// the members outside the anchor's depth-d group fall into runs of equal
// group; each run's representative (run[lane % |run|], lane = the
// primitive's stripe) is one hop from the anchor and anchors the rest of
// its run from depth d+1; the run holding the anchor continues from d+1
// with the same anchor. A multicast sends data down the hops (stage
// d-1); a reduction folds it up the hops (stage L-d), a representative
// with followers ("relay") first folding its own contribution and theirs
// into a per-primitive scratch accumulator. Ring chains (ring > 1) link
// the representatives of the ring's blocks and hang one tree per block.
#include <algorithm>
#include <array>
#include <set>

#include "planning.hpp"

namespace hiccl {

namespace {

// FNV-1a of "<step>|<kind>|<root>|<send buf>:<off>+<count>|<recv buf>:<off>
// |<op>|<root participates>,<leaf>,..." — the key the reference names
// staging and scratch buffers with (factorize.cpp:45-57).
std::string fingerprint(int step, const Primitive& p) {
  std::string key;
  key.reserve(96);
  key += std::to_string(step) + '|' + to_string(p.kind) + '|' + std::to_string(p.root) + '|';
  key += p.send.buffer + ':' + std::to_string(p.send.offset) + '+' + std::to_string(p.send.count);
  key += '|' + p.recv.buffer + ':' + std::to_string(p.recv.offset);
  key += '|' + std::to_string((int)p.op) + '|' + (p.root_participates ? '1' : '0');
  for (Rank r : p.leaves) key += ',' + std::to_string(r);
  return hex16(fnv1a64(key));
}

struct Hop {
  Rank near;    // already holds the data (multicast) / collects it (reduction)
  Rank far;     // representative of a group `near` is not in
  int depth;    // tree depth of the hop
  bool relays;  // `far` anchors followers of its own
};

std::vector<Hop> spanning_tree(const MachineDescriptor& m, int lane, Rank anchor,
                               std::vector<Rank> members, int depth) {
  struct Pending {
    Rank anchor;
    std::vector<Rank> members;
    int depth;
  };
  std::vector<Hop> hops;
  std::vector<Pending> work;
  work.push_back({anchor, std::move(members), depth});
  while (!work.empty()) {
    Pending job = std::move(work.back());
    work.pop_back();
    if (job.members.empty() || job.depth > m.num_levels()) continue;
    const int span = m.group_size(job.depth);
    const int home = job.anchor / span;
    auto it = job.members.begin();
    while (it != job.members.end()) {
      const int group = *it / span;
      const auto end = std::find_if(it, job.members.end(), [&](Rank r) { return r / span != group; });
      std::vector<Rank> run(it, end);
      it = end;
      if (group == home) {
        work.push_back({job.anchor, std::move(run), job.depth + 1});
        continue;
      }
      const Rank rep = run[lane % run.size()];
      hops.push_back({job.anchor, rep, job.depth, run.size() > 1});
      run.erase(std::find(run.begin(), run.end(), rep));
      work.push_back({rep, std::move(run), job.depth + 1});
    }
  }
  return hops;
}

struct Loc {
  std::string buffer;
  int64_t offset = 0;
};

// One primitive's transfers, stages relative to the primitive.
class PrimitiveLowering {
 public:
  PrimitiveLowering(const Primitive& p, const MachineDescriptor& m, int ring, std::string scratch)
      : p_(p), m_(m), L_(m.num_levels()), ring_(ring), lane_(p.stripe),
        send_{p.send.buffer, p.send.offset}, recv_{p.recv.buffer, p.recv.offset},
        scratch_{std::move(scratch), 0} {}

  std::vector<P2PTransfer> run() {
    if (p_.kind == PrimitiveKind::multicast)
      multicast();
    else
      reduction();
    initialize_accumulators();
    densify_stages();
    return std::move(out_);
  }
  bool scratch_used() const { return scratch_used_; }

 private:
  void add(Rank src, const Loc& from, Rank dst, const Loc& to, bool reduce, int stage) {
    P2PTransfer t;
    t.src = src;
    t.dst = dst;
    t.src_buffer = from.buffer;
    t.src_offset = from.offset;
    t.dst_buffer = to.buffer;
    t.dst_offset = to.offset;
    t.count = p_.recv.count;
    t.reduce = reduce;
    t.op = p_.op;
    t.stage = stage;
    t.level = src == dst ? L_ : m_.crossing_level(src, dst);
    t.stripe = lane_;
    out_.push_back(std::move(t));
  }

  // Ring blocks (p / ring ranks each), the root's first, then every block
  // holding members in wrap-around order (factorize.cpp:302-315); empty
  // when the members all sit in the root's block or there is no ring.
  std::vector<std::vector<Rank>> ring_blocks(const std::vector<Rank>& members) const {
    if (ring_ <= 1 || members.empty()) return {};
    const int size = m_.world_size() / ring_;
    const int home = p_.root / size;
    std::vector<std::vector<Rank>> by_block(ring_);
    for (Rank r : members) by_block[r / size].push_back(r);
    if (by_block[home].size() == members.size()) return {};
    std::vector<std::vector<Rank>> chain;
    for (int i = 0; i < ring_; ++i) {
      auto& b = by_block[(home + i) % ring_];
      if (i == 0 || !b.empty()) chain.push_back(std::move(b));
    }
    return chain;
  }

  // Depth below which a ring block assembles. A block is assembled by a
  // tree from its representative over the others (block 0: the root,
  // which is no member); when that tree would start past the last level
  // the reference silently loses those members — refuse instead.
  int block_depth(const std::vector<std::vector<Rank>>& chain) const {
    const int bd = m_.depth_of_block(m_.world_size() / ring_);
    bool stranded = bd + 1 > L_ && !chain[0].empty();
    for (size_t i = 1; i < chain.size(); ++i) stranded |= bd + 1 > L_ && chain[i].size() > 1;
    if (stranded)
      throw Error(ErrorCode::InvalidConfig,
                  "ring blocks of " + std::to_string(m_.world_size() / ring_) +
                      " ranks are no group of the hierarchy: assembling them would "
                      "drop members");
    return bd;
  }

  static std::vector<Rank> without(const std::vector<Rank>& v, Rank r) {
    std::vector<Rank> out;
    for (Rank x : v)
      if (x != r) out.push_back(x);
    return out;
  }

  // ---- multicast: data flows down the hops ----
  void multicast() {
    if (p_.root_participates && !p_.in_place()) add(p_.root, send_, p_.root, recv_, false, 0);
    if (p_.leaves.empty()) return;
    const auto chain = ring_blocks(p_.leaves);
    if (chain.empty()) {
      for (const Hop& h : spanning_tree(m_, lane_, p_.root, p_.leaves, 1))
        add(h.near, h.near == p_.root ? send_ : recv_, h.far, recv_, false, h.depth - 1);
      return;
    }
    // chain hops rep[i-1] -> rep[i] at stage i-1, then every block's tree
    const int len = (int)chain.size();
    const int bd = block_depth(chain);
    std::vector<Rank> rep{p_.root};
    for (int i = 1; i < len; ++i) {
      rep.push_back(chain[i][lane_ % chain[i].size()]);
      add(rep[i - 1], i == 1 ? send_ : recv_, rep[i], recv_, false, i - 1);
    }
    for (int i = 0; i < len; ++i) {
      const Loc& origin = i == 0 ? send_ : recv_;
      for (const Hop& h : spanning_tree(m_, lane_, rep[i], without(chain[i], rep[i]), bd + 1))
        add(h.near, h.near == rep[i] ? origin : recv_, h.far, recv_, false,
            (len - 1) + (h.depth - bd - 1));
    }
  }

  // ---- reduction: data folds up the hops ----
  void fold_tree(Rank collector, const Loc& into, const std::vector<Rank>& members, int depth) {
    for (const Hop& h : spanning_tree(m_, lane_, collector, members, depth)) {
      add(h.far, h.relays ? scratch_ : send_, h.near, h.near == collector ? into : scratch_, true,
          L_ - h.depth);
      if (h.relays) seed_scratch(h.far);
    }
  }

  void seed_scratch(Rank r) {
    scratch_used_ = true;
    add(r, send_, r, scratch_, true, 0);
  }

  void reduction() {
    const auto chain = ring_blocks(p_.leaves);
    if (chain.empty()) {
      fold_tree(p_.root, recv_, p_.leaves, 1);
    } else {
      const int len = (int)chain.size();
      const int bd = block_depth(chain);
      std::vector<Rank> rep{p_.root};
      std::vector<Loc> acc{recv_};
      fold_tree(p_.root, recv_, chain[0], bd + 1);  // the root is no leaf
      for (int i = 1; i < len; ++i) {
        rep.push_back(chain[i][lane_ % chain[i].size()]);
        if (i == len - 1 && chain[i].size() == 1) {  // lone chain end forwards its send
          acc.push_back(send_);
          continue;
        }
        acc.push_back(scratch_);
        seed_scratch(rep[i]);
        fold_tree(rep[i], scratch_, without(chain[i], rep[i]), bd + 1);
      }
      // hops toward the root, farthest block first
      for (int j = len - 2; j >= 0; --j)
        add(rep[j + 1], acc[j + 1], rep[j], acc[j], true, (L_ - bd) + (len - 2 - j));
    }
    if (p_.root_participates && !p_.in_place()) add(p_.root, send_, p_.root, recv_, true, 0);
  }

  // Every accumulator (rank, buffer) a reduction folds into is
  // initialized by its first writer in (stage, src, src buffer, src
  // offset) order, which becomes a plain copy — unless the root reduces
  // in place, its recv already holding its own contribution
  // (factorize.cpp:323-335).
  void initialize_accumulators() {
    const bool preinit = p_.kind == PrimitiveKind::reduction && p_.root_participates &&
                         p_.in_place();
    std::map<std::pair<Rank, std::string>, size_t> first;
    for (size_t k = 0; k < out_.size(); ++k) {
      const P2PTransfer& t = out_[k];
      if (!t.reduce) continue;
      if (preinit && t.dst == p_.root && t.dst_buffer == p_.recv.buffer) continue;
      auto [it, fresh] = first.try_emplace({t.dst, t.dst_buffer}, k);
      const P2PTransfer& best = out_[it->second];
      if (!fresh && std::tie(t.stage, t.src, t.src_buffer, t.src_offset) <
                        std::tie(best.stage, best.src, best.src_buffer, best.src_offset))
        it->second = k;
    }
    for (const auto& [key, k] : first) out_[k].reduce = false;
  }

  void densify_stages() {
    std::set<int> used;
    for (const auto& t : out_) used.insert(t.stage);
    std::vector<int> ranks(used.begin(), used.end());
    for (auto& t : out_)
      t.stage = (int)(std::lower_bound(ranks.begin(), ranks.end(), t.stage) - ranks.begin());
  }

  const Primitive& p_;
  const MachineDescriptor& m_;
  const int L_, ring_, lane_;
  const Loc send_, recv_, scratch_;
  bool scratch_used_ = false;
  std::vector<P2PTransfer> out_;
};

BufferRef part_of(const BufferRef& r, const SplitRange& s) {
  return BufferRef{r.buffer, r.offset + s.offset, s.count};
}

Primitive make(PrimitiveKind kind, Rank root, std::vector<Rank> leaves, BufferRef send,
               BufferRef recv, ReduceOp op, int lane) {
  Primitive p;
  p.kind = kind;
  p.root = root;
  p.leaves = std::move(leaves);
  p.send = std::move(send);
  p.recv = std::move(recv);
  p.op = op;
  p.stripe = lane;
  return p;
}

// Striping (factorize.cpp:451-585): a primitive whose leaves leave the
// root's node is cut into s balanced chunks; chunk c travels through
// lane root q_c (the root, then the lowest other GPUs of its node). The
// intra-node part (root -> q_c scatter, or the per-lane partial
// reductions) goes before an inserted fence, the cross-node part (q_c's
// multicast, or the gather of the partials to the root) after it.
CollectiveProgram stripe(const CollectiveProgram& program, const MachineDescriptor& m, int s) {
  CollectiveProgram out(program.world_size());
  for (const auto& [name, d] : program.buffers())
    out.declare_buffer(name, d.length, d.input, d.internal);
  const int g = m.gpus_per_node();
  bool any = false;
  auto emit = [&](std::vector<Primitive>& prims) {
    if (prims.empty()) return;
    if (any) out.add_fence();
    any = true;
    for (Primitive& p : prims) out.append_primitive(std::move(p));
  };

  const auto& steps = program.steps();
  for (int si = 0; si < (int)steps.size(); ++si) {
    std::vector<Primitive> intra, cross;
    for (const Primitive& prim : steps[si]) {
      const int node = m.node_of(prim.root);
      const bool leaves_node = std::any_of(prim.leaves.begin(), prim.leaves.end(),
                                           [&](Rank r) { return m.node_of(r) != node; });
      if (!leaves_node) {
        intra.push_back(prim);
        continue;
      }
      std::vector<Rank> lane_root{prim.root};
      for (Rank r = node * g; r < (node + 1) * g && (int)lane_root.size() < s; ++r)
        if (r != prim.root) lane_root.push_back(r);
      const std::string staging = "__stage." + fingerprint(si, prim);
      auto staged = [&](const SplitRange& part) {
        return BufferRef{staging, part.offset, part.count};
      };
      bool staging_used = false;
      const bool mc = prim.kind == PrimitiveKind::multicast;
      if (mc && prim.root_participates && !prim.in_place()) {
        Primitive self = make(PrimitiveKind::multicast, prim.root, {}, prim.send, prim.recv,
                              ReduceOp::sum, 0);
        self.root_participates = true;
        intra.push_back(std::move(self));
      }
      std::vector<Rank> contributors = prim.leaves;  // reductions: everyone folding in
      if (!mc && prim.root_participates)
        contributors.insert(std::upper_bound(contributors.begin(), contributors.end(), prim.root),
                            prim.root);
      for (int c = 0; c < s; ++c) {
        const SplitRange part = balanced_split(prim.send.count, s, c);
        if (part.count == 0) continue;
        const Rank q = lane_root[c];
        if (mc) {
          const bool q_is_leaf = std::binary_search(prim.leaves.begin(), prim.leaves.end(), q);
          const BufferRef landing = q_is_leaf ? part_of(prim.recv, part) : staged(part);
          staging_used |= !q_is_leaf;
          if (c > 0)  // the root hands chunk c to its lane root: a one-leaf reduction (a copy)
            intra.push_back(make(PrimitiveKind::reduction, q, {prim.root},
                                 part_of(prim.send, part), landing, prim.op, c));
          std::vector<Rank> rest;
          for (Rank l : prim.leaves)
            if (l != q) rest.push_back(l);
          if (!rest.empty())
            cross.push_back(make(PrimitiveKind::multicast, q, std::move(rest),
                                 c == 0 ? part_of(prim.send, part) : landing,
                                 part_of(prim.recv, part), ReduceOp::sum, c));
        } else {
          std::vector<Rank> others;
          for (Rank r : contributors)
            if (r != q) others.push_back(r);
          Primitive partial = make(PrimitiveKind::reduction, q, std::move(others),
                                   part_of(prim.send, part),
                                   c == 0 ? part_of(prim.recv, part) : staged(part), prim.op, c);
          partial.root_participates =
              std::binary_search(contributors.begin(), contributors.end(), q);
          intra.push_back(std::move(partial));
          if (c > 0) {
            staging_used = true;
            cross.push_back(make(PrimitiveKind::reduction, prim.root, {q}, staged(part),
                                 part_of(prim.recv, part), prim.op, c));
          }
        }
      }
      if (staging_used) out.declare_buffer(staging, prim.recv.count, false, true);
    }
    emit(intra);
    emit(cross);
  }
  return out;
}

}  // namespace

// A primitive whose participating root reads its send range and writes an
// overlapping but different recv range of the same buffer (a shifted
// in-place copy or reduction) passes the reference's validate(), but its
// lowering reads the send range while the root's own recv writes are
// landing, in whatever order the stages give: the reference's symbolic
// oracle rejects such plans (tests/test_random_programs.py). Refused.
static void refuse_shifted_self_overlap(const CollectiveProgram& program) {
  for (const auto& step : program.steps())
    for (const Primitive& p : step)
      if (p.root_participates && p.send.overlaps(p.recv) && !p.in_place())
        throw Error(ErrorCode::ReadWriteRace,
                    "primitive rooted at " + std::to_string(p.root) + " reads '" + p.send.buffer +
                        "'[" + std::to_string(p.send.offset) + ", " + std::to_string(p.send.end()) +
                        ") and writes the overlapping, shifted [" + std::to_string(p.recv.offset) +
                        ", " + std::to_string(p.recv.end()) + ") on the same rank");
}

StagedPlan lower(const CollectiveProgram& program, const MachineDescriptor& machine,
                 const OptimizationConfig& config) {
  if (const auto v = program.validate(); !v.empty())
    throw Error(v.front().code, "program invalid: " + v.front().message);
  refuse_shifted_self_overlap(program);
  require_valid_machine(machine, program.world_size());
  require_valid_config(config, machine);

  const CollectiveProgram striped =
      config.stripe > 1 ? stripe(program, machine, config.stripe) : program;

  StagedPlan plan;
  plan.world_size = striped.world_size();
  plan.element_size = machine.element_size();
  plan.stripe = config.stripe;
  plan.ring = config.ring;
  plan.source_program_id = program.id();
  plan.buffers = striped.buffers();

  // Steps run back to back: a step's transfers start where the previous
  // step's longest primitive ended; a fence sits at every step boundary.
  std::vector<P2PTransfer> all;
  std::vector<int> boundary;
  int next = 0;
  const auto& steps = striped.steps();
  for (int si = 0; si < (int)steps.size(); ++si) {
    int width = 0;
    for (const Primitive& prim : steps[si]) {
      const std::string scratch = "__acc." + fingerprint(si, prim);
      PrimitiveLowering lowering(prim, machine, config.ring, scratch);
      for (P2PTransfer& t : lowering.run()) {
        width = std::max(width, t.stage + 1);
        t.stage += next;
        t.step = si;
        all.push_back(std::move(t));
      }
      if (lowering.scratch_used())
        plan.buffers[scratch] = BufferDecl{prim.recv.count, false, true};
    }
    next += width;
    if (si + 1 < (int)steps.size()) boundary.push_back(next);
  }

  // Renumber the occupied stages densely; a fence keeps its place unless
  // it would open the plan, close it, or repeat the previous fence.
  std::vector<int> occupied;
  for (const auto& t : all) occupied.push_back(t.stage);
  std::sort(occupied.begin(), occupied.end());
  occupied.erase(std::unique(occupied.begin(), occupied.end()), occupied.end());
  auto dense = [&](int stage) {
    return (int)(std::lower_bound(occupied.begin(), occupied.end(), stage) - occupied.begin());
  };
  for (auto& t : all) t.stage = dense(t.stage);
  for (int b : boundary) {
    const int st = dense(b);
    if (st > 0 && st < (int)occupied.size() && (plan.fences.empty() || plan.fences.back().stage != st))
      plan.fences.push_back(FenceBoundary{st, true});
  }
  plan.num_stages = (int)occupied.size();

  sort_canonical(all, Clock::stage);
  for (auto& t : all) t.slot = t.stage;
  link_dependencies(all, Clock::stage, &plan.fences);
  plan.transfers = std::move(all);
  return plan;
}

}  // namespace hiccl
