// The machine a plan is lowered for, and the optimization knobs.
//
// A hierarchy is a list of top-down factors of the world size p: depth 0
// is everyone, depth d splits every depth-(d-1) group into hierarchy[d-1]
// contiguous rank blocks, depth L = hierarchy.size() is single ranks.
// `gpus_per_node` (g) says where the "node" boundary sits: it must equal
// the product of some suffix of the factors. On one B200 box every level
// is the same NVSwitch fabric, so a hierarchy only shapes the plan (the
// paper's virtual hierarchies); `transport` is the paper's
// per-level "library" label.
//
// Same group arithmetic as the reference's MachineDescriptor
// (proj/include/hiercoll/machine.hpp:48-89, machine.cpp:50-89) for the
// parts lowering reads; the reference's NIC model belongs to its CPU cost
// simulator and is not on the execution path.
#pragma once

#include <string>
#include <vector>

#include "hiccl/types.hpp"

namespace hiccl {

class MachineDescriptor {
 public:
  MachineDescriptor() = default;
  /// Every level labelled `transport` ("IPC": peer loads/stores over NVLink).
  static MachineDescriptor uniform(std::vector<int> hierarchy, int gpus_per_node,
                                   const std::string& transport = "IPC");

  const std::vector<int>& hierarchy() const { return factors_; }
  int gpus_per_node() const { return node_size_; }
  int element_size() const { return element_size_; }
  const std::string& transport(int level) const { return transport_.at(level); }
  void set_transport(int level, const std::string& t) { transport_.at(level) = t; }

  int world_size() const { return block_.empty() ? 0 : block_[0]; }
  int num_levels() const { return (int)factors_.size(); }
  /// Ranks per group at `depth` (0: everyone, num_levels(): one).
  int group_size(int depth) const;
  int group_index(Rank rank, int depth) const { return rank / group_size(depth); }
  /// Shallowest depth at which a and b sit in different groups
  /// (num_levels() when a == b).
  int crossing_level(Rank a, Rank b) const;
  /// Depth whose groups are the nodes (group size == gpus_per_node).
  int node_depth() const;
  int node_count() const { return world_size() / node_size_; }
  int node_of(Rank r) const { return r / node_size_; }
  /// First depth whose groups hold at most `ranks` ranks (reference
  /// factorize.cpp:317-321: where a ring block's assembly tree starts).
  int depth_of_block(int ranks) const;

  /// Reasons this description cannot serve a p-rank program (empty: ok).
  std::vector<Violation> check(int p) const;

 private:
  std::vector<int> factors_;
  std::vector<int> block_;  // block_[d] = group size at depth d, d = 0..L
  std::vector<std::string> transport_;
  int node_size_ = 1;
  int element_size_ = 4;
};

/// Throws InvalidMachine with the first reason check() reports.
void require_valid_machine(const MachineDescriptor& m, int p);

/// Striping s, ring node count n, pipeline depth m (reference
/// machine.hpp:105-109).
struct OptimizationConfig {
  int stripe = 1;
  int ring = 1;
  int pipeline = 1;
};

/// The reference's limits (machine.cpp:172-194): 1 <= s <= g,
/// 1 <= ring <= node count with ring | node count, m >= 1. Ring blocks
/// that no hierarchy level groups are refused later, by lower(), exactly
/// when a block assembly would drop members (see plan.hpp).
std::vector<Violation> validate_config(const OptimizationConfig& cfg,
                                       const MachineDescriptor& m);
void require_valid_config(const OptimizationConfig& cfg, const MachineDescriptor& m);

}  // namespace hiccl
