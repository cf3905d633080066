// Machine description and optimization knobs (reference:
// proj/include/hiercoll/machine.hpp:25-114). The hierarchy vector holds
// top-down integer factors of p; contiguous rank blocks form the groups
// of each level. On the B200 box every level is the same NVSwitch fabric:
// the hierarchy shapes the plan ("virtual hierarchy"),
// `transport` labels which executor lowering a level uses.
#pragma once

#include <string>
#include <utility>
#include <vector>

#include "hiccl/types.hpp"

namespace hiccl {

enum class Binding : uint8_t { packed = 0, round_robin = 1, bijective = 2 };
std::string to_string(Binding b);
Binding binding_from_string(const std::string& s);

/// Per-level link parameters (machine.hpp:35-39). `transport` is the
/// paper's per-level "library": "IPC" (peer loads/stores
/// over NVLink, the default), "NVLS" (reserved for multimem lowering).
struct LevelLink {
  double alpha = 0.0;
  double bandwidth = 0.0;
  std::string transport;
};

struct MachineDescriptor {
  std::vector<int> hierarchy;
  std::vector<LevelLink> levels;
  int gpus_per_node = 1;
  int nics_per_node = 1;
  double nic_bandwidth = 0.0;
  Binding binding = Binding::packed;
  int element_size = 4;

  int world_size() const;
  int num_levels() const { return (int)hierarchy.size(); }
  /// Group size at depth (0 = everyone, num_levels() = singleton).
  int group_size(int depth) const;
  int group_index(Rank rank, int depth) const;
  std::pair<Rank, Rank> group_span(Rank rank, int depth) const;
  /// Shallowest depth separating a and b; num_levels() when a == b.
  int crossing_level(Rank a, Rank b) const;
  int node_depth() const;
  int node_count() const { return world_size() / gpus_per_node; }
  int node_of(Rank r) const { return r / gpus_per_node; }
  Rank local_rank(Rank r) const { return r % gpus_per_node; }
  bool level_crosses_nodes(int level) const { return level <= node_depth(); }
  int nic_of(Rank rank) const;

  std::string serialize() const;
  static MachineDescriptor deserialize(const std::string& text);
  static MachineDescriptor load(const std::string& path);

  /// Uniform description used by tests and the presets: every level
  /// gets (alpha, bandwidth, transport); one NIC per node at 25 GB/s
  /// (same fixture as the reference's tests/test_common.hpp:25-38).
  static MachineDescriptor uniform(std::vector<int> hierarchy, int gpus_per_node,
                                   const std::string& transport = "IPC",
                                   double alpha = 1e-6, double bandwidth = 100e9);
};

std::vector<Violation> validate_machine(const MachineDescriptor& m, int p);
void require_valid_machine(const MachineDescriptor& m, int p);

struct GroupInfo {
  int id;
  std::vector<Rank> members;
};
GroupInfo group_of(Rank rank, int depth, const MachineDescriptor& m);

/// Striping s, ring node count n, pipeline depth m (machine.hpp:105-109).
struct OptimizationConfig {
  int stripe = 1;
  int ring = 1;
  int pipeline = 1;
};

/// The reference's rules (machine.cpp:172-194). Ring blocks that no
/// hierarchy level groups are caught later, by lower(), exactly when a
/// block assembly would drop members (see plan.hpp).
std::vector<Violation> validate_config(const OptimizationConfig& cfg,
                                       const MachineDescriptor& m);
void require_valid_config(const OptimizationConfig& cfg, const MachineDescriptor& m);

/// Depth of the first hierarchy level whose groups hold at most
/// `block_size` ranks (reference factorize.cpp:317-321).
int depth_of_block(const MachineDescriptor& m, int block_size);

}  // namespace hiccl
