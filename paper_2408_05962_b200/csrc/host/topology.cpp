// Hierarchy arithmetic: group sizes are precomputed once per description
// (block_[d] = ranks per depth-d group), so every query the factorizer
// makes — group of a rank, level at which two ranks part, node depth — is
// a division against that table.
#include "hiccl/machine.hpp"

namespace hiccl {

namespace {
Violation machine_problem(std::string why) {
  Violation v;
  v.code = ErrorCode::InvalidMachine;
  v.message = std::move(why);
  return v;
}
}  // namespace

MachineDescriptor MachineDescriptor::uniform(std::vector<int> hierarchy, int gpus_per_node,
                                             const std::string& transport) {
  MachineDescriptor m;
  m.factors_ = std::move(hierarchy);
  m.transport_.assign(m.factors_.size(), transport);
  m.node_size_ = gpus_per_node;
  // block sizes top-down; a non-positive factor leaves the table short
  // and check() reports it
  int64_t ranks = 1;
  for (int f : m.factors_) ranks *= f > 0 ? f : 1;
  m.block_.push_back((int)ranks);
  for (int f : m.factors_) {
    if (f < 1) break;
    m.block_.push_back(m.block_.back() / f);
  }
  return m;
}

int MachineDescriptor::group_size(int depth) const {
  if (depth < 0 || depth >= (int)block_.size())
    throw Error(ErrorCode::InvalidMachine,
                "no hierarchy depth " + std::to_string(depth) + " in a " +
                    std::to_string(num_levels()) + "-level machine");
  return block_[depth];
}

int MachineDescriptor::crossing_level(Rank a, Rank b) const {
  const int L = num_levels();
  for (int d = 1; d <= L; ++d)
    if (a / block_[d] != b / block_[d]) return d;
  return L;
}

int MachineDescriptor::node_depth() const {
  for (int d = (int)block_.size() - 1; d >= 0; --d)
    if (block_[d] == node_size_) return d;
  throw Error(ErrorCode::InvalidMachine, "node size " + std::to_string(node_size_) +
                                             " is no group size of the hierarchy");
}

int MachineDescriptor::depth_of_block(int ranks) const {
  int d = 0;
  while (d < num_levels() && block_[d] > ranks) ++d;
  return d;
}

std::vector<Violation> MachineDescriptor::check(int p) const {
  std::vector<Violation> out;
  if (factors_.empty()) {
    out.push_back(machine_problem("the hierarchy has no levels"));
    return out;
  }
  bool factors_ok = true;
  for (size_t i = 0; i < factors_.size(); ++i)
    if (factors_[i] < 1) {
      out.push_back(machine_problem("level " + std::to_string(i + 1) + " has factor " +
                                    std::to_string(factors_[i])));
      factors_ok = false;
    }
  if (factors_ok && world_size() != p)
    out.push_back(machine_problem("the hierarchy spans " + std::to_string(world_size()) +
                                  " ranks, the program " + std::to_string(p)));
  if (transport_.size() != factors_.size())
    out.push_back(machine_problem("one transport label per level is required"));
  if (element_size_ < 1) out.push_back(machine_problem("element size must be positive"));
  if (node_size_ < 1) {
    out.push_back(machine_problem("gpus_per_node must be positive"));
  } else if (factors_ok) {
    if (world_size() % node_size_ != 0) {
      out.push_back(machine_problem(std::to_string(node_size_) + " GPUs per node do not divide " +
                                    std::to_string(world_size()) + " ranks"));
    } else {
      bool is_group = false;
      for (int b : block_) is_group |= b == node_size_;
      if (!is_group)
        out.push_back(machine_problem("no trailing product of the hierarchy equals " +
                                      std::to_string(node_size_) + " GPUs per node"));
    }
  }
  return out;
}

void require_valid_machine(const MachineDescriptor& m, int p) {
  const auto v = m.check(p);
  if (!v.empty()) throw Error(ErrorCode::InvalidMachine, v.front().message);
}

std::vector<Violation> validate_config(const OptimizationConfig& cfg,
                                       const MachineDescriptor& m) {
  std::vector<Violation> out;
  auto refuse = [&out](std::string why) {
    Violation v;
    v.code = ErrorCode::InvalidConfig;
    v.message = std::move(why);
    out.push_back(std::move(v));
  };
  const int g = m.gpus_per_node(), nodes = m.node_count();
  if (cfg.stripe < 1 || cfg.stripe > g)
    refuse("stripe count " + std::to_string(cfg.stripe) + " outside [1, " + std::to_string(g) +
           "] (GPUs per node)");
  if (cfg.ring < 1 || cfg.ring > nodes)
    refuse("ring of " + std::to_string(cfg.ring) + " outside [1, " + std::to_string(nodes) +
           "] (nodes)");
  else if (nodes % cfg.ring != 0)
    refuse("ring of " + std::to_string(cfg.ring) + " does not split " + std::to_string(nodes) +
           " nodes evenly");
  if (cfg.pipeline < 1) refuse("pipeline depth " + std::to_string(cfg.pipeline) + " < 1");
  return out;
}

void require_valid_config(const OptimizationConfig& cfg, const MachineDescriptor& m) {
  const auto v = validate_config(cfg, m);
  if (!v.empty()) throw Error(ErrorCode::InvalidConfig, v.front().message);
}

}  // namespace hiccl
