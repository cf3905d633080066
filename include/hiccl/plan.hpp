// Point-to-point plans: a program lowered for a machine (striping, ring
// chains, hierarchical trees), put in canonical order with def-use
// dependencies, optionally pipelined over m channels.
// The data contract is the reference factorizer's and pipeliner's
// (proj/include/hiercoll/factorize.hpp:28-113, pipeline.hpp:23-45): plans
// — and therefore the floating-point fold order the executor reproduces —
// match the reference's transfer for transfer, byte for byte when
// serialized.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "hiccl/machine.hpp"
#include "hiccl/program.hpp"

namespace hiccl {

/// One chunk movement (factorize.hpp:33-52). src == dst is a local copy.
/// `reduce` folds into a live accumulator, otherwise overwrite.
struct P2PTransfer {
  int id = -1;
  Rank src = 0, dst = 0;
  std::string src_buffer;
  int64_t src_offset = 0;
  std::string dst_buffer;
  int64_t dst_offset = 0;
  int64_t count = 0;
  bool reduce = false;
  ReduceOp op = ReduceOp::sum;
  int stage = 0;
  int level = 0;
  int stripe = 0;
  int channel = 0;
  int slot = 0;
  int step = 0;
  std::vector<int> deps;

  bool is_local() const { return src == dst; }
};

/// Stage at which a program step begins; `aligned` iff every dependency
/// crossing it connects identical ranges (factorize.hpp:58-61).
struct FenceBoundary {
  int stage = 0;
  bool aligned = true;
};

struct StagedPlan {
  int world_size = 0;
  int element_size = 4;
  int stripe = 1;
  int ring = 1;
  int num_stages = 0;
  std::string source_program_id;
  std::map<std::string, BufferDecl> buffers;
  std::vector<FenceBoundary> fences;
  std::vector<P2PTransfer> transfers;

  int64_t total_bytes() const;
  std::string serialize() const;
  static StagedPlan deserialize(const std::string& text);
};

/// Overlapped schedule (pipeline.hpp:31-38): every transfer replicated on
/// `depth` channels, channel c at slot stage + c.
struct PipelinedPlan {
  StagedPlan base;
  int depth = 1;
  int slots = 0;

  std::string serialize() const;
  static PipelinedPlan deserialize(const std::string& text);
};

/// validate -> stripe -> per-step ring/tree lowering -> fence offsets ->
/// stage compaction -> canonical ids -> deps (factorize.cpp:587-662).
/// Throws InvalidConfig where the reference would silently drop members
/// (a ring block that no hierarchy level below the root groups).
StagedPlan lower(const CollectiveProgram& program, const MachineDescriptor& machine,
                 const OptimizationConfig& config);

/// pipeline.cpp:76-132
PipelinedPlan pipeline(const StagedPlan& plan, int depth);

/// p x p bytes at `slot` (pipeline.cpp:134-145).
std::vector<std::vector<int64_t>> comm_matrix(const PipelinedPlan& plan, int slot);

/// Bytes moved between different blocks of node_size ranks (factorize.cpp:670-676).
int64_t inter_node_bytes(const StagedPlan& plan, int node_size);

}  // namespace hiccl
