// Point-to-point plans: what a program becomes once lowered for a machine
// (striping, ring chains, hierarchical trees), put in canonical order with
// its def-use edges, and optionally pipelined over m channels.
//
// The fields and their meaning are the reference factorizer's and
// pipeliner's data contract (proj/include/hiercoll/factorize.hpp:28-113,
// pipeline.hpp:23-45): a plan here equals the reference's transfer for
// transfer — serialized, byte for byte — which is what fixes the
// floating-point fold order the device executor reproduces.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "hiccl/machine.hpp"
#include "hiccl/program.hpp"

namespace hiccl {

// One chunk moving from (src, src_buffer, src_offset) to (dst, dst_buffer,
// dst_offset), `count` elements; overwrites, or folds into the live
// destination with `op` when `reduce` (factorize.hpp:33-52).
struct P2PTransfer {
  int id = -1;  // position in the canonical order
  Rank src = 0, dst = 0;  // equal: a copy on one rank
  std::string src_buffer, dst_buffer;
  int64_t src_offset = 0, dst_offset = 0, count = 0;
  bool reduce = false;
  ReduceOp op = ReduceOp::sum;
  int stage = 0, level = 0, stripe = 0;  // where lowering put it
  int channel = 0, slot = 0;             // pipelining: channel c runs at slot stage + c
  int step = 0;                          // the program step it lowers
  std::vector<int> deps;                 // ids it reads after (read-after-write edges)

  bool is_local() const { return src == dst; }
};

// First stage of a program step. `aligned`: every dependency across it
// joins identical ranges, so pipelining may overlap the steps on either
// side; otherwise the pipeline drains there (factorize.hpp:58-61).
struct FenceBoundary {
  int stage = 0;
  bool aligned = true;
};

// The lowered transfer DAG with its buffers and fences.
struct StagedPlan {
  int world_size = 0, element_size = 4;
  int stripe = 1, ring = 1;  // the knobs it was lowered with
  int num_stages = 0;
  std::string source_program_id;
  std::map<std::string, BufferDecl> buffers;
  std::vector<FenceBoundary> fences;
  std::vector<P2PTransfer> transfers;

  int64_t total_bytes() const;
  std::string serialize() const;
  static StagedPlan deserialize(const std::string& text);
};

// The overlapped schedule (pipeline.hpp:31-38): each transfer cut into
// `depth` balanced channels, channel c at slot stage + c.
struct PipelinedPlan {
  StagedPlan base;
  int depth = 1;
  int slots = 0;

  std::string serialize() const;
  static PipelinedPlan deserialize(const std::string& text);
};

// validate, stripe, lower each step's primitives (ring chains, trees),
// offset by fences, compact stages, canonical ids, dependency edges
// (factorize.cpp:587-662). Refuses with InvalidConfig the plans the
// reference would lower wrongly: ring blocks no hierarchy level below the
// root groups (members would be dropped), shifted self-overlapping
// primitives, pipelined writes reordered across aligned fences.
StagedPlan lower(const CollectiveProgram& program, const MachineDescriptor& machine,
                 const OptimizationConfig& config);

PipelinedPlan pipeline(const StagedPlan& plan, int depth);  // pipeline.cpp:76-132

// Bytes rank i sends rank j at `slot`, p x p (pipeline.cpp:134-145).
std::vector<std::vector<int64_t>> comm_matrix(const PipelinedPlan& plan, int slot);

// Bytes crossing between blocks of node_size consecutive ranks
// (factorize.cpp:670-676).
int64_t inter_node_bytes(const StagedPlan& plan, int node_size);

}  // namespace hiccl
