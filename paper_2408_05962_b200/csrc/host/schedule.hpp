// Plan -> executor schedule.
//
// The reference executor (engine.cpp:285-330) applies transfers one at a
// time in (slot, id) order. The device executor runs a slot's transfers
// concurrently, so this pass derives from the pipelined plan everything
// the concurrent execution needs to give bit-identical results:
//
//  * write groups — every slot's writes are cut into maximal segments of
//    a destination buffer covered by the same set of transfers; a
//    segment's contributors, in id order (the copy, if any, first — it is
//    the lowest id because slot_less orders copies before reduces,
//    pipeline.cpp:30-35), become ONE fused item: acc = first source (or
//    the live destination), then fold every later source in id order,
//    one store. That is exactly the reference's sequence of folds.
//  * phases — if a slot ever reads what the same slot writes (never seen
//    in the reference's plans, checked here anyway), the later item moves
//    to a later phase of the slot so the sequential order is kept.
//  * waits — cross-step RAW, WAR and WAW hazards between items become
//    "executor X finished step s" edges, realized on the device as
//    epoch-tagged flag words written with release semantics (fences as
//    flags, not host synchronization).
//
// Pure host code: no CUDA headers, so the CPU tests exercise it directly.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hiccl/plan.hpp"

namespace hiccl {

struct Loc {
  int rank = 0;
  int buffer = 0;  // index into Schedule::buffer_names
  int64_t offset = 0;
};

struct WorkItem {
  int step = 0;            // global (slot, phase) step
  int exec = 0;            // executor that runs it
  Loc dst;
  int64_t count = 0;
  ReduceOp op = ReduceOp::sum;
  bool reads_dst = false;  // accumulate onto the live destination first
  std::vector<Loc> srcs;   // fold order; when reads_dst, srcs[0] == dst
  std::vector<int> transfer_ids;  // contributors (debug / tests)
  // Range that decides the tile -> CTA assignment (layout.cpp); -1: dst.
  // A staging copy tiles like the fold that consumes it.
  int64_t tile_key = -1;
  bool staging = false;  // a push into the destination's staging (CopyMode::staged)
};

struct StepWait {
  int exec;  // wait until this executor ...
  int step;  // ... has finished this global step
};

struct ExecProgram {
  std::vector<std::vector<int>> items_by_step;  // item indices per global step
  std::vector<std::vector<StepWait>> waits;     // per global step (deduplicated)
  std::vector<bool> publish;                    // someone waits on this step
};

struct Schedule {
  int world_size = 0;
  int num_execs = 1;
  std::vector<int> rank_to_exec;
  std::vector<std::string> buffer_names;  // plan map order
  std::vector<BufferDecl> buffer_decls;
  std::vector<int> step_slot;   // global step -> slot
  std::vector<int> step_phase;  // global step -> phase within slot
  std::vector<WorkItem> items;
  std::vector<ExecProgram> execs;
  int max_sources = 0;
  int max_phases = 1;
  int staging_buffer = -1;  // index of the synthetic "__hiccl.staging" buffer (staged / ll)
  bool ll = false;          // staging holds tagged lines (CopyMode::ll)
  int64_t ll_half = 0;      // ll: byte distance between the two arena copies

  // Executor whose memory holds (rank, buffer): rank_to_exec[rank] for user
  // buffers; internal buffers may live with their only reader (push).
  std::vector<std::vector<int>> home;  // [rank][buffer]
  // Internal-buffer arena layout: byte offset of (rank, buffer) inside
  // the arena of home[rank][buffer]; -1 when that rank never touches it.
  std::vector<std::vector<int64_t>> arena_offset;  // [rank][buffer]
  std::vector<int64_t> arena_bytes;                // [exec]
  std::vector<std::vector<int64_t>> extent;        // [rank][buffer] elements touched
};

// pull: copies run on the destination's executor; push: on the source's;
// staged: push, and every remote source of a reduction is first pushed
// into a staging range on the destination, which then folds locally in
// the plan's order (all cross-GPU traffic becomes stores).
// ll (low latency): every remote source, copies included, is pushed into
// staging as tagged lines (8 payload bytes + the launch tag per 16-byte
// store); the consumer polls the tags instead of waiting on step flags, and
// no executor touches another's user buffers, so launches need no entry or
// exit barrier and no system-scope fence.
enum class CopyMode { pull = 0, push = 1, staged = 2, ll = 3 };

/// Build the schedule. `element_size` sizes the arena; copies run on the
/// destination's executor (pull) or the source's (push); reductions
/// always run where they land (pull-reduce: remote loads, one local store).
Schedule build_schedule(const PipelinedPlan& plan, const std::vector<int>& rank_to_exec,
                        int num_execs, int element_size, CopyMode copy_mode);

/// Replays a schedule sequentially the way the executor would and
/// checks, transfer by transfer, that every contributor is present once
/// and that no hazard is left without an ordering edge. Throws
/// DependencyViolation on failure (used by the tests).
void verify_schedule(const PipelinedPlan& plan, const Schedule& s);

/// The numeric half of verify_schedule, cheap enough for every executor:
/// the plan's sequential (slot, id) execution and the schedule's
/// step-by-step concurrent execution, replayed on segments (maximal ranges
/// every element of which sees the same operations) instead of elements.
/// Throws DependencyViolation when they differ; false when the plan cuts
/// its buffers into more than `max_segments` segments (not checked).
bool replay_schedule(const PipelinedPlan& plan, const Schedule& s, int64_t max_segments);

}  // namespace hiccl
