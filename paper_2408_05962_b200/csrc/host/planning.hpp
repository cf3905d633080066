// Internal helpers shared by the lowering (factor.cpp), the ordering and
// pipelining passes (order.cpp) and the plan persistence (plan_io.cpp).
#pragma once

#include <vector>

#include "hiccl/plan.hpp"
#include "json.hpp"

namespace hiccl {

/// Which clock orders a plan: stages (a lowered plan) or slots (a
/// pipelined one). The canonical orders differ only in that key and in
/// where the channel ranks among the tie-breakers (reference
/// factorize.cpp:360-365 and pipeline.cpp:30-35).
enum class Clock { stage, slot };

/// Sorts into canonical order and numbers the transfers 0..n-1.
void sort_canonical(std::vector<P2PTransfer>& ts, Clock clock);

/// Def-use edges: a transfer depends on every transfer of an earlier
/// stage/slot that writes into its source range or, when it reduces, into
/// its destination range. With `fences`, a fence that such an edge crosses
/// between non-identical ranges is marked misaligned (the pipeliner must
/// drain there). Reference: factorize.cpp:377-414, pipeline.cpp:43-72.
void link_dependencies(std::vector<P2PTransfer>& ts, Clock clock,
                       std::vector<FenceBoundary>* fences);

json::Value buffers_to_json(const std::map<std::string, BufferDecl>& decls);
json::Value staged_plan_json(const StagedPlan& p);
StagedPlan staged_plan_from(const json::Value& j);

}  // namespace hiccl
