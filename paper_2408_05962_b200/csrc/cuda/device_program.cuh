// Device-side program tables of the persistent executor. Built on the
// host from a Schedule (csrc/host/schedule.hpp) with every address
// already resolved into this device's view (local, peer-mapped or
// IPC-opened), so the kernel never translates names or ranks.
#pragma once

#include <cstdint>

namespace hiccl::dev {

// One fused write group: dst = fold(src[0], src[1], ..., src[n-1]) over
// `count` elements, in exactly that order (the reference's id order).
struct Item {
  uint64_t dst;         // device address
  int64_t count;        // elements
  uint32_t src_first;   // index into Program::srcs
  uint16_t n_src;       // >= 1
  uint8_t op;           // 0 sum, 1 max (ignored when n_src == 1)
  uint8_t flags;        // kVec | kMcReduce | kMcStore
  uint32_t tile_first;  // first tile of this item within its step
  uint32_t n_tiles;
};
static_assert(sizeof(Item) == 32, "Item layout");

// Item flags.
constexpr uint8_t kVec = 1;       // dst and every src congruent mod 16 bytes
constexpr uint8_t kMcReduce = 2;  // src[0] is a multicast address: multimem.ld_reduce
constexpr uint8_t kMcStore = 4;   // dst is a multicast address: multimem.st

// One global (slot, phase) step as seen by this executor.
struct Step {
  uint32_t item_first;
  uint32_t n_items;
  uint32_t n_tiles;
  uint32_t wait_first;
  uint32_t n_waits;
  uint16_t publish;  // 1: some executor waits on this step -> arrive + publish
  uint16_t uniform;  // 1: every item has n_tiles == n_tiles / n_items -> interleave
  uint32_t tile_elems;  // per-step tile size: small steps use small tiles so
                        // every CTA gets work (threads * {1,2,4,8} * 16 bytes)
};

// "executor `exec` has published at least epoch_base + k".
struct Wait {
  uint32_t exec;
  uint32_t k;
};

// Flag word protocol, per epoch e (one epoch per start()), S steps:
//   value e*(S+2) + 0      executor started (its inputs are ready)
//   value e*(S+2) + 1 + s  executor finished global step s
//   value e*(S+2) + S + 1  executor finished everything
// Values only grow (red.release.sys.max), so a wait is one comparison.
struct Program {
  const Step* steps;
  const Item* items;
  const uint64_t* srcs;
  const Wait* waits;
  uint64_t* flags;                 // this executor's flag words [num_execs]
  uint64_t* const* peer_flags;     // every executor's flag words (this device's view)
  unsigned long long* arrive;      // [num_steps + 1] CTA arrival counters
  unsigned int* status;            // device word: 0 ok, 1 watchdog fired (sticky)
  int num_steps;
  int num_execs;
  int self;
  unsigned long long* trace;       // [num_steps + 4] globaltimer stamps (see kernels.cuh)
  long long timeout_ns;            // <= 0: no watchdog
};

constexpr int kMaxExecs = 64;

}  // namespace hiccl::dev
