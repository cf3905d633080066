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
  uint32_t base_cta;    // tile l runs on CTA (base_cta + l) % gridDim
  uint32_t n_tiles;
};
static_assert(sizeof(Item) == 32, "Item layout");

// Item flags.
constexpr uint8_t kVec = 1;       // dst and every src congruent mod 16 bytes
constexpr uint8_t kMcReduce = 2;  // src[0] is a multicast address: multimem.ld_reduce
constexpr uint8_t kMcStore = 4;   // dst is a multicast address: multimem.st
constexpr uint8_t kLLStore = 8;   // dst is tagged-line staging in a peer (CopyMode::ll)
constexpr uint8_t kLLLoad = 16;   // some src is tagged-line staging (address bit 63 set)
constexpr uint8_t kTma = 32;      // local copy, 16-byte aligned, whole 16-byte vectors
constexpr uint8_t kAlign16 = 64;  // point-to-point fold, every address 16-byte aligned,
                                  // whole vectors: may be staged through shared memory
constexpr uint64_t kLLBit = 1ULL << 63;

// One global (slot, phase) step as seen by this executor.
struct Step {
  uint32_t item_first;
  uint32_t n_items;
  uint32_t n_tiles;
  uint16_t publish;  // 0: nobody waits; 1: only this executor's CTAs wait (GPU-scope
                     // release to its own words); 2: system-scope release to every executor
  uint16_t max_rounds;  // max over items of ceil(n_tiles / gridDim)
  uint32_t tile_elems;  // per-step tile size: small steps use small tiles so
                        // every CTA gets work (threads * {1,2,4,8} * 16 bytes)
  uint16_t barrier;     // 1: CTA barrier before the step (own earlier tiles)
  uint16_t tma;         // 1: every item is a local 16-byte-aligned copy: thread 0
                        // streams the CTA's tiles with TMA bulk copies (kernels.cuh);
                        // 2: every item is kAlign16: staged folds (kernels.cuh)
  uint16_t cta_lo;      // the step's tiles run on CTAs [cta_lo, cta_lo + cta_n)
  uint16_t cta_n;       // (alternating halves let consecutive steps overlap)
  uint16_t tile_publish;  // 1: publish progress after every tile (tile-level waiters)
  uint16_t pad;
};

// "CTA `cta` (kAllCtas: every CTA) of executor `exec` has published at
// least epoch_base + k" — i.e. finished global step k - 1.
struct Wait {
  uint16_t exec;
  uint16_t cta;
  uint32_t k;
};
constexpr uint16_t kAllCtas = 0xFFFF;

// A tile-level wait: before this CTA's tile `at` of the step (its ordinal),
// CTA `cta` of `exec` must have published at least epoch_base + k, where a
// producer's tile with ordinal o of step s publishes s * T + o + 1 and a
// finished step s publishes (s + 1) * T (T = Program::tile_stride).
struct TileWait {
  uint16_t exec;
  uint16_t cta;
  uint32_t k;
  uint32_t at;
  uint32_t pad;
};
constexpr int kMaxCtas = 1024;

// Flag words, per epoch e (one epoch per start()), S steps. Executor words
// flags[x], x < kMaxExecs:
//   e*(S+2) + 0      executor x started (its inputs are ready)
//   e*(S+2) + S + 1  executor x finished everything
// CTA words flags[kMaxExecs + x*kMaxCtas + c]:
//   e*(S+2) + 1 + s  CTA c of executor x finished global step s
// Producers raise the words in every executor's array (relaxed system-scope
// max after one release fence); values only grow, a wait is a comparison.
struct Program {
  const Step* steps;
  const Item* items;
  const uint64_t* srcs;
  const uint2* cta_waits;          // [num_steps * gridDim] {first, count} into waits
  const Wait* waits;
  uint64_t* flags;                 // this executor's flag words (layout above)
  uint64_t* const* peer_flags;     // every executor's flag words (this device's view)
  unsigned long long* arrive;      // [num_steps + 2]; [num_steps] counts this launch's exit arrivals (reset by the last),
                                   // [num_steps + 1] = epoch of the last finished launch
  unsigned int* status;            // device word: 0 ok, 1 watchdog fired (sticky)
  unsigned int* status_mirror;     // host-mapped copy of status[0..4] (read by wait())
  int num_steps;
  int num_execs;
  int self;
  unsigned long long* trace;       // [num_steps + 4] globaltimer stamps (see kernels.cuh)
  long long timeout_ns;            // <= 0: no watchdog
  // Tagged-line mode (CopyMode::ll): no entry / exit barrier; a line of
  // epoch e carries tag (uint32)e and lives in arena copy e & 1, ll_half
  // bytes apart.
  int ll;
  unsigned long long ll_half;
  // steps / items / srcs live in one 16-byte-aligned image; when smem_bytes
  // > 0 the kernel copies it (image_bytes) plus this CTA's cta_waits entries
  // into dynamic shared memory at entry.
  const void* image;
  int image_bytes;
  int smem_bytes;
  int tma;                         // some step is a TMA step (smem_bytes >= 2 * kTmaChunk)
  // Some item reads or writes through a multicast (NVLS) address while
  // other accesses reach the same memory through unicast addresses:
  // fence.proxy.alias at every flag hand-off (see kernels.cuh).
  int alias_fence;
  // Checked mode (HICCL_CHECK_DEPS=1): per (step, CTA) {first, count} into
  // `checks` — producer (executor, CTA, step + 1) flags re-read before the
  // CTA's tiles run; a producer not yet done sets status bit 2 and records
  // the first violation in status[1..4]. Null otherwise.
  const uint2* cta_checks;
  const Wait* checks;
  // Test hook (checked mode only): executor `delay_exec` sleeps `delay_ns`
  // before each of its steps.
  int delay_exec;
  long long delay_ns;
  int solo;  // profiling hook: no entry / exit barrier (HICCL_PROFILE_SOLO)
  // staged folds: stages of fold_stage_bytes in the dynamic shared memory
  unsigned int fold_stages;
  unsigned int fold_stage_bytes;
  // Tile-granular progress: words advance tile_stride (T) per step; per
  // (step, CTA) {first, count} into tile_waits (sorted by `at`), or null.
  unsigned int tma_stages;  // TMA copy steps: stages of kTmaChunk in flight (2..kTmaMaxStages)
  unsigned int tile_stride;
  unsigned int tile_pub_every;  // publish after every k-th tile (the step end always publishes)
  const uint2* cta_tile_waits;
  const TileWait* tile_waits;
};
constexpr unsigned kStatusTimeout = 1u, kStatusDepViolation = 2u;
constexpr unsigned kTmaChunk = 32 * 1024;  // per stage (tools/tmacopy.cu)
constexpr int kTmaMaxStages = 4;
constexpr int kMaxProgramSmem = 96 * 1024;

constexpr int kMaxExecs = 64;

}  // namespace hiccl::dev
