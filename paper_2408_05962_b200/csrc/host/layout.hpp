// Device layout of a schedule and its tile-granular synchronization.
//
// build_layout() decides, for one executor, how each global step becomes
// device items and tiles: item order (peer rotation), NVLS lowering
// (multimem.ld_reduce / multimem.st where buffers sit in a multicast
// window), tile size, and the tile -> CTA assignment (tile t runs on CTA
// t mod G; equal-size items are interleaved tile by tile).
//
// analyze_sync() then derives, from every executor's layout, which CTA of
// which executor each CTA must wait for before each of its steps: every
// RAW / WAR / WAW hazard between two tiles becomes "CTA c of executor E has
// finished step s". When producer and consumer tile the same range the
// same way (pipelined chains), a consumer CTA waits for exactly one
// producer CTA instead of the whole producing executor — the paper's
// fine-grain dependencies across fences at tile grain.
//
// Pure host code, deterministic: every executor computes the same result
// for every other executor (that is how a producer knows what to publish).
#pragma once

#include <cstdint>
#include <vector>

#include "schedule.hpp"

namespace hiccl {

struct AbsRef {
  int rank = 0;
  int buffer = 0;
  int64_t offset = 0;
  bool multicast = false;  // the same (buffer, offset) of every rank, via the switch
  bool ll = false;         // tagged-line staging (CopyMode::ll): ordered by its tags
};

// mc_reduce_store: multimem.ld_reduce of every rank's range, multimem.st of
// the result into the same range of every rank, per tile (fuse_nvls).
enum class ItemKind : uint8_t { p2p = 0, mc_reduce = 1, mc_store = 2, mc_reduce_store = 3 };

struct AbsItem {
  AbsRef dst;
  std::vector<AbsRef> srcs;
  int64_t count = 0;
  ReduceOp op = ReduceOp::sum;
  ItemKind kind = ItemKind::p2p;
  uint32_t n_tiles = 0;
  // Tile l of this item runs on CTA (base_cta + l) % G. The base is a
  // function of the destination range alone, so a range produced in one
  // step and consumed in a later one (chains, reduce-scatter -> all-gather)
  // is tiled onto the same CTAs: the consumer CTA waits for one producer CTA.
  uint32_t base_cta = 0;
  int64_t tile_key = 0;  // range offset the base is derived from
};

struct StepLayout {
  int tile_elems = 0;
  uint32_t n_tiles = 0;  // over all items
  // The step's tiles run on CTAs [cta_lo, cta_lo + cta_n). With alternating
  // halves (LayoutParams::alt_halves) consecutive steps use disjoint halves
  // of the grid, so one half's fence / wait / ramp overlaps the other half's
  // transfer (half the SMs saturate NVLink, tools/nvlinkbench.cu).
  int cta_lo = 0;
  int cta_n = 1;
  std::vector<AbsItem> items;
};

struct ExecLayout {
  std::vector<StepLayout> steps;
};

struct LayoutParams {
  int ctas = 1;       // G, identical on every executor
  int threads = 512;
  int esize = 4;
  int dtype = 0;      // HC_* code, decides which NVLS reductions exist
  std::vector<bool> multicast;  // per plan buffer: bound to an NVLS window
  int max_tile_vec = 8;         // tile = threads * {1,2,4,8 (max)} * 16 bytes
  bool alt_halves = false;      // steps alternate between the grid's halves
  // Tile-granular progress (analyze_sync): a consumer tile waits for the
  // producer tiles it conflicts with, not for the producer CTAs' whole steps.
  bool tile_sync = false;
};

/// Grid size every executor uses when the caller does not fix one: one CTA
/// per SM, fewer when no step of any executor has two 16-byte vectors per
/// thread for every CTA.
int auto_ctas(const Schedule& s, int esize, int threads, int sms);

// Payload bytes per tile in tagged-line schedules (one warp, 2 lines a lane).
constexpr int kLLTileBytes = 512;

ExecLayout build_layout(const Schedule& s, int exec, const LayoutParams& lp);

/// Default for LayoutParams::alt_halves: pipelined schedules (>= 4 steps)
/// whose steps are at most 8 MiB per executor. Measured at p = 4
/// (profiles/r1/experiments/alt_halves_p4.txt): chains of 2-8 MiB steps
/// 5-15% faster; larger steps 8-16% slower (half the grid no longer keeps
/// enough in flight).
bool want_alt_halves(const Schedule& s, int esize);

/// NVLS reduce-then-multicast fusion over every executor's layout (all
/// executors run it on the same input and get the same result). An
/// mc_reduce item of step s1 whose result range is multicast in place by an
/// mc_store of a later step s2 of the same executor (all-reduce =
/// reduce-scatter . all-gather) becomes one mc_reduce_store item at s1: each
/// tile is reduced through the switch and multicast straight back, so the
/// egress-bound reduction and the ingress-bound multicast overlap instead of
/// running as two link-bound phases. Fused only when no access of any
/// executor in steps [s1, s2) touches the multicast range (other than the
/// reduction itself), so every value read or written keeps the plan's order.
/// Returns the number of fused pairs.
int fuse_nvls(const Schedule& s, std::vector<ExecLayout>& layouts);

/// CTA that runs tile `local` of `item` (the device loop enumerates the
/// same assignment: for CTA lo + b, item i, tiles l = (b - base_i) mod n + kn).
inline int tile_cta(const AbsItem& it, uint32_t local, const StepLayout& L) {
  return L.cta_lo + (int)((it.base_cta + local) % (uint32_t)L.cta_n);
}

struct CtaWait {
  int exec;
  int cta;   // -1: every CTA of `exec`
  int step;  // wait until that CTA (those CTAs) finished this global step ...
  // ... or, for a tile-level wait (tile_sync), only up to its tile `value`:
  // progress word >= epoch base + value, value = step * T + ordinal + 1
  // (T = ExecSync::tile_stride; a finished step s publishes (s + 1) * T),
  // checked before this CTA's tile `at` of the step (its ordinal).
  int64_t value = -1;  // -1: step-level, (step + 1) * T
  int at = 0;
  int64_t target(int T) const { return value >= 0 ? value : (int64_t)(step + 1) * T; }
};

/// Ordinal of every tile of a step on its CTA, in the device loop's order
/// (rounds, then items from a CTA-dependent one): ord[item][local tile].
std::vector<std::vector<uint32_t>> tile_ordinals(const StepLayout& L);

struct ExecSync {
  // waits[step][cta]: what CTA `cta` of this executor waits for before
  // running its tiles of `step` (only CTAs with tiles in the step).
  std::vector<std::vector<std::vector<CtaWait>>> waits;
  // Per step: 0 nobody waits on it; 1 only CTAs of this executor wait
  // (GPU-scope release to its own flag words); 2 another executor waits,
  // or the step's writes land in peer memory (system-scope release to
  // every executor's words).
  std::vector<uint8_t> publish;
  // Per step: the CTA barriers before it, because one of its tiles depends
  // on a tile the same CTA ran earlier (tagged-line schedules only: there
  // the barrier replaces a flag round).
  std::vector<uint8_t> barrier;
  // required[step][cta]: every (executor, CTA, step) whose tiles conflict
  // with this CTA's tiles of `step` — the waits before compression into
  // whole-executor waits. The checked launch mode (HICCL_CHECK_DEPS=1)
  // re-reads each producer's flag before the CTA's tiles run and reports
  // DependencyViolation if one has not finished its step.
  std::vector<std::vector<std::vector<CtaWait>>> required;
  // tile_waits[step][cta]: tile-level waits (tile_sync), sorted by `at`.
  std::vector<std::vector<std::vector<CtaWait>>> tile_waits;
  // Per step: publish progress after every tile (someone waits at tile grain).
  std::vector<uint8_t> tile_publish;
  int tile_stride = 1;  // T: progress words advance T per step (1: no tile sync)
  int64_t paired = 0;         // single-CTA waits
  int64_t whole = 0;          // whole-executor waits
};

std::vector<ExecSync> analyze_sync(const Schedule& s, const std::vector<ExecLayout>& layouts,
                                   const LayoutParams& lp);

/// Independent check (tests): replays every hazard pair of tiles and
/// confirms a wait (possibly transitive through the same CTA's earlier
/// waits is NOT assumed) covers it. Throws DependencyViolation.
void verify_sync(const Schedule& s, const std::vector<ExecLayout>& layouts,
                 const std::vector<ExecSync>& sync, const LayoutParams& lp);

}  // namespace hiccl
