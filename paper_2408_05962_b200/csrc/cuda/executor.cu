// Host side of the persistent executor: schedule -> device tables,
// buffers/arena/flags, cooperative launch, C ABI (include/hiccl.h).
#include <nvtx3/nvtx3.hpp>
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../host/capi_common.hpp"
#include "../host/layout.hpp"
#include "hiccl/model.hpp"
#include "../host/schedule.hpp"
#include "hiccl.h"
#include "kernels.cuh"

using namespace hiccl;

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(ErrorCode::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

int element_size(int dtype) {
  switch (dtype) {
    case HC_F32: return 4;
    case HC_BF16: return 2;
    case HC_F16: return 2;
    case HC_I32: return 4;
    case HC_I64: return 8;
    case HC_F64: return 8;
    case HC_U8: return 1;
  }
  throw Error(ErrorCode::InvalidConfig, "unknown dtype " + std::to_string(dtype));
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class T>
T* upload(const std::vector<T>& v, std::vector<void*>& owned) {
  if (v.empty()) return nullptr;
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, v.size() * sizeof(T)), "cudaMalloc(table)");
  owned.push_back(p);
  cuda_check(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice),
             "cudaMemcpy(table)");
  return (T*)p;
}

constexpr int kStatusWords = 5;  // [0] bits, [1..4] first dependency violation

bool env_flag(const char* name) {
  const char* v = std::getenv(name);
  return v && atoi(v) != 0;
}

// Every schedule an executor runs is first replayed against the plan's
// sequential execution (replay_schedule: exact, on segments, milliseconds
// at any byte count); a schedule-compiler bug then fails create / commit
// with DependencyViolation instead of computing wrong bytes.
// HICCL_VERIFY_SCHEDULE=0 skips it.
Schedule checked_schedule(const PipelinedPlan& plan, const std::vector<int>& rank_to_exec,
                          int num_execs, int esize, CopyMode mode) {
  Schedule s = build_schedule(plan, rank_to_exec, num_execs, esize, mode);
  static const bool skip = std::getenv("HICCL_VERIFY_SCHEDULE") &&
                           atoi(std::getenv("HICCL_VERIFY_SCHEDULE")) == 0;
  if (!skip) replay_schedule(plan, s, 1LL << 22);
  return s;
}

CopyMode copy_mode_of(int m) {
  if (m < 0 || m > 3)
    throw Error(ErrorCode::InvalidConfig, "copy_mode must be 0 pull, 1 push, 2 staged, 3 ll, 4 auto");
  return (CopyMode)m;
}

// copy_mode 4: push or tagged lines by the cost model (model.hpp). A pure
// function of the plan, element size and rank map, so every executor of a
// world resolves it the same way.
int resolve_auto_mode(const PipelinedPlan& plan, int esize, const std::vector<int>& r2e,
                      int num_execs) {
  const int p = plan.base.world_size;
  bool contiguous = p % num_execs == 0;
  for (int r = 0; r < p && contiguous; ++r) contiguous = r2e[r] == r / (p / num_execs);
  if (!contiguous || num_execs == 1) return 1;
  for (const auto& [name, d] : plan.base.buffers)
    if (!d.internal && (double)d.length * esize > 64.0 * (1 << 20)) return 1;
  const B200Model m;
  const int rpg = p / num_execs;
  return predict(plan, esize, m, rpg, 3).seconds < predict(plan, esize, m, rpg, 1).seconds ? 3 : 1;
}

using KernelFn = void (*)(dev::Program);

template <bool LL, bool TS>
KernelFn kernel_for_mode(int dtype) {
  switch (dtype) {
    case HC_F32: return dev::persistent_executor<0, LL, TS>;
    case HC_BF16: return dev::persistent_executor<1, LL, TS>;
    case HC_F16: return dev::persistent_executor<2, LL, TS>;
    case HC_I32: return dev::persistent_executor<3, LL, TS>;
    case HC_I64: return dev::persistent_executor<4, LL, TS>;
    case HC_F64: return dev::persistent_executor<5, LL, TS>;
    case HC_U8: return dev::persistent_executor<6, LL, TS>;
  }
  throw Error(ErrorCode::InvalidConfig, "unknown dtype");
}

KernelFn kernel_for(int dtype, bool ll, bool ts = false) {
  // tagged lines have their own protocol; tile sync is a bandwidth-kernel variant
  return ll ? kernel_for_mode<true, false>(dtype)
            : ts ? kernel_for_mode<false, true>(dtype) : kernel_for_mode<false, false>(dtype);
}

}  // namespace

struct hc_exec {
  PipelinedPlan plan;
  hc_exec_config cfg{};
  std::vector<int> rank_to_exec;
  Schedule sched;
  int esize = 4;
  int device = 0;
  // copy_mode 4 resolved to tagged lines at creation: commit() may still
  // switch to push when NVLS windows get bound and the model prefers them
  // (the arena was sized for both schedules)
  bool auto_ll = false;

  void* arena = nullptr;
  size_t arena_bytes = 0;
  uint64_t* flags = nullptr;
  unsigned long long* arrive = nullptr;
  unsigned long long* trace = nullptr;  // device stamps of the last launch
  unsigned int* status_dev = nullptr;  // watchdog word (device)
  unsigned int* status_host = nullptr;  // host-mapped mirror the kernel writes when it sets a bit
  unsigned int* status_mapped = nullptr;  // its device address
  cudaStream_t own_stream = nullptr;    // executors sharing a device: private non-blocking stream
  bool poisoned = false;
  std::vector<void*> peer_arena;
  std::vector<uint64_t*> peer_flags;
  std::map<std::pair<int, std::string>, std::pair<char*, size_t>> bindings;
  std::map<std::string, char*> multicast;  // buffer name -> multicast address (NVLS)

  std::vector<void*> tables;  // device allocations owned by commit
  dev::Program prog{};
  bool committed = false;
  int ctas = 0, threads = 0;
  cudaEvent_t done = nullptr;
  bool launched = false;     // a non-captured launch to wait for
  bool ever_started = false;  // any start(), captured ones included
  size_t step_words_steps = 0;  // step count the arrive words were sized for
  unsigned words_T = 1;         // tile stride of the committed program
  bool tile_mode = false;       // the tile-sync kernel variant
  hc_exec_stats stats{};

  ~hc_exec() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (launched && done) cudaEventSynchronize(done);
    for (void* p : tables) cudaFree(p);
    for (void* p : retired) cudaFree(p);
    if (arena) cudaFree(arena);
    if (flags) cudaFree(flags);
    if (arrive) cudaFree(arrive);
    if (trace) cudaFree(trace);
    if (status_dev) cudaFree(status_dev);
    if (status_host) cudaFreeHost(status_host);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (done) cudaEventDestroy(done);
    if (prev >= 0) cudaSetDevice(prev);
  }

  // A re-commit replaces the tables, but CUDA graphs captured from earlier
  // start() calls still point at the old ones: retire them, free at destroy.
  std::vector<void*> retired;
  void free_tables() {
    retired.insert(retired.end(), tables.begin(), tables.end());
    tables.clear();
  }

  char* address(const Loc& l, int64_t count) {
    const BufferDecl& d = sched.buffer_decls[l.buffer];
    const std::string& name = sched.buffer_names[l.buffer];
    if (d.internal) {
      const int x = sched.home[l.rank][l.buffer];
      char* base = x == cfg.exec_index ? (char*)arena : (char*)peer_arena[x];
      if (!base)
        throw Error(ErrorCode::BadBufferRef,
                    "arena of executor " + std::to_string(x) + " not bound (hc_exec_bind_peer_arena)");
      const int64_t off = sched.arena_offset[l.rank][l.buffer];
      if (off < 0) throw Error(ErrorCode::BadBufferRef, "internal buffer not laid out: " + name);
      return base + off + l.offset * esize;
    }
    auto it = bindings.find({l.rank, name});
    if (it == bindings.end())
      throw Error(ErrorCode::BadBufferRef, "buffer '" + name + "' of rank " +
                                               std::to_string(l.rank) + " is not bound");
    if ((size_t)((l.offset + count) * esize) > it->second.second)
      throw Error(ErrorCode::BadBufferRef, "buffer '" + name + "' of rank " +
                                               std::to_string(l.rank) + " is smaller than the plan needs");
    return it->second.first + l.offset * esize;
  }

  // Device address of an abstract reference, as seen from this device.
  char* resolve(const AbsRef& r, int64_t count) {
    if (r.multicast) {
      auto it = multicast.find(sched.buffer_names[r.buffer]);
      if (it == multicast.end())
        throw Error(ErrorCode::BadBufferRef, "no multicast binding for " + sched.buffer_names[r.buffer]);
      return it->second + r.offset * esize;
    }
    return address(Loc{r.rank, r.buffer, r.offset}, count);
  }

  // Local per-schedule device words (step arrival counters, trace).
  // Flag words only grow: launch e of an S-step schedule with tile stride T
  // publishes values in [e (S + 2) T, (e + 1)(S + 2) T). When a re-commit
  // changes S or T after launches (captured or not), the epoch restarts
  // above every value ever published, so no stale word satisfies a new
  // wait; every executor has run the same launches, so all compute the
  // same epoch.
  unsigned long long published_floor() {
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize(recommit)");
    unsigned long long e = 0;
    cuda_check(cudaMemcpy(&e, arrive + step_words_steps + 1, sizeof e, cudaMemcpyDeviceToHost),
               "cudaMemcpy(epoch)");
    return (e + 1) * (unsigned long long)(step_words_steps + 2) * words_T;
  }
  void set_epoch_above(unsigned long long floor, unsigned T) {
    const unsigned long long unit = (unsigned long long)(step_words_steps + 2) * T;
    const unsigned long long e0 = (floor + unit - 1) / unit;
    cuda_check(cudaMemcpy(arrive + step_words_steps + 1, &e0, sizeof e0, cudaMemcpyHostToDevice),
               "cudaMemcpy(epoch)");
    words_T = T;
  }
  void alloc_step_words() {
    unsigned long long floor = 0;
    if (arrive) {
      floor = published_floor();
      cudaFree(arrive);
    }
    if (trace) cudaFree(trace);
    arrive = nullptr;
    trace = nullptr;
    const size_t nsteps = sched.step_slot.size();
    cuda_check(cudaMalloc(&arrive, sizeof(unsigned long long) * (nsteps + 2)), "cudaMalloc(arrive)");
    cuda_check(cudaMemset(arrive, 0, sizeof(unsigned long long) * (nsteps + 2)), "cudaMemset(arrive)");
    step_words_steps = nsteps;
    if (floor) set_epoch_above(floor, words_T);
    cuda_check(cudaMalloc(&trace, sizeof(unsigned long long) * (nsteps + 4 + 128)), "cudaMalloc(trace)");
    cuda_check(cudaMemset(trace, 0, sizeof(unsigned long long) * (nsteps + 4 + 128)), "cudaMemset(trace)");
  }

  void commit() {
    DeviceGuard g(device);
    free_tables();
    const int self = cfg.exec_index;
    if (auto_ll && !multicast.empty() && !ever_started) {
      // every executor binds the same windows, so all make the same choice
      const B200Model m;
      if (predict_nvls(plan, cfg.dtype, m).seconds < predict(plan, esize, m, 1, 3).seconds) {
        cfg.copy_mode = 1;
        sched = checked_schedule(plan, rank_to_exec, cfg.num_execs, esize, CopyMode::push);
        alloc_step_words();
      }
      auto_ll = false;
    }
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    const int max_threads = sched.ll ? dev::kLLThreads : 512;
    // multimem bodies run best with 256-thread CTAs (half the multicast
    // requests in flight per SM of the 512-thread point-to-point body:
    // 1 GiB fused all-reduce at p=4 2.34 ms against 2.40-2.47 ms,
    // profiles/r1/nvls/tile_sweep_p4.txt)
    bool nvls_window = !sched.ll && !multicast.empty() && cfg.num_execs == sched.world_size;
    threads = cfg.threads > 0 ? cfg.threads : nvls_window ? 256 : max_threads;
    if (threads % 32 || threads < 64 || threads > max_threads)
      throw Error(ErrorCode::InvalidConfig, "threads must be a multiple of 32 in [64, " +
                                                std::to_string(max_threads) + "]");
    KernelFn fn = kernel_for(cfg.dtype, sched.ll);  // occupancy: the variants share launch bounds
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, threads, 0),
               "occupancy");
    // executors sharing the device split its co-resident capacity, so all
    // of their persistent grids run at once
    const int sharing = std::max(1, cfg.execs_per_device);
    const int max_ctas = std::min(per_sm * prop.multiProcessorCount / sharing, dev::kMaxCtas);
    if (max_ctas < 1)
      throw Error(ErrorCode::InvalidConfig, std::to_string(sharing) + " executors cannot share one device");
    // The grid size is a function of the schedule alone, so every executor
    // picks the same G (tile -> CTA maps must agree across executors).
    ctas = cfg.ctas > 0 ? cfg.ctas
                        : std::min(max_ctas, auto_ctas(sched, esize, threads, prop.multiProcessorCount));
    if (ctas > max_ctas)
      throw Error(ErrorCode::InvalidConfig, "ctas " + std::to_string(ctas) +
                                                " exceed co-resident capacity " + std::to_string(max_ctas));

    LayoutParams lp;
    lp.ctas = ctas;
    lp.threads = threads;
    lp.esize = esize;
    lp.dtype = cfg.dtype;
    if (const char* kv = std::getenv("HICCL_TILE_VEC")) lp.max_tile_vec = std::max(1, std::min(8, atoi(kv)));
    lp.alt_halves = want_alt_halves(sched, esize);
    if (const char* ah = std::getenv("HICCL_ALT_HALVES")) lp.alt_halves = atoi(ah) != 0;
    lp.multicast.assign(sched.buffer_names.size(), false);
    for (size_t b = 0; b < sched.buffer_names.size(); ++b)
      lp.multicast[b] = multicast.count(sched.buffer_names[b]) > 0;
    // Tile-granular progress (HICCL_TILE_SYNC=1; every executor of a world
    // must agree): not with NVLS windows, tagged lines or the checked mode
    // (whose producer checks are step-level).
    lp.tile_sync = env_flag("HICCL_TILE_SYNC") && multicast.empty() && !sched.ll &&
                   !env_flag("HICCL_CHECK_DEPS");
    std::vector<ExecLayout> layouts;
    for (int e = 0; e < cfg.num_execs; ++e) layouts.push_back(build_layout(sched, e, lp));
    if (!std::getenv("HICCL_NO_NVLS_FUSE")) fuse_nvls(sched, layouts);
    const std::vector<ExecSync> sync = analyze_sync(sched, layouts, lp);
    const ExecLayout& L = layouts[self];
    const ExecSync& Y = sync[self];
    tile_mode = lp.tile_sync;
    fn = kernel_for(cfg.dtype, sched.ll, tile_mode);
    if ((unsigned)Y.tile_stride != words_T) {
      if (ever_started) set_epoch_above(published_floor(), (unsigned)Y.tile_stride);
      words_T = (unsigned)Y.tile_stride;
    }
    const int nsteps = (int)L.steps.size();

    std::vector<dev::Step> steps(nsteps);
    std::vector<dev::Item> items;
    std::vector<uint64_t> srcs;
    std::vector<uint2> cta_waits((size_t)nsteps * ctas, make_uint2(0, 0));
    std::vector<dev::Wait> waits;
    // Checked mode (debug): producer flags re-read before every step's
    // tiles (kernels.cuh check_producers). Test hooks, checked mode only:
    // HICCL_TEST_DROP_WAITS=1 drops every wait, HICCL_TEST_DELAY_EXEC=x
    // makes executor x sleep HICCL_TEST_DELAY_NS (default 2 ms) per step.
    const bool checked = env_flag("HICCL_CHECK_DEPS");
    const bool drop_waits = checked && env_flag("HICCL_TEST_DROP_WAITS");
    std::vector<uint2> cta_checks(checked ? (size_t)nsteps * ctas : 0, make_uint2(0, 0));
    std::vector<dev::Wait> checks;
    std::vector<uint2> cta_tile_waits(lp.tile_sync ? (size_t)nsteps * ctas : 0, make_uint2(0, 0));
    std::vector<dev::TileWait> tile_waits;
    stats = hc_exec_stats{};
    const bool use_tma = !sched.ll && !std::getenv("HICCL_NO_TMA");
    bool any_tma = false, any_staged = false;
    // Staged folds (kernels.cuh staged_fold_step): 0 off, 1 steps whose
    // folds are all local (default), 2 every eligible step (HICCL_STAGED)
    // Default 1: C1 455 vs 479 us, p = 8 virtual all-reduce 777 vs 839 us
    // (profiles/r2/staged_fold_ab.txt).
    const int staged_mode = sched.ll ? 0
                            : std::getenv("HICCL_STAGED") ? atoi(std::getenv("HICCL_STAGED")) : 1;
    for (int s = 0; s < nsteps; ++s) {
      const StepLayout& SL = L.steps[s];
      dev::Step& st = steps[s];
      st.item_first = (uint32_t)items.size();
      st.n_items = (uint32_t)SL.items.size();
      st.n_tiles = SL.n_tiles;
      st.tile_elems = (uint32_t)SL.tile_elems;
      uint32_t rounds = 0;
      for (const AbsItem& a : SL.items)
        rounds = std::max<uint32_t>(rounds, (a.n_tiles + SL.cta_n - 1) / SL.cta_n);
      st.cta_lo = (uint16_t)SL.cta_lo;
      st.cta_n = (uint16_t)SL.cta_n;
      if (rounds > 0xFFFF) throw Error(ErrorCode::InvalidConfig, "step too large for the grid");
      st.max_rounds = (uint16_t)rounds;
      st.publish = Y.publish[s];
      st.barrier = Y.barrier[s];
      // steps followed or waiting tile by tile run the register body (the
      // TMA / staged bodies publish and wait per step)
      bool tile_involved = Y.tile_publish[s] != 0;
      for (int c = 0; c < ctas; ++c) tile_involved |= !Y.tile_waits[s][c].empty();
      bool all_tma = !SL.items.empty() && !tile_involved,
           all_staged = !SL.items.empty() && staged_mode > 0 && !tile_involved;
      for (const AbsItem& a : SL.items) {
        dev::Item it{};
        char* dst = resolve(a.dst, a.count);
        it.dst = (uint64_t)dst;
        it.count = a.count;
        it.src_first = (uint32_t)srcs.size();
        it.n_src = (uint16_t)a.srcs.size();
        it.op = (uint8_t)a.op;
        bool vec = true, ll_load = false;
        for (const AbsRef& r : a.srcs) {
          char* p = resolve(r, a.count);
          srcs.push_back((uint64_t)p | (r.ll ? dev::kLLBit : 0));
          vec &= ((uint64_t)p % 16) == ((uint64_t)dst % 16);
          ll_load |= r.ll;
        }
        uint8_t kind = a.kind == ItemKind::mc_reduce ? dev::kMcReduce
                       : a.kind == ItemKind::mc_store ? dev::kMcStore
                       : a.kind == ItemKind::mc_reduce_store ? (uint8_t)(dev::kMcReduce | dev::kMcStore)
                                                             : 0;
        if (kind) {
          if (!vec || (uint64_t)dst % 16)
            throw Error(ErrorCode::BadBufferRef, "NVLS window buffers must be 16-byte aligned");
          ++stats.nvls_items;
        }
        if (a.dst.ll) kind |= dev::kLLStore;
        if (ll_load) kind |= dev::kLLLoad;
        // local 16-byte-aligned copy of whole vectors -> TMA eligible
        if (use_tma && !kind && a.srcs.size() == 1 && !a.dst.multicast && !a.srcs[0].multicast &&
            sched.home[a.dst.rank][a.dst.buffer] == self &&
            sched.home[a.srcs[0].rank][a.srcs[0].buffer] == self &&
            (uint64_t)dst % 16 == 0 && srcs.back() % 16 == 0 && (a.count * esize) % 16 == 0)
          kind |= dev::kTma;
        all_tma &= (kind & dev::kTma) != 0;
        // staged-fold eligible: plain fold, every address 16-byte aligned,
        // whole vectors, at most 8 sources (and, in mode 1, all local)
        bool aligned = !(kind & ~dev::kTma) && !a.dst.multicast && a.srcs.size() <= 8 &&
                       (uint64_t)dst % 16 == 0 && (a.count * esize) % 16 == 0;
        bool local = aligned && sched.home[a.dst.rank][a.dst.buffer] == self;  // (multicast: rank -1)
        for (size_t j = 0; j < a.srcs.size(); ++j) {
          aligned &= !a.srcs[j].multicast && srcs[srcs.size() - a.srcs.size() + j] % 16 == 0;
          local &= !a.srcs[j].multicast && sched.home[a.srcs[j].rank][a.srcs[j].buffer] == self;
        }
        if (aligned) kind |= dev::kAlign16;
        all_staged &= aligned && (staged_mode == 2 || local);
        it.flags = (uint8_t)((vec ? dev::kVec : 0) | kind);
        it.base_cta = a.base_cta;
        it.n_tiles = a.n_tiles;
        items.push_back(it);
        // traffic accounting (plan view)
        const int64_t bytes = a.count * esize;
        for (const AbsRef& r : a.srcs) {
          stats.bytes_in += bytes;
          if (r.multicast || sched.home[r.rank][r.buffer] != self) stats.remote_bytes += bytes;
        }
        stats.bytes_out += bytes;
        if (a.dst.multicast || sched.home[a.dst.rank][a.dst.buffer] != self)
          stats.remote_bytes += a.dst.ll ? 2 * ((bytes + 7) / 8 * 8) : bytes;
      }
      st.tma = all_tma ? 1 : all_staged ? 2 : 0;
      stats.tma_steps += st.tma == 1;
      stats.staged_steps += st.tma == 2;
      any_tma |= all_tma;
      any_staged |= !all_tma && all_staged;
      if (checked)
        for (int c = 0; c < ctas; ++c) {
          const auto& need = Y.required[s][c];
          cta_checks[(size_t)s * ctas + c] = make_uint2((uint32_t)checks.size(), (uint32_t)need.size());
          for (const CtaWait& w : need)
            checks.push_back(dev::Wait{(uint16_t)w.exec, (uint16_t)w.cta,
                                       (uint32_t)((w.step + 1) * Y.tile_stride)});
        }
      for (int c = 0; c < ctas; ++c) {
        static const std::vector<CtaWait> none;
        const auto& list = drop_waits ? none : Y.waits[s][c];
        cta_waits[(size_t)s * ctas + c] = make_uint2((uint32_t)waits.size(), (uint32_t)list.size());
        for (const CtaWait& w : list) {
          waits.push_back(dev::Wait{(uint16_t)w.exec, w.cta < 0 ? dev::kAllCtas : (uint16_t)w.cta,
                                    (uint32_t)w.target(Y.tile_stride)});
          if (w.cta < 0) ++stats.whole_waits;
          else ++stats.paired_waits;
        }
      }
      st.tile_publish = Y.tile_publish[s];
      if (lp.tile_sync)
        for (int c = 0; c < ctas; ++c) {
          const auto& list = Y.tile_waits[s][c];
          cta_tile_waits[(size_t)s * ctas + c] =
              make_uint2((uint32_t)tile_waits.size(), (uint32_t)list.size());
          for (const CtaWait& w : list) {
            tile_waits.push_back(dev::TileWait{(uint16_t)w.exec, (uint16_t)w.cta,
                                               (uint32_t)w.target(Y.tile_stride), (uint32_t)w.at, 0});
            ++stats.paired_waits;
          }
        }
    }
    std::vector<uint64_t*> pf(cfg.num_execs);
    for (int x = 0; x < cfg.num_execs; ++x) {
      pf[x] = x == self ? flags : peer_flags[x];
      if (!pf[x])
        throw Error(ErrorCode::BadBufferRef,
                    "flags of executor " + std::to_string(x) + " not bound (hc_exec_bind_peer_flags)");
    }
    // steps | items | srcs as one 16-byte-aligned image (the kernel copies
    // it to shared memory when it fits, kernels.cuh)
    auto align16 = [](size_t v) { return (v + 15) / 16 * 16; };
    const size_t o_items = align16(steps.size() * sizeof(dev::Step));
    const size_t o_srcs = o_items + align16(items.size() * sizeof(dev::Item));
    const size_t image_bytes = o_srcs + align16(srcs.size() * sizeof(uint64_t));
    std::vector<unsigned char> image(std::max<size_t>(image_bytes, 16), 0);
    if (!steps.empty()) std::memcpy(image.data(), steps.data(), steps.size() * sizeof(dev::Step));
    if (!items.empty()) std::memcpy(image.data() + o_items, items.data(), items.size() * sizeof(dev::Item));
    if (!srcs.empty()) std::memcpy(image.data() + o_srcs, srcs.data(), srcs.size() * sizeof(uint64_t));
    unsigned char* img = upload(image, tables);
    prog.image = img;
    prog.image_bytes = (int)image_bytes;
    prog.steps = reinterpret_cast<const dev::Step*>(img);
    prog.items = reinterpret_cast<const dev::Item*>(img + o_items);
    prog.srcs = reinterpret_cast<const uint64_t*>(img + o_srcs);
    const size_t smem = image_bytes + (size_t)nsteps * sizeof(uint2);
    const bool use_smem = sched.ll && smem <= (size_t)dev::kMaxProgramSmem &&
                          !std::getenv("HICCL_NO_SMEM_PROGRAM");
    // staged folds: HICCL_FOLD_STAGES x HICCL_FOLD_STAGE_KB (default 2 x 64 KB)
    prog.fold_stages = std::getenv("HICCL_FOLD_STAGES")
                           ? (unsigned)std::max(2, std::min(dev::kFoldStages, atoi(std::getenv("HICCL_FOLD_STAGES"))))
                           : 2u;
    prog.fold_stage_bytes = std::getenv("HICCL_FOLD_STAGE_KB")
                                ? (unsigned)std::max(8, atoi(std::getenv("HICCL_FOLD_STAGE_KB"))) * 1024u
                                : dev::kFoldStageBytes;
    if (prog.fold_stages * prog.fold_stage_bytes > 200u * 1024u)
      prog.fold_stage_bytes = 200u * 1024u / prog.fold_stages / 1024u * 1024u;
    // TMA copy steps: stages of 32 KB in flight — 2 by default, 3 when the
    // staged folds' shared memory is there anyway (C1 412 -> 400 us, p = 8
    // virtual all-reduce 771 -> 768 us; 4: 399 / 792; a lone 1 GiB copy is
    // fastest with 2); HICCL_TMA_STAGES overrides
    const char* ts_env = std::getenv("HICCL_TMA_STAGES");
    const unsigned forced_tma =
        ts_env ? (unsigned)std::max(2, std::min(dev::kTmaMaxStages, atoi(ts_env))) : 0u;
    const size_t fold_smem = any_staged ? (size_t)prog.fold_stages * prog.fold_stage_bytes : 0;
    const size_t tma_smem = any_tma ? (size_t)(forced_tma ? forced_tma : 2u) * dev::kTmaChunk : 0;
    prog.smem_bytes = use_smem ? (int)smem : (int)std::max(fold_smem, tma_smem);
    prog.tma_stages =
        forced_tma ? forced_tma
                   : (unsigned)std::max<size_t>(2, std::min<size_t>(3, (size_t)prog.smem_bytes / dev::kTmaChunk));
    prog.tma = (any_tma ? 1 : 0) | (any_staged ? 2 : 0);
    // HICCL_NO_ALIAS_FENCE=1: measurement only (what the proxy fences cost)
    prog.alias_fence = stats.nvls_items > 0 && !env_flag("HICCL_NO_ALIAS_FENCE") ? 1 : 0;
    if (prog.smem_bytes > 48 * 1024)
      cuda_check(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      prog.smem_bytes),
                 "cudaFuncSetAttribute(smem)");
    prog.cta_checks = checked ? upload(cta_checks, tables) : nullptr;
    prog.checks = checked && !checks.empty() ? upload(checks, tables) : nullptr;
    prog.delay_exec = -1;
    prog.delay_ns = 0;
    if (checked && std::getenv("HICCL_TEST_DELAY_EXEC")) {
      prog.delay_exec = atoi(std::getenv("HICCL_TEST_DELAY_EXEC"));
      prog.delay_ns = std::getenv("HICCL_TEST_DELAY_NS") ? atoll(std::getenv("HICCL_TEST_DELAY_NS"))
                                                         : 2000000;
    }
    // HICCL_PROFILE_SOLO=1: no entry / exit barrier, so a profiler that
    // serializes kernels can replay one executor of a schedule with no
    // cross-executor waits (tools/profile_links.py); never for real runs.
    prog.solo = env_flag("HICCL_PROFILE_SOLO") ? 1 : 0;
    prog.tile_stride = (unsigned)Y.tile_stride;
    prog.tile_pub_every = std::getenv("HICCL_TILE_PUB") ? (unsigned)std::max(1, atoi(std::getenv("HICCL_TILE_PUB"))) : 1u;
    prog.cta_tile_waits = lp.tile_sync ? upload(cta_tile_waits, tables) : nullptr;
    prog.tile_waits = lp.tile_sync && !tile_waits.empty() ? upload(tile_waits, tables) : nullptr;
    prog.cta_waits = upload(cta_waits, tables);
    prog.waits = upload(waits, tables);
    prog.peer_flags = upload(pf, tables);
    prog.flags = flags;
    prog.arrive = arrive;
    prog.status = status_dev;
    prog.status_mirror = status_mapped;
    prog.num_steps = nsteps;
    prog.num_execs = cfg.num_execs;
    prog.self = self;
    prog.trace = trace;
    prog.timeout_ns = cfg.timeout_s > 0 ? (long long)(cfg.timeout_s * 1e9) : 0;
    prog.ll = sched.ll ? 1 : 0;
    prog.ll_half = (unsigned long long)sched.ll_half;

    stats.num_steps = nsteps;
    stats.copy_mode = cfg.copy_mode;
    stats.num_items = (int)items.size();
    stats.num_waits = (int)waits.size();
    stats.ctas = ctas;
    stats.threads = threads;
    stats.arena_bytes = (int64_t)arena_bytes;
    committed = true;
  }

  void start(cudaStream_t stream) {
    if (!committed) throw Error(ErrorCode::InvalidConfig, "hc_exec_start before hc_exec_commit");
    if (poisoned) throw Error(ErrorCode::Timeout, "executor poisoned by an earlier watchdog timeout");
    DeviceGuard g(device);
    if (!stream && own_stream) stream = own_stream;
    dev::Program p = prog;
    void* args[] = {&p};
    KernelFn fn = kernel_for(cfg.dtype, sched.ll, tile_mode);
    // Cooperative (co-resident CTAs) launch that stream capture accepts:
    // start() may be recorded into a CUDA graph and replayed; the epoch is
    // kept on the device.
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(ctas);
    lc.blockDim = dim3(threads);
    lc.dynamicSmemBytes = (size_t)prog.smem_bytes;
    lc.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    // HICCL_PLAIN_LAUNCH=1: no cooperative attribute (co-residency then
    // rests on the grid cap alone; the watchdog reports a grid that never
    // became resident as HC_TIMEOUT)
    static const bool plain = std::getenv("HICCL_PLAIN_LAUNCH") && atoi(std::getenv("HICCL_PLAIN_LAUNCH"));
    lc.numAttrs = plain ? 0 : 1;
    cuda_check(cudaLaunchKernelExC(&lc, (const void*)fn, args), "cudaLaunchKernelEx(cooperative)");
    ever_started = true;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(stream, &cap), "cudaStreamIsCapturing");
    if (cap == cudaStreamCaptureStatusNone) {
      // the status bits reach the host through the mapped mirror, so
      // start() is one launch and one event record, and wait() / query()
      // never touch the legacy stream
      cuda_check(cudaEventRecord(done, stream), "cudaEventRecord");
      launched = true;
    }
  }

  void wait() {
    if (!launched) {
      // only captured launches (CUDA graph replays the host never sees):
      // the caller has synchronized their stream; read the status mirror
      if (ever_started) check_watchdog();
      return;
    }
    DeviceGuard g(device);
    cuda_check(cudaEventSynchronize(done), "cudaEventSynchronize");
    check_watchdog();
  }

  // After `done` completed: the pinned copy holds the word as the kernel left it.
  void check_watchdog() {
    const volatile unsigned int* w = status_host;
    const unsigned int st = w[0];
    if (st & dev::kStatusDepViolation) {
      poisoned = true;
      throw Error(ErrorCode::DependencyViolation,
                  "step " + std::to_string(w[1]) + " of CTA " + std::to_string(w[2]) +
                      " was about to run before CTA " + std::to_string(w[3] & 0xFFFF) +
                      " of executor " + std::to_string(w[3] >> 16) + " finished step " +
                      std::to_string(w[4] / words_T - 1));
    }
    if (st) {
      poisoned = true;
      throw Error(ErrorCode::Timeout, "flag wait exceeded the watchdog timeout");
    }
  }
};

namespace {
using hiccl::capi::guard;

// cuMemGetAddressRange through the runtime's driver entry point, so the
// library never links libcuda directly (it must load on CPU-only hosts).
using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (AddrRangeFn) nullptr;
    return (AddrRangeFn)f;
  }();
  return fn;
}
}  // namespace

extern "C" {

hc_status hc_exec_create(const hc_plan* plan, const hc_exec_config* cfg, hc_exec** out) {
  return guard([&] {
    if (!plan || !cfg || !out) throw Error(ErrorCode::InvalidConfig, "null argument");
    auto ex = std::make_unique<hc_exec>();
    ex->plan = capi::plan_of(plan);
    ex->cfg = *cfg;
    const int p = ex->plan.base.world_size;
    if (cfg->num_execs < 1 || cfg->num_execs > dev::kMaxExecs)
      throw Error(ErrorCode::InvalidConfig, "num_execs out of range");
    if (cfg->exec_index < 0 || cfg->exec_index >= cfg->num_execs)
      throw Error(ErrorCode::InvalidConfig, "exec_index out of range");
    if (cfg->rank_to_exec)
      ex->rank_to_exec.assign(cfg->rank_to_exec, cfg->rank_to_exec + p);
    else if (cfg->num_execs == 1)
      ex->rank_to_exec.assign(p, 0);
    else
      throw Error(ErrorCode::InvalidConfig, "rank_to_exec required with several executors");
    ex->cfg.rank_to_exec = nullptr;
    ex->esize = element_size(cfg->dtype);
    ex->device = cfg->device;
    if (cfg->copy_mode == 4)
      ex->cfg.copy_mode = resolve_auto_mode(ex->plan, ex->esize, ex->rank_to_exec, cfg->num_execs);
    ex->sched = checked_schedule(ex->plan, ex->rank_to_exec, cfg->num_execs, ex->esize,
                                 copy_mode_of(ex->cfg.copy_mode));
    ex->peer_arena.assign(cfg->num_execs, nullptr);
    ex->peer_flags.assign(cfg->num_execs, nullptr);
    int64_t arena = ex->sched.arena_bytes[cfg->exec_index];
    if (cfg->copy_mode == 4 && ex->cfg.copy_mode == 3 && cfg->num_execs == p) {
      ex->auto_ll = true;  // commit() may fall back to push for NVLS windows
      const Schedule push = build_schedule(ex->plan, ex->rank_to_exec, cfg->num_execs, ex->esize,
                                           CopyMode::push);
      arena = std::max(arena, push.arena_bytes[cfg->exec_index]);
    }

    DeviceGuard g(ex->device);
    ex->arena_bytes = (size_t)arena;
    cuda_check(cudaMalloc(&ex->arena, std::max<size_t>(ex->arena_bytes, 256)), "cudaMalloc(arena)");
    // zero: no staging line may carry a valid tag before it is written
    cuda_check(cudaMemset(ex->arena, 0, std::max<size_t>(ex->arena_bytes, 256)), "cudaMemset(arena)");
    const size_t flag_words = dev::kMaxExecs + (size_t)dev::kMaxExecs * dev::kMaxCtas;
    cuda_check(cudaMalloc(&ex->flags, sizeof(uint64_t) * flag_words), "cudaMalloc(flags)");
    cuda_check(cudaMemset(ex->flags, 0, sizeof(uint64_t) * flag_words), "cudaMemset(flags)");
    ex->alloc_step_words();
    cuda_check(cudaMalloc(&ex->status_dev, kStatusWords * sizeof(unsigned int)), "cudaMalloc(status)");
    cuda_check(cudaMemset(ex->status_dev, 0, kStatusWords * sizeof(unsigned int)), "cudaMemset(status)");
    cuda_check(cudaHostAlloc((void**)&ex->status_host, kStatusWords * sizeof(unsigned int),
                             cudaHostAllocPortable | cudaHostAllocMapped),
               "cudaHostAlloc(status)");
    std::memset(ex->status_host, 0, kStatusWords * sizeof(unsigned int));
    cuda_check(cudaHostGetDevicePointer((void**)&ex->status_mapped, ex->status_host, 0),
               "cudaHostGetDevicePointer(status)");
    if (cfg->execs_per_device > 1)
      cuda_check(cudaStreamCreateWithFlags(&ex->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&ex->done, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    *out = ex.release();
  });
}

void hc_exec_destroy(hc_exec* ex) { delete ex; }

hc_status hc_exec_bind_buffer(hc_exec* ex, int rank, const char* name, void* ptr, size_t bytes) {
  return guard([&] {
    if (rank < 0 || rank >= ex->plan.base.world_size)
      throw Error(ErrorCode::RankOutOfRange, "rank " + std::to_string(rank));
    auto it = ex->plan.base.buffers.find(name);
    if (it == ex->plan.base.buffers.end())
      throw Error(ErrorCode::BadBufferRef, std::string("plan has no buffer '") + name + "'");
    if (it->second.internal)
      throw Error(ErrorCode::BadBufferRef, std::string("'") + name + "' is internal staging");
    if (!ptr) throw Error(ErrorCode::BadBufferRef, "null buffer pointer");
    ex->bindings[{rank, name}] = {(char*)ptr, bytes};
    ex->committed = false;
  });
}

hc_status hc_exec_bind_multicast(hc_exec* ex, const char* name, void* mc_ptr) {
  return guard([&] {
    auto it = ex->plan.base.buffers.find(name);
    if (it == ex->plan.base.buffers.end())
      throw Error(ErrorCode::BadBufferRef, std::string("plan has no buffer '") + name + "'");
    if (it->second.internal)
      throw Error(ErrorCode::BadBufferRef, std::string("'") + name + "' is internal staging");
    if (mc_ptr)
      ex->multicast[name] = (char*)mc_ptr;
    else
      ex->multicast.erase(name);
    ex->committed = false;
  });
}

hc_status hc_exec_local_arena(hc_exec* ex, void** ptr, size_t* bytes) {
  return guard([&] {
    *ptr = ex->arena;
    *bytes = ex->arena_bytes;
  });
}

hc_status hc_exec_bind_peer_arena(hc_exec* ex, int peer, void* ptr) {
  return guard([&] {
    if (peer < 0 || peer >= ex->cfg.num_execs) throw Error(ErrorCode::RankOutOfRange, "peer");
    ex->peer_arena[peer] = ptr;
    ex->committed = false;
  });
}

hc_status hc_exec_local_flags(hc_exec* ex, void** ptr, size_t* bytes) {
  return guard([&] {
    *ptr = ex->flags;
    *bytes = sizeof(uint64_t) * (dev::kMaxExecs + (size_t)dev::kMaxExecs * dev::kMaxCtas);
  });
}

hc_status hc_exec_bind_peer_flags(hc_exec* ex, int peer, void* ptr) {
  return guard([&] {
    if (peer < 0 || peer >= ex->cfg.num_execs) throw Error(ErrorCode::RankOutOfRange, "peer");
    ex->peer_flags[peer] = (uint64_t*)ptr;
    ex->committed = false;
  });
}

// NVTX ranges (header-only nvtx3: free unless a profiler is attached)
// around the three host calls of Comm::init / start / wait.
hc_status hc_exec_commit(hc_exec* ex) {
  nvtx3::scoped_range r{"hiccl init (commit)"};
  return guard([&] { ex->commit(); });
}

hc_status hc_exec_start(hc_exec* ex, void* stream) {
  nvtx3::scoped_range r{"hiccl start"};
  return guard([&] { ex->start((cudaStream_t)stream); });
}

hc_status hc_exec_wait(hc_exec* ex) {
  nvtx3::scoped_range r{"hiccl wait"};
  return guard([&] { ex->wait(); });
}

hc_status hc_exec_query(hc_exec* ex, int* done) {
  return guard([&] {
    if (!ex->launched) {
      *done = 1;
      return;
    }
    DeviceGuard g(ex->device);
    cudaError_t e = cudaEventQuery(ex->done);
    if (e == cudaErrorNotReady) {
      *done = 0;
      return;
    }
    cuda_check(e, "cudaEventQuery");
    *done = 1;
    ex->check_watchdog();
  });
}

hc_status hc_exec_get_trace(hc_exec* ex, int64_t* out, int n) {
  return guard([&] {
    const int base_n = (int)ex->sched.step_slot.size() + 4;
    if (n < base_n) throw Error(ErrorCode::InvalidConfig, "trace needs " + std::to_string(base_n) + " entries");
    const int need = std::min(n, base_n + 128);  // + per-warp debug stamps (ll)
    if (!ex->launched) throw Error(ErrorCode::InvalidConfig, "no launch to trace");
    DeviceGuard g(ex->device);
    cuda_check(cudaEventSynchronize(ex->done), "cudaEventSynchronize");
    std::vector<unsigned long long> t(need);
    cuda_check(cudaMemcpy(t.data(), ex->trace, need * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
               "read trace");
    for (int i = 0; i < need; ++i) out[i] = (int64_t)t[i];
  });
}

hc_status hc_exec_get_stats(const hc_exec* ex, hc_exec_stats* out) {
  return guard([&] { *out = ex->stats; });
}

hc_status hc_enable_peer_access(const int* devices, int n) {
  return guard([&] {
    for (int i = 0; i < n; ++i) {
      DeviceGuard g(devices[i]);
      for (int j = 0; j < n; ++j) {
        if (i == j || devices[i] == devices[j]) continue;
        int can = 0;
        cuda_check(cudaDeviceCanAccessPeer(&can, devices[i], devices[j]), "cudaDeviceCanAccessPeer");
        if (!can)
          throw Error(ErrorCode::CudaError, "device " + std::to_string(devices[i]) +
                                                " cannot access peer " + std::to_string(devices[j]));
        cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          continue;
        }
        cuda_check(e, "cudaDeviceEnablePeerAccess");
      }
    }
  });
}

hc_status hc_ipc_export(void* ptr, unsigned char handle[64], size_t* offset) {
  return guard([&] {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    CUdeviceptr base = 0;
    size_t size = 0;
    AddrRangeFn fn = addr_range_fn();
    if (!fn || fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
      throw Error(ErrorCode::CudaError, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    cuda_check(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, 64);
    *offset = (size_t)((CUdeviceptr)ptr - base);
  });
}

hc_status hc_ipc_import(const unsigned char handle[64], size_t offset, int device, void** ptr) {
  return guard([&] {
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* base = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    *ptr = (char*)base + offset;
  });
}

hc_status hc_device_range(const void* ptr, void** base, size_t* bytes) {
  return guard([&] {
    CUdeviceptr b = 0;
    size_t n = 0;
    AddrRangeFn fn = addr_range_fn();
    if (!fn || fn(&b, &n, (CUdeviceptr)ptr) != CUDA_SUCCESS)
      throw Error(ErrorCode::BadBufferRef, "pointer is not device memory (cuMemGetAddressRange)");
    *base = (void*)b;
    *bytes = n;
  });
}

hc_status hc_ipc_close(void* base_ptr) {
  return guard([&] { cuda_check(cudaIpcCloseMemHandle(base_ptr), "cudaIpcCloseMemHandle"); });
}

hc_status hc_device_alloc(int device, size_t bytes, void** ptr) {
  return guard([&] {
    DeviceGuard g(device);
    cuda_check(cudaMalloc(ptr, std::max<size_t>(bytes, 16)), "cudaMalloc");
  });
}

hc_status hc_device_free(int device, void* ptr) {
  return guard([&] {
    DeviceGuard g(device);
    cuda_check(cudaFree(ptr), "cudaFree");
  });
}

hc_status hc_device_count(int* n) {
  return guard([&] {
    *n = 0;
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      *n = 0;
    }
  });
}

hc_status hc_device_sync(int device) {
  return guard([&] {
    DeviceGuard g(device);
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  });
}

hc_status hc_device_fill(int device, void* ptr, int64_t count, int dtype, uint64_t seed, int rank,
                         int64_t index_base, void* stream) {
  return guard([&] {
    DeviceGuard g(device);
    if (count <= 0) return;
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((count + threads - 1) / threads, 148 * 16);
    cudaStream_t s = (cudaStream_t)stream;
    switch (dtype) {
      case HC_F32: dev::fill_kernel<0><<<blocks, threads, 0, s>>>(ptr, count, seed, rank, index_base); break;
      case HC_BF16: dev::fill_kernel<1><<<blocks, threads, 0, s>>>(ptr, count, seed, rank, index_base); break;
      case HC_F16: dev::fill_kernel<2><<<blocks, threads, 0, s>>>(ptr, count, seed, rank, index_base); break;
      case HC_I32: dev::fill_kernel<3><<<blocks, threads, 0, s>>>(ptr, count, seed, rank, index_base); break;
      case HC_I64: dev::fill_kernel<4><<<blocks, threads, 0, s>>>(ptr, count, seed, rank, index_base); break;
      case HC_F64: dev::fill_kernel<5><<<blocks, threads, 0, s>>>(ptr, count, seed, rank, index_base); break;
      case HC_U8: dev::fill_kernel<6><<<blocks, threads, 0, s>>>(ptr, count, seed, rank, index_base); break;
      default: throw Error(ErrorCode::InvalidConfig, "unknown dtype");
    }
    cuda_check(cudaGetLastError(), "fill_kernel launch");
  });
}

}  // extern "C"
