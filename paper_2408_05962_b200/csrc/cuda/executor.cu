// Host side of the persistent executor: schedule -> device tables,
// buffers/arena/flags, cooperative launch, C ABI (include/hiccl.h).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../host/capi_common.hpp"
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

using KernelFn = void (*)(dev::Program, unsigned long long);

KernelFn kernel_for(int dtype) {
  switch (dtype) {
    case HC_F32: return dev::persistent_executor<0>;
    case HC_BF16: return dev::persistent_executor<1>;
    case HC_F16: return dev::persistent_executor<2>;
    case HC_I32: return dev::persistent_executor<3>;
    case HC_I64: return dev::persistent_executor<4>;
    case HC_F64: return dev::persistent_executor<5>;
    case HC_U8: return dev::persistent_executor<6>;
  }
  throw Error(ErrorCode::InvalidConfig, "unknown dtype");
}

}  // namespace

struct hc_exec {
  PipelinedPlan plan;
  hc_exec_config cfg{};
  std::vector<int> rank_to_exec;
  Schedule sched;
  int esize = 4;
  int device = 0;

  void* arena = nullptr;
  size_t arena_bytes = 0;
  uint64_t* flags = nullptr;
  unsigned long long* arrive = nullptr;
  unsigned long long* trace = nullptr;  // device stamps of the last launch
  unsigned int* status_dev = nullptr;  // watchdog word, read back after completion
  bool poisoned = false;
  std::vector<void*> peer_arena;
  std::vector<uint64_t*> peer_flags;
  std::map<std::pair<int, std::string>, std::pair<char*, size_t>> bindings;
  std::map<std::string, char*> multicast;  // buffer name -> multicast address (NVLS)

  std::vector<void*> tables;  // device allocations owned by commit
  dev::Program prog{};
  bool committed = false;
  int ctas = 0, threads = 0;
  unsigned long long epoch = 0;
  cudaEvent_t done = nullptr;
  bool launched = false;
  hc_exec_stats stats{};

  ~hc_exec() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (launched && done) cudaEventSynchronize(done);
    for (void* p : tables) cudaFree(p);
    if (arena) cudaFree(arena);
    if (flags) cudaFree(flags);
    if (arrive) cudaFree(arrive);
    if (trace) cudaFree(trace);
    if (status_dev) cudaFree(status_dev);
    if (done) cudaEventDestroy(done);
    if (prev >= 0) cudaSetDevice(prev);
  }

  void free_tables() {
    for (void* p : tables) cudaFree(p);
    tables.clear();
  }

  char* address(const Loc& l, int64_t count) {
    const BufferDecl& d = sched.buffer_decls[l.buffer];
    const std::string& name = sched.buffer_names[l.buffer];
    if (d.internal) {
      const int x = rank_to_exec[l.rank];
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

  struct Emit {
    char* dst;
    std::vector<char*> srcs;
    int64_t count;
    ReduceOp op;
    uint8_t flags;  // dev::kMcReduce / dev::kMcStore
  };

  char* multicast_of(int buffer) const {
    auto it = multicast.find(sched.buffer_names[buffer]);
    return it == multicast.end() ? nullptr : it->second;
  }

  bool nvls_reduce_supported(ReduceOp op) const {
    switch (cfg.dtype) {
      case HC_F32: case HC_BF16: case HC_F16: return op == ReduceOp::sum;
      case HC_I32: return true;
      default: return false;
    }
  }

  // One step of this executor -> device items. With NVLS windows bound
  // (hc_exec_bind_multicast), and one rank per executor:
  //  * a write group that folds the same (buffer, offset) of EVERY rank
  //    becomes one multimem.ld_reduce item (reduced in the switch);
  //  * copies of one source range to the same (buffer, offset) of every
  //    other rank (the source's own range being that range, or also
  //    targeted) become one multimem.st item.
  // Everything else keeps the point-to-point form.
  std::vector<Emit> lower_step(const std::vector<int>& order, int self) {
    std::vector<Emit> out;
    const int P = sched.world_size;
    bool nvls = !multicast.empty() && cfg.num_execs == P;
    if (nvls) {
      std::vector<int> seen(cfg.num_execs, 0);
      for (int r = 0; r < P; ++r) nvls &= !seen[rank_to_exec[r]]++;
    }
    auto aligned = [&](const char* a) { return ((uintptr_t)a % 16) == 0; };
    std::vector<bool> used(order.size(), false);
    for (size_t i = 0; i < order.size(); ++i) {
      if (used[i]) continue;
      const WorkItem& w = sched.items[order[i]];
      const bool whole_vectors = (w.count * esize) % 16 == 0;
      if (nvls && whole_vectors && !w.reads_dst && (int)w.srcs.size() == P &&
          nvls_reduce_supported(w.op)) {
        char* mc = multicast_of(w.srcs[0].buffer);
        bool all = mc != nullptr;
        std::vector<int> hit(P, 0);
        for (const Loc& l : w.srcs) {
          all &= l.buffer == w.srcs[0].buffer && l.offset == w.srcs[0].offset;
          hit[l.rank]++;
        }
        for (int r = 0; r < P; ++r) all &= hit[r] == 1;
        char* dst = address(w.dst, w.count);
        char* src = all ? mc + w.srcs[0].offset * esize : nullptr;
        if (all && aligned(dst) && aligned(src)) {
          out.push_back(Emit{dst, {src}, w.count, w.op, dev::kMcReduce});
          used[i] = true;
          continue;
        }
      }
      const bool copy = !w.reads_dst && w.srcs.size() == 1;
      if (nvls && whole_vectors && copy && rank_to_exec[w.srcs[0].rank] == self &&
          multicast_of(w.dst.buffer)) {
        // gather the same-source copies of this step
        const Loc& s0 = w.srcs[0];
        std::vector<size_t> group;
        std::vector<int> hit(P, 0);
        for (size_t j = i; j < order.size(); ++j) {
          if (used[j]) continue;
          const WorkItem& x = sched.items[order[j]];
          if (x.reads_dst || x.srcs.size() != 1 || x.count != w.count) continue;
          const Loc& sx = x.srcs[0];
          if (sx.rank != s0.rank || sx.buffer != s0.buffer || sx.offset != s0.offset) continue;
          if (x.dst.buffer != w.dst.buffer || x.dst.offset != w.dst.offset) continue;
          group.push_back(j);
          hit[x.dst.rank] = 1;
        }
        // the multicast also writes the source rank's own copy of the range
        const bool self_ok = hit[s0.rank] || (s0.buffer == w.dst.buffer && s0.offset == w.dst.offset);
        bool all = self_ok;
        for (int r = 0; r < P; ++r) all &= hit[r] || r == s0.rank;
        char* mc = multicast_of(w.dst.buffer) + w.dst.offset * esize;
        char* src = address(s0, w.count);
        if (all && aligned(mc) && aligned(src)) {
          for (size_t j : group) used[j] = true;
          out.push_back(Emit{mc, {src}, w.count, w.op, dev::kMcStore});
          continue;
        }
      }
      Emit e{address(w.dst, w.count), {}, w.count, w.op, 0};
      for (const Loc& l : w.srcs) e.srcs.push_back(address(l, w.count));
      out.push_back(std::move(e));
      used[i] = true;
    }
    for (size_t i = 0; i < order.size(); ++i) {  // traffic accounting (plan view)
      const WorkItem& w = sched.items[order[i]];
      const int64_t bytes = w.count * esize;
      for (const Loc& l : w.srcs) {
        stats.bytes_in += bytes;
        if (rank_to_exec[l.rank] != self) stats.remote_bytes += bytes;
      }
      stats.bytes_out += bytes;
      if (rank_to_exec[w.dst.rank] != self) stats.remote_bytes += bytes;
    }
    return out;
  }

  void commit() {
    DeviceGuard g(device);
    free_tables();
    const int self = cfg.exec_index;
    const int nsteps = (int)sched.step_slot.size();
    const ExecProgram& ep = sched.execs[self];
    int first_rank = 0;
    while (first_rank < sched.world_size && rank_to_exec[first_rank] != self) ++first_rank;

    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    threads = cfg.threads > 0 ? cfg.threads : 512;
    if (threads % 32 || threads < 64 || threads > 512)
      throw Error(ErrorCode::InvalidConfig, "threads must be a multiple of 32 in [64, 512]");
    KernelFn fn = kernel_for(cfg.dtype);
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, threads, 0),
               "occupancy");
    const int max_ctas = per_sm * prop.multiProcessorCount;
    // Grid: one CTA per SM, fewer when no step has enough bytes to give
    // every CTA at least two 16-byte vectors per thread (small messages
    // then pay for fewer arrivals and fences).
    int64_t max_step_bytes = 0;
    for (int s = 0; s < nsteps; ++s) {
      int64_t b = 0;
      for (int k : ep.items_by_step[s]) b += sched.items[k].count * esize;
      max_step_bytes = std::max(max_step_bytes, b);
    }
    const int64_t min_tile = (int64_t)threads * 16 * 2;
    const int auto_ctas = (int)std::max<int64_t>(
        1, std::min<int64_t>(prop.multiProcessorCount, (max_step_bytes + min_tile - 1) / min_tile));
    ctas = cfg.ctas > 0 ? cfg.ctas : std::min(max_ctas, auto_ctas);
    if (ctas > max_ctas)
      throw Error(ErrorCode::InvalidConfig, "ctas " + std::to_string(ctas) +
                                                " exceed co-resident capacity " + std::to_string(max_ctas));

    std::vector<dev::Step> steps(nsteps);
    std::vector<dev::Item> items;
    std::vector<uint64_t> srcs;
    std::vector<dev::Wait> waits;
    stats = hc_exec_stats{};
    for (int s = 0; s < nsteps; ++s) {
      dev::Step& st = steps[s];
      st.item_first = (uint32_t)items.size();
      st.wait_first = (uint32_t)waits.size();
      uint32_t tiles = 0;
      // Peer rotation: order this step's items by the distance from our
      // first rank to the peer they talk to, so executors start on
      // different peers instead of all hitting rank 0 first.
      std::vector<int> order = ep.items_by_step[s];
      const int me = first_rank;
      auto peer_of = [&](const WorkItem& w) {
        if (rank_to_exec[w.dst.rank] != self) return w.dst.rank;  // push: remote write
        for (const Loc& l : w.srcs)
          if (rank_to_exec[l.rank] != self) return l.rank;
        return w.dst.rank;
      };
      const int P = sched.world_size;
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return (peer_of(sched.items[a]) - me + P) % P < (peer_of(sched.items[b]) - me + P) % P;
      });
      // Resolve addresses; lower onto NVLS where buffers sit in a window.
      std::vector<Emit> emits = lower_step(order, self);
      // Tile size of this step: the largest of threads * {8,4,2,1} vectors
      // that still gives every CTA a tile.
      int kv = dev::kTileVec;
      for (; kv > 1; kv /= 2) {
        const int64_t te = (int64_t)threads * kv * 16 / esize;
        int64_t nt = 0;
        for (const Emit& e : emits) nt += (e.count + te - 1) / te;
        if (nt >= ctas) break;
      }
      const int tile_elems = threads * kv * 16 / esize;
      st.tile_elems = (uint32_t)tile_elems;
      uint32_t first_tiles = 0;
      bool uniform = !emits.empty();
      for (const Emit& e : emits) {
        dev::Item it{};
        it.dst = (uint64_t)e.dst;
        it.count = e.count;
        it.src_first = (uint32_t)srcs.size();
        it.n_src = (uint16_t)e.srcs.size();
        it.op = (uint8_t)e.op;
        bool vec = true;
        for (char* a : e.srcs) {
          srcs.push_back((uint64_t)a);
          vec &= ((uint64_t)a % 16) == ((uint64_t)e.dst % 16);
        }
        it.flags = (uint8_t)((vec ? dev::kVec : 0) | e.flags);
        if (e.flags) ++stats.nvls_items;
        it.tile_first = tiles;
        it.n_tiles = (uint32_t)((e.count + tile_elems - 1) / tile_elems);
        if (tiles == 0) first_tiles = it.n_tiles;
        uniform &= it.n_tiles == first_tiles;
        tiles += it.n_tiles;
        items.push_back(it);
      }
      st.n_items = (uint32_t)items.size() - st.item_first;
      st.n_tiles = tiles;
      for (const StepWait& w : ep.waits[s]) waits.push_back(dev::Wait{(uint32_t)w.exec, (uint32_t)(w.step + 1)});
      st.n_waits = (uint32_t)waits.size() - st.wait_first;
      if (st.n_waits > (uint32_t)threads)
        throw Error(ErrorCode::InvalidConfig, "more wait edges than threads");
      st.publish = ep.publish[s] ? 1 : 0;
      st.uniform = (uniform && st.n_items > 1) ? 1 : 0;
    }
    std::vector<uint64_t*> pf(cfg.num_execs);
    for (int x = 0; x < cfg.num_execs; ++x) {
      pf[x] = x == self ? flags : peer_flags[x];
      if (!pf[x])
        throw Error(ErrorCode::BadBufferRef,
                    "flags of executor " + std::to_string(x) + " not bound (hc_exec_bind_peer_flags)");
    }
    prog.steps = upload(steps, tables);
    prog.items = upload(items, tables);
    prog.srcs = upload(srcs, tables);
    prog.waits = upload(waits, tables);
    prog.peer_flags = upload(pf, tables);
    prog.flags = flags;
    prog.arrive = arrive;
    prog.status = status_dev;
    prog.num_steps = nsteps;
    prog.num_execs = cfg.num_execs;
    prog.self = self;
    prog.trace = trace;
    prog.timeout_ns = cfg.timeout_s > 0 ? (long long)(cfg.timeout_s * 1e9) : 0;

    stats.num_steps = nsteps;
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
    ++epoch;
    dev::Program p = prog;
    unsigned long long e = epoch;
    void* args[] = {&p, &e};
    KernelFn fn = kernel_for(cfg.dtype);
    cuda_check(cudaLaunchCooperativeKernel((const void*)fn, dim3(ctas), dim3(threads), args, 0, stream),
               "cudaLaunchCooperativeKernel");
    cuda_check(cudaEventRecord(done, stream), "cudaEventRecord");
    launched = true;
  }

  void wait() {
    if (!launched) return;
    DeviceGuard g(device);
    cuda_check(cudaEventSynchronize(done), "cudaEventSynchronize");
    check_watchdog();
  }

  void check_watchdog() {
    unsigned int st = 0;
    cuda_check(cudaMemcpy(&st, status_dev, sizeof st, cudaMemcpyDeviceToHost), "read watchdog");
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
    ex->sched = build_schedule(ex->plan, ex->rank_to_exec, cfg->num_execs, ex->esize,
                               cfg->copy_mode ? CopyMode::push : CopyMode::pull);
    ex->peer_arena.assign(cfg->num_execs, nullptr);
    ex->peer_flags.assign(cfg->num_execs, nullptr);

    DeviceGuard g(ex->device);
    ex->arena_bytes = (size_t)ex->sched.arena_bytes[cfg->exec_index];
    cuda_check(cudaMalloc(&ex->arena, std::max<size_t>(ex->arena_bytes, 256)), "cudaMalloc(arena)");
    cuda_check(cudaMalloc(&ex->flags, sizeof(uint64_t) * dev::kMaxExecs), "cudaMalloc(flags)");
    cuda_check(cudaMemset(ex->flags, 0, sizeof(uint64_t) * dev::kMaxExecs), "cudaMemset(flags)");
    const size_t nsteps = ex->sched.step_slot.size();
    cuda_check(cudaMalloc(&ex->arrive, sizeof(unsigned long long) * (nsteps + 1)), "cudaMalloc(arrive)");
    cuda_check(cudaMemset(ex->arrive, 0, sizeof(unsigned long long) * (nsteps + 1)), "cudaMemset(arrive)");
    cuda_check(cudaMalloc(&ex->trace, sizeof(unsigned long long) * (nsteps + 4)), "cudaMalloc(trace)");
    cuda_check(cudaMalloc(&ex->status_dev, sizeof(unsigned int)), "cudaMalloc(status)");
    cuda_check(cudaMemset(ex->status_dev, 0, sizeof(unsigned int)), "cudaMemset(status)");
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
    *bytes = sizeof(uint64_t) * dev::kMaxExecs;
  });
}

hc_status hc_exec_bind_peer_flags(hc_exec* ex, int peer, void* ptr) {
  return guard([&] {
    if (peer < 0 || peer >= ex->cfg.num_execs) throw Error(ErrorCode::RankOutOfRange, "peer");
    ex->peer_flags[peer] = (uint64_t*)ptr;
    ex->committed = false;
  });
}

hc_status hc_exec_commit(hc_exec* ex) { return guard([&] { ex->commit(); }); }

hc_status hc_exec_start(hc_exec* ex, void* stream) {
  return guard([&] { ex->start((cudaStream_t)stream); });
}

hc_status hc_exec_wait(hc_exec* ex) { return guard([&] { ex->wait(); }); }

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
    const int need = (int)ex->sched.step_slot.size() + 4;
    if (n < need) throw Error(ErrorCode::InvalidConfig, "trace needs " + std::to_string(need) + " entries");
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
