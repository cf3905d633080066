// hiccl::Comm<T> — the paper's user API over
// the C ABI in hiccl.h. Header-only: include it and link libhiccl.so.
//
//   hiccl::Comm<float> comm(rank, world, device, allgather);   // one process per GPU
//   for (int j = 0; j < p; ++j)                                 // reduce-scatter
//     comm.add_reduction(send + j * n, recv + j * n, n, all, j, hiccl::op::sum);
//   comm.add_fence();
//   for (int i = 0; i < p; ++i)                                 // all-gather in place
//     comm.add_multicast(recv + i * n, recv + i * n, n, i, others(i));
//   comm.init({p}, {"IPC"}, /*ring*/ 1, /*stripe*/ 1, /*pipeline*/ 1);
//   comm.start(stream);  ...  comm.wait();
//
// With send/recv from comm.alloc_nvls(count) and library {"NVLS"}, the same
// composition runs through the NVSwitch (multimem, fused per tile).
//
// Every rank registers the same composition with its own pointers
// (PAPER.md:238-239). A pointer is mapped to (buffer, element offset): the
// buffer is the device allocation that contains it, numbered in order of
// first use, so allocations must correspond across ranks (the same call
// sequence on every rank). The reference's equivalent is
// CollectiveProgram::add_* over named BufferRefs (composition.hpp:80-90),
// lowered by lower() + pipeline() (factorize.hpp:107, pipeline.hpp:40) and
// executed by execute_plan() (engine.hpp:127); here init() lowers once
// (persistent) and start()/wait() launch and join the
// persistent sm_100a executor.
//
// Bootstrap: the paper uses MPI for setup. `allgather`
// receives this process's blob and must return every process's blob in
// rank order (wrap MPI_Allgather, torch.distributed, a socket, ...).
#pragma once

#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hiccl.h"

#if __has_include(<cuda_bf16.h>)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#define HICCL_HAVE_CUDA_HALF 1
#endif

namespace hiccl {

enum class op { sum = HC_OP_SUM, max = HC_OP_MAX };

template <class T> struct dtype_of;
template <> struct dtype_of<float> { static constexpr int value = HC_F32; };
template <> struct dtype_of<double> { static constexpr int value = HC_F64; };
template <> struct dtype_of<int32_t> { static constexpr int value = HC_I32; };
template <> struct dtype_of<int64_t> { static constexpr int value = HC_I64; };
template <> struct dtype_of<uint8_t> { static constexpr int value = HC_U8; };
#ifdef HICCL_HAVE_CUDA_HALF
// 16-bit floats: widen to fp32, add, round to nearest even after every
// fold (the executor and the oracle state the same rule)
template <> struct dtype_of<__nv_bfloat16> { static constexpr int value = HC_BF16; };
template <> struct dtype_of<__half> { static constexpr int value = HC_F16; };
#endif

/// Raised for any non-OK status; `status` is 1 + the reference ErrorCode.
class CommError : public std::runtime_error {
 public:
  CommError(int status, const std::string& what) : std::runtime_error(what), status(status) {}
  int status;
};

inline void check(hc_status s) {
  if (s != HC_OK) throw CommError(s, hc_last_error());
}

using Allgather = std::function<std::vector<std::string>(const std::string&)>;

template <class T, int DT = dtype_of<T>::value>
class Comm {
 public:
  /// One process per GPU: this process serves `rank` of `world` ranks on `device`.
  Comm(int rank, int world, int device, Allgather allgather)
      : rank_(rank), world_(world), device_(device), allgather_(std::move(allgather)) {
    check(hc_program_create(world, &prog_));
  }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  ~Comm() {
    if (exec_) hc_exec_destroy(exec_);
    for (void* base : imported_) hc_ipc_close(base);
    for (auto& w : windows_) hc_window_destroy(w.win);
    if (plan_) hc_plan_destroy(plan_);
    if (prog_) hc_program_destroy(prog_);
  }

  /// Symmetric device memory for `count` elements inside an NVSwitch
  /// multicast window (the per-level library "NVLS"). Collective: every rank
  /// calls it with the same count, in the same order, before init(). Pointers
  /// into it compose like any other; init() binds the window's multicast
  /// address too, so every-rank reductions and in-place every-rank
  /// multicasts over it run as multimem.ld_reduce / multimem.st (an
  /// all-reduce as one fused reduce+multicast pass). Freed with the Comm.
  T* alloc_nvls(size_t count) {
    if (plan_) throw CommError(HC_INVALID_CONFIG, "alloc_nvls after init()");
    const size_t align = size_t(2) << 20;
    const size_t bytes = (count * sizeof(T) + align - 1) / align * align;
    Window w{};
    unsigned char h[64] = {0};
    if (rank_ == 0) {
      check(hc_window_open(device_, world_, bytes, nullptr, &w.win));
      check(hc_window_export(w.win, h));
    }
    const std::vector<std::string> hs = allgather_(std::string(reinterpret_cast<char*>(h), 64));
    if ((int)hs.size() != world_ || hs[0].size() != 64)
      throw CommError(HC_INTERNAL, "allgather returned wrong size");
    if (rank_ != 0)
      check(hc_window_open(device_, world_, bytes,
                           reinterpret_cast<const unsigned char*>(hs[0].data()), &w.win));
    allgather_(std::string());  // every member added its device before anyone binds
    check(hc_window_bind(w.win));
    check(hc_window_export_memory(w.win, h));
    const std::vector<std::string> mems = allgather_(std::string(reinterpret_cast<char*>(h), 64));
    w.peer.assign(world_, nullptr);
    for (int r = 0; r < world_; ++r)
      if (r != rank_)
        check(hc_window_import_memory(w.win, reinterpret_cast<const unsigned char*>(mems[r].data()),
                                      &w.peer[r]));
    allgather_(std::string());
    size_t got = 0;
    check(hc_window_pointers(w.win, 0, &w.uc, &w.mc, &got));
    w.peer[rank_] = w.uc;
    Buffer b{"buf" + std::to_string(buffers_.size()), static_cast<char*>(w.uc), bytes,
             (int)windows_.size()};
    check(hc_program_declare_buffer(prog_, b.name.c_str(), (int64_t)(bytes / sizeof(T)), 1, 0));
    windows_.push_back(std::move(w));
    buffers_.push_back(b);
    return reinterpret_cast<T*>(b.base);
  }

  /// Comm<T>::add_multicast(sendbuf, recvbuf, count, i, j_vec):
  /// rank i's send range replicates into recv of every rank in j_vec.
  void add_multicast(T* sendbuf, T* recvbuf, size_t count, int i, std::vector<int> j_vec) {
    auto s = locate(sendbuf, count), r = locate(recvbuf, count);
    check(hc_program_add_multicast(prog_, s.first.c_str(), s.second, r.first.c_str(), r.second,
                                   (int64_t)count, i, j_vec.data(), (int)j_vec.size()));
  }

  /// Comm<T>::add_reduction(sendbuf, recvbuf, count, i_vec, j, op):
  /// the send ranges of i_vec fold with `o` into rank j's recv range.
  void add_reduction(T* sendbuf, T* recvbuf, size_t count, std::vector<int> i_vec, int j,
                     op o = op::sum) {
    auto s = locate(sendbuf, count), r = locate(recvbuf, count);
    check(hc_program_add_reduction(prog_, s.first.c_str(), s.second, r.first.c_str(), r.second,
                                   (int64_t)count, i_vec.data(), (int)i_vec.size(), j, (int)o));
  }

  /// Comm<T>::add_fence(): later primitives depend on earlier ones.
  void add_fence() { check(hc_program_add_fence(prog_)); }

  /// init(hierarchy, library, ring, stripe, pipeline):
  /// lower + pipeline once, build this rank's executor, exchange IPC handles.
  void init(std::vector<int> hierarchy, std::vector<std::string> library, int ring = 1,
            int stripe = 1, int pipeline = 1, int gpus_per_node = 0) {
    std::vector<const char*> lib;
    for (auto& l : library) lib.push_back(l.c_str());
    int p = 1;
    for (int h : hierarchy) p *= h;
    hc_machine_desc m{hierarchy.data(), (int)hierarchy.size(), gpus_per_node ? gpus_per_node : p,
                      library.empty() ? nullptr : lib.data()};
    check(hc_plan_lower(prog_, &m, ring, stripe, pipeline, &plan_));
    std::vector<int> r2e(world_);
    for (int r = 0; r < world_; ++r) r2e[r] = r;
    // copy mode: the cost model's choice (4 = auto), unless a level names
    // the NVLS library — an explicit request for switch reductions /
    // multicasts, which only the point-to-point push schedule lowers to
    bool nvls = false;
    for (auto& l : library) nvls |= l == "NVLS";
    hc_exec_config cfg{device_, rank_, world_, r2e.data(), DT, 0, 0, nvls ? 1 : 4, 60.0, 1};
    check(hc_exec_create(plan_, &cfg, &exec_));
    // bootstrap blob: arena, flags, then every user buffer of this rank
    std::string blob;
    void* ptr = nullptr;
    size_t bytes = 0;
    check(hc_exec_local_arena(exec_, &ptr, &bytes));
    append_handle(blob, ptr);
    check(hc_exec_local_flags(exec_, &ptr, &bytes));
    append_handle(blob, ptr);
    for (auto& b : buffers_) {
      if (b.window >= 0) {  // every member's address is known from the window
        const Window& w = windows_[b.window];
        for (int r = 0; r < world_; ++r)
          check(hc_exec_bind_buffer(exec_, r, b.name.c_str(), w.peer[r], b.bytes));
        check(hc_exec_bind_multicast(exec_, b.name.c_str(), w.mc));
        continue;
      }
      check(hc_exec_bind_buffer(exec_, rank_, b.name.c_str(), b.base, b.bytes));
      append_handle(blob, b.base);
      blob.append(reinterpret_cast<const char*>(&b.bytes), sizeof b.bytes);
    }
    const std::vector<std::string> all = allgather_(blob);
    if ((int)all.size() != world_) throw CommError(HC_INTERNAL, "allgather returned wrong size");
    for (int peer = 0; peer < world_; ++peer) {
      if (peer == rank_) continue;
      const std::string& pb = all[peer];
      size_t at = 0;
      check(hc_exec_bind_peer_arena(exec_, peer, open(pb, at)));
      check(hc_exec_bind_peer_flags(exec_, peer, open(pb, at)));
      for (auto& b : buffers_) {
        if (b.window >= 0) continue;
        void* ptr = open(pb, at);
        size_t bytes = 0;
        if (at + sizeof bytes > pb.size()) throw CommError(HC_PARSE_ERROR, "short bootstrap blob");
        std::memcpy(&bytes, pb.data() + at, sizeof bytes);
        at += sizeof bytes;
        check(hc_exec_bind_buffer(exec_, peer, b.name.c_str(), ptr, bytes));
      }
    }
    check(hc_exec_commit(exec_));
  }

  /// Non-blocking start on `stream` (cudaStream_t; nullptr = default).
  void start(void* stream = nullptr) { check(hc_exec_start(exec_, stream)); }
  /// Blocks until this rank's buffers are reusable.
  void wait() { check(hc_exec_wait(exec_)); }

  hc_exec_stats stats() const {
    hc_exec_stats s{};
    check(hc_exec_get_stats(exec_, &s));
    return s;
  }
  std::string plan_json() const {
    char* s = nullptr;
    check(hc_plan_serialize(plan_, &s));
    std::string out(s);
    hc_free(s);
    return out;
  }

 private:
  struct Buffer {
    std::string name;
    char* base;
    size_t bytes;
    int window = -1;  // index into windows_ (alloc_nvls), or -1
  };
  struct Window {
    hc_window* win = nullptr;
    void* uc = nullptr;       // this member's memory
    void* mc = nullptr;       // multicast address on this device
    std::vector<void*> peer;  // every member's memory as mapped here
  };

  // Device allocation containing p -> (buffer name, element offset). A new
  // allocation becomes buffer "buf<k>", declared as an input (user memory
  // is always initialized) of its full length, so the reference's eager
  // checks (composition.cpp:114-153) fire inside add_* as they do there.
  std::pair<std::string, int64_t> locate(T* p, size_t count) {
    if (plan_) throw CommError(HC_INVALID_CONFIG, "add_* after init()");
    char* c = reinterpret_cast<char*>(p);
    for (auto& b : buffers_)
      if (c >= b.base && c < b.base + b.bytes) return {b.name, offset_in(b, c)};
    void* base = nullptr;
    size_t bytes = 0;
    check(hc_device_range(p, &base, &bytes));
    Buffer b{"buf" + std::to_string(buffers_.size()), static_cast<char*>(base), bytes, -1};
    check(hc_program_declare_buffer(prog_, b.name.c_str(), (int64_t)(bytes / sizeof(T)), 1, 0));
    buffers_.push_back(b);
    return {b.name, offset_in(buffers_.back(), c)};
  }

  static int64_t offset_in(const Buffer& b, const char* c) {
    const int64_t off = (int64_t)(c - b.base);
    if (off % (int64_t)sizeof(T)) throw CommError(HC_BAD_BUFFER_REF, "misaligned pointer");
    return off / (int64_t)sizeof(T);
  }

  static void append_handle(std::string& blob, void* ptr) {
    unsigned char h[64];
    size_t off = 0;
    check(hc_ipc_export(ptr, h, &off));
    blob.append(reinterpret_cast<const char*>(h), 64);
    blob.append(reinterpret_cast<const char*>(&off), sizeof off);
  }

  void* open(const std::string& blob, size_t& at) {
    if (at + 64 + sizeof(size_t) > blob.size()) throw CommError(HC_PARSE_ERROR, "short bootstrap blob");
    const std::string key = blob.substr(at, 64);
    size_t off = 0;
    std::memcpy(&off, blob.data() + at + 64, sizeof off);
    at += 64 + sizeof off;
    auto it = opened_.find(key);
    if (it == opened_.end()) {
      void* base = nullptr;
      check(hc_ipc_import(reinterpret_cast<const unsigned char*>(key.data()), 0, device_, &base));
      imported_.push_back(base);
      it = opened_.emplace(key, base).first;
    }
    return static_cast<char*>(it->second) + off;
  }

  int rank_, world_, device_;
  Allgather allgather_;
  hc_program* prog_ = nullptr;
  hc_plan* plan_ = nullptr;
  hc_exec* exec_ = nullptr;
  std::vector<Buffer> buffers_;
  std::vector<Window> windows_;
  std::map<std::string, void*> opened_;
  std::vector<void*> imported_;
};

}  // namespace hiccl
