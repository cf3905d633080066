// The persistent sm_100a executor kernel.
//
// Replaces the reference's transfer loop (engine.cpp:285-330). One grid
// per executor (GPU), co-resident (cooperative launch), walks the global
// steps in order. Per step a CTA
//   1. waits — only if it has tiles here — for the executors / steps its
//      items depend on (acquire loads of local flag words that peers
//      raise over NVLink with release reductions),
//   2. runs its tiles: 128-bit loads of every source of a fused write
//      group (peer addresses go straight over NVLink/NVSwitch; local ones
//      hit HBM), the fold in registers in the reference's order, one
//      128-bit store,
//   3. if anyone depends on this step: arrives on the step counter; the
//      last CTA to arrive publishes "step done" to every executor.
// No host synchronization between steps, no reduction kernels, no copy
// engines: fences become flag edges between exactly the executors that
// share data.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdint>
#include <type_traits>

#include "device_program.cuh"

namespace hiccl::dev {

// ---------------------------------------------------------------- flags

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void red_relaxed_sys_max(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// Multicast (multimem.*) and unicast accesses reach the same physical
// memory through different virtual addresses, which the PTX memory model
// treats as different proxies: they are ordered only by a causality path
// that passes through a proxy fence (fence.proxy.alias) — in any thread on
// that path ("proxy-preserved base causality order"). Every cross-CTA or
// cross-GPU hand-off here is release (producer) -> acquire (consumer), so
// one fence per hand-off on the consumer side suffices: each waiting thread
// fences right after its acquire, before the barrier that releases the
// CTA's readers; the producer's writes precede that fence in causality
// order through the release / acquire pair. (The first version fenced in
// every thread on both sides, profiles/r2/alias_fence_cost*.jsonl.) Only in
// launches with NVLS items.
__device__ __forceinline__ void fence_proxy_alias(const Program& P) {
  if (P.alias_fence) asm volatile("fence.proxy.alias;" ::: "memory");
}

__device__ __forceinline__ long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Sticky status bits (watchdog, dependency violation), mirrored into a
// host-mapped word so wait() reads them without a copy per launch.
__device__ __forceinline__ void set_status(const Program& P, unsigned bits) {
  const unsigned old = atomicOr(P.status, bits);
  if (P.status_mirror) {
    *reinterpret_cast<volatile unsigned*>(P.status_mirror) = old | bits;
    __threadfence_system();
  }
}

// Spin until *p >= target. Returns the observed value, or 0 when the
// watchdog fired (status set, caller unwinds).
__device__ __forceinline__ uint64_t wait_at_least(const Program& P, const uint64_t* p,
                                                  uint64_t target) {
  uint64_t v = ld_acquire_sys(p);
  if (v >= target) return v;
  const long long t0 = P.timeout_ns > 0 ? globaltimer() : 0;
  unsigned spins = 0;
  while ((v = ld_acquire_sys(p)) < target) {
    if (++spins > 64) __nanosleep(64);
    if ((spins & 255) == 0) {
      if (*(volatile unsigned int*)P.status) return 0;  // another CTA timed out
      if (P.timeout_ns > 0 && globaltimer() - t0 > P.timeout_ns) {
        set_status(P, kStatusTimeout);
        return 0;
      }
    }
  }
  return v;
}

// Release pattern: ONE system-scope fence, then relaxed reductions to
// every executor's flag word, issued back to back (a release per
// reduction would serialize one NVLink round trip per peer).
__device__ __forceinline__ void publish_all(const Program& P, uint64_t value) {
  fence_acq_rel_sys();
  for (int x = 0; x < P.num_execs; ++x) red_relaxed_sys_max(P.peer_flags[x] + P.self, value);
}

// Only CTAs of this executor wait: GPU-scope release to its own word.
__device__ __forceinline__ void publish_cta_local(const Program& P, uint64_t value) {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  const size_t at = kMaxExecs + (size_t)P.self * kMaxCtas + blockIdx.x;
  asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(P.flags + at), "l"(value) : "memory");
}

// Same, for this CTA's progress word in every executor's CTA array.
__device__ __forceinline__ void publish_cta(const Program& P, uint64_t value) {
  fence_acq_rel_sys();
  const size_t at = kMaxExecs + (size_t)P.self * kMaxCtas + blockIdx.x;
  for (int x = 0; x < P.num_execs; ++x) red_relaxed_sys_max(P.peer_flags[x] + at, value);
}

__device__ __forceinline__ const uint64_t* cta_flag(const Program& P, int exec, int cta) {
  return P.flags + kMaxExecs + (size_t)exec * kMaxCtas + cta;
}

// ------------------------------------------------------------ element ops
// Fold rules (stated once, mirrored by oracle/numeric_exec.c):
//   f32/f64 sum: one IEEE add per fold (no contraction, no reassociation)
//   bf16/f16 sum: widen to f32, add, round-to-nearest-even after every fold
//   integer sum: wrapping add;  max: (acc < v) ? v : acc

template <int DT> struct Elem;
template <> struct Elem<0> { using T = float; };
template <> struct Elem<1> { using T = __nv_bfloat16; };
template <> struct Elem<2> { using T = __half; };
template <> struct Elem<3> { using T = int32_t; };
template <> struct Elem<4> { using T = long long; };
template <> struct Elem<5> { using T = double; };
template <> struct Elem<6> { using T = uint8_t; };

template <int DT, int OP>
__device__ __forceinline__ typename Elem<DT>::T fold1(typename Elem<DT>::T a,
                                                      typename Elem<DT>::T b) {
  if constexpr (DT == 1) {
    const float x = __bfloat162float(a), y = __bfloat162float(b);
    if constexpr (OP == 0) return __float2bfloat16_rn(__fadd_rn(x, y));
    else return (x < y) ? b : a;
  } else if constexpr (DT == 2) {
    const float x = __half2float(a), y = __half2float(b);
    if constexpr (OP == 0) return __float2half_rn(__fadd_rn(x, y));
    else return (x < y) ? b : a;
  } else if constexpr (DT == 0) {
    if constexpr (OP == 0) return __fadd_rn(a, b);
    else return (a < b) ? b : a;
  } else if constexpr (DT == 5) {
    if constexpr (OP == 0) return __dadd_rn(a, b);
    else return (a < b) ? b : a;
  } else if constexpr (DT == 3) {
    if constexpr (OP == 0) return (int32_t)((uint32_t)a + (uint32_t)b);
    else return (a < b) ? b : a;
  } else if constexpr (DT == 4) {
    if constexpr (OP == 0) return (long long)((unsigned long long)a + (unsigned long long)b);
    else return (a < b) ? b : a;
  } else {
    if constexpr (OP == 0) return (uint8_t)(a + b);
    else return (a < b) ? b : a;
  }
}

// Fold of one 32-bit word holding 1, 2 or 4 elements (4-byte-or-smaller
// types), register-only (no local-memory arrays).
template <int DT, int OP>
__device__ __forceinline__ uint32_t fold_word(uint32_t a, uint32_t b) {
  if constexpr (DT == 0) {
    const float x = __uint_as_float(a), y = __uint_as_float(b);
    return __float_as_uint(OP == 0 ? __fadd_rn(x, y) : ((x < y) ? y : x));
  } else if constexpr (DT == 3) {
    const int x = (int)a, y = (int)b;
    return OP == 0 ? a + b : (uint32_t)((x < y) ? y : x);
  } else if constexpr (DT == 6) {
    return OP == 0 ? __vadd4(a, b) : __vmaxu4(a, b);
  } else if constexpr (DT == 1) {
    __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a);
    __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162*>(&b);
    __nv_bfloat162 r;
    r.x = fold1<1, OP>(x.x, y.x);
    r.y = fold1<1, OP>(x.y, y.y);
    return *reinterpret_cast<uint32_t*>(&r);
  } else {
    static_assert(DT == 2, "16-bit float");
    __half2 x = *reinterpret_cast<__half2*>(&a);
    __half2 y = *reinterpret_cast<__half2*>(&b);
    __half2 r;
    r.x = fold1<2, OP>(x.x, y.x);
    r.y = fold1<2, OP>(x.y, y.y);
    return *reinterpret_cast<uint32_t*>(&r);
  }
}

template <int DT, int OP>
__device__ __forceinline__ uint64_t fold_dword(uint64_t a, uint64_t b) {
  if constexpr (DT == 5) {
    const double x = __longlong_as_double((long long)a), y = __longlong_as_double((long long)b);
    return (uint64_t)__double_as_longlong(OP == 0 ? __dadd_rn(x, y) : ((x < y) ? y : x));
  } else {
    static_assert(DT == 4, "64-bit integer");
    const long long x = (long long)a, y = (long long)b;
    return OP == 0 ? a + b : (uint64_t)((x < y) ? y : x);
  }
}

template <int DT, int OP>
__device__ __forceinline__ uint4 fold16(uint4 a, uint4 b) {
  if constexpr (DT == 4 || DT == 5) {
    const uint64_t lo = fold_dword<DT, OP>(((uint64_t)a.y << 32) | a.x, ((uint64_t)b.y << 32) | b.x);
    const uint64_t hi = fold_dword<DT, OP>(((uint64_t)a.w << 32) | a.z, ((uint64_t)b.w << 32) | b.z);
    return make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
  } else {
    return make_uint4(fold_word<DT, OP>(a.x, b.x), fold_word<DT, OP>(a.y, b.y),
                      fold_word<DT, OP>(a.z, b.z), fold_word<DT, OP>(a.w, b.w));
  }
}

// ------------------------------------------------------------ tile bodies

// A tile is kTileVec 16-byte vectors per thread of the destination.
constexpr int kTileVec = 8;
// Loads in flight per thread per batch; a group of NS sources folds U =
// kBatch / NS destination vectors per batch so every source load of the
// batch is issued before the first fold (one round trip per batch instead
// of one per source).
#ifndef HICCL_FOLD_BATCH
#define HICCL_FOLD_BATCH 8
#endif
constexpr int kBatch = HICCL_FOLD_BATCH;
// Plain copies keep fewer vectors in flight per thread: measured on B200,
// 4 outstanding 16-byte loads per thread beat 8 for HBM-bound copies and
// match them over NVLink.
#ifndef HICCL_COPY_BATCH
#define HICCL_COPY_BATCH 4
#endif
constexpr int kCopyBatch = HICCL_COPY_BATCH;

template <int DT, int OP, int NS>
__device__ __forceinline__ void fold_vectors_ns(uint4* __restrict__ dst,
                                                const uint64_t* __restrict__ srcs,
                                                int64_t byte_off, int nvec) {
  constexpr int U = NS == 1 ? kCopyBatch : (kBatch / NS > 0 ? kBatch / NS : 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  const uint4* s[NS];
#pragma unroll
  for (int j = 0; j < NS; ++j) s[j] = reinterpret_cast<const uint4*>(__ldg(srcs + j) + byte_off);
  int v0 = 0;
  // full batches: no predication
  for (; v0 + nt * U <= nvec; v0 += nt * U) {
    uint4 x[NS][U];
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u) x[j][u] = __ldcg(s[j] + v0 + u * nt + tid);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint4 acc = x[0][u];
#pragma unroll
      for (int j = 1; j < NS; ++j) acc = fold16<DT, OP>(acc, x[j][u]);
      __stcg(dst + v0 + u * nt + tid, acc);
    }
  }
  // remainder (< one batch): the same batch shape with indices clamped into
  // the tile (always-valid loads, stores masked), so a short tile still has
  // all of its loads in flight at once
  if (v0 < nvec) {
    uint4 x[NS][U];
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = min(v0 + u * nt + tid, nvec - 1);
        x[j][u] = __ldcg(s[j] + v);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * nt + tid;
      uint4 acc = x[0][u];
#pragma unroll
      for (int j = 1; j < NS; ++j) acc = fold16<DT, OP>(acc, x[j][u]);
      if (v < nvec) __stcg(dst + v, acc);
    }
  }
}

// Any number of sources: batches of kBatch destination vectors, sources
// folded one after the other.
template <int DT, int OP>
__device__ __forceinline__ void fold_vectors_any(uint4* __restrict__ dst,
                                                 const uint64_t* __restrict__ srcs, int n_src,
                                                 int64_t byte_off, int nvec) {
  constexpr int U = 4;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int v0 = 0; v0 < nvec; v0 += nt * U) {
    uint4 acc[U];
    const uint4* s0 = reinterpret_cast<const uint4*>(__ldg(srcs) + byte_off);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * nt + tid;
      if (v < nvec) acc[u] = __ldcg(s0 + v);
    }
    for (int j = 1; j < n_src; ++j) {
      const uint4* sj = reinterpret_cast<const uint4*>(__ldg(srcs + j) + byte_off);
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = v0 + u * nt + tid;
        if (v < nvec) x[u] = __ldcg(sj + v);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = fold16<DT, OP>(acc[u], x[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * nt + tid;
      if (v < nvec) __stcg(dst + v, acc[u]);
    }
  }
}

template <int DT, int OP>
__device__ __forceinline__ void fold_vectors(uint4* __restrict__ dst,
                                             const uint64_t* __restrict__ srcs, int n_src,
                                             int64_t byte_off, int nvec) {
  switch (n_src) {
    case 1: fold_vectors_ns<DT, OP, 1>(dst, srcs, byte_off, nvec); return;
    case 2: fold_vectors_ns<DT, OP, 2>(dst, srcs, byte_off, nvec); return;
    case 3: fold_vectors_ns<DT, OP, 3>(dst, srcs, byte_off, nvec); return;
    case 4: fold_vectors_ns<DT, OP, 4>(dst, srcs, byte_off, nvec); return;
    case 5: fold_vectors_ns<DT, OP, 5>(dst, srcs, byte_off, nvec); return;
    case 6: fold_vectors_ns<DT, OP, 6>(dst, srcs, byte_off, nvec); return;
    case 7: fold_vectors_ns<DT, OP, 7>(dst, srcs, byte_off, nvec); return;
    case 8: fold_vectors_ns<DT, OP, 8>(dst, srcs, byte_off, nvec); return;
    default: fold_vectors_any<DT, OP>(dst, srcs, n_src, byte_off, nvec); return;
  }
}

template <int DT, int OP>
__device__ __forceinline__ void fold_scalars(uint64_t dst, const uint64_t* __restrict__ srcs,
                                             int n_src, int64_t elem_lo, int64_t elem_hi) {
  using T = typename Elem<DT>::T;
  using R = typename std::conditional<sizeof(T) == 1, uint8_t,
            typename std::conditional<sizeof(T) == 2, unsigned short,
            typename std::conditional<sizeof(T) == 4, unsigned int,
                                      unsigned long long>::type>::type>::type;
  for (int64_t i = elem_lo + threadIdx.x; i < elem_hi; i += blockDim.x) {
    R raw = __ldcg(reinterpret_cast<const R*>(__ldg(srcs)) + i);
    T acc = *reinterpret_cast<T*>(&raw);
    for (int j = 1; j < n_src; ++j) {
      R r = __ldcg(reinterpret_cast<const R*>(__ldg(srcs + j)) + i);
      acc = fold1<DT, OP>(acc, *reinterpret_cast<T*>(&r));
    }
    reinterpret_cast<T*>(dst)[i] = acc;
  }
}

// ------------------------------------------------------------ tagged lines
// CopyMode::ll: a 16-byte line {w0, tag, w1, tag} carries 8 payload bytes
// (bytes [8l, 8l + 8) of the range); each 8-byte half is written and read
// as one access, so a half whose tag matches holds this launch's word. The
// reader polls the lines it needs instead of waiting for step flags.

__device__ __forceinline__ void st_line(uint64_t addr, uint64_t v, uint32_t tag) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(addr), "r"((uint32_t)v),
               "r"(tag), "r"((uint32_t)(v >> 32)), "r"(tag) : "memory");
}

__device__ __forceinline__ uint4 ld_line_once(uint64_t addr) {
  uint4 r;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(addr) : "memory");
  return r;
}

// Poll one line until both halves carry `tag`. When the watchdog fires (or
// fired elsewhere) it returns 0 with the status word set; the kernel's
// next flag wait then unwinds.
__device__ __forceinline__ uint64_t ld_line(const Program& P, uint64_t addr, uint32_t tag) {
  uint32_t a, b, c, d;
  unsigned spins = 0;
  long long t0 = 0;
  while (true) {
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(addr) : "memory");
    if (b == tag && d == tag) break;
    if ((++spins & 1023) == 0) {
      if (*(volatile unsigned int*)P.status) return 0;
      if (P.timeout_ns > 0) {
        const long long now = globaltimer();
        if (!t0) t0 = now;
        else if (now - t0 > P.timeout_ns) {
          set_status(P, kStatusTimeout);
          return 0;
        }
      }
    }
  }
  return (uint64_t)a | ((uint64_t)c << 32);
}

// nb (<= 8) payload bytes at addr, little-endian, as whole elements of ESZ bytes.
template <int ESZ>
__device__ __forceinline__ uint64_t ld_bytes_slow(uint64_t addr, int nb) {
  uint64_t v = 0;
  for (int k = 0; k < nb; k += ESZ) {
    uint64_t e;
    if constexpr (ESZ == 1) e = __ldcg(reinterpret_cast<const unsigned char*>(addr + k));
    else if constexpr (ESZ == 2) e = __ldcg(reinterpret_cast<const unsigned short*>(addr + k));
    else if constexpr (ESZ == 4) e = __ldcg(reinterpret_cast<const unsigned int*>(addr + k));
    else e = __ldcg(reinterpret_cast<const unsigned long long*>(addr + k));
    v |= e << (8 * k);
  }
  return v;
}

template <int ESZ>
__device__ __forceinline__ uint64_t ld_bytes(uint64_t addr, int nb) {
  if (nb == 8 && (addr & 7) == 0) return __ldcg(reinterpret_cast<const unsigned long long*>(addr));
  return ld_bytes_slow<ESZ>(addr, nb);
}

template <int ESZ>
__device__ __forceinline__ void st_bytes_slow(uint64_t addr, uint64_t v, int nb) {
  for (int k = 0; k < nb; k += ESZ) {
    const uint64_t e = v >> (8 * k);
    if constexpr (ESZ == 1) __stcg(reinterpret_cast<unsigned char*>(addr + k), (unsigned char)e);
    else if constexpr (ESZ == 2) __stcg(reinterpret_cast<unsigned short*>(addr + k), (unsigned short)e);
    else if constexpr (ESZ == 4) __stcg(reinterpret_cast<unsigned int*>(addr + k), (unsigned int)e);
    else __stcg(reinterpret_cast<unsigned long long*>(addr + k), (unsigned long long)e);
  }
}

template <int ESZ>
__device__ __forceinline__ void st_bytes(uint64_t addr, uint64_t v, int nb) {
  if (nb == 8 && (addr & 7) == 0) {
    __stcg(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)v);
    return;
  }
  st_bytes_slow<ESZ>(addr, v, nb);
}

template <int DT, int OP>
__device__ __forceinline__ uint64_t fold8(uint64_t a, uint64_t b) {
  if constexpr (DT == 4 || DT == 5) {
    return fold_dword<DT, OP>(a, b);
  } else {
    return (uint64_t)fold_word<DT, OP>((uint32_t)a, (uint32_t)b) |
           ((uint64_t)fold_word<DT, OP>((uint32_t)(a >> 32), (uint32_t)(b >> 32)) << 32);
  }
}

// Line l of a source: tagged staging (bit 63) or plain memory.
template <int ESZ>
__device__ __forceinline__ uint64_t ll_fetch(const Program& P, uint64_t a, int64_t l, int nb,
                                             uint32_t tag, uint64_t ll_off) {
  if (a & kLLBit) return ld_line(P, (a & ~kLLBit) + ll_off + l * 16, tag);
  return ld_bytes<ESZ>(a + l * 8, nb);
}

// One line of a tagged-line item, any alignment / partial length (slow path).
template <int DT, int OP>
__device__ __forceinline__ void ll_line_slow(const Program& P, const Item& it, const uint64_t* srcs,
                                          int64_t l, int nb, uint32_t tag, uint64_t ll_off) {
  constexpr int esz = sizeof(typename Elem<DT>::T);
  if (it.flags & kLLStore) {
    st_line(it.dst + ll_off + l * 16, ld_bytes<esz>(srcs[0] + l * 8, nb), tag);
    return;
  }
  uint64_t acc = 0;
  for (int j = 0; j < it.n_src; ++j) {
    const uint64_t a = srcs[j];
    const uint64_t v = (a & kLLBit) ? ld_line(P, (a & ~kLLBit) + ll_off + l * 16, tag)
                                    : ld_bytes<esz>(a + l * 8, nb);
    acc = j == 0 ? v : fold8<DT, OP>(acc, v);
  }
  st_bytes<esz>(it.dst + l * 8, acc, nb);
}

// Fold of up to NS sources over lines [l0, l_end) of a tile (aligned, full
// lines): every source's line loads of a batch are issued before any tag
// is checked, so the batch costs one memory round trip, not one per source;
// until every tag matches, the whole batch is reloaded.
template <int DT, int OP, int NS, int UB>
__device__ __forceinline__ void ll_fold_lines(const Program& P, const Item& it,
                                              const uint64_t* srcs, int64_t l0, int64_t l_end,
                                              int lane, int lanes, uint32_t tag, uint64_t ll_off) {
  const int n = it.n_src;
  uint64_t a[NS];
  uint32_t ll_mask = 0;
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    a[j] = j < n ? srcs[j] : 0;
    if (a[j] & kLLBit) {
      a[j] = (a[j] & ~kLLBit) + ll_off;
      ll_mask |= 1u << j;
    }
  }
  for (int64_t lb = l0; lb < l_end; lb += (int64_t)lanes * UB) {
    uint4 r[NS][UB];
    unsigned spins = 0;
    long long t0 = 0;
    while (true) {
      bool ok = true;
#pragma unroll
      for (int j = 0; j < NS; ++j)
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int64_t l = lb + (int64_t)u * lanes + lane;
          if (j < n && l < l_end) {
            if (ll_mask >> j & 1) {
              r[j][u] = ld_line_once(a[j] + l * 16);
              ok &= r[j][u].y == tag && r[j][u].w == tag;
            } else {
              const unsigned long long v =
                  __ldcg(reinterpret_cast<const unsigned long long*>(a[j] + l * 8));
              r[j][u] = make_uint4((uint32_t)v, tag, (uint32_t)(v >> 32), tag);
            }
          }
        }
      if (ok) break;
      if ((++spins & 1023) == 0) {
        if (*(volatile unsigned int*)P.status) break;
        if (P.timeout_ns > 0) {
          const long long now = globaltimer();
          if (!t0) t0 = now;
          else if (now - t0 > P.timeout_ns) {
            set_status(P, kStatusTimeout);
            break;
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int64_t l = lb + (int64_t)u * lanes + lane;
      if (l >= l_end) continue;
      uint64_t acc = 0;
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        if (j < n) {
          const uint64_t v = (uint64_t)r[j][u].x | ((uint64_t)r[j][u].z << 32);
          acc = j == 0 ? v : fold8<DT, OP>(acc, v);
        }
      }
      __stcg(reinterpret_cast<unsigned long long*>(it.dst + l * 8), acc);
    }
  }
}

// One tile of a tagged-line item, run by one warp (`lanes` threads; the
// CTA's warps take its tiles round robin, so small items of one step run
// side by side): a push of plain local data into a peer's
// staging (kLLStore), or a fold whose sources include staging (kLLLoad),
// in the plan's order, into plain local memory. Each thread keeps kLLBatch
// lines of one source in flight and re-polls the batch until every tag
// matches; ranges with 8-byte-misaligned plain addresses and the partial
// last line take the per-line slow path.
constexpr int kLLBatch = 4;

template <int DT, int OP>
__device__ __forceinline__ void run_tile_ll(const Program& P, const Item& it, const uint64_t* srcs,
                                         int64_t tile, int tile_elems, uint32_t tag,
                                         uint64_t ll_off, int lane, int lanes) {
  constexpr int esz = sizeof(typename Elem<DT>::T);
  constexpr int U = kLLBatch;
  const int64_t lo = tile * (int64_t)tile_elems;
  const int64_t hi = lo + tile_elems < it.count ? lo + tile_elems : it.count;
  const int64_t b1 = hi * esz;  // tiles start on a 16-byte multiple of the range
  const int64_t l0 = lo * esz / 8, lfull = b1 / 8, l1 = (b1 + 7) / 8;
  const int64_t nt = lanes, tid = lane;
  uint64_t plain_or = (it.flags & kLLStore) ? 0 : it.dst;
  for (int j = 0; j < it.n_src; ++j) {
    const uint64_t a = srcs[j];
    if (!(a & kLLBit)) plain_or |= a;
  }
  const int64_t fast_end = (plain_or & 7) ? l0 : lfull;
  for (int64_t l = fast_end + tid; l < l1; l += nt)
    ll_line_slow<DT, OP>(P, it, srcs, l, (int)(b1 - l * 8 < 8 ? b1 - l * 8 : 8), tag, ll_off);
  if (it.flags & kLLStore) {
    const uint64_t src = srcs[0], dst = it.dst + ll_off;
    for (int64_t lb = l0; lb < fast_end; lb += nt * U) {
      uint64_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t l = lb + u * nt + tid;
        if (l < fast_end) v[u] = __ldcg(reinterpret_cast<const unsigned long long*>(src + l * 8));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t l = lb + u * nt + tid;
        if (l < fast_end) st_line(dst + l * 16, v[u], tag);
      }
    }
    return;
  }
  if (it.n_src <= 4) {
    ll_fold_lines<DT, OP, 4, 2>(P, it, srcs, l0, fast_end, lane, lanes, tag, ll_off);
    return;
  }
  for (int64_t lb = l0; lb < fast_end; lb += nt * U) {
    uint64_t acc[U];
    for (int j = 0; j < it.n_src; ++j) {
      const uint64_t a = srcs[j];
      uint64_t v[U];
      if (a & kLLBit) {
        const uint64_t base = (a & ~kLLBit) + ll_off;
        unsigned spins = 0;
        long long t0 = 0;
        while (true) {
          bool ok = true;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t l = lb + u * nt + tid;
            if (l < fast_end) {
              const uint4 r = ld_line_once(base + l * 16);
              v[u] = (uint64_t)r.x | ((uint64_t)r.z << 32);
              ok &= r.y == tag && r.w == tag;
            }
          }
          if (ok) break;
          if ((++spins & 1023) == 0) {
            if (*(volatile unsigned int*)P.status) break;
            if (P.timeout_ns > 0) {
              const long long now = globaltimer();
              if (!t0) t0 = now;
              else if (now - t0 > P.timeout_ns) {
                set_status(P, kStatusTimeout);
                break;
              }
            }
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t l = lb + u * nt + tid;
          if (l < fast_end) v[u] = __ldcg(reinterpret_cast<const unsigned long long*>(a + l * 8));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = j == 0 ? v[u] : fold8<DT, OP>(acc[u], v[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t l = lb + u * nt + tid;
      if (l < fast_end) __stcg(reinterpret_cast<unsigned long long*>(it.dst + l * 8), acc[u]);
    }
  }
}

// ------------------------------------------------------------ TMA copies
// Local HBM copies run at ~6.7 TB/s as a 2-stage TMA bulk pipeline
// (global -> shared with an mbarrier, shared -> global bulk groups) against
// ~6.3 TB/s for the best LDG/STG body (tools/tmacopy.cu, 1 GiB). Over
// NVLink both reach the same link ceiling (tools/tmapeer.cu), so only steps
// made entirely of local copies use it. Thread 0 streams the CTA's tiles;
// the chunk counter (and with it the mbarrier phases) runs across steps.

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void tma_chunk_load(char* sdst, uint64_t gsrc, uint32_t bytes, uint64_t* mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void tma_chunk_store(uint64_t gdst, const char* ssrc, uint32_t bytes,
                                                uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n TMA_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TMA_WAIT_%=;\n}\n" ::"r"(smem_u32(mbar)), "r"(parity) : "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Thread 0 only. `n` counts the chunks this CTA issued in the launch.
__device__ __forceinline__ void tma_copy_step(const Program& P, const Step& st, char* stage,
                                           uint64_t* mbar, uint32_t& n, int esz,
                                           const uint2* cache) {
  // S stages of kTmaChunk: chunk k lands in stage k % S (mbarrier parity
  // (k / S) & 1); loads run S - 1 chunks ahead of the bulk stores, and a
  // stage is reloaded only once the store of the chunk before it has read
  // it (bulk groups complete in order).
  const uint32_t S = P.tma_stages;
  const uint32_t G = st.cta_n, b = blockIdx.x - st.cta_lo;  // caller: b < G
  // earlier steps' generic-proxy writes (acquired by this CTA's waits) must
  // be visible to the bulk loads
  asm volatile("fence.proxy.async.global;" ::: "memory");
  // pending stores (thread 0 only) in shared memory: a dynamically indexed
  // register array would cost the kernel a stack frame
  __shared__ uint64_t ring_dst[kTmaMaxStages];
  __shared__ uint32_t ring_bytes[kTmaMaxStages];
  const uint32_t n0 = n;
  auto store = [&](uint32_t j) {  // chunk j (launch-wide index) has been loaded
    const uint32_t slot = j % S;
    tma_chunk_store(ring_dst[slot], stage + (size_t)slot * kTmaChunk, ring_bytes[slot], mbar + slot,
                    (j / S) & 1);
  };
  for (uint32_t round = 0; round < st.max_rounds; ++round) {
    for (uint32_t j = 0; j < st.n_items; ++j) {
      const uint32_t jj = (j + b) % st.n_items;
      const uint32_t idx = st.item_first + jj;
      uint32_t n_tiles, local;
      if (cache) {
        n_tiles = cache[jj].x;
        local = cache[jj].y + round * G;
      } else {
        n_tiles = __ldg(&P.items[idx].n_tiles);
        local = (b + G - __ldg(&P.items[idx].base_cta) % G) % G + round * G;
      }
      if (local >= n_tiles) continue;
      const uint64_t dst = __ldg(&P.items[idx].dst);
      const int64_t count = __ldg(&P.items[idx].count);
      const uint64_t src = __ldg(P.srcs + __ldg(&P.items[idx].src_first));
      const int64_t lo = (int64_t)local * st.tile_elems * esz;
      const int64_t hi_e = ((int64_t)local + 1) * st.tile_elems < count ? ((int64_t)local + 1) * st.tile_elems : count;
      const int64_t hi = hi_e * esz;
      for (int64_t off = lo; off < hi; off += kTmaChunk) {
        const uint32_t bytes = (uint32_t)(hi - off < (int64_t)kTmaChunk ? hi - off : kTmaChunk);
        const uint32_t slot = n % S;
        // the stage's previous chunk (n - S) was stored at the last step of
        // this loop; its bulk store must have read the stage
        if (n >= S) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        ring_dst[slot] = dst + off;
        ring_bytes[slot] = bytes;
        tma_chunk_load(stage + (size_t)slot * kTmaChunk, src + off, bytes, mbar + slot);
        if (n + 1 >= n0 + S) store(n + 1 - S);
        ++n;
      }
    }
  }
  // the chunks still in flight
  for (uint32_t j = (n >= n0 + S - 1 ? n + 1 - S : n0); j < n; ++j) store(j);
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // the bulk writes, complete, become visible to generic-proxy readers
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------ staged folds
// A step whose items are all 16-byte-aligned point-to-point folds (local or
// peer sources, up to 8) can run through shared memory as a
// producer / consumer pipeline: warp 0 streams the CTA's tiles in chunks,
// one bulk copy (cp.async.bulk, TMA) per source into a stage, and the
// other warps fold each landed stage from shared memory in the reference's
// order and store the result. `full` mbarriers (TMA transaction counts)
// hand a stage to the consumers, `empty` mbarriers (one arrival per
// consumer warp) hand it back, so several stages are always in flight and
// no CTA-wide barrier sits between chunks. The register body instead keeps
// one batch of loads in flight per thread and waits a full round trip per
// batch.
constexpr int kFoldStages = 6;                  // upper bound (smem_bytes decides)
constexpr uint32_t kFoldStageBytes = 64 * 1024;  // default stage size

// This CTA's tiles of a step in the order of the register loop.
struct TileCursor {
  uint32_t round = 0, j = 0;
  uint32_t idx = 0;
  int64_t pos = 0, end = 0;  // bytes within the item
  uint32_t ns = 0, chunk = 0;
  bool live = false;

  const uint2* cache = nullptr;  // per item {n_tiles, this CTA's first tile} (shared memory)

  __device__ bool next_tile(const Program& P, const Step& st, uint32_t b, uint32_t G, int esz,
                            uint32_t stage_bytes) {
    while (round < st.max_rounds) {
      while (j < st.n_items) {
        const uint32_t jj = (j + b) % st.n_items;
        const uint32_t i = st.item_first + jj;
        ++j;
        uint32_t n_tiles, local;
        if (cache) {
          n_tiles = cache[jj].x;
          local = cache[jj].y + round * G;
        } else {
          n_tiles = __ldg(&P.items[i].n_tiles);
          local = (b + G - __ldg(&P.items[i].base_cta) % G) % G + round * G;
        }
        if (local >= n_tiles) continue;
        const int64_t count = __ldg(&P.items[i].count);
        const int64_t lo = (int64_t)local * st.tile_elems;
        const int64_t hi = lo + st.tile_elems < count ? lo + st.tile_elems : count;
        idx = i;
        pos = lo * esz;
        end = hi * esz;
        ns = __ldg(&P.items[i].n_src);
        chunk = (stage_bytes / ns) & ~15u;
        return true;
      }
      j = 0;
      ++round;
    }
    return false;
  }
  // the next chunk [off, off + bytes) of the current or a later tile
  __device__ bool next_chunk(const Program& P, const Step& st, uint32_t b, uint32_t G, int esz,
                             uint32_t stage_bytes, int64_t& off, uint32_t& bytes) {
    if (!live || pos >= end) {
      live = next_tile(P, st, b, G, esz, stage_bytes);
      if (!live) return false;
    }
    off = pos;
    bytes = (uint32_t)(end - pos < (int64_t)chunk ? end - pos : chunk);
    pos += bytes;
    return true;
  }
};

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int DT, int OP, int NS>
__device__ __forceinline__ void fold_stage_ns(uint4* __restrict__ dst, const char* stage,
                                              uint32_t chunk, int nvec, int c, int nc) {
#pragma unroll 2
  for (int v = c; v < nvec; v += nc) {
    uint4 x[NS];
#pragma unroll
    for (int j = 0; j < NS; ++j) x[j] = *reinterpret_cast<const uint4*>(stage + j * chunk + v * 16);
    uint4 acc = x[0];
#pragma unroll
    for (int j = 1; j < NS; ++j) acc = fold16<DT, OP>(acc, x[j]);
    __stcg(dst + v, acc);
  }
}

template <int DT, int OP>
__device__ __forceinline__ void fold_stage(uint4* dst, const char* stage, uint32_t chunk, int ns,
                                           int nvec, int c, int nc) {
  switch (ns) {
    case 1: fold_stage_ns<DT, OP, 1>(dst, stage, chunk, nvec, c, nc); return;
    case 2: fold_stage_ns<DT, OP, 2>(dst, stage, chunk, nvec, c, nc); return;
    case 3: fold_stage_ns<DT, OP, 3>(dst, stage, chunk, nvec, c, nc); return;
    case 4: fold_stage_ns<DT, OP, 4>(dst, stage, chunk, nvec, c, nc); return;
    case 5: fold_stage_ns<DT, OP, 5>(dst, stage, chunk, nvec, c, nc); return;
    case 6: fold_stage_ns<DT, OP, 6>(dst, stage, chunk, nvec, c, nc); return;
    case 7: fold_stage_ns<DT, OP, 7>(dst, stage, chunk, nvec, c, nc); return;
    default: fold_stage_ns<DT, OP, 8>(dst, stage, chunk, nvec, c, nc); return;
  }
}

// Every thread of the CTA. `n` (shared) counts the chunks staged in this
// launch: chunk k uses stage k % S; its full / empty phases are k / S.
// The checked-mode and staged-fold bodies are inlined behind their runtime
// branches: as calls, the ABI's saved registers cost the main loop a 232-byte
// stack frame and ~9% on C1 (profiles/r2/aux_inline_ab.txt).
#ifdef HICCL_NOINLINE_AUX
#define HICCL_AUX __noinline__
#else
#define HICCL_AUX __forceinline__
#endif

template <int DT>
__device__ HICCL_AUX void staged_fold_step(const Program& P, const Step& st, char* stages,
                                              uint64_t* full, uint64_t* empty, uint32_t& n,
                                              const uint2* cache) {
  constexpr int esz = sizeof(typename Elem<DT>::T);
  const uint32_t G = st.cta_n, b = blockIdx.x - st.cta_lo;
  const uint32_t S = P.fold_stages, SB = P.fold_stage_bytes;
  const uint32_t n0 = n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t used = 0;  // chunks of this step
  if (warp == 0) {
    if (lane == 0) {
      // earlier steps' generic-proxy writes (acquired by this CTA's waits)
      // must be visible to the bulk loads
      asm volatile("fence.proxy.async.global;" ::: "memory");
      TileCursor cur;
      cur.cache = cache;
      int64_t off;
      uint32_t bytes;
      while (cur.next_chunk(P, st, b, G, esz, SB, off, bytes)) {
        const uint32_t k = n0 + used++;
        const uint32_t slot = k % S;
        if (k >= S) mbar_wait(empty + slot, ((k / S) - 1) & 1);  // consumers freed it
        char* stage = stages + (size_t)slot * SB;
        const uint64_t* srcs = P.srcs + __ldg(&P.items[cur.idx].src_first);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(smem_u32(full + slot)), "r"(bytes * cur.ns) : "memory");
        for (uint32_t j = 0; j < cur.ns; ++j)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(smem_u32(stage + j * cur.chunk)), "l"(__ldg(srcs + j) + off), "r"(bytes),
              "r"(smem_u32(full + slot)) : "memory");
      }
      n = n0 + used;
    }
  } else {
    const int c = threadIdx.x - 32, nc = blockDim.x - 32;
    TileCursor cur;
    cur.cache = cache;
    int64_t off;
    uint32_t bytes;
    uint32_t k = n0;
    while (cur.next_chunk(P, st, b, G, esz, SB, off, bytes)) {
      const uint32_t slot = k % S;
      mbar_wait(full + slot, (k / S) & 1);
      uint4* dst = reinterpret_cast<uint4*>(__ldg(&P.items[cur.idx].dst) + off);
      const char* stage = stages + (size_t)slot * SB;
      if (__ldg(&P.items[cur.idx].op) == 0 || cur.ns == 1)
        fold_stage<DT, 0>(dst, stage, cur.chunk, (int)cur.ns, (int)(bytes / 16), c, nc);
      else
        fold_stage<DT, 1>(dst, stage, cur.chunk, (int)cur.ns, (int)(bytes / 16), c, nc);
      // generic-proxy reads of the stage before the async-proxy refill
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + slot)) : "memory");
      ++k;
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ NVLS bodies
// multimem.ld_reduce: the switch reads the same offset from every member of
// the multicast object and returns the reduction (accumulated in fp32 for
// 16-bit floats). Only dtype/op pairs the hardware supports are lowered
// (executor.cu): f32/bf16/f16 sum, i32 sum/max.

template <int DT, int OP>
__device__ __forceinline__ uint4 mc_ld_reduce(const uint4* mc) {
  uint4 v;
  if constexpr (DT == 0) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  } else if constexpr (DT == 1) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  } else if constexpr (DT == 2) {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(mc) : "memory");
  } else if constexpr (DT == 3) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(mc);
    uint32_t r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (OP == 0)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.s32 %0, [%1];" : "=r"(r[k]) : "l"(p + k) : "memory");
      else
        asm volatile("multimem.ld_reduce.relaxed.sys.global.max.s32 %0, [%1];" : "=r"(r[k]) : "l"(p + k) : "memory");
    }
    v = make_uint4(r[0], r[1], r[2], r[3]);
  } else {
    v = make_uint4(0, 0, 0, 0);  // never lowered
  }
  return v;
}

__device__ __forceinline__ void mc_store(uint4* mc, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// MODE: kMcStore (local load -> multicast store), kMcReduce (switch
// reduction -> local store) or both (switch reduction -> multicast store:
// the fused all-reduce tile, egress and ingress traffic overlapping).
template <int DT, int OP, int MODE>
__device__ __forceinline__ void nvls_vectors(const Item& it, const uint64_t* srcs, int64_t byte_off,
                                             int nvec) {
  constexpr bool REDUCE = (MODE & kMcReduce) != 0, MCAST = (MODE & kMcStore) != 0;
  constexpr int U = 4;
  const int tid = threadIdx.x, nt = blockDim.x;
  const uint4* src = reinterpret_cast<const uint4*>(__ldg(srcs) + byte_off);
  uint4* dst = reinterpret_cast<uint4*>(it.dst + byte_off);
  int v0 = 0;
  for (; v0 + nt * U <= nvec; v0 += nt * U) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (REDUCE) x[u] = mc_ld_reduce<DT, OP>(src + v0 + u * nt + tid);
      else x[u] = __ldcg(src + v0 + u * nt + tid);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if constexpr (MCAST) mc_store(dst + v0 + u * nt + tid, x[u]);
      else __stcg(dst + v0 + u * nt + tid, x[u]);
    }
  }
  if (v0 < nvec) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = min(v0 + u * nt + tid, nvec - 1);
      if constexpr (REDUCE) x[u] = mc_ld_reduce<DT, OP>(src + v);
      else x[u] = __ldcg(src + v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = v0 + u * nt + tid;
      if (v < nvec) {
        if constexpr (MCAST) mc_store(dst + v, x[u]);
        else __stcg(dst + v, x[u]);
      }
    }
  }
}

template <int DT, int OP, bool LL>
__device__ void run_tile(const Program& P, const Item& it, const uint64_t* srcs, int64_t tile,
                         int tile_elems, uint32_t tag, uint64_t ll_off) {
  using T = typename Elem<DT>::T;
  constexpr int esz = sizeof(T);
  if constexpr (LL) {
    // every item of a tagged-line schedule (plain local folds too: the
    // mode is for small messages, where a lean kernel beats wide vectors)
    run_tile_ll<DT, OP>(P, it, srcs, tile, tile_elems, tag, ll_off, threadIdx.x & 31, 32);
    return;
  }
  const int64_t lo = tile * (int64_t)tile_elems;
  const int64_t hi = lo + tile_elems < it.count ? lo + tile_elems : it.count;
  if (it.flags & (kMcReduce | kMcStore)) {
    // lowered items are 16-byte aligned with a whole number of vectors;
    // a multicast store is a bit copy (every dtype), switch reductions are
    // lowered only for f32/bf16/f16/i32 (layout.cpp nvls_reduce_ok)
    const int nv = (int)((hi - lo) * esz / 16);
    if constexpr (DT == 0 || DT == 1 || DT == 2 || DT == 3) {
      if ((it.flags & (kMcReduce | kMcStore)) == (kMcReduce | kMcStore))
        nvls_vectors<DT, OP, kMcReduce | kMcStore>(it, srcs, lo * esz, nv);
      else if (it.flags & kMcReduce)
        nvls_vectors<DT, OP, kMcReduce>(it, srcs, lo * esz, nv);
      else
        nvls_vectors<DT, OP, kMcStore>(it, srcs, lo * esz, nv);
    } else {
      if (!(it.flags & kMcReduce)) nvls_vectors<DT, OP, kMcStore>(it, srcs, lo * esz, nv);
    }
    return;
  }
  if (!(it.flags & kVec)) {
    // Misaligned sources: element-wise (every address advances by the
    // same index i, so pass base addresses and absolute indices).
    fold_scalars<DT, OP>(it.dst, srcs, it.n_src, lo, hi);
    return;
  }
  // All addresses share the same misalignment; peel to a 16-byte boundary.
  const int mis = (int)(it.dst % 16);
  int64_t head = mis ? (16 - mis) / esz : 0;
  const int64_t vlo = lo + (head < hi - lo ? head : hi - lo);
  const int64_t nv = (hi - vlo) * esz / 16;
  const int64_t vhi = vlo + nv * (16 / esz);
  if (vlo > lo) fold_scalars<DT, OP>(it.dst, srcs, it.n_src, lo, vlo);
  if (nv > 0)
    fold_vectors<DT, OP>(reinterpret_cast<uint4*>(it.dst + vlo * esz), srcs, it.n_src,
                         vlo * esz, (int)nv);
  if (vhi < hi) fold_scalars<DT, OP>(it.dst, srcs, it.n_src, vhi, hi);
}

// ------------------------------------------------------------ the kernel

constexpr uint32_t kSmemItems = 1024;
// Tagged-line kernels run 256-thread CTAs (tiles are per warp, so the grid
// supplies the parallelism) and get 255 registers for their batched polls.
constexpr int kLLThreads = 256;

// LL: the tagged-line variant (CopyMode::ll); a separate instantiation so
// the bandwidth path's register allocation does not carry its code.
//
// Checked mode: every producer tile this CTA's tiles of step s conflict
// with must have finished (its CTA's flag reached the step) — whatever the
// wait tables said. The runtime counterpart of the reference executor's
// "deps done" check (engine.cpp:302-306): a consumer tile about to run
// before its producer step fails the launch with DependencyViolation.
__device__ HICCL_AUX void check_producers(const Program& P, int s, uint64_t base) {
  const uint2 ci = P.cta_checks[(size_t)s * gridDim.x + blockIdx.x];
  for (uint32_t e = threadIdx.x; e < ci.y; e += blockDim.x) {
    const Wait w = P.checks[ci.x + e];
    if (ld_acquire_sys(cta_flag(P, w.exec, w.cta)) >= base + w.k) continue;
    if (atomicOr(P.status, kStatusDepViolation) & kStatusDepViolation) continue;
    const unsigned detail[4] = {(unsigned)s, blockIdx.x, ((unsigned)w.exec << 16) | w.cta, w.k};
    for (int i = 0; i < 4; ++i) {
      P.status[1 + i] = detail[i];
      if (P.status_mirror) reinterpret_cast<volatile unsigned*>(P.status_mirror)[1 + i] = detail[i];
    }
    set_status(P, kStatusDepViolation);
  }
  __syncthreads();
}

// The launch's epoch lives on the device (arrive[num_steps + 1], bumped by
// the last CTA to finish), so a captured CUDA graph replays launches with
// fresh epochs and no host involvement.
// TS: the tile-sync variant (tile-level waits and per-tile publishes in the
// tile loop; a separate instantiation so the plain kernel's register
// allocation does not carry them).
template <int DT, bool LL, bool TS = false>
__global__ void __launch_bounds__(LL ? kLLThreads : 512, 1) persistent_executor(Program P) {
  __shared__ int aborted;                // a wait of this CTA hit the watchdog
  __shared__ uint2 s_items[kSmemItems];  // current step: {n_tiles, this CTA's first tile}
  extern __shared__ __align__(128) unsigned char s_prog[];
  __shared__ __align__(8) uint64_t s_tma_bar[kTmaMaxStages];  // TMA stage mbarriers (non-LL kernel)
  __shared__ uint32_t s_tma_chunks;                 // thread 0: TMA chunks issued so far
  __shared__ __align__(8) uint64_t s_fold_full[kFoldStages];   // staged folds: stage landed
  __shared__ __align__(8) uint64_t s_fold_empty[kFoldStages];  // staged folds: stage free
  __shared__ uint32_t s_fold_chunks;                 // staged-fold chunks so far (launch)
  const unsigned long long epoch =
      *reinterpret_cast<volatile unsigned long long*>(P.arrive + P.num_steps + 1) + 1;
  const uint64_t T = P.tile_stride;  // progress units per step (1 without tile sync)
  const uint64_t base = epoch * (uint64_t)(P.num_steps + 2) * T;
  const int tid = threadIdx.x;

  // Entry barrier: peers may read our inputs / write our outputs only
  // after this grid (and so every earlier kernel on our stream) started.
  // Trace (per launch, read by hc_exec_get_trace): [0] grid entry,
  // [1] entry barrier passed, [2 + s] step s published, [S + 2] last CTA
  // finished, [S + 3] exit barrier passed.
  //
  // Tagged-line mode has no entry barrier: nobody reads or writes another
  // executor's buffers except the staging lines, and a producer fills arena
  // copy e & 1 of a consumer only once that consumer has entered epoch e-1
  // (so finished reading copy e & 1 in epoch e-2). "Entered" needs no
  // fence: the previous launch's reads completed at the kernel boundary.
  // Tagged-line (small-message) programs run from shared memory: the step /
  // item / source tables (one contiguous image) and this CTA's wait index
  // are copied in while the entry flags are checked, so no dependent global
  // load sits on a step's critical path. (The bandwidth kernel keeps its
  // tables in global memory: its fold loops need every register.)
  const Step* steps = P.steps;
  const Item* items = P.items;
  const uint64_t* srcs_tab = P.srcs;
  const uint2* my_waits = nullptr;
  if constexpr (LL) {
    if (P.smem_bytes) {
      const uint4* g = reinterpret_cast<const uint4*>(P.image);
      uint4* d = reinterpret_cast<uint4*>(s_prog);
      for (int i = tid; i < P.image_bytes / 16; i += blockDim.x) d[i] = __ldg(g + i);
      uint2* c = reinterpret_cast<uint2*>(s_prog + P.image_bytes);
      for (int i = tid; i < P.num_steps; i += blockDim.x)
        c[i] = __ldg(&P.cta_waits[(size_t)i * gridDim.x + blockIdx.x]);
      const char* img = reinterpret_cast<const char*>(P.image);
      steps = reinterpret_cast<const Step*>(s_prog + (reinterpret_cast<const char*>(P.steps) - img));
      items = reinterpret_cast<const Item*>(s_prog + (reinterpret_cast<const char*>(P.items) - img));
      srcs_tab = reinterpret_cast<const uint64_t*>(s_prog + (reinterpret_cast<const char*>(P.srcs) - img));
      my_waits = c;
    }
  }
  const uint32_t tag = (uint32_t)epoch;
  const uint64_t ll_off = (epoch & 1) ? P.ll_half : 0;
  // A lone executor (every rank on one GPU) has no peer to wait for:
  // stream order already separates its launches; its "started" word is a
  // GPU-scope relaxed update with no fence.
  if (blockIdx.x == 0 && tid == 0) {
    P.trace[0] = globaltimer();
    if (LL || P.num_execs == 1) {
      for (int x = 0; x < P.num_execs; ++x) red_relaxed_sys_max(P.peer_flags[x] + P.self, base);
    } else {
      publish_all(P, base);
    }
  }
  if (tid == 0) {
    aborted = 0;
    s_tma_chunks = 0;
    s_fold_chunks = 0;
    if (!LL && P.tma) {
      for (int i = 0; i < kTmaMaxStages; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_tma_bar[i])));
      for (int i = 0; i < kFoldStages; ++i) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_fold_full[i])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&s_fold_empty[i])),
                     "r"((int)(blockDim.x >> 5) - 1));
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  {
    const uint64_t need = LL ? base - (P.num_steps + 2) * T : base;
    if (tid < P.num_execs && !P.solo) {
      if (wait_at_least(P, P.flags + tid, need) < need) aborted = 1;
      fence_proxy_alias(P);
    }
    __syncthreads();
  }
  if (aborted) return;
  if (blockIdx.x == 0 && tid == 0) P.trace[1] = globaltimer();

  for (int s = 0; s < P.num_steps; ++s) {
    const Step st = LL ? steps[s] : P.steps[s];
    if (st.barrier) __syncthreads();
    if (P.delay_ns > 0 && P.self == P.delay_exec && tid == 0) {
      const long long t0 = globaltimer();
      while (globaltimer() - t0 < P.delay_ns) __nanosleep(1000);
    }
    if (st.n_tiles) {
      // Tile-granular dependencies: the CTAs (of any executor) whose tiles
      // this CTA's tiles read or overwrite, as computed on the host.
      const uint2 wi = (LL && my_waits) ? my_waits[s]
                                        : __ldg(&P.cta_waits[(size_t)s * gridDim.x + blockIdx.x]);
      if (wi.y) {
        bool waited = false;
        for (uint32_t e = 0; e < wi.y; ++e) {
          const Wait w = P.waits[wi.x + e];
          const uint64_t target = base + w.k;
          if (w.cta == kAllCtas) {
            for (uint32_t c = tid; c < gridDim.x; c += blockDim.x) {
              if (wait_at_least(P, cta_flag(P, w.exec, c), target) < target) aborted = 1;
              waited = true;
            }
          } else if (tid == (int)(e % blockDim.x)) {
            if (wait_at_least(P, cta_flag(P, w.exec, w.cta), target) < target) aborted = 1;
            waited = true;
          }
        }
        if (waited) fence_proxy_alias(P);
        __syncthreads();
        if (aborted) return;
      }
#ifndef HICCL_LEAN
      if (P.cta_checks) check_producers(P, s, base);
#endif
      // the step's tiles run on CTAs [cta_lo, cta_lo + cta_n)
      const bool mine = blockIdx.x >= st.cta_lo && blockIdx.x - st.cta_lo < st.cta_n;
      // The step's (n_tiles, this CTA's first tile) per item, staged in
      // shared memory by every thread: the tile enumeration visits every
      // (round, item) pair, which would otherwise cost two dependent global
      // loads each (for the TMA paths: on one thread).
      const bool cached = mine && !(LL && my_waits) && st.n_items <= kSmemItems;
      if (cached) {
        const uint32_t G = st.cta_n, b = blockIdx.x - st.cta_lo;
        __syncthreads();  // the previous step's table is no longer read
        for (uint32_t i = tid; i < st.n_items; i += blockDim.x) {
          const uint32_t idx = st.item_first + i;
          const uint32_t nt_i = __ldg(&P.items[idx].n_tiles), bc = __ldg(&P.items[idx].base_cta);
          s_items[i] = make_uint2(nt_i, (b + G - bc % G) % G);
        }
        __syncthreads();
      }
      if (!mine) {
      } else if (!LL && st.tma == 1) {
        if (tid == 0)
          tma_copy_step(P, st, reinterpret_cast<char*>(s_prog), s_tma_bar, s_tma_chunks,
                        (int)sizeof(typename Elem<DT>::T), cached ? s_items : nullptr);
#ifndef HICCL_LEAN
      } else if (!LL && st.tma == 2) {
        staged_fold_step<DT>(P, st, reinterpret_cast<char*>(s_prog), s_fold_full, s_fold_empty,
                             s_fold_chunks, cached ? s_items : nullptr);
#endif
      } else {
      // Tile l of item i runs on CTA (base_i + l) mod G, so a range
      // produced by CTA b in one step is consumed by CTA b in the next
      // (tile-granular dependencies). Rounds visit the items starting at a
      // CTA-dependent item, so every wave spreads over every peer. Item and
      // source tables are immutable for the kernel's lifetime.
      const uint32_t G = st.cta_n, b = blockIdx.x - st.cta_lo;
      uint32_t k = 0;  // LL: this CTA's tiles go to its warps round robin
      const uint32_t nw = blockDim.x >> 5, warp = tid >> 5;
      // LL timeline of CTA 0 (debug slots after the step stamps): per step
      // s < 4 and warp w < 16, when the warp started and finished its tiles
      const bool stamp = LL && b == 0 && (tid & 31) == 0 && s < 4 && warp < 16;
      if (stamp) P.trace[P.num_steps + 4 + (s * 16 + warp) * 2] = globaltimer();
      // tile-level progress: waits before a given tile of this CTA, and a
      // publish after each tile when someone follows this step tile by tile
      uint32_t ord = 0, tw = 0, tw_n = 0;
      const TileWait* tws = nullptr;
      if (TS && !LL && P.cta_tile_waits) {
        const uint2 t2 = __ldg(&P.cta_tile_waits[(size_t)s * gridDim.x + blockIdx.x]);
        tws = P.tile_waits + t2.x;
        tw_n = t2.y;
      }
      for (uint32_t round = 0; round < st.max_rounds; ++round) {
        for (uint32_t j = 0; j < st.n_items; ++j) {
          const uint32_t jj = (j + b) % st.n_items;
          const uint32_t idx = st.item_first + jj;
          uint32_t n_tiles, first;
          if (cached) {
            const uint2 c = s_items[jj];
            n_tiles = c.x;
            first = c.y;
          } else {
            if constexpr (LL) {
              n_tiles = items[idx].n_tiles;
              first = (b + G - items[idx].base_cta % G) % G;
            } else {
              n_tiles = __ldg(&P.items[idx].n_tiles);
              first = (b + G - __ldg(&P.items[idx].base_cta) % G) % G;
            }
          }
          const uint32_t local = first + round * G;
          if (local >= n_tiles) continue;
          if constexpr (LL) {
            if (k++ % nw != warp) continue;
          }
          Item it;
          if constexpr (LL) {
            it = items[idx];
          } else {
            it.dst = __ldg(&P.items[idx].dst);
            it.count = __ldg(&P.items[idx].count);
            it.src_first = __ldg(&P.items[idx].src_first);
            it.n_src = __ldg(&P.items[idx].n_src);
            it.op = __ldg(&P.items[idx].op);
            it.flags = __ldg(&P.items[idx].flags);
          }
          const uint64_t* srcs = (LL ? srcs_tab : P.srcs) + it.src_first;
          if constexpr (TS && !LL) {
            if (tw < tw_n && __ldg(&tws[tw].at) == ord) {
              uint32_t e = tw;
              for (; e < tw_n && __ldg(&tws[e].at) == ord; ++e)
                if (tid == (int)((e - tw) % blockDim.x)) {
                  const uint64_t target = base + __ldg(&tws[e].k);
                  if (wait_at_least(P, cta_flag(P, __ldg(&tws[e].exec), __ldg(&tws[e].cta)), target) < target)
                    aborted = 1;
                }
              tw = e;
              __syncthreads();
              if (aborted) return;
            }
          }
          if (it.op == 0 || it.n_src == 1)
            run_tile<DT, 0, LL>(P, it, srcs, local, st.tile_elems, tag, ll_off);
          else
            run_tile<DT, 1, LL>(P, it, srcs, local, st.tile_elems, tag, ll_off);
          if constexpr (TS && !LL) {
            if (st.tile_publish && (ord + 1) % P.tile_pub_every == 0) {
              __syncthreads();
              if (tid == 0) {
                if (st.publish == 1) publish_cta_local(P, base + s * T + ord + 1);
                else publish_cta(P, base + s * T + ord + 1);
              }
            }
            ++ord;
          }
        }
      }
      if (stamp) P.trace[P.num_steps + 4 + (s * 16 + warp) * 2 + 1] = globaltimer();
      }
    }
    if (st.publish) {
      __syncthreads();
      if (tid == 0) {
        if (st.publish == 1) publish_cta_local(P, base + (s + 1) * T);
        else publish_cta(P, base + (s + 1) * T);
        if (blockIdx.x == 0) P.trace[2 + s] = globaltimer();
      }
    } else if (blockIdx.x == 0 && tid == 0) {
      P.trace[2 + s] = globaltimer();  // thread 0's own view (no barrier)
    }
  }

  // Exit. With peers and no tagged lines, a barrier: our buffers are
  // reusable once every executor is done (GPU-scope release per CTA; the
  // last CTA's system-scope fence in publish_all is cumulative over
  // everything it acquired via the counter). Tagged-line launches and a
  // lone executor need none: every byte owed to a peer already sits in its
  // staging lines, or there is no peer.
  const bool barrier = !LL && P.num_execs > 1 && !P.solo;
  __syncthreads();
  if (tid == 0) {
    if (barrier) __threadfence();
    const unsigned long long old = atomicAdd(P.arrive + P.num_steps, 1ULL);
    if (old + 1 == gridDim.x) {  // per-launch count: any grid size per commit
      if (barrier) __threadfence();
      P.arrive[P.num_steps] = 0;          // nobody of this launch touches it again
      P.arrive[P.num_steps + 1] = epoch;  // every CTA has read it
      if (barrier) publish_all(P, base + (P.num_steps + 1) * T);
      P.trace[P.num_steps + 2] = globaltimer();
    }
  }
  if (blockIdx.x == 0) {
    if (barrier && tid < P.num_execs) {
      wait_at_least(P, P.flags + tid, base + (P.num_steps + 1) * T);
      fence_proxy_alias(P);
    }
    __syncthreads();
    if (tid == 0) P.trace[P.num_steps + 3] = globaltimer();
  }
}

// ------------------------------------------------------------ data generator
// h = splitmix64(seed ^ (rank << 40) ^ index); shared with the oracle.

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

template <int DT>
__global__ void fill_kernel(void* out, int64_t n, uint64_t seed, int rank, int64_t index_base) {
  using T = typename Elem<DT>::T;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = splitmix64(seed ^ ((uint64_t)rank << 40) ^ (uint64_t)(index_base + i));
    const float f = __fmul_rn((float)(h >> 40), 5.9604644775390625e-08f) * 2.0f - 1.0f;
    T v;
    if constexpr (DT == 0) v = f;
    else if constexpr (DT == 1) v = __float2bfloat16_rn(f);
    else if constexpr (DT == 2) v = __float2half_rn(f);
    else if constexpr (DT == 3) v = (int32_t)((h >> 33) & 0xFFFF);
    else if constexpr (DT == 4) v = (long long)((h >> 33) & 0xFFFF);
    else if constexpr (DT == 5) v = (double)f;
    else v = (uint8_t)(h >> 56);
    reinterpret_cast<T*>(out)[i] = v;
  }
}

}  // namespace hiccl::dev
