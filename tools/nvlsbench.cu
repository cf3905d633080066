// Development microbenchmark: NVSwitch multimem throughput, one process
// driving every visible GPU (hiccl NVLS window from libhiccl.so).
//   R  reduce-scatter: multimem.ld_reduce (switch reads every member) -> local store
//   S  all-gather:     local load -> multimem.st (switch writes every member)
//   F  all-reduce:     multimem.ld_reduce -> multimem.st of the same tile
//   R1 reduce:         GPU 0 alone ld_reduces all S bytes (single issuer)
//   S1 broadcast:      GPU 0 alone multicasts all S bytes (single issuer)
// GPU r works on chunk r of S bytes (R, S, F); reports per-GPU link bytes and busbw.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Iinclude -o tools/nvlsbench tools/nvlsbench.cu \
//        -Lpaper_2408_05962_b200/lib -lhiccl -Xlinker -rpath,$PWD/paper_2408_05962_b200/lib
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "hiccl.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint4 ldred(const uint4* p) {
  uint4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mst(uint4* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w) : "memory");
}

// MODE 0 = R, 1 = S, 2 = F (R1 / S1 launch MODE 0 / 1 on GPU 0 only)
template <int MODE, int U>
__global__ void __launch_bounds__(1024) body(const uint4* src, uint4* dst, long nvec) {
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U; base < nvec; base += stride) {
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long v = base + u * blockDim.x + threadIdx.x;
      if (v < nvec) a[u] = MODE == 1 ? __ldcg(src + v) : ldred(src + v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long v = base + u * blockDim.x + threadIdx.x;
      if (v < nvec) {
        if (MODE == 0) __stcg(dst + v, a[u]);
        else mst(dst + v, a[u]);
      }
    }
  }
}

using Fn = void (*)(const uint4*, uint4*, long);
template <int MODE>
Fn pick(int u) {
  switch (u) {
    case 1: return body<MODE, 1>;
    case 2: return body<MODE, 2>;
    case 4: return body<MODE, 4>;
    case 8: return body<MODE, 8>;
    default: return body<MODE, 16>;
  }
}

int main(int argc, char** argv) {
  const size_t S = argc > 1 ? strtoull(argv[1], nullptr, 0) : (1ull << 30);
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  std::vector<int> devs(n);
  for (int i = 0; i < n; ++i) devs[i] = i;
  hc_window* w = nullptr;
  if (hc_window_create(devs.data(), n, 2 * S, &w) != 0) {
    fprintf(stderr, "window: %s\n", hc_last_error());
    return 1;
  }
  std::vector<char*> uc(n), mc(n);
  for (int i = 0; i < n; ++i) {
    void *u = nullptr, *m = nullptr;
    size_t b = 0;
    hc_window_pointers(w, i, &u, &m, &b);
    uc[i] = (char*)u;
    mc[i] = (char*)m;
    CK(cudaSetDevice(i));
    CK(cudaMemset(uc[i], 0, 2 * S));
  }
  for (int i = 0; i < n; ++i) { CK(cudaSetDevice(i)); CK(cudaDeviceSynchronize()); }
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(i));
    CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[i]));
    CK(cudaEventCreate(&e1[i]));
  }
  const size_t chunk = S / n;
  const long nvec = (long)(chunk / 16);
  const char* names[] = {"R", "S", "F", "R1", "S1"};
  const int us[] = {2, 4, 8, 16};
  const int ths[] = {256, 512, 1024};
  const int cps[] = {1, 2, 4};
  const int first_mode = argc > 2 ? atoi(argv[2]) : 0;
  for (int mode = first_mode; mode < 5; ++mode)
    for (int u : us)
      for (int th : ths)
        for (int cpsm : cps) {
          if (th * cpsm > 2048) continue;
          const int km = mode == 3 ? 0 : mode == 4 ? 1 : mode;
          const bool single = mode >= 3;
          Fn fn = km == 0 ? pick<0>(u) : km == 1 ? pick<1>(u) : pick<2>(u);
          cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
          int occ = 0;
          CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, th, 0));
          if (occ < cpsm) continue;
          const int grid = 148 * cpsm;
          float best = 1e30f;
          for (int rep = 0; rep < 4; ++rep) {
            const int users = single ? 1 : n;
            for (int i = 0; i < users; ++i) {
              CK(cudaSetDevice(i));
              const size_t off = (size_t)i * chunk;
              const uint4* src = (const uint4*)(km == 1 ? uc[i] + off : mc[i] + off);
              uint4* dst = (uint4*)(km == 0 ? uc[i] + S + off : mc[i] + S + off);
              CK(cudaEventRecord(e0[i], st[i]));
              fn<<<grid, th, 0, st[i]>>>(src, dst, single ? (long)(S / 16) : nvec);
              CK(cudaGetLastError());
              CK(cudaEventRecord(e1[i], st[i]));
            }
            float worst = 0;
            for (int i = 0; i < users; ++i) {
              CK(cudaSetDevice(i));
              CK(cudaEventSynchronize(e1[i]));
              float ms = 0;
              CK(cudaEventElapsedTime(&ms, e0[i], e1[i]));
              worst = ms > worst ? ms : worst;
            }
            if (rep > 0 && worst < best) best = worst;
          }
          // per GPU link bytes (egress, ingress) for S bytes per rank
          const double c = (double)chunk, s = (double)S;
          double eg = 0, in = 0, busf = 1;
          if (mode == 0) { eg = s; in = c; busf = (n - 1.0) / n; }
          if (mode == 1) { eg = c; in = s; busf = (n - 1.0) / n; }
          if (mode == 2) { eg = s + c; in = s + c; busf = 2.0 * (n - 1) / n; }
          if (mode == 3) { eg = s; in = s; busf = 1; }  // every GPU serves S; GPU 0 draws S
          if (mode == 4) { eg = s; in = s; busf = 1; }  // GPU 0 sends S; every GPU lands S
          const double t = best / 1e3;
          printf("{\"mode\": \"%s\", \"p\": %d, \"U\": %d, \"threads\": %d, \"ctas\": %d, \"us\": %.1f, "
                 "\"egress_gbs\": %.1f, \"ingress_gbs\": %.1f, \"busbw\": %.1f}\n",
                 names[mode], n, u, th, grid, best * 1e3, eg / t / 1e9, in / t / 1e9, s / t / 1e9 * busf);
          fflush(stdout);
        }
  hc_window_destroy(w);
  return 0;
}
