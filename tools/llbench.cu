// Development microbenchmark: tagged-line (LL) exchange latency between two
// B200s (one process, peer access). (A) a persistent kernel doing N
// exchanges in a loop; (B) one exchange per kernel launch, N launches
// captured in a CUDA graph per device (normal and cooperative launches).
// Every poll is bounded by %globaltimer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/llbench tools/llbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ long long gt() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

// one exchange: every thread stores its lines into the peer's buffer, then
// polls its own buffer for the same tag
__device__ int g_store_mode = 0;  // 0 st.volatile, 1 st.relaxed.sys, 2 weak st.global, 3 weak .cg

template <int M>
__device__ __forceinline__ void st16(uint4* p, uint32_t a, uint32_t t) {
  if constexpr (M == 0) asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(t), "r"(a), "r"(t) : "memory");
  else if constexpr (M == 1) asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(t), "r"(a), "r"(t) : "memory");
  else if constexpr (M == 2) asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(t), "r"(a), "r"(t) : "memory");
  else asm volatile("st.global.cg.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(t), "r"(a), "r"(t) : "memory");
}

__device__ __forceinline__ bool exchange(uint4* peer, uint4* mine, int lines, uint32_t tag, long long deadline) {
  const int m = g_store_mode;
  for (int l = threadIdx.x; l < lines; l += blockDim.x) {
    if (m == 0) st16<0>(peer + l, l, tag);
    else if (m == 1) st16<1>(peer + l, l, tag);
    else if (m == 2) st16<2>(peer + l, l, tag);
    else st16<3>(peer + l, l, tag);
  }
  for (int l = threadIdx.x; l < lines; l += blockDim.x) {
    while (true) {
      uint32_t a, b, c, d;
      asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(mine + l) : "memory");
      if (b == tag && d == tag) break;
      if (gt() > deadline) return false;
    }
  }
  return true;
}

__global__ void loop_kernel(uint4* peer, uint4* mine, int lines, int n, long long* out) {
  const long long t0 = gt();
  const int per = lines / gridDim.x;  // this CTA's share
  for (int e = 1; e <= n; ++e) {
    uint4* p = peer + (e & 1) * lines + blockIdx.x * per;
    uint4* m = mine + (e & 1) * lines + blockIdx.x * per;
    if (!exchange(p, m, per, (uint32_t)e, t0 + 2000000000LL)) { out[0] = -1; return; }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (gt() - t0) / n;
}

// one exchange per launch; the epoch is a device counter bumped at exit
__global__ void once_kernel(uint4* peer, uint4* mine, int lines, unsigned long long* epoch, long long* stamps) {
  const unsigned long long e = *(volatile unsigned long long*)epoch + 1;
  const long long t0 = gt();
  uint4* p = peer + (e & 1) * lines;
  uint4* m = mine + (e & 1) * lines;
  exchange(p, m, lines, (uint32_t)e, t0 + 2000000000LL);
  __syncthreads();
  if (threadIdx.x == 0) {
    stamps[2 * (e % 512)] = t0;
    stamps[2 * (e % 512) + 1] = gt();
    *epoch = e;
  }
}

int main() {
  int nd = 0;
  CK(cudaGetDeviceCount(&nd));
  if (nd < 2) { printf("needs 2 GPUs\n"); return 0; }
  uint4* buf[2];
  long long* out[2];
  unsigned long long* ep[2];
  cudaStream_t s[2];
  const int max_lines = 1 << 16;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d], 2 * max_lines * sizeof(uint4)));
    CK(cudaMallocManaged(&out[d], 4096 * sizeof(long long)));
    CK(cudaMalloc(&ep[d], 8));
    CK(cudaStreamCreateWithFlags(&s[d], cudaStreamNonBlocking));
  }
  for (int mode = 0; mode < 4; ++mode)
  for (int grid : {4, 64}) for (int lines : {8192, 131072 / 2}) {
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaMemcpyToSymbol(g_store_mode, &mode, sizeof(int))); }
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaMemset(buf[d], 0, 2 * max_lines * sizeof(uint4))); CK(cudaDeviceSynchronize()); }
    const int n = 500;
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); loop_kernel<<<grid, 512, 0, s[d]>>>(buf[1 - d], buf[d], lines, n, out[d]); }
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaStreamSynchronize(s[d])); }
    printf("store mode %d persistent loop: %7d B payload, %3d CTAs x 512: %lld ns per exchange\n", mode, lines * 8, grid, out[0][0]);
  }
  for (int lines : {64, 1024, 16384}) {
    for (int threads : {64, 512}) {
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaMemset(buf[d], 0, 2 * max_lines * sizeof(uint4))); CK(cudaDeviceSynchronize()); }
      const int n = 2000;
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); loop_kernel<<<1, threads, 0, s[d]>>>(buf[1 - d], buf[d], lines, n, out[d]); }
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaStreamSynchronize(s[d])); }
      printf("persistent loop: %6d B payload, %3d threads: %lld ns per exchange\n", lines * 8, threads, out[0][0]);
    }
  }
  // (B) graph of N single-exchange launches per device
  for (int coop = 0; coop < 2; ++coop) for (int lines : {64, 1024}) {
    const int n = 200;
    cudaGraphExec_t ge[2];
    for (int d = 0; d < 2; ++d) {
      cudaSetDevice(d);
      CK(cudaMemset(buf[d], 0, 2 * max_lines * sizeof(uint4)));
      CK(cudaMemset(ep[d], 0, 8));
      CK(cudaDeviceSynchronize());
      cudaGraph_t g;
      CK(cudaStreamBeginCapture(s[d], cudaStreamCaptureModeThreadLocal));
      for (int i = 0; i < n; ++i) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(1); lc.blockDim = dim3(64); lc.stream = s[d];
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = coop;
        lc.attrs = at; lc.numAttrs = 1;
        uint4* pp = buf[1 - d]; uint4* mm = buf[d]; int ln = lines; unsigned long long* e = ep[d]; long long* st = out[d];
        void* args[] = {&pp, &mm, &ln, &e, &st};
        CK(cudaLaunchKernelExC(&lc, (const void*)once_kernel, args));
      }
      CK(cudaStreamEndCapture(s[d], &g));
      CK(cudaGraphInstantiate(&ge[d], g, 0));
    }
    cudaEvent_t a[2], b[2];
    for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaEventCreate(&a[d]); cudaEventCreate(&b[d]); }
    for (int rep = 0; rep < 2; ++rep) {
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaEventRecord(a[d], s[d]); CK(cudaGraphLaunch(ge[d], s[d])); cudaEventRecord(b[d], s[d]); }
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaStreamSynchronize(s[d])); }
    }
    float ms[2];
    for (int d = 0; d < 2; ++d) cudaEventElapsedTime(&ms[d], a[d], b[d]);
    // in-kernel time and gap between consecutive launches on device 0
    long long in_sum = 0, gap_sum = 0; int cnt = 0;
    for (int e = 2 * n - 50; e < 2 * n - 1; ++e) {
      const long long s0 = out[0][2 * (e % 512)], e0 = out[0][2 * (e % 512) + 1], s1 = out[0][2 * ((e + 1) % 512)];
      in_sum += e0 - s0; gap_sum += s1 - e0; ++cnt;
    }
    printf("graph of %d launches (coop=%d), %5d B payload: %.2f us per launch (dev0 %.2f dev1 %.2f ms); in-kernel %.2f us, gap %.2f us\n",
           n, coop, lines * 8, ms[0] * 1e3 / n, ms[0], ms[1], in_sum / 1e3 / cnt, gap_sum / 1e3 / cnt);
    // cross-device start skew (globaltimer assumed common)
    long long sk = 0;
    for (int e = 2 * n - 50; e < 2 * n; ++e) sk += out[0][2 * (e % 512)] - out[1][2 * (e % 512)];
    printf("   mean start(dev0) - start(dev1): %.2f us\n", sk / 1e3 / 50);
  }
  return 0;
}
