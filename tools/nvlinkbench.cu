// Development microbenchmark: raw peer read / write bandwidth between two
// B200s over NVLink (one process, peer access), uni- and bidirectional.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U>
__global__ void __launch_bounds__(512) copy(const uint4* __restrict__ src, uint4* __restrict__ dst, long nvec) {
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U; base < nvec; base += stride) {
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long v = base + u * blockDim.x + threadIdx.x; if (v < nvec) a[u] = __ldcg(src + v); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long v = base + u * blockDim.x + threadIdx.x; if (v < nvec) __stcg(dst + v, a[u]); }
  }
}

int main() {
  const long bytes = 1L << 30, n = bytes / 16;
  uint4 *a[2], *b[2];
  cudaStream_t s[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d)); CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&a[d], bytes)); CK(cudaMalloc(&b[d], bytes)); cudaMemset(a[d], d, bytes);
    cudaStreamCreate(&s[d]); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]);
  }
  int grids[] = {74, 148, 296};
  for (int mode = 0; mode < 4; ++mode) {  // 0 read uni, 1 read bi, 2 write uni, 3 write bi
    for (int g : grids) for (int U : {4, 8}) {
      float best = 1e9;
      for (int it = 0; it < 4; ++it) {
        for (int d = 0; d < 2; ++d) {
          if ((mode == 0 || mode == 2) && d == 1) continue;
          cudaSetDevice(d);
          const uint4* src = (mode < 2) ? a[1 - d] : a[d];
          uint4* dst = (mode < 2) ? b[d] : b[1 - d];
          cudaEventRecord(e0[d], s[d]);
          if (U == 4) copy<4><<<g, 512, 0, s[d]>>>(src, dst, n); else copy<8><<<g, 512, 0, s[d]>>>(src, dst, n);
          cudaEventRecord(e1[d], s[d]);
        }
        float worst = 0;
        for (int d = 0; d < 2; ++d) {
          if ((mode == 0 || mode == 2) && d == 1) continue;
          cudaSetDevice(d); cudaEventSynchronize(e1[d]);
          float ms; cudaEventElapsedTime(&ms, e0[d], e1[d]); if (ms > worst) worst = ms;
        }
        if (it > 0 && worst < best) best = worst;
      }
      const char* names[] = {"peer READ  uni", "peer READ  bi ", "peer WRITE uni", "peer WRITE bi "};
      printf("%s grid=%d U=%d: %.3f ms  %.0f GB/s per direction\n", names[mode], g, U, best, bytes / best / 1e6);
    }
  }
  return 0;
}
