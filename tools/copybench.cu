// Development microbenchmark: load/store flavours for the executor's copy body.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

template <int MODE>
__device__ __forceinline__ uint4 ld(const uint4* p) {
  if constexpr (MODE == 0) return *p;
  else if constexpr (MODE == 1) return __ldcg(p);
  else { uint4 v; asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p)); return v; }
}
template <int MODE>
__device__ __forceinline__ void st(uint4* p, uint4 v) {
  if constexpr (MODE == 0) *p = v;
  else if constexpr (MODE == 1) __stcg(p, v);
  else __stcs(p, v);
}

template <int MODE, int U, bool SYNC>
__global__ void __launch_bounds__(512) tiles(const uint4* __restrict__ src, uint4* __restrict__ dst, long nvec) {
  const int nt = blockDim.x;
  const long tile = (long)nt * U;
  const long ntiles = (nvec + tile - 1) / tile;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (SYNC) __syncthreads();
    const long base = t * tile;
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long v = base + u * nt + threadIdx.x; if (v < nvec) a[u] = ld<MODE>(src + v); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long v = base + u * nt + threadIdx.x; if (v < nvec) st<MODE>(dst + v, a[u]); }
  }
}

template <class K>
float timeit(K k, int grid, int block, const uint4* s, uint4* d, long n) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, block>>>(s, d, n);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) k<<<grid, block>>>(s, d, n);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10;
}

int main() {
  const long bytes = 1L << 30; const long n = bytes / 16;
  uint4 *s, *d; cudaMalloc(&s, bytes); cudaMalloc(&d, bytes); cudaMemset(s, 1, bytes);
  int grids[] = {148, 296, 592, 1184};
#define RUN(M, U, S) for (int g : grids) { float ms = timeit(tiles<M, U, S>, g, 512, s, d, n); printf("mode=%d U=%d sync=%d grid=%d: %.3f ms %.0f GB/s\n", M, U, S, g, ms, 2.0 * bytes / ms / 1e6); }
  RUN(0, 4, false) RUN(1, 4, false) RUN(2, 4, false) RUN(0, 4, true) RUN(1, 4, true) RUN(0, 8, false) RUN(0, 2, false) RUN(1, 8, false)
  return 0;
}
