// Development microbenchmark: p GPUs, every GPU moves 1/p-size chunks to or
// from every peer concurrently (the all-to-all pattern of reduce-scatter /
// all-gather), peer loads (pull) or peer stores (push).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) move(const uint4* const* src, uint4* const* dst, int npeer, long nvec) {
  // tile interleave over peers: tile t -> peer t % npeer
  const long tile = 512L * 8;
  const long tiles_per_peer = (nvec + tile - 1) / tile;
  const long total = tiles_per_peer * npeer;
  for (long t = blockIdx.x; t < total; t += gridDim.x) {
    const int peer = t % npeer;
    const long base = (t / npeer) * tile;
    const uint4* s = src[peer];
    uint4* d = dst[peer];
    uint4 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { long v = base + u * 512 + threadIdx.x; if (v < nvec) a[u] = __ldcg(s + v); }
#pragma unroll
    for (int u = 0; u < 8; ++u) { long v = base + u * 512 + threadIdx.x; if (v < nvec) __stcg(d + v, a[u]); }
  }
}

int main() {
  int p = 0;
  cudaGetDeviceCount(&p);
  const long chunk = (1L << 30) / p;  // per peer
  std::vector<uint4*> in(p), out(p);
  for (int d = 0; d < p; ++d) {
    cudaSetDevice(d);
    for (int e = 0; e < p; ++e) if (e != d) cudaDeviceEnablePeerAccess(e, 0);
    cudaMalloc(&in[d], chunk * p); cudaMalloc(&out[d], chunk * p);
  }
  for (int mode = 0; mode < 2; ++mode) {  // 0 pull, 1 push
    std::vector<uint4**> dsrc(p), ddst(p);
    for (int d = 0; d < p; ++d) {
      std::vector<uint4*> s, t;
      for (int e = 0; e < p; ++e) {
        if (e == d) continue;
        if (mode == 0) { s.push_back((uint4*)((char*)in[e] + d * chunk)); t.push_back((uint4*)((char*)out[d] + e * chunk)); }
        else { s.push_back((uint4*)((char*)in[d] + e * chunk)); t.push_back((uint4*)((char*)out[e] + d * chunk)); }
      }
      cudaSetDevice(d);
      cudaMalloc(&dsrc[d], sizeof(uint4*) * (p - 1)); cudaMalloc(&ddst[d], sizeof(uint4*) * (p - 1));
      cudaMemcpy(dsrc[d], s.data(), sizeof(uint4*) * (p - 1), cudaMemcpyHostToDevice);
      cudaMemcpy(ddst[d], t.data(), sizeof(uint4*) * (p - 1), cudaMemcpyHostToDevice);
    }
    std::vector<cudaEvent_t> a(p), b(p);
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      for (int d = 0; d < p; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); }
      for (int d = 0; d < p; ++d) {
        cudaSetDevice(d); cudaEventCreate(&a[d]); cudaEventCreate(&b[d]);
        cudaEventRecord(a[d]); move<<<148, 512>>>(dsrc[d], ddst[d], p - 1, chunk / 16); cudaEventRecord(b[d]);
      }
      float worst = 0;
      for (int d = 0; d < p; ++d) { cudaSetDevice(d); cudaEventSynchronize(b[d]); float ms; cudaEventElapsedTime(&ms, a[d], b[d]); if (ms > worst) worst = ms; }
      if (it && worst < best) best = worst;
    }
    printf("p=%d %s all-to-all chunks of %ld MiB: %.3f ms, %.0f GB/s per GPU per direction\n", p,
           mode ? "PUSH" : "PULL", chunk >> 20, best, (double)chunk * (p - 1) / best / 1e6);
  }
  return 0;
}
