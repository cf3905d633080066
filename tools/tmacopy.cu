// Development microbenchmark: 1 GiB HBM copy, LDG/STG (the executor's body)
// against a TMA bulk-copy pipeline (cp.async.bulk global->shared with an
// mbarrier, shared->global bulk groups), one elected thread per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmacopy tools/tmacopy.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) ldst(const uint4* __restrict__ src, uint4* __restrict__ dst, long nvec) {
  constexpr int U = 4;
  const long stride = (long)gridDim.x * blockDim.x * U;
  for (long base = (long)blockIdx.x * blockDim.x * U; base < nvec; base += stride) {
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long v = base + u * blockDim.x + threadIdx.x; if (v < nvec) a[u] = __ldcg(src + v); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long v = base + u * blockDim.x + threadIdx.x; if (v < nvec) __stcg(dst + v, a[u]); }
  }
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(m)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_addr(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_addr(m)) : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// chunks of C bytes, K stages; chunk i of this CTA = blockIdx.x + i * gridDim.x
__global__ void tma_copy(const char* __restrict__ src, char* __restrict__ dst, long bytes, int C, int K) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[8];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < K; ++s) mbar_init(&mbar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long nchunks = (bytes + C - 1) / C;
  const long mine = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto chunk_bytes = [&](long i) {
    const long c = blockIdx.x + i * gridDim.x;
    const long lo = c * C;
    return (uint32_t)(bytes - lo < C ? bytes - lo : C);
  };
  auto issue_load = [&](long i) {
    const int s = (int)(i % K);
    const long c = blockIdx.x + i * gridDim.x;
    const uint32_t b = chunk_bytes(i);
    mbar_expect(&mbar[s], b);
    bulk_load(smem + (size_t)s * C, src + c * C, b, &mbar[s]);
  };
  for (long j = 0; j < K - 1 && j < mine; ++j) issue_load(j);
  for (long i = 0; i < mine; ++i) {
    const long j = i + K - 1;
    if (j < mine) {
      if (j >= K) bulk_wait_read0();  // the store that last used stage j % K has read it
      issue_load(j);
    }
    const int s = (int)(i % K);
    mbar_wait(&mbar[s], (uint32_t)((i / K) & 1));
    const long c = blockIdx.x + i * gridDim.x;
    bulk_store(dst + c * C, smem + (size_t)s * C, chunk_bytes(i));
  }
  bulk_wait0();
}

int main() {
  const long bytes = 1L << 30;
  char *s, *d;
  cudaMalloc(&s, bytes); cudaMalloc(&d, bytes); cudaMemset(s, 1, bytes); cudaMemset(d, 0, bytes);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto report = [&](const char* what, float ms) { printf("%-40s %.3f ms  %.0f GB/s (r+w)\n", what, ms, 2.0 * bytes / ms / 1e6); };
  {
    for (int i = 0; i < 3; ++i) ldst<<<148, 512>>>((const uint4*)s, (uint4*)d, bytes / 16);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) ldst<<<148, 512>>>((const uint4*)s, (uint4*)d, bytes / 16);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); report("ldg/stg 148x512 U=4", ms / 10);
  }
  cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int per_sm : {1, 2, 4})
    for (int C : {16384, 32768, 49152})
      for (int K : {2, 3, 4, 6}) {
        const size_t smem = (size_t)C * K;
        if (smem * per_sm > 220 * 1024) continue;
        const int grid = 148 * per_sm;
        for (int i = 0; i < 2; ++i) tma_copy<<<grid, 32, smem>>>(s, d, bytes, C, K);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) tma_copy<<<grid, 32, smem>>>(s, d, bytes, C, K);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        char buf[96]; snprintf(buf, sizeof buf, "tma %d/SM C=%dK K=%d", per_sm, C / 1024, K);
        report(buf, ms / 10);
      }
  // correctness of the last configuration
  char h[64];
  cudaMemcpy(h, d + bytes - 64, 64, cudaMemcpyDeviceToHost);
  printf("tail byte %d (expect 1)\n", h[63]);
  return 0;
}
