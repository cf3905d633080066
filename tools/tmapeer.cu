// Development microbenchmark: TMA bulk copies over NVLink (push / pull) against
// LDG/STG, 1 GiB, one process with two GPUs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmapeer tools/tmapeer.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(1024) ldst(const uint4* __restrict__ src, uint4* __restrict__ dst, long nvec) {
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


// (one process, two GPUs with peer access) push = local -> peer, pull = peer -> local
int main() {
  int nd = 0; cudaGetDeviceCount(&nd);
  if (nd < 2) { printf("needs 2 GPUs\n"); return 0; }
  const long bytes = 1L << 30;
  char *buf_a[2], *buf_b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d); cudaDeviceEnablePeerAccess(1 - d, 0);
    cudaMalloc(&buf_a[d], bytes); cudaMalloc(&buf_b[d], bytes);
    cudaMemset(buf_a[d], 1 + d, bytes); cudaMemset(buf_b[d], 0, bytes);
    cudaStreamCreate(&st[d]); cudaEventCreate(&e0[d]); cudaEventCreate(&e1[d]);
    cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  }
  // mode: 0 push ldst, 1 push tma, 2 pull ldst, 3 pull tma; bi: both GPUs at once
  const char* names[] = {"push ldg/stg", "push tma", "pull ldg/stg", "pull tma"};
  for (int bi = 0; bi < 2; ++bi)
    for (int mode = 0; mode < 4; ++mode)
      for (int C : {16384, 32768})
        for (int K : {2, 3}) {
          if (mode % 2 == 0 && (C != 16384 || K != 2)) continue;  // ldst: one config
          float best = 1e9;
          for (int rep = 0; rep < 3; ++rep) {
            for (int d = 0; d < 2; ++d) {
              if (!bi && d == 1) continue;
              cudaSetDevice(d);
              const char* src = mode < 2 ? buf_a[d] : buf_a[1 - d];
              char* dst = mode < 2 ? buf_b[1 - d] : buf_b[d];
              cudaEventRecord(e0[d], st[d]);
              for (int i = 0; i < 5; ++i) {
                if (mode % 2 == 0) ldst<4><<<148, 512, 0, st[d]>>>((const uint4*)src, (uint4*)dst, bytes / 16);
                else tma_copy<<<148, 32, (size_t)C * K, st[d]>>>(src, dst, bytes, C, K);
              }
              cudaEventRecord(e1[d], st[d]);
            }
            float ms = 0;
            for (int d = 0; d < 2; ++d) {
              if (!bi && d == 1) continue;
              cudaSetDevice(d); cudaEventSynchronize(e1[d]);
              float m; cudaEventElapsedTime(&m, e0[d], e1[d]); ms = m > ms ? m : ms;
            }
            best = ms / 5 < best ? ms / 5 : best;
          }
          cudaError_t e = cudaGetLastError();
          printf("%s %-14s C=%2dK K=%d: %.3f ms  %.0f GB/s per direction %s\n", bi ? "bidir" : "unidir",
                 names[mode], C / 1024, K, best, bytes / best / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
  return 0;
}
