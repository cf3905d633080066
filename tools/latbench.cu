// Development microbenchmark: the fixed costs of one executor launch on
// two B200s (one process, peer access): kernel launch, system fences, flag
// round trips over NVLink, dependent local / remote load latency.
// Every spin loop is bounded by %globaltimer (no hang if a peer is late).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/latbench tools/latbench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ long long gt() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint64_t ld_acq(const uint64_t* p) { uint64_t v; asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint64_t ld_rlx(const uint64_t* p) { uint64_t v; asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ uint64_t ld_vol(const uint64_t* p) { uint64_t v; asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_rlx(uint64_t* p, uint64_t v) { asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) { asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ void fence_ar() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_sc() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__global__ void empty_kernel() {}

// out[0] = ns per iteration of the selected fence with `stores` prior stores to `peer`
__global__ void fence_cost(int kind, uint64_t* peer, int stores, long long* out) {
  const int iters = 200;
  long long t0 = gt();
  for (int i = 0; i < iters; ++i) {
    for (int k = 0; k < stores; ++k) peer[k * 16] = i;
    if (kind == 0) fence_ar(); else if (kind == 1) fence_sc(); else if (kind == 2) fence_gpu(); else __threadfence_system();
  }
  out[0] = (gt() - t0) / iters;
}

// Dependent pointer chase; out = ns per load.
__global__ void chase(const uint64_t* p, int n, long long* out) {
  uint64_t i = 0;
  long long t0 = gt();
  for (int k = 0; k < n; ++k) i = __ldcg(p + i);
  out[0] = (gt() - t0) / n + (i == 12345678 ? 1 : 0);
}

// Ping-pong: GPU `me` (0 or 1). my_flag lives on my GPU, peer_flag on the
// peer (written by me remotely). mode 0: spin ld.acquire.sys, publish
// fence+red; 1: spin ld.relaxed + fence after, publish st.release;
// 2: spin volatile, publish red w/o fence.
__global__ void pingpong(int me, uint64_t* my_flag, uint64_t* peer_flag, int rounds, int mode,
                         long long* out) {
  long long t0 = gt();
  const long long deadline = t0 + 2000000000LL;
  for (int r = 1; r <= rounds; ++r) {
    if (me == 0 || r > 0) {
      if (me == 0) {
        if (mode == 0) { fence_ar(); red_rlx(peer_flag, r); }
        else if (mode == 1) st_rel(peer_flag, r);
        else red_rlx(peer_flag, r);
      }
      // wait for the answer
      while (true) {
        uint64_t v = mode == 0 ? ld_acq(my_flag) : mode == 1 ? ld_rlx(my_flag) : ld_vol(my_flag);
        if (v >= (uint64_t)r) break;
        if (gt() > deadline) { out[0] = -1; return; }
      }
      if (mode == 1) fence_ar();
      if (me == 1) {
        if (mode == 0) { fence_ar(); red_rlx(peer_flag, r); }
        else if (mode == 1) st_rel(peer_flag, r);
        else red_rlx(peer_flag, r);
      }
    }
  }
  out[0] = (gt() - t0) / rounds;
}

// Start skew across CTAs of one launch: out[b] = globaltimer at CTA entry.
__global__ void cta_start(long long* out) { if (threadIdx.x == 0) out[blockIdx.x] = gt(); }

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  uint64_t* buf[2];
  uint64_t* flags[2];
  long long* out[2];
  cudaStream_t s[2];
  const int nd = ndev >= 2 ? 2 : 1;
  for (int d = 0; d < nd; ++d) {
    CK(cudaSetDevice(d));
    if (nd == 2) CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d], 64 << 20));
    CK(cudaMalloc(&flags[d], 4096));
    CK(cudaMemset(flags[d], 0, 4096));
    CK(cudaMallocManaged(&out[d], 4096 * sizeof(long long)));
    CK(cudaStreamCreate(&s[d]));
  }
  CK(cudaSetDevice(0));
  // 1. launch overhead, back to back
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {1, 148}) for (int coop = 0; coop < 2; ++coop) {
    const int n = 200;
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0, s[0]);
      for (int i = 0; i < n; ++i) {
        if (coop) {
          void* args[] = {nullptr};
          CK(cudaLaunchCooperativeKernel((void*)empty_kernel, grid, 512, args, 0, s[0]));
        } else {
          empty_kernel<<<grid, 512, 0, s[0]>>>();
        }
      }
      cudaEventRecord(e1, s[0]);
      CK(cudaEventSynchronize(e1));
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("launch grid=%d coop=%d: %.2f us per launch (back to back)\n", grid, coop, ms * 1e3 / n);
  }
  // 1b. CTA start skew
  cta_start<<<148, 512, 0, s[0]>>>(out[0]);
  CK(cudaStreamSynchronize(s[0]));
  { long long lo = out[0][0], hi = out[0][0];
    for (int b = 0; b < 148; ++b) { lo = out[0][b] < lo ? out[0][b] : lo; hi = out[0][b] > hi ? out[0][b] : hi; }
    printf("cta start skew over 148 CTAs: %lld ns\n", hi - lo); }
  // 2. fence costs (local and with remote stores)
  const char* fname[] = {"fence.acq_rel.sys", "fence.sc.sys", "fence.acq_rel.gpu", "__threadfence_system"};
  for (int kind = 0; kind < 4; ++kind) for (int stores : {0, 1, 8}) for (int remote = 0; remote < nd; ++remote) {
    fence_cost<<<1, 1, 0, s[0]>>>(kind, remote ? buf[1] : buf[0], stores, out[0]);
    CK(cudaStreamSynchronize(s[0]));
    printf("%-22s stores=%d %s: %lld ns\n", fname[kind], stores, remote ? "remote" : "local ", out[0][0]);
  }
  // 3. dependent load latency, local (L2-resident) and remote
  {
    const int n = 1000;
    uint64_t* h = new uint64_t[n * 64];
    for (int i = 0; i < n * 64; ++i) h[i] = 0;
    for (int i = 0; i < n; ++i) h[i * 64] = ((i + 1) % n) * 64;  // stride 512 B
    for (int d = 0; d < nd; ++d) { cudaSetDevice(d); CK(cudaMemcpy(buf[d], h, n * 64 * 8, cudaMemcpyHostToDevice)); }
    cudaSetDevice(0);
    for (int remote = 0; remote < nd; ++remote) {
      for (int rep = 0; rep < 2; ++rep) {
        chase<<<1, 1, 0, s[0]>>>(remote ? buf[1] : buf[0], n, out[0]);
        CK(cudaStreamSynchronize(s[0]));
      }
      printf("dependent load latency %s: %lld ns\n", remote ? "remote (NVLink)" : "local (L2)", out[0][0]);
    }
    delete[] h;
  }
  // 4. ping-pong round trips between GPUs (both kernels resident at once)
  if (nd == 2) {
    const char* mname[] = {"fence+red / ld.acquire", "st.release / ld.relaxed+fence", "red / ld.volatile (no fence)"};
    for (int mode = 0; mode < 3; ++mode) {
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaMemset(flags[d], 0, 4096)); CK(cudaDeviceSynchronize()); }
      const int rounds = 2000;
      for (int d = 0; d < 2; ++d) {
        cudaSetDevice(d);
        pingpong<<<1, 1, 0, s[d]>>>(d, flags[d], flags[1 - d], rounds, mode, out[d]);
      }
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); CK(cudaStreamSynchronize(s[d])); }
      printf("ping-pong %-32s: %lld ns per round trip\n", mname[mode], out[0][0]);
    }
  }
  return 0;
}
