// The paper's Listing 2 through hiccl::Comm<float>:
// all-reduce composed as reduce-scatter, fence, in-place all-gather, one
// process per GPU, bootstrap over files in a shared directory. Checks the
// result bit for bit against the fold order of the plan (ascending source
// rank per chunk, one IEEE add per fold).
//
//   comm_demo <rank> <world> <device> <count_per_rank> <bootdir> [pipeline] [nvls|bf16|f16]...
//
// With "nvls" the buffers come from Comm::alloc_nvls and init() names the
// NVLS library: the switch reduces in its own order (fp32 accumulation), so
// the check is |got - fold| <= rtol * sum |x| (rtol 1e-6 f32, 1e-2 16-bit)
// instead of bit equality. "bf16" / "f16" run Comm<__nv_bfloat16> /
// Comm<__half>: every fold widens to fp32, adds, rounds to nearest even.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "hiccl/comm.hpp"

static std::vector<std::string> file_allgather(const std::string& dir, int rank, int world,
                                               const std::string& blob) {
  static int round = 0;  // one file set per call (alloc_nvls exchanges several times)
  const std::string tag = dir + "/blob." + std::to_string(round++) + ".";
  const std::string mine = tag + std::to_string(rank);
  {
    std::ofstream(mine + ".tmp", std::ios::binary) << blob;
  }
  std::rename((mine + ".tmp").c_str(), mine.c_str());
  std::vector<std::string> all(world);
  for (int r = 0; r < world; ++r) {
    const std::string f = tag + std::to_string(r);
    for (int tries = 0;; ++tries) {
      std::ifstream in(f, std::ios::binary);
      if (in) {
        std::stringstream ss;
        ss << in.rdbuf();
        all[r] = ss.str();
        break;
      }
      if (tries > 60000) throw std::runtime_error("bootstrap timeout");
      usleep(1000);
    }
  }
  return all;
}

template <class T> struct Num;
template <> struct Num<float> {
  static constexpr int dt = HC_F32;
  static float f(float v) { return v; }
  static float add(float a, float b) { return a + b; }
  static constexpr float rtol = 1e-6f;
};
template <> struct Num<__nv_bfloat16> {
  static constexpr int dt = HC_BF16;
  static float f(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __nv_bfloat16 add(__nv_bfloat16 a, __nv_bfloat16 b) { return __float2bfloat16_rn(f(a) + f(b)); }
  static constexpr float rtol = 1e-2f;
};
template <> struct Num<__half> {
  static constexpr int dt = HC_F16;
  static float f(__half v) { return __half2float(v); }
  static __half add(__half a, __half b) { return __float2half_rn(f(a) + f(b)); }
  static constexpr float rtol = 1e-2f;
};

template <class T>
int run(int rank, int world, int device, size_t n, const std::string& dir, int pipeline, bool nvls) {
  using N = Num<T>;
  T *send = nullptr, *recv = nullptr;
  hiccl::Comm<T> comm(rank, world, device, [&](const std::string& b) {
    return file_allgather(dir, rank, world, b);
  });
  if (nvls) {
    send = comm.alloc_nvls(world * n);
    recv = comm.alloc_nvls(world * n);
  } else {
    cudaMalloc(&send, world * n * sizeof(T));
    cudaMalloc(&recv, world * n * sizeof(T));
  }
  std::vector<int> all(world);
  for (int r = 0; r < world; ++r) all[r] = r;
  for (int j = 0; j < world; ++j)
    comm.add_reduction(send + j * n, recv + j * n, n, all, j, hiccl::op::sum);
  if (world > 1) {
    comm.add_fence();
    for (int i = 0; i < world; ++i) {
      std::vector<int> others;
      for (int r = 0; r < world; ++r)
        if (r != i) others.push_back(r);
      comm.add_multicast(recv + i * n, recv + i * n, n, i, others);
    }
  }
  comm.init({world}, {nvls ? "NVLS" : "IPC"}, /*ring*/ 1, /*stripe*/ 1, pipeline);
  hiccl::check(hc_device_fill(device, send, (int64_t)(world * n), N::dt, 42, rank, 0, nullptr));
  cudaDeviceSynchronize();
  for (int it = 0; it < 3; ++it) {
    comm.start();
    comm.wait();
  }
  // expected: per element, fold ascending ranks (plan order)
  std::vector<T> got(world * n), in(world * n), acc(world * n);
  std::vector<float> mag(world * n);
  cudaMemcpy(got.data(), recv, got.size() * sizeof(T), cudaMemcpyDeviceToHost);
  T* tmp = nullptr;
  cudaMalloc(&tmp, in.size() * sizeof(T));
  for (int r = 0; r < world; ++r) {
    hiccl::check(hc_device_fill(device, tmp, (int64_t)in.size(), N::dt, 42, r, 0, nullptr));
    cudaMemcpy(in.data(), tmp, in.size() * sizeof(T), cudaMemcpyDeviceToHost);
    for (size_t k = 0; k < in.size(); ++k) {
      acc[k] = r == 0 ? in[k] : N::add(acc[k], in[k]);
      mag[k] = r == 0 ? std::fabs(N::f(in[k])) : mag[k] + std::fabs(N::f(in[k]));
    }
  }
  cudaFree(tmp);
  size_t bad = 0;
  for (size_t k = 0; k < acc.size(); ++k)
    bad += nvls ? std::fabs(N::f(acc[k]) - N::f(got[k])) > N::rtol * mag[k]
                : std::memcmp(&acc[k], &got[k], sizeof(T)) != 0;
  const hc_exec_stats st = comm.stats();
  std::printf("rank %d/%d: %zu mismatches of %zu, %d items, %d steps, %d nvls items, %zu-byte elements\n",
              rank, world, bad, acc.size(), st.num_items, st.num_steps, st.nvls_items, sizeof(T));
  if (!nvls) {
    cudaFree(send);
    cudaFree(recv);
  }
  return bad ? 1 : 0;
}

int main(int argc, char** argv) {
  if (argc < 6) return 2;
  const int rank = atoi(argv[1]), world = atoi(argv[2]), device = atoi(argv[3]);
  const size_t n = strtoull(argv[4], nullptr, 10);
  const std::string dir = argv[5];
  const int pipeline = argc > 6 ? atoi(argv[6]) : 1;
  bool nvls = false;
  std::string type = "f32";
  for (int a = 7; a < argc; ++a) {
    if (std::string(argv[a]) == "nvls") nvls = true;
    else type = argv[a];
  }
  cudaSetDevice(device);
  try {
    if (type == "bf16") return run<__nv_bfloat16>(rank, world, device, n, dir, pipeline, nvls);
    if (type == "f16") return run<__half>(rank, world, device, n, dir, pipeline, nvls);
    return run<float>(rank, world, device, n, dir, pipeline, nvls);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rank %d: %s\n", rank, e.what());
    return 3;
  }
}
