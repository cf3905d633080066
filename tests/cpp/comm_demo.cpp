// The paper's Listing 2 through hiccl::Comm<float>:
// all-reduce composed as reduce-scatter, fence, in-place all-gather, one
// process per GPU, bootstrap over files in a shared directory. Checks the
// result bit for bit against the fold order of the plan (ascending source
// rank per chunk, one IEEE add per fold).
//
//   comm_demo <rank> <world> <device> <count_per_rank> <bootdir> [pipeline] [nvls]
//
// With "nvls" the buffers come from Comm::alloc_nvls and init() names the
// NVLS library: the switch reduces in its own order (fp32 accumulation), so
// the check is |got - fold| <= 1e-6 * sum |x| instead of bit equality.
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

int main(int argc, char** argv) {
  if (argc < 6) return 2;
  const int rank = atoi(argv[1]), world = atoi(argv[2]), device = atoi(argv[3]);
  const size_t n = strtoull(argv[4], nullptr, 10);
  const std::string dir = argv[5];
  const int pipeline = argc > 6 ? atoi(argv[6]) : 1;
  const bool nvls = argc > 7 && std::string(argv[7]) == "nvls";
  cudaSetDevice(device);
  float *send = nullptr, *recv = nullptr;
  try {
    hiccl::Comm<float> comm(rank, world, device, [&](const std::string& b) {
      return file_allgather(dir, rank, world, b);
    });
    if (nvls) {
      send = comm.alloc_nvls(world * n);
      recv = comm.alloc_nvls(world * n);
    } else {
      cudaMalloc(&send, world * n * sizeof(float));
      cudaMalloc(&recv, world * n * sizeof(float));
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
    hiccl::check(hc_device_fill(device, send, (int64_t)(world * n), HC_F32, 42, rank, 0, nullptr));
    cudaDeviceSynchronize();
    for (int it = 0; it < 3; ++it) {
      comm.start();
      comm.wait();
    }
    // expected: per element, fold ascending ranks (plan order), fp32 adds
    std::vector<float> got(world * n), in(world * n), acc(world * n), mag(world * n);
    cudaMemcpy(got.data(), recv, got.size() * sizeof(float), cudaMemcpyDeviceToHost);
    float* tmp = nullptr;
    cudaMalloc(&tmp, in.size() * sizeof(float));
    for (int r = 0; r < world; ++r) {
      hiccl::check(hc_device_fill(device, tmp, (int64_t)in.size(), HC_F32, 42, r, 0, nullptr));
      cudaMemcpy(in.data(), tmp, in.size() * sizeof(float), cudaMemcpyDeviceToHost);
      for (size_t k = 0; k < in.size(); ++k) {
        acc[k] = r == 0 ? in[k] : acc[k] + in[k];
        mag[k] = r == 0 ? std::fabs(in[k]) : mag[k] + std::fabs(in[k]);
      }
    }
    cudaFree(tmp);
    size_t bad = 0;
    for (size_t k = 0; k < acc.size(); ++k)
      bad += nvls ? std::fabs(acc[k] - got[k]) > 1e-6f * mag[k] : std::memcmp(&acc[k], &got[k], 4) != 0;
    const hc_exec_stats st = comm.stats();
    std::printf("rank %d/%d: %zu mismatches of %zu, %d items, %d steps, %d nvls items\n", rank, world,
                bad, acc.size(), st.num_items, st.num_steps, st.nvls_items);
    if (!nvls) {
      cudaFree(send);
      cudaFree(recv);
    }
    return bad ? 1 : 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "rank %d: %s\n", rank, e.what());
    return 3;
  }
}
