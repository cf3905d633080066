// NVLS windows: symmetric device memory bound to an NVSwitch multicast
// object (CUDA multicast objects, driver API reached through the runtime's
// entry-point table so libhiccl.so never links libcuda directly).
//
// A window spans one device per executor. Every member owns `bytes` of
// physical memory (cuMemCreate) mapped at a unicast address; the multicast
// object maps the same offsets of every member at one multicast address,
// where `multimem.ld_reduce` reads-and-reduces across all members inside
// the switch and `multimem.st` writes to all members at once. Executors
// lower eligible reduction groups / multicasts onto it (executor.cu).
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../host/capi_common.hpp"
#include "hiccl.h"

using namespace hiccl;

namespace {

struct Driver {
  decltype(&cuMulticastCreate) mcCreate = nullptr;
  decltype(&cuMulticastAddDevice) mcAddDevice = nullptr;
  decltype(&cuMulticastBindMem) mcBindMem = nullptr;
  decltype(&cuMulticastUnbind) mcUnbind = nullptr;
  decltype(&cuMulticastGetGranularity) mcGranularity = nullptr;
  decltype(&cuMemCreate) memCreate = nullptr;
  decltype(&cuMemRelease) memRelease = nullptr;
  decltype(&cuMemAddressReserve) addrReserve = nullptr;
  decltype(&cuMemAddressFree) addrFree = nullptr;
  decltype(&cuMemMap) memMap = nullptr;
  decltype(&cuMemUnmap) memUnmap = nullptr;
  decltype(&cuMemSetAccess) memSetAccess = nullptr;
  decltype(&cuMemGetAllocationGranularity) allocGranularity = nullptr;
  decltype(&cuMemExportToShareableHandle) exportHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) importHandle = nullptr;
  decltype(&cuDeviceGet) deviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) deviceGetAttribute = nullptr;
  decltype(&cuGetErrorString) errorString = nullptr;
  bool ok = false;
};

template <class F>
void entry(const char* name, F& fn, bool& ok) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !f) {
    ok = false;
    return;
  }
  fn = reinterpret_cast<F>(f);
}

const Driver& drv() {
  static Driver d = [] {
    Driver x;
    x.ok = true;
    entry("cuMulticastCreate", x.mcCreate, x.ok);
    entry("cuMulticastAddDevice", x.mcAddDevice, x.ok);
    entry("cuMulticastBindMem", x.mcBindMem, x.ok);
    entry("cuMulticastUnbind", x.mcUnbind, x.ok);
    entry("cuMulticastGetGranularity", x.mcGranularity, x.ok);
    entry("cuMemCreate", x.memCreate, x.ok);
    entry("cuMemRelease", x.memRelease, x.ok);
    entry("cuMemAddressReserve", x.addrReserve, x.ok);
    entry("cuMemAddressFree", x.addrFree, x.ok);
    entry("cuMemMap", x.memMap, x.ok);
    entry("cuMemUnmap", x.memUnmap, x.ok);
    entry("cuMemSetAccess", x.memSetAccess, x.ok);
    entry("cuMemGetAllocationGranularity", x.allocGranularity, x.ok);
    entry("cuMemExportToShareableHandle", x.exportHandle, x.ok);
    entry("cuMemImportFromShareableHandle", x.importHandle, x.ok);
    entry("cuDeviceGet", x.deviceGet, x.ok);
    entry("cuDeviceGetAttribute", x.deviceGetAttribute, x.ok);
    entry("cuGetErrorString", x.errorString, x.ok);
    return x;
  }();
  return d;
}

void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = nullptr;
  if (drv().errorString) drv().errorString(r, &s);
  throw Error(ErrorCode::CudaError, std::string(what) + ": " + (s ? s : "CUDA driver error"));
}

void rt_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(ErrorCode::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct hc_window {
  struct Member {
    int device = -1;
    CUmemGenericAllocationHandle mem = 0;
    CUdeviceptr uc = 0;  // unicast mapping of this member's memory
    CUdeviceptr mc = 0;  // multicast mapping on this member's device
  };
  CUmemGenericAllocationHandle mc = 0;
  size_t size = 0;       // per member, rounded to the multicast granularity
  size_t gran = 0;       // recommended multicast granularity (mapping alignment)
  int n_members = 0;
  bool single_process = true;
  int exported_fd = -1;
  std::vector<Member> local;  // members driven by this process
  bool bound = false;
  int mem_fd = -1;            // exported physical memory of local[0] (multi-process)
  struct Peer {
    CUmemGenericAllocationHandle mem = 0;
    CUdeviceptr uc = 0;
  };
  std::vector<Peer> peers;    // imported unicast mappings of other members

  ~hc_window() {
    const Driver& d = drv();
    for (auto& m : local) {
      int prev = -1;
      cudaGetDevice(&prev);
      cudaSetDevice(m.device);
      cudaDeviceSynchronize();
      if (m.mc) {
        d.memUnmap(m.mc, size);
        d.addrFree(m.mc, size);
      }
      if (m.uc) {
        d.memUnmap(m.uc, size);
        d.addrFree(m.uc, size);
      }
      if (bound && m.mem) {
        CUdevice dev;
        d.deviceGet(&dev, m.device);
        d.mcUnbind(mc, dev, 0, size);
      }
      if (m.mem) d.memRelease(m.mem);
      if (prev >= 0) cudaSetDevice(prev);
    }
    for (auto& p : peers) {
      if (p.uc) {
        d.memUnmap(p.uc, size);
        d.addrFree(p.uc, size);
      }
      if (p.mem) d.memRelease(p.mem);
    }
    if (mc) d.memRelease(mc);
    if (exported_fd >= 0) close(exported_fd);
    if (mem_fd >= 0) close(mem_fd);
  }

  CUmemAllocationProp mem_prop(int device) const {
    CUmemAllocationProp p{};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return p;
  }

  void add_device(Member& m) {
    CUdevice dev;
    cu_check(drv().deviceGet(&dev, m.device), "cuDeviceGet");
    int supported = 0;
    cu_check(drv().deviceGetAttribute(&supported, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev),
             "cuDeviceGetAttribute");
    if (!supported)
      throw Error(ErrorCode::CudaError, "device " + std::to_string(m.device) +
                                            " does not support NVSwitch multicast");
    cu_check(drv().mcAddDevice(mc, dev), "cuMulticastAddDevice");
  }

  // Physical memory, bind, unicast + multicast mappings for one member.
  // `access` lists the devices that may touch the unicast mapping.
  void bind_member(Member& m, const std::vector<int>& access) {
    const Driver& d = drv();
    rt_check(cudaSetDevice(m.device), "cudaSetDevice");
    CUmemAllocationProp prop = mem_prop(m.device);
    cu_check(d.memCreate(&m.mem, size, &prop, 0), "cuMemCreate");
    cu_check(d.mcBindMem(mc, 0, m.mem, 0, size, 0), "cuMulticastBindMem");
    std::vector<CUmemAccessDesc> desc;
    for (int a : access) {
      CUmemAccessDesc x{};
      x.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      x.location.id = a;
      x.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      desc.push_back(x);
    }
    cu_check(d.addrReserve(&m.uc, size, gran, 0, 0), "cuMemAddressReserve(uc)");
    cu_check(d.memMap(m.uc, size, 0, m.mem, 0), "cuMemMap(uc)");
    cu_check(d.memSetAccess(m.uc, size, desc.data(), desc.size()), "cuMemSetAccess(uc)");
    CUmemAccessDesc self{};
    self.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    self.location.id = m.device;
    self.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cu_check(d.addrReserve(&m.mc, size, gran, 0, 0), "cuMemAddressReserve(mc)");
    cu_check(d.memMap(m.mc, size, 0, mc, 0), "cuMemMap(mc)");
    cu_check(d.memSetAccess(m.mc, size, &self, 1), "cuMemSetAccess(mc)");
    rt_check(cudaMemset((void*)m.uc, 0, size), "cudaMemset(window)");
    rt_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  }

  void create_object(int n, size_t bytes, bool exportable) {
    const Driver& d = drv();
    if (!d.ok) throw Error(ErrorCode::CudaError, "CUDA driver lacks the multicast API");
    CUmulticastObjectProp prop{};
    prop.numDevices = (unsigned)n;
    prop.size = bytes;
    prop.handleTypes = exportable ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : 0;
    cu_check(d.mcGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED),
             "cuMulticastGetGranularity");
    size = round_up(std::max<size_t>(bytes, 1), gran);
    prop.size = size;
    cu_check(d.mcCreate(&mc, &prop), "cuMulticastCreate");
  }
};

namespace {
using hiccl::capi::guard;

size_t granular_size(int n, size_t bytes, size_t* gran_out) {
  const Driver& d = drv();
  if (!d.ok) throw Error(ErrorCode::CudaError, "CUDA driver lacks the multicast API");
  CUmulticastObjectProp prop{};
  prop.numDevices = (unsigned)n;
  prop.size = bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  cu_check(d.mcGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED),
           "cuMulticastGetGranularity");
  *gran_out = gran;
  return round_up(std::max<size_t>(bytes, 1), gran);
}
}  // namespace

extern "C" {

hc_status hc_window_create(const int* devices, int n, size_t bytes, hc_window** out) {
  return guard([&] {
    if (n < 1 || !devices) throw Error(ErrorCode::InvalidConfig, "window needs devices");
    int prev = -1;
    cudaGetDevice(&prev);
    auto w = std::make_unique<hc_window>();
    w->n_members = n;
    w->single_process = true;
    rt_check(cudaSetDevice(devices[0]), "cudaSetDevice");
    cudaFree(nullptr);  // context
    w->create_object(n, bytes, false);
    w->local.resize(n);
    for (int i = 0; i < n; ++i) {
      w->local[i].device = devices[i];
      rt_check(cudaSetDevice(devices[i]), "cudaSetDevice");
      cudaFree(nullptr);
      w->add_device(w->local[i]);
    }
    std::vector<int> all(devices, devices + n);
    for (int i = 0; i < n; ++i) w->bind_member(w->local[i], all);
    w->bound = true;
    if (prev >= 0) cudaSetDevice(prev);
    *out = w.release();
  });
}

hc_status hc_window_open(int device, int n_members, size_t bytes, const unsigned char* handle,
                         hc_window** out) {
  return guard([&] {
    int prev = -1;
    cudaGetDevice(&prev);
    rt_check(cudaSetDevice(device), "cudaSetDevice");
    cudaFree(nullptr);
    auto w = std::make_unique<hc_window>();
    w->n_members = n_members;
    w->single_process = false;
    if (!handle) {
      w->create_object(n_members, bytes, true);
      int fd = -1;
      cu_check(drv().exportHandle(&fd, w->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
               "cuMemExportToShareableHandle");
      w->exported_fd = fd;
    } else {
      // handle = { int32 pid, int32 fd } of the creating process; take a
      // copy of its descriptor with pidfd_getfd (same host, same user).
      int32_t pid = 0, rfd = 0;
      std::memcpy(&pid, handle, 4);
      std::memcpy(&rfd, handle + 4, 4);
      const int pidfd = (int)syscall(SYS_pidfd_open, pid, 0);
      if (pidfd < 0) throw Error(ErrorCode::CudaError, "pidfd_open failed");
      const int fd = (int)syscall(SYS_pidfd_getfd, pidfd, rfd, 0);
      close(pidfd);
      if (fd < 0) throw Error(ErrorCode::CudaError, "pidfd_getfd failed (ptrace permission?)");
      w->size = granular_size(n_members, bytes, &w->gran);
      cu_check(drv().importHandle(&w->mc, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
               "cuMemImportFromShareableHandle");
      close(fd);
    }
    w->local.resize(1);
    w->local[0].device = device;
    w->add_device(w->local[0]);
    if (prev >= 0) cudaSetDevice(prev);
    *out = w.release();
  });
}

hc_status hc_window_export(hc_window* w, unsigned char handle[64]) {
  return guard([&] {
    if (w->exported_fd < 0) throw Error(ErrorCode::InvalidConfig, "window was not created here");
    std::memset(handle, 0, 64);
    const int32_t pid = (int32_t)getpid(), fd = w->exported_fd;
    std::memcpy(handle, &pid, 4);
    std::memcpy(handle + 4, &fd, 4);
  });
}

hc_status hc_window_bind(hc_window* w) {
  return guard([&] {
    if (w->bound) return;
    int prev = -1;
    cudaGetDevice(&prev);
    for (auto& m : w->local) w->bind_member(m, {m.device});
    w->bound = true;
    if (prev >= 0) cudaSetDevice(prev);
  });
}

// Peer unicast access across processes: each member exports its physical
// memory as a POSIX descriptor; peers take a copy with pidfd_getfd and map it.
hc_status hc_window_export_memory(hc_window* w, unsigned char handle[64]) {
  return guard([&] {
    if (!w->bound || w->local.size() != 1) throw Error(ErrorCode::InvalidConfig, "bind first");
    if (w->mem_fd < 0)
      cu_check(drv().exportHandle(&w->mem_fd, w->local[0].mem, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
               "cuMemExportToShareableHandle(memory)");
    std::memset(handle, 0, 64);
    const int32_t pid = (int32_t)getpid(), fd = w->mem_fd;
    std::memcpy(handle, &pid, 4);
    std::memcpy(handle + 4, &fd, 4);
  });
}

hc_status hc_window_import_memory(hc_window* w, const unsigned char handle[64], void** uc) {
  return guard([&] {
    if (!w->bound || w->local.size() != 1) throw Error(ErrorCode::InvalidConfig, "bind first");
    int32_t pid = 0, rfd = 0;
    std::memcpy(&pid, handle, 4);
    std::memcpy(&rfd, handle + 4, 4);
    const int pidfd = (int)syscall(SYS_pidfd_open, pid, 0);
    if (pidfd < 0) throw Error(ErrorCode::CudaError, "pidfd_open failed");
    const int fd = (int)syscall(SYS_pidfd_getfd, pidfd, rfd, 0);
    close(pidfd);
    if (fd < 0) throw Error(ErrorCode::CudaError, "pidfd_getfd failed (ptrace permission?)");
    int prev = -1;
    cudaGetDevice(&prev);
    rt_check(cudaSetDevice(w->local[0].device), "cudaSetDevice");
    hc_window::Peer peer;
    const Driver& d = drv();
    cu_check(d.importHandle(&peer.mem, (void*)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
             "cuMemImportFromShareableHandle(memory)");
    close(fd);
    cu_check(d.addrReserve(&peer.uc, w->size, w->gran, 0, 0), "cuMemAddressReserve(peer)");
    cu_check(d.memMap(peer.uc, w->size, 0, peer.mem, 0), "cuMemMap(peer)");
    CUmemAccessDesc a{};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = w->local[0].device;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cu_check(d.memSetAccess(peer.uc, w->size, &a, 1), "cuMemSetAccess(peer)");
    w->peers.push_back(peer);
    *uc = (void*)peer.uc;
    if (prev >= 0) cudaSetDevice(prev);
  });
}

hc_status hc_window_pointers(hc_window* w, int member, void** uc, void** mc, size_t* bytes) {
  return guard([&] {
    if (!w->bound) throw Error(ErrorCode::InvalidConfig, "window not bound yet");
    if (member < 0 || member >= (int)w->local.size())
      throw Error(ErrorCode::RankOutOfRange, "window member not driven by this process");
    *uc = (void*)w->local[member].uc;
    *mc = (void*)w->local[member].mc;
    *bytes = w->size;
  });
}

void hc_window_destroy(hc_window* w) { delete w; }

hc_status hc_nvls_supported(int device, int* supported) {
  return guard([&] {
    *supported = 0;
    if (!drv().ok) return;
    CUdevice dev;
    if (drv().deviceGet(&dev, device) != CUDA_SUCCESS) return;
    int s = 0;
    if (drv().deviceGetAttribute(&s, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) == CUDA_SUCCESS)
      *supported = s;
  });
}

}  // extern "C"
