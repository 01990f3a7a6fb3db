// ABI plumbing: version, error strings, device query.
#include <cuda_runtime.h>

#include <atomic>

#include "pcb_common.cuh"
#include "pcb_launch.cuh"

namespace pcb {
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v < 1) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}
}  // namespace pcb

extern "C" int pcb_abi_version(void) { return PCB_ABI_VERSION; }

extern "C" const char* pcb_error_string(int code) {
  switch (code) {
    case 0: return "success";
    case PCB_EINVAL: return "popcorn_b200: invalid argument (size or null pointer)";
    case PCB_EUNSUP: return "popcorn_b200: unsupported shape/variant for this kernel";
    case PCB_ENODEV: return "popcorn_b200: no sm_100 (B200) CUDA device";
    case -4: return "popcorn_b200: dataset parse error (see info/text)";
    default: break;
  }
  if (code > 0) return cudaGetErrorString((cudaError_t)code);
  return "popcorn_b200: unknown error";
}

extern "C" int pcb_device_info(int device, int* sm, int* major, int* minor) {
  int mj = 0, mn = 0, s = 0;
  cudaError_t e = cudaDeviceGetAttribute(&mj, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) return (int)e;
  cudaDeviceGetAttribute(&mn, cudaDevAttrComputeCapabilityMinor, device);
  cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, device);
  if (sm) *sm = s;
  if (major) *major = mj;
  if (minor) *minor = mn;
  return mj == 10 ? 0 : PCB_ENODEV;
}

extern "C" long long pcb_launch_count(void) { return pcb::g_launches.load(std::memory_order_relaxed); }
