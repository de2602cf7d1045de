// C-ABI plumbing: error string, version, capability probe. Entry points live beside their kernels
// (leaf.cu, merge.cu, solve.cu, gemm.cu); all are declared in include/hps_b200.h.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace hps {
static thread_local char g_err[1024] = "";
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace hps

// Number of kernels this library has launched in this process (bench.py's gpu_launches).
extern "C" long long hps_launch_count(void) { return hps::g_launches.load(); }

extern "C" const char* hps_last_error(void) { return hps::g_err; }

extern "C" int hps_version(void) { return 1; }

// 0 when a device with compute capability 10.x is visible, HPS_ERR_CUDA otherwise.
extern "C" int hps_device_check(int* major, int* minor, int* sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    hps::set_error("cudaGetDevice: %s", cudaGetErrorString(e));
    return HPS_ERR_CUDA;
  }
  cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
  if (*major != 10) {
    hps::set_error("built for sm_100a, found sm_%d%d", *major, *minor);
    return HPS_ERR_CUDA;
  }
  return HPS_OK;
}
