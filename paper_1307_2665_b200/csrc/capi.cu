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

// ---------------------------------------------------------------------------------------------
// Contexts (ctx.cuh)
// ---------------------------------------------------------------------------------------------
#include <map>
#include <utility>

#include "ctx.cuh"

namespace hps {

int check_ctx(const Ctx* c, const char* fn) {
  if (!c) {
    set_error("%s: null hps_ctx_t", fn);
    return HPS_ERR_ARG;
  }
  int dev = -1;
  HPS_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev != c->device) {
    set_error("%s: context of device %d used while device %d is current", fn, c->device, dev);
    return HPS_ERR_ARG;
  }
  return HPS_OK;
}

double* Ctx::splitk_scratch(size_t n, cudaStream_t st) {
  const int r = role(st);
  if (n > splitk_n[r]) {
    // no allocation inside a stream capture (it would invalidate the capture): the caller then
    // runs without split-K. BuildGraph warms up first, so captures normally find it allocated.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    double* fresh = nullptr;
    if (cudaMalloc(&fresh, n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    if (splitk[r]) retired.push_back(splitk[r]);
    splitk[r] = fresh;
    splitk_n[r] = n;
  }
  return splitk[r];
}

double* Ctx::emu_scratch(size_t n, cudaStream_t st) {
  const int r = role(st);
  if (n > emu_n[r]) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    double* fresh = nullptr;
    if (cudaMalloc(&fresh, n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    if (emu_buf[r]) retired.push_back(emu_buf[r]);
    emu_buf[r] = fresh;
    emu_n[r] = n;
  }
  return emu_buf[r];
}

double* Ctx::gather_scratch(size_t n, cudaStream_t st) {
  const int r = role(st);
  if (n > gather_n[r]) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    double* fresh = nullptr;
    if (cudaMalloc(&fresh, n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    if (gather_buf[r]) retired.push_back(gather_buf[r]);
    gather_buf[r] = fresh;
    gather_n[r] = n;
  }
  return gather_buf[r];
}

int ensure_smem_attr(const void* kernel, int device, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(kernel, device);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return HPS_OK;
  HPS_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[key] = bytes;
  return HPS_OK;
}

}  // namespace hps

extern "C" int hps_ctx_create(int device, hps_ctx_t* out) {
  using namespace hps;
  if (!out) {
    set_error("hps_ctx_create: null out");
    return HPS_ERR_ARG;
  }
  *out = nullptr;
  int prev = 0;
  HPS_CUDA_CHECK(cudaGetDevice(&prev));
  HPS_CUDA_CHECK(cudaSetDevice(device));
  Ctx* c = new Ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  bool ok = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithPriority(&c->ahead, cudaStreamNonBlocking, hi) == cudaSuccess;
  ok = ok && cudaStreamCreateWithPriority(&c->ahead_side, cudaStreamNonBlocking, hi) == cudaSuccess;
  for (int i = 0; i < 64 && ok; ++i) ok = cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming) == cudaSuccess;
  cudaSetDevice(prev);
  if (!ok) {
    set_error("hps_ctx_create: stream/event creation failed on device %d: %s", device,
              cudaGetErrorString(cudaGetLastError()));
    hps_ctx_destroy(reinterpret_cast<hps_ctx_t>(c));
    return HPS_ERR_CUDA;
  }
  c->streams_ok = true;
  *out = reinterpret_cast<hps_ctx_t>(c);
  return HPS_OK;
}

extern "C" int hps_ctx_destroy(hps_ctx_t handle) {
  using namespace hps;
  Ctx* c = reinterpret_cast<Ctx*>(handle);
  if (!c) return HPS_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();  // nothing of this context may still run
  for (auto s : {c->side, c->ahead, c->ahead_side})
    if (s) cudaStreamDestroy(s);
  for (auto e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& row : c->probe)
    for (auto e : row)
      if (e) cudaEventDestroy(e);
  for (auto p : c->splitk)
    if (p) cudaFree(p);
  for (auto p : c->emu_buf)
    if (p) cudaFree(p);
  for (auto p : c->gather_buf)
    if (p) cudaFree(p);
  if (c->emu && c->emu_free) c->emu_free(c->emu);
  for (auto p : c->retired) cudaFree(p);
  cudaGetLastError();
  cudaSetDevice(prev);
  delete c;
  return HPS_OK;
}

extern "C" int hps_ctx_set_option(hps_ctx_t handle, int option, long long value) {
  hps::Ctx* c = reinterpret_cast<hps::Ctx*>(handle);
  if (!c || option < 0 || option >= HPS_OPT_COUNT) {
    hps::set_error("hps_ctx_set_option: bad context or option %d", option);
    return HPS_ERR_ARG;
  }
  std::lock_guard<std::mutex> lk(c->mu);
  c->opt[option] = value;
  return HPS_OK;
}

extern "C" long long hps_ctx_get_option(hps_ctx_t handle, int option) {
  hps::Ctx* c = reinterpret_cast<hps::Ctx*>(handle);
  if (!c || option < 0 || option >= HPS_OPT_COUNT) return -1;
  return c->opt[option];
}

extern "C" int hps_ctx_device(hps_ctx_t handle) {
  hps::Ctx* c = reinterpret_cast<hps::Ctx*>(handle);
  return c ? c->device : -1;
}
