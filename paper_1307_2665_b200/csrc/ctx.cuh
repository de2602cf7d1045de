// Library context (hps_ctx_t in include/hps_b200.h): everything that used to be process-global.
// One context per (device, concurrent build): it owns the library's side streams (the recursive
// interface inverse's fork stream and the look-ahead pair), their event ring, the split-K scratch
// of each stream role and the tuning options. Two builds in flight on two streams use two
// contexts, so they never share scratch. Calls are thread-compatible per context.
#pragma once
#include <mutex>
#include <vector>

#include "common.cuh"
#include "hps_b200.h"



namespace hps {

struct Ctx {
  int device = 0;
  int sms = 148;
  // defaults: split-K on, group-M 16, fork on, 2 leaf CTAs/SM, no free SMs, no profiling, FP64 GEMM
  // emulation for K >= 512 and >= 2^32 multiply-adds: the modular scheme with 14 moduli
  // (FP64-equivalent accuracy; the 8-slice scheme when moduli = 0), <= 8 GB of products, int8
  // products on this library's tcgen05 kernel
  long long opt[HPS_OPT_COUNT] = {1, 16, 1, 2, 0, 0, 8, 1LL << 32, 512, 14, 8192, 0, 0, 0, 1};
  // side streams: 1 = fork (recursive inverse), 2/3 = look-ahead inverse pair (highest priority)
  cudaStream_t side = nullptr, ahead = nullptr, ahead_side = nullptr;
  bool streams_ok = false;
  cudaEvent_t ev[64] = {};
  int next_ev = 0;
  // split-K partial sums per stream role (0 caller's stream, 1 side, 2 ahead, 3 ahead_side). An
  // outgrown buffer is retired, not freed, until destroy: a captured CUDA graph may reference it.
  double* splitk[4] = {};
  size_t splitk_n[4] = {};
  std::vector<void*> retired;
  // look-ahead profiling (HPS_OPT_PROFILE_AHEAD)
  cudaEvent_t probe[32][4] = {};
  int probe_depth = -1;
  std::mutex mu;

  int role(cudaStream_t st) const {
    if (!streams_ok || st == nullptr) return 0;
    return st == side ? 1 : st == ahead ? 2 : st == ahead_side ? 3 : 0;
  }
  cudaEvent_t record_on(cudaStream_t st) {
    cudaEvent_t e = ev[next_ev];
    next_ev = (next_ev + 1) & 63;
    cudaEventRecord(e, st);
    return e;
  }
  double* splitk_scratch(size_t n, cudaStream_t st);
  // FP64-emulation state (emu.cu: cuBLASLt handle, plans) and its scratch per stream role
  void* emu = nullptr;
  void (*emu_free)(void*) = nullptr;
  double* emu_buf[4] = {};
  size_t emu_n[4] = {};
  double* emu_scratch(size_t n, cudaStream_t st);
  // gathered operands (the batched solve's boundary rows), per stream role
  double* gather_buf[4] = {};
  size_t gather_n[4] = {};
  double* gather_scratch(size_t n, cudaStream_t st);
};

// Context of a C-ABI call: a valid handle whose device is the caller's current device.
int check_ctx(const Ctx* c, const char* fn);
#define HPS_CTX(c, handle)                                 \
  ::hps::Ctx* c = reinterpret_cast<::hps::Ctx*>(handle);   \
  do {                                                     \
    const int _cs = ::hps::check_ctx(c, __func__);         \
    if (_cs != HPS_OK) return _cs;                         \
  } while (0)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device).
int ensure_smem_attr(const void* kernel, int device, int bytes);

}  // namespace hps
