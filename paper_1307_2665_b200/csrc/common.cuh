// Shared device helpers for the HPS B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define HPS_OK 0
#define HPS_ERR_LEAF_RESONANCE 1
#define HPS_ERR_MERGE_RESONANCE 2
#define HPS_ERR_CUDA 3
#define HPS_ERR_NCCL 4
#define HPS_ERR_ARG 5

namespace hps {

void set_error(const char* fmt, ...);
void count_launch();  // every kernel launch of this library bumps a process-wide counter

#define HPS_CUDA_CHECK(expr)                                                              \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      ::hps::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return HPS_ERR_CUDA;                                                                \
    }                                                                                     \
  } while (0)

#define HPS_LAUNCH_CHECK()            \
  do {                                \
    ::hps::count_launch();            \
    HPS_CUDA_CHECK(cudaGetLastError()); \
  } while (0)

// DMMA: D(8x8) += A(8x4, row) * B(4x8, col), one f64 each for A/B per lane, two for C.
// Lane layout (g = lane>>2, t = lane&3): a = A[g][t], b = B[t][g], c = C[g][2t..2t+1].
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy global -> shared; zero-fills when !pred.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Explicit shared-memory store. Copy loops over a register array written with plain stores get
// turned into memcpy by LLVM, which forces the array into local memory; this keeps it in registers.
__device__ __forceinline__ void sts64(double* p, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(smem_u32(p)), "d"(v) : "memory");
}

// Reciprocal for pivots: MUFU approximation + 2 Newton steps (error ~1 ulp). About 60 cycles,
// against ~230 for the IEEE division sequence, which sits on every pivot step's critical path.
// Named barriers (ids 1..15; 0 is __syncthreads): sync waits, arrive only signals.
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r);
  r = fma(r, fma(-x, r, 1.0), r);
  return r;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide max of non-negative doubles (all threads get the result). `red` >= 32 doubles.
__device__ __forceinline__ double block_max(double v, double* red) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = lane < nw ? red[lane] : 0.0;
  r = warp_max(r);
  return r;
}

}  // namespace hps
