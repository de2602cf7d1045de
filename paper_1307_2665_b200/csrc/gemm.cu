// Host launcher for the DMMA GEMM (tile selection) + the C-ABI test hook.
#include <algorithm>
#include <cstdlib>

#include "gemm.cuh"

namespace hps {

__global__ void k_splitk_reduce(GemmParams p) {
  const long long mn = (long long)p.M * p.N;
  const long long total = mn * p.batch;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long b = e / mn, rc = e - b * mn;
    const int r = (int)(rc / p.N), c = (int)(rc - (long long)r * p.N);
    const double* P = p.partial + b * p.split * mn + rc;
    double s = 0.0;
    for (int k = 0; k < p.split; ++k) s += P[k * mn];
    double* dst = p.C + b * p.strideC + (long long)r * p.ldc + c;
    double v = p.alpha * s;
    if (p.beta != 0.0) v += p.beta * *dst;
    if (p.blk_j1a) v += blk_value(p, (int)b, r, c);
    if (p.nonfinite && !isfinite(v)) atomicMax(p.nonfinite, (int)b + p.batch_offset);
    *dst = v;
  }
}

// Split-K scratch: growing device buffers, one per stream role (the caller's stream, the library's
// side stream where the interface inverse runs independent GEMMs, and the look-ahead pair), in
// HPS_SCRATCH_SLOTS independent sets. hps_set_scratch_slot(s) selects the set for the calling host
// thread's later enqueues, so two builds in flight on two streams (solver.Pipeline(streams=2))
// never share one. Builds repeat the same shapes, so they settle after the first build. An
// outgrown buffer is never freed: a captured CUDA graph (solver.BuildGraph) may still reference it.
int stream_role(cudaStream_t st);  // merge.cu: 0 caller, 1 fork side, 2/3 look-ahead inverse pair
constexpr int HPS_SCRATCH_SLOTS = 4;
static double* g_splitk[HPS_SCRATCH_SLOTS][4] = {};
static size_t g_splitk_n[HPS_SCRATCH_SLOTS][4] = {};
static thread_local int t_scratch_slot = 0;
static double* splitk_scratch(size_t n, cudaStream_t st) {
  const int role = stream_role(st), set = t_scratch_slot;
  if (n > g_splitk_n[set][role]) {
    // no allocation inside a stream capture (it would invalidate the capture): the caller then
    // runs without split-K. BuildGraph warms up first, so captures normally find it allocated.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
    double* fresh = nullptr;
    if (cudaMalloc(&fresh, n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    g_splitk[set][role] = fresh;
    g_splitk_n[set][role] = n;
  }
  return g_splitk[set][role];
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC = true>
static int launch_cfg(const GemmParams& p, cudaStream_t stream) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = dgemm_dmma_kernel<BM, BN, BK, WM, WN, STAGES, VEC>;
  static bool attr_set = false;  // per-instantiation
  if (!attr_set) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    attr_set = true;
  }
  // split-K when the tile grid cannot fill the GPU and K is long (top levels, batched solve)
  const long long tiles = (long long)((p.N + BN - 1) / BN) * ((p.M + BM - 1) / BM) * p.batch;
  int split = 1;
  static const int allow = getenv("HPS_SPLITK") ? atoi(getenv("HPS_SPLITK")) : 1;
  if (allow && tiles < 148 && p.K >= 8 * BK) {
    split = (int)std::min<long long>((2 * 148 + tiles - 1) / tiles, p.K / (4 * BK));
    split = std::max(1, std::min(split, 16));
    while (split > 1 && (long long)split * p.batch > 65535) --split;
  }
  GemmParams q = p;
  if (split > 1) {
    q.split = split;
    q.partial = splitk_scratch((size_t)split * p.batch * (size_t)p.M * p.N, stream);
    if (!q.partial) q.split = 1;
  }
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.batch * q.split);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, stream>>>(q);
  HPS_LAUNCH_CHECK();
  if (q.split > 1) {
    const long long total = (long long)p.M * p.N * p.batch;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
    k_splitk_reduce<<<blocks, 256, 0, stream>>>(q);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

// 64 x 64 paired-fragment kernel (gemm.cuh): MINB CTAs per SM, split-K to fill 148 * MINB slots.
template <int BK, int STAGES, int MINB>
static int launch_cfg64(const GemmParams& p, cudaStream_t stream) {
  using Cfg = Gemm64Cfg<BK, STAGES>;
  auto kern = dgemm64_kernel<BK, STAGES, MINB>;
  static bool attr_set = false;
  if (!attr_set) {
    HPS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem));
    attr_set = true;
  }
  const long long tiles = (long long)((p.N + 63) / 64) * ((p.M + 63) / 64) * p.batch;
  int split = 1;
  static const int allow = getenv("HPS_SPLITK") ? atoi(getenv("HPS_SPLITK")) : 1;
  const long long slots = 148LL * MINB;
  static const int mode = getenv("HPS_SPLIT_MODE") ? atoi(getenv("HPS_SPLIT_MODE")) : 1;  // 1: measured better (r01)
  if (mode == 0 && allow && tiles < slots && p.K >= 4 * BK) {
    split = (int)std::min<long long>((2 * slots + tiles - 1) / tiles, p.K / (2 * BK));
    split = std::max(1, std::min(split, 16));
    while (split > 1 && (long long)split * p.batch > 65535) --split;
  }
  if (mode == 1 && allow && 2 * tiles < slots && p.K >= 8 * BK) {  // about one wave
    split = (int)std::min<long long>((slots + tiles - 1) / tiles, p.K / (4 * BK));
    split = std::max(1, std::min(split, 16));
    while (split > 1 && (long long)split * p.batch > 65535) --split;
  }
  GemmParams q = p;
  if (split > 1) {
    q.split = split;
    q.partial = splitk_scratch((size_t)split * p.batch * (size_t)p.M * p.N, stream);
    if (!q.partial) q.split = 1;
  }
  static const int group_m = getenv("HPS_GEMM_GROUP_M") ? atoi(getenv("HPS_GEMM_GROUP_M")) : 16;
  q.group_m = group_m;
  dim3 grid((p.N + 63) / 64, (p.M + 63) / 64, p.batch * q.split);
  kern<<<grid, 128, Cfg::kSmem, stream>>>(q);
  HPS_LAUNCH_CHECK();
  if (q.split > 1) {
    const long long total = (long long)p.M * p.N * p.batch;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
    k_splitk_reduce<<<blocks, 256, 0, stream>>>(q);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

int dgemm_launch(const GemmParams& p, cudaStream_t stream) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return HPS_OK;
  if (p.K <= 0) {
    set_error("dgemm: K=%d", p.K);
    return HPS_ERR_ARG;
  }
  const bool vec = !(p.K % 16 != 0 || p.N % 2 != 0 || (p.ldb % 2) || (p.ldc % 2) || (p.lda % 2) ||
                     (p.strideA % 2) || (p.strideB % 2) || (p.strideC % 2) ||
                     (reinterpret_cast<uintptr_t>(p.A) & 15) || (reinterpret_cast<uintptr_t>(p.B) & 15) ||
                     (reinterpret_cast<uintptr_t>(p.C) & 15));
  if (p.batch > 65535) {  // gridDim.z limit: launch in batch chunks
    for (int b0 = 0; b0 < p.batch; b0 += 65535) {
      GemmParams q = p;
      q.batch = std::min(65535, p.batch - b0);
      q.A += (long long)b0 * p.strideA;
      q.B += (long long)b0 * p.strideB;
      q.C += (long long)b0 * p.strideC;
      if (q.Bidx) q.Bidx += (long long)b0 * p.strideBidx;
      q.batch_offset = p.batch_offset + b0;
      int st = dgemm_launch(q, stream);
      if (st != HPS_OK) return st;
    }
    return HPS_OK;
  }
  if (!vec) return launch_cfg<64, 64, 16, 2, 2, 3, false>(p, stream);  // any shape (e.g. q = 21)
  // 64 x 64 paired-fragment tiles, BK 16, 3 stages, 3 CTAs per SM: measured best of
  // {BK 16/32} x {2,3,4 stages} x {2,3,4 CTAs/SM} on the merge shapes (tools/gemm_variants.sh)
  // Narrow row-gather GEMMs (the batched solve with b <= 64: one 64-column tile, small M,
  // latency-bound on the index-then-row loads) measured 7-12 us per depth faster on the LDS.64
  // 64 x 64 kernel below; at b = 256 the paired kernel wins (cfg5 solve 97.8 vs 104.3 ms).
  static const int v64 = getenv("HPS_GEMM64") ? atoi(getenv("HPS_GEMM64")) : 1;
  // K <= 32 (the bottom merge depths: K = n3 = 16 or 32, one or two k tiles): two stages are enough
  // and the smaller footprint fits 4 CTAs per SM, more tiles in flight for these memory-bound shapes
  static const int smallk = getenv("HPS_SMALLK") ? atoi(getenv("HPS_SMALLK")) : 1;
  // M <= 32 (the merge S = X^-1 R GEMMs of the bottom depths, n3 = 16 or 32): row tiles of 16/32
  static const int smallm_s = getenv("HPS_SMALLM_S") ? atoi(getenv("HPS_SMALLM_S")) : 1;
  if (smallm_s && !p.Bidx && p.M <= 16 && p.N >= 64) return launch_cfg<16, 64, 16, 1, 2, 3>(p, stream);
  if (smallm_s && !p.Bidx && p.M <= 32 && p.N >= 64) return launch_cfg<32, 64, 16, 1, 2, 3>(p, stream);
  // 96 x 96 (the leaf-pair merges' T GEMM): 48 x 48 tiles cover it exactly (64 x 64 tiles: 56%)
  static const int t96 = getenv("HPS_T96") ? atoi(getenv("HPS_T96")) : 1;
  if (t96 && !p.Bidx && p.M == 96 && p.N == 96) return launch_cfg<48, 48, 16, 2, 2, 2>(p, stream);
  if (v64 && !(p.Bidx && p.N <= 64) && smallk && p.K <= 32) return launch_cfg64<16, 2, 4>(p, stream);
  if (v64 && !(p.Bidx && p.N <= 64)) return launch_cfg64<16, 3, 3>(p, stream);
  // narrow row-gather GEMMs with few rows (the batched solve's bottom depths: M = n3 = 16 or 32):
  // tiles as tall as the problem instead of 64-row tiles that are 50-75% padding
  static const int smallm = getenv("HPS_SMALLM") ? atoi(getenv("HPS_SMALLM")) : 1;
  if (smallm && p.Bidx && p.N <= 64 && p.M <= 16) return launch_cfg<16, 64, 16, 1, 2, 3>(p, stream);
  if (smallm && p.Bidx && p.N <= 64 && p.M <= 32) return launch_cfg<32, 64, 16, 1, 2, 3>(p, stream);
  double tiles128 = double((p.M + 127) / 128) * double((p.N + 127) / 128) * p.batch;
  // HPS_GEMM64=0: the previous tiling (128 x 128 x 16, 8 warps of 64 x 32, one CTA per SM)
  if (p.M >= 128 && p.N >= 128 && tiles128 >= 148.0) return launch_cfg<128, 128, 16, 2, 4, 4>(p, stream);
  return launch_cfg<64, 64, 16, 2, 2, 3>(p, stream);
}

}  // namespace hps

extern "C" int hps_set_scratch_slot(int slot) {
  if (slot < 0 || slot >= hps::HPS_SCRATCH_SLOTS) {
    hps::set_error("hps_set_scratch_slot: slot %d not in [0, %d)", slot, hps::HPS_SCRATCH_SLOTS);
    return HPS_ERR_ARG;
  }
  hps::t_scratch_slot = slot;
  return HPS_OK;
}

extern "C" int hps_dgemm_batched(int M, int N, int K, int batch, double alpha, const double* A, long long lda,
                                 long long strideA, const double* B, long long ldb, long long strideB,
                                 const int* Bidx, long long strideBidx, double beta, double* C, long long ldc,
                                 long long strideC, void* stream) {
  hps::GemmParams p{M, N, K, batch, A, lda, strideA, B, ldb, strideB, Bidx, strideBidx, C, ldc, strideC,
                    alpha, beta, nullptr};
  return hps::dgemm_launch(p, static_cast<cudaStream_t>(stream));
}
