// Host launcher for the DMMA GEMM (tile selection) + the C-ABI test hook.
#include <algorithm>
#include <cstdlib>

#include "ctx.cuh"
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

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC = true>
static int launch_cfg(const GemmParams& p, Ctx& cx, cudaStream_t stream) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = dgemm_dmma_kernel<BM, BN, BK, WM, WN, STAGES, VEC>;
  const int as = ensure_smem_attr((const void*)kern, cx.device, (int)Cfg::kSmem);
  if (as != HPS_OK) return as;
  // split-K when the tile grid cannot fill the GPU and K is long (top levels, batched solve)
  const long long tiles = (long long)((p.N + BN - 1) / BN) * ((p.M + BM - 1) / BM) * p.batch;
  int split = 1;
  const long long sms = cx.sms;
  if (cx.opt[HPS_OPT_SPLITK] && tiles < sms && p.K >= 8 * BK) {
    split = (int)std::min<long long>((2 * sms + tiles - 1) / tiles, p.K / (4 * BK));
    split = std::max(1, std::min(split, 16));
    while (split > 1 && (long long)split * p.batch > 65535) --split;
  }
  GemmParams q = p;
  if (split > 1) {
    q.split = split;
    q.partial = cx.splitk_scratch((size_t)split * p.batch * (size_t)p.M * p.N, stream);
    if (!q.partial) q.split = 1;
  }
  dim3 grid((p.N + BN - 1) / BN, (p.M + BM - 1) / BM, p.batch * q.split);
  kern<<<grid, Cfg::kThreads, Cfg::kSmem, stream>>>(q);
  HPS_LAUNCH_CHECK();
  if (q.split > 1) {
    const long long total = (long long)p.M * p.N * p.batch;
    const int blocks = (int)std::min<long long>((total + 255) / 256, sms * 8);
    k_splitk_reduce<<<blocks, 256, 0, stream>>>(q);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

// 64 x 64 paired-fragment kernel (gemm.cuh): MINB CTAs per SM, split-K to fill 148 * MINB slots.
template <int BK, int STAGES, int MINB>
static int launch_cfg64(const GemmParams& p, Ctx& cx, cudaStream_t stream) {
  using Cfg = Gemm64Cfg<BK, STAGES>;
  auto kern = dgemm64_kernel<BK, STAGES, MINB>;
  const int as = ensure_smem_attr((const void*)kern, cx.device, (int)Cfg::kSmem);
  if (as != HPS_OK) return as;
  const long long tiles = (long long)((p.N + 63) / 64) * ((p.M + 63) / 64) * p.batch;
  int split = 1;
  const long long sms = cx.sms;
  const long long slots = sms * MINB;
  if (cx.opt[HPS_OPT_SPLITK] && 2 * tiles < slots && p.K >= 8 * BK) {  // about one wave (measured best, r01)
    split = (int)std::min<long long>((slots + tiles - 1) / tiles, p.K / (4 * BK));
    split = std::max(1, std::min(split, 16));
    while (split > 1 && (long long)split * p.batch > 65535) --split;
  } else if (cx.opt[HPS_OPT_SPLITK] && p.Bidx && tiles < 4 * slots && p.K >= 16 * BK) {
    // the batched solve's top depths (one to a few boxes, long K): a tile grid just over a wave
    // (e.g. 512 tiles on 444 slots) leaves most SMs idle in its last wave; pick the split with the
    // best wave fill, 3% per extra split for the partial sums' pass
    double best = 0.0;
    for (int s = 1; s <= 8 && (long long)s * 4 * BK <= p.K && (long long)s * p.batch <= 65535; ++s) {
      const long long t = tiles * s, waves = (t + slots - 1) / slots;
      const double eff = (double)t / (double)(waves * slots) - 0.03 * (s - 1);
      if (eff > best + 1e-9) {
        best = eff;
        split = s;
      }
    }
  }
  GemmParams q = p;
  if (split > 1) {
    q.split = split;
    q.partial = cx.splitk_scratch((size_t)split * p.batch * (size_t)p.M * p.N, stream);
    if (!q.partial) q.split = 1;
  }
  q.group_m = (int)cx.opt[HPS_OPT_GEMM_GROUP_M];
  dim3 grid((p.N + 63) / 64, (p.M + 63) / 64, p.batch * q.split);
  kern<<<grid, 128, Cfg::kSmem, stream>>>(q);
  HPS_LAUNCH_CHECK();
  if (q.split > 1) {
    const long long total = (long long)p.M * p.N * p.batch;
    const int blocks = (int)std::min<long long>((total + 255) / 256, sms * 8);
    k_splitk_reduce<<<blocks, 256, 0, stream>>>(q);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

int emu_gemm(const GemmParams& p, Ctx& cx, cudaStream_t st);  // emu.cu

int dgemm_launch(const GemmParams& p, Ctx& cx, cudaStream_t stream) {
  if (p.M <= 0 || p.N <= 0 || p.batch <= 0) return HPS_OK;
  if (p.K <= 0) {
    set_error("dgemm: K=%d", p.K);
    return HPS_ERR_ARG;
  }
  if (p.emu_ok && (cx.opt[HPS_OPT_EMU_MODULI] > 0 || cx.opt[HPS_OPT_EMU_SLICES] > 0)) {
    const int r = emu_gemm(p, cx, stream);
    if (r != 1) return r;  // 1: not eligible here, run on DMMA
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
      int st = dgemm_launch(q, cx, stream);
      if (st != HPS_OK) return st;
    }
    return HPS_OK;
  }
  if (!vec) return launch_cfg<64, 64, 16, 2, 2, 3, false>(p, cx, stream);  // any shape (e.g. q = 21)
  // Measured best per shape class (round 1, tools/gemm_shapes.py):
  // * M <= 32, N >= 64 (the merge S = X^-1 R GEMMs of the bottom depths, n3 = 16 or 32): 16/32-row tiles;
  // * 96 x 96 (the leaf-pair merges' T GEMM): 48 x 48 tiles cover it exactly (64 x 64 tiles: 56%);
  // * K <= 32 (bottom merge depths): the 64 x 64 paired-fragment kernel with 2 stages, 4 CTAs/SM;
  // * otherwise the 64 x 64 paired-fragment kernel (BK 16, 3 stages, 3 CTAs/SM; the shape cuBLAS
  //   picks on sm_100), except narrow row-gather GEMMs (the batched solve, N <= 64), which are
  //   latency-bound on the index-then-row loads and run 7-12 us per depth faster on LDS.64 tiles
  //   as tall as the problem (M <= 32) or 64 x 64 (at b = 256 the paired kernel wins: 97.8 vs 104.3 ms).
  if (!p.Bidx && p.M <= 16 && p.N >= 64) return launch_cfg<16, 64, 16, 1, 2, 3>(p, cx, stream);
  if (!p.Bidx && p.M <= 32 && p.N >= 64) return launch_cfg<32, 64, 16, 1, 2, 3>(p, cx, stream);
  if (!p.Bidx && p.M == 96 && p.N == 96) return launch_cfg<48, 48, 16, 2, 2, 2>(p, cx, stream);
  // row-gather GEMMs (the batched solve) with few rows (the bottom depths, n3 <= 32): 16 / 32-row
  // tiles, as tall as the problem, instead of 64-row tiles that are mostly padding
  if (p.Bidx && p.M <= 16) return launch_cfg<16, 64, 16, 1, 2, 3>(p, cx, stream);
  if (p.Bidx && p.M <= 32) return launch_cfg<32, 64, 16, 1, 2, 3>(p, cx, stream);
  const bool narrow_gather = p.Bidx && p.N <= 64;
  if (!narrow_gather && p.K <= 32) return launch_cfg64<16, 2, 4>(p, cx, stream);
  if (!narrow_gather) return launch_cfg64<16, 3, 3>(p, cx, stream);
  if (p.M <= 16) return launch_cfg<16, 64, 16, 1, 2, 3>(p, cx, stream);
  if (p.M <= 32) return launch_cfg<32, 64, 16, 1, 2, 3>(p, cx, stream);
  return launch_cfg<64, 64, 16, 2, 2, 3>(p, cx, stream);
}

}  // namespace hps

extern "C" int hps_dgemm_batched(hps_ctx_t ctx, int M, int N, int K, int batch, double alpha, const double* A, long long lda,
                                 long long strideA, const double* B, long long ldb, long long strideB,
                                 const int* Bidx, long long strideBidx, double beta, double* C, long long ldc,
                                 long long strideC, void* stream) {
  hps::GemmParams p{M, N, K, batch, A, lda, strideA, B, ldb, strideB, Bidx, strideBidx, C, ldc, strideC,
                    alpha, beta, nullptr};
  p.emu_ok = true;
  HPS_CTX(cx, ctx);
  return hps::dgemm_launch(p, *cx, static_cast<cudaStream_t>(stream));
}
