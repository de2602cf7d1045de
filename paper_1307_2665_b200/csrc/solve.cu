// Downward pass (reference solver.py:303-316): for every parent at one depth,
//   u[I_i(box)] = S_box u[I_e(box)]
// for a batch of boundary vectors. u is node-major (N x ldu, RHS contiguous). I_e rows are
// gathered through the per-depth id table. I_i is contiguous (start0 + b*n3 ...), so the output
// is a plain strided store. Large batches go through the DMMA GEMM (B-row gather). For
// nrhs <= 8 a warp-per-row kernel streams S once (HBM-bound, like a batched GEMV).
#include "common.cuh"
#include "ctx.cuh"
#include "gemm.cuh"

namespace hps {

template <int NR>
__global__ void __launch_bounds__(256) k_solve_small(const double* __restrict__ S, const int* __restrict__ Ie,
                                                     long long ii_start0, int n3, int ne,
                                                     double* __restrict__ u, int ldu) {
  const int b = blockIdx.x;
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n3) return;
  const double* Sr = S + ((long long)b * n3 + r) * ne;
  const int* ie = Ie + (long long)b * ne;
  double acc[NR];
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = 0.0;
  // 8 columns per lane per step, every S value and index loaded before the dependent u gathers:
  // more loads in flight per warp on the HBM-bound S stream (the loop was load -> load chained)
  for (int c = lane; c < ne; c += 256) {  // predicated: short rows (ne < 256) take one pass
    double sv[8];
    int iv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool ok = c + 32 * k < ne;
      sv[k] = ok ? __ldcs(Sr + c + 32 * k) : 0.0;  // S is read once per solve: stream it past L2
      iv[k] = ok ? __ldg(ie + c + 32 * k) : -1;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (iv[k] >= 0) {
        const double* uc = u + (long long)iv[k] * ldu;
#pragma unroll
        for (int j = 0; j < NR; ++j) acc[j] = fma(sv[k], uc[j], acc[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NR; ++j) acc[j] = warp_sum(acc[j]);
  if (lane < NR) {
    double v = acc[0];
#pragma unroll
    for (int j = 1; j < NR; ++j)
      if (lane == j) v = acc[j];
    u[(ii_start0 + (long long)b * n3 + r) * ldu + lane] = v;
  }
}

// Bg[b][k][0..nrhs) = u[Ie[b][k]][0..nrhs): the boundary values of every box at one depth as a
// plain (ne x nrhs) operand, so the batched product can run as the FP64 emulation on the int8
// tensor cores (emu.cu), which takes no row gather. One warp per row.
__global__ void __launch_bounds__(256) k_solve_gather(const double* __restrict__ u, int ldu, const int* __restrict__ Ie,
                                                      int ne, int nrhs, long long rows, double* __restrict__ Bg) {
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const double* src = u + (long long)__ldg(Ie + row) * ldu;
  double* dst = Bg + row * nrhs;
  for (int j = lane; j < nrhs; j += 32) dst[j] = src[j];
}

}  // namespace hps

using namespace hps;

extern "C" int hps_solve_level(hps_ctx_t ctx, int nbatch, int n3, int ne, const double* S, const int* Ie, long long ii_start0,
                               double* u, int ldu, int nrhs, void* stream) {
  HPS_CTX(cx, ctx);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (nbatch <= 0 || nrhs <= 0) return HPS_OK;
  if (nrhs > ldu) {
    set_error("hps_solve_level: nrhs > ldu");
    return HPS_ERR_ARG;
  }
  if (nrhs <= 8) {
    dim3 grid(nbatch, (n3 + 7) / 8);
    switch (nrhs) {
#define HPS_SOLVE_CASE(R) \
  case R: k_solve_small<R><<<grid, 256, 0, st>>>(S, Ie, ii_start0, n3, ne, u, ldu); break;
      HPS_SOLVE_CASE(1) HPS_SOLVE_CASE(2) HPS_SOLVE_CASE(3) HPS_SOLVE_CASE(4)
      HPS_SOLVE_CASE(5) HPS_SOLVE_CASE(6) HPS_SOLVE_CASE(7) HPS_SOLVE_CASE(8)
#undef HPS_SOLVE_CASE
    }
    HPS_LAUNCH_CHECK();
    return HPS_OK;
  }
  // GEMM: C = u rows [start0 + b*n3, +n3), A = S[b] (n3 x ne), B = u[Ie[b]] (ne x nrhs)
  GemmParams p{n3, nrhs, ne, nbatch, S, ne, (long long)n3 * ne, u, ldu, 0, Ie, ne,
               u + ii_start0 * ldu, ldu, (long long)n3 * ldu, 1.0, 0.0, nullptr};
  // With HPS_OPT_EMU_SOLVE, large FP64-bound depths (K = ne >= the emulation threshold) gather B
  // once into a plain (ne x nrhs) operand per box and run through the FP64 emulation on the int8
  // tensor cores (which takes no row gather).
  const bool emu_on = cx->opt[HPS_OPT_EMU_SOLVE] && cx->opt[HPS_OPT_EMU_MODULI] > 0;
  const double work = (double)n3 * nrhs * ne * nbatch;
  const bool emu_here = emu_on && nrhs >= 64 && ne >= cx->opt[HPS_OPT_EMU_MIN_K] &&
                        work >= (double)cx->opt[HPS_OPT_EMU_MIN_WORK] && n3 % 4 == 0 && nrhs % 4 == 0 && ne % 16 == 0;
  if (emu_here) {
    const long long rows = (long long)nbatch * ne;
    double* Bg = cx->gather_scratch((size_t)rows * nrhs, st);
    if (Bg) {
      k_solve_gather<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(u, ldu, Ie, ne, nrhs, rows, Bg);
      HPS_LAUNCH_CHECK();
      p.B = Bg;
      p.ldb = nrhs;
      p.strideB = (long long)ne * nrhs;
      p.Bidx = nullptr;
      p.strideBidx = 0;
      p.emu_ok = true;
    }
  }
  return dgemm_launch(p, *cx, st);
}
