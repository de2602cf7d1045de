// FP64 GEMM emulated on the int8 tensor cores (Ozaki scheme, fixed-point slices), for the large merge
// GEMMs (S = X^-1 R, T = blk + C S: merge.py:108, 118).
//
// B200 has ~37 TF/s of FP64 (DMMA) but ~2.5 POPS of dense int8 through the 5th-gen tensor cores (the
// measured cuBLASLt IMMA rate on 32768 x 32768 x 8192, tools/int8_probe.py). With every row of A and
// column of B scaled by a power of two into (-1/2, 1/2) and cut into s balanced base-2^7 digits (int8
// in [-64, 64]),
//
//   A = diag(2^e) sum_i 2^(-7(i+1)) A_i,   B = sum_j 2^(-7(j+1)) B_j diag(2^f),
//   A B = diag(2^e) [ sum_{t < s} 2^(-7(t+2)) C_t ] diag(2^f) + (dropped t >= s terms),
//   C_t = sum_{i+j=t} A_i B_j  =  [A_0 | ... | A_t] [B_t; ...; B_0]   (one int8 GEMM, K' = (t+1) K),
//
// every C_t is EXACT in int32 (|C_t| <= (t+1) K 64^2 < 2^31 for K <= 8192 s^-1 2^13... checked below),
// and the only rounding is the digit truncation (2^-(7s+1) of the row / column maximum) and s fp64
// additions. s = 8 (56 bits, the default) keeps the normwise error at or below a DGEMM's
// (~K 2^-53 |A||B|). The products run on cuBLASLt's int8 GEMM (a plain library GEMM); the scaling,
// digit splitting, fp64 accumulation and the merge epilogue (the block-diagonal addend, the
// non-finite flag) are the kernels here. Used by dgemm_launch when the context enables it
// (HPS_OPT_EMU_SLICES) and the GEMM is large and plain (beta = 0, no row gather).
#include <cublasLt.h>

#include <algorithm>
#include <map>
#include <tuple>

#include "common.cuh"
#include "ctx.cuh"
#include "gemm.cuh"

namespace hps {

// e[b][i] with |A_i| < 2^(e - 1): x = a 2^-e in (-1/2, 1/2). One warp per row.
__global__ void k_emu_row_exp(const double* __restrict__ A, long long lda, long long sA, int M, int K, int* __restrict__ e) {
  const int b = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= M) return;
  const double* Ar = A + (long long)b * sA + (long long)r * lda;
  double m = 0.0;
  for (int k = lane; k < K; k += 32) m = fmax(m, fabs(Ar[k]));
  m = warp_max(m);
  if (lane == 0) {
    int ex = 0;
    if (m > 0.0) frexp(m, &ex);  // m = f 2^ex, f in [1/2, 1)
    e[(long long)b * M + r] = ex + 1;
  }
}

// f[b][j] with |B[:, j]| < 2^(f - 1). 32 columns x 8 row slices per CTA (coalesced row reads).
__global__ void __launch_bounds__(256) k_emu_col_exp(const double* __restrict__ B, long long ldb, long long sB, int K, int N,
                                                    int* __restrict__ f) {
  __shared__ double red[8][33];
  const int b = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  const double* Bb = B + (long long)b * sB + j;
  double m = 0.0;
  if (j < N)
    for (int k = ty; k < K; k += 8) m = fmax(m, fabs(Bb[(long long)k * ldb]));
  red[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && j < N) {
#pragma unroll
    for (int r = 1; r < 8; ++r) m = fmax(m, red[r][tx]);
    int ex = 0;
    if (m > 0.0) frexp(m, &ex);
    f[(long long)b * N + j] = ex + 1;
  }
}

// 2^ex as a double (normal range)
__device__ __forceinline__ double pow2(int ex) { return __longlong_as_double((long long)(1023 + ex) << 52); }

// digits of the rows of A: out[b][i][t K + k], t = 0 (most significant) .. s - 1; 4 k per thread.
__global__ void k_emu_split_rows(const double* __restrict__ A, long long lda, long long sA, int M, int K,
                                 const int* __restrict__ e, int s, signed char* __restrict__ out) {
  const int b = blockIdx.z, r = blockIdx.y;
  const int k4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k4 >= K) return;  // K % 16 == 0
  const double sc = pow2(-e[(long long)b * M + r]);
  const double* Ar = A + (long long)b * sA + (long long)r * lda + k4;
  double x[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) x[u] = Ar[u] * sc;  // exact (power of two)
  char4* o = reinterpret_cast<char4*>(out + ((long long)b * M + r) * (long long)s * K + k4);
  for (int t = 0; t < s; ++t) {
    signed char d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double y = x[u] * 128.0;  // exact
      const double q = rint(y);       // |q| <= 64
      x[u] = y - q;                   // exact, in [-1/2, 1/2]
      d[u] = (signed char)q;
    }
    o[(long long)t * (K / 4)] = make_char4(d[0], d[1], d[2], d[3]);
  }
}

// digits of the columns of B, transposed and in reversed slice order:
// out[b][j][(s - 1 - t) K + k] = digit t of B[k][j] 2^-f_j. Tile: 32 k x 64 j through shared memory.
__global__ void __launch_bounds__(256) k_emu_split_cols(const double* __restrict__ B, long long ldb, long long sB, int K,
                                                       int N, const int* __restrict__ f, int s,
                                                       signed char* __restrict__ out) {
  __shared__ signed char sd[8][64][33];
  const int b = blockIdx.z;
  const int k0 = blockIdx.y * 32, j0 = blockIdx.x * 64;
  const double* Bb = B + (long long)b * sB;
  for (int idx = threadIdx.x; idx < 32 * 64; idx += blockDim.x) {
    const int kk = idx / 64, jj = idx % 64;
    const int k = k0 + kk, j = j0 + jj;
    double x = (k < K && j < N) ? Bb[(long long)k * ldb + j] * pow2(-f[(long long)b * N + j]) : 0.0;
    for (int t = 0; t < s; ++t) {
      const double y = x * 128.0;
      const double d = rint(y);
      x = y - d;
      sd[t][jj][kk] = (signed char)d;
    }
  }
  __syncthreads();
  signed char* ob = out + (long long)b * N * s * K;
  for (int idx = threadIdx.x; idx < s * 64 * 8; idx += blockDim.x) {  // 4 bytes per store
    const int k4 = (idx % 8) * 4, rest = idx / 8, jj = rest % 64, t = rest / 64;
    const int k = k0 + k4, j = j0 + jj;
    if (k < K && j < N)
      *reinterpret_cast<char4*>(ob + (long long)j * s * K + (long long)(s - 1 - t) * K + k) =
          make_char4(sd[t][jj][k4], sd[t][jj][k4 + 1], sd[t][jj][k4 + 2], sd[t][jj][k4 + 3]);
  }
}

// acc (the output matrix) = (first ? 0 : acc) + sum_g C_(t0 - g) 2^-(7(t0 - g + 2)), g < ng (the
// smallest terms first); the last pass (down to t = 0) also applies the row / column scales, alpha,
// the merge's block-diagonal addend and the non-finite flag. Rows on blockIdx.y (grid-stride), 4
// columns per thread (int4 / 2 x double2 accesses; N % 4 == 0). Ct holds ng int32 M x N buffers.
constexpr int EMU_GROUP = 4;  // diagonals accumulated per pass (int32 buffers alive at once)
__global__ void __launch_bounds__(256) k_emu_accum(const int* __restrict__ Ct, long long sCt, int M, int N,
                                                  GemmParams p, int t0, int ng, int first, int last,
                                                  const int* __restrict__ e, const int* __restrict__ f) {
  const int b = blockIdx.z;
  const int c4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  bool bad = false;
  if (c4 < N) {
    for (int r = blockIdx.y; r < M; r += gridDim.y) {
      double* dst = p.C + (long long)b * p.strideC + (long long)r * p.ldc + c4;
      double v[4] = {0.0, 0.0, 0.0, 0.0};
      if (!first) {
        const double2 o0 = *reinterpret_cast<const double2*>(dst), o1 = *reinterpret_cast<const double2*>(dst + 2);
        v[0] = o0.x;
        v[1] = o0.y;
        v[2] = o1.x;
        v[3] = o1.y;
      }
      for (int g = 0; g < ng; ++g) {
        const double sc = pow2(-7 * (t0 - g + 2));
        const int4 ci = *reinterpret_cast<const int4*>(Ct + g * sCt + ((long long)b * M + r) * N + c4);
        v[0] = fma((double)ci.x, sc, v[0]);  // exact product (int32 x power of two)
        v[1] = fma((double)ci.y, sc, v[1]);
        v[2] = fma((double)ci.z, sc, v[2]);
        v[3] = fma((double)ci.w, sc, v[3]);
      }
      if (last) {
        const int er = e[(long long)b * M + r];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int ex = er + f[(long long)b * N + c4 + u];
          double w = v[u] * pow2(ex / 2) * pow2(ex - ex / 2);  // exact; two factors keep each in range
          w *= p.alpha;
          if (p.blk_j1a) w += blk_value(p, b, r, c4 + u);
          bad |= !isfinite(w);
          v[u] = w;
        }
      }
      *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[1]);
      *reinterpret_cast<double2*>(dst + 2) = make_double2(v[2], v[3]);
    }
  }
  if (last && p.nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicMax(p.nonfinite, b + p.batch_offset);
}

struct EmuPlan {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  cublasLtMatmulAlgo_t algo;
  bool ok = false;
};

struct EmuState {
  cublasLtHandle_t lt = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 32u << 20;
  std::map<std::tuple<int, int, int, int, int>, EmuPlan> plans;  // (M, N, k', batch, s) -> plan
};

static EmuState* emu_state(Ctx& cx) {
  if (!cx.emu) {
    auto* s = new EmuState();
    if (cublasLtCreate(&s->lt) != CUBLAS_STATUS_SUCCESS || cudaMalloc(&s->ws, s->ws_bytes) != cudaSuccess) {
      cudaGetLastError();
      delete s;
      return nullptr;
    }
    cx.emu = s;
    cx.emu_free = [](void* p) {
      auto* s = static_cast<EmuState*>(p);
      for (auto& kv : s->plans) {
        EmuPlan& pl = kv.second;
        if (pl.a) cublasLtMatrixLayoutDestroy(pl.a);
        if (pl.b) cublasLtMatrixLayoutDestroy(pl.b);
        if (pl.c) cublasLtMatrixLayoutDestroy(pl.c);
        if (pl.op) cublasLtMatmulDescDestroy(pl.op);
      }
      if (s->ws) cudaFree(s->ws);
      if (s->lt) cublasLtDestroy(s->lt);
      delete s;
    };
  }
  return static_cast<EmuState*>(cx.emu);
}

// Plan of C_t (int32, M x N row-major) = Adig[:, 0:k'] (M x k', row stride sK) * Bdig^T window
// (N x k', row stride sK), batched. In cuBLASLt's column-major terms: C^T (N x M) = op_T(Bw) op_N(Aw).
static EmuPlan* emu_plan(EmuState* es, int M, int N, int kp, int sK, int batch) {
  auto key = std::make_tuple(M, N, kp, sK, batch);
  auto it = es->plans.find(key);
  if (it != es->plans.end()) return it->second.ok ? &it->second : nullptr;
  EmuPlan& pl = es->plans[key];
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  bool ok = cublasLtMatmulDescCreate(&pl.op, CUBLAS_COMPUTE_32I, CUDA_R_32I) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&pl.a, CUDA_R_8I, kp, N, sK) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&pl.b, CUDA_R_8I, kp, M, sK) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&pl.c, CUDA_R_32I, N, M, N) == CUBLAS_STATUS_SUCCESS;
  if (ok && batch > 1) {
    const long long sa = (long long)N * sK, sb = (long long)M * sK, sc = (long long)M * N;
    ok = cublasLtMatrixLayoutSetAttribute(pl.a, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof(batch)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.a, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof(sa)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.b, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof(batch)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.b, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sb, sizeof(sb)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.c, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof(batch)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.c, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof(sc)) == 0;
  }
  if (ok) {
    cublasLtMatmulPreference_t pref = nullptr;
    ok = cublasLtMatmulPreferenceCreate(&pref) == CUBLAS_STATUS_SUCCESS;
    ok = ok && cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &es->ws_bytes,
                                                    sizeof(es->ws_bytes)) == CUBLAS_STATUS_SUCCESS;
    cublasLtMatmulHeuristicResult_t res{};
    int n = 0;
    ok = ok && cublasLtMatmulAlgoGetHeuristic(es->lt, pl.op, pl.a, pl.b, pl.c, pl.c, pref, 1, &res, &n) ==
                   CUBLAS_STATUS_SUCCESS && n > 0;
    if (ok) pl.algo = res.algo;
    if (pref) cublasLtMatmulPreferenceDestroy(pref);
  }
  pl.ok = ok;
  return ok ? &pl : nullptr;
}

// Returns HPS_OK when the GEMM ran emulated, 1 when the caller should run it on DMMA instead (not
// eligible, no scratch inside a graph capture, or no cuBLASLt plan), an error code on failure.
int emu_gemm(const GemmParams& p, Ctx& cx, cudaStream_t st) {
  const int s = (int)cx.opt[HPS_OPT_EMU_SLICES];
  if (s <= 0 || p.Bidx || p.beta != 0.0 || p.split > 1) return 1;
  const double work = (double)p.M * p.N * p.K;
  // it pays where a GEMM is FP64-bound: K >= HPS_OPT_EMU_MIN_K (each output element costs 2 K DMMA flops
  // against ~56 bytes of accumulation traffic plus 72 K int8 operations)
  if (work * p.batch < (double)cx.opt[HPS_OPT_EMU_MIN_WORK] || p.K < cx.opt[HPS_OPT_EMU_MIN_K] || p.M % 4 ||
      p.N % 4 || p.K % 16)
    return 1;
  if ((reinterpret_cast<uintptr_t>(p.C) & 15) || (p.ldc % 2) || (p.strideC % 2)) return 1;
  if ((long long)(s) * p.K * 64 * 64 >= (1LL << 31)) return 1;  // C_t must stay exact in int32
  EmuState* es = emu_state(cx);
  if (!es) return 1;
  const long long sK = (long long)s * p.K;
  const size_t a_bytes = (size_t)p.batch * p.M * sK, b_bytes = (size_t)p.batch * p.N * sK;
  const size_t c1 = (size_t)p.batch * p.M * p.N, c_bytes = EMU_GROUP * c1 * sizeof(int);
  const size_t e_bytes = (size_t)p.batch * (p.M + p.N) * sizeof(int);
  const size_t need = (a_bytes + b_bytes + c_bytes + e_bytes + 4 * 256) / sizeof(double) + 1;
  double* scratch = cx.emu_scratch(need, st);
  if (!scratch) return 1;
  char* base = reinterpret_cast<char*>(scratch);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  signed char* Ad = reinterpret_cast<signed char*>(base);
  signed char* Bd = reinterpret_cast<signed char*>(base + align(a_bytes));
  int* Ct = reinterpret_cast<int*>(base + align(a_bytes) + align(b_bytes));
  int* e = reinterpret_cast<int*>(reinterpret_cast<char*>(Ct) + align(c_bytes));
  int* f = e + (size_t)p.batch * p.M;
  // plans for every diagonal first (host only), so nothing is enqueued when one is missing
  EmuPlan* plans[16];
  for (int t = 0; t < s; ++t)
    if (!(plans[t] = emu_plan(es, p.M, p.N, (t + 1) * p.K, (int)sK, p.batch))) return 1;
  k_emu_row_exp<<<dim3((p.M + 7) / 8, p.batch), 256, 0, st>>>(p.A, p.lda, p.strideA, p.M, p.K, e);
  HPS_LAUNCH_CHECK();
  k_emu_col_exp<<<dim3((p.N + 31) / 32, p.batch), 256, 0, st>>>(p.B, p.ldb, p.strideB, p.K, p.N, f);
  HPS_LAUNCH_CHECK();
  k_emu_split_rows<<<dim3((p.K / 4 + 255) / 256, p.M, p.batch), 256, 0, st>>>(p.A, p.lda, p.strideA, p.M, p.K, e, s,
                                                                               Ad);
  HPS_LAUNCH_CHECK();
  k_emu_split_cols<<<dim3((p.N + 63) / 64, (p.K + 31) / 32, p.batch), 256, 0, st>>>(p.B, p.ldb, p.strideB, p.K, p.N, f,
                                                                                  s, Bd);
  HPS_LAUNCH_CHECK();
  const int one = 1, zero = 0;
  const dim3 agrid((p.N / 4 + 255) / 256, (unsigned)std::min<long long>(p.M, std::max<long long>(1, (long long)cx.sms * 16 / ((p.N / 4 + 255) / 256))), p.batch);
  for (int t0 = s - 1; t0 >= 0; t0 -= EMU_GROUP) {  // smallest terms first, EMU_GROUP diagonals per pass
    const int ng = std::min(EMU_GROUP, t0 + 1);
    for (int g = 0; g < ng; ++g) {
      const int t = t0 - g;
      const EmuPlan* pl = plans[t];
      const signed char* Aw = Bd + (long long)(s - 1 - t) * p.K;  // cuBLASLt "A": Bdig window (N x k')
      const signed char* Bw = Ad;                                  // cuBLASLt "B": Adig prefix (M x k')
      int* Cg = Ct + g * c1;
      if (cublasLtMatmul(es->lt, pl->op, &one, Aw, pl->a, Bw, pl->b, &zero, Cg, pl->c, Cg, pl->c, &pl->algo, es->ws,
                         es->ws_bytes, st) != CUBLAS_STATUS_SUCCESS) {
        set_error("emu_gemm: cublasLtMatmul failed (M=%d N=%d K=%d t=%d)", p.M, p.N, p.K, t);
        return HPS_ERR_CUDA;
      }
      count_launch();
    }
    k_emu_accum<<<agrid, 256, 0, st>>>(Ct, (long long)c1, p.M, p.N, p, t0, ng, t0 == s - 1, t0 - ng < 0, e, f);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

}  // namespace hps
