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
// (HPS_OPT_EMU_SLICES) and the GEMM is large and plain (beta = 0, no row gather; the modular scheme
// also takes beta != 0).
#include <cublasLt.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <type_traits>

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

// Shape / alignment test shared by both schemes: it pays where a GEMM is FP64-bound, K >=
// HPS_OPT_EMU_MIN_K (each output element costs 2 K DMMA flops against the per-element conversion
// and reconstruction traffic).
static bool emu_eligible(const GemmParams& p, const Ctx& cx, bool beta_ok = false) {
  if (p.Bidx || (p.beta != 0.0 && !beta_ok) || (p.beta != 0.0 && p.blk_j1a) || p.split > 1) return false;
  const double work = (double)p.M * p.N * p.K;
  if (work * p.batch < (double)cx.opt[HPS_OPT_EMU_MIN_WORK] || p.K < cx.opt[HPS_OPT_EMU_MIN_K] || p.M % 4 ||
      p.N % 4 || p.K % 16)
    return false;
  return !((reinterpret_cast<uintptr_t>(p.C) & 15) || (p.ldc % 2) || (p.strideC % 2));
}

// Slice scheme. Returns HPS_OK when the GEMM ran emulated, 1 when the caller should run it on DMMA
// instead (not eligible, no scratch inside a graph capture, or no cuBLASLt plan), an error code on
// failure.
static int emu_gemm_slices(const GemmParams& p, Ctx& cx, cudaStream_t st) {
  const int s = (int)cx.opt[HPS_OPT_EMU_SLICES];
  if (s <= 0 || !emu_eligible(p, cx)) return 1;
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


// ---------------------------------------------------------------------------------------------
// Modular scheme (Chinese remainder theorem; Ozaki, Uchino & Imamura's "scheme II", restated).
//
// Rows of A and columns of B are scaled by powers of two and rounded to integers,
//   A' = rint(diag(2^sig) A),  B' = rint(B diag(2^tau)),  with ||A'_i||_2 <= 2^PA, ||B'_j||_2 <= 2^PB,
// so by Cauchy-Schwarz every entry of the exact integer product C' = A'B' is at most 2^(PA + PB) <=
// Mod / 8 in magnitude, Mod = m_0 ... m_(n-1) (pairwise coprime, <= 256). Per modulus the residues
// A'_l = A' mod m_l, B'_l = B' mod m_l (symmetric, int8) give C_l = A'_l B'_l exactly in int32 (|C_l|
// <= K 2^14), one int8 GEMM each, and
//   C' = sum_l (C_l mod m_l) w_l  (mod Mod),  w_l = (Mod / m_l) ((Mod / m_l)^-1 mod m_l),
// recovered in fp64 from an exact high part (w_l rounded to a multiple of 2^E, 42 significant bits:
// sums of r w_hi are exact) plus a low part, and the quotient by Mod rounded away (|C'| <= Mod / 8
// keeps it unambiguous). C = diag(2^-sig) C' diag(2^-tau). The only rounding is that of A' and B'
// (<= 1/2 per entry, relative to the row / column 2-norm 2^-PA, 2^-PB) and the final fp64 sum: with
// 14 moduli (Mod ~ 2^110.2, PA = 53, PB = 54) the product error is at or below a DGEMM's, for n
// int8 GEMMs instead of the slice scheme's s (s + 1) / 2 = 36.
// ---------------------------------------------------------------------------------------------
constexpr int CRT_MAX = 16;
struct CrtConst {
  int n, PA, PB, E;
  double m[CRT_MAX], inv_m[CRT_MAX];  // residues of the scaled operands (fp64, exact)
  int mi[CRT_MAX], minv[CRT_MAX];     // reduction of int32 products: minv = floor(2^32 / m)
  double W[CRT_MAX], wlo[CRT_MAX];    // w_l = W_l 2^E + wlo_l, W_l integer, |wlo_l| <= 2^(E - 1)
  double Mh, Mlo;                     // Mod = Mh 2^E + Mlo
  double shi0, slo0;                  // -kCrtBias sum W_l (exact), -kCrtBias sum wlo_l: the sums start here
  double twoE_over_M, inv_M, twoE;
  double gP[(CRT_MAX + 2) / 3], ginvP[(CRT_MAX + 2) / 3];  // residue groups: products of moduli 3g..3g+2 (< 2^24)
};

static const int kModuli[CRT_MAX] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};

// Reconstruction arithmetic (k_crt_accum), with r_l = C_l mod m_l in [-128, 127], n <= 16 and
// E = bits - 36 (Mod < 2^bits), all in fp64. The residue byte b_l = r_l + 128 enters as the double
// d_l = 4096 + b_l = r_l + kCrtBias, built with ONE byte permute (the byte dropped into mantissa
// bits 8..15 of the high word 0x40B00000; low word 0), so the sums run over d_l from a bias-
// cancelling start value instead of converting and unbiasing every residue:
//   shi = shi0 + sum d_l W_l = sum r_l W_l   exact: |W_l| <= 2^35 + 1, d_l < 2^12.1, every partial sum
//                                            an integer below 2^51 (shi0 = -kCrtBias sum W_l, exact)
//   slo = slo0 + sum d_l wlo_l = sum r_l wlo_l   exact as well: wlo_l is w_l's remainder rounded to a
//                                            multiple of 2^(E - 34) (<= 34 significant bits), which
//                                            shifts C' by at most 14 * 128 * 2^(E - 35) = 2^(bits - 60)
//   q   = rint(shi 2^E / Mod + slo / Mod)   |C'| <= Mod / 8 leaves a 3/8 margin to the rounding edge
//   C'  = (shi - q Mh) 2^E + (slo - q Mlo)  the first factor exact (an integer < 2^47)
// so C' carries an absolute error ~2^(bits - 60): 1/16 ulp of the largest |C'| ~ 2^(bits - 4), and a
// thousand times below the rounding of A' and B' themselves (~sqrt(K) 2^(PB - 1) >= 2^(bits / 2 + 3)).
// Both sums being exact, zero residues give an exact zero and the result does not depend on order.
constexpr double kCrtBias = 4224.0;  // 4096 (the permuted double's leading one) + 128 (the byte's bias)
static bool crt_constants(int n, CrtConst& c) {
  if (n < 2 || n > CRT_MAX) return false;
  typedef unsigned __int128 u128;
  typedef __int128 i128;
  u128 Mod = 1;
  for (int l = 0; l < n; ++l) Mod *= (u128)kModuli[l];
  int bits = 0;  // Mod < 2^bits
  while (bits < 128 && (u128(1) << bits) <= Mod) ++bits;
  const int flo = bits - 1;  // 2^flo <= Mod
  // |C'| <= 2^(PA + PB) <= 2^(flo - 3) <= Mod / 8
  c.n = n;
  c.PA = (flo - 3) / 2;
  c.PB = flo - 3 - c.PA;
  c.E = bits - 36;
  auto to_double = [](i128 v) {
    const bool neg = v < 0;
    u128 u = neg ? (u128)(-v) : (u128)v;
    const double d = (double)(unsigned long long)(u >> 64) * 18446744073709551616.0 + (double)(unsigned long long)(u & ~0ULL);
    return neg ? -d : d;
  };
  // v = hi 2^E + lo, hi integer, |lo| <= 2^(E - 1); keep > 0: lo rounded to a multiple of 2^(E - 34)
  // (at most 34 significant bits, so that sums of d_l wlo_l are exact too)
  auto split = [&](i128 v, double& hi, double& lo, bool keep33) {
    const i128 unit = (i128)1 << c.E;
    const i128 qv = v >= 0 ? (v + unit / 2) >> c.E : -((-v + unit / 2) >> c.E);
    hi = to_double(qv);  // |qv| < 2^37: exact
    i128 rem = v - qv * unit;
    if (keep33) {
      const i128 u2 = (i128)1 << (c.E - 34);
      rem = (rem >= 0 ? (rem + u2 / 2) / u2 : -((-rem + u2 / 2) / u2)) * u2;
    }
    lo = to_double(rem);
  };
  const double dMod = to_double((i128)Mod);
  for (int l = 0; l < n; ++l) {
    const long long m = kModuli[l];
    const u128 Ml = Mod / (u128)m;
    const long long r = (long long)(Ml % (u128)m);
    long long y = 1;
    while ((r * y) % m != 1) ++y;  // m <= 256: direct search
    const u128 w = (Ml * (u128)y) % Mod;
    const i128 ws = (w > Mod / 2) ? (i128)w - (i128)Mod : (i128)w;
    c.m[l] = (double)m;
    c.inv_m[l] = 1.0 / (double)m;
    c.mi[l] = (int)m;
    c.minv[l] = (int)((1ULL << 32) / (unsigned long long)m);
    split(ws, c.W[l], c.wlo[l], true);
  }
  split((i128)Mod, c.Mh, c.Mlo, false);
  double sw = 0.0, swl = 0.0;  // integers (in units of 1 and 2^(E - 34)) below 2^40: both sums exact
  for (int l = 0; l < n; ++l) { sw += c.W[l]; swl += c.wlo[l]; }
  c.shi0 = -kCrtBias * sw;  // 13 x 40 bits: exact
  c.slo0 = -kCrtBias * swl;
  c.twoE = ldexp(1.0, c.E);
  c.twoE_over_M = c.twoE / dMod;
  c.inv_M = 1.0 / dMod;
  for (int g = 0; 3 * g < n; ++g) {
    double P = 1.0;
    for (int l = 3 * g; l < std::min(n, 3 * g + 3); ++l) P *= (double)kModuli[l];  // < 2^24, exact
    // a short last group (n % 3 != 0): a power-of-two multiple of the product reduces just as well
    // (every modulus of the group divides it) and keeps the first quotient x / P below 2^51 for
    // |x| up to 2^61 (16 moduli; with P = 193 alone the 1.5 * 2^52 shift no longer rounded it)
    while (P < 0x1p20) P *= 2.0;
    c.gP[g] = P;
    c.ginvP[g] = 1.0 / P;
  }
  return true;
}

// sig[b][i] (tau[b][j]): the power of two that brings row i of A (column j of B) to 2-norm < 2^P;
// INT_MIN marks a non-finite row / column (its outputs become NaN, as a DGEMM's would be non-finite).
// The squares are summed after an exact power-of-two prescale by the maximum (no overflow).
// x 2^e, exact for |e| <= 1022 (one multiply by a constructed power of two), else ldexp
__device__ __forceinline__ double crt_ldexp(double x, int e) {
  if (e >= -1022 && e <= 1023) return x * __longlong_as_double((long long)(e + 1023) << 52);
  return ldexp(x, e);
}
// The exponent from the maximum mx and the sum of squares ss of a row / column, accumulated unscaled
// in one pass; valid when mx is in [2^-450, 2^450] (no square overflows, every square that matters
// for the norm stays normal). Returns INT_MIN for a non-finite row, 0 for a zero row, INT_MAX when
// the caller must rescale (mx outside that range).
__device__ __forceinline__ int crt_exponent_1pass(double mx, double ss, int P) {
  if (!isfinite(mx) || !isfinite(ss)) return isfinite(mx) ? INT_MAX : INT_MIN;
  if (mx == 0.0) return 0;
  if (mx < 0x1p-450 || mx > 0x1p450) return INT_MAX;
  int ex;
  frexp(sqrt(ss) * (1.0 + 0x1p-30), &ex);  // ||row|| < 2^ex (an upper bound despite rounding)
  return P - ex;
}
// Rescaled second pass (rare): squares of x 2^-em, mx < 2^em
__device__ __forceinline__ int crt_exponent_scaled(double ss_scaled, int em, int P) {
  int ex;
  frexp(sqrt(ss_scaled) * (1.0 + 0x1p-30), &ex);
  return P - ex - em;
}

__global__ void k_crt_row_scale(const double* __restrict__ A, long long lda, long long sA, int M, int K, int P,
                                int* __restrict__ sig) {
  const int b = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= M) return;
  const double* Ar = A + (long long)b * sA + (long long)r * lda;
  double mx[4] = {0.0, 0.0, 0.0, 0.0}, ss[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = lane; k < K; k += 128) {  // K % 16 == 0: four independent loads per lane
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = k + 32 * u < K ? __ldg(Ar + k + 32 * u) : 0.0;
      mx[u] = fmax(mx[u], fabs(v));
      ss[u] = fma(v, v, ss[u]);
    }
  }
  const double m = warp_max(fmax(fmax(mx[0], mx[1]), fmax(mx[2], mx[3])));
  const double q = warp_sum((ss[0] + ss[1]) + (ss[2] + ss[3]));
  int e = crt_exponent_1pass(m, q, P);
  if (e == INT_MAX) {  // rescale by the maximum and sum again
    int em;
    frexp(m, &em);
    double s2 = 0.0;
    for (int k = lane; k < K; k += 32) {
      const double v = ldexp(Ar[k], -em);
      s2 = fma(v, v, s2);
    }
    e = crt_exponent_scaled(warp_sum(s2), em, P);
  }
  if (lane == 0) sig[(long long)b * M + r] = e;
}

// 32 columns x 8 row slices per CTA (coalesced row reads), 8 rows in flight per thread
__global__ void __launch_bounds__(256) k_crt_col_scale(const double* __restrict__ B, long long ldb, long long sB, int K,
                                                      int N, int P, int* __restrict__ tau) {
  __shared__ double red[2][8][33];
  __shared__ int ex[32];
  const int b = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + tx;
  const double* Bb = B + (long long)b * sB + j;
  double mx[4] = {0.0, 0.0, 0.0, 0.0}, ss[4] = {0.0, 0.0, 0.0, 0.0};
  if (j < N)
    for (int k = ty; k < K; k += 64) {  // 8 loads in flight per thread
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = k + 8 * u < K ? __ldg(Bb + (long long)(k + 8 * u) * ldb) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        mx[u & 3] = fmax(mx[u & 3], fabs(v[u]));
        ss[u & 3] = fma(v[u], v[u], ss[u & 3]);
      }
    }
  red[0][ty][tx] = fmax(fmax(mx[0], mx[1]), fmax(mx[2], mx[3]));
  red[1][ty][tx] = (ss[0] + ss[1]) + (ss[2] + ss[3]);
  __syncthreads();
  if (ty == 0) {
    double m = red[0][0][tx], q = red[1][0][tx];
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      m = fmax(m, red[0][r][tx]);
      q += red[1][r][tx];
    }
    ex[tx] = crt_exponent_1pass(m, q, P);
    red[0][0][tx] = m;
  }
  __syncthreads();
  if (ex[tx] == INT_MAX) {  // rare: rescale this column by its maximum and sum again
    int em;
    frexp(red[0][0][tx], &em);
    double s2 = 0.0;
    for (int k = ty; k < K; k += 8) {
      const double v = ldexp(Bb[(long long)k * ldb], -em);
      s2 = fma(v, v, s2);
    }
    red[1][ty][tx] = s2;
  }
  __syncthreads();
  if (ty == 0 && j < N) {
    int e = ex[tx];
    if (e == INT_MAX) {
      double q = 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r) q += red[1][r][tx];
      int em;
      frexp(red[0][0][tx], &em);
      e = crt_exponent_scaled(q, em, P);
    }
    tau[(long long)b * N + j] = e;
  }
}

// Residues of the integer x (|x| <= 2^61, exact in fp64) modulo every m_l, each in [-128, 128]
// (+128 only for m = 256, whose byte wraps to the same class), as the low bytes of r[l]. Two levels,
// all on the FP64 pipe and without range fixes: y = x mod P_g for the product P_g < 2^24 of three
// moduli (the quotient rounded through the 1.5 * 2^52 shift may be one off, so |y| <= 1.5 P_g <
// 2^25, exact), then y mod m_l with an exact quotient (y / m_l is far from the half-integers its
// rounding could confuse), read out through the same shift.
constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
template <int NM>
__device__ __forceinline__ void crt_residues(double x, const CrtConst& c, int (&r)[NM]) {
#pragma unroll
  for (int g = 0; g < (NM + 2) / 3; ++g) {
    const double q = fma(x, c.ginvP[g], kShift) - kShift;
    const double y = fma(-c.gP[g], q, x);
    const double ys = y + kShift;  // exact; then y - m ql + kShift in one exact fma
#pragma unroll
    for (int l = 3 * g; l < (3 * g + 3 < NM ? 3 * g + 3 : NM); ++l) {
      const double ql = fma(y, c.inv_m[l], kShift) - kShift;
      r[l] = __double2loint(fma(-c.m[l], ql, ys));
    }
  }
}

// residues of the scaled rows of A: out[l][b][i][k]; 4 k per thread
template <int NM>
__global__ void __launch_bounds__(256) k_crt_split_rows(const double* __restrict__ A, long long lda, long long sA, int M,
                                                       int K, int batch, const int* __restrict__ sig, CrtConst c,
                                                       signed char* __restrict__ out) {
  const int b = blockIdx.z, r = blockIdx.y;
  const int k4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k4 >= K) return;  // K % 16 == 0
  const int sg = sig[(long long)b * M + r];
  const double* Ar = A + (long long)b * sA + (long long)r * lda + k4;
  int res[4][NM];
#pragma unroll
  for (int u = 0; u < 4; ++u) crt_residues<NM>(sg == INT_MIN ? 0.0 : rint(crt_ldexp(Ar[u], sg)), c, res[u]);
  const long long plane = (long long)batch * M * K;
  unsigned* o = reinterpret_cast<unsigned*>(out + ((long long)b * M + r) * K + k4);
#pragma unroll
  for (int l = 0; l < NM; ++l)
    o[l * (plane / 4)] = (res[0][l] & 0xFF) | ((res[1][l] & 0xFF) << 8) | ((res[2][l] & 0xFF) << 16) | (res[3][l] << 24);
}

// residues of the scaled columns of B, transposed: out[l][b][j][k]. Tile: 32 k x 64 j through
// shared memory; each thread 8 consecutive k of one column (two packed words per modulus).
template <int NM>
__global__ void __launch_bounds__(256) k_crt_split_cols(const double* __restrict__ B, long long ldb, long long sB, int K,
                                                       int N, int batch, const int* __restrict__ tau, CrtConst c,
                                                       signed char* __restrict__ out) {
  __shared__ unsigned sd[NM][64][9];  // 32 k bytes per (l, j) + a padding word
  const int b = blockIdx.z;
  const int k0 = blockIdx.y * 32, j0 = blockIdx.x * 64;
  const double* Bb = B + (long long)b * sB;
  const int jj = threadIdx.x % 64, kq = threadIdx.x / 64;  // k = k0 + 8 kq + i
  const int j = j0 + jj;
  const int tj = j < N ? tau[(long long)b * N + j] : INT_MIN;
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = k0 + 8 * kq + i;
    x[i] = (k < K && tj != INT_MIN) ? __ldg(Bb + (long long)k * ldb + j) : 0.0;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int res[4][NM];
#pragma unroll
    for (int i = 0; i < 4; ++i) crt_residues<NM>(rint(crt_ldexp(x[4 * h + i], tj == INT_MIN ? 0 : tj)), c, res[i]);
#pragma unroll
    for (int l = 0; l < NM; ++l)
      sd[l][jj][2 * kq + h] =
          (res[0][l] & 0xFF) | ((res[1][l] & 0xFF) << 8) | ((res[2][l] & 0xFF) << 16) | (res[3][l] << 24);
  }
  __syncthreads();
  const long long plane = (long long)batch * N * K;
  signed char* ob = out + (long long)b * N * K;
  for (int idx = threadIdx.x; idx < NM * 64 * 8; idx += blockDim.x) {  // 4 bytes per store
    const int w = idx % 8, rest = idx / 8, jr = rest % 64, l = rest / 64;
    const int k = k0 + 4 * w, jg = j0 + jr;
    if (k < K && jg < N) *reinterpret_cast<unsigned*>(ob + l * plane + (long long)jg * K + k) = sd[l][jr][w];
  }
}

// ---------------------------------------------------------------------------------------------
// Residues on the integer pipes (HPS_OPT_EMU_SPLIT 1, the default): the FP64-pipe version above
// spends ~63 FP64 operations per element and is bound by that pipe. Here the scaled integer y (|y| <=
// 2^61) is converted once (cvt.rni.s64.f64) and shifted to v = y + S > 0, S a multiple of every
// modulus of a group (the first eight moduli; the rest), so v = y modulo each of them. The eight
// bytes d_i of v feed a small int8 tensor-core product (legacy mma.sync m16n8k32, u8 x s8):
//   c_l = sum_i d_i (256^i mod m_l)     (symmetric constants: |c_l| < 2^18) is congruent to y.
// A lane holds two elements (MMA rows g and g + 8); an MMA row is four consecutive elements (one per
// lane of a quad), and the B fragment is block-diagonal over those four slots, so one MMA yields 2
// moduli x 4 slots for 16 + 16 elements and 7 MMAs cover 14 moduli. Then
//   q = floor((c + h) / m) = (c minv + h minv + 2^20) >> 32   (exact for |c| < 2^18: minv = floor(2^32 /
//                                        m) + 1, the 2^20 outweighs minv's excess times a negative c)
//   r = c - q m in [-h, m - 1 - h], h = floor(m / 2): a signed byte congruent to y,
// two integer multiply-adds per residue; the four slots of a row are packed into one word with byte
// permutes and one quad shuffle. ~65 instructions per element instead of ~167.
struct ResTab {
  unsigned clo[CRT_MAX], chi[CRT_MAX];  // 256^i mod m as signed bytes, i = 0..3 and 4..7
  unsigned minv[CRT_MAX], kq[CRT_MAX];  // floor(2^32 / m) + 1, and h * minv + 2^20 (< 2^32)
  int m[CRT_MAX];
  unsigned long long shift[2];          // S of the moduli 0..7 and of the moduli 8..
};
static bool res_tab(int n, ResTab& t) {
  typedef unsigned __int128 u128;
  for (int grp = 0; grp < 2; ++grp) {
    u128 P = 1;
    for (int l = 8 * grp; l < std::min(n, 8 * grp + 8); ++l) P *= (u128)kModuli[l];
    const u128 lo = (u128)1 << 61, hi = ((u128)1 << 64) - ((u128)1 << 61);  // v = y + S in (0, 2^64) for |y| <= 2^61
    u128 S = P * std::max<u128>(1, ((u128)1 << 62) / P);
    if (S < lo || S > hi) return false;
    t.shift[grp] = (unsigned long long)S;
  }
  for (int l = 0; l < CRT_MAX; ++l) {
    const int m = kModuli[l < n ? l : 0];
    unsigned lo = 0, hi = 0;
    long long pw = 1;
    for (int i = 0; i < 8; ++i) {
      int c = (int)(pw % m);
      if (c >= (m + 1) / 2) c -= m;  // [-128, 127]
      (i < 4 ? lo : hi) |= (unsigned)(c & 0xFF) << (8 * (i & 3));
      pw = (pw * 256) % m;
    }
    t.clo[l] = lo;
    t.chi[l] = hi;
    t.minv[l] = (unsigned)((1ULL << 32) / (unsigned long long)m) + 1u;
    t.kq[l] = (unsigned)(m / 2) * t.minv[l] + (1u << 20);
    t.m[l] = m;
  }
  return true;
}

// keeps a per-lane constant in its register: ptxas otherwise re-reads the parameter bank (an indexed
// LDC through the address-divergence unit) at every use, which then bounds the kernel. A shuffle
// from the own lane is opaque to it.
__device__ __forceinline__ void res_pin(unsigned& x) {
  asm volatile("{\n\t.reg .u32 l;\n\tmov.u32 l, %%laneid;\n\tshfl.sync.idx.b32 %0, %0, l, 31, 0xffffffff;\n\t}" : "+r"(x));
}
__device__ __forceinline__ void res_pin(int& x) {
  asm volatile("{\n\t.reg .u32 l;\n\tmov.u32 l, %%laneid;\n\tshfl.sync.idx.b32 %0, %0, l, 31, 0xffffffff;\n\t}" : "+r"(x));
}

template <int NM>
struct ResFrag {  // a lane's constants: B fragments of the NJ MMAs and the reduction constants of its moduli
  static constexpr int NJ = (NM + 1) / 2;
  unsigned b0[NJ], b1[NJ];
  int minv[NJ], negm[NJ];
  long long kq[NJ];
  __device__ __forceinline__ void init(const ResTab& t, int lane) {
    const int g = lane >> 2, tq = lane & 3;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int lb = 2 * j + (g >> 2);  // B column g: modulus lb, element slot g & 3
      const bool on = tq == (g & 3) && lb < NM;
      b0[j] = on ? t.clo[lb < NM ? lb : 0] : 0u;
      b1[j] = on ? t.chi[lb < NM ? lb : 0] : 0u;
      const int lc = 2 * j + (tq >> 1) < NM ? 2 * j + (tq >> 1) : 0;  // C columns 2 tq, 2 tq + 1: modulus lc
      negm[j] = -t.m[lc];
      minv[j] = (int)t.minv[lc];
      unsigned k = t.kq[lc];
      res_pin(b0[j]);
      res_pin(b1[j]);
      res_pin(negm[j]);
      res_pin(minv[j]);
      res_pin(k);
      kq[j] = (long long)k;
    }
  }
};

// w[j]: the residues modulo m_(2j + (tq >> 1)) of four consecutive elements as one word of signed
// bytes. y0 is this lane's element of the first 32 (element index = lane), y1 of the second 32. Even
// lanes receive the word of elements 4g .. 4g + 3, odd lanes that of elements 32 + 4g .. 32 + 4g + 3.
template <int NM>
__device__ __forceinline__ void res_words(long long y0, long long y1, const ResFrag<NM>& f, const ResTab& t, int lane,
                                          unsigned (&w)[ResFrag<NM>::NJ]) {
  const bool odd = lane & 1;
#pragma unroll
  for (int j = 0; j < ResFrag<NM>::NJ; ++j) {
    const unsigned long long S = t.shift[j >= 4 ? 1 : 0];  // MMA j: moduli 2j, 2j + 1
    const unsigned long long v0 = (unsigned long long)y0 + S, v1 = (unsigned long long)y1 + S;
    int c0, c1, c2, c3;
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%10, %10, %10, %10};"
                 : "=r"(c0), "=r"(c1), "=r"(c2), "=r"(c3)
                 : "r"((unsigned)v0), "r"((unsigned)v1), "r"((unsigned)(v0 >> 32)), "r"((unsigned)(v1 >> 32)), "r"(f.b0[j]),
                   "r"(f.b1[j]), "r"(0));
    auto red = [&](int c) {  // c - m floor((c + h) / m)
      const int q = (int)(((long long)c * (long long)f.minv[j] + f.kq[j]) >> 32);
      return (unsigned)(q * f.negm[j] + c);
    };
    const unsigned pg = __byte_perm(red(c0), red(c1), 0x0040), pg8 = __byte_perm(red(c2), red(c3), 0x0040);
    const unsigned recv = __shfl_xor_sync(0xffffffffu, odd ? pg : pg8, 1);
    w[j] = __byte_perm(odd ? recv : pg, odd ? pg8 : recv, 0x5410);
  }
}

// x 2^e rounded to an integer (ties to even, as rint), e fixed per row / column: one multiply when 2^e
// is a normal number
__device__ __forceinline__ long long res_scaled(double x, int e, double pw, bool direct) {
  return __double2ll_rn(direct ? x * pw : ldexp(x, e));
}

// residues of the scaled rows of A: out[l][b][i][k]; a warp takes 256 consecutive k of a row in 4
// steps of 64 (the 8 loads of a lane issued first); 128 threads, 5 CTAs per SM (96 registers)
template <int NM>
__global__ void __launch_bounds__(128, 5) k_crt_split_rows_mma(const double* __restrict__ A, long long lda, long long sA,
                                                              int M, int K, int batch, const int* __restrict__ sig,
                                                              ResTab t, signed char* __restrict__ out) {
  constexpr int NJ = ResFrag<NM>::NJ;
  const int b = blockIdx.z, r = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kbeg = (blockIdx.x * 4 + warp) * 256;
  if (kbeg >= K) return;
  ResFrag<NM> f;
  f.init(t, lane);
  const int sg = sig[(long long)b * M + r];
  const bool direct = sg >= -1022 && sg <= 1023;
  const double pw = __longlong_as_double((long long)((direct ? sg : 0) + 1023) << 52);
  const double* Ar = A + (long long)b * sA + (long long)r * lda;
  double x[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int k = kbeg + 32 * s + lane;
    x[s] = (k < K && sg != INT_MIN) ? __ldg(Ar + k) : 0.0;
  }
  const long long plane = (long long)batch * M * K;
  const int g = lane >> 2, tq = lane & 3;
  const int lmine = tq >> 1, koff = (lane & 1) * 32 + 4 * g;
  // this lane's word of modulus 2j + lmine at step s: obase + 2 j plane + 64 s
  signed char* obase = out + ((long long)b * M + r) * K + lmine * plane + kbeg + koff;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int k0 = kbeg + 64 * s;
    if (k0 >= K) break;
    unsigned w[NJ];
    res_words<NM>(res_scaled(x[2 * s], sg, pw, direct), res_scaled(x[2 * s + 1], sg, pw, direct), f, t, lane, w);
    if (k0 + koff < K) {
      signed char* o = obase + 64 * s;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        if (2 * j + lmine < NM) *reinterpret_cast<unsigned*>(o) = w[j];
        o += 2 * plane;
      }
    }
  }
}

// residues of the scaled columns of B, transposed: out[l][b][j][k]. CTA tile 32 k x 64 j in three
// phases through shared memory: (1) coalesced row reads, each element scaled by its column's power of
// two and converted to an integer; (2) warp w takes columns 16w .. 16w + 15: per step a lane holds
// the integers of (k = 4s + tq, j = g) and (k = 4s + tq, j = 8 + g), so a quad = four consecutive k
// of one column = one output word, staged at [l][j][s]; (3) the 32 bytes of every (l, j) leave as
// full sectors (8 lanes x 4 bytes).
template <int NM>
struct ResColsSmem {
  static constexpr int SY = 68;           // integer tile row stride (64-bit words; == 4 mod 16: phase 2's quad reads are conflict-free)
  static constexpr int SL = 64 * 9 + 16;  // words per modulus: 64 columns x (8 words + 1 pad), + 16 so that a lane pair's two moduli take different banks
  static constexpr int kBytes = 32 * SY * 8 + NM * SL * 4;
};
template <int NM>
__global__ void __launch_bounds__(128, 4) k_crt_split_cols_mma(const double* __restrict__ B, long long ldb, long long sB,
                                                              int K, int N, int batch, const int* __restrict__ tau,
                                                              ResTab t, signed char* __restrict__ out) {
  constexpr int NJ = ResFrag<NM>::NJ;
  constexpr int SY = ResColsSmem<NM>::SY, SL = ResColsSmem<NM>::SL;
  extern __shared__ __align__(16) unsigned char res_smem[];
  long long* sy = reinterpret_cast<long long*>(res_smem);               // 32 x SY integers
  unsigned* so = reinterpret_cast<unsigned*>(res_smem + 32 * SY * 8);  // [l][j][s]: NM x SL words
  const int b = blockIdx.z, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int j0 = blockIdx.x * 64, k0 = blockIdx.y * 32;
  {  // phase 1: thread -> column pair 2 (tid % 32), rows tid / 32 + 4 i
    const int jc = j0 + 2 * lane;
    const int t0 = jc < N ? tau[(long long)b * N + jc] : INT_MIN, t1 = jc + 1 < N ? tau[(long long)b * N + jc + 1] : INT_MIN;
    const int e0 = t0 == INT_MIN ? 0 : t0, e1 = t1 == INT_MIN ? 0 : t1;
    const bool d0 = e0 >= -1022 && e0 <= 1023, d1 = e1 >= -1022 && e1 <= 1023;
    const double p0 = __longlong_as_double((long long)((d0 ? e0 : 0) + 1023) << 52);
    const double p1 = __longlong_as_double((long long)((d1 ? e1 : 0) + 1023) << 52);
    const double* Bb = B + (long long)b * sB + jc;
    const bool vec = jc + 1 < N && !(ldb & 1) && !(reinterpret_cast<uintptr_t>(B) & 15) && !(sB & 1);
    double2 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int k = k0 + warp + 4 * i;
      x[i] = make_double2(0.0, 0.0);
      if (k < K) {
        if (vec) {
          x[i] = __ldg(reinterpret_cast<const double2*>(Bb + (long long)k * ldb));
        } else {
          if (jc < N) x[i].x = __ldg(Bb + (long long)k * ldb);
          if (jc + 1 < N) x[i].y = __ldg(Bb + (long long)k * ldb + 1);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int kr = warp + 4 * i;
      const long long y0 = t0 == INT_MIN ? 0 : res_scaled(x[i].x, e0, p0, d0);
      const long long y1 = t1 == INT_MIN ? 0 : res_scaled(x[i].y, e1, p1, d1);
      *reinterpret_cast<longlong2*>(&sy[kr * SY + 2 * lane]) = make_longlong2(y0, y1);
    }
  }
  ResFrag<NM> f;
  f.init(t, lane);
  __syncthreads();
  {  // phase 2
    const int jl = 16 * warp + g;  // local columns jl and jl + 8
    const int jm = (lane & 1) ? jl + 8 : jl, lmine = tq >> 1;
#pragma unroll 2
    for (int s = 0; s < 8; ++s) {
      unsigned w[NJ];
      res_words<NM>(sy[(4 * s + tq) * SY + jl], sy[(4 * s + tq) * SY + jl + 8], f, t, lane, w);
#pragma unroll
      for (int j = 0; j < NJ; ++j)
        if (2 * j + lmine < NM) so[(2 * j + lmine) * SL + jm * 9 + s] = w[j];
    }
  }
  __syncthreads();
  const long long plane = (long long)batch * N * K;
  signed char* ob = out + (long long)b * N * K;
  for (int idx = tid; idx < NM * 64 * 8; idx += 128) {  // 4 bytes per store
    const int wq = idx % 8, rest = idx / 8, jr = rest % 64, l = rest / 64;
    const int k = k0 + 4 * wq, jg = j0 + jr;
    if (k < K && jg < N) *reinterpret_cast<unsigned*>(ob + l * plane + (long long)jg * K + k) = so[l * SL + jr * 9 + wq];
  }
}

#define HPS_CRT_SWITCH(n, CALL)                                                                            \
  switch (n) {                                                                                             \
    case 2: CALL(2); break; case 3: CALL(3); break; case 4: CALL(4); break; case 5: CALL(5); break;        \
    case 6: CALL(6); break; case 7: CALL(7); break; case 8: CALL(8); break; case 9: CALL(9); break;        \
    case 10: CALL(10); break; case 11: CALL(11); break; case 12: CALL(12); break; case 13: CALL(13); break; \
    case 14: CALL(14); break; case 15: CALL(15); break; case 16: CALL(16); break;                          \
  }

// (C_l mod m_l) + 128 in [0, 255] of an int32 product (|v| < 2^30; as mod_byte in i8gemm.cu)
__device__ __forceinline__ unsigned crt_biased(int v, int m, int minv) {
  const unsigned x = (unsigned)(v + m * ((1 << 30) / m + 1));
  const int q = (int)__umulhi(x, (unsigned)minv);
  int r = (int)x - q * m;
  r = r >= m ? r - m : r;
  r = r > 127 ? r - m : r;
  return (unsigned)(r + 128);
}
// biased residue byte K of the packed word x -> the exact double 4096 + b = r + kCrtBias: one byte
// permute drops the byte into mantissa bits 8..15 of the high word 0x40B00000 (2^12). Only the high
// word of d is rewritten (its low word stays the zero it was initialised with), so no move is spent
// on the low half of every temporary.
template <int K>
__device__ __forceinline__ void crt_biased_double(double& d, unsigned x) {
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %0;\n\tprmt.b32 hi, %1, 0x40B00000, %2;\n\tmov.b64 %0, {lo, hi};\n\t}"
      : "+d"(d)
      : "r"(x), "n"(0x7604 + (K << 4)));
}
// 2^e for |e| <= 1022 (exact scale of the outputs), else ldexp
__device__ __forceinline__ double crt_scale(double x, int e) {
  if (e >= -1022 && e <= 1023) return x * __longlong_as_double((long long)(e + 1023) << 52);
  return ldexp(x, e);
}

template <typename TIn>
struct CrtIn;
template <>
struct CrtIn<int> {  // cuBLASLt int32 products: reduced here
  typedef int4 V;
  static __device__ __forceinline__ void biased(const V& x, const CrtConst& c, int l, double (&d)[4]) {
    crt_biased_double<0>(d[0], crt_biased(x.x, c.mi[l], c.minv[l]));
    crt_biased_double<0>(d[1], crt_biased(x.y, c.mi[l], c.minv[l]));
    crt_biased_double<0>(d[2], crt_biased(x.z, c.mi[l], c.minv[l]));
    crt_biased_double<0>(d[3], crt_biased(x.w, c.mi[l], c.minv[l]));
  }
};
template <>
struct CrtIn<unsigned char> {  // the tcgen05 kernel's biased residues, 4 per word
  typedef unsigned V;
  static __device__ __forceinline__ void biased(const V& x, const CrtConst&, int, double (&d)[4]) {
    crt_biased_double<0>(d[0], x);
    crt_biased_double<1>(d[1], x);
    crt_biased_double<2>(d[2], x);
    crt_biased_double<3>(d[3], x);
  }
};

// Reconstruction of the output columns [j0, j0 + nc) from the NM products of that panel
// (Cl[l][b][i][0..nc): int32 products, or biased int8 residues), with the row / column scales,
// alpha, the merge's block-diagonal addend and the non-finite flag. Rows on blockIdx.y (grid-stride),
// 4 columns per thread; all NM loads of a row are issued before the arithmetic (one byte permute and
// two fma per residue, no conversions). Everything that depends on the columns only is set up
// before the row loop: the column scales as doubles (times alpha), their block-diagonal map entries;
// per row the scale is one product of two powers of two (rows or columns whose exponents leave the
// normal range take crt_scale instead), and the residue planes are walked with one pointer.
// (Two rows per step, for more loads in flight, was slower: 8.2 vs 6.3 ms on 64 x 4096 x 4096 outputs.)
struct CrtCols {
  int tj[4];
  double csa[4];   // alpha 2^-tj (fast path)
  bool fast;       // every tj finite and within the fast range, alpha's exponent small
  int tjmin, tjmax;
  int cm[4];       // block-diagonal addend: column map entries
  bool ctop[4];    //   and the half each column lies in
};
constexpr int kCrtFastExp = 960;  // |sig|, |tau|, |sig + tau| up to here: 2^-e built and multiplied directly

template <int NM, typename TIn>
__device__ __forceinline__ void crt_row(const typename CrtIn<TIn>::V (&in)[NM], int sr, const CrtCols& cc, int b, int r,
                                        int col0, const GemmParams& p, const CrtConst& c, bool& bad) {
  double shi[4] = {c.shi0, c.shi0, c.shi0, c.shi0}, slo[4] = {c.slo0, c.slo0, c.slo0, c.slo0};
  double d[4] = {0.0, 0.0, 0.0, 0.0};  // r + kCrtBias (high words rewritten per modulus)
#pragma unroll
  for (int l = 0; l < NM; ++l) {
    CrtIn<TIn>::biased(in[l], c, l, d);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      shi[u] = fma(d[u], c.W[l], shi[u]);  // exact
      slo[u] = fma(d[u], c.wlo[l], slo[u]);  // exact
    }
  }
  double v[4];
  const bool fast = cc.fast && (unsigned)(sr + kCrtFastExp) <= 2u * kCrtFastExp &&
                    (unsigned)(sr + cc.tjmin + kCrtFastExp) <= 2u * kCrtFastExp &&
                    (unsigned)(sr + cc.tjmax + kCrtFastExp) <= 2u * kCrtFastExp;
  const double rs = __hiloint2double((int)((unsigned)(1023 - sr) << 20), 0);  // 2^-sr (used on the fast path only)
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double q = rint(fma(shi[u], c.twoE_over_M, slo[u] * c.inv_M));
    const double cp = fma(fma(-q, c.Mh, shi[u]), c.twoE, fma(-q, c.Mlo, slo[u]));
    if (fast) {
      v[u] = cp * (rs * cc.csa[u]);  // rs csa: an exact power-of-two scaling of alpha; one rounding
    } else {
      const double w = (sr == INT_MIN || cc.tj[u] == INT_MIN) ? __longlong_as_double(0x7ff8000000000000LL)
                                                               : crt_scale(cp, -(sr + cc.tj[u]));
      v[u] = w * p.alpha;
    }
  }
  if (p.blk_j1a) {  // T = blkdiag(Ta11, Tb22) + C S: the addend of this row's half
    const int n1 = p.M >> 1;
    const bool top = r < n1;
    const int gb = b + p.batch_offset;
    const double* src = (top ? p.blk.a(gb) : p.blk.bb(gb)) + (long long)(top ? p.blk_j1a[r] : p.blk_j2b[r - n1]) * p.blk.m;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (cc.ctop[u] == top) v[u] += src[cc.cm[u]];
  }
  double* dst = p.C + (long long)b * p.strideC + (long long)r * p.ldc + col0;
  if (p.beta != 0.0) {  // C = alpha A B + beta C
    const double2 o0 = *reinterpret_cast<const double2*>(dst), o1 = *reinterpret_cast<const double2*>(dst + 2);
    v[0] = fma(p.beta, o0.x, v[0]);
    v[1] = fma(p.beta, o0.y, v[1]);
    v[2] = fma(p.beta, o1.x, v[2]);
    v[3] = fma(p.beta, o1.y, v[3]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) bad |= !isfinite(v[u]);
  *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(dst + 2) = make_double2(v[2], v[3]);
}

template <int NM, typename TIn>
__global__ void __launch_bounds__(256, 4) k_crt_accum(const TIn* __restrict__ Cl, int M, int nc, int j0, GemmParams p,
                                                  CrtConst c, const int* __restrict__ sig,
                                                  const int* __restrict__ tau) {
  typedef typename CrtIn<TIn>::V V4;
  const int b = blockIdx.z;
  const int c4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const long long plane = (long long)p.batch * M * nc;
  bool bad = false;
  if (c4 < nc) {
    CrtCols cc;
    int ea;
    frexp(p.alpha, &ea);
    cc.fast = p.alpha != 0.0 && isfinite(p.alpha) && ea >= -30 && ea <= 30;
    cc.tjmin = INT_MAX;
    cc.tjmax = INT_MIN;
    const int n1 = p.M >> 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int col = j0 + c4 + u;
      const int t = tau[(long long)b * p.N + col];
      cc.tj[u] = t;
      cc.fast = cc.fast && (unsigned)(t + kCrtFastExp) <= 2u * kCrtFastExp;
      cc.tjmin = min(cc.tjmin, t);
      cc.tjmax = max(cc.tjmax, t);
      cc.csa[u] = __hiloint2double((int)((unsigned)(1023 - (cc.fast ? t : 0)) << 20), 0) * p.alpha;
      cc.ctop[u] = col < n1;
      cc.cm[u] = p.blk_j1a ? (cc.ctop[u] ? p.blk_j1a[col] : p.blk_j2b[col - n1]) : 0;
    }
    // 32-bit indices in units of V4 (four elements): n planes hold < 2^32 of them under the scratch
    // cap (<= 8 GB, emu_gemm_crt), so a load costs one index add and one wide multiply-add
    const V4* base = reinterpret_cast<const V4*>(Cl);
    const unsigned planeV = (unsigned)(plane >> 2), ncV = (unsigned)nc >> 2;
    const unsigned idx0 = (unsigned)b * (unsigned)M * ncV + ((unsigned)c4 >> 2);
    for (int r = blockIdx.y; r < M; r += gridDim.y) {
      unsigned idx = idx0 + (unsigned)r * ncV;
      V4 in[NM];
#pragma unroll
      for (int l = 0; l < NM; ++l) {
        in[l] = __ldcs(base + idx);
        idx += planeV;
      }
      crt_row<NM, TIn>(in, sig[(long long)b * M + r], cc, b, r, j0 + c4, p, c, bad);
    }
  }
  if (p.nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicMax(p.nonfinite, b + p.batch_offset);
}

template <typename TIn>
static void crt_accum_launch(int n, dim3 grid, cudaStream_t st, const TIn* Cl, int M, int nc, int j0,
                             const GemmParams& p, const CrtConst& c, const int* sig, const int* tau) {
#define HPS_CRT_CASE(NM) \
  case NM: k_crt_accum<NM, TIn><<<grid, 256, 0, st>>>(Cl, M, nc, j0, p, c, sig, tau); break;
  switch (n) {
    HPS_CRT_CASE(2) HPS_CRT_CASE(3) HPS_CRT_CASE(4) HPS_CRT_CASE(5) HPS_CRT_CASE(6) HPS_CRT_CASE(7)
    HPS_CRT_CASE(8) HPS_CRT_CASE(9) HPS_CRT_CASE(10) HPS_CRT_CASE(11) HPS_CRT_CASE(12) HPS_CRT_CASE(13)
    HPS_CRT_CASE(14) HPS_CRT_CASE(15) HPS_CRT_CASE(16)
  }
#undef HPS_CRT_CASE
}

// Plan of the panel products: C_l[b] (int32, M x nc row-major) = Ares_l[b] (M x K) * Bres_l[b]^T
// rows [j0, j0 + nc) (each nc x K; consecutive (l, b) operands strideB = N K apart), all n * batch
// of them in one strided-batched call. Column-major terms: C^T (nc x M) = op_T(Bw) op_N(Aw).
static EmuPlan* crt_plan(EmuState* es, int M, int nc, int K, long long strideB, int nbatch) {
  auto key = std::make_tuple(M, nc, K, (int)(strideB / K), -nbatch);  // negative batch: CRT plans
  auto it = es->plans.find(key);
  if (it != es->plans.end()) return it->second.ok ? &it->second : nullptr;
  EmuPlan& pl = es->plans[key];
  cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
  bool ok = cublasLtMatmulDescCreate(&pl.op, CUBLAS_COMPUTE_32I, CUDA_R_32I) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&pl.a, CUDA_R_8I, K, nc, K) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&pl.b, CUDA_R_8I, K, M, K) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&pl.c, CUDA_R_32I, nc, M, nc) == CUBLAS_STATUS_SUCCESS;
  if (ok && nbatch > 1) {
    const long long sa = strideB, sb = (long long)M * K, sc = (long long)M * nc;
    ok = cublasLtMatrixLayoutSetAttribute(pl.a, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &nbatch, sizeof(nbatch)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.a, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sa, sizeof(sa)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.b, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &nbatch, sizeof(nbatch)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.b, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sb, sizeof(sb)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.c, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &nbatch, sizeof(nbatch)) == 0 &&
         cublasLtMatrixLayoutSetAttribute(pl.c, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &sc, sizeof(sc)) == 0;
  }
  if (ok) {
    cublasLtMatmulPreference_t pref = nullptr;
    ok = cublasLtMatmulPreferenceCreate(&pref) == CUBLAS_STATUS_SUCCESS;
    ok = ok && cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &es->ws_bytes,
                                                    sizeof(es->ws_bytes)) == CUBLAS_STATUS_SUCCESS;
    cublasLtMatmulHeuristicResult_t res{};
    int nres = 0;
    ok = ok && cublasLtMatmulAlgoGetHeuristic(es->lt, pl.op, pl.a, pl.b, pl.c, pl.c, pref, 1, &res, &nres) ==
                   CUBLAS_STATUS_SUCCESS && nres > 0;
    if (ok) pl.algo = res.algo;
    if (pref) cublasLtMatmulPreferenceDestroy(pref);
  }
  pl.ok = ok;
  return ok ? &pl : nullptr;
}

bool i8gemm_mod_ok(int M, int N, int nc, int K, int nmod);  // i8gemm.cu
int i8gemm_mod(const signed char* A, const signed char* B, unsigned char* R, int M, int N, int nc, int j0, int K, int nz,
               int batch, const int* moduli, int nmod, bool pair, Ctx& cx, cudaStream_t st);

static int emu_gemm_crt(const GemmParams& p, Ctx& cx, cudaStream_t st) {
  const int n = (int)cx.opt[HPS_OPT_EMU_MODULI];
  if (!emu_eligible(p, cx, true) || p.K >= (1 << 16)) return 1;  // |C_l| <= K 2^14 < 2^30
  CrtConst c;
  if (!crt_constants(n, c)) return 1;
  // output column panels: the n products of a panel fit the scratch cap; panel widths are multiples
  // of 256 (the kernel's tile width) where the cap allows
  const bool own = cx.opt[HPS_OPT_EMU_ENGINE] != 1;  // 0: tcgen05 single CTAs, 2: CTA pairs, 1: cuBLASLt
  const size_t elt = own ? 1 : sizeof(int);  // the tcgen05 kernel stores residues, cuBLASLt int32 sums
  // at most 8 GB of products: k_crt_accum indexes them with 32 bits (in units of four elements)
  const size_t cap = (size_t)std::min<long long>(8192, std::max<long long>(1, cx.opt[HPS_OPT_EMU_SCRATCH_MB])) << 20;
  const size_t per_col = (size_t)n * p.batch * p.M * elt;
  const size_t maxc = std::max<size_t>(32, cap / per_col);
  int nc;
  if (maxc >= (size_t)p.N) {
    nc = p.N;
  } else {
    const int np = (int)((p.N + maxc - 1) / maxc);
    const int q = maxc >= 256 ? 256 : 32;
    nc = std::min<int>((int)(maxc / q * q), ((p.N + np - 1) / np + q - 1) / q * q);
  }
  const bool use_own = own && i8gemm_mod_ok(p.M, p.N, nc, p.K, n) && (p.N % nc == 0 || (p.N % nc) % 32 == 0);
  const size_t per = use_own ? 1 : sizeof(int);
  const size_t a_bytes = (size_t)n * p.batch * p.M * p.K, b_bytes = (size_t)n * p.batch * p.N * p.K;
  const size_t c_bytes = (size_t)n * p.batch * p.M * nc * per;
  const size_t e_bytes = (size_t)p.batch * (p.M + p.N) * sizeof(int);
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t need = (align(a_bytes) + align(b_bytes) + align(c_bytes) + e_bytes) / sizeof(double) + 1;
  EmuState* es = use_own ? nullptr : emu_state(cx);
  if (!use_own && !es) return 1;
  double* scratch = cx.emu_scratch(need, st);
  if (!scratch) return 1;
  char* base = reinterpret_cast<char*>(scratch);
  signed char* Ar = reinterpret_cast<signed char*>(base);
  signed char* Br = reinterpret_cast<signed char*>(base + align(a_bytes));
  void* Cl = base + align(a_bytes) + align(b_bytes);
  int* sig = reinterpret_cast<int*>(reinterpret_cast<char*>(Cl) + align(c_bytes));
  int* tau = sig + (size_t)p.batch * p.M;
  const int nb = n * p.batch;
  EmuPlan *full = nullptr, *tail = nullptr;
  if (!use_own) {
    full = crt_plan(es, p.M, nc, p.K, (long long)p.N * p.K, nb);
    tail = (p.N % nc) ? crt_plan(es, p.M, p.N % nc, p.K, (long long)p.N * p.K, nb) : nullptr;
    if (!full || ((p.N % nc) && !tail)) return 1;
  }
  k_crt_row_scale<<<dim3((p.M + 7) / 8, p.batch), 256, 0, st>>>(p.A, p.lda, p.strideA, p.M, p.K, c.PA, sig);
  HPS_LAUNCH_CHECK();
  k_crt_col_scale<<<dim3((p.N + 31) / 32, p.batch), 256, 0, st>>>(p.B, p.ldb, p.strideB, p.K, p.N, c.PB, tau);
  HPS_LAUNCH_CHECK();
  // the operands' residue bytes: A rows and B columns (transposed), K-contiguous; 16-byte stores need
  // K % 16 == 0 (emu_eligible) and 256-byte aligned planes (align above)
  if (cx.opt[HPS_OPT_EMU_SPLIT] != 0) {  // integer pipes + int8 MMA (default)
    ResTab rt;
    if (!res_tab(n, rt)) return 1;
#define HPS_SPLIT_ROWS(NM)                                                                                          \
  k_crt_split_rows_mma<NM><<<dim3((p.K + 1023) / 1024, p.M, p.batch), 128, 0, st>>>(p.A, p.lda, p.strideA, p.M, p.K, \
                                                                                    p.batch, sig, rt, Ar)
    HPS_CRT_SWITCH(n, HPS_SPLIT_ROWS)
#undef HPS_SPLIT_ROWS
    HPS_LAUNCH_CHECK();
#define HPS_SPLIT_COLS(NM)                                                                                      \
  {                                                                                                             \
    const int as = ensure_smem_attr((const void*)k_crt_split_cols_mma<NM>, cx.device, ResColsSmem<NM>::kBytes); \
    if (as != HPS_OK) return as;                                                                                \
    k_crt_split_cols_mma<NM><<<dim3((p.N + 63) / 64, (p.K + 31) / 32, p.batch), 128, ResColsSmem<NM>::kBytes, st>>>( \
        p.B, p.ldb, p.strideB, p.K, p.N, p.batch, tau, rt, Br);                                                 \
  }
    HPS_CRT_SWITCH(n, HPS_SPLIT_COLS)
#undef HPS_SPLIT_COLS
    HPS_LAUNCH_CHECK();
  } else {  // FP64 pipe
#define HPS_SPLIT_ROWS(NM)                                                                                   \
  k_crt_split_rows<NM><<<dim3((p.K / 4 + 255) / 256, p.M, p.batch), 256, 0, st>>>(p.A, p.lda, p.strideA, p.M, p.K, \
                                                                                 p.batch, sig, c, Ar)
    HPS_CRT_SWITCH(n, HPS_SPLIT_ROWS)
#undef HPS_SPLIT_ROWS
    HPS_LAUNCH_CHECK();
#define HPS_SPLIT_COLS(NM)                                                                                        \
  k_crt_split_cols<NM><<<dim3((p.N + 63) / 64, (p.K + 31) / 32, p.batch), 256, 0, st>>>(p.B, p.ldb, p.strideB, p.K, \
                                                                                      p.N, p.batch, tau, c, Br)
    HPS_CRT_SWITCH(n, HPS_SPLIT_COLS)
#undef HPS_SPLIT_COLS
    HPS_LAUNCH_CHECK();
  }
  const int one = 1, zero = 0;
  for (int j0 = 0; j0 < p.N; j0 += nc) {
    const int w = std::min(nc, p.N - j0);
    if (use_own) {
      const int r = i8gemm_mod(Ar, Br, reinterpret_cast<unsigned char*>(Cl), p.M, p.N, w, j0, p.K, nb, p.batch,
                               kModuli, n, cx.opt[HPS_OPT_EMU_ENGINE] == 2, cx, st);
      if (r != HPS_OK) return r;
    } else {
      const EmuPlan* pl = w == nc ? full : tail;
      const signed char* Bw = Br + (long long)j0 * p.K;  // cuBLASLt "A": residue rows [j0, j0 + w) of B^T
      if (cublasLtMatmul(es->lt, pl->op, &one, Bw, pl->a, Ar, pl->b, &zero, Cl, pl->c, Cl, pl->c, &pl->algo, es->ws,
                         es->ws_bytes, st) != CUBLAS_STATUS_SUCCESS) {
        set_error("emu_gemm_crt: cublasLtMatmul failed (M=%d N=%d K=%d panel %d)", p.M, p.N, p.K, j0);
        return HPS_ERR_CUDA;
      }
      count_launch();
    }
    const int bx = (w / 4 + 255) / 256;
    const dim3 grid(bx, (unsigned)std::min<long long>(p.M, std::max<long long>(1, (long long)cx.sms * 16 / bx)), p.batch);
    if (use_own)
      crt_accum_launch<unsigned char>(n, grid, st, reinterpret_cast<const unsigned char*>(Cl), p.M, w, j0, p, c, sig, tau);
    else
      crt_accum_launch<int>(n, grid, st, reinterpret_cast<const int*>(Cl), p.M, w, j0, p, c, sig, tau);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

int emu_gemm(const GemmParams& p, Ctx& cx, cudaStream_t st) {
  if (cx.opt[HPS_OPT_EMU_MODULI] > 0) return emu_gemm_crt(p, cx, st);
  return emu_gemm_slices(p, cx, st);
}

}  // namespace hps
