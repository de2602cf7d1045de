// Pivoted LU of the large interface systems (n3 > 128) and the solve S = X^-1 R through it.
//
// Reference: merge.py:106-110 factors X = T33a - T33b with LAPACK getrf (partial pivoting) and
// solves with getrs. Here, for the (deflated) X of every merge at one depth, batched:
//
//   P X = L U          blocked right-looking LU, outer blocks of NB = 128 columns, inner panels of
//                      W = 16 columns. A panel pivots over the FULL remaining column (rows
//                      [c, n)), never only inside a block. The panel kernel (k_lu_panel) is one
//                      thread-block cluster per matrix: C = ceil(rows / 1024) CTAs of 1024 threads,
//                      one row per thread, the panel rows mirrored in each CTA's shared memory.
//                      Per pivot step: warp/CTA argmax, the CTA candidates exchanged through
//                      distributed shared memory under one cluster barrier, the pivot row read from
//                      its owner's shared memory, rank-1 update in registers. Rows are swapped
//                      LAPACK-style (sequential swaps, ipiv) when the panel is written back;
//                      k_swap_trsm16 applies the swaps to the other columns and solves the panel's
//                      16-row strip inside its 128-block; the 128-row strip solve U12 = L11^-1 A12
//                      is the same recursive triangular solve, the trailing updates the DMMA GEMM.
//   S = U^-1 L^-1 P R  row gather by the pivot permutation, then two recursive triangular solves
//                      in place: the bulk as DMMA GEMMs, 16-row diagonal strips by forward / back
//                      substitution in registers (k_strip16, one thread per column).
//
// Flops: 2/3 n^3 (LU) + 2 n^2 ne (two solves), against 2 n^3 + 2 n^2 ne for an explicit inverse.
#include <algorithm>

#include "common.cuh"
#include "ctx.cuh"
#include "gemm.cuh"
#include "lu.cuh"

namespace hps {

namespace lu {
constexpr int R = 1024;   // rows per CTA of the panel kernel (one per thread)
constexpr int W = 16;     // panel width
constexpr int SR = W + 1; // shared-memory row stride (doubles)
constexpr int NB = 128;   // outer block
constexpr int KEYBITS = 14;  // row index bits inside the argmax key (rows < 16384)
constexpr size_t PANEL_SMEM = sizeof(double) * (size_t)R * SR;
}  // namespace lu

__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int o) {
  unsigned lo = (unsigned)v, hi = (unsigned)(v >> 32);
  lo = __shfl_xor_sync(0xffffffffu, lo, o);
  hi = __shfl_xor_sync(0xffffffffu, hi, o);
  return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// generic address of the same shared-memory object in CTA `rank` of the cluster
template <typename T>
__device__ __forceinline__ T* map_rank(T* p, unsigned rank) {
  T* out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
  return out;
}

// One W-column panel of every matrix: rows [c0, n), columns [c0, c0 + w). grid = (C, batch),
// cluster (C, 1, 1). On exit the panel holds L (unit, below the diagonal) and U (on and above it)
// with the rows in LAPACK order, and ipiv[c0 + j] is the row swapped with c0 + j at step j.
__global__ void __launch_bounds__(lu::R, 1) k_lu_panel(double* A, int n, long long strideA, int c0, int w,
                                                    int* ipiv, int* status, int status_base) {
  extern __shared__ __align__(16) double s_rows[];  // [R][SR]
  __shared__ unsigned long long s_warp[lu::R / 32];
  __shared__ unsigned long long s_cand[2][16];      // CTA candidates (read from rank 0's copy)
  __shared__ double s_prow[lu::W];
  __shared__ int s_piv[lu::W];
  __shared__ int s_list_pos[2 * lu::W], s_list_row[2 * lu::W];
  __shared__ int s_nlist;
  const unsigned C = gridDim.x;
  const unsigned rank = C > 1 ? cluster_ctarank() : 0;
  const int b = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Ab = A + (long long)b * strideA;
  const int g = c0 + (int)rank * lu::R + tid;  // this thread's row
  const bool valid = g < n;
  double a[lu::W];
#pragma unroll
  for (int k = 0; k < lu::W; ++k) a[k] = (valid && k < w) ? Ab[(long long)g * n + c0 + k] : 0.0;
  double* myrow = s_rows + tid * lu::SR;
#pragma unroll
  for (int k = 0; k < lu::W; ++k) myrow[k] = a[k];
  bool done = false;
  bool singular = false;
#pragma unroll
  for (int j = 0; j < lu::W; ++j) {  // unrolled: a[] stays in registers
    if (j >= w) break;
    // ---- argmax |a[j]| over the active rows (ties: smallest row) ----
    unsigned long long key = 0;
    if (valid && !done) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(a[j]));
      key = (bits & ~((1ULL << lu::KEYBITS) - 1)) | (unsigned long long)((1 << lu::KEYBITS) - 1 - (g - c0));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = shfl_xor_u64(key, o);
      key = other > key ? other : key;
    }
    if (lane == 0) s_warp[warp] = key;
    __syncthreads();
    if (warp == 0) {
      unsigned long long k2 = s_warp[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = shfl_xor_u64(k2, o);
        k2 = other > k2 ? other : k2;
      }
      if (lane == 0) {
        if (C > 1)
          *map_rank(&s_cand[j & 1][rank], 0u) = k2;  // publish this CTA's candidate at rank 0
        else
          s_cand[j & 1][0] = k2;
      }
    }
    if (C > 1) cluster_sync_all();
    else __syncthreads();
    // ---- every CTA picks the winner and fetches the pivot row from its owner ----
    if (warp == 0) {
      unsigned long long best = 0;
      if (lane < (int)C) best = C > 1 ? *map_rank(&s_cand[j & 1][lane], 0u) : s_cand[j & 1][0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = shfl_xor_u64(best, o);
        best = other > best ? other : best;
      }
      const int prow = c0 + (1 << lu::KEYBITS) - 1 - (int)(best & ((1ULL << lu::KEYBITS) - 1));
      const unsigned owner = (unsigned)((prow - c0) / lu::R);
      const int local = (prow - c0) - (int)owner * lu::R;
      const double* src = s_rows + local * lu::SR;
      if (C > 1 && owner != rank) src = map_rank(src, owner);
      if (lane < lu::W) s_prow[lane] = (lane < w) ? src[lane] : 0.0;
      if (lane == 0) s_piv[j] = (best >> lu::KEYBITS) == 0 ? -1 - prow : prow;  // < 0: zero pivot column
    }
    __syncthreads();
    int p = s_piv[j];
    if (p < 0) {
      singular = true;
      p = -1 - p;
    }
    if (g == p) done = true;
    if (valid && !done) {
      const double piv = s_prow[j];
      const double l = p == s_piv[j] ? a[j] / piv : 0.0;
      a[j] = l;
      myrow[j] = l;
#pragma unroll
      for (int k = 0; k < lu::W; ++k)
        if (k > j && k < w) {
          a[k] = fma(-l, s_prow[k], a[k]);
          myrow[k] = a[k];
        }
    }
  }
  // ---- LAPACK-order write-back: emulate the sequential swaps (one thread per CTA, same result) ----
  if (tid == 0) {
    int nl = 0;
    for (int j = 0; j < w; ++j) {
      int p = s_piv[j];
      if (p < 0) p = -1 - p;
      const int t = c0 + j;
      int pp = p;  // current position of original row p
      for (int k = 0; k < nl; ++k)
        if (s_list_row[k] == p) pp = s_list_pos[k];
      int rt = t;  // original row now at position t
      int kt = -1, kp = -1;
      for (int k = 0; k < nl; ++k) {
        if (s_list_pos[k] == t) {
          rt = s_list_row[k];
          kt = k;
        }
        if (s_list_pos[k] == pp) kp = k;
      }
      if (kt < 0) {
        kt = nl++;
        s_list_pos[kt] = t;
      }
      s_list_row[kt] = p;
      if (pp != t) {
        if (kp < 0) {
          kp = nl++;
          s_list_pos[kp] = pp;
        }
        s_list_row[kp] = rt;
      }
      if (rank == 0) ipiv[(long long)b * n + t] = pp;
    }
    s_nlist = nl;
    if (singular && status && rank == 0) atomicMax(status, status_base + b);
  }
  __syncthreads();
  if (valid) {
    int dst = g;
    for (int k = 0; k < s_nlist; ++k)
      if (s_list_row[k] == g) dst = s_list_pos[k];
#pragma unroll
    for (int k = 0; k < lu::W; ++k)
      if (k < w) Ab[(long long)dst * n + c0 + k] = a[k];
  }
  if (C > 1) cluster_sync_all();  // no CTA leaves while another may still read its shared memory
}

// For every column outside the panel [c0, c0 + w): the panel's row swaps (ipiv[c0 .. c0 + w)).
// Columns in [c0 + w, tend) then get the strip solve U12 = L11^-1 A12 of the panel's w rows.
// One thread per column; grid = (ceil(n / 128), batch).
__global__ void __launch_bounds__(128) k_swap_trsm16(double* A, int n, long long strideA, int c0, int w,
                                                    const int* __restrict__ ipiv, int tend) {
  __shared__ double sL[lu::W][lu::W];
  __shared__ int sp[lu::W];
  const int b = blockIdx.y;
  double* Ab = A + (long long)b * strideA;
  for (int i = threadIdx.x; i < lu::W * lu::W; i += blockDim.x) {
    const int r = i / lu::W, c = i % lu::W;
    sL[r][c] = (r < w && c < w) ? Ab[(long long)(c0 + r) * n + c0 + c] : 0.0;
  }
  if (threadIdx.x < lu::W) sp[threadIdx.x] = threadIdx.x < w ? ipiv[(long long)b * n + c0 + threadIdx.x] : 0;
  __syncthreads();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n || (col >= c0 && col < c0 + w)) return;
  for (int j = 0; j < w; ++j) {
    const int r1 = c0 + j, r2 = sp[j];
    if (r2 != r1) {
      double* p1 = Ab + (long long)r1 * n + col;
      double* p2 = Ab + (long long)r2 * n + col;
      const double t = *p1;
      *p1 = *p2;
      *p2 = t;
    }
  }
  if (col >= c0 + w && col < tend) {
    double x[lu::W];
#pragma unroll
    for (int r = 0; r < lu::W; ++r) x[r] = r < w ? Ab[(long long)(c0 + r) * n + col] : 0.0;
#pragma unroll
    for (int r = 1; r < lu::W; ++r) {
      double s = x[r];
#pragma unroll
      for (int k = 0; k < lu::W; ++k)
        if (k < r) s = fma(-sL[r][k], x[k], s);
      x[r] = s;
    }
#pragma unroll
    for (int r = 0; r < lu::W; ++r)
      if (r < w) Ab[(long long)(c0 + r) * n + col] = x[r];
  }
}

// Strip solve with a diagonal block of the LU factors: the w-row strip B (w <= 16, columns
// [0, ncols); B points at its first row) <- T^-1 B, T = X[r0 : r0 + w, r0 : r0 + w], unit lower
// (LOWER) or upper. One thread per column, the strip column and T in registers / shared memory.
template <bool LOWER>
__global__ void __launch_bounds__(128) k_strip16(const double* __restrict__ X, int n, long long strideX, int r0, int w,
                                                double* __restrict__ B, long long ldb, long long strideB, int ncols) {
  __shared__ double sT[lu::W][lu::W + 1];
  const int b = blockIdx.y;
  const double* T = X + (long long)b * strideX + (long long)r0 * n + r0;
  for (int i = threadIdx.x; i < lu::W * lu::W; i += blockDim.x) {
    const int r = i / lu::W, c = i % lu::W;
    sT[r][c] = (r < w && c < w) ? T[(long long)r * n + c] : (r == c ? 1.0 : 0.0);
  }
  __syncthreads();
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= ncols) return;
  double* Bb = B + (long long)b * strideB + col;
  double x[lu::W];
#pragma unroll
  for (int r = 0; r < lu::W; ++r) x[r] = r < w ? Bb[(long long)r * ldb] : 0.0;
  if (LOWER) {
#pragma unroll
    for (int r = 1; r < lu::W; ++r) {
      double s = x[r];
#pragma unroll
      for (int k = 0; k < r; ++k) s = fma(-sT[r][k], x[k], s);
      x[r] = s;
    }
  } else {
#pragma unroll
    for (int r = lu::W - 1; r >= 0; --r) {
      double s = x[r];
#pragma unroll
      for (int k = r + 1; k < lu::W; ++k) s = fma(-sT[r][k], x[k], s);
      x[r] = s / sT[r][r];
    }
  }
#pragma unroll
  for (int r = 0; r < lu::W; ++r)
    if (r < w) Bb[(long long)r * ldb] = x[r];
}

// perm[i] = original row that ends at position i after the sequential swaps ipiv (one thread per
// matrix: n steps).
__global__ void k_ipiv_to_perm(const int* __restrict__ ipiv, int n, int* __restrict__ perm) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  int* pm = perm + (long long)b * n;
  const int* ip = ipiv + (long long)b * n;
  for (int i = 0; i < n; ++i) pm[i] = i;
  for (int i = 0; i < n; ++i) {
    const int r = ip[i];
    if (r != i) {
      const int t = pm[i];
      pm[i] = pm[r];
      pm[r] = t;
    }
  }
}

// dst[b][i][:] = src[b][perm[b][i]][:] (ne columns), one warp per row.
__global__ void k_permute_rows(const double* __restrict__ src, long long strideS, const int* __restrict__ perm,
                               int n, int ne, double* __restrict__ dst, long long strideD) {
  const int b = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= n) return;
  const double* s = src + (long long)b * strideS + (long long)perm[(long long)b * n + r] * ne;
  double* d = dst + (long long)b * strideD + (long long)r * ne;
  for (int c = lane; c < ne; c += 32) d[c] = s[c];
}

static int gemm(Ctx& cx, int M, int N, int K, int batch, double alpha, const double* A, long long lda, long long sA,
                const double* B, long long ldb, long long sB, double beta, double* C, long long ldc, long long sC,
                cudaStream_t st, int* nonfinite = nullptr) {
  GemmParams p{M, N, K, batch, A, lda, sA, B, ldb, sB, nullptr, 0, C, ldc, sC, alpha, beta, nonfinite};
  return dgemm_launch(p, cx, st);
}

#define LU_TRY(x)                  \
  do {                             \
    int _s = (x);                  \
    if (_s != HPS_OK) return _s;   \
  } while (0)

LuWs lu_ws(void* base, int n, int batch) {
  LuWs w;
  int* ip = static_cast<int*>(base);
  w.ipiv = ip;
  w.perm = ip + (size_t)batch * n;
  return w;
}

size_t lu_ws_bytes(int n, int batch) { return sizeof(int) * 2 * (size_t)batch * n + 64; }

// B (w rows of ncols, row stride ldb, batch stride sB) <- T^-1 B for T = X[r0 : r0 + w, r0 : r0 + w]
// (unit lower or upper), recursively: the bulk as DMMA GEMMs, 16-row strips by k_strip16.
static int trsm(Ctx& cx, bool lower, const double* X, int n, int batch, int r0, int w, double* B, long long ldb,
                long long sB, int ncols, cudaStream_t st) {
  if (w <= 0 || ncols <= 0) return HPS_OK;
  const long long sX = (long long)n * n;
  if (w <= lu::W) {
    if (lower)
      k_strip16<true><<<dim3((ncols + 127) / 128, batch), 128, 0, st>>>(X, n, sX, r0, w, B, ldb, sB, ncols);
    else
      k_strip16<false><<<dim3((ncols + 127) / 128, batch), 128, 0, st>>>(X, n, sX, r0, w, B, ldb, sB, ncols);
    HPS_LAUNCH_CHECK();
    return HPS_OK;
  }
  const int nb = (w + lu::W - 1) / lu::W;
  const int h = ((nb + 1) / 2) * lu::W;
  double* B2 = B + (long long)h * ldb;
  if (lower) {
    LU_TRY(trsm(cx, true, X, n, batch, r0, h, B, ldb, sB, ncols, st));
    LU_TRY(gemm(cx, w - h, ncols, h, batch, -1.0, X + (long long)(r0 + h) * n + r0, n, sX, B, ldb, sB, 1.0, B2, ldb,
                sB, st));
    return trsm(cx, true, X, n, batch, r0 + h, w - h, B2, ldb, sB, ncols, st);
  }
  LU_TRY(trsm(cx, false, X, n, batch, r0 + h, w - h, B2, ldb, sB, ncols, st));
  LU_TRY(gemm(cx, h, ncols, w - h, batch, -1.0, X + (long long)r0 * n + r0 + h, n, sX, B2, ldb, sB, 1.0, B, ldb, sB,
              st));
  return trsm(cx, false, X, n, batch, r0, h, B, ldb, sB, ncols, st);
}

static int launch_panel(Ctx& cx, double* X, int n, int batch, int c0, int w, int* ipiv, int* status,
                        int status_base, cudaStream_t st) {
  const int rows = n - c0;
  const int C = (rows + lu::R - 1) / lu::R;
  if (C > 16) {
    set_error("lu: interface of %d rows exceeds the panel kernel (16 CTAs x %d rows)", rows, lu::R);
    return HPS_ERR_ARG;
  }
  LU_TRY(ensure_smem_attr((const void*)k_lu_panel, cx.device, (int)lu::PANEL_SMEM));
  if (C > 8) {
    static bool np_set[16] = {};
    if (!np_set[cx.device & 15]) {
      HPS_CUDA_CHECK(cudaFuncSetAttribute(k_lu_panel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      np_set[cx.device & 15] = true;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)C, (unsigned)batch, 1);
  cfg.blockDim = dim3(lu::R, 1, 1);
  cfg.dynamicSmemBytes = lu::PANEL_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HPS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_lu_panel, X, n, (long long)n * n, c0, w, ipiv, status, status_base));
  count_launch();
  return HPS_OK;
}

// P X = L U in place for `batch` n x n matrices (stride n^2); ipiv / perm in ws.
int lu_factor(Ctx& cx, double* X, int n, int batch, const LuWs& ws, int* status, int status_base, cudaStream_t st) {
  const long long sX = (long long)n * n;
  for (int c = 0; c < n; c += lu::NB) {
    const int bw = std::min(lu::NB, n - c);
    for (int cc = c; cc < c + bw; cc += lu::W) {
      const int w = std::min(lu::W, c + bw - cc);
      LU_TRY(launch_panel(cx, X, n, batch, cc, w, ws.ipiv, status, status_base, st));
      k_swap_trsm16<<<dim3((n + 127) / 128, batch), 128, 0, st>>>(X, n, sX, cc, w, ws.ipiv, c + bw);
      HPS_LAUNCH_CHECK();
      const int rest = c + bw - cc - w;
      if (rest > 0 && n - cc - w > 0)
        LU_TRY(gemm(cx, n - cc - w, rest, w, batch, -1.0, X + (long long)(cc + w) * n + cc, n, sX,
                    X + (long long)cc * n + cc + w, n, sX, 1.0, X + (long long)(cc + w) * n + cc + w, n, sX, st));
    }
    const int right = n - c - bw;
    if (right > 0) {
      // U12 = L11^-1 A12, then the rank-bw update of the trailing matrix
      double* A12 = X + (long long)c * n + c + bw;
      LU_TRY(trsm(cx, true, X, n, batch, c, bw, A12, n, sX, right, st));
      LU_TRY(gemm(cx, right, right, bw, batch, -1.0, X + (long long)(c + bw) * n + c, n, sX, A12, n, sX, 1.0,
                  X + (long long)(c + bw) * n + c + bw, n, sX, st));
    }
  }
  k_ipiv_to_perm<<<batch, 32, 0, st>>>(ws.ipiv, n, ws.perm);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

__global__ void k_nonfinite_rows(const double* __restrict__ S, long long per, int* status, int status_base) {
  const int b = blockIdx.y;
  const double* Sb = S + (long long)b * per;
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per; i += (long long)gridDim.x * blockDim.x)
    bad |= !isfinite(Sb[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicMax(status, status_base + b);
}

// S = U^-1 L^-1 P R for the factored X (lu_factor), all matrices of the batch. R: n x ne per
// matrix (read only); S_out: n x ne per matrix. status flags a non-finite S (MergeResonanceError).
int lu_solve(Ctx& cx, const double* X, int n, int batch, const LuWs& ws, const double* R, int ne, double* S_out,
             int* status, int status_base, cudaStream_t st) {
  const long long sB = (long long)n * ne;
  k_permute_rows<<<dim3((n + 7) / 8, batch), 256, 0, st>>>(R, sB, ws.perm, n, ne, S_out, sB);
  HPS_LAUNCH_CHECK();
  LU_TRY(trsm(cx, true, X, n, batch, 0, n, S_out, ne, sB, ne, st));
  LU_TRY(trsm(cx, false, X, n, batch, 0, n, S_out, ne, sB, ne, st));
  if (status) {
    k_nonfinite_rows<<<dim3((unsigned)std::min<long long>(cx.sms, (sB + 255) / 256), batch), 256, 0, st>>>(
        S_out, sB, status, status_base);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

}  // namespace hps

using namespace hps;

// Test hook: LU-factor `batch` n x n matrices in place (X) and solve X S = R (S written to S_out).
extern "C" size_t hps_lu_workspace_bytes(int n, int batch) { return lu_ws_bytes(n, batch); }

extern "C" int hps_lu_solve_batched(hps_ctx_t ctx, int n, int ne, int batch, double* X, const double* R,
                                    double* S_out, int* ipiv_out, void* ws, size_t ws_bytes, int* status,
                                    void* stream) {
  HPS_CTX(cx, ctx);
  if (n <= 0 || ne <= 0 || batch <= 0 || ws_bytes < lu_ws_bytes(n, batch)) {
    set_error("hps_lu_solve_batched: bad arguments n=%d ne=%d ws=%zu", n, ne, ws_bytes);
    return HPS_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LuWs w = lu_ws(ws, n, batch);
  LU_TRY(lu_factor(*cx, X, n, batch, w, status, 0, st));
  LU_TRY(lu_solve(*cx, X, n, batch, w, R, ne, S_out, status, 0, st));
  if (ipiv_out)
    HPS_CUDA_CHECK(cudaMemcpyAsync(ipiv_out, w.ipiv, sizeof(int) * (size_t)n * batch, cudaMemcpyDeviceToDevice, st));
  return HPS_OK;
}
