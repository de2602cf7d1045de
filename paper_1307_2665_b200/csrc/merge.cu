// Level-batched DtN merge (reference merge.py:92-119), B200 design:
//
//   X  = Ta[j3a,j3a] - Tb[j3b,j3b]                 (gather, HBM-bound)
//   Xd = X + sigma * V V^T                          (deflate the analytic corner null modes)
//   Xi = Xd^{-1}                                    (in-smem Gauss-Jordan for n3 <= 128, else
//                                                    recursive 2x2 block inverse on DMMA GEMMs)
//   S  = Xi [-Ta[j3a,j1a] | Tb[j3b,j2b]]            (DMMA GEMM)
//   T  = blkdiag(Ta[j1a,j1a], Tb[j2b,j2b]) + [Ta[j1a,j3a]; Tb[j2b,j3b]] S   (DMMA GEMM, beta = 1)
//
// Why deflate: with the reference's corner-averaged L1 (leafops.py:143-179), X is exactly singular
// at every depth <= 2L-2. Its null space is known in closed form: one
// vector per interior vertex on the cut line. On the two segments meeting at the vertex the
// vector holds the Chebyshev-endpoint Lagrange polynomial sampled at the Gauss nodes. Both
// X V = 0 and [Ta13; Tb23] V = 0, so any solution of X S = R gives the same parent T. Adding
// sigma V V^T makes the system nonsingular and well conditioned (cond 1e2..1e3 measured). Its
// solution is the particular S with V^T S = 0. That S is reproducible, while the reference's raw
// S is rounding noise along V. T matches the reference (parity-gated in tests/).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "ctx.cuh"
#include "gemm.cuh"
#include "lu.cuh"

namespace hps {

// ---------------------------------------------------------------------------------------------
// Gathers: one warp per output row, lanes over columns (maps come in runs of q -> coalesced).
// ---------------------------------------------------------------------------------------------
// ChildRef (children of merge b) lives in gemm.cuh: the T GEMM epilogue reads the blkdiag through it.

// dst[c] = sign * src[map[c]] for c < n by one warp: 4 elements per lane per step, all index loads
// before the value loads (independent loads in flight together instead of load -> load chains)
__device__ __forceinline__ void warp_gather(double* __restrict__ dst, const double* __restrict__ src,
                                            const int* __restrict__ map, int n, double sign, int lane) {
  int c = lane;
  for (; c + 96 < n; c += 128) {
    const int i0 = __ldg(map + c), i1 = __ldg(map + c + 32), i2 = __ldg(map + c + 64), i3 = __ldg(map + c + 96);
    const double v0 = src[i0], v1 = src[i1], v2 = src[i2], v3 = src[i3];
    dst[c] = sign * v0;
    dst[c + 32] = sign * v1;
    dst[c + 64] = sign * v2;
    dst[c + 96] = sign * v3;
  }
  for (; c < n; c += 32) dst[c] = sign * src[__ldg(map + c)];
}

__global__ void k_gather_xr(ChildRef ch, const int* __restrict__ j1a, const int* __restrict__ j2b,
                            const int* __restrict__ j3a, const int* __restrict__ j3b, int n3, int ne,
                            double* __restrict__ X, double* __restrict__ R,
                            unsigned long long* __restrict__ diagmax) {
  const int b = blockIdx.x;
  const int r = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= n3) return;
  const int n1 = ne / 2;
  const double* Ta = ch.a(b) + (long long)j3a[r] * ch.m;
  const double* Tb = ch.bb(b) + (long long)j3b[r] * ch.m;
  double* Xr = X ? X + ((long long)b * n3 + r) * n3 : nullptr;
  double* Rr = R + ((long long)b * n3 + r) * ne;
  if (X) for (int c = lane; c < n3; c += 32) {  // X == nullptr: precomputed (look-ahead), R only
    const double v = Ta[j3a[c]] - Tb[j3b[c]];
    Xr[c] = v;
    // max |diag X| for the deflation shift: non-negative doubles order like their bit patterns,
    // so an integer atomicMax is exact and independent of the CTA order
    if (c == r && diagmax) atomicMax(diagmax + b, (unsigned long long)__double_as_longlong(fabs(v)));
  }
  warp_gather(Rr, Ta, j1a, n1, -1.0, lane);
  warp_gather(Rr + n1, Tb, j2b, n1, 1.0, lane);
}

// C[b] (ne x n3), one warp per row (n3 >= 32)
__global__ void k_gather_c_rows(ChildRef ch, const int* __restrict__ j1a, const int* __restrict__ j2b,
                                const int* __restrict__ j3a, const int* __restrict__ j3b, int n3, int ne,
                                double* __restrict__ Cm) {
  const int b = blockIdx.x;
  const int r = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= ne) return;
  const int n1 = ne / 2;
  const bool top = r < n1;
  const double* src = top ? ch.a(b) + (long long)j1a[r] * ch.m : ch.bb(b) + (long long)j2b[r - n1] * ch.m;
  warp_gather(Cm + ((long long)b * ne + r) * n3, src, top ? j3a : j3b, n3, 1.0, lane);
}

// C[b] (ne x n3), element-parallel (one thread per 4 entries, 256-entry strides), for narrow rows
// (n3 = 16 at the leaf pairs would leave half of every row warp idle); measured faster below 32
// columns, slower above
__global__ void k_gather_c(ChildRef ch, const int* __restrict__ j1a, const int* __restrict__ j2b,
                           const int* __restrict__ j3a, const int* __restrict__ j3b, int n3, int ne,
                           double* __restrict__ Cm) {
  const int b = blockIdx.x;
  const int n1 = ne / 2;
  const long long total = (long long)ne * n3;
  const double* Ta = ch.a(b);
  const double* Tb = ch.bb(b);
  double* Cb = Cm + (long long)b * total;
  for (long long e0 = (long long)blockIdx.y * 1024 + threadIdx.x; e0 < total; e0 += (long long)gridDim.y * 1024) {
    long long src[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {  // all index loads first
      const long long e = e0 + 256 * k;
      src[k] = -1;
      if (e < total) {
        const int r = (int)(e / n3), c = (int)(e - (long long)r * n3);
        src[k] = r < n1 ? (long long)__ldg(j1a + r) * ch.m + __ldg(j3a + c)
                        : (long long)__ldg(j2b + r - n1) * ch.m + __ldg(j3b + c);
      }
    }
    double v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long e = e0 + 256 * k;
      v[k] = src[k] >= 0 ? ((int)(e / n3) < n1 ? Ta : Tb)[src[k]] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (src[k] >= 0) Cb[e0 + 256 * k] = v[k];
  }
}


// ---------------------------------------------------------------------------------------------
// Look-ahead of the parent's interface matrix (hps_merge_level_ahead). While depth d+1 still has
// its big T GEMM to run, the parent depth's X = Ta[pj3a, pj3a] - Tb[pj3b, pj3b] only needs the
// pj3 rows and columns of the two children, T = blk + C S:
//   X = (blk_a - blk_b)[pj3, pj3] + [Ca[pj3a, :] | -Cb[pj3b, :]] [Sa[:, pj3a]; Sb[:, pj3b]],
// one GEMM with K = 2 n3 over gathered operands. The parent's deflation and inverse then run on a
// high-priority stream beside the T GEMM.
// ---------------------------------------------------------------------------------------------
// One warp per parent row r: Ag[b][r] = [Cm[2b][pj3a[r]] | -Cm[2b+1][pj3b[r]]] and
// X[b][r][c] = blk_2b(pj3a[r], pj3a[c]) - blk_2b+1(pj3b[r], pj3b[c]).
__global__ void k_ahead_rows(ChildRef ch, const int* __restrict__ j1a, const int* __restrict__ j2b, int n3, int ne,
                             const double* __restrict__ Cm, const int* __restrict__ pj3a,
                             const int* __restrict__ pj3b, int pn3, double* __restrict__ Ag, double* __restrict__ X) {
  const int b = blockIdx.x;
  const int r = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= pn3) return;
  const int n1 = ne / 2, ia = pj3a[r], ib = pj3b[r];
  const double* Ca = Cm + ((long long)(2 * b) * ne + ia) * n3;
  const double* Cb = Cm + ((long long)(2 * b + 1) * ne + ib) * n3;
  double* Ar = Ag + ((long long)b * pn3 + r) * (2 * n3);
  for (int k = lane; k < n3; k += 32) {
    Ar[k] = Ca[k];
    Ar[n3 + k] = -Cb[k];
  }
  // X row: the block-diagonal addends of the two children (zero off their diagonal blocks). The
  // row half (j1a / j2b side) of ia and ib is fixed per row, so only the column maps vary.
  double* Xr = X + ((long long)b * pn3 + r) * pn3;
  const bool ta = ia < n1, tb = ib < n1;
  const double* rowa = (ta ? ch.a(2 * b) : ch.bb(2 * b)) + (long long)(ta ? j1a[ia] : j2b[ia - n1]) * ch.m;
  const double* rowb = (tb ? ch.a(2 * b + 1) : ch.bb(2 * b + 1)) + (long long)(tb ? j1a[ib] : j2b[ib - n1]) * ch.m;
  auto colmap = [&](int j, bool top) { return (j < n1) == top ? (top ? j1a[j] : j2b[j - n1]) : -1; };
  int c = lane;
  for (; c + 32 < pn3; c += 64) {
    const int ja0 = __ldg(pj3a + c), jb0 = __ldg(pj3b + c), ja1 = __ldg(pj3a + c + 32), jb1 = __ldg(pj3b + c + 32);
    const int ma0 = colmap(ja0, ta), mb0 = colmap(jb0, tb), ma1 = colmap(ja1, ta), mb1 = colmap(jb1, tb);
    const double a0 = ma0 >= 0 ? rowa[ma0] : 0.0, b0 = mb0 >= 0 ? rowb[mb0] : 0.0;
    const double a1 = ma1 >= 0 ? rowa[ma1] : 0.0, b1 = mb1 >= 0 ? rowb[mb1] : 0.0;
    Xr[c] = a0 - b0;
    Xr[c + 32] = a1 - b1;
  }
  for (; c < pn3; c += 32) {
    const int ma = colmap(pj3a[c], ta), mb = colmap(pj3b[c], tb);
    Xr[c] = (ma >= 0 ? rowa[ma] : 0.0) - (mb >= 0 ? rowb[mb] : 0.0);
  }
}

// One warp per row k of Bg[b] (2 n3 x pn3): S[2b][k][pj3a[c]] (k < n3), S[2b+1][k - n3][pj3b[c]].
__global__ void k_ahead_bg(const double* __restrict__ S, int n3, int ne, const int* __restrict__ pj3a,
                           const int* __restrict__ pj3b, int pn3, double* __restrict__ Bg) {
  const int b = blockIdx.x;
  const int k = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (k >= 2 * n3) return;
  const bool top = k < n3;
  const double* Sr = S + ((long long)(2 * b + (top ? 0 : 1)) * n3 + (top ? k : k - n3)) * ne;
  const int* map = top ? pj3a : pj3b;
  double* Br = Bg + ((long long)b * 2 * n3 + k) * pn3;
  for (int c = lane; c < pn3; c += 32) Br[c] = Sr[map[c]];
}

// max |diag X| per matrix (the deflation shift), as the exact integer max of the bit patterns.
__global__ void k_diagmax(const double* __restrict__ X, int n, unsigned long long* __restrict__ diagmax) {
  const int b = blockIdx.x;
  unsigned long long m = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long v = (unsigned long long)__double_as_longlong(fabs(X[((long long)b * n + i) * n + i]));
    m = v > m ? v : m;
  }
  atomicMax(diagmax + b, m);
}

// Corner-mode projector entry (V V^T)[r][c] for an interface of n = nseg * q nodes.
__device__ __forceinline__ double vvt(int r, int c, int q, int nseg, const double* vs, const double* ve) {
  int sr = r / q, sc = c / q, lr = r - sr * q, lc = c - sc * q;
  if (sr == sc) {
    double v = 0.0;
    if (sr >= 1) v += vs[lr] * vs[lc];
    if (sr <= nseg - 2) v += ve[lr] * ve[lc];
    return v;
  }
  if (sc == sr + 1) return ve[lr] * vs[lc];
  if (sr == sc + 1) return vs[lr] * ve[lc];
  return 0.0;
}

// Blocked Gauss-Jordan inverse (n <= 8*NT) with partial pivoting (ties to the smallest row; implicit
// row order: row p_k is eliminated at step k and inv(X)[k][p_j] = B[p_k][j] in the in-place result
// B, the write-out applies that permutation), built for a short critical path:
//  * the matrix lives in registers in DMMA C-fragment layout: warp w owns columns 16w..16w+15,
//    lane (g, tq) holds a[r][c][h] = A(8r + g, 16w + 8c + 2tq + h);
//  * pivots go in blocks of 8 (one 8-column tile). The warp owning the tile factors it alone
//    (REDUX argmax, shuffles, no CTA barrier). A block of GJ steps acts on every other column as
//    I + W E_P^T, with W = (panel after the block) - E_P (E_P: unit vectors at the 8 pivot rows);
//  * every other tile then takes A += W A[P, :] on DMMA (k = 8: two m8n8k4 k-steps);
//  * look-ahead: the owner of the next tile updates that tile first and factors it while the
//    other warps run their updates, so one __syncthreads per 8 pivots.
// Sizes that are not a multiple of 8 are padded with identity rows/columns.
#ifdef HPS_GJ_PROFILE
__device__ long long g_gj_prof[8];
extern "C" int hps_debug_gj_profile(long long* out, int reset) {
  if (reset) {
    long long z[8] = {};
    cudaMemcpyToSymbol(g_gj_prof, z, sizeof(z));
    return 0;
  }
  cudaMemcpyFromSymbol(out, g_gj_prof, sizeof(long long) * 8);
  return 0;
}
#endif
template <int NT>
__global__ void __launch_bounds__(NT * 16) k_gj_blk(double* X, long long lda, long long strideX, int n, int* status,
                                                   int status_base) {
  constexpr int NM = 8 * NT, W = NT / 2, RPL = NM / 32 > 0 ? NM / 32 : 1;
  static_assert(NT % 2 == 0 && W >= 1 && NM <= 128, "NT (row index must fit in 7 bits)");
  __shared__ double sW[2][NM][9];     // panel of the current / next block after its 8 GJ steps
  __shared__ int sP[2][8];            // pivot rows of the block
  __shared__ double sAP[W][8][17];    // per warp: A[P, its 16 columns] before the block update
  __shared__ double sDum[10];         // store sink for lanes that do not hold a staged row (never read)
  __shared__ unsigned sCand[4][2];    // multi-warp panel: each warp's (hi, lo) argmax candidate
  __shared__ __align__(16) double sRowP[2][8];  // 2-warp panel: the pivot row (by pivot parity)
  __shared__ unsigned char usedrow[NM];
  __shared__ int pivrow[NM], rowstep[NM];
  __shared__ int s_sing;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, tq = lane & 3;
  double* Xb = X + (long long)blockIdx.x * strideX;
  double a[NT][2][2];
#pragma unroll
  for (int r = 0; r < NT; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int R = 8 * r + g, C = 16 * warp + 8 * c + 2 * tq + h;
        a[r][c][h] = (R < n && C < n) ? Xb[(long long)R * lda + C] : (R == C ? 1.0 : 0.0);
      }
  for (int i = threadIdx.x; i < NM; i += blockDim.x) usedrow[i] = 0;
  if (threadIdx.x == 0) s_sing = 0;

  // Factor the 8 columns of my tile C (block kb) with 8 sequential GJ steps, one warp, row layout:
  // the tile goes through shared memory so lane l holds rows l + 32i, all 8 columns.
  auto panel = [&](auto cc, int kb) {
    constexpr int C = decltype(cc)::value;
    double(*Pb)[9] = sW[kb & 1];
#pragma unroll
    for (int r = 0; r < NT; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) Pb[8 * r + g][2 * tq + h] = a[r][C][h];
    __syncwarp();
    double pr[RPL][8];
    bool used[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int R = lane + 32 * i;
      used[i] = R >= NM || usedrow[R];
#pragma unroll
      for (int j = 0; j < 8; ++j) pr[i][j] = R < NM ? Pb[R][j] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      // argmax |x| over the unused rows with two REDUX: the high word of |x| exactly, then the low
      // word with its 7 lowest mantissa bits replaced by (127 - row), so the smallest row wins
      // exact ties (and ties within 2^-45 relative). 2 REDUX instead of 3 (tools/microbench/
      // panel_ablate.cu: 628 vs 760 cycles per pivot).
      unsigned bh = 0u, bl = 0u;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const unsigned long long kb = used[i] ? 0ull : (unsigned long long)__double_as_longlong(fabs(pr[i][t]));
        const unsigned h = (unsigned)(kb >> 32);
        const unsigned l = used[i] ? 0u : ((((unsigned)kb) & ~127u) | (127u - (unsigned)(lane + 32 * i)));
        if (h > bh || (h == bh && l > bl)) { bh = h; bl = l; }
      }
      const unsigned mh = __reduce_max_sync(0xffffffffu, bh);
      const unsigned ml = __reduce_max_sync(0xffffffffu, bh == mh ? bl : 0u);
      const int p = 127 - (int)(ml & 127u);
      const int pl = p & 31, pi = p >> 5;
      double rp[8];
#pragma unroll
      for (int i = 0; i < RPL; ++i)
        if (pi == i) {  // warp-uniform
          if (lane == pl) used[i] = true;
#pragma unroll
          for (int j = 0; j < 8; ++j) rp[j] = __shfl_sync(0xffffffffu, pr[i][j], pl);
        }
      const double piv = rp[t];
      const double inv = fast_rcp(piv);
#pragma unroll
      for (int j = 0; j < 8; ++j) rp[j] = j == t ? inv : rp[j] * inv;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const double f = pr[i][t];
        pr[i][t] = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) pr[i][j] = fma(-f, rp[j], pr[i][j]);
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const bool mine = pi == i && lane == pl;
#pragma unroll
        for (int j = 0; j < 8; ++j) pr[i][j] = mine ? rp[j] : pr[i][j];
      }
      if (lane == 0) {
        sP[kb & 1][t] = p;
        usedrow[p] = 1;
        pivrow[8 * kb + t] = p;
        rowstep[p] = 8 * kb + t;
        if (piv == 0.0) s_sing = 1;
      }
    }
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int R = lane + 32 * i;
      if (R < NM)
#pragma unroll
        for (int j = 0; j < 8; ++j) Pb[R][j] = pr[i][j];
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < NT; ++r)
#pragma unroll
      for (int h = 0; h < 2; ++h) a[r][C][h] = Pb[8 * r + g][2 * tq + h];
  };
  // Multi-warp panel (n > 32): the tile's owner (role 0) and PW - 1 helper warps (roles 1.., the
  // other warps of the owner's aligned group of PW) factor the 8 columns together, NM / (32 PW)
  // rows per lane. Per pivot: a 2-REDUX argmax in each warp, the candidates exchanged through
  // shared memory (named barrier over the PW warps), the pivot row published by its lane (second
  // barrier).
  constexpr int PW = NT >= 16 ? 4 : 2;
  constexpr int BAR_PANEL2 = 1, HALF = NM / PW, RPL2 = NM >= 32 * PW ? NM / (32 * PW) : 1;
  auto panel2 = [&](auto cc, int kb, int role) {
    constexpr int C = decltype(cc)::value;
    double(*Pb)[9] = sW[kb & 1];
    if (role == 0) {
#pragma unroll
      for (int r = 0; r < NT; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) Pb[8 * r + g][2 * tq + h] = a[r][C][h];
    }
    bar_sync(BAR_PANEL2, 32 * PW);
    double pr[RPL2][8];
    bool used[RPL2];
#pragma unroll
    for (int i = 0; i < RPL2; ++i) {
      const int R = role * HALF + lane + 32 * i;
      used[i] = usedrow[R];
#pragma unroll
      for (int j = 0; j < 8; ++j) pr[i][j] = Pb[R][j];
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      unsigned bh = 0u, bl = 0u;
#pragma unroll
      for (int i = 0; i < RPL2; ++i) {
        const int R = role * HALF + lane + 32 * i;
        const unsigned long long kb2 = used[i] ? 0ull : (unsigned long long)__double_as_longlong(fabs(pr[i][t]));
        const unsigned h = (unsigned)(kb2 >> 32);
        const unsigned l = used[i] ? 0u : ((((unsigned)kb2) & ~127u) | (127u - (unsigned)R));
        if (h > bh || (h == bh && l > bl)) { bh = h; bl = l; }
      }
      const unsigned mh = __reduce_max_sync(0xffffffffu, bh);
      const unsigned ml = __reduce_max_sync(0xffffffffu, bh == mh ? bl : 0u);
      if (lane == 0) { sCand[role][0] = mh; sCand[role][1] = ml; }
      bar_sync(BAR_PANEL2, 32 * PW);
      unsigned wh = sCand[0][0], wl = sCand[0][1];
#pragma unroll
      for (int w2 = 1; w2 < PW; ++w2) {
        const unsigned h2 = sCand[w2][0], l2 = sCand[w2][1];
        if (h2 > wh || (h2 == wh && l2 > wl)) { wh = h2; wl = l2; }
      }
      const int p = 127 - (int)(wl & 127u);
      const int prole = p / HALF, pq = p - prole * HALF, pl = pq & 31, pi = pq >> 5;
      if (role == prole && lane == pl) {
#pragma unroll
        for (int i = 0; i < RPL2; ++i)
          if (pi == i) {
            used[i] = true;
#pragma unroll
            for (int j = 0; j < 8; j += 2)
              *reinterpret_cast<double2*>(&sRowP[t & 1][j]) = make_double2(pr[i][j], pr[i][j + 1]);
          }
      }
      bar_sync(BAR_PANEL2, 32 * PW);
      double rp[8];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(&sRowP[t & 1][j]);
        rp[j] = v.x;
        rp[j + 1] = v.y;
      }
      const double piv = rp[t];
      const double inv = fast_rcp(piv);
#pragma unroll
      for (int j = 0; j < 8; ++j) rp[j] = j == t ? inv : rp[j] * inv;
#pragma unroll
      for (int i = 0; i < RPL2; ++i) {
        const double f = pr[i][t];
        pr[i][t] = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) pr[i][j] = fma(-f, rp[j], pr[i][j]);
      }
#pragma unroll
      for (int i = 0; i < RPL2; ++i) {
        const bool mine = role == prole && pi == i && lane == pl;
#pragma unroll
        for (int j = 0; j < 8; ++j) pr[i][j] = mine ? rp[j] : pr[i][j];
      }
      if (role == 0 && lane == 0) {
        sP[kb & 1][t] = p;
        usedrow[p] = 1;
        pivrow[8 * kb + t] = p;
        rowstep[p] = 8 * kb + t;
        if (piv == 0.0) s_sing = 1;
      }
    }
#pragma unroll
    for (int i = 0; i < RPL2; ++i) {
      const int R = role * HALF + lane + 32 * i;
#pragma unroll
      for (int j = 0; j < 8; ++j) Pb[R][j] = pr[i][j];
    }
    bar_sync(BAR_PANEL2, 32 * PW);
    if (role == 0) {
#pragma unroll
      for (int r = 0; r < NT; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) a[r][C][h] = Pb[8 * r + g][2 * tq + h];
    }
  };
  constexpr bool TWO = NT >= 8;  // two-warp panel when each warp gets >= 1 row per lane
  // A[:, my tile C] += Panel(kb) A[P(kb), tile C]; the pivot rows were zeroed when staged
  auto update_tile = [&](auto cc, int kb) {
    constexpr int C = decltype(cc)::value;
    const double(*Pb)[9] = sW[kb & 1];
    const double b0 = sAP[warp][tq][8 * C + g], b1 = sAP[warp][4 + tq][8 * C + g];
#pragma unroll
    for (int r = 0; r < NT; ++r) {
      dmma_8x8x4(a[r][C][0], a[r][C][1], Pb[8 * r + g][tq], b0);
      dmma_8x8x4(a[r][C][0], a[r][C][1], Pb[8 * r + g][4 + tq], b1);
    }
  };
  using C0 = std::integral_constant<int, 0>;
  using C1 = std::integral_constant<int, 1>;

  __syncthreads();
#ifdef HPS_GJ_PROFILE
  const long long p00 = clock64();
#endif
  if constexpr (TWO) {
    if (warp < PW) panel2(C0{}, 0, warp);
  } else {
    if (warp == 0) panel(C0{}, 0);
  }
#ifdef HPS_GJ_PROFILE
  if (warp == 0 && lane == 0 && blockIdx.x == 0) atomicAdd((unsigned long long*)&g_gj_prof[6], (unsigned long long)(clock64() - p00));
#endif
  __syncthreads();
#ifdef HPS_GJ_PROFILE
  long long pacc[6] = {0, 0, 0, 0, 0, 0};
#endif
  for (int kb = 0; kb < NT; ++kb) {
#ifdef HPS_GJ_PROFILE
    long long q0 = clock64(), q1 = q0, q2 = q0, q3 = q0;
#endif
    const int own = kb >> 1, ownc = kb & 1;  // tile of block kb: already final
    const bool keep0 = warp == own && ownc == 0, keep1 = warp == own && ownc == 1;
    // stage my pivot rows of block kb, zeroing them in the tiles that take the update:
    // a_new = a + Panel A_P on non-pivot rows, a_new = Panel A_P on pivot rows (no cancellation)
    // which of my register slots hold a pivot row of block kb (rows 8r + g), and its position t:
    // a static loop over the slots then stages them with redirected stores (no dynamic register
    // indexing, no indirect branches)
    unsigned zmask = 0u;
    unsigned long long tpos = 0ull;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int p = sP[kb & 1][t];
      if (g == (p & 7)) {
        zmask |= 1u << (p >> 3);
        tpos |= (unsigned long long)t << (4 * (p >> 3));
      }
    }
#pragma unroll
    for (int r = 0; r < NT; ++r) {
      const bool piv = (zmask >> r) & 1u;
      const int t = (int)((tpos >> (4 * r)) & 15ull);
      double* d = piv ? &sAP[warp][t][2 * tq] : sDum;
      d[0] = a[r][0][0];
      d[1] = a[r][0][1];
      d[8] = a[r][1][0];
      d[9] = a[r][1][1];
      const bool z0 = piv && !keep0, z1 = piv && !keep1;
      a[r][0][0] = z0 ? 0.0 : a[r][0][0];
      a[r][0][1] = z0 ? 0.0 : a[r][0][1];
      a[r][1][0] = z1 ? 0.0 : a[r][1][0];
      a[r][1][1] = z1 ? 0.0 : a[r][1][1];
    }
    __syncwarp();
#ifdef HPS_GJ_PROFILE
    q1 = clock64();
#endif
    const int nx = kb + 1, nown = nx >> 1, nownc = nx & 1;
    if (nx < NT && warp == nown) {
      if (nownc == 0) {
        update_tile(C0{}, kb);
#ifdef HPS_GJ_PROFILE
        q2 = clock64();
#endif
        if constexpr (TWO) panel2(C0{}, nx, 0); else panel(C0{}, nx);
#ifdef HPS_GJ_PROFILE
        q3 = clock64();
#endif
        if (!keep1) update_tile(C1{}, kb);
      } else {
        update_tile(C1{}, kb);
#ifdef HPS_GJ_PROFILE
        q2 = clock64();
#endif
        if constexpr (TWO) panel2(C1{}, nx, 0); else panel(C1{}, nx);
#ifdef HPS_GJ_PROFILE
        q3 = clock64();
#endif
        if (!keep0) update_tile(C0{}, kb);
      }
    } else if (TWO && nx < NT && (warp ^ nown) < PW) {
      // helper of the next panel: one of my tile updates, the panel, then the other update
      if (!keep0) update_tile(C0{}, kb);
      panel2(C0{}, nx, warp ^ nown);  // (the helper's tile index is unused)
      if (!keep1) update_tile(C1{}, kb);
    } else {
      if (!keep0) update_tile(C0{}, kb);
      if (!keep1) update_tile(C1{}, kb);
    }
#ifdef HPS_GJ_PROFILE
    long long q4 = clock64();
#endif
    __syncthreads();
#ifdef HPS_GJ_PROFILE
    long long q5 = clock64();
    if (warp == nown && nx < NT) { pacc[0] += q1 - q0; pacc[1] += q2 - q1; pacc[2] += q3 - q2; pacc[3] += q4 - q3; pacc[4] += q5 - q4; pacc[5] += q5 - q0; }
#endif
  }
#ifdef HPS_GJ_PROFILE
  if (lane == 0 && blockIdx.x == 0)
    for (int q = 0; q < 6; ++q) atomicAdd((unsigned long long*)&g_gj_prof[q], (unsigned long long)pacc[q]);
#endif
  // inv(X)[rowstep[R]][pivrow[C]] = B[R][C]
#pragma unroll
  for (int r = 0; r < NT; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int R = 8 * r + g, C = 16 * warp + 8 * c + 2 * tq + h;
        if (R < n && C < n) Xb[(long long)rowstep[R] * lda + pivrow[C]] = a[r][c][h];
      }
  if (s_sing && status && threadIdx.x == 0) atomicMax(status, status_base + (int)blockIdx.x);
}

// Deflation X += sigma V V^T, sigma = max |diag X| (reduced by k_gather_xr before any CTA here
// modifies a diagonal block): one CTA per (segment row, merge).
__global__ void k_deflate(double* X, int n, int q, const double* __restrict__ vs, const double* __restrict__ ve,
                          const unsigned long long* __restrict__ diagmax) {
  const int b = blockIdx.x, sr = blockIdx.y;
  double* Xb = X + (long long)b * n * n;
  const double sigma = __longlong_as_double((long long)diagmax[b]);
  const int nseg = n / q;
  const int c0 = max(0, sr - 1) * q, c1 = min(nseg, sr + 2) * q;
  const int w = c1 - c0;
  for (int idx = threadIdx.x; idx < q * w; idx += blockDim.x) {
    int r = sr * q + idx / w, c = c0 + idx % w;
    Xb[(long long)r * n + c] += sigma * vvt(r, c, q, nseg, vs, ve);
  }
}

// In-place batched inverse of n x n blocks (n <= 128), stride lda: blocked Gauss-Jordan.
static int inverse_small(double* X, long long lda, long long strideX, int n, int batch, int* status,
                         int status_base, cudaStream_t st) {
  if (n > 128) {
    set_error("inverse_small: n=%d > 128", n);
    return HPS_ERR_ARG;
  }
  if (n <= 16)
    k_gj_blk<2><<<batch, 32, 0, st>>>(X, lda, strideX, n, status, status_base);
  else if (n <= 32)
    k_gj_blk<4><<<batch, 64, 0, st>>>(X, lda, strideX, n, status, status_base);
  else if (n <= 64)
    k_gj_blk<8><<<batch, 128, 0, st>>>(X, lda, strideX, n, status, status_base);
  else
    k_gj_blk<16><<<batch, 256, 0, st>>>(X, lda, strideX, n, status, status_base);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

static int gemm(Ctx& cx, int M, int N, int K, int batch, double alpha, const double* A, long long lda, long long sA,
                const double* B, long long ldb, long long sB, double beta, double* C, long long ldc, long long sC,
                cudaStream_t st, int* nonfinite = nullptr) {
  GemmParams p{M, N, K, batch, A, lda, sA, B, ldb, sB, nullptr, 0, C, ldc, sC, alpha, beta, nonfinite};
  p.emu_ok = true;  // the block inverse's large GEMMs may run emulated on the int8 tensor cores
  return dgemm_launch(p, cx, st);
}

#define HPS_TRY(x)            \
  do {                        \
    int _s = (x);             \
    if (_s != HPS_OK) return _s; \
  } while (0)

// Recursive 2x2 block inverse, in place, batched (all matrices n x n with leading dim lda).
//   A11 <- inv(A11); T12 = A11 A12; T21 = A21 A11; A22 <- A22 - A21 T12; A22 <- inv(A22)
//   A12 <- -T12 A22; A21 <- -A22 T21; A11 <- A11 - A12 T21
// Base blocks (<= 128) use pivoted Gauss-Jordan in registers. The independent GEMM pairs of each
// level run concurrently on the context's fork stream (fork/join through its event ring; captured
// CUDA graphs get parallel branches).
static int inverse_rec(Ctx& cx, double* A, long long lda, long long strideA, int n, int batch, double* tmp,
                       int* status, int status_base, cudaStream_t st, cudaStream_t side = nullptr) {
  if (n <= 128) return inverse_small(A, lda, strideA, n, batch, status, status_base, st);
  const int h = n / 2, h2 = n - h;  // unequal halves allowed (q = 21 gives n3 = 21 * 2^j)
  double* A11 = A;
  double* A12 = A + h;
  double* A21 = A + (long long)h * lda;
  double* A22 = A21 + h;
  double* T12 = tmp;                              // h x h2
  double* T21 = tmp + (long long)batch * h * h2;  // h2 x h
  double* deeper = T21 + (long long)batch * h * h2;
  const long long sT = (long long)h * h2;
  const bool fork = cx.opt[HPS_OPT_INV_FORK] && cx.streams_ok;
  if (!side) side = cx.side;
  cudaStream_t s2 = fork ? side : st;
  HPS_TRY(inverse_rec(cx, A11, lda, strideA, h, batch, deeper, status, status_base, st, side));
  if (fork) HPS_CUDA_CHECK(cudaStreamWaitEvent(s2, cx.record_on(st), 0));
  // T21 = A21 inv(A11) on the side stream, T12 = inv(A11) A12 and the Schur update on the main one
  HPS_TRY(gemm(cx, h2, h, h, batch, 1.0, A21, lda, strideA, A11, lda, strideA, 0.0, T21, h, sT, s2));
  HPS_TRY(gemm(cx, h, h2, h, batch, 1.0, A11, lda, strideA, A12, lda, strideA, 0.0, T12, h2, sT, st));
  HPS_TRY(gemm(cx, h2, h2, h, batch, -1.0, A21, lda, strideA, T12, h2, sT, 1.0, A22, lda, strideA, st));
  HPS_TRY(inverse_rec(cx, A22, lda, strideA, h2, batch, deeper, status, status_base, st, side));
  if (fork) HPS_CUDA_CHECK(cudaStreamWaitEvent(s2, cx.record_on(st), 0));
  // A21 = -inv(S) T21 on the side stream (after T21 there), A12 = -T12 inv(S) on the main one
  HPS_TRY(gemm(cx, h2, h, h2, batch, -1.0, A22, lda, strideA, T21, h, sT, 0.0, A21, lda, strideA, s2));
  HPS_TRY(gemm(cx, h, h2, h2, batch, -1.0, T12, h2, sT, A22, lda, strideA, 0.0, A12, lda, strideA, st));
  if (fork) HPS_CUDA_CHECK(cudaStreamWaitEvent(st, cx.record_on(s2), 0));  // join: T21 and A21 done
  HPS_TRY(gemm(cx, h, h, h2, batch, -1.0, A12, lda, strideA, T21, h, sT, 1.0, A11, lda, strideA, st));
  return HPS_OK;
}

static size_t inverse_rec_tmp_doubles(int n, int batch) {
  if (n <= 128) return 0;  // the Gauss-Jordan base needs no workspace
  const int h = n / 2, h2 = n - h;
  return 2ull * batch * h * h2 + std::max(inverse_rec_tmp_doubles(h, batch), inverse_rec_tmp_doubles(h2, batch));
}

// Merge workspace of one depth: X (inverted in place for n3 <= 128, LU-factored for n3 > 128), R,
// C, the LU pivots (n3 > 128) and the per-merge deflation shifts.
// Merge workspace of one depth: X (inverted in place, or LU-factored with pivoting), R, C; for
// n3 > 128 also the probe image w = X_d v of the inverse's residual check, the block-inverse
// recursion's temporaries and the LU pivots; the per-merge deflation shifts.
struct MergeWs {
  double *X, *R, *C;
  double *probe = nullptr, *rtmp = nullptr;
  LuWs lu;
  unsigned long long* diagmax;
};
static size_t merge_aux_bytes(int nbatch, int n3) {
  if (n3 <= 128) return 0;
  const size_t d = (size_t)nbatch * n3 + inverse_rec_tmp_doubles(n3, nbatch);
  return ((d * sizeof(double) + lu_ws_bytes(n3, nbatch)) + 255) & ~size_t(255);
}
static MergeWs merge_ws(void* ws, int nbatch, int n3, int ne) {
  MergeWs w;
  w.X = static_cast<double*>(ws);
  w.R = w.X + (size_t)nbatch * n3 * n3;
  w.C = w.R + (size_t)nbatch * n3 * ne;
  double* aux = w.C + (size_t)nbatch * ne * n3;
  if (n3 > 128) {
    w.probe = aux;
    w.rtmp = w.probe + (size_t)nbatch * n3;
    w.lu = lu_ws(w.rtmp + inverse_rec_tmp_doubles(n3, nbatch), n3, nbatch);
  }
  w.diagmax = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(aux) + merge_aux_bytes(nbatch, n3));
  return w;
}

// Residual check of the fast block inverse (n3 > 128). Before the inversion w = X_d v for a fixed
// +-1 probe v (k_resid_image); afterwards r = X_d^-1 w - v (k_resid_check, in the same call, or in the
// parent depth's call when the look-ahead inverted X, so the check stays off the look-ahead's
// critical path). The recursive 2x2 block inverse pivots only inside 128-blocks, so a near-singular
// leading block would go unnoticed; max|r| above 1e-6 (or non-finite) raises the merge's status word
// to HPS_STATUS_PIVOT + b and the host re-runs that depth with the pivoted LU. One warp per row.
__device__ __forceinline__ double probe_v(int i) { return ((i * 2654435761u) >> 13) & 1 ? 1.0 : -1.0; }
__global__ void k_resid_image(const double* __restrict__ X, int n, double* __restrict__ w) {
  const int b = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= n) return;
  const double* Xr = X + ((long long)b * n + r) * n;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s = fma(Xr[c], probe_v(c), s);
  s = warp_sum(s);
  if (lane == 0) w[(long long)b * n + r] = s;
}
__global__ void k_resid_check(const double* __restrict__ Xi, int n, const double* __restrict__ w, int* status,
                              int status_base) {
  const int b = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= n) return;
  const double* Xr = Xi + ((long long)b * n + r) * n;
  const double* wb = w + (long long)b * n;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s = fma(Xr[c], wb[c], s);
  s = warp_sum(s) - probe_v(r);
  if (lane == 0 && !(fabs(s) <= 1e-6) && status) atomicMax(status, HPS_STATUS_PIVOT + status_base + b);
}
static int resid_image(const MergeWs& W, const double* X, int n3, int nbatch, cudaStream_t st) {
  k_resid_image<<<dim3((n3 + 7) / 8, nbatch), 256, 0, st>>>(X, n3, W.probe);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}
static int resid_check(const MergeWs& W, const double* Xi, int n3, int nbatch, int* status, int status_base,
                       cudaStream_t st) {
  k_resid_check<<<dim3((n3 + 7) / 8, nbatch), 256, 0, st>>>(Xi, n3, W.probe, status, status_base);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

}  // namespace hps

using namespace hps;

extern "C" size_t hps_merge_workspace_bytes(int nbatch, int n3, int ne) {
  const size_t d = size_t(nbatch) * (size_t(n3) * n3 + 2ull * n3 * ne + 1);
  return d * sizeof(double) + merge_aux_bytes(nbatch, n3) + 256;
}

// HPS_OPT_PROFILE_AHEAD (eager builds only, dev tool): timing events at the look-ahead fork (0),
// the end of the parent inverse on the look-ahead stream (1), the end of the T GEMM (2) and the
// join (3), per depth; hps_debug_ahead_times reads the elapsed times relative to event 0.
static void ahead_probe(Ctx& cx, int k, cudaStream_t s) {
  if (!cx.opt[HPS_OPT_PROFILE_AHEAD] || cx.probe_depth < 0 || cx.probe_depth >= 32) return;
  cudaEvent_t& e = cx.probe[cx.probe_depth][k];
  if (!e) cudaEventCreate(&e);
  cudaEventRecord(e, s);
}
extern "C" int hps_debug_ahead_times(hps_ctx_t ctx, int depth, float* out) {  // ms since the fork
  Ctx* cx = reinterpret_cast<Ctx*>(ctx);
  if (!cx || depth < 0 || depth >= 32 || !cx->probe[depth][0]) return 1;
  for (int k = 1; k < 4; ++k) cudaEventElapsedTime(out + k - 1, cx->probe[depth][0], cx->probe[depth][k]);
  return 0;
}
extern "C" void hps_debug_ahead_depth(hps_ctx_t ctx, int depth) {
  if (ctx) reinterpret_cast<Ctx*>(ctx)->probe_depth = depth;
}

// Parent-depth look-ahead of hps_merge_level_ahead (see k_ahead_rows).
struct AheadArgs {
  const int* pmaps;       // parent depth's split maps (j1a, j2b, j3a, j3b)
  int pn3, pne;
  const double* pvmode;   // parent depth's corner-mode vectors (2q)
  void* pws;              // the parent depth's merge workspace (X inverted in place there)
  size_t pws_bytes;
  int* pstatus;
  int pstatus_base;
};

static int merge_level_impl(Ctx& cx, int nbatch, int n3, int ne, int m, int q, const double* T_child, long long child_stride,
                            const int* child_idx, const int* maps, const double* vmode, double* S_out, double* T_out,
                            void* ws, size_t ws_bytes, int* status, int status_base, bool pre_inverted,
                            const AheadArgs* ah, cudaStream_t st, int flags = 0) {
  if (nbatch <= 0) return HPS_OK;
  if (ne % 2 || n3 % q || m != ne / 2 + n3 || ws_bytes < hps_merge_workspace_bytes(nbatch, n3, ne)) {
    set_error("hps_merge_level: bad arguments n3=%d ne=%d m=%d q=%d ws=%zu", n3, ne, m, q, ws_bytes);
    return HPS_ERR_ARG;
  }
  const int n1 = ne / 2;
  const int* j1a = maps;
  const int* j2b = maps + n1;
  const int* j3a = maps + 2 * n1;
  const int* j3b = j3a + n3;
  const MergeWs W = merge_ws(ws, nbatch, n3, ne);
  double* X = W.X;
  double* R = W.R;
  double* Cm = W.C;
  unsigned long long* diagmax = W.diagmax;
  // n3 <= 128: in-register Gauss-Jordan inverse (partial pivoting over the whole matrix). n3 > 128:
  // the recursive block inverse with its residual check (fast; HPS_MERGE_PIVOTED unset), or the
  // pivoted LU + triangular solves (HPS_MERGE_PIVOTED: what the host asks for after a failed check).
  const bool big = n3 > 128 && (flags & HPS_MERGE_PIVOTED);
  const bool checked = n3 > 128 && !big;
  const bool deflate = n3 > q;  // deflate the n3/q - 1 corner null modes
  ChildRef ch{T_child, child_stride, child_idx, m};
  if (!pre_inverted && deflate) HPS_CUDA_CHECK(cudaMemsetAsync(diagmax, 0, sizeof(unsigned long long) * nbatch, st));
  // pre_inverted: X was formed, deflated and inverted (n3 <= 128) or LU-factored (n3 > 128) by the
  // child depth's look-ahead; R and C only
  k_gather_xr<<<dim3(nbatch, (n3 + 7) / 8), 256, 0, st>>>(ch, j1a, j2b, j3a, j3b, n3, ne, pre_inverted ? nullptr : X,
                                                        R, (deflate && !pre_inverted) ? diagmax : nullptr);
  HPS_LAUNCH_CHECK();
  if (n3 < 32)
    k_gather_c<<<dim3(nbatch, (unsigned)std::min<long long>(((long long)ne * n3 + 1023) / 1024, 65535)), 256, 0,
                 st>>>(ch, j1a, j2b, j3a, j3b, n3, ne, Cm);
  else
    k_gather_c_rows<<<dim3(nbatch, (ne + 7) / 8), 256, 0, st>>>(ch, j1a, j2b, j3a, j3b, n3, ne, Cm);
  HPS_LAUNCH_CHECK();
  if (pre_inverted && checked)  // the look-ahead inverted X: its residual check runs here
    HPS_TRY(resid_check(W, X, n3, nbatch, status, status_base, st));
  if (!pre_inverted) {
    if (deflate) {
      k_deflate<<<dim3(nbatch, n3 / q), 256, 0, st>>>(X, n3, q, vmode, vmode + q, diagmax);
      HPS_LAUNCH_CHECK();
    }
    if (big) {
      HPS_TRY(lu_factor(cx, X, n3, nbatch, W.lu, status, status_base, st));
    } else if (checked) {
      HPS_TRY(resid_image(W, X, n3, nbatch, st));
      HPS_TRY(inverse_rec(cx, X, n3, (long long)n3 * n3, n3, nbatch, W.rtmp, status, status_base, st));
      HPS_TRY(resid_check(W, X, n3, nbatch, status, status_base, st));
    } else
      HPS_TRY(inverse_small(X, n3, (long long)n3 * n3, n3, nbatch, status, status_base, st));
  }
  if (!S_out) return HPS_OK;  // interface only (hps_merge_interface): X factored, R and C gathered
  // S = X^-1 R; a non-finite S raises the status word to the merge index (MergeResonanceError)
  if (big)
    HPS_TRY(lu_solve(cx, X, n3, nbatch, W.lu, R, ne, S_out, status, status_base, st));
  else {
    GemmParams sp{n3, ne, n3, nbatch, X, n3, (long long)n3 * n3, R, ne, (long long)n3 * ne, nullptr, 0, S_out, ne,
                  (long long)n3 * ne, 1.0, 0.0, status};
    sp.emu_ok = true;
    HPS_TRY(dgemm_launch(sp, cx, st));
  }
  if (ah != nullptr && !(cx.streams_ok && (nbatch % 2) == 0)) {
    // the caller would treat the parent's X as inverted: refuse instead of skipping silently
    set_error("hps_merge_level_ahead: look-ahead needs an even nbatch (got %d) and the context's streams", nbatch);
    return HPS_ERR_ARG;
  }
  const bool ahead = ah != nullptr;
  if (ahead) {
    // parent X from the pj3 rows / columns of this depth's T (before the T GEMM): gathered
    // operands in the parent workspace's R and C regions, X into its X region
    const int P = nbatch / 2, pn3 = ah->pn3, pne = ah->pne, pn1 = pne / 2;
    if (pn3 % q || ah->pws_bytes < hps_merge_workspace_bytes(P, pn3, pne)) {
      set_error("hps_merge_level_ahead: bad parent arguments pn3=%d pne=%d ws=%zu", pn3, pne, ah->pws_bytes);
      return HPS_ERR_ARG;
    }
    const int* pj3a = ah->pmaps + 2 * pn1;
    const int* pj3b = pj3a + pn3;
    const MergeWs PW = merge_ws(ah->pws, P, pn3, pne);
    double* pX = PW.X;
    double* pR = PW.R;
    double* pC = PW.C;
    unsigned long long* pdiag = PW.diagmax;
    double* Ag = pR;  // P x pn3 x 2 n3  (2 n3 <= pne)
    double* Bg = pC;  // P x 2 n3 x pn3
    k_ahead_rows<<<dim3(P, (pn3 + 7) / 8), 256, 0, st>>>(ch, j1a, j2b, n3, ne, Cm, pj3a, pj3b, pn3, Ag, pX);
    HPS_LAUNCH_CHECK();
    k_ahead_bg<<<dim3(P, (2 * n3 + 7) / 8), 256, 0, st>>>(S_out, n3, ne, pj3a, pj3b, pn3, Bg);
    HPS_LAUNCH_CHECK();
    HPS_TRY(gemm(cx, pn3, pn3, 2 * n3, P, 1.0, Ag, 2 * n3, (long long)pn3 * 2 * n3, Bg, pn3, (long long)2 * n3 * pn3,
                 1.0, pX, pn3, (long long)pn3 * pn3, st));
    const bool pdefl = pn3 > q;
    if (pdefl) {
      HPS_CUDA_CHECK(cudaMemsetAsync(pdiag, 0, sizeof(unsigned long long) * P, st));
      k_diagmax<<<P, 256, 0, st>>>(pX, pn3, pdiag);
      HPS_LAUNCH_CHECK();
    }
    // fork: deflate + invert the parent X on the high-priority look-ahead stream
    ahead_probe(cx, 0, st);
    HPS_CUDA_CHECK(cudaStreamWaitEvent(cx.ahead, cx.record_on(st), 0));
    if (pdefl) {
      k_deflate<<<dim3(P, pn3 / q), 256, 0, cx.ahead>>>(pX, pn3, q, ah->pvmode, ah->pvmode + q, pdiag);
      HPS_LAUNCH_CHECK();
    }
    if (pn3 > 128 && (flags & HPS_MERGE_PARENT_PIVOTED))
      HPS_TRY(lu_factor(cx, pX, pn3, P, PW.lu, ah->pstatus, ah->pstatus_base, cx.ahead));
    else if (pn3 > 128) {  // residual image now, the check in the parent's call
      HPS_TRY(resid_image(PW, pX, pn3, P, cx.ahead));
      HPS_TRY(inverse_rec(cx, pX, pn3, (long long)pn3 * pn3, pn3, P, PW.rtmp, ah->pstatus, ah->pstatus_base, cx.ahead,
                          cx.ahead_side));
    }
    else
      HPS_TRY(inverse_small(pX, pn3, (long long)pn3 * pn3, pn3, P, ah->pstatus, ah->pstatus_base, cx.ahead));
    ahead_probe(cx, 1, cx.ahead);
  }
  {  // T = blkdiag(Ta[j1a, j1a], Tb[j2b, j2b]) + C S, the blkdiag read by the GEMM epilogue
    GemmParams gp{ne, ne, n3, nbatch, Cm, n3, (long long)ne * n3, S_out, ne, (long long)n3 * ne, nullptr, 0,
                  T_out, ne, (long long)ne * ne, 1.0, 0.0, nullptr};
    gp.blk = ch;
    gp.blk_j1a = j1a;
    gp.blk_j2b = j2b;
    gp.emu_ok = true;
    HPS_TRY(dgemm_launch(gp, cx, st));
  }
  if (ahead) ahead_probe(cx, 2, st);
  if (ahead) HPS_CUDA_CHECK(cudaStreamWaitEvent(st, cx.record_on(cx.ahead), 0));  // join
  if (ahead) ahead_probe(cx, 3, st);
  return HPS_OK;
}

extern "C" int hps_merge_level(hps_ctx_t ctx, int nbatch, int n3, int ne, int m, int q, const double* T_child,
                               long long child_stride, const int* child_idx, const int* maps, const double* vmode,
                               double* S_out, double* T_out, void* ws, size_t ws_bytes, int* status,
                               int status_base, void* stream) {
  HPS_CTX(cx, ctx);
  return merge_level_impl(*cx, nbatch, n3, ne, m, q, T_child, child_stride, child_idx, maps, vmode, S_out, T_out, ws,
                          ws_bytes, status, status_base, false, nullptr, static_cast<cudaStream_t>(stream));
}

extern "C" int hps_merge_level_ahead(hps_ctx_t ctx, int nbatch, int n3, int ne, int m, int q, const double* T_child,
                                     long long child_stride, const int* child_idx, const int* maps,
                                     const double* vmode, double* S_out, double* T_out, void* ws, size_t ws_bytes,
                                     int* status, int status_base, int pre_inverted, const int* pmaps, int pn3,
                                     int pne, const double* pvmode, void* pws, size_t pws_bytes, int* pstatus,
                                     int pstatus_base, int flags, void* stream) {
  HPS_CTX(cx, ctx);
  AheadArgs ah{pmaps, pn3, pne, pvmode, pws, pws_bytes, pstatus, pstatus_base};
  return merge_level_impl(*cx, nbatch, n3, ne, m, q, T_child, child_stride, child_idx, maps, vmode, S_out, T_out, ws,
                          ws_bytes, status, status_base, pre_inverted != 0, pmaps ? &ah : nullptr,
                          static_cast<cudaStream_t>(stream), flags);
}

// Batched in-place inverse (n <= 128 uses the register Gauss-Jordan kernel directly, larger n the
// recursive block inverse). Exposed for unit tests and micro-benchmarks.
extern "C" size_t hps_inverse_workspace_bytes(int n, int batch) {
  return inverse_rec_tmp_doubles(n, batch) * sizeof(double) + 256;
}

extern "C" int hps_inverse_batched(hps_ctx_t ctx, int n, int batch, double* X, long long lda, long long strideX, void* ws,
                                   size_t ws_bytes, int* status, void* stream) {
  if (ws_bytes < hps_inverse_workspace_bytes(n, batch) || n <= 0) {
    set_error("hps_inverse_batched: bad arguments n=%d ws=%zu", n, ws_bytes);
    return HPS_ERR_ARG;
  }
  HPS_CTX(cx, ctx);
  return inverse_rec(*cx, X, lda, strideX, n, batch, static_cast<double*>(ws), status, 0,
                     static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------------------------------------
// Split merge for the distributed top depths (parallel.py): the owner of a parent forms and factors
// its interface system (hps_merge_interface), every rank of the parent's group solves a column panel
// of S and multiplies it into a column panel of T (hps_interface_solve + hps_dgemm_batched), and the
// owner assembles T = blkdiag + panels (hps_merge_assemble). Per-element arithmetic is that of
// hps_merge_level (same kernels, same summation order), so with split-K off the two agree bitwise.
// ---------------------------------------------------------------------------------------------
namespace hps {
__global__ void k_iota_rows(int* perm, int n, int batch) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * batch; i += gridDim.x * blockDim.x) perm[i] = i % n;
}

// T[b][r][c] = blkdiag(Ta[j1a, j1a], Tb[j2b, j2b])[r][c] + panels[c / w][b][r][c % w], one warp per row.
__global__ void k_merge_assemble(ChildRef ch, const int* __restrict__ j1a, const int* __restrict__ j2b, int ne,
                                 const double* __restrict__ panels, int w, int nbatch, double* __restrict__ T) {
  const int b = blockIdx.y;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= ne) return;
  const int n1 = ne / 2;
  const bool top = r < n1;
  const double* src = top ? ch.a(b) : ch.bb(b);
  const int rm = top ? j1a[r] : j2b[r - n1];
  double* Tr = T + ((long long)b * ne + r) * ne;
  for (int c = lane; c < ne; c += 32) {
    const int p = c / w, cc = c - p * w;
    double v = panels[(((long long)p * nbatch + b) * ne + r) * w + cc];
    double blk = 0.0;
    if ((c < n1) == top) blk = src[(long long)rm * ch.m + (top ? j1a[c] : j2b[c - n1])];
    Tr[c] = v + blk;
  }
}
}  // namespace hps

extern "C" int hps_merge_interface(hps_ctx_t ctx, int nbatch, int n3, int ne, int m, int q, const double* T_child,
                                   long long child_stride, const int* child_idx, const int* maps, const double* vmode,
                                   double* Xf_out, int* perm_out, double* R_out, double* C_out, void* ws,
                                   size_t ws_bytes, int* status, int status_base, int flags, void* stream) {
  HPS_CTX(cx, ctx);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HPS_TRY(merge_level_impl(*cx, nbatch, n3, ne, m, q, T_child, child_stride, child_idx, maps, vmode, nullptr,
                           nullptr, ws, ws_bytes, status, status_base, false, nullptr, st, flags));
  const bool lu_form = n3 > 128 && (flags & HPS_MERGE_PIVOTED);
  const MergeWs W = merge_ws(ws, nbatch, n3, ne);
  const size_t nX = (size_t)nbatch * n3 * n3, nR = (size_t)nbatch * n3 * ne;
  if (Xf_out) HPS_CUDA_CHECK(cudaMemcpyAsync(Xf_out, W.X, nX * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (R_out) HPS_CUDA_CHECK(cudaMemcpyAsync(R_out, W.R, nR * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (C_out) HPS_CUDA_CHECK(cudaMemcpyAsync(C_out, W.C, nR * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (perm_out) {
    if (lu_form) {
      HPS_CUDA_CHECK(cudaMemcpyAsync(perm_out, W.lu.perm, (size_t)nbatch * n3 * sizeof(int), cudaMemcpyDeviceToDevice, st));
    } else {
      k_iota_rows<<<std::max(1, std::min(1024, (n3 * nbatch + 255) / 256)), 256, 0, st>>>(perm_out, n3, nbatch);
      HPS_LAUNCH_CHECK();
    }
  }
  return HPS_OK;
}

extern "C" int hps_interface_solve(hps_ctx_t ctx, int n3, int ncols, int batch, const double* Xf, const int* perm,
                                   const double* R, double* S_out, int* status, int status_base, int flags,
                                   void* stream) {
  HPS_CTX(cx, ctx);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n3 <= 0 || ncols <= 0 || batch <= 0) {
    set_error("hps_interface_solve: bad arguments n3=%d ncols=%d", n3, ncols);
    return HPS_ERR_ARG;
  }
  if (!(n3 > 128 && (flags & HPS_MERGE_PIVOTED)))  // Xf is the explicit inverse
    return gemm(*cx, n3, ncols, n3, batch, 1.0, Xf, n3, (long long)n3 * n3, R, ncols, (long long)n3 * ncols, 0.0,
                S_out, ncols, (long long)n3 * ncols, st, status);
  LuWs w;
  w.perm = const_cast<int*>(perm);
  return lu_solve(*cx, Xf, n3, batch, w, R, ncols, S_out, status, status_base, st);
}

extern "C" int hps_merge_assemble(hps_ctx_t ctx, int nbatch, int ne, int m, const double* T_child,
                                  long long child_stride, const int* child_idx, const int* maps, const double* panels,
                                  int npanels, double* T_out, void* stream) {
  HPS_CTX(cx, ctx);
  (void)cx;
  if (npanels <= 0 || ne % npanels || ne % 2) {
    set_error("hps_merge_assemble: ne=%d not divisible into %d panels", ne, npanels);
    return HPS_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ChildRef ch{T_child, child_stride, child_idx, m};
  k_merge_assemble<<<dim3((ne + 7) / 8, nbatch), 256, 0, st>>>(ch, maps, maps + ne / 2, ne, panels, ne / npanels,
                                                              nbatch, T_out);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}
