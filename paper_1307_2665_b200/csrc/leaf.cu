// Leaf stage (reference leafops.py:217-302 + solver.py:226-246), one CTA per coefficient group.
//
//   1. Assemble A = -c11 D1sq - 2 c12 D12 - c22 D2sq + c1 D1 + c2 D2 + diag(c) on the fly from the
//      1-D factors. The same per-entry op sequence as the reference is used, so the entries are
//      bitwise equal. Only the augmented system M = [A_ii | A_ie | probe] (ni x (ni+nb+1)) is
//      materialised, in a per-CTA global scratch slot. 148 slots x 400 KB stay resident in L2.
//   2. Blocked Gaussian elimination with partial pivoting on M (panel in shared memory, rank-NB
//      trailing updates). This is the same factorisation family as LAPACK gesv in the reference.
//   3. Blocked back substitution X = U^{-1} Y, probe condition estimate (leafops.py:293-294),
//      Psi = -X[:, :nb].
//   4. DtN epilogue T = (L43[:,J_e] + L43[:,J_i] Psi) L1 (solver.py:241-242).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "leaf.cuh"

namespace hps {

constexpr int LEAF_NB = 16;
constexpr int LEAF_THREADS = 256;



__global__ void __launch_bounds__(LEAF_THREADS) k_leaf(LeafArgs a) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  __shared__ int s_piv;
  const int p = a.p, p2 = p * p;
  const int ni = (p - 2) * (p - 2), nb = 4 * (p - 1), ng = 4 * p;
  const int ncols = ni + nb + 1;
  const int ldm = ncols + 1;  // even
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;

  // shared memory carve-up
  double* coef = sm;                  // 6 * p2
  double* Dx = coef + 6 * p2;         // p2
  double* Dy = Dx + p2;
  double* Dxx = Dy + p2;
  double* Dyy = Dxx + p2;
  double* P = Dyy + p2;               // ni * NB panel
  double* Ub = P + ni * LEAF_NB;      // NB * ncols
  double* T1 = Ub + LEAF_NB * ncols;  // ng * nb
  int* ipiv = reinterpret_cast<int*>(T1 + ng * nb);  // ni
  int* Ji = ipiv + ni;                // ni
  int* Je = Ji + ni;                  // nb

  const double* cDx = a.consts;
  const double* cL43e = a.consts + 4 * p2;
  const double* cL43i = cL43e + ng * nb;
  const double* cL1 = cL43i + ng * ni;
  const double* cprobe = cL1 + nb * ng;

  for (int i = tid; i < 4 * p2; i += nt) Dx[i] = cDx[i];
  for (int i = tid; i < ni; i += nt) Ji[i] = a.idx[i];
  for (int i = tid; i < nb; i += nt) Je[i] = a.idx[ni + i];

  double* M = a.scratch + (long long)blockIdx.x * a.scratch_stride;

  for (int grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    __syncthreads();
    for (int f = 0; f < 6; ++f) {
      const double* src = a.field[f] ? a.field[f] + (long long)grp * p2 : nullptr;
      for (int i = tid; i < p2; i += nt) coef[f * p2 + i] = src ? src[i] : a.scalar[f];
    }
    __syncthreads();

    // ---- 1. assemble M = [A_ii | A_ie | probe], row abs-sum of A_ii for the norm ----
    double rowmax = 0.0;
    for (int r = warp; r < ni; r += nt / 32) {
      const int na = Ji[r], ia = na / p, ja = na - ia * p;
      double rs = 0.0;
      for (int c = lane; c < ncols; c += 32) {
        double v;
        if (c == ncols - 1) {
          v = cprobe[r];
        } else {
          const int nbn = c < ni ? Ji[c] : Je[c - ni];
          const int ib = nbn / p, jb = nbn - ib * p;
          double acc = 0.0;
          if (a.present[0] && ja == jb) acc += coef[0 * p2 + na] * (-Dxx[ia * p + ib]);
          if (a.present[1]) acc += coef[1 * p2 + na] * (-2.0 * (Dx[ia * p + ib] * Dy[ja * p + jb]));
          if (a.present[2] && ia == ib) acc += coef[2 * p2 + na] * (-Dyy[ja * p + jb]);
          if (a.present[3] && ja == jb) acc += coef[3 * p2 + na] * Dx[ia * p + ib];
          if (a.present[4] && ia == ib) acc += coef[4 * p2 + na] * Dy[ja * p + jb];
          if (nbn == na) acc += coef[5 * p2 + na];
          v = acc;
          if (c < ni) rs += fabs(v);
        }
        M[(long long)r * ldm + c] = v;
      }
      rs = warp_sum(rs);
      rowmax = fmax(rowmax, rs);
    }
    const double anorm = block_max(rowmax, red);
    __syncthreads();

    // ---- 2. blocked GE with partial pivoting ----
    for (int k0 = 0; k0 < ni; k0 += LEAF_NB) {
      const int kb = min(LEAF_NB, ni - k0);
      const int rows = ni - k0;
      for (int e = tid; e < rows * kb; e += nt) {
        int i = e / kb, j = e - i * kb;
        P[i * LEAF_NB + j] = M[(long long)(k0 + i) * ldm + k0 + j];
      }
      __syncthreads();
      for (int j = 0; j < kb; ++j) {
        if (warp == 0) {
          double best = -1.0;
          int bi = j;
          for (int i = j + lane; i < rows; i += 32) {
            double v = fabs(P[i * LEAF_NB + j]);
            if (v > best) { best = v; bi = i; }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_xor_sync(0xffffffffu, best, o);
            int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
          }
          if (lane == 0) { s_piv = bi; ipiv[k0 + j] = k0 + bi; }
        }
        __syncthreads();
        const int pr = s_piv;
        if (pr != j && tid < kb) {
          double t0 = P[j * LEAF_NB + tid];
          P[j * LEAF_NB + tid] = P[pr * LEAF_NB + tid];
          P[pr * LEAF_NB + tid] = t0;
        }
        __syncthreads();
        const double inv = 1.0 / P[j * LEAF_NB + j];
        for (int i = j + 1 + tid; i < rows; i += nt) P[i * LEAF_NB + j] *= inv;
        __syncthreads();
        const int w = kb - j - 1;
        if (w > 0)
          for (int e = tid; e < (rows - j - 1) * w; e += nt) {
            int i = j + 1 + e / w, c = j + 1 + e % w;
            P[i * LEAF_NB + c] -= P[i * LEAF_NB + j] * P[j * LEAF_NB + c];
          }
        __syncthreads();
      }
      // U11 rows back to M (L part stays in smem; L is not needed after this panel)
      for (int e = tid; e < kb * kb; e += nt) {
        int i = e / kb, j = e - i * kb;
        if (j >= i) M[(long long)(k0 + i) * ldm + k0 + j] = P[i * LEAF_NB + j];
      }
      // row swaps + U12 = L11^{-1} M12 on trailing columns (one column per thread)
      const int c0 = k0 + kb;
      const int wt = ncols - c0;
      for (int cc = tid; cc < wt; cc += nt) {
        const int c = c0 + cc;
        double x[LEAF_NB];
        for (int j = 0; j < kb; ++j) {
          const int pj = ipiv[k0 + j];
          if (pj != k0 + j) {
            double t0 = M[(long long)(k0 + j) * ldm + c];
            M[(long long)(k0 + j) * ldm + c] = M[(long long)pj * ldm + c];
            M[(long long)pj * ldm + c] = t0;
          }
        }
#pragma unroll
        for (int j = 0; j < LEAF_NB; ++j) {
          if (j < kb) {
            double v = M[(long long)(k0 + j) * ldm + c];
            for (int i = 0; i < j; ++i) v -= P[j * LEAF_NB + i] * x[i];
            x[j] = v;
            Ub[j * ncols + cc] = v;
            M[(long long)(k0 + j) * ldm + c] = v;
          }
        }
      }
      __syncthreads();
      // trailing update rows k0+kb.., cols c0..
      const int tr = rows - kb;
      for (int e = tid; e < tr * wt; e += nt) {
        const int i = e / wt, cc = e - i * wt;
        double* dst = M + (long long)(c0 + i) * ldm + c0 + cc;
        double v = *dst;
        const double* Lr = P + (kb + i) * LEAF_NB;
        for (int j = 0; j < kb; ++j) v -= Lr[j] * Ub[j * ncols + cc];
        *dst = v;
      }
      __syncthreads();
    }

    // ---- 3. back substitution X = U^{-1} Y (Y = columns ni..ncols-1), blocked by NB rows ----
    const int nr = ncols - ni;  // nb + 1 right-hand sides
    for (int kend = ni; kend > 0; kend -= LEAF_NB) {
      const int k0 = max(0, kend - LEAF_NB);
      const int kb = kend - k0;
      // Y_blk -= U[blk, kend:] X[kend:]
      for (int e = tid; e < kb * nr; e += nt) {
        const int i = e / nr, c = e - i * nr;
        const double* Ur = M + (long long)(k0 + i) * ldm;
        double v = Ur[ni + c];
        for (int k = kend; k < ni; ++k) v -= Ur[k] * M[(long long)k * ldm + ni + c];
        Ub[i * ncols + c] = v;
      }
      __syncthreads();
      // triangular solve within the block, one RHS column per thread
      for (int c = tid; c < nr; c += nt) {
        for (int i = kb - 1; i >= 0; --i) {
          const double* Ur = M + (long long)(k0 + i) * ldm;
          double v = Ub[i * ncols + c];
          for (int k = i + 1; k < kb; ++k) v -= Ur[k0 + k] * Ub[k * ncols + c];
          v /= Ur[k0 + i];
          Ub[i * ncols + c] = v;
        }
        for (int i = 0; i < kb; ++i) M[(long long)(k0 + i) * ldm + ni + c] = Ub[i * ncols + c];
      }
      __syncthreads();
    }

    // ---- probe condition estimate (leafops.py:293-294) ----
    double pm = 0.0;
    for (int r = tid; r < ni; r += nt) pm = fmax(pm, fabs(M[(long long)r * ldm + ncols - 1]));
    pm = block_max(pm, red);
    if (tid == 0) a.cond[grp] = anorm * pm / a.probe_max;

    // ---- Psi = -X[:, :nb] ----
    double* Psi = a.Psi + (long long)grp * ni * nb;
    for (int e = tid; e < ni * nb; e += nt) {
      const int r = e / nb, c = e - r * nb;
      Psi[e] = -M[(long long)r * ldm + ni + c];
    }
    __syncthreads();
    // ---- T1 = L43e + L43i Psi  (ng x nb), then T = T1 L1 (ng x ng) ----
    for (int e = tid; e < ng * nb; e += nt) {
      const int i = e / nb, c = e - i * nb;
      const double* Lr = cL43i + (long long)i * ni;
      double dot = 0.0;
      for (int k = 0; k < ni; ++k) dot += Lr[k] * Psi[(long long)k * nb + c];
      T1[e] = cL43e[e] + dot;
    }
    __syncthreads();
    double* T = a.T + (long long)grp * ng * ng;
    for (int e = tid; e < ng * ng; e += nt) {
      const int i = e / ng, c = e - i * ng;
      double dot = 0.0;
      for (int k = 0; k < nb; ++k) dot += T1[i * nb + k] * cL1[k * ng + c];
      T[e] = dot;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// p = 16 fast path (the BASELINE configs): block Gauss-Jordan on the augmented system with implicit
// partial pivoting, register-resident panels and DMMA rank-16 updates.
//
// The augmented matrix M = [A_ii | A_ie | probe] (196 x 257, stored 200 x 260 with zero padding)
// lives in a per-CTA global scratch slot (2 CTAs/SM x 148 x 416 KB, L2-resident). For each panel
// of 16 columns:
//   a. thread r loads its row's panel entries (orig) and factors the panel over the active rows:
//      partial pivoting by block argmax, no physical row swaps;
//   b. W = (L11 U11)^{-1} M[P, trailing]  (16 x <=244, one trailing column per thread);
//   c. M[r, trailing] -= orig_r * W  for every row r not in P: DMMA with A = orig rows (smem),
//      B = W (smem), C = M tile (L2).
// After 13 panels, row p_k of M holds x_k (Gauss-Jordan: no back substitution phase). The DtN
// epilogue T = (L43e + L43i Psi) L1 also runs on DMMA.
// ---------------------------------------------------------------------------------------------
#ifdef HPS_LEAF_PROFILE
__device__ long long g_leaf_prof[1024][8];
#define PROF_T(var) long long var = clock64()
#define PROF_ADD(slot, t0) do { if (threadIdx.x == 0) g_leaf_prof[blockIdx.x][slot] += clock64() - (t0); } while (0)
#else
#define PROF_T(var)
#define PROF_ADD(slot, t0)
#endif
namespace l16 {
constexpr int NI = 196, NB = 60, NG = 64, NCOLS = 257, LDM = 260, MROWS = 200;
constexpr int SA = 20;   // A16 row stride (== 4 mod 16: conflict-free A fragments)
constexpr int SB = 264;  // W row stride (== 8 mod 16: conflict-free B fragments); >= 256 columns
constexpr int ST1 = 68;  // T1 row stride
constexpr int SMEM_D = MROWS * SA + 16 * SB + 16 * 17 + 32;  // doubles
constexpr size_t SMEM = SMEM_D * sizeof(double) + sizeof(int) * (NI + NI + NB) + 64;
}  // namespace l16

template <int THREADS>
__global__ void __launch_bounds__(THREADS, 512 / THREADS) k_leaf16(LeafArgs a) {
  using namespace l16;
  extern __shared__ __align__(16) double sm[];
  __shared__ double redv[32];
  __shared__ int redi[32];
  __shared__ int s_sing;
  double* sA16 = sm;                 // MROWS x SA
  double* sW = sA16 + MROWS * SA;    // 16 x SB
  double* sLU = sW + 16 * SB;        // 16 x 17
  double* sProw = sLU + 16 * 17;     // 2 x 16 (double-buffered pivot row)
  int* sPiv = reinterpret_cast<int*>(sProw + 32);  // NI: pivot row of step k
  int* Ji = sPiv + NI;
  int* Je = Ji + NI;
  // assembly-phase aliases (inside sA16/sW)
  double* coef = sm;                 // 6 * 256
  double* Dx = coef + 6 * 256;       // 4 * 256 (Dx, Dy, Dxx, Dyy)
  double* Dy = Dx + 256;
  double* Dxx = Dy + 256;
  double* Dyy = Dxx + 256;
  double* sT1 = sm;                  // 64 x ST1 (epilogue)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const double* cL43e = a.consts + 4 * 256;
  const double* cL43i = cL43e + NG * NB;
  const double* cL1 = cL43i + NG * NI;
  const double* cprobe = cL1 + NB * NG;
  for (int i = tid; i < NI; i += THREADS) Ji[i] = a.idx[i];
  for (int i = tid; i < NB; i += THREADS) Je[i] = a.idx[NI + i];
  double* M = a.scratch + (long long)blockIdx.x * a.scratch_stride;

  for (int grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    __syncthreads();
    for (int i = tid; i < 4 * 256; i += THREADS) Dx[i] = a.consts[i];
    for (int f = 0; f < 6; ++f) {
      const double* src = a.field[f] ? a.field[f] + (long long)grp * 256 : nullptr;
      for (int i = tid; i < 256; i += THREADS) coef[f * 256 + i] = src ? src[i] : a.scalar[f];
    }
    if (tid == 0) s_sing = 0;
    __syncthreads();
    PROF_T(t_asm);

    // ---- assemble (same per-entry op sequence as leafops.py:217-233) ----
    double rowmax = 0.0;
    for (int r = warp; r < MROWS; r += THREADS / 32) {
      double rs = 0.0;
      double* Mr = M + (long long)r * LDM;
      if (r >= NI) {
        for (int c = lane; c < LDM; c += 32) Mr[c] = 0.0;
        continue;
      }
      const int na = Ji[r], ia = na >> 4, ja = na & 15;
      for (int c = lane; c < LDM; c += 32) {
        double v = 0.0;
        if (c == NCOLS - 1) {
          v = cprobe[r];
        } else if (c < NCOLS - 1) {
          const int nbn = c < NI ? Ji[c] : Je[c - NI];
          const int ib = nbn >> 4, jb = nbn & 15;
          double acc = 0.0;
          if (a.present[0] && ja == jb) acc += coef[0 * 256 + na] * (-Dxx[ia * 16 + ib]);
          if (a.present[1]) acc += coef[1 * 256 + na] * (-2.0 * (Dx[ia * 16 + ib] * Dy[ja * 16 + jb]));
          if (a.present[2] && ia == ib) acc += coef[2 * 256 + na] * (-Dyy[ja * 16 + jb]);
          if (a.present[3] && ja == jb) acc += coef[3 * 256 + na] * Dx[ia * 16 + ib];
          if (a.present[4] && ia == ib) acc += coef[4 * 256 + na] * Dy[ja * 16 + jb];
          if (nbn == na) acc += coef[5 * 256 + na];
          v = acc;
          if (c < NI) rs += fabs(v);
        }
        Mr[c] = v;
      }
      rs = warp_sum(rs);
      rowmax = fmax(rowmax, rs);
    }
    // block max of the row abs-sums (reuse redv)
    rowmax = warp_max(rowmax);
    if (lane == 0) redv[warp] = rowmax;
    __syncthreads();
    double anorm = 0.0;
#pragma unroll
    for (int w = 0; w < THREADS / 32; ++w) anorm = fmax(anorm, redv[w]);
    __syncthreads();

    PROF_ADD(0, t_asm);
    // ---- block Gauss-Jordan, 13 panels ----
    int mystep = -1;
    bool act = tid < NI;
    for (int kp = 0; kp < (NI + 15) / 16; ++kp) {
      const int k0 = kp * 16;
      const int kb = min(16, NI - k0);
      PROF_T(t_pan);
      double orig[16], work[16];
      if (tid < NI) {
        const double2* row = reinterpret_cast<const double2*>(M + (long long)tid * LDM + k0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          double2 v = row[j];
          orig[2 * j] = (2 * j < kb) ? v.x : 0.0;
          orig[2 * j + 1] = (2 * j + 1 < kb) ? v.y : 0.0;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) orig[j] = 0.0;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) work[j] = orig[j];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < kb) {
          double cand = act ? fabs(work[j]) : -1.0;
          int ci = tid;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, cand, o);
            const int oi = __shfl_xor_sync(0xffffffffu, ci, o);
            if (ov > cand || (ov == cand && oi < ci)) { cand = ov; ci = oi; }
          }
          if (lane == 0) { redv[warp] = cand; redi[warp] = ci; }
          __syncthreads();
          {  // every warp reduces the per-warp candidates (identical result): no broadcast barrier
            constexpr int NW = THREADS / 32;
            double v = lane < NW ? redv[lane] : -2.0;
            int vi = lane < NW ? redi[lane] : 0x7fffffff;
#pragma unroll
            for (int o = NW / 2; o > 0; o >>= 1) {
              const double ov = __shfl_xor_sync(0xffffffffu, v, o);
              const int oi = __shfl_xor_sync(0xffffffffu, vi, o);
              if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
            }
            vi = __shfl_sync(0xffffffffu, vi, 0);
            if (tid == 0) sPiv[k0 + j] = vi;
            if (tid == vi) {
              act = false;
              mystep = k0 + j;
              if (work[j] == 0.0) s_sing = 1;
#pragma unroll
              for (int c = 0; c < 16; ++c) sts64(sProw + (j & 1) * 16 + c, work[c]);
            }
          }
          __syncthreads();
          if (act) {
            const double* pr = sProw + (j & 1) * 16;  // double-buffered: no barrier after the update
            const double l = work[j] * fast_rcp(pr[j]);
            work[j] = l;
#pragma unroll
            for (int c = j + 1; c < 16; ++c) work[c] = fma(-l, pr[c], work[c]);
          }
        }
      }
      PROF_ADD(1, t_pan);
      PROF_T(t_w);
      const bool inP = mystep >= k0 && mystep < k0 + kb;
      if (inP) {
        const int r = mystep - k0;
#pragma unroll
        for (int c = 0; c < 16; ++c) sts64(sLU + r * 17 + c, work[c]);
      }
      if (tid < MROWS) {
#pragma unroll
        for (int j = 0; j < 16; ++j) sts64(sA16 + tid * SA + j, (tid < NI && !inP) ? -orig[j] : 0.0);
      }
      __syncthreads();
      // W = U11^{-1} L11^{-1} M[P, c0:]
      const int c0 = k0 + kb;
      const int nT = LDM - c0;
      const int nTp = (nT + 127) & ~127;  // W is padded with zero columns to whole 128-chunks
      for (int cc = tid; cc < nTp; cc += THREADS) {
        double y[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) y[r] = (r < kb && cc < nT) ? M[(long long)sPiv[k0 + r] * LDM + c0 + cc] : 0.0;
#pragma unroll
        for (int r = 1; r < 16; ++r)
#pragma unroll
          for (int b = 0; b < r; ++b) y[r] = fma(-sLU[r * 17 + b], y[b], y[r]);
#pragma unroll
        for (int r = 15; r >= 0; --r) {
          if (r < kb) {
#pragma unroll
            for (int b = r + 1; b < 16; ++b) y[r] = fma(-sLU[r * 17 + b], y[b], y[r]);
            y[r] = y[r] / sLU[r * 17 + r];
          } else {
            y[r] = 0.0;
          }
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) sts64(sW + r * SB + cc, y[r]);
        if (cc < nT)
#pragma unroll
          for (int r = 0; r < 16; ++r)
            if (r < kb) M[(long long)sPiv[k0 + r] * LDM + c0 + cc] = y[r];
      }
      __syncthreads();
      // M[:, c0:] += (-orig) * W on DMMA. Warp = row tiles of 8 (A fragments kept in registers);
      // columns in chunks of 128 = 16 DMMA tiles whose C loads are all issued before the first
      // DMMA, so one L2 round trip covers 16 tiles.
      PROF_ADD(2, t_w);
      PROF_T(t_u);
      const int nchunk = (nT + 127) >> 7;
      for (int item = warp; item < (MROWS / 8) * nchunk; item += THREADS / 32) {
        const int r0 = (item / nchunk) * 8;
        const int cb = (item % nchunk) * 128;
        double af[4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) af[ks] = sA16[(r0 + g) * SA + 4 * ks + tq];
        double* Mr = M + (long long)(r0 + g) * LDM + c0;
        {
          double acc[16][2];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = cb + 8 * j + 2 * tq;
            if (col < nT) {
              const double2 v = *reinterpret_cast<const double2*>(Mr + col);
              acc[j][0] = v.x;
              acc[j][1] = v.y;
            } else {
              acc[j][0] = acc[j][1] = 0.0;
            }
          }
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            if (4 * ks < kb) {
              const double* Wr = sW + (4 * ks + tq) * SB + cb + g;
#pragma unroll
              for (int j = 0; j < 16; ++j) dmma_8x8x4(acc[j][0], acc[j][1], af[ks], Wr[8 * j]);
            }
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int col = cb + 8 * j + 2 * tq;
            if (col < nT) *reinterpret_cast<double2*>(Mr + col) = make_double2(acc[j][0], acc[j][1]);
          }
        }
      }
      PROF_ADD(3, t_u);
      PROF_T(t_ub);
      __syncthreads();
      PROF_ADD(4, t_ub);
    }
    PROF_T(t_ep);

    // ---- X rows in step order; probe condition estimate; Psi = -X[:, :NB] ----
    double* Psi = a.Psi + (long long)grp * NI * NB;
    double pm = 0.0;
    for (int e = tid; e < NI * (NB + 1); e += THREADS) {
      const int k = e / (NB + 1), c = e - k * (NB + 1);
      const double v = M[(long long)sPiv[k] * LDM + NI + c];
      if (c < NB) __stcs(Psi + k * NB + c, -v);
      else pm = fmax(pm, fabs(v));
    }
    pm = warp_max(pm);
    if (lane == 0) redv[warp] = pm;
    __syncthreads();
    if (tid == 0) {
      double m = 0.0;
      for (int w = 0; w < THREADS / 32; ++w) m = fmax(m, redv[w]);
      const double cnd = anorm * m / a.probe_max;
      a.cond[grp] = (s_sing || !isfinite(cnd)) ? INFINITY : cnd;
    }
    __syncthreads();
    // ---- T1 = L43e + L43i Psi (64 x 60), warp = 8 rows x 64 cols ----
    if (warp < 8) {
      const int r0 = warp * 8;
      double acc[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
      const double* Arow = cL43i + (long long)(r0 + g) * NI;
      for (int ks = 0; ks < NI; ks += 4) {
        const double af = __ldg(Arow + ks + tq);
        const double* Brow = Psi + (long long)(ks + tq) * NB;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = 8 * j + g;
          const double bf = col < NB ? Brow[col] : 0.0;
          dmma_8x8x4(acc[j][0], acc[j][1], af, bf);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = 8 * j + 2 * tq;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = col + h;
          sT1[(r0 + g) * ST1 + cc] = cc < NB ? __ldg(cL43e + (r0 + g) * NB + cc) + acc[j][h] : 0.0;
        }
      }
    }
    __syncthreads();
    // ---- T = T1 L1 (64 x 64), K = 60 ----
    if (warp < 8) {
      const int r0 = warp * 8;
      double acc[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
      for (int ks = 0; ks < NB; ks += 4) {
        const double af = sT1[(r0 + g) * ST1 + ks + tq];
        const double* Brow = cL1 + (ks + tq) * NG;
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_8x8x4(acc[j][0], acc[j][1], af, __ldg(Brow + 8 * j + g));
      }
      double* T = a.T + (long long)grp * NG * NG;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        __stcs(reinterpret_cast<double2*>(T + (r0 + g) * NG + 8 * j + 2 * tq), make_double2(acc[j][0], acc[j][1]));
    }
    PROF_ADD(5, t_ep);
  }
}

size_t leaf_smem_bytes(int p) {
  const int p2 = p * p, ni = (p - 2) * (p - 2), nb = 4 * (p - 1), ng = 4 * p, ncols = ni + nb + 1;
  return sizeof(double) * (6 * p2 + 4 * p2 + ni * LEAF_NB + LEAF_NB * ncols + ng * nb) +
         sizeof(int) * (2 * ni + nb) + 64;
}

int leaf_grid(int ngroups) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max(1, std::min(ngroups, sms));
}

}  // namespace hps

using namespace hps;

static int leaf16_threads() {
  static int t = getenv("HPS_LEAF16_THREADS") ? atoi(getenv("HPS_LEAF16_THREADS")) : 256;
  return t == 512 ? 512 : 256;
}
static int leaf16_grid(int ngroups) {
  static int per_sm = getenv("HPS_LEAF_CTAS_PER_SM") ? atoi(getenv("HPS_LEAF_CTAS_PER_SM"))
                                                     : (leaf16_threads() == 512 ? 1 : 2);
  return std::max(1, std::min(ngroups, per_sm * leaf_grid(1 << 30)));
}

#ifdef HPS_LEAF_PROFILE
extern "C" int hps_debug_leaf_profile(long long* out, int reset) {
  if (reset) {
    static long long z[1024][8] = {};
    cudaMemcpyToSymbol(g_leaf_prof, z, sizeof(z));
    return 0;
  }
  cudaMemcpyFromSymbol(out, g_leaf_prof, sizeof(long long) * 1024 * 8);
  return 0;
}
#endif

extern "C" size_t hps_leaf_workspace_bytes(int p, int ngroups) {
  if (p == 16)
    return sizeof(double) * std::max((size_t)leaf16_grid(ngroups) * l16::MROWS * l16::LDM,
                                     (size_t)leaf16v3_grid(ngroups) * leaf16v3_scratch_doubles()) + 256;
  const int ni = (p - 2) * (p - 2), nb = 4 * (p - 1);
  const long long ldm = ni + nb + 2;
  return sizeof(double) * (size_t)leaf_grid(ngroups) * ni * ldm + 256;
}

// Optional L2 persistence window over the per-CTA leaf scratch (HPS_LEAF_L2PERSIST=1): the scratch
// is re-read and re-written by every panel, everything else is touched once. Reset on scope exit.
struct L2Window {
  cudaStream_t st;
  bool on = false;
  L2Window(cudaStream_t s, void* base, size_t bytes) : st(s) {
    static const int persist = getenv("HPS_LEAF_L2PERSIST") ? atoi(getenv("HPS_LEAF_L2PERSIST")) : 0;
    if (!persist) return;
    int dev = 0, maxp = 0, maxw = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (maxp <= 0 || maxw <= 0) return;
    const size_t win = std::min(bytes, (size_t)maxw);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min((size_t)maxp, win));
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = base;
    v.accessPolicyWindow.num_bytes = win;
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)maxp / (double)win);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    on = cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
    cudaGetLastError();
  }
  ~L2Window() {
    if (!on) return;
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
    cudaGetLastError();
  }
};

extern "C" int hps_leaf_stage(int p, int ngroups, const double* const* fields, const double* scalars,
                              const double* consts, const int* idx, double probe_max, double* Psi, double* T,
                              double* cond, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ngroups <= 0) return HPS_OK;
  if (p < 3 || p > 32 || ws_bytes < hps_leaf_workspace_bytes(p, ngroups)) {
    set_error("hps_leaf_stage: bad arguments p=%d ws=%zu", p, ws_bytes);
    return HPS_ERR_ARG;
  }
  LeafArgs a{};
  a.p = p;
  a.ngroups = ngroups;
  for (int f = 0; f < 6; ++f) {
    a.field[f] = fields[f];
    a.scalar[f] = scalars[f];
    a.present[f] = fields[f] != nullptr || scalars[f] != 0.0;
  }
  a.consts = consts;
  a.idx = idx;
  a.probe_max = probe_max;
  a.Psi = Psi;
  a.T = T;
  a.cond = cond;
  const int ni = (p - 2) * (p - 2), nb = 4 * (p - 1);
  a.scratch = static_cast<double*>(ws);
  static const int leaf_v = getenv("HPS_LEAF_V") ? atoi(getenv("HPS_LEAF_V")) : 3;
  if (p == 16 && !getenv("HPS_LEAF_GENERIC") && leaf_v == 3) {
    L2Window window(st, ws, (size_t)leaf16v3_grid(ngroups) * leaf16v3_scratch_doubles() * sizeof(double));
    return launch_leaf16v3(a, st);
  }
  if (p == 16 && !getenv("HPS_LEAF_GENERIC")) {
    a.scratch_stride = (long long)l16::MROWS * l16::LDM;
    static bool attr = false;
    if (!attr) {
      HPS_CUDA_CHECK(cudaFuncSetAttribute(k_leaf16<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l16::SMEM));
      HPS_CUDA_CHECK(cudaFuncSetAttribute(k_leaf16<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)l16::SMEM));
      attr = true;
    }
    // Keep as much of the per-CTA scratch in L2 as the persisting carve-out allows: the scratch is
    // re-read and re-written by every panel, everything else is touched once.
    L2Window window(st, ws, (size_t)leaf16_grid(ngroups) * a.scratch_stride * sizeof(double));
    if (leaf16_threads() == 512)
      k_leaf16<512><<<leaf16_grid(ngroups), 512, l16::SMEM, st>>>(a);
    else
      k_leaf16<256><<<leaf16_grid(ngroups), 256, l16::SMEM, st>>>(a);
    HPS_LAUNCH_CHECK();
    return HPS_OK;
  }
  a.scratch_stride = (long long)ni * (ni + nb + 2);
  const size_t smem = leaf_smem_bytes(p);
  HPS_CUDA_CHECK(cudaFuncSetAttribute(k_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_leaf<<<leaf_grid(ngroups), LEAF_THREADS, smem, st>>>(a);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}
