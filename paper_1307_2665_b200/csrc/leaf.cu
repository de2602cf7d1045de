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
#include "ctx.cuh"
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

size_t leaf_smem_bytes(int p) {
  const int p2 = p * p, ni = (p - 2) * (p - 2), nb = 4 * (p - 1), ng = 4 * p, ncols = ni + nb + 1;
  return sizeof(double) * (6 * p2 + 4 * p2 + ni * LEAF_NB + LEAF_NB * ncols + ng * nb) +
         sizeof(int) * (2 * ni + nb) + 64;
}

int leaf_grid(const Ctx& cx, int ngroups) { return std::max(1, std::min(ngroups, cx.sms)); }

}  // namespace hps

using namespace hps;

extern "C" size_t hps_leaf_workspace_bytes(hps_ctx_t ctx, int p, int ngroups) {
  // ctx NULL: the sizes for a default context on a 148-SM B200 (a host-only query)
  static const Ctx dflt;
  const Ctx* cx = ctx ? reinterpret_cast<const Ctx*>(ctx) : &dflt;
  if (p == 16) return sizeof(double) * (size_t)leaf16v3_grid(*cx, ngroups) * leaf16v3_scratch_doubles() + 256;
  const int ni = (p - 2) * (p - 2), nb = 4 * (p - 1);
  const long long ldm = ni + nb + 2;
  return sizeof(double) * (size_t)leaf_grid(*cx, ngroups) * ni * ldm + 256;
}

extern "C" int hps_leaf_stage(hps_ctx_t ctx, int p, int ngroups, const double* const* fields, const double* scalars,
                              const double* consts, const int* idx, double probe_max, double* Psi, double* T,
                              double* cond, void* ws, size_t ws_bytes, void* stream) {
  HPS_CTX(cx, ctx);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ngroups <= 0) return HPS_OK;
  if (p < 3 || p > 32 || ws_bytes < hps_leaf_workspace_bytes(ctx, p, ngroups)) {
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
  if (p == 16) return launch_leaf16v3(a, *cx, st);
  a.scratch_stride = (long long)ni * (ni + nb + 2);
  const size_t smem = leaf_smem_bytes(p);
  const int as = ensure_smem_attr((const void*)k_leaf, cx->device, (int)smem);
  if (as != HPS_OK) return as;
  k_leaf<<<leaf_grid(*cx, ngroups), LEAF_THREADS, smem, st>>>(a);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}
