// Leaf stage, p = 16, v3: right-looking blocked LU with implicit partial pivoting and look-ahead.
// Reference math: leafops.py:217-302, solver.py:226-246. Same outputs as the v2/generic kernels:
// Psi = -A_ii^{-1} A_ie, the probe condition estimate, and T = (L43e + L43i Psi) L1.
//
// One CTA per coefficient group, 2 CTAs per SM, 8 warps in two roles:
//   * panel warps 0-3 own physical rows (thread t: rows t and t+128) and factor a 16-column panel
//     in registers. Partial pivoting: a REDUX argmax over the active rows. No row swaps: a pivot
//     row just leaves the active set.
//   * update warps 4-7 apply the rank-16 update of the previous panel on DMMA, over the compact
//     list of still-active rows only. They update the next panel's columns first, then signal
//     the panel warps through a named barrier, so factor(k+1) overlaps update(k) on the
//     remaining columns.
// After the last panel, a blocked back substitution (leaf3_backsub: Y staged in shared memory,
// precomputed inverses of the 16x16 diagonal blocks, everything on DMMA) yields X = U^{-1} Y.
// The augmented matrix lives in a per-CTA global scratch slot (200 x 260 fp64, L2-resident),
// followed by the 13 diagonal-block inverses.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "ctx.cuh"
#include "leaf.cuh"

namespace hps {
#ifdef HPS_LEAF_PROFILE
__device__ long long g_leaf3_prof[1024][16];
#define P3_T(v) long long v = clock64()
#define P3_ADD(slot, t0, who) do { if ((who)) atomicAdd((unsigned long long*)&g_leaf3_prof[blockIdx.x][slot], (unsigned long long)(clock64() - (t0))); } while (0)
#else
#define P3_T(v)
#define P3_ADD(slot, t0, who)
#endif
namespace l3 {
constexpr int NI = 196, NB = 60, NG = 64, NCOLS = 257, LDM = 260, MROWS = 200;
constexpr int THREADS = 256;
constexpr int NPW = 4;  // panel warps
constexpr int SA = 20;  // multiplier row stride (== 4 mod 16)
constexpr int SB = 260; // U12 row stride (== 4 mod 16: the DMMA B-fragment loads are conflict-free)
constexpr int ST1 = 68;
constexpr int NPANEL = (NI + 15) / 16;  // 13
constexpr int OFF_A16 = 0;                         // 2 x MROWS x SA
constexpr int OFF_U12 = OFF_A16 + 2 * MROWS * SA;  // 16 x SB
constexpr int OFF_LU = OFF_U12 + 16 * SB;          // 16 x 17
constexpr int OFF_PROW = OFF_LU + 16 * 17;         // 2 x 16
constexpr int BS_OFF_U = NI * 64;                  // back substitution: Y (NI x 64), then 2 x Uinv
constexpr int NDBL = std::max(OFF_PROW + 32, BS_OFF_U + 2 * 16 * 20);
constexpr int NINT = 2 * MROWS + NI + NI + NB + 64;
constexpr size_t SMEM = (size_t)NDBL * 8 + (size_t)NINT * 4 + 64;
constexpr int BAR_PANEL = 1;      // panel warps only (128 threads)
}  // namespace l3



// Back substitution X = U^{-1} Y for the 13 pivot blocks, Psi = -X out, T1 = L43e + L43i Psi staged
// in shared memory (64 x ST1 at OFF_U12) for the T epilogue. Returns this thread's max |X[:, probe]|.
__device__ __noinline__ double leaf3_backsub(double* __restrict__ M, const int* __restrict__ sPiv, double* __restrict__ Psi,
                                             const double* __restrict__ cL43i, const double* __restrict__ cL43e) {
  using namespace l3;
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  (void)lane;
    // ================= back substitution (right-looking), fused with T1 = L43i Psi =================
    // Y (the 64 right-hand-side columns of every pivot row, in pivot-step order) is staged once
    // into shared memory (XOR-swizzled rows of 64), so the 13-block chain never waits on L2.
    //   once:   Uinv_k = U11_k^{-1} for all 13 diagonal blocks (one column per thread), to global;
    //   per block, from the last:
    //     X_kp = Uinv_kp Y_kp on DMMA (warp w: columns 8w..8w+7, in place), Psi rows out;
    //     T1 += L43i[:, blk] (-X_kp) and Y_j -= U[P_j, blk] X_kp (j < kp), all warps on DMMA, with
    //     Uinv (cp.async) and the U / L43i fragments (registers) loaded one block ahead.
    double* sYb = sm;                       // NI x 64 (swizzled)
    double* sUb = sm + BS_OFF_U;            // 2 x 16 x SUI: Uinv of the block (cp.async)
    constexpr int SUI = 20;                 // == 4 mod 16: conflict-free A fragments
    double* UinvG = M + (long long)MROWS * LDM;  // 13 x 16 x 16 in the CTA's scratch slot
    auto yidx = [](int r, int c) { return r * 64 + (c ^ ((r & 7) << 3)); };
    double t1acc[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) t1acc[j][0] = t1acc[j][1] = 0.0;
    double pm = 0.0;
    P3_T(t_st);
    {  // U11 blocks -> smem (13 x 16 x 16, zero outside the block), then Uinv columns -> global
      for (int e = tid; e < NPANEL * 128; e += THREADS) {
        const int blk = e >> 7, r = (e >> 3) & 15, c = (e & 7) * 2, k0 = 16 * blk, kb = min(16, NI - k0);
        double2 v = make_double2(0.0, 0.0);
        if (r < kb) v = *reinterpret_cast<const double2*>(M + (long long)sPiv[k0 + r] * LDM + k0 + c);
        if (c >= kb) v.x = 0.0;
        if (c + 1 >= kb) v.y = 0.0;
        *reinterpret_cast<double2*>(sm + blk * 256 + r * 16 + c) = v;
      }
      __syncthreads();
      if (tid < NPANEL * 16) {
        const int blk = tid >> 4, c = tid & 15, kb = min(16, NI - 16 * blk);
        const double* U = sm + blk * 256;
        double v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = r == c ? 1.0 : 0.0;
#pragma unroll
        for (int r = 15; r >= 0; --r) {
          if (r <= c && r < kb) {
            const double x = v[r] * fast_rcp(U[r * 16 + r]);
            v[r] = x;
#pragma unroll
            for (int b = 0; b < r; ++b) v[b] = fma(-U[b * 16 + r], x, v[b]);
          }
        }
        double* out = UinvG + blk * 256 + c;
#pragma unroll
        for (int r = 0; r < 16; ++r) out[r * 16] = (c < kb && r < kb) ? v[r] : 0.0;
      }
      __syncthreads();  // Uinv (global) visible to the cp.async readers below; U11 staging dead
    }
    auto load_uinv = [&](int kp, int buf) {  // 16 rows x 16 doubles, 8 x 16 B per row (threads 0-127)
      if (tid < 128) {
        const int r = tid >> 3, c = (tid & 7) * 2;
        cp_async16(sUb + buf * 16 * SUI + r * SUI + c, UinvG + kp * 256 + r * 16 + c, true);
      }
      cp_async_commit();
    };
    // A fragments loaded into registers one block ahead: U[P_j, blk] for this warp's Y-update
    // items (it = warp + 8m) and -L43i[8w+g, blk] for its T1 rows
    double afU[3][4], afT[4];
    auto load_frags = [&](int kp) {
      const int k0 = 16 * kp, kb = min(16, NI - k0);
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int ri = (warp + 8 * m) * 8 + g;
        const bool rv = ri < k0;
        const double* Urow = M + (long long)(rv ? sPiv[ri] : 0) * LDM + k0;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) afU[m][ks] = (rv && 4 * ks < kb) ? Urow[4 * ks + tq] : 0.0;
      }
      const double* Arow = cL43i + (long long)(warp * 8 + g) * NI + k0;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) afT[ks] = 4 * ks < kb ? -__ldg(Arow + 4 * ks + tq) : 0.0;
    };
    load_uinv(NPANEL - 1, (NPANEL - 1) & 1);
    load_frags(NPANEL - 1);
    for (int e = tid; e < NI * 32; e += THREADS) {
      const int r = e >> 5, c = (e & 31) * 2;
      const double2 v = *reinterpret_cast<const double2*>(M + (long long)sPiv[r] * LDM + NI + c);
      *reinterpret_cast<double2*>(sYb + yidx(r, c)) = v;
    }
    for (int kp = NPANEL - 1; kp >= 0; --kp) {
      const int k0 = 16 * kp, kb = min(16, NI - k0), buf = kp & 1;
      if (kp == NPANEL - 1) P3_ADD(10, t_st, tid == 0);
      P3_T(t_w);
      cp_async_wait<0>();
      __syncthreads();  // Y_kp final, Uinv_kp staged, previous block's readers done
      P3_ADD(11, t_w, tid == 0);
      P3_T(t_s);
      if (kp > 0) load_uinv(kp - 1, buf ^ 1);
      {  // X_kp = Uinv_kp Y_kp: this warp's 8 columns, both 8-row halves, in place
        const double* Ui = sUb + buf * 16 * SUI;
        double x0[2] = {0.0, 0.0}, x1[2] = {0.0, 0.0};
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          if (4 * ks < kb) {
            const double b = sYb[yidx(k0 + 4 * ks + tq, 8 * warp + g)];
            dmma_8x8x4(x0[0], x0[1], Ui[g * SUI + 4 * ks + tq], b);
            dmma_8x8x4(x1[0], x1[1], Ui[(g + 8) * SUI + 4 * ks + tq], b);
          }
        __syncwarp();
        const int col = 8 * warp + 2 * tq;
        if (g < kb) {
          *reinterpret_cast<double2*>(sYb + yidx(k0 + g, col)) = make_double2(x0[0], x0[1]);
          if (col < NB) __stcs(reinterpret_cast<double2*>(Psi + (long long)(k0 + g) * NB + col), make_double2(-x0[0], -x0[1]));
        }
        if (g + 8 < kb) {
          *reinterpret_cast<double2*>(sYb + yidx(k0 + g + 8, col)) = make_double2(x1[0], x1[1]);
          if (col < NB) __stcs(reinterpret_cast<double2*>(Psi + (long long)(k0 + g + 8) * NB + col), make_double2(-x1[0], -x1[1]));
        }
        if (col == NB) pm = fmax(pm, fmax(g < kb ? fabs(x0[0]) : 0.0, g + 8 < kb ? fabs(x1[0]) : 0.0));
      }
      __syncthreads();
      P3_ADD(12, t_s, tid == 0);
      P3_T(t_u);
      // T1 rows 8w..8w+7 += L43i[:, blk] (-X_kp)
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        if (4 * ks < kb) {
          const int xr = k0 + 4 * ks + tq;
#pragma unroll
          for (int j = 0; j < 8; ++j) dmma_8x8x4(t1acc[j][0], t1acc[j][1], afT[ks], sYb[yidx(xr, 8 * j + g)]);
        }
      // Y_j -= U[P_j, blk] X_kp for the pivot steps j < k0 (8-row items it = warp + 8m)
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int it = warp + 8 * m;
        if (it * 8 < k0) {
          const int yr = it * 8 + g;
          double acc[8][2];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double2 v = *reinterpret_cast<const double2*>(sYb + yidx(yr, 8 * j + 2 * tq));
            acc[j][0] = v.x;
            acc[j][1] = v.y;
          }
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            if (4 * ks < kb) {
              const double af = -afU[m][ks];
              const int xr = k0 + 4 * ks + tq;
#pragma unroll
              for (int j = 0; j < 8; ++j) dmma_8x8x4(acc[j][0], acc[j][1], af, sYb[yidx(xr, 8 * j + g)]);
            }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<double2*>(sYb + yidx(yr, 8 * j + 2 * tq)) = make_double2(acc[j][0], acc[j][1]);
        }
      }
      if (kp > 0) load_frags(kp - 1);  // in flight across the next block's barrier + solve
      P3_ADD(13, t_u, tid == 0);
    }
    __syncthreads();
    // T1 (+ L43e) -> smem
    double* sT1 = sm + OFF_U12;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int col = 8 * j + 2 * tq;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = col + h;
        sT1[(warp * 8 + g) * ST1 + cc] = cc < NB ? __ldg(cL43e + (warp * 8 + g) * NB + cc) + t1acc[j][h] : 0.0;
      }
    }
    return pm;
}

__global__ void __launch_bounds__(l3::THREADS, 2) k_leaf16v3(LeafArgs a) {
  using namespace l3;
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long s_key[NPW];
  __shared__ int s_idx[NPW];
  __shared__ int s_cnt[2 * NPW];
  __shared__ int s_nact[2];
  __shared__ int s_sing;
  __shared__ int s_next;  // work-stealing counter for the trailing update
  __shared__ double s_red[8];
  double* sA16 = sm + OFF_A16;
  double* sU12 = sm + OFF_U12;
  double* sLU = sm + OFF_LU;
  double* sProw = sm + OFF_PROW;
  int* ib = reinterpret_cast<int*>(sm + NDBL);
  int* sAct = ib;               // 2 x MROWS
  int* sPiv = sAct + 2 * MROWS; // NI: physical row eliminated at step k
  int* Ji = sPiv + NI;
  int* Je = Ji + NI;
  // assembly-phase aliases
  double* coef = sA16;          // 6 x 256
  double* Dx = coef + 6 * 256;  // Dx, Dy, Dxx, Dyy
  double* Dy = Dx + 256;
  double* Dxx = Dy + 256;
  double* Dyy = Dxx + 256;
  int* colmap = sAct;           // node (i, j) -> M column, at [i * 17 + j] (272 <= 2 * MROWS)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  // the panel warps are the CTA's LAST warps: the issue arbiter favours the highest warp id, and the
  // pivot chain they run is the critical path
  const bool pwarp = warp >= THREADS / 32 - NPW;
  const int pw = warp - (THREADS / 32 - NPW), ptid = tid - 32 * (THREADS / 32 - NPW);
  const double* cL43e = a.consts + 4 * 256;
  const double* cL43i = cL43e + NG * NB;
  const double* cL1 = cL43i + NG * NI;
  const double* cprobe = cL1 + NB * NG;
  for (int i = tid; i < NI; i += THREADS) Ji[i] = a.idx[i];
  for (int i = tid; i < NB; i += THREADS) Je[i] = a.idx[NI + i];
  double* M = a.scratch + (long long)blockIdx.x * a.scratch_stride;

  for (int grp = blockIdx.x; grp < a.ngroups; grp += gridDim.x) {
    __syncthreads();
    // ================= assembly (leafops.py:217-233, same per-entry op order) =================
    P3_T(t_asm);
    for (int i = tid; i < 4 * 256; i += THREADS) Dx[i] = a.consts[i];
    for (int f = 0; f < 6; ++f) {
      const double* src = a.field[f] ? a.field[f] + (long long)grp * 256 : nullptr;
      for (int i = tid; i < 256; i += THREADS) coef[f * 256 + i] = src ? src[i] : a.scalar[f];
    }
    for (int i = tid; i < 16 * 17; i += THREADS) colmap[i] = -1;
    if (tid == 0) s_sing = 0;
    __syncthreads();
    for (int i = tid; i < NI; i += THREADS) colmap[(Ji[i] >> 4) * 17 + (Ji[i] & 15)] = i;
    for (int i = tid; i < NB; i += THREADS) colmap[(Je[i] >> 4) * 17 + (Je[i] & 15)] = NI + i;
    // zero-fill M (vectorised), probe column
    for (int e = tid; e < MROWS * LDM / 2; e += THREADS)
      reinterpret_cast<double2*>(M)[e] = make_double2(0.0, 0.0);
    __syncthreads();
    const bool dense = a.present[1] != 0;  // c12 != 0 couples every (i', j'): dense rows
    double rowmax = 0.0;
    for (int r = warp; r < NI; r += THREADS / 32) {
      double* Mr = M + (long long)r * LDM;
      const int na = Ji[r], ia = na >> 4, ja = na & 15;
      double rs = 0.0;
      auto entry = [&](int ib_, int jb_) {
        double acc = 0.0;
        if (a.present[0] && ja == jb_) acc += coef[0 * 256 + na] * (-Dxx[ia * 16 + ib_]);
        if (a.present[1]) acc += coef[1 * 256 + na] * (-2.0 * (Dx[ia * 16 + ib_] * Dy[ja * 16 + jb_]));
        if (a.present[2] && ia == ib_) acc += coef[2 * 256 + na] * (-Dyy[ja * 16 + jb_]);
        if (a.present[3] && ja == jb_) acc += coef[3 * 256 + na] * Dx[ia * 16 + ib_];
        if (a.present[4] && ia == ib_) acc += coef[4 * 256 + na] * Dy[ja * 16 + jb_];
        if (ib_ == ia && jb_ == ja) acc += coef[5 * 256 + na];
        return acc;
      };
      if (dense) {
        for (int c = lane; c < NCOLS - 1; c += 32) {
          const int nbn = c < NI ? Ji[c] : Je[c - NI];
          const double v = entry(nbn >> 4, nbn & 15);
          Mr[c] = v;
          if (c < NI) rs += fabs(v);
        }
      } else {
        // nonzeros only: the grid row (ib, ja) and the grid column (ia, jb) through node (ia, ja)
        const int which = lane >> 4, t = lane & 15;  // lanes 0-15: vary ib; 16-31: vary jb (skip the diagonal)
        const int ib_ = which == 0 ? t : ia, jb_ = which == 0 ? ja : t;
        if (!(which == 1 && t == ja)) {
          const int col = colmap[ib_ * 17 + jb_];
          const double v = entry(ib_, jb_);
          Mr[col] = v;
          if (col < NI) rs += fabs(v);
        }
      }
      if (lane == 0) Mr[NCOLS - 1] = cprobe[r];
      rs = warp_sum(rs);
      rowmax = fmax(rowmax, rs);
    }
    rowmax = warp_max(rowmax);
    if (lane == 0) s_red[warp] = rowmax;
    __syncthreads();
    double anorm = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) anorm = fmax(anorm, s_red[w]);

    // ================= blocked LU with look-ahead =================
    // panel-warp state: rows r0 = ptid, r1 = ptid + 128
    const int r0 = ptid, r1 = ptid + 128;
    // a row is active until it becomes a pivot row (step >= 0); derived, not stored, to save registers
#define act0 (step0 < 0 && pwarp)
#define act1 (step1 < 0 && pwarp && ptid < NI - 128)
    int step0 = -1, step1 = -1;
    int cidx0 = -1, cidx1 = -1;  // compact index of r0 / r1 in the last active list

    auto factor = [&](int k) {  // panel warps only
      const int k0 = 16 * k, kb = min(16, NI - k0);
      double w0[16], w1[16];
#pragma unroll
      for (int j = 0; j < 16; j += 2) {
        double2 v0 = make_double2(0.0, 0.0), v1 = make_double2(0.0, 0.0);
        if (act0 && j < kb) v0 = *reinterpret_cast<const double2*>(M + (long long)r0 * LDM + k0 + j);
        if (act1 && j < kb) v1 = *reinterpret_cast<const double2*>(M + (long long)r1 * LDM + k0 + j);
        w0[j] = v0.x; w0[j + 1] = (j + 1 < kb) ? v0.y : 0.0;
        w1[j] = v1.x; w1[j + 1] = (j + 1 < kb) ? v1.y : 0.0;
      }
      if (k > 0) {  // apply panel k-1's rank-16 update to this panel's columns of my rows (registers)
        const int kbp = 16;  // every panel but the last is full
        const double* Ap = sA16 + ((k - 1) & 1) * MROWS * SA;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < kbp) {
            const double a0 = act0 ? Ap[cidx0 * SA + j] : 0.0;
            const double a1 = act1 ? Ap[cidx1 * SA + j] : 0.0;
            const double* Ur = sU12 + j * SB;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const double u = Ur[c];
              w0[c] = fma(a0, u, w0[c]);
              w1[c] = fma(a1, u, w1[c]);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c >= kb) { w0[c] = 0.0; w1[c] = 0.0; }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < kb) {
          const unsigned long long k0key = act0 ? (unsigned long long)__double_as_longlong(fabs(w0[j])) : 0ull;
          const unsigned long long k1key = act1 ? (unsigned long long)__double_as_longlong(fabs(w1[j])) : 0ull;
          unsigned long long key = k0key;
          int idx = act0 ? r0 : 0x7fffffff;
          if (act1 && (k1key > key || (k1key == key && r1 < idx))) { key = k1key; idx = r1; }
          const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
          const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
          const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
          const int wi = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)idx : 0xffffffffu);
          if (lane == 0) {
            s_key[pw] = ((unsigned long long)mhi << 32) | mlo;
            s_idx[pw] = wi;
          }
          bar_sync(BAR_PANEL, NPW * 32);
          unsigned long long bk = s_key[0];
          int p = s_idx[0];
#pragma unroll
          for (int w = 1; w < NPW; ++w) {
            const unsigned long long kk = s_key[w];
            const int ii = s_idx[w];
            if (kk > bk || (kk == bk && ii < p)) { bk = kk; p = ii; }
          }
          double* pr = sProw + (j & 1) * 16;
          if (r0 == p) {
            step0 = k0 + j;
            if (w0[j] == 0.0) s_sing = 1;
#pragma unroll
            for (int c = 0; c < 16; ++c) sts64(pr + c, w0[c]);
          }
          if (r1 == p) {
            step1 = k0 + j;
            if (w1[j] == 0.0) s_sing = 1;
#pragma unroll
            for (int c = 0; c < 16; ++c) sts64(pr + c, w1[c]);
          }
          if (ptid == 0) sPiv[k0 + j] = p;
          bar_sync(BAR_PANEL, NPW * 32);
          const double inv = fast_rcp(pr[j]);
          if (act0) {
            const double l = w0[j] * inv;
            w0[j] = l;
#pragma unroll
            for (int c = j + 1; c < 16; ++c) w0[c] = fma(-l, pr[c], w0[c]);
          }
          if (act1) {
            const double l = w1[j] * inv;
            w1[j] = l;
#pragma unroll
            for (int c = j + 1; c < 16; ++c) w1[c] = fma(-l, pr[c], w1[c]);
          }
        }
      }
      // pivot rows of this panel: LU11 rows to smem, U part into M
      if (step0 >= k0 && step0 < k0 + kb) {
        const int rr = step0 - k0;
#pragma unroll
        for (int c = 0; c < 16; ++c) sts64(sLU + rr * 17 + c, w0[c]);
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c >= rr && c < kb) M[(long long)r0 * LDM + k0 + c] = w0[c];
      }
      if (step1 >= k0 && step1 < k0 + kb) {
        const int rr = step1 - k0;
#pragma unroll
        for (int c = 0; c < 16; ++c) sts64(sLU + rr * 17 + c, w1[c]);
#pragma unroll
        for (int c = 0; c < 16; ++c)
          if (c >= rr && c < kb) M[(long long)r1 * LDM + k0 + c] = w1[c];
      }
      // compact list of rows still active, with their (negated) multipliers for the update
      const unsigned b0 = __ballot_sync(0xffffffffu, act0), b1 = __ballot_sync(0xffffffffu, act1);
      if (lane == 0) { s_cnt[pw] = __popc(b0); s_cnt[NPW + pw] = __popc(b1); }
      bar_sync(BAR_PANEL, NPW * 32);
      int off0 = 0, off1 = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < NPW; ++w) {
        if (w < pw) { off0 += s_cnt[w]; off1 += s_cnt[NPW + w]; }
        tot += s_cnt[w];
      }
      off1 += tot;
#pragma unroll
      for (int w = 0; w < NPW; ++w) tot += s_cnt[NPW + w];
      const unsigned lt = (1u << lane) - 1u;
      const int buf = k & 1;
      int* act = sAct + buf * MROWS;
      double* A16 = sA16 + buf * MROWS * SA;
      if (act0) {
        const int i = off0 + __popc(b0 & lt);
        cidx0 = i;
        act[i] = r0;
#pragma unroll
        for (int j = 0; j < 16; ++j) sts64(A16 + i * SA + j, j < kb ? -w0[j] : 0.0);
      }
      if (act1) {
        const int i = off1 + __popc(b1 & lt);
        cidx1 = i;
        act[i] = r1;
#pragma unroll
        for (int j = 0; j < 16; ++j) sts64(A16 + i * SA + j, j < kb ? -w1[j] : 0.0);
      }
      if (ptid == 0) s_nact[buf] = tot;
    };

#undef act0
#undef act1
    // rank-kb update of M[act rows][c0 + [cbeg, cend)] by the update warps (uw = 0..3). Work item:
    // 8 rows x CW columns whose C loads are all issued before the DMMAs (one L2 round trip); CW = 64
    // keeps a warp's DMMA burst at 32, so the panel warps' FP64 operations queue behind less.
    // uw >= 0: static round-robin over 4 update warps; uw < 0: pull items from s_next (any warp).
    auto update = [&](int k, int cbeg, int cend, int uw) {
#ifndef HPS_LEAF_CW
#define HPS_LEAF_CW 64  // 128: 4-5% slower once the panel warps have issue priority (longer DMMA bursts ahead of their FP64 ops); 32: the same as 64
#endif
      constexpr int CW = HPS_LEAF_CW, NJ = CW / 8;
      const int k0 = 16 * k, kb = min(16, NI - k0), c0 = k0 + kb, nT = LDM - c0;
      const int buf = k & 1;
      const int nact = s_nact[buf];
      const int* act = sAct + buf * MROWS;
      const double* A16 = sA16 + buf * MROWS * SA;
      const int nrt = (nact + 7) >> 3;
      const int ncw = (cend - cbeg + CW - 1) / CW;
      const int lim = min(cend, nT);
      const int nitems = nrt * ncw;
      for (int it = uw >= 0 ? uw : 0;;) {
        if (uw < 0) {
          int v = 0;
          if (lane == 0) v = atomicAdd(&s_next, 1);
          it = __shfl_sync(0xffffffffu, v, 0);
        }
        if (it >= nitems) break;
        const int rt = it / ncw, cb = cbeg + (it - rt * ncw) * CW;
        const int ri = rt * 8 + g;
        const bool rv = ri < nact;
        const int row = rv ? act[ri] : 0;
        double af[4];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) af[ks] = rv ? A16[ri * SA + 4 * ks + tq] : 0.0;
        double* Mr = M + (long long)row * LDM + c0;
        double acc[NJ][2];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int col = cb + 8 * j + 2 * tq;
          if (rv && col < lim) {
            const double2 v = *reinterpret_cast<const double2*>(Mr + col);
            acc[j][0] = v.x;
            acc[j][1] = v.y;
          } else {
            acc[j][0] = acc[j][1] = 0.0;
          }
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          if (4 * ks < kb) {
            const double* Ur = sU12 + (4 * ks + tq) * SB + cb + g;
#pragma unroll
            for (int j = 0; j < NJ; ++j)
              if (cb + 8 * j < lim) dmma_8x8x4(acc[j][0], acc[j][1], af[ks], Ur[8 * j]);
          }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int col = cb + 8 * j + 2 * tq;
          if (rv && col < lim) *reinterpret_cast<double2*>(Mr + col) = make_double2(acc[j][0], acc[j][1]);
        }
        if (uw >= 0) it += 4;
      }
    };

    P3_ADD(0, t_asm, tid == 0);
    P3_T(t_f0);
    if (pwarp) factor(0);
    __syncthreads();
    P3_ADD(1, t_f0, tid == 0);
    for (int k = 0; k < NPANEL; ++k) {
      P3_T(t_u12);
      const int k0 = 16 * k, kb = min(16, NI - k0), c0 = k0 + kb, nT = LDM - c0;
      // U12 = L11^{-1} M[P_k, c0:] (one trailing column per thread)
      for (int cc = tid; cc < 256; cc += THREADS) {
        double y[16];
#pragma unroll
        for (int r = 0; r < 16; ++r)
          y[r] = (r < kb && cc < nT) ? M[(long long)sPiv[k0 + r] * LDM + c0 + cc] : 0.0;
#pragma unroll
        for (int r = 1; r < 16; ++r)
          if (r < kb)
#pragma unroll
            for (int b = 0; b < r; ++b) y[r] = fma(-sLU[r * 17 + b], y[b], y[r]);
#pragma unroll
        for (int r = 0; r < 16; ++r) sts64(sU12 + r * SB + cc, y[r]);
        if (cc < nT)
#pragma unroll
          for (int r = 0; r < 16; ++r)
            if (r < kb) M[(long long)sPiv[k0 + r] * LDM + c0 + cc] = y[r];
      }
      if (tid == 0) s_next = 0;
      __syncthreads();
      P3_ADD(2, t_u12, tid == 0);
      P3_T(t_main);
      // The next panel's columns are updated by the panel warps themselves inside factor(k+1)
      // (in registers, for their own rows), so the update warps start right after them and
      // nobody waits for a look-ahead hand-off.
      const bool ahead = k + 1 < NPANEL;
      const int la = ahead ? min(16, NI - 16 * (k + 1)) : 0;  // exactly the next panel's columns
      if (!pwarp) {
        P3_ADD(3, t_main, tid == 128);
        update(k, la, nT, -1);
        P3_ADD(4, t_main, tid == 128);
      } else {
        if (ahead) {
          P3_ADD(5, t_main, tid == 0);
          factor(k + 1);
          P3_ADD(6, t_main, tid == 0);
        }
        update(k, la, nT, -1);  // join the remaining trailing update
      }
      __syncthreads();
      P3_ADD(7, t_main, tid == 0);
    }
    P3_T(t_bs);

    // back substitution + T1 in a separate (non-inlined) function: its registers do not perturb
    // the allocation of the factorisation loop above
    double pm = leaf3_backsub(M, sPiv, a.Psi + (long long)grp * NI * NB, cL43i, cL43e);
    P3_ADD(8, t_bs, tid == 0);
    P3_T(t_ep);
    // probe condition estimate (leafops.py:293-294)
    pm = warp_max(pm);
    if (lane == 0) s_red[warp] = pm;
    __syncthreads();
    if (tid == 0) {
      double mx = 0.0;
      for (int w = 0; w < 8; ++w) mx = fmax(mx, s_red[w]);
      const double cnd = anorm * mx / a.probe_max;
      a.cond[grp] = (s_sing || !isfinite(cnd)) ? INFINITY : cnd;
    }
    double* sT1 = sU12;  // 64 x ST1, written by leaf3_backsub
    __syncthreads();
    {
      const int rr0 = warp * 8;
      double acc[8][2];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;
      for (int ks = 0; ks < NB; ks += 4) {
        const double af = sT1[(rr0 + g) * ST1 + ks + tq];
        const double* Brow = cL1 + (ks + tq) * NG;
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_8x8x4(acc[j][0], acc[j][1], af, __ldg(Brow + 8 * j + g));
      }
      double* T = a.T + (long long)grp * NG * NG;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        __stcs(reinterpret_cast<double2*>(T + (rr0 + g) * NG + 8 * j + 2 * tq), make_double2(acc[j][0], acc[j][1]));
    }
    P3_ADD(9, t_ep, tid == 0);
  }
}

#ifdef HPS_LEAF_PROFILE
extern "C" int hps_debug_leaf3_profile(long long* out, int reset) {
  if (reset) {
    static long long z[1024][16] = {};
    cudaMemcpyToSymbol(g_leaf3_prof, z, sizeof(z));
    return 0;
  }
  cudaMemcpyFromSymbol(out, g_leaf3_prof, sizeof(long long) * 1024 * 16);
  return 0;
}
#endif

size_t leaf16v3_scratch_doubles() { return (size_t)l3::MROWS * l3::LDM + (size_t)l3::NPANEL * 256; }

int leaf16v3_grid(const Ctx& cx, int ngroups) {
  // HPS_OPT_LEAF_FREE_SMS: size the grid for that many fewer SMs (experiment: SMs left to a
  // concurrent stream's merges in solver.Pipeline)
  const int per_sm = (int)std::max(1LL, cx.opt[HPS_OPT_LEAF_CTAS_PER_SM]);
  const int sms = std::max(1, cx.sms - (int)cx.opt[HPS_OPT_LEAF_FREE_SMS]);
  // the smallest grid with the same leaves per CTA as a full one: the grid-stride loop's critical
  // path is unchanged, and the spare CTA slots let other streams' small kernels (the next
  // problem's grouping in solver.Pipeline) run beside the leaf stage (cfg2: 293 of 296)
  const int full = std::max(1, std::min(ngroups, per_sm * sms));
  const int per_cta = (ngroups + full - 1) / full;
  return std::max(1, (ngroups + per_cta - 1) / per_cta);
}

int launch_leaf16v3(LeafArgs& a, Ctx& cx, cudaStream_t st) {
  const int as = ensure_smem_attr((const void*)k_leaf16v3, cx.device, (int)l3::SMEM);
  if (as != HPS_OK) return as;
  a.scratch_stride = (long long)leaf16v3_scratch_doubles();
  k_leaf16v3<<<leaf16v3_grid(cx, a.ngroups), l3::THREADS, l3::SMEM, st>>>(a);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

}  // namespace hps
