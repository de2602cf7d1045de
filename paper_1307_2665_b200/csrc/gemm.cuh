// Batched fp64 GEMM on the DMMA pipe (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), sm_100a.
//
//   C[b] = alpha * A[b] * B[b] + beta * C[b]     (all row-major)
//
// B rows may be gathered through an index table (the solve's u[I_e] gather). This one kernel
// carries every bulk flop of the merge levels (S = X^-1 R, T += C S, the recursive interface
// inverse) and of the batched solve. tcgen05 has no f64 kind on sm_100a, so DMMA is the FP64
// tensor path (measured 37.1 TF/s peak on B200 vs 34.2 for DFMA; profiles/fp64_peak_r01.json).
//
// Tiling: CTA tile BM x BN x BK, STAGES-deep cp.async pipeline. Smem strides are padded so every
// fragment load is a 2-wavefront LDS.64 (A: stride = BK+4 doubles, B: stride = BN+8 doubles).
#pragma once
#include "common.cuh"

namespace hps {

// Children of merge b in a level-batched tree (merge.cu): T matrices at T + idx[2b]*stride and
// T + idx[2b+1]*stride (idx null: children 2b, 2b+1), each m x m.
struct ChildRef {
  const double* T;
  long long stride;
  const int* idx;
  int m;
  __device__ __forceinline__ const double* a(int b) const {
    return T + (long long)(idx ? idx[2 * b] : 2 * b) * stride;
  }
  __device__ __forceinline__ const double* bb(int b) const {
    return T + (long long)(idx ? idx[2 * b + 1] : 2 * b + 1) * stride;
  }
};

struct GemmParams {
  int M, N, K, batch;
  const double* A; long long lda, strideA;
  const double* B; long long ldb, strideB;
  const int* Bidx; long long strideBidx;  // optional: row k of B[b] is B[b] + Bidx[b*strideBidx + k]*ldb
  double* C; long long ldc, strideC;
  double alpha, beta;
  int* nonfinite;  // optional: set to max batch index with a non-finite output
  int batch_offset = 0;  // added to the reported batch index (batch-chunked launches)
  int split = 1;         // split-K factor (blockIdx.z = batch * split + s)
  double* partial = nullptr;  // split > 1: raw partial sums [batch][split][M][N]
  // Optional fused block-diagonal addend of the merge update T = blkdiag(Ta11, Tb22) + C S
  // (replaces beta * C): for merge b (= batch index + batch_offset), n1 = M / 2,
  // blk[r][c] = Ta[j1a[r]][j1a[c]] (r, c < n1), Tb[j2b[r-n1]][j2b[c-n1]] (r, c >= n1), else 0.
  ChildRef blk{nullptr, 0, nullptr, 0};
  const int* blk_j1a = nullptr;
  const int* blk_j2b = nullptr;
  int group_m = 0;  // 64 x 64 kernel: grouped tile rasterisation (0 = row-major)
  bool emu_ok = false;  // may run as the int8-sliced FP64 emulation (emu.cu) when the context enables it
};

__device__ __forceinline__ double blk_value(const GemmParams& p, int b, int r, int c) {
  const int n1 = p.M >> 1;
  const bool top = r < n1;
  if ((c < n1) != top) return 0.0;
  const int gb = b + p.batch_offset;
  const double* src = top ? p.blk.a(gb) : p.blk.bb(gb);
  const int rm = top ? p.blk_j1a[r] : p.blk_j2b[r - n1];
  const int cm = top ? p.blk_j1a[c] : p.blk_j2b[c - n1];
  return src[(long long)rm * p.blk.m + cm];
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int kThreads = WM * WN * 32;
  static constexpr int SA = BK + 4;
  static constexpr int SB = BN + 8;
  static constexpr int kStageA = BM * SA;
  static constexpr int kStageB = BK * SB;
  static constexpr size_t kSmem = size_t(STAGES) * (kStageA + kStageB) * sizeof(double);
  static constexpr int TM = BM / WM / 8;
  static constexpr int TN = BN / WN / 8;
  static_assert(BM % (WM * 8) == 0 && BN % (WN * 8) == 0 && BK % 4 == 0, "tile");
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool VEC = true>
__global__ void __launch_bounds__(WM* WN * 32)
dgemm_dmma_kernel(GemmParams p) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * Cfg::kStageA;

  const int b = blockIdx.z / p.split;
  const int ks_idx = blockIdx.z - b * p.split;
  const int m0 = blockIdx.y * BM;
  const int n0 = blockIdx.x * BN;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int g = lane >> 2, t = lane & 3;

  const double* A = p.A + (long long)b * p.strideA;
  const double* B = p.B + (long long)b * p.strideB;
  const int* Bidx = p.Bidx ? p.Bidx + (long long)b * p.strideBidx : nullptr;
  double* C = p.C + (long long)b * p.strideC;

  const int kt_all = VEC ? p.K / BK : (p.K + BK - 1) / BK;  // VEC: K % BK == 0 (launcher)
  const int kt_per = (kt_all + p.split - 1) / p.split;
  const int kt0 = ks_idx * kt_per;
  const int ktiles = max(0, min(kt_all, kt0 + kt_per) - kt0);

  auto load_stage = [&](int stage, int kt) {
    const int k0 = (kt0 + kt) * BK;
    if constexpr (!VEC) {  // any shape / alignment: predicated scalar loads, zero padding
      double* a_dst = sA + stage * Cfg::kStageA;
      for (int e = tid; e < BM * BK; e += Cfg::kThreads) {
        const int r = e / BK, c = e - r * BK;
        const int gr = m0 + r, gk = k0 + c;
        a_dst[r * Cfg::SA + c] = (gr < p.M && gk < p.K) ? A[(long long)gr * p.lda + gk] : 0.0;
      }
      double* b_dst = sB + stage * Cfg::kStageB;
      for (int e = tid; e < BK * BN; e += Cfg::kThreads) {
        const int r = e / BN, c = e - r * BN;
        const int gk = k0 + r, gc = n0 + c;
        double v = 0.0;
        if (gk < p.K && gc < p.N) {
          const long long row = Bidx ? (long long)Bidx[gk] : (long long)gk;
          v = B[row * p.ldb + gc];
        }
        b_dst[r * Cfg::SB + c] = v;
      }
      return;
    }
    double* a_dst = sA + stage * Cfg::kStageA;
    constexpr int A_CHUNKS = BM * BK / 2;
#pragma unroll
    for (int c = tid; c < A_CHUNKS; c += Cfg::kThreads) {
      int r = c / (BK / 2), cc = c % (BK / 2);
      int gr = m0 + r;
      bool ok = gr < p.M;
      const double* src = A + (long long)(ok ? gr : 0) * p.lda + k0 + 2 * cc;
      cp_async16(a_dst + r * Cfg::SA + 2 * cc, src, ok);
    }
    double* b_dst = sB + stage * Cfg::kStageB;
    constexpr int B_CHUNKS = BK * BN / 2;
#pragma unroll
    for (int c = tid; c < B_CHUNKS; c += Cfg::kThreads) {
      int r = c / (BN / 2), cc = c % (BN / 2);
      int gc = n0 + 2 * cc;
      bool ok = gc < p.N;
      long long row = Bidx ? (long long)Bidx[k0 + r] : (long long)(k0 + r);
      const double* src = B + row * p.ldb + (ok ? gc : 0);
      cp_async16(b_dst + r * Cfg::SB + 2 * cc, src, ok);
    }
  };

  double acc[Cfg::TM][Cfg::TN][2];
#pragma unroll
  for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  const int a_row0 = wm * (BM / WM) + g;
  const int b_col0 = wn * (BN / WN) + g;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {  // prefetch tile kt + STAGES - 1 into the slot freed last iteration
      int nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* a_s = sA + (kt % STAGES) * Cfg::kStageA;
    const double* b_s = sB + (kt % STAGES) * Cfg::kStageB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::TM], bf[Cfg::TN];
#pragma unroll
      for (int i = 0; i < Cfg::TM; ++i) af[i] = a_s[(a_row0 + i * 8) * Cfg::SA + kk + t];
#pragma unroll
      for (int j = 0; j < Cfg::TN; ++j) bf[j] = b_s[(kk + t) * Cfg::SB + b_col0 + j * 8];
#pragma unroll
      for (int i = 0; i < Cfg::TM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::TN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  if (p.split > 1) {  // raw partial sums; k_splitk_reduce applies alpha/beta in a fixed order
    double* P = p.partial + ((long long)b * p.split + ks_idx) * (long long)p.M * p.N;
#pragma unroll
    for (int i = 0; i < Cfg::TM; ++i) {
      int r = m0 + a_row0 + i * 8;
      if (r >= p.M) continue;
#pragma unroll
      for (int j = 0; j < Cfg::TN; ++j) {
        int c = n0 + wn * (BN / WN) + j * 8 + 2 * t;
        if constexpr (!VEC) {
          if (c < p.N) P[(long long)r * p.N + c] = acc[i][j][0];
          if (c + 1 < p.N) P[(long long)r * p.N + c + 1] = acc[i][j][1];
        } else if (c < p.N) {
          *reinterpret_cast<double2*>(P + (long long)r * p.N + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        }
      }
    }
    return;
  }
  bool bad = false;
#pragma unroll
  for (int i = 0; i < Cfg::TM; ++i) {
    int r = m0 + a_row0 + i * 8;
    if (r >= p.M) continue;
#pragma unroll
    for (int j = 0; j < Cfg::TN; ++j) {
      int c = n0 + wn * (BN / WN) + j * 8 + 2 * t;
      if (c >= p.N) continue;
      double* dst = C + (long long)r * p.ldc + c;
      if constexpr (!VEC) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (c + h < p.N) {
            double v = p.alpha * acc[i][j][h];
            if (p.beta != 0.0) v += p.beta * dst[h];
            if (p.blk_j1a) v += blk_value(p, b, r, c + h);
            bad |= !isfinite(v);
            dst[h] = v;
          }
        continue;
      }
      double2 v;
      v.x = p.alpha * acc[i][j][0];
      v.y = p.alpha * acc[i][j][1];
      if (p.beta != 0.0) {
        double2 o = *reinterpret_cast<const double2*>(dst);
        v.x += p.beta * o.x;
        v.y += p.beta * o.y;
      }
      if (p.blk_j1a) {
        v.x += blk_value(p, b, r, c);
        v.y += blk_value(p, b, r, c + 1);
      }
      bad |= !isfinite(v.x) || !isfinite(v.y);
      *reinterpret_cast<double2*>(dst) = v;
    }
  }
  if (p.nonfinite && bad) atomicMax(p.nonfinite, b + p.batch_offset);
}

// 64 x 64 CTA tile, 4 warps of 32 x 32, several CTAs per SM (the shape cuBLAS picks for DGEMM on
// sm_100). Fragments are loaded in pairs with LDS.128:
//  * k pairing: in every 8-deep k block, DMMA k-step s in {0,1} gives lane tq the k index
//    2*tq + s, so a lane's A fragments of both steps, A[m][2tq], A[m][2tq+1], are adjacent;
//  * n pairing: in every 16-column block, DMMA j in {0,1} takes column 2c + j for its fragment
//    column c, so B[k][2g], B[k][2g+1] feed both DMMAs, and each lane ends up owning 4
//    consecutive output columns per row.
// Smem strides: A row = BK + 8 doubles (== 8 mod 16), B row = 64 + 2 doubles (== 2 mod 8): every
// quarter-warp's 16-byte loads hit 8 distinct bank groups.
template <int BK, int STAGES>
struct Gemm64Cfg {
  static constexpr int BM = 64, BN = 64, kThreads = 128;
  static constexpr int SA = BK + 8;
  static constexpr int SB = BN + 2;
  static constexpr int kStageA = BM * SA;
  static constexpr int kStageB = BK * SB;
  static constexpr size_t kSmem = size_t(STAGES) * (kStageA + kStageB) * sizeof(double);
};

template <int BK, int STAGES, int MINB>
__global__ void __launch_bounds__(128, MINB) dgemm64_kernel(GemmParams p) {
  using Cfg = Gemm64Cfg<BK, STAGES>;
  constexpr int BM = 64, BN = 64;
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * Cfg::kStageA;
  const int b = blockIdx.z / p.split;
  const int ks_idx = blockIdx.z - b * p.split;
  // Grouped rasterisation (p.group_m > 0, large grids): consecutive CTAs walk down group_m tile rows
  // before moving right, so the ~444 CTAs of a wave share ~sqrt(444) row and column panels of A and
  // B in L2 instead of streaming all of B once per wave of tile rows.
  int tile_m = blockIdx.y, tile_n = blockIdx.x;
  if (p.group_m > 0 && (int)gridDim.y > p.group_m) {
    const int pid = blockIdx.y * gridDim.x + blockIdx.x, per_group = p.group_m * gridDim.x;
    const int first_m = (pid / per_group) * p.group_m;
    const int gsize = min((int)gridDim.y - first_m, p.group_m);
    tile_m = first_m + (pid % per_group) % gsize;
    tile_n = (pid % per_group) / gsize;
  }
  const int m0 = tile_m * BM, n0 = tile_n * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  const double* A = p.A + (long long)b * p.strideA;
  const double* B = p.B + (long long)b * p.strideB;
  const int* Bidx = p.Bidx ? p.Bidx + (long long)b * p.strideBidx : nullptr;
  double* C = p.C + (long long)b * p.strideC;
  const int kt_all = p.K / BK;
  const int kt_per = (kt_all + p.split - 1) / p.split;
  const int kt0 = ks_idx * kt_per;
  const int ktiles = max(0, min(kt_all, kt0 + kt_per) - kt0);

  // Each thread copies the same 4 A chunks and 4 B chunks (16 B) of every stage: source pointers
  // and smem offsets are computed once and advanced by BK per k tile.
  constexpr int NCA = BM * BK / 2 / 128, NCB = BK * BN / 2 / 128;
  static_assert(NCA * 128 == BM * BK / 2 && NCB * 128 == BK * BN / 2, "chunks");
  const double* a_src[NCA];
  int a_off[NCA];
  bool a_ok[NCA];
#pragma unroll
  for (int i = 0; i < NCA; ++i) {
    const int c = tid + 128 * i, r = c / (BK / 2), cc = c % (BK / 2);
    a_ok[i] = m0 + r < p.M;
    a_src[i] = A + (long long)(a_ok[i] ? m0 + r : 0) * p.lda + (long long)kt0 * BK + 2 * cc;
    a_off[i] = r * Cfg::SA + 2 * cc;
  }
  const double* b_src[NCB];
  int b_off[NCB], b_row[NCB];
  bool b_ok[NCB];
#pragma unroll
  for (int i = 0; i < NCB; ++i) {
    const int c = tid + 128 * i, r = c / (BN / 2), cc = c % (BN / 2);
    b_ok[i] = n0 + 2 * cc < p.N;
    b_row[i] = r;
    b_src[i] = B + (b_ok[i] ? n0 + 2 * cc : 0) + (Bidx ? 0 : ((long long)kt0 * BK + r) * p.ldb);
    b_off[i] = r * Cfg::SB + 2 * cc;
  }
  const long long b_step = (long long)BK * p.ldb;
  auto load_stage = [&](int stage, int kt) {
    double* a_dst = sA + stage * Cfg::kStageA;
#pragma unroll
    for (int i = 0; i < NCA; ++i) cp_async16(a_dst + a_off[i], a_src[i] + kt * BK, a_ok[i]);
    double* b_dst = sB + stage * Cfg::kStageB;
    if (Bidx) {
      const int k0 = (kt0 + kt) * BK;
#pragma unroll
      for (int i = 0; i < NCB; ++i)
        cp_async16(b_dst + b_off[i], b_src[i] + (long long)Bidx[k0 + b_row[i]] * p.ldb, b_ok[i]);
    } else {
#pragma unroll
      for (int i = 0; i < NCB; ++i) cp_async16(b_dst + b_off[i], b_src[i] + kt * b_step, b_ok[i]);
    }
  };

  double acc[4][2][2][2];  // [m block][n pair][j][h]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[i][q][j][0] = acc[i][q][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }
  const int arow = wm * 32 + g;       // + 8 i
  const int bcol = wn * 32 + 2 * g;   // + 16 q
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* a_s = sA + (kt % STAGES) * Cfg::kStageA;
    const double* b_s = sB + (kt % STAGES) * Cfg::kStageB;
#pragma unroll
    for (int kb = 0; kb < BK; kb += 8) {
      double2 af[4], bf[2][2];  // af[i] = steps 0/1; bf[s][q] = (j0, j1)
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = *reinterpret_cast<const double2*>(a_s + (arow + 8 * i) * Cfg::SA + kb + 2 * t);
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
        for (int q = 0; q < 2; ++q)
          bf[s2][q] = *reinterpret_cast<const double2*>(b_s + (kb + 2 * t + s2) * Cfg::SB + bcol + 16 * q);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          dmma_8x8x4(acc[i][q][0][0], acc[i][q][0][1], af[i].x, bf[0][q].x);
          dmma_8x8x4(acc[i][q][1][0], acc[i][q][1][1], af[i].x, bf[0][q].y);
        }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          dmma_8x8x4(acc[i][q][0][0], acc[i][q][0][1], af[i].y, bf[1][q].x);
          dmma_8x8x4(acc[i][q][1][0], acc[i][q][1][1], af[i].y, bf[1][q].y);
        }
    }
  }
  cp_async_wait<0>();

  // lane (g, t) owns rows arow + 8i, columns bcol' + 16q + 4t + {0,1,2,3} (= 2h + j)
  const int ccol0 = n0 + wn * 32 + 4 * t;
  if (p.split > 1) {
    double* P = p.partial + ((long long)b * p.split + ks_idx) * (long long)p.M * p.N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = m0 + arow + 8 * i;
      if (r >= p.M) continue;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = ccol0 + 16 * q;
        double* dst = P + (long long)r * p.N + c;
        if (c < p.N) *reinterpret_cast<double2*>(dst) = make_double2(acc[i][q][0][0], acc[i][q][1][0]);
        if (c + 2 < p.N) *reinterpret_cast<double2*>(dst + 2) = make_double2(acc[i][q][0][1], acc[i][q][1][1]);
      }
    }
    return;
  }
  if (p.blk_j1a) {
    // merge update T = blkdiag + C S: gather all 32 block-diagonal addends of this lane first
    // (maps, then the child entries, all independent loads in flight together), then store
    const int n1 = p.M >> 1, gb = b + p.batch_offset;
    const double* Ta = p.blk.a(gb);
    const double* Tb = p.blk.bb(gb);
    const double* rs[4];
    bool rtop[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = min(m0 + arow + 8 * i, p.M - 1);
      rtop[i] = r < n1;
      rs[i] = rtop[i] ? Ta + (long long)p.blk_j1a[r] * p.blk.m : Tb + (long long)p.blk_j2b[r - n1] * p.blk.m;
    }
    int cm[2][4];
    bool ctop[2][4];
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = min(ccol0 + 16 * q + k, p.N - 1);
        ctop[q][k] = c < n1;
        cm[q][k] = ctop[q][k] ? p.blk_j1a[c] : p.blk_j2b[c - n1];
      }
    // column 16q + 4t + (2h + j) holds acc[i][q][j][h]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double v = rtop[i] == ctop[q][k] ? __ldg(rs[i] + cm[q][k]) : 0.0;
          acc[i][q][k & 1][k >> 1] = fma(p.alpha, acc[i][q][k & 1][k >> 1], v);
        }
  }
  const double alpha = p.blk_j1a ? 1.0 : p.alpha;  // (applied above when the addend was fused)
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + arow + 8 * i;
    if (r >= p.M) continue;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c = ccol0 + 16 * q;
      double* dst = C + (long long)r * p.ldc + c;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (c + 2 * h >= p.N) continue;
        double2 v = make_double2(alpha * acc[i][q][0][h], alpha * acc[i][q][1][h]);
        if (p.beta != 0.0) {
          const double2 o = *reinterpret_cast<const double2*>(dst + 2 * h);
          v.x += p.beta * o.x;
          v.y += p.beta * o.y;
        }
        bad |= !isfinite(v.x) || !isfinite(v.y);
        *reinterpret_cast<double2*>(dst + 2 * h) = v;
      }
    }
  }
  if (p.nonfinite && bad) atomicMax(p.nonfinite, b + p.batch_offset);
}

// C[b] = alpha * sum_s P[b][s] + beta * C[b], deterministic summation order.
__global__ void k_splitk_reduce(GemmParams p);

// Launch with a tile shape picked from the problem size (split-K scratch and options from the
// context). Returns HPS_OK or an error code.
struct Ctx;
int dgemm_launch(const GemmParams& p, Ctx& cx, cudaStream_t stream);

}  // namespace hps
