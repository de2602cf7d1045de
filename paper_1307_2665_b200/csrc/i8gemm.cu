// Batched int8 GEMM with a modular epilogue on the 5th-generation tensor cores (tcgen05), for the
// modular FP64 emulation of the merge GEMMs (emu.cu; merge.py:108, 118):
//
//   R[z][i][j] = ((sum_k A[z][i][k] B[z][j0 + j][k]) mod m_(z / batch)) + 128,  in [0, 255] (uint8:
//                the symmetric residue in [-128, 127], biased),
//   A: [nz][M][K] int8, B: [nz][N][K] int8 (both K-contiguous), j < nc (an output column panel).
//
// Persistent, warp-specialised, one CTA per SM (320 threads):
//   warp 0    TMA producer: 128 x 128 B (A) and 256 x 128 B (B) boxes with the 128-byte swizzle
//             into a 4-stage shared-memory ring (full / empty mbarriers, expect-tx byte counts);
//   warp 1    allocates all 512 TMEM columns and issues tcgen05.mma.kind::i8 (M = 128, N = 256,
//             K = 32 per instruction; 4 per stage) into one of two 256-column int32 accumulators,
//             releases each stage with tcgen05.commit, and signals the epilogue;
//   (both role warps run their loops converged and let one elect.sync lane issue: the descriptors
//   stay in uniform registers, with no per-instruction waterfall loop; 7% faster than lane 0 alone)
//   warps 2-9 epilogue: tcgen05.ld 32x32b (two warps per 32-lane quadrant of TMEM, each half of the
//             columns; warp w may only touch quadrant w % 4), the exact
//             int32 sums reduced mod m (multiply-high quotient, no conversions), 32 bytes per row
//             chunk stored; the accumulator is released to the MMA warp while the next tile's
//             MMAs run in the other one.
// Tiles are ordered in groups of G tile rows so that the concurrent wave's A panels stay in L2.
#include <cuda.h>

#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "ctx.cuh"

namespace hps {
namespace i8 {

constexpr int BM = 128, BN = 256, BK = 128;  // BK: bytes = int8 elements of K per stage
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int EPI_WARPS = 8;  // two per TMEM lane quadrant, each half of the tile's columns
constexpr int THREADS = 64 + 32 * EPI_WARPS;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int MAX_MOD = 16;

struct ModTab {
  int m[MAX_MOD];
  int minv[MAX_MOD];
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// Bounded wait: a protocol error traps (a launch failure) instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (long long i = 0;; ++i) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    if (ok) return;
    if (i > (1LL << 26)) __trap();
  }
}
__device__ __forceinline__ void tma_load3(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
// one lane of a converged warp (elect.sync): the warp runs a role's loop together (warp-uniform
// values stay in uniform registers) and only the elected lane issues the TMA / MMA instruction
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor of a K-major tile with the 128-byte swizzle: rows of 128 bytes,
// 8-row (1024-byte) core-matrix groups; start address >> 4, LBO 16 B (unused when swizzled), SBO
// 1024 B, descriptor version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor: D s32, A / B signed int8, both K-major, N >> 3, M >> 4.
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Tile t -> (z, tile row, tile column): z outermost, then groups of G tile rows swept column by column,
// so a wave's A row panels (G x BM x K bytes, sized on the host to ~32 MB) stay in L2 while B streams.
__device__ __forceinline__ void tile_coords(long long t, int tm, int tn, int G, int& z, int& mi, int& ni) {
  const long long per = (long long)tm * tn;
  z = (int)(t / per);
  const int r = (int)(t - (long long)z * per);
  const int g = r / (G * tn), first = g * G, gs = min(G, tm - first);
  const int rr = r - g * G * tn;
  mi = first + rr % gs;
  ni = rr / gs;
}

// The biased symmetric residue ((v mod m) in [128 - m, 127]) + 128 of |v| < 2^30, in five integer
// operations. With off = m (floor(2^30 / m) + 1) + (m - 128), t = v + off is in [0, 2^31 + 2m) and
// congruent to v - 128, and for r' = t mod m the result is r' + (256 - m) whichever half v mod m lies
// in (v mod m = r' + 128 - m <= 127 if r' + 128 >= m, else r' + 128 > 127 and the representative is
// r' + 128 - m: both give r' + 256 - m), so no centring test. The multiply-high quotient (minv =
// floor(2^32 / m)) is the floor or one less, so t - q m is in [0, 2m): one unsigned-min correction.
__device__ __forceinline__ uint32_t mod_raw(uint32_t u, int m, int minv, int off) {  // r' = (v + off) mod m
  const unsigned t = u + (unsigned)off;
  const unsigned r = t - __umulhi(t, (unsigned)minv) * (unsigned)m;
  return min(r, r - (unsigned)m);
}
// four of them as a word of bytes; the + (256 - m) is added to all four at once (r' + 256 - m <= 255:
// no carry between the bytes)
__device__ __forceinline__ uint32_t mod_bytes4(const uint32_t* v, int m, int minv, int off) {
  const uint32_t lo = __byte_perm(mod_raw(v[0], m, minv, off), mod_raw(v[1], m, minv, off), 0x0040);
  const uint32_t hi = __byte_perm(mod_raw(v[2], m, minv, off), mod_raw(v[3], m, minv, off), 0x0040);
  return __byte_perm(lo, hi, 0x5410) + (uint32_t)(256 - m) * 0x01010101u;
}

__global__ void __launch_bounds__(THREADS, 1)
    k_i8gemm_mod(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M, int nc, int j0,
                 int K, int nz, int batch, int G, ModTab mt, unsigned char* __restrict__ R) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  // bars: full[STAGES], empty[STAGES], tfull[2], tempty[2]; then the TMEM base address
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);
  const uint32_t sbase = su32(smem);
  const uint32_t full0 = su32(bars), empty0 = full0 + 8 * STAGES, tfull0 = empty0 + 8 * STAGES, tempty0 = tfull0 + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = (M + BM - 1) / BM, tn = (nc + BN - 1) / BN;
  const long long tiles = (long long)nz * tm * tn;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    }
    __syncwarp();
    int s = 0;
    uint32_t ph = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
      int z, mi, ni;
      tile_coords(t, tm, tn, G, z, mi, ni);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        const uint32_t fb = full0 + 8 * s;
        const uint32_t dst = sbase + s * STAGE_BYTES;
        if (elect_one()) {
          mbar_expect_tx(fb, STAGE_BYTES);
          tma_load3(dst, &ta, fb, kb * BK, mi * BM, z);
          tma_load3(dst + A_BYTES, &tb, fb, kb * BK, j0 + ni * BN, z);
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(tempty0 + 8 * acc, aph ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * BN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(full0 + 8 * s, ph);
        tc_fence_after();
        const uint64_t a0 = sw128_desc(sbase + s * STAGE_BYTES);
        const uint64_t b0 = sw128_desc(sbase + s * STAGE_BYTES + A_BYTES);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 32; ++k)  // +32 bytes along K inside the swizzle atom: +2 in the >> 4 address
            umma_i8(d, a0 + 2 * k, b0 + 2 * k, (kb | k) != 0);
          umma_commit(empty0 + 8 * s);
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      if (elect_one()) umma_commit(tfull0 + 8 * acc);
      __syncwarp();
    }
  } else {
    const int q = warp & 3;                  // TMEM lane quadrant this warp may access
    const int half = (warp - 2) / 4;         // which half of the columns
    int it = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      int z, mi, ni;
      tile_coords(t, tm, tn, G, z, mi, ni);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(tfull0 + 8 * acc, aph);
      tc_fence_after();
      const int row = mi * BM + q * 32 + lane;
      const int l = z / batch;
      const int m = mt.m[l];
      const int minv = mt.minv[l], off = m * ((1 << 30) / m + 1) + (m - 128);
      unsigned char* dst = R + ((long long)z * M + row) * nc + ni * BN;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + c * 32, v);
        if (row < M && ni * BN + c * 32 < nc) {
          uint32_t w[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            w[i] = mod_bytes4(v + 4 * i, m, minv, off);
          uint4* o = reinterpret_cast<uint4*>(dst + c * 32);
          o[0] = make_uint4(w[0], w[1], w[2], w[3]);
          o[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8 * acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// ------------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 256 tile. Each
// CTA stages its 128 rows of A and its 128 rows (half) of B per k-block (32 KB; 6 stages), so the
// L2 -> SM traffic per MMA is 2/3 of the single-CTA tile's; the even CTA's one lane issues
// tcgen05.mma.cta_group::2 (M = 256, N = 256) over both CTAs' shared memory, and each CTA's TMEM
// holds its 128 accumulator rows. Both CTAs' TMA loads complete on the even CTA's full barrier;
// the MMA commits are multicast to both CTAs' empty / tmem-full barriers; both CTAs' epilogue warps
// release an accumulator on the even CTA's tmem-empty barrier (8 arrivals).
// ------------------------------------------------------------------------------------------------
namespace pair {
constexpr int BM = 256, BN = 256, BK = 128;  // pair tile; per CTA: 128 rows of A, 128 rows of B
constexpr int STAGES = 6;
constexpr int A_BYTES = 128 * BK, B_BYTES = 128 * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}  // namespace pair

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank0(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void tma_load3_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar_rank0, int c0, int c1,
                                               int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_rank0), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void umma_i8_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(pair::kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {  // arrive on `bar` in both CTAs
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_i8gemm_mod_pair(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M, int nc,
                      int j0, int K, int nz, int batch, int G, ModTab mt, unsigned char* __restrict__ R) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + pair::STAGES * pair::STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * pair::STAGES + 4);
  const uint32_t sbase = su32(smem);
  const uint32_t full0 = su32(bars), empty0 = full0 + 8 * pair::STAGES, tfull0 = empty0 + 8 * pair::STAGES, tempty0 = tfull0 + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int tm = (M + pair::BM - 1) / pair::BM, tn = (nc + pair::BN - 1) / pair::BN;
  const long long tiles = (long long)nz * tm * tn;
  const int nk = (K + pair::BK - 1) / pair::BK;
  const long long cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < pair::STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);   // used in the even CTA: its producer's expect-tx arrival
      mbar_init(empty0 + 8 * s, 1);  // one multicast commit per use
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 2 * EPI_WARPS);  // even CTA: the epilogue warps of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    }
    __syncwarp();
    int s = 0;
    uint32_t ph = 0;
    for (long long t = cid; t < tiles; t += ncl) {
      int z, mi, ni;
      tile_coords(t, tm, tn, G, z, mi, ni);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(empty0 + 8 * s, ph ^ 1);
        const uint32_t fb = full0 + 8 * s;
        const uint32_t fb0 = map_to_rank0(fb);
        const uint32_t dst = sbase + s * pair::STAGE_BYTES;
        if (elect_one()) {
          if (rank == 0) mbar_expect_tx(fb, 2 * pair::STAGE_BYTES);  // both CTAs' bytes land on the even CTA's barrier
          tma_load3_pair(dst, &ta, fb0, kb * pair::BK, mi * pair::BM + (int)rank * 128, z);
          tma_load3_pair(dst + pair::A_BYTES, &tb, fb0, kb * pair::BK, j0 + ni * pair::BN + (int)rank * 128, z);
        }
        __syncwarp();
        if (++s == pair::STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (long long t = cid; t < tiles; t += ncl, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(tempty0 + 8 * acc, aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * pair::BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint64_t a0 = sw128_desc(sbase + s * pair::STAGE_BYTES);
          const uint64_t b0 = sw128_desc(sbase + s * pair::STAGE_BYTES + pair::A_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < pair::BK / 32; ++k) umma_i8_pair(d, a0 + 2 * k, b0 + 2 * k, (kb | k) != 0);
            umma_commit_pair(empty0 + 8 * s);
          }
          __syncwarp();
          if (++s == pair::STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if (elect_one()) umma_commit_pair(tfull0 + 8 * acc);
        __syncwarp();
      }
    }
  } else {
    const int q = warp & 3;
    const int half = (warp - 2) / 4;
    const uint32_t tempty_rank0 = map_to_rank0(tempty0);
    int it = 0;
    for (long long t = cid; t < tiles; t += ncl, ++it) {
      int z, mi, ni;
      tile_coords(t, tm, tn, G, z, mi, ni);
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(tfull0 + 8 * acc, aph);
      tc_fence_after();
      const int row = mi * pair::BM + (int)rank * 128 + q * 32 + lane;
      const int l = z / batch;
      const int m = mt.m[l];
      const int minv = mt.minv[l], off = m * ((1 << 30) / m + 1) + (m - 128);
      unsigned char* dst = R + ((long long)z * M + row) * nc + ni * pair::BN;
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * pair::BN;
#pragma unroll 1
      for (int c = half * (pair::BN / 64); c < (half + 1) * (pair::BN / 64); ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + c * 32, v);
        if (row < M && ni * pair::BN + c * 32 < nc) {
          uint32_t w[8];
#pragma unroll
          for (int i = 0; i < 8; ++i)
            w[i] = mod_bytes4(v + 4 * i, m, minv, off);
          uint4* o = reinterpret_cast<uint4*>(dst + c * 32);
          o[0] = make_uint4(w[0], w[1], w[2], w[3]);
          o[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_rank0 + 8 * acc);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

// [nz][rows][K] int8, boxes of 128 K-bytes x box_rows rows x 1, 128-byte swizzle, zero fill out of bounds
static bool make_map(CUtensorMap* map, const void* base, int K, int rows, int nz, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * (cuuint64_t)rows};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace i8

// Eligibility of the tcgen05 path for a panel product (the caller falls back to cuBLASLt otherwise).
bool i8gemm_mod_ok(int M, int N, int nc, int K, int nmod) {
  return i8::encode_fn() != nullptr && nmod <= i8::MAX_MOD && K % 16 == 0 && N % 16 == 0 && nc % 32 == 0 && M > 0 &&
         nc > 0;
}

// R[z][i][j] (uint8, [nz][M][nc]) = (A[z] B[z][j0 + j]^T) mod moduli[z / batch] + 128; see the top of
// the file. pair: the CTA-pair kernel (256 x 256 tiles), else the single-CTA one (128 x 256).
int i8gemm_mod(const signed char* A, const signed char* B, unsigned char* R, int M, int N, int nc, int j0, int K, int nz,
               int batch, const int* moduli, int nmod, bool pair, Ctx& cx, cudaStream_t st) {
  CUtensorMap ta, tb;
  const int abox = pair ? 128 : i8::BM, bbox = pair ? 128 : i8::BN;
  if (!i8::make_map(&ta, A, K, M, nz, abox) || !i8::make_map(&tb, B, K, N, nz, bbox)) {
    set_error("i8gemm_mod: cuTensorMapEncodeTiled failed (M=%d N=%d K=%d nz=%d)", M, N, K, nz);
    return HPS_ERR_CUDA;
  }
  i8::ModTab mt;
  for (int l = 0; l < i8::MAX_MOD; ++l) {
    mt.m[l] = l < nmod ? moduli[l] : 1;
    mt.minv[l] = (int)((1ULL << 32) / (unsigned long long)mt.m[l]);
  }
  // tile-row group: ~32 MB of A row panels (or the option's override)
  const int bm = pair ? i8::pair::BM : i8::BM;
  const int tm = (M + bm - 1) / bm;
  int G = cx.opt[HPS_OPT_EMU_TILE_GROUP] > 0 ? (int)cx.opt[HPS_OPT_EMU_TILE_GROUP]
                                              : (int)std::max<long long>(1, (32LL << 20) / ((long long)bm * K));
  G = std::max(1, std::min(G, tm));
  if (pair) {
    int st_attr = ensure_smem_attr(reinterpret_cast<const void*>(&i8::k_i8gemm_mod_pair), cx.device, i8::pair::SMEM);
    if (st_attr != HPS_OK) return st_attr;
    const long long tiles = (long long)nz * ((M + i8::pair::BM - 1) / i8::pair::BM) * ((nc + i8::pair::BN - 1) / i8::pair::BN);
    const int grid = 2 * (int)std::min<long long>(tiles, cx.sms / 2);
    i8::k_i8gemm_mod_pair<<<grid, i8::THREADS, i8::pair::SMEM, st>>>(ta, tb, M, nc, j0, K, nz, batch, G, mt, R);
  } else {
    int st_attr = ensure_smem_attr(reinterpret_cast<const void*>(&i8::k_i8gemm_mod), cx.device, i8::SMEM);
    if (st_attr != HPS_OK) return st_attr;
    const long long tiles = (long long)nz * ((M + i8::BM - 1) / i8::BM) * ((nc + i8::BN - 1) / i8::BN);
    const int grid = (int)std::min<long long>(tiles, cx.sms);
    i8::k_i8gemm_mod<<<grid, i8::THREADS, i8::SMEM, st>>>(ta, tb, M, nc, j0, K, nz, batch, G, mt, R);
  }
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

}  // namespace hps

extern "C" int hps_i8gemm_mod(hps_ctx_t ctx, const signed char* A, const signed char* B, unsigned char* R, int M, int N,
                              int nc, int j0, int K, int nz, int batch, const int* moduli, int nmod, int engine,
                              void* stream) {
  HPS_CTX(cx, ctx);
  if (!hps::i8gemm_mod_ok(M, N, nc, K, nmod) || nz <= 0 || batch <= 0 || nz % batch || nz / batch > nmod ||
      j0 < 0 || j0 + nc > N || K >= (1 << 16) || (engine != 0 && engine != 2)) {
    hps::set_error("hps_i8gemm_mod: unsupported arguments (M=%d N=%d nc=%d j0=%d K=%d nz=%d batch=%d engine=%d)", M, N,
                   nc, j0, K, nz, batch, engine);
    return HPS_ERR_ARG;
  }
  for (int l = 0; l < nmod; ++l)
    if (moduli[l] < 2 || moduli[l] > 256) {
      hps::set_error("hps_i8gemm_mod: modulus %d out of range", moduli[l]);
      return HPS_ERR_ARG;
    }
  return hps::i8gemm_mod(A, B, R, M, N, nc, j0, K, nz, batch, moduli, nmod, engine == 2, *cx,
                         static_cast<cudaStream_t>(stream));
}
