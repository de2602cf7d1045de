// Ablation of the single-warp 8-column GJ panel step of k_gj_blk (rows: lane + 32 i, RPL = 4).
// MODE bits: 1 = fixed pivot (no REDUX), 2 = no reciprocal (inv = 1), 4 = pivot row by selects +
// shuffles instead of a uniform branch, 8 = skip the update FMAs.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double fast_rcp(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r); r = fma(r, fma(-x, r, 1.0), r); return r;
}
template <int MODE>
__global__ void panel(double* X, long long* cyc, int reps) {
  constexpr int RPL = 4;
  const int lane = threadIdx.x;
  double pr[RPL][8];
  bool used[RPL];
  for (int i = 0; i < RPL; ++i) { used[i] = false; for (int j = 0; j < 8; ++j) pr[i][j] = X[(lane + 32 * i) * 8 + j]; }
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      int p;
      if (MODE & 1) {
        p = (rep * 8 + t) & 127;
      } else if (MODE & 16) {  // 2 REDUX: exact hi word, then lo word with the row index in its low 7 bits
        unsigned bh = 0u, bl = 0u;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const unsigned long long kb = used[i] ? 0ull : (unsigned long long)__double_as_longlong(fabs(pr[i][t]));
          const unsigned h = (unsigned)(kb >> 32);
          const unsigned l = used[i] ? 0u : (((unsigned)kb) & ~127u) | (127u - (unsigned)(lane + 32 * i));
          if (h > bh || (h == bh && l > bl)) { bh = h; bl = l; }
        }
        const unsigned mh = __reduce_max_sync(~0u, bh);
        const unsigned ml = __reduce_max_sync(~0u, bh == mh ? bl : 0u);
        p = 127 - (int)(ml & 127u);
      } else if (MODE & 32) {  // butterfly shuffles, exact (key, smallest index)
        unsigned long long best = 0ull; int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const unsigned long long key = used[i] ? 0ull : (unsigned long long)__double_as_longlong(fabs(pr[i][t]));
          const int idx = used[i] ? 0x7fffffff : lane + 32 * i;
          if (key > best || (key == best && idx < bi)) { best = key; bi = idx; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const unsigned long long k2 = __shfl_xor_sync(~0u, best, o);
          const int i2 = __shfl_xor_sync(~0u, bi, o);
          if (k2 > best || (k2 == best && i2 < bi)) { best = k2; bi = i2; }
        }
        p = bi;
      } else {
        unsigned long long best = 0ull; int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const unsigned long long key = used[i] ? 0ull : (unsigned long long)__double_as_longlong(fabs(pr[i][t]));
          const int idx = used[i] ? 0x7fffffff : lane + 32 * i;
          if (key > best || (key == best && idx < bi)) { best = key; bi = idx; }
        }
        const unsigned hi = (unsigned)(best >> 32), lo = (unsigned)best;
        const unsigned mhi = __reduce_max_sync(~0u, hi);
        const unsigned mlo = __reduce_max_sync(~0u, hi == mhi ? lo : 0u);
        p = (int)__reduce_min_sync(~0u, (hi == mhi && lo == mlo) ? (unsigned)bi : ~0u);
      }
      const int pl = p & 31, pi = p >> 5;
      double rp[8];
      if (MODE & 4) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          double v = pr[0][j];
#pragma unroll
          for (int i = 1; i < RPL; ++i) v = (pi == i) ? pr[i][j] : v;
          rp[j] = __shfl_sync(~0u, v, pl);
        }
      } else {
#pragma unroll
        for (int i = 0; i < RPL; ++i)
          if (pi == i) {
#pragma unroll
            for (int j = 0; j < 8; ++j) rp[j] = __shfl_sync(~0u, pr[i][j], pl);
          }
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) used[i] = used[i] || (pi == i && lane == pl);
      if (rep % 16 == 15) for (int i = 0; i < RPL; ++i) used[i] = false;  // keep rows available
      const double piv = rp[t];
      const double inv = (MODE & 2) ? 1.0 : fast_rcp(piv);
#pragma unroll
      for (int j = 0; j < 8; ++j) rp[j] = j == t ? inv : rp[j] * inv;
      if (!(MODE & 8)) {
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const double f = pr[i][t];
          pr[i][t] = 0.0;
#pragma unroll
          for (int j = 0; j < 8; ++j) pr[i][j] = fma(-f, rp[j], pr[i][j]);
        }
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const bool mine = pi == i && lane == pl;
#pragma unroll
        for (int j = 0; j < 8; ++j) pr[i][j] = mine ? rp[j] : pr[i][j];
      }
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < RPL; ++i) for (int j = 0; j < 8; ++j) X[(lane + 32 * i) * 8 + j] = pr[i][j];
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  double* X; long long* cyc; cudaMalloc(&X, 128 * 8 * 8); cudaMalloc(&cyc, 8);
  static double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = 1.0 + (double)((i * 7919) % 13) / 13.0 + (i % 9 == 0 ? 30 : 0);
  long long c; const int reps = 64;
#define RUN(M, name) cudaMemcpy(X, h, sizeof(h), cudaMemcpyHostToDevice); panel<M><<<1, 32>>>(X, cyc, reps); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("%-40s %8.1f cyc/pivot\n", name, c / (8.0 * reps));
  RUN(0, "full");
  RUN(16, "argmax: 2 REDUX, index in low bits");
  RUN(32, "argmax: butterfly shuffles");
  RUN(18, "2 REDUX + no reciprocal");
  RUN(4, "pivot row via selects + shfl");
  RUN(1, "fixed pivot (no REDUX)");
  RUN(2, "no reciprocal");
  RUN(8, "no update FMAs");
  RUN(3, "no REDUX, no reciprocal");
  RUN(11, "no REDUX, no rcp, no update");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
