// Phase timing of the register Gauss-Jordan step (k_gj2 layout: RPL=4, CPW=16, W=8, n=128).
// Stamps per step for warp 0 (owner of columns 0..15) and warp 7 (never an owner in steps 0..14).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sts64(double* p, double v) { asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(smem_u32(p)), "d"(v) : "memory"); }
__device__ __forceinline__ double fast_rcp(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(r, fma(-x, r, 1.0), r); r = fma(r, fma(-x, r, 1.0), r); return r;
}
constexpr int RPL = 4, CPW = 16, W = 8, NMAX = 128;
__global__ void __launch_bounds__(256) gj(double* X, int n, long long* prof) {
  __shared__ double colbuf[2][NMAX];
  __shared__ double s_inv[2];
  __shared__ int s_p[2];
  __shared__ __align__(16) double rowbuf[W][CPW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cbase = warp * CPW;
  double a[RPL][CPW];
  bool used[RPL];
  for (int i = 0; i < RPL; ++i) { used[i] = false; for (int j = 0; j < CPW; ++j) a[i][j] = X[(lane + 32 * i) * n + cbase + j]; }
  long long acc[6] = {0, 0, 0, 0, 0, 0};
  auto publish = [&](int kn, int jl) {
    double v[RPL];
#pragma unroll
    for (int j = 0; j < CPW; ++j) if (j == jl) { for (int i = 0; i < RPL; ++i) v[i] = a[i][j]; }
    unsigned long long bestkey = 0ull; int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      sts64(&colbuf[kn & 1][lane + 32 * i], v[i]);
      const unsigned long long key = used[i] ? 0ull : (unsigned long long)__double_as_longlong(fabs(v[i]));
      const int idx = used[i] ? 0x7fffffff : lane + 32 * i;
      if (key > bestkey || (key == bestkey && idx < bi)) { bestkey = key; bi = idx; }
    }
    const unsigned hi = (unsigned)(bestkey >> 32), lo = (unsigned)bestkey;
    const unsigned mhi = __reduce_max_sync(~0u, hi);
    const unsigned mlo = __reduce_max_sync(~0u, hi == mhi ? lo : 0u);
    const int p = (int)__reduce_min_sync(~0u, (hi == mhi && lo == mlo) ? (unsigned)bi : ~0u);
    const int pl = p & 31, pi = p >> 5;
    double pv = 0.0;
#pragma unroll
    for (int i = 0; i < RPL; ++i) if (pi == i) pv = __shfl_sync(~0u, v[i], pl);
    if (lane == 0) { s_p[kn & 1] = p; s_inv[kn & 1] = fast_rcp(pv); }
  };
  __syncthreads();
  if (warp == 0) publish(0, 0);
  __syncthreads();
  for (int k = 0; k < 15; ++k) {
    long long t0 = clock64();
    const int bb = k & 1;
    const int p = s_p[bb];
    const double inv = s_inv[bb];
    const int pl = p & 31, pi = p >> 5;
    double f[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) f[i] = colbuf[bb][lane + 32 * i] * inv;
    double rp[CPW];
#ifdef SHFL
#pragma unroll
    for (int i = 0; i < RPL; ++i)
      if (pi == i) {
        if (lane == pl) used[i] = true;
#pragma unroll
        for (int j = 0; j < CPW; ++j) rp[j] = __shfl_sync(~0u, a[i][j], pl);
      }
#else
#pragma unroll
    for (int i = 0; i < RPL; ++i)
      if (pi == i && lane == pl) {
        used[i] = true;
#pragma unroll
        for (int j = 0; j < CPW; j += 2) *reinterpret_cast<double2*>(&rowbuf[warp][j]) = make_double2(a[i][j], a[i][j + 1]);
      }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CPW; j += 2) { const double2 v = *reinterpret_cast<const double2*>(&rowbuf[warp][j]); rp[j] = v.x; rp[j + 1] = v.y; }
#endif
    long long t1 = clock64();
    const int kw = k / CPW;
    if (warp == kw) {
      const int kj = k - kw * CPW;
#pragma unroll
      for (int j = 0; j < CPW; ++j) if (j == kj) { rp[j] = 1.0; for (int i = 0; i < RPL; ++i) a[i][j] = 0.0; }
    }
    long long t2 = t1, t3 = t1;
    const int k1 = k + 1, ow = k1 / CPW;
    if (k1 < n && warp == ow) {
      const int j1 = k1 - ow * CPW;
#pragma unroll
      for (int j = 0; j < CPW; ++j)
        if (j == j1) {
#pragma unroll
          for (int i = 0; i < RPL; ++i) { a[i][j] = fma(-f[i], rp[j], a[i][j]); if (pi == i && lane == pl) a[i][j] = rp[j] * inv; }
        }
      t2 = clock64();
#ifndef NO_PUBLISH
      publish(k1, j1);
#else
      if (lane == 0) { s_p[k1 & 1] = k1; s_inv[k1 & 1] = 0.5; }
#endif
      t3 = clock64();
#pragma unroll
      for (int j = 0; j < CPW; ++j)
        if (j != j1) {
#pragma unroll
          for (int i = 0; i < RPL; ++i) a[i][j] = fma(-f[i], rp[j], a[i][j]);
        }
    } else {
#ifndef NO_UPDATE
#pragma unroll
      for (int j = 0; j < CPW; ++j)
#pragma unroll
        for (int i = 0; i < RPL; ++i) a[i][j] = fma(-f[i], rp[j], a[i][j]);
#endif
    }
#ifndef NO_FIX
#pragma unroll
    for (int i = 0; i < RPL; ++i)
      if (pi == i && lane == pl) {
#pragma unroll
        for (int j = 0; j < CPW; ++j) a[i][j] = rp[j] * inv;
      }
#endif
    long long t4 = clock64();
#ifndef NO_BAR
    __syncthreads();
#else
    __syncwarp();
#endif
    long long t5 = clock64();
    acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3; acc[4] += t5 - t4; acc[5] += t5 - t0;
  }
  if (lane == 0 && (warp == 0 || warp == 7)) for (int q = 0; q < 6; ++q) prof[(warp == 7) * 6 + q] = acc[q];
  for (int i = 0; i < RPL; ++i) for (int j = 0; j < CPW; ++j) X[(lane + 32 * i) * n + cbase + j] = a[i][j];
}
int main() {
  const int n = 128;
  double* X; long long* prof; cudaMalloc(&X, n * n * 8); cudaMalloc(&prof, 12 * 8);
  static double h[n * n];
  for (int i = 0; i < n * n; ++i) h[i] = (i % (n + 1) == 0 ? 50.0 : 0.0) + (double)((i * 7919) % 13) / 13.0;
  cudaMemcpy(X, h, n * n * 8, cudaMemcpyHostToDevice);
  gj<<<1, 256>>>(X, n, prof);
  cudaMemcpy(X, h, n * n * 8, cudaMemcpyHostToDevice);
  gj<<<1, 256>>>(X, n, prof);
  long long hp[12]; cudaMemcpy(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost);
  const char* nm[6] = {"load+shfl", "col j1 upd", "publish", "rest upd+fix", "barrier", "total"};
  for (int w = 0; w < 2; ++w) { printf("%s:", w ? "warp7" : "warp0(owner)"); for (int q = 0; q < 6; ++q) printf("  %s %.0f", nm[q], hp[w * 6 + q] / 15.0); printf("\n"); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
