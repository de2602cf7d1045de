// Ablation of the per-pivot-step cost of the register Gauss-Jordan (RPL=1, CPW=8, W=4, n=32).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sts64(double* p, double v) { asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(smem_u32(p)), "d"(v) : "memory"); }

template <int MODE>  // bit0: skip barrier, bit1: p = k (no argmax), bit2: inv = piv (no divide)
__global__ void gj(double* X, int n, long long* cyc) {
  constexpr int RPL = 1, CPW = 8;
  __shared__ double colbuf[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a[RPL][CPW];
  bool used[RPL];
  for (int j = 0; j < CPW; ++j) a[0][j] = X[lane * 32 + warp * CPW + j];
  used[0] = lane >= n;
  if (warp == 0) colbuf[0][lane] = a[0][0];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 50; ++rep)
  for (int k = 0; k < n; ++k) {
    const double* ck = colbuf[k & 1];
    double cv[RPL];
    cv[0] = ck[lane];
    int p;
    if (MODE & 2) {
      p = k;
    } else {
      unsigned long long key = used[0] ? 0ull : (unsigned long long)__double_as_longlong(fabs(cv[0]));
      int bi = used[0] ? 0x7fffffff : lane;
      unsigned hi = key >> 32, lo = (unsigned)key;
      unsigned mhi = __reduce_max_sync(~0u, hi);
      unsigned mlo = __reduce_max_sync(~0u, hi == mhi ? lo : 0u);
      p = (int)__reduce_min_sync(~0u, (hi == mhi && lo == mlo) ? (unsigned)bi : ~0u);
    }
    const int pl = p & 31;
    const double piv = ck[p];
    const double inv = (MODE & 4) ? piv : 1.0 / piv;
    if (lane == pl) used[0] = true;
    double rp[CPW];
#pragma unroll
    for (int j = 0; j < CPW; ++j) rp[j] = __shfl_sync(~0u, a[0][j], pl) * inv;
    const int kw = k / CPW;
    if (warp == kw) {
      const int kj = k - kw * CPW;
#pragma unroll
      for (int j = 0; j < CPW; ++j) if (j == kj) { rp[j] = inv; a[0][j] = 0.0; }
    }
    const double f = cv[0];
    const bool prow = lane == pl;
#pragma unroll
    for (int j = 0; j < CPW; ++j) { double v = fma(-f, rp[j], a[0][j]); a[0][j] = prow ? rp[j] : v; }
    if (k + 1 < n && warp == (k + 1) / CPW) {
      const int j1 = (k + 1) - warp * CPW;
#pragma unroll
      for (int j = 0; j < CPW; ++j) if (j == j1) sts64(&colbuf[(k + 1) & 1][lane], a[0][j]);
    }
    if (!(MODE & 1)) __syncthreads(); else __syncwarp();
  }
  long long t1 = clock64();
  for (int j = 0; j < CPW; ++j) X[lane * 32 + warp * CPW + j] = a[0][j];
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* X; long long* cyc; cudaMalloc(&X, 32 * 32 * 8); cudaMalloc(&cyc, 8);
  double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = (i % 33 == 0 ? 40.0 : 0.0) + (double)((i * 7919) % 13) / 13.0;
  long long c;
#define RUN(M, name) cudaMemcpy(X, h, 8192, cudaMemcpyHostToDevice); gj<M><<<1, 128>>>(X, 32, cyc); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("%-28s %8.1f cyc/step\n", name, c / (50.0 * 32));
  RUN(0, "full");
  RUN(1, "no barrier");
  RUN(2, "no argmax");
  RUN(4, "no divide");
  RUN(7, "none of the three");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
