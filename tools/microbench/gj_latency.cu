// Latency probe: per-pivot-step cost of a single-warp 32x32 Gauss-Jordan (no barriers) vs the
// building blocks (REDUX argmax, DP reciprocal, shuffles), timed with clock64 inside the kernel.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gj32_warp(double* X, long long* cyc, int reps) {
  const int lane = threadIdx.x;
  double a[32];
  for (int j = 0; j < 32; ++j) a[j] = X[lane * 32 + j];
  bool used = false;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      unsigned long long key = used ? 0ull : (unsigned long long)__double_as_longlong(fabs(a[k]));
      unsigned hi = key >> 32, lo = (unsigned)key;
      unsigned mhi = __reduce_max_sync(~0u, hi);
      unsigned mlo = __reduce_max_sync(~0u, hi == mhi ? lo : 0u);
      int p = (int)__reduce_min_sync(~0u, (hi == mhi && lo == mlo) ? (unsigned)lane : ~0u);
      double piv = __shfl_sync(~0u, a[k], p);
      double inv = 1.0 / piv;
      if (lane == p) used = true;
      double f = a[k];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        double rp = __shfl_sync(~0u, a[j], p) * inv;
        double v = fma(-f, rp, a[j]);
        a[j] = (lane == p) ? rp : v;
      }
      a[k] = (lane == p) ? inv : -f * inv;
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int j = 0; j < 32; ++j) s += a[j];
  X[lane] = s;
  if (lane == 0) cyc[0] = t1 - t0;
}

__global__ void redux_chain(long long* cyc, unsigned* out, int n) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __reduce_max_sync(~0u, v) + threadIdx.x;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void rcp_chain(long long* cyc, double* out, int n) {
  double v = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = 1.0 / v + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void dfma_chain(long long* cyc, double* out, int n) {
  double v = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = fma(v, 0.999999, 1e-7);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void shfl_chain(long long* cyc, double* out, int n) {
  double v = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_sync(~0u, v, (threadIdx.x + 1) & 31) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void bar_chain(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* X; long long* cyc; unsigned* u; double* d;
  cudaMalloc(&X, 32 * 32 * 8); cudaMalloc(&cyc, 8); cudaMalloc(&u, 4096); cudaMalloc(&d, 8192);
  double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = (i % 33 == 0 ? 40.0 : 0.0) + (double)((i * 7919) % 13) / 13.0;
  cudaMemcpy(X, h, 8192, cudaMemcpyHostToDevice);
  long long c;
  int reps = 100;
  gj32_warp<<<1, 32>>>(X, cyc, reps); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("gj32 single warp: %.1f cycles per pivot step\n", (double)c / (reps * 32));
  int n = 10000;
  redux_chain<<<1, 32>>>(cyc, u, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("REDUX.MAX dependent: %.1f cyc\n", (double)c / n);
  rcp_chain<<<1, 32>>>(cyc, d, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("1.0/x + 1 dependent: %.1f cyc\n", (double)c / n);
  dfma_chain<<<1, 32>>>(cyc, d, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("DFMA dependent: %.1f cyc\n", (double)c / n);
  shfl_chain<<<1, 32>>>(cyc, d, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("SHFL f64 + DADD dependent: %.1f cyc\n", (double)c / n);
  bar_chain<<<1, 256>>>(cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("BAR.SYNC 8 warps: %.1f cyc\n", (double)c / n);
  bar_chain<<<1, 128>>>(cyc, n); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); printf("BAR.SYNC 4 warps: %.1f cyc\n", (double)c / n);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
