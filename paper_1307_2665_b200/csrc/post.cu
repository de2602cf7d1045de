// Post-processing on the device (reference solver.py:349-400):
//   hps_leaf_fields  : per listed leaf, the p x p Chebyshev field W = [L1 u[I_e] ; Psi_g L1 u[I_e]]
//                      scattered by J_e / J_i (solver.py:349-356, _leaf_field), for nrhs columns;
//   hps_eval_points  : out[t] = rx[t]^T W[slot[t]] ry[t] (post_process / boundary_flux_at: the
//                      derivative versions fold Dx or Dy into the weights on the host);
//   hps_gauge_sides  : Gauss values on the 4 sides re-tabulated from W (the L4 blocks: Qx W[:,0],
//                      Qy W[p-1,:], Qx W[:,p-1], Qy W[0,:], leafops.py:191-198), leaf I_e order;
//   hps_gauge_gather : u[node] = mean of its owners' side values (1 or 2 leaves); nodes flagged as
//                      outer boundary keep their input value. Deterministic (no atomics).
// The fields are invariant under the interface null modes, so the re-tabulated u is
// a gauge-fixed Gauss-node solution.
#include <algorithm>

#include "common.cuh"

namespace hps {

constexpr int POST_RHS = 64;  // right-hand sides per pass of k_leaf_fields

// One CTA per listed leaf. smem: ue[4q][nr], we[nb][nr].
__global__ void __launch_bounds__(256) k_leaf_fields(int nlist, int p, const double* __restrict__ U, int ldu,
                                                     int r0, int nr, const int* __restrict__ leaves,
                                                     const int* __restrict__ leaf_Ie, const int* __restrict__ gid,
                                                     const double* __restrict__ L1, const double* __restrict__ Psi,
                                                     const int* __restrict__ J_i, const int* __restrict__ J_e,
                                                     double* __restrict__ W, int ldw) {
  extern __shared__ double sm[];
  const int q4 = 4 * p, nb = 4 * (p - 1), ni = (p - 2) * (p - 2), p2 = p * p;
  double* ue = sm;            // q4 x nr
  double* we = sm + q4 * nr;  // nb x nr
  for (int s = blockIdx.x; s < nlist; s += gridDim.x) {
    const int leaf = leaves[s];
    const int* Ie = leaf_Ie + (long long)leaf * q4;
    const double* Ps = Psi + (long long)gid[leaf] * ni * nb;
    double* Ws = W + (long long)s * p2 * ldw + r0;
    __syncthreads();
    for (int e = threadIdx.x; e < q4 * nr; e += blockDim.x) {
      const int k = e / nr, r = e - k * nr;
      ue[e] = U[(long long)Ie[k] * ldu + r0 + r];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nb * nr; e += blockDim.x) {
      const int i = e / nr, r = e - i * nr;
      const double* L = L1 + (long long)i * q4;
      double acc = 0.0;
      for (int k = 0; k < q4; ++k) acc = fma(__ldg(L + k), ue[k * nr + r], acc);
      we[e] = acc;
      Ws[(long long)J_e[i] * ldw + r] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < ni * nr; e += blockDim.x) {
      const int i = e / nr, r = e - i * nr;
      const double* P = Ps + (long long)i * nb;
      double acc = 0.0;
      for (int k = 0; k < nb; ++k) acc = fma(__ldg(P + k), we[k * nr + r], acc);
      Ws[(long long)J_i[i] * ldw + r] = acc;
    }
  }
}

// One warp per target: out[t][r] = sum_ij rx[t][i] W[slot[t]][i p + j][r] ry[t][j].
__global__ void k_eval_points(int npts, int p, const double* __restrict__ W, int ldw, int nrhs,
                              const int* __restrict__ slot, const double* __restrict__ rx,
                              const double* __restrict__ ry, double* __restrict__ out) {
  const int t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= npts) return;
  const int p2 = p * p;
  const double* Wt = W + (long long)slot[t] * p2 * ldw;
  const double* x = rx + (long long)t * p;
  const double* y = ry + (long long)t * p;
  for (int r = 0; r < nrhs; ++r) {
    double acc = 0.0;
    for (int e = lane; e < p2; e += 32) {
      const int i = e / p, j = e - i * p;
      acc = fma(x[i] * y[j], Wt[(long long)e * ldw + r], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) out[(long long)t * nrhs + r] = acc;
  }
}

// One CTA per listed leaf: side[s][k][r], k over the leaf's 4p Gauss boundary nodes (S, E, N, W).
__global__ void k_gauge_sides(int nlist, int p, const double* __restrict__ W, int ldw, int nrhs,
                              const double* __restrict__ Qx, const double* __restrict__ Qy,
                              double* __restrict__ side) {
  const int q4 = 4 * p, p2 = p * p;
  for (int s = blockIdx.x; s < nlist; s += gridDim.x) {
    const double* Ws = W + (long long)s * p2 * ldw;
    double* out = side + (long long)s * q4 * nrhs;
    for (int e = threadIdx.x; e < q4 * nrhs; e += blockDim.x) {
      const int k = e / nrhs, r = e - k * nrhs;
      const int sd = k / p, m = k - sd * p;
      const double* Q = (sd & 1) ? Qy + (long long)m * p : Qx + (long long)m * p;
      double acc = 0.0;
      for (int l = 0; l < p; ++l) {
        int g;  // grid index i * p + j of the l-th Chebyshev node along the side
        switch (sd) {
          case 0: g = l * p; break;            // S: W[l][0]
          case 1: g = (p - 1) * p + l; break;  // E: W[p-1][l]
          case 2: g = l * p + p - 1; break;    // N: W[l][p-1]
          default: g = l; break;               // W: W[0][l]
        }
        acc = fma(__ldg(Q + l), Ws[(long long)g * ldw + r], acc);
      }
      out[e] = acc;
    }
  }
}

// u_out[node][r]: src[2 node], src[2 node + 1] index side rows (leaf slot * 4p + k); -1 = none.
// A node whose first source is -1 keeps u_in (outer boundary: the Dirichlet data).
__global__ void k_gauge_gather(int N, int nrhs, const double* __restrict__ side, const int* __restrict__ src,
                               const double* __restrict__ u_in, int ldu_in, double* __restrict__ u_out,
                               int ldu_out) {
  const long long total = (long long)N * nrhs;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int node = (int)(e / nrhs), r = (int)(e - (long long)node * nrhs);
    const int a = src[2 * node], b = src[2 * node + 1];
    double v;
    if (a < 0)
      v = u_in[(long long)node * ldu_in + r];
    else if (b < 0)
      v = side[(long long)a * nrhs + r];
    else
      v = 0.5 * (side[(long long)a * nrhs + r] + side[(long long)b * nrhs + r]);
    u_out[(long long)node * ldu_out + r] = v;
  }
}

}  // namespace hps

using namespace hps;

extern "C" int hps_leaf_fields(int nlist, int p, const double* U, int ldu, int nrhs, const int* leaves,
                               const int* leaf_Ie, const int* gid, const double* L1, const double* Psi,
                               const int* J_i, const int* J_e, double* W, void* stream) {
  if (nlist <= 0 || nrhs <= 0) return HPS_OK;
  if (p < 3 || p > 32 || ldu < nrhs) {
    set_error("hps_leaf_fields: bad arguments p=%d ldu=%d nrhs=%d", p, ldu, nrhs);
    return HPS_ERR_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = std::min(nlist, 148 * 8);
  for (int r0 = 0; r0 < nrhs; r0 += POST_RHS) {
    const int nr = std::min(POST_RHS, nrhs - r0);
    const size_t smem = sizeof(double) * (size_t)(4 * p + 4 * (p - 1)) * nr;
    if (smem > 48 * 1024) {
      static bool attr = false;
      if (!attr) {
        HPS_CUDA_CHECK(cudaFuncSetAttribute(k_leaf_fields, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)(sizeof(double) * (4 * 32 + 4 * 31) * POST_RHS)));
        attr = true;
      }
    }
    k_leaf_fields<<<grid, 256, smem, st>>>(nlist, p, U, ldu, r0, nr, leaves, leaf_Ie, gid, L1, Psi, J_i, J_e, W,
                                           nrhs);
    HPS_LAUNCH_CHECK();
  }
  return HPS_OK;
}

extern "C" int hps_eval_points(int npts, int p, const double* W, int nrhs, const int* slot, const double* rx,
                               const double* ry, double* out, void* stream) {
  if (npts <= 0 || nrhs <= 0) return HPS_OK;
  k_eval_points<<<(npts + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(npts, p, W, nrhs, nrhs, slot, rx,
                                                                                ry, out);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

extern "C" int hps_gauge_sides(int nlist, int p, const double* W, int nrhs, const double* Qx, const double* Qy,
                               double* side, void* stream) {
  if (nlist <= 0 || nrhs <= 0) return HPS_OK;
  k_gauge_sides<<<std::min(nlist, 148 * 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(nlist, p, W, nrhs, nrhs,
                                                                                          Qx, Qy, side);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

extern "C" int hps_gauge_gather(int N, int nrhs, const double* side, const int* src, const double* u_in,
                                int ldu_in, double* u_out, int ldu_out, void* stream) {
  if (N <= 0 || nrhs <= 0) return HPS_OK;
  const long long total = (long long)N * nrhs;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  k_gauge_gather<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(N, nrhs, side, src, u_in, ldu_in, u_out,
                                                                       ldu_out);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}
