// Leaf grouping on the device (solver.py:208-222 of the reference groups leaves whose coefficient
// sample rows are bitwise equal, so the leaf stage factors each distinct leaf operator once).
//   hps_leaf_hash:   one warp per leaf: a wrapping 64-bit dot product of the sample bit patterns
//                    with position-dependent odd weights (splitmix64 of the word index).
//   hps_leaf_verify: one warp per leaf: bitwise compare of the leaf's rows with its representative's;
//                    any mismatch (a hash collision) sets *mismatch and the host regroups exactly.
#include <cstdint>

#include "common.cuh"

namespace hps {

struct FieldSet {
  const double* f[6];
  int nf;
};

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void k_leaf_hash(int n_leaf, int row_len, FieldSet fs, unsigned long long* __restrict__ hash) {
  const int leaf = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (leaf >= n_leaf) return;
  unsigned long long h = 0ull;
  for (int f = 0; f < fs.nf; ++f) {
    const unsigned long long* row =
        reinterpret_cast<const unsigned long long*>(fs.f[f]) + (long long)leaf * row_len;
    for (int i = lane; i < row_len; i += 32)
      h += __ldg(row + i) * (splitmix64((unsigned long long)(f * row_len + i)) | 1ull);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if (lane == 0) hash[leaf] = h;
}

__global__ void k_leaf_verify(int n_leaf, int row_len, FieldSet fs, const long long* __restrict__ rep_of,
                              int* __restrict__ mismatch) {
  const int leaf = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (leaf >= n_leaf) return;
  const long long rep = rep_of[leaf];
  if (rep == leaf) return;
  bool diff = rep < 0 || rep >= n_leaf;
  for (int f = 0; f < fs.nf && !diff; ++f) {
    const unsigned long long* a = reinterpret_cast<const unsigned long long*>(fs.f[f]) + (long long)leaf * row_len;
    const unsigned long long* b = reinterpret_cast<const unsigned long long*>(fs.f[f]) + rep * row_len;
    for (int i = lane; i < row_len; i += 32) diff |= __ldg(a + i) != __ldg(b + i);
  }
  if (__any_sync(0xffffffffu, diff) && lane == 0) atomicOr(mismatch, 1);
}

static int fieldset(int nfields, const double* const* fields, FieldSet& fs) {
  if (nfields < 1 || nfields > 6) {
    set_error("leaf grouping: nfields=%d (1..6)", nfields);
    return HPS_ERR_ARG;
  }
  fs.nf = nfields;
  for (int f = 0; f < 6; ++f) fs.f[f] = f < nfields ? fields[f] : nullptr;
  return HPS_OK;
}

}  // namespace hps

using namespace hps;

// hash[leaf] over the nfields sample rows (row_len doubles each) of every leaf.
extern "C" int hps_leaf_hash(int n_leaf, int row_len, int nfields, const double* const* fields,
                             unsigned long long* hash, void* stream) {
  if (n_leaf <= 0) return HPS_OK;
  FieldSet fs;
  const int s = fieldset(nfields, fields, fs);
  if (s != HPS_OK) return s;
  k_leaf_hash<<<(n_leaf + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(n_leaf, row_len, fs, hash);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}

// *mismatch |= 1 if any leaf's rows differ bitwise from those of rep_of[leaf].
extern "C" int hps_leaf_verify(int n_leaf, int row_len, int nfields, const double* const* fields,
                               const long long* rep_of, int* mismatch, void* stream) {
  if (n_leaf <= 0) return HPS_OK;
  FieldSet fs;
  const int s = fieldset(nfields, fields, fs);
  if (s != HPS_OK) return s;
  k_leaf_verify<<<(n_leaf + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(n_leaf, row_len, fs, rep_of,
                                                                                 mismatch);
  HPS_LAUNCH_CHECK();
  return HPS_OK;
}
