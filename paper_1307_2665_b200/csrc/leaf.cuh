// Shared declarations of the leaf-stage kernels (leaf.cu: generic p; leaf3.cu: the p = 16 kernel).
#pragma once
#include "common.cuh"

namespace hps {

struct LeafArgs {
  int p, ngroups;
  // coefficient samples, rows = group representatives (ngroups x p^2); null => scalar
  const double* field[6];
  double scalar[6];
  int present[6];  // 0 => scalar zero, term skipped (leafops.py:220-221)
  const double* consts;  // Dx, Dy, Dxx, Dyy, L43e, L43i, L1, probe
  const int* idx;        // J_i, J_e
  double probe_max;
  double* Psi;   // ngroups x ni x nb
  double* T;     // ngroups x 4p x 4p
  double* cond;  // ngroups
  double* scratch;
  long long scratch_stride;  // doubles per CTA slot
};

// p = 16: blocked LU with warp-specialised panels (leaf3.cu). scratch_stride is set by the launcher.
struct Ctx;
size_t leaf16v3_scratch_doubles();
int leaf16v3_grid(const Ctx& cx, int ngroups);
int launch_leaf16v3(LeafArgs& a, Ctx& cx, cudaStream_t st);

}  // namespace hps
