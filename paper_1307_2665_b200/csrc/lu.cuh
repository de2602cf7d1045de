// Pivoted blocked LU of the large interface systems and the solve through it (lu.cu).
#pragma once
#include "common.cuh"

namespace hps {

struct Ctx;
struct LuWs {
  int* ipiv = nullptr;  // batch x n: LAPACK-style sequential row swaps
  int* perm = nullptr;  // batch x n: resulting permutation (row i of P X = row perm[i] of X)
};
LuWs lu_ws(void* base, int n, int batch);
size_t lu_ws_bytes(int n, int batch);
// P X = L U in place (batch x n x n, stride n^2); a zero pivot column raises *status to status_base + b.
int lu_factor(Ctx& cx, double* X, int n, int batch, const LuWs& ws, int* status, int status_base, cudaStream_t st);
// S = X^-1 R = U^-1 L^-1 P R (R, S: batch x n x ne); a non-finite S raises *status.
int lu_solve(Ctx& cx, const double* X, int n, int batch, const LuWs& ws, const double* R, int ne, double* S_out,
             int* status, int status_base, cudaStream_t st);

}  // namespace hps
