/* hps_b200.h -- C ABI of the B200-native HPS build/solve hot path (libhps_b200.so).
 *
 * All pointers are DEVICE pointers unless noted. All matrices are fp64 row-major. `stream` is a
 * cudaStream_t passed as void*. Every entry point returns a status code. On HPS_ERR_* the call
 * sets a message, readable through hps_last_error(). Numerical failures are reported through
 * device-side status words (-1 = ok), so a whole build can be enqueued without host syncs.
 *
 * Reference interfaces replaced (the reference is pure Python; these are its BLAS/LAPACK call
 * sites):
 *   hps_leaf_stage   <- solver._leaf_stage chunk loop, solver.py:226-246
 *                       (assemble_operator leafops.py:217-233, interior_solve_batch
 *                        leafops.py:273-295, DtN product solver.py:241-242)
 *   hps_merge_level  <- merge.merge_dtn, merge.py:92-119, for all 2^d parents of one depth
 *   hps_lu_solve_batched <- scipy.linalg.lu_factor / lu_solve (LAPACK getrf/getrs), merge.py:106-110
 *                       (the dense-branch loop body of solver.build, solver.py:266-285)
 *   hps_solve_level  <- SolutionOperator.apply inside solver.solve, solver.py:93-97 / 312-315,
 *                       for all parents of one depth and a batch of right-hand sides
 *   hps_dgemm_batched <- the BLAS dgemm behind `@` (merge.py:118, solver.py:71 apply_global_dtn)
 *   hps_leaf_hash / hps_leaf_verify <- the leaf grouping of solver._leaf_stage, solver.py:208-222
 *                       (np.unique over the stacked coefficient sample rows)
 *   hps_leaf_fields / hps_eval_points <- _leaf_field + the barycentric evaluation of post_process and
 *                       boundary_flux_at, solver.py:349-400
 *   hps_tree_sizes / hps_tree_layout <- grid.build_tree, grid.py:204-322 (host code)
 *   hps_gauge_sides / hps_gauge_gather <- (new) Gauss-node solution
 *                       re-tabulated from the leaf fields with the L4 blocks (leafops.py:191-198)
 */
#ifndef HPS_B200_H
#define HPS_B200_H
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_OK 0
#define HPS_ERR_LEAF_RESONANCE 1
#define HPS_ERR_MERGE_RESONANCE 2
#define HPS_ERR_CUDA 3
#define HPS_ERR_NCCL 4
#define HPS_ERR_ARG 5

/* Library context: owns the library's side streams (interface-inverse fork stream, look-ahead
 * pair), their events, the split-K scratch and the tuning options of one device. Create one per
 * device and per build in flight (two concurrent builds on two streams use two contexts). Calls
 * taking a context are thread-compatible per context; the context's device must be current.
 * hps_ctx_destroy synchronises its device and frees everything the context allocated. */
typedef struct hps_ctx_s* hps_ctx_t;
#define HPS_OPT_SPLITK 0            /* split-K of under-filled GEMMs (1); 0: every GEMM batch-invariant */
#define HPS_OPT_GEMM_GROUP_M 1      /* grouped tile rasterisation of the 64x64 GEMM (16; 0 row-major) */
#define HPS_OPT_INV_FORK 2          /* block-inverse GEMM pairs on the fork stream (1) */
#define HPS_OPT_LEAF_CTAS_PER_SM 3  /* leaf kernel CTAs per SM (2) */
#define HPS_OPT_LEAF_FREE_SMS 4     /* leaf grid sized for this many fewer SMs (0) */
#define HPS_OPT_PROFILE_AHEAD 5     /* timing events around the look-ahead inverse (0; dev tool) */
#define HPS_OPT_EMU_SLICES 6        /* FP64 GEMM emulation on the int8 tensor cores, slice scheme: 7-bit slices
                                       per operand, s (s + 1) / 2 int8 products (0 = off; used when
                                       HPS_OPT_EMU_MODULI is 0); the merges' S / T GEMMs and hps_dgemm_batched */
#define HPS_OPT_EMU_MIN_WORK 7      /* emulate GEMMs with M N K batch >= this (2^32) */
#define HPS_OPT_EMU_MIN_K 8         /* ... and K >= this (512): below it the residue and reconstruction passes
                                       cost more than DMMA saves */
#define HPS_OPT_EMU_MODULI 9        /* FP64 GEMM emulation, modular scheme: one int8 product per modulus
                                       (14, FP64-equivalent; 6..16; 0 = off) with Chinese-remainder
                                       reconstruction; takes precedence over HPS_OPT_EMU_SLICES */
#define HPS_OPT_EMU_SCRATCH_MB 10   /* cap on the modular scheme's product scratch (8192 MB) */
#define HPS_OPT_EMU_ENGINE 11       /* int8 products of the modular scheme: this library's tcgen05 kernel (TMA +
                                       TMEM, residues reduced in its epilogue) on single CTAs, 128 x 256 tiles (0)
                                       or CTA pairs, 256 x 256 tiles (2); cuBLASLt IMMA (1) */
#define HPS_OPT_EMU_TILE_GROUP 12   /* tile rows per group of the tcgen05 kernel's tile order (0: ~32 MB of A) */
#define HPS_OPT_EMU_SOLVE 13        /* batched solve (b >= 64) through the emulation too (0: DMMA; measured slower
                                       at b = 256: S is read once, its residues cost about what DMMA saves) */
#define HPS_OPT_EMU_SPLIT 14        /* operand residues of the modular scheme: integer pipes + a small int8 MMA per
                                       element pair (1) or the FP64 pipe (0) */
#define HPS_OPT_COUNT 15
int hps_ctx_create(int device, hps_ctx_t* out);
int hps_ctx_destroy(hps_ctx_t ctx);
int hps_ctx_set_option(hps_ctx_t ctx, int option, long long value);
long long hps_ctx_get_option(hps_ctx_t ctx, int option); /* -1 on a bad context or option */
int hps_ctx_device(hps_ctx_t ctx);

const char* hps_last_error(void);
int hps_version(void);
int hps_device_check(int* major, int* minor, int* sms);
/* Kernels launched by this library so far in this process (benchmark accounting). */
long long hps_launch_count(void);
/* Host-side tree / node layout (<- grid.build_tree, grid.py:204-322): sizes,
 * then the arrays, all HOST pointers and caller-allocated. hps_tree_sizes fills n3/ne/m per depth
 * d < 2L (arrays of max(2L, 1) entries) and returns N, the number of Gauss nodes (-1 on bad
 * arguments). hps_tree_layout writes points[N][2], on_vertical[N], leaf_cells[4^L][2],
 * leaf_I_e[4^L][4q], and per depth Ie[d] ([2^d][ne]) and maps[d] (j1a[ne/2], j2b[ne/2], j3a[n3],
 * j3b[n3]); gauss01[q] = (Gauss-Legendre nodes + 1) / 2. Bit-exact with the reference layout. */
long long hps_tree_sizes(int L, int q, long long* n3, long long* ne, long long* m);
int hps_tree_layout(int L, int q, double x_lo, double y_lo, double width, double height, const double* gauss01,
                    double* points, unsigned char* on_vertical, long long* leaf_cells, long long* leaf_I_e,
                    long long* const* Ie, long long* const* maps);

/* Leaf stage for `ngroups` distinct coefficient groups (leaves with bitwise-equal samples share a
 * group, solver.py:208-222).
 *   fields[6]  host array of device pointers (ngroups x p^2 samples, x1-major grid) or NULL
 *   scalars[6] host array; used where fields[f] == NULL; a scalar 0 skips the term
 *   consts     Dx, Dy, Dx@Dx, Dy@Dy (p^2 each), L43[:,J_e] (4p x nb), L43[:,J_i] (4p x ni),
 *              L1 (nb x 4p), probe (ni); ni = (p-2)^2, nb = 4(p-1)
 *   idx        int32 J_i (ni), J_e (nb)
 * Outputs: Psi (ngroups x ni x nb), T (ngroups x 4p x 4p), cond (ngroups, probe estimate of
 * leafops.py:293-294; the caller raises LeafResonanceError if cond > 1e13). */
size_t hps_leaf_workspace_bytes(hps_ctx_t ctx, int p, int ngroups); /* ctx NULL: default 148-SM context */
int hps_leaf_stage(hps_ctx_t ctx, int p, int ngroups, const double* const* fields, const double* scalars,
                   const double* consts, const int* idx, double probe_max, double* Psi, double* T,
                   double* cond, void* ws, size_t ws_bytes, void* stream);

/* All 2^d merges of one depth. Children of merge b are T_child + child_idx[2b(+1)]*child_stride
 * (child_idx NULL => 2b, 2b+1), each m x m with m = ne/2 + n3.
 *   maps   int32 j1a (ne/2), j2b (ne/2), j3a (n3), j3b (n3)   (merge.py:27-89 split positions)
 *   vmode  q start + q end values of the corner null mode on one interface segment
 * Outputs S_out (nbatch x n3 x ne), T_out (nbatch x ne x ne). *status (device int, init -1) is raised to
 * the largest merge index whose interface system is singular or whose S is non-finite
 * (MergeResonanceError, merge.py:106-112). */
size_t hps_merge_workspace_bytes(int nbatch, int n3, int ne);
int hps_merge_level(hps_ctx_t ctx, int nbatch, int n3, int ne, int m, int q, const double* T_child,
                    long long child_stride, const int* child_idx, const int* maps,
                    const double* vmode, double* S_out, double* T_out, void* ws, size_t ws_bytes,
                    int* status, int status_base, void* stream);
/* Interface factorisation of n3 > 128 (flags of hps_merge_level_ahead / hps_merge_interface /
 * hps_interface_solve). Default: the recursive 2x2 block inverse (DMMA GEMMs over 128-blocks, each
 * inverted by pivoted Gauss-Jordan) followed by a residual check X_d (X_d^-1 v) - v on a +-1 probe;
 * above 1e-6 (or non-finite) the depth's status word becomes HPS_STATUS_PIVOT + merge index and the
 * caller re-runs the depth with HPS_MERGE_PIVOTED: the pivoted LU of hps_lu_solve_batched (partial
 * pivoting over the whole column, as LAPACK getrf in merge.py:106-110). HPS_MERGE_PARENT_PIVOTED asks
 * the same for the look-ahead's parent depth. n3 <= 128 always uses pivoted Gauss-Jordan. */
#define HPS_MERGE_PIVOTED 1
#define HPS_MERGE_PARENT_PIVOTED 2
#define HPS_STATUS_PIVOT (1 << 24)

/* hps_merge_level plus a look-ahead for the parent depth (the next call): before this depth's big
 * T GEMM, the parent's interface matrix X = Ta[pj3a, pj3a] - Tb[pj3b, pj3b] is formed from the pj3
 * rows / columns of this depth's T = blk + C S (one GEMM over gathered operands), deflated and
 * inverted in the parent's workspace `pws` on a high-priority library stream, concurrently with the
 * T GEMM; the call joins it before returning. The parent's call then passes pre_inverted = 1 (with
 * the same workspace) and skips its own X gather, deflation and inverse. pmaps = NULL: no
 * look-ahead. nbatch must be even when pmaps is set. */
int hps_merge_level_ahead(hps_ctx_t ctx, int nbatch, int n3, int ne, int m, int q, const double* T_child,
                          long long child_stride, const int* child_idx, const int* maps, const double* vmode,
                          double* S_out, double* T_out, void* ws, size_t ws_bytes, int* status, int status_base,
                          int pre_inverted, const int* pmaps, int pn3, int pne, const double* pvmode, void* pws,
                          size_t pws_bytes, int* pstatus, int pstatus_base, int flags, void* stream);

/* Split merge of the distributed top depths (parallel.py): the parent's owner runs
 * hps_merge_interface (gathers, deflation, factorisation: the in-place inverse for n3 <= 128, the
 * pivoted LU for n3 > 128; outputs the factored X, its row permutation (identity for n3 <= 128), R
 * and C, each nbatch-batched like hps_merge_level's workspace); every rank of the parent's group
 * solves a column panel S_p = X^-1 R[:, panel] (hps_interface_solve) and forms T_p = C S_p
 * (hps_dgemm_batched); the owner assembles T = blkdiag(Ta11, Tb22) + [T_0 | T_1 | ...]
 * (hps_merge_assemble; panels laid out [npanels][nbatch][ne][ne / npanels]). Same per-element
 * arithmetic as hps_merge_level. */
int hps_merge_interface(hps_ctx_t ctx, int nbatch, int n3, int ne, int m, int q, const double* T_child,
                        long long child_stride, const int* child_idx, const int* maps, const double* vmode,
                        double* Xf_out, int* perm_out, double* R_out, double* C_out, void* ws, size_t ws_bytes,
                        int* status, int status_base, int flags, void* stream);
int hps_interface_solve(hps_ctx_t ctx, int n3, int ncols, int batch, const double* Xf, const int* perm,
                        const double* R, double* S_out, int* status, int status_base, int flags, void* stream);
int hps_merge_assemble(hps_ctx_t ctx, int nbatch, int ne, int m, const double* T_child, long long child_stride,
                       const int* child_idx, const int* maps, const double* panels, int npanels, double* T_out,
                       void* stream);

/* u[ii_start0 + b*n3 + r, :nrhs] = sum_c S[b][r][c] * u[Ie[b][c], :nrhs] for all nbatch parents of
 * one depth; u is node-major with leading dimension ldu (solver.py:312-315). */
int hps_solve_level(hps_ctx_t ctx, int nbatch, int n3, int ne, const double* S, const int* Ie, long long ii_start0,
                    double* u, int ldu, int nrhs, void* stream);

/* In-place inverse of `batch` n x n matrices: partial-pivoting Gauss-Jordan for n <= 128 (what the
 * merges use there); above 128 a recursive 2x2 block inverse on the DMMA GEMM, which pivots only
 * inside its 128-blocks (a utility; the merges factor n3 > 128 with hps_lu_solve_batched's LU).
 * *status as above. */
size_t hps_inverse_workspace_bytes(int n, int batch);
int hps_inverse_batched(hps_ctx_t ctx, int n, int batch, double* X, long long lda, long long strideX, void* ws,
                        size_t ws_bytes, int* status, void* stream);

/* Pivoted LU (partial pivoting over the whole column, LAPACK getrf row order; merge.py:106-110) of
 * `batch` n x n matrices X (stride n^2, overwritten by L\U), then S = X^-1 R (R, S: n x ne per
 * matrix) by two triangular solves. ipiv_out (optional, device, batch x n): LAPACK-style 0-based
 * swap rows. *status (init -1) is raised to b for a zero pivot column or a non-finite S. This is
 * the factorisation hps_merge_level uses for interfaces of n3 > 128. */
size_t hps_lu_workspace_bytes(int n, int batch);
int hps_lu_solve_batched(hps_ctx_t ctx, int n, int ne, int batch, double* X, const double* R, double* S_out,
                         int* ipiv_out, void* ws, size_t ws_bytes, int* status, void* stream);

/* C[b] = alpha A[b] B[b] + beta C[b]; optional B-row gather Bidx (NULL = none). K % 16 == 0. */
int hps_dgemm_batched(hps_ctx_t ctx, int M, int N, int K, int batch, double alpha, const double* A, long long lda,
                      long long strideA, const double* B, long long ldb, long long strideB,
                      const int* Bidx, long long strideBidx, double beta, double* C, long long ldc,
                      long long strideC, void* stream);

/* The int8 residue products of the modular FP64 emulation (the core of hps_dgemm_batched's emulated
 * path, merge.py:108/118), exposed for tests and benchmarks: for z < nz and the output column panel
 * [j0, j0 + nc),
 *   R[z][i][j] = ((sum_k A[z][i][k] B[z][j0 + j][k]) mod moduli[z / batch]) + 128   (uint8, [nz][M][nc])
 * with A int8 [nz][M][K], B int8 [nz][N][K] (K contiguous), 2 <= moduli[l] <= 256, K % 16 == 0,
 * N % 16 == 0, nc % 32 == 0, K < 65536. engine: 0 = tcgen05 single-CTA kernel, 2 = CTA-pair
 * kernel. Device pointers; stream is a cudaStream_t. */
int hps_i8gemm_mod(hps_ctx_t ctx, const signed char* A, const signed char* B, unsigned char* R, int M, int N, int nc,
                   int j0, int K, int nz, int batch, const int* moduli, int nmod, int engine, void* stream);

/* Leaf grouping (solver.py:208-222). fields: HOST array of nfields (1..6) DEVICE pointers, each to
 * n_leaf x row_len fp64 samples. hps_leaf_hash writes a 64-bit hash of every leaf's rows;
 * hps_leaf_verify sets *mismatch (device int) to 1 if some leaf's rows differ bitwise from those of
 * leaf rep_of[leaf], i.e. the hash grouping had a collision and must be redone exactly. */
int hps_leaf_hash(int n_leaf, int row_len, int nfields, const double* const* fields,
                  unsigned long long* hash, void* stream);
int hps_leaf_verify(int n_leaf, int row_len, int nfields, const double* const* fields,
                    const long long* rep_of, int* mismatch, void* stream);

/* Post-processing (solver.py:349-400). U: N x ldu node-major solution (nrhs columns used).
 * hps_leaf_fields: for s < nlist, leaf = leaves[s]: W[s][i*p+j][r] (ldw = nrhs) = the p x p Chebyshev
 *   field of RHS r: w_e = L1 u[leaf_Ie[leaf][0..4p)], w_i = Psi[gid[leaf]] w_e, scattered by J_e / J_i.
 *   L1: 4(p-1) x 4p; Psi: groups x (p-2)^2 x 4(p-1).
 * hps_eval_points: out[t][r] = sum_ij rx[t][i] W[slot[t]][i*p+j][r] ry[t][j] (rx, ry: npts x p).
 * hps_gauge_sides: side[s][k][r] = Gauss value at the k-th I_e node of listed leaf s re-tabulated from
 *   W[s] (sides S, E, N, W: Qx W[:,0], Qy W[p-1,:], Qx W[:,p-1], Qy W[0,:]; Qx, Qy: p x p).
 * hps_gauge_gather: u_out[node][r] = mean of side rows src[2 node], src[2 node + 1] (-1: absent);
 *   src[2 node] == -1 keeps u_in[node][r]. */
int hps_leaf_fields(int nlist, int p, const double* U, int ldu, int nrhs, const int* leaves,
                    const int* leaf_Ie, const int* gid, const double* L1, const double* Psi,
                    const int* J_i, const int* J_e, double* W, void* stream);
int hps_eval_points(int npts, int p, const double* W, int nrhs, const int* slot, const double* rx,
                    const double* ry, double* out, void* stream);
int hps_gauge_sides(int nlist, int p, const double* W, int nrhs, const double* Qx, const double* Qy,
                    double* side, void* stream);
int hps_gauge_gather(int N, int nrhs, const double* side, const int* src, const double* u_in,
                     int ldu_in, double* u_out, int ldu_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
