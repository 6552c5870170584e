/*
 * skeweig_stages.h -- stage-level C-ABI entry points of the sm_100a path, used by
 * the parity tests (kernel-level checks on shared inputs, SURVEY §4 tier 2) and by
 * bench.py for per-kernel roofline numbers.  Same conventions as skeweig.h
 * (FP64, column-major, device pointers unless stated, synchronous, caller-owned
 * arrays, workspace from skew_set_workspace sized for the same n).
 */
#ifndef SKEWEIG_STAGES_H
#define SKEWEIG_STAGES_H
#include "skeweig.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Full-to-band reduction (Eqs. (6)-(8)) of the skew A (strictly
 * lower, destroyed).  On return the band (width b = ctx band width) is in
 * A[c+1 .. c+b, c].  When Vout != NULL: Vout (n x npanel*b, ldv >= n, zero-filled by
 * the callee) receives V_j in columns j*b..j*b+b-1 at rows r0_j = (j+1)b.., with
 * explicit unit diagonal; Tout (b x npanel*b) the compact-WY T_j
 * (Q_j = I - V_j T_j V_j^T, Eq. (6)); tau_out (npanel*b) the tau's.
 * *npanel_out = number of panels = max(0, floor((n-2)/b)). */
int skew_stage_reduce_to_band(skew_ctx ctx, int64_t n, double* A, int64_t lda,
                              double* Vout, int64_t ldv, double* Tout, double* tau_out,
                              int64_t* npanel_out);

/* Band-to-tridiagonal bulge chasing of the band matrix given in
 * LOWER BAND STORAGE AB (ldab >= b+1): AB[d + c*ldab] = B[c+d, c], 0 <= d <= b.
 * alpha_out (n-1): Lemma-1 off-diagonals, alpha_k = -T[k+1,k] (reading R2).
 * When X != NULL (n x ncols, ldx): X <- Q2 X with B = Q2 T Q2^T (BT2 path). */
int skew_stage_band_to_tridiag(skew_ctx ctx, int64_t n, int b, const double* AB, int64_t ldab,
                               double* alpha_out, double* X, int64_t ldx, int64_t ncols);

/* Tridiagonal stage (Lemma 1 + bisection + inverse iteration, PAPER.md:248-262,
 * 616-617): top-nev eigenpairs of tridiag(alpha, 0, alpha) (size n).
 * lambda (nev) descending; Q (n x nev, ldq) or NULL for eigenvalues only. */
int skew_stage_tridiag_eig(skew_ctx ctx, int64_t n, const double* alpha, int64_t nev,
                           double* lambda, double* Q, int64_t ldq);

/* Kernel accounting for measurement.  Every kernel launch of the library belongs to
 * one of SKEW_KERNEL_CLASSES classes (skew_kernel_class_name); skew_kernel_stats
 * returns, for the last call, the number of launches per class and -- when
 * profiling is on -- the summed device time (ms) of each class measured with CUDA
 * events recorded on the context stream around the launches.  The last class,
 * "collectives", times the NCCL / virtual-group collectives of a distributed solve
 * (panel broadcast, skew-SYMM allreduce, band allreduce, eigenvalue allgather). */
#define SKEW_KERNEL_CLASSES 21
int skew_set_profiling(skew_ctx ctx, int on);
int skew_kernel_stats(skew_ctx ctx, double* ms_out, int64_t* launches_out, int count);
const char* skew_kernel_class_name(int cls);

/* The rank-2k update's lower-triangular tile schedule (host function, no GPU needed):
 * fills tm_out / tn_out (capacity cap) with the (row tile, column tile) pairs the
 * skew rank-2k kernel of rank `rank` of `nranks` visits on a trailing matrix of order
 * ntm*128 (128-row x 64-column tiles of the TMA-fed kernel; 1D block-cyclic ownership of the
 * 64-wide column blocks, rank(q) = (q - qoff) mod nranks with qoff = 0 here), in launch order:
 * tile (tm, tn) covers rows [128 tm, 128 tm + 128) and columns [64 tn, 64 tn + 64) and is
 * visited iff it meets the strictly lower triangle.  Returns the count (or -i for argument i).
 * Tests check that the ranks' sets partition the lower triangle (tests/test_tile_schedule.py). */
int64_t skew_tile_schedule(int64_t ntm, int nranks, int rank, int64_t* tm_out, int64_t* tn_out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
