/*
 * skeweig.h -- C-ABI of the B200-native (sm_100a) two-stage skew-symmetric
 * eigensolver (Penke, Marek, Vorwerk, Draxl, Benner, arXiv 1912.04062).
 *
 * Problem (Algorithm 1): for a real skew-symmetric
 * A = -A^T (n x n), return the eigenpairs A z_k = i*lambda_k z_k with lambda_k > 0,
 * the nev <= floor(n/2) LARGEST, in descending order (the other half are the
 * conjugate pairs -i*lambda_k, conj(z_k)).  Eigenvectors are unit
 * 2-norm; their phase is free (reading R7).
 *
 * Route (ELPA2 flavour): full->band (panel QR + skew rank-2k
 * update, Eqs. (6)-(8)), band->tridiagonal bulge chasing
 * (PAPER.md:446-462), Lemma 1 link to tridiag(alpha, 0, alpha)
 * solved by bisection + inverse iteration, Q <- D Q_diag
 * (PAPER.md:307-311), then the two back-transformations on [Re | Im] as one real
 * n x 2nev matrix.
 *
 * Conventions (all entry points):
 *  - FP64, column-major, 0-based, 64-bit sizes.
 *  - A skew input is read from its STRICTLY LOWER triangle only; the diagonal and
 *    upper triangle are never read.
 *  - Array pointers of skew_eig / skew_eig_range / skew_eigvals / skew_eig_bse may be
 *    DEVICE pointers (cudaMalloc / torch) or HOST pointers (pageable or pinned).  The
 *    library detects the kind with cudaPointerGetAttributes; host inputs are staged
 *    through the workspace (the workspace must then be sized with SKEW_WS_HOST_STAGING).
 *    Zre and Zim must be of the same kind.  The BSE pipeline stages
 *    (skew_bse_build_M, skew_bse_backtransform) and the stage entry points take device
 *    pointers only.
 *  - Non-finite input (a NaN or Inf in the triangle that is read) is an argument error
 *    (-3, the A or M argument), detected before any reduction starts.
 *  - Ownership: every array belongs to the caller.  A (or M) is INPUT AND
 *    DESTROYED when it is a device array (it receives reflectors and the band;
 *    contents unspecified on return, LAPACK convention); a host A is not modified.
 *    Outputs must not alias inputs.
 *  - The library never allocates device memory in a solve: it uses the caller's
 *    workspace (skew_workspace_size / skew_set_workspace).
 *  - Calls are synchronous: work is enqueued on the context stream and the
 *    stream is synchronised before returning, so the status is final.
 *  - One context must not be used by two host threads at once; distinct
 *    contexts are independent.
 *
 * Status codes: 0 ok; -i: the i-th argument is invalid (LAPACK INFO style, the
 * context counts as argument 1); positive codes below.
 */
#ifndef SKEWEIG_H
#define SKEWEIG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKEW_OK 0
#define SKEW_ERR_NOCONV 1          /* inverse iteration did not converge for some vectors */
#define SKEW_ERR_NOT_DEFINITE 4    /* BSE: Cholesky pivot <= n*eps*max(diag M) */
#define SKEW_ERR_CUDA 10           /* a CUDA runtime error (message: skew_last_error) */
#define SKEW_ERR_NCCL 11
#define SKEW_ERR_WORKSPACE 12      /* workspace missing or too small */
#define SKEW_ERR_NOT_IMPLEMENTED 13

/* workspace flags */
#define SKEW_WS_VECTORS 1          /* eigenvectors requested (else eigenvalues only) */
#define SKEW_WS_HOST_STAGING 2     /* room to stage host A (n x n) */
#define SKEW_WS_BSE 4              /* room for the BSE front-end (Cholesky factor) */
#define SKEW_WS_BSE_BACKTRANSFORM 8 /* room for skew_bse_backtransform's scratch (16 n2 nev bytes) */
#define SKEW_WS_ONESTEP 16         /* size for skew_eig_onestep (with SKEW_WS_VECTORS for vectors) */

/* skew_eig_bse flags */
#define SKEW_BSE_HAMILTONIAN_Y 1   /* return y = J L z (H y = -i lambda y, H = -J M) instead of z */

typedef struct skew_ctx_s* skew_ctx;

/* Create a context on CUDA device `device` that enqueues on `cuda_stream`
 * (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream; NULL = legacy
 * default stream).  The internal band width is b = 64 (fixed: the panel, bulge-chase and
 * BT2 kernels are built for it; reading R10).  Tunables are read from the
 * environment once here: SKEWEIG_BT1_MERGE (panels per BT1 block reflector, 1..8,
 * default 8), SKEWEIG_REORTH_W (reorthogonalisation window, default 32). */
int skew_ctx_create(skew_ctx* out, int device, void* cuda_stream);
int skew_ctx_destroy(skew_ctx ctx);

/* Multi-GPU (one process per GPU).  skew_get_unique_id fills 128 bytes (an NCCL unique
 * id) on one rank; the caller distributes them (e.g. torch.distributed) and every rank
 * calls skew_ctx_create_dist with the same bytes.  On such a context the solve entry
 * points are collective: every rank passes the SAME A; the full->band reduction is
 * distributed by b-wide column blocks (1D block-cyclic, owner of column c = (c/64) mod
 * nranks; NCCL broadcast of each panel's V, T, tau and allreduce of the skew-SYMM
 * products); the band is combined with an allreduce; the eigenvectors
 * are sharded by skew_eig_range (each rank its own [k0, k1)).
 * Returns SKEW_ERR_NCCL on communicator failure. */
int skew_get_unique_id(char id[128]);
int skew_ctx_create_dist(skew_ctx* out, int device, void* cuda_stream, int nranks, int rank, const char id[128]);

/* Virtual ranks (test harness for the distributed path on ONE device): skew_vgroup_create
 * makes a group of nranks; skew_ctx_create_virtual makes the context of rank `rank` in it
 * (all on `device`).  Each rank's solve must be called from its own host thread (the
 * collectives meet at host barriers; the contexts may share one stream).  The distributed
 * algorithm is the one of skew_ctx_create_dist (same ownership, partitions, ghost windows);
 * the collectives are device copies and a fixed-order sum kernel that read the peers'
 * buffers.  The group allocates its own reduction scratch (cudaMalloc) and must outlive its
 * contexts.  Returns -i for a bad argument i. */
int skew_vgroup_create(int nranks, void** out);
int skew_vgroup_destroy(void* group);
int skew_ctx_create_virtual(skew_ctx* out, int device, void* cuda_stream, void* group, int nranks, int rank);

/* Bytes of device workspace a solve of order n with nev pairs needs (flags:
 * SKEW_WS_*).  The caller allocates it (e.g. a torch uint8 tensor) and passes it
 * with skew_set_workspace; it must stay alive while the context uses it. */
int skew_workspace_size(skew_ctx ctx, int64_t n, int64_t nev, int flags, size_t* bytes);
int skew_set_workspace(skew_ctx ctx, void* dptr, size_t bytes);

/* Eigenpairs (Algorithm 1, ELPA2 flavour, half spectrum).
 *   n        >= 1
 *   A        n x n (lda >= n), strictly lower triangle read; destroyed if device
 *   nev      1 <= nev <= floor(n/2)
 *   lambda   nev doubles out, lambda_0 >= lambda_1 >= ... > 0
 *   Zre, Zim n x nev each (ldz >= n): z_k = Zre[:,k] + i Zim[:,k]
 * Returns 0, -i (bad argument i), SKEW_ERR_NOCONV, SKEW_ERR_CUDA, SKEW_ERR_WORKSPACE. */
int skew_eig(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev,
             double* lambda, double* Zre, double* Zim, int64_t ldz);

/* Same solve, eigenvectors of the index range [k0, k1) only (0 <= k0 < k1 <= nev):
 * lambda receives all nev eigenvalues, Zre/Zim (n x (k1-k0), ldz) the vectors
 * z_{k0} .. z_{k1-1}.  This is the per-rank call of the multi-GPU path (DESIGN.md
 * "Multi-GPU": each rank owns a contiguous eigenpair range; the back-transforms of
 * different ranges are independent). */
int skew_eig_range(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev, int64_t k0, int64_t k1,
                   double* lambda, double* Zre, double* Zim, int64_t ldz);

/* Eigenvalues only (Algorithm 1 steps 1-2): the nev largest lambda_k, descending. */
int skew_eigvals(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev, double* lambda);

/* BSE form (steps 2-3): M (n x n, n even, symmetric positive
 * definite, lower triangle incl. diagonal read) -> M = L L^T (Cholesky) -> W = L^T J L
 * with J = [[0, I], [-I, 0]] -> eigenpairs of the skew W as in skew_eig.
 *   M       device: destroyed, receives L (lower triangle, upper zeroed); host: staged
 *           through the workspace (size it with SKEW_WS_BSE | SKEW_WS_HOST_STAGING), not
 *           modified
 *   flags   0, or SKEW_BSE_HAMILTONIAN_Y: Zre/Zim receive y_k = J L z_k instead of z_k
 *           (H y_k = -i lambda_k y_k for H = -J M; not normalised, ||y_k|| =
 *           ||L z_k||); needs Zre/Zim
 *   Zre/Zim both NULL (eigenvalues only) or both non-NULL, same pointer kind
 * On a pivot <= n*eps*max_i M_ii returns SKEW_ERR_NOT_DEFINITE with the 1-based pivot
 * index in *pivot_out.  Argument numbers: ctx 1, n 2, M 3, ldm 4,
 * nev 5, flags 6, lambda 7, Zre 8, Zim 9, ldz 10. */
int skew_eig_bse(skew_ctx ctx, int64_t n, double* M, int64_t ldm, int64_t nev, int flags,
                 double* lambda, double* Zre, double* Zim, int64_t ldz, int64_t* pivot_out);

/* One-step route (the paper's ELPA1-style GPU variant, PAPER.md:359-404,
 * Eqs. (2)-(5), Fig. 4): A reduced directly to tridiagonal form, one Householder
 * reflector per column, blocked by 64 columns (a skew matrix-vector product over the
 * trailing matrix per column, a skew rank-128 update per panel); then the same tridiagonal
 * solve and D assembly, and ONE back-transformation with the n-2 reflectors (merged compact
 * WY, the BT1 kernels).  Same result as skew_eig (eigenvalues to rounding; eigenvectors up
 * to phase).  DEVICE arrays only; Zre = Zim = NULL for eigenvalues only.  Workspace: size
 * with skew_workspace_size(ctx, n, nev, SKEW_WS_ONESTEP | SKEW_WS_VECTORS, ...).  Arguments
 * and status codes as skew_eig (host pointers: -i). */
int skew_eig_onestep(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev,
                     double* lambda, double* Zre, double* Zim, int64_t ldz);

/* Full BSE H_BS pipeline, step 1 (Eq. (10)):
 * M = [[Re(A+B), Im(A-B)], [-Im(A+B), Re(A-B)]] for H_BS = [[A, B], [-B-bar, -A-bar]]
 * (Eq. (9)), A = A^H and B = B^T.  A, B: device, n x n complex128 stored as interleaved
 * (re, im) doubles, column-major, leading dimensions lda, ldb >= n (in complex elements);
 * only read, caller-owned.  M: device, 2n x 2n real column-major, ldm >= 2n, fully
 * written.  Hermitian / symmetric structure is not checked (definiteness is: skew_eig_bse
 * reports SKEW_ERR_NOT_DEFINITE).  Asynchronous on the context stream.  Returns SKEW_OK
 * or -k for a bad k-th argument (host pointers are rejected). */
int skew_bse_build_M(skew_ctx ctx, int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                     double* M, int64_t ldm);

/* Full BSE H_BS pipeline, step 4 (PAPER.md:604-606 with Theorem 1):
 * x_k = Q J L z_k, Q = [[I, -iI], [I, iI]] / sqrt(2), J = [[0, I], [-I, 0]], so that
 * H_BS x_k = lambda_k x_k.  L: device, n2 x n2 lower-triangular Cholesky factor (as left
 * in M by skew_eig_bse; entries above the diagonal are ignored), ldl >= n2, n2 even.
 * Zre/Zim: device, n2 x nev (ldz >= n2), the skew_eig_bse eigenvectors.  X: device,
 * n2 x nev complex128 interleaved, ldx >= n2 (complex elements), fully written; each
 * column is normalised to unit 2-norm (phase free, reading R7).  Scratch
 * (16 n2 nev + 8 nev bytes) comes from the context workspace: size it with
 * skew_workspace_size(ctx, n2, nev, SKEW_WS_BSE_BACKTRANSFORM | ...).  Asynchronous on
 * the context stream.  Returns SKEW_OK, -k for a bad k-th argument or SKEW_ERR_WORKSPACE. */
int skew_bse_backtransform(skew_ctx ctx, int64_t n2, const double* L, int64_t ldl, int64_t nev,
                           const double* Zre, const double* Zim, int64_t ldz, double* X, int64_t ldx);

/* Per-stage device times (ms) of the last solve, measured with CUDA events on the
 * context stream: [0] full->band, [1] band->tridiagonal, [2] tridiagonal solve,
 * [3] back-transform 2 (bulge reflectors), [4] back-transform 1 (block
 * reflectors), [5] output, [6] BSE front-end.  `count` <= 7. */
int skew_stage_times(skew_ctx ctx, double* ms_out, int count);

/* Number of non-converged inverse-iteration vectors in the last solve. */
int64_t skew_last_nfail(skew_ctx ctx);
const char* skew_status_string(int status);
const char* skew_last_error(skew_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* SKEWEIG_H */
