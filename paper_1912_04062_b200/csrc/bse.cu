// bse.cu -- BSE-form front end (SURVEY §8(b) entry point skew_eig_bse):
//   step 2: M = L L^T (blocked right-looking Cholesky: diagonal-block factor, panel
//           TRSM, DMMA SYRK trailing update on the lower triangle);
//   step 3: W = L^T J L, J = [[0, I], [-I, 0]]:
//           W11 = S - S^T with S = L11^T L21,  W21 = -L22^T L11,  W22 = 0
//           (block expansion of L^T (J L)).
// NotDefinite when a pivot <= n*eps*max_i M_ii (reading R18).
#include "common.cuh"
#include "gemm_dmma.cuh"
#include "tma_gemm.cuh"
#include "internal.h"
#include <algorithm>
#include <cfloat>

namespace sk {

static constexpr int kCholNB = 64;

__global__ void diag_max_kernel(const double* M, int64_t ldm, int64_t n, double* out) {
  __shared__ double red[256];
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, M[SK_IDX(i, i, ldm)]);
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

// unblocked Cholesky of the nb x nb diagonal block at (j0, j0); status[0] = first failing pivot (1-based)
__global__ void chol_diag_kernel(double* M, int64_t ldm, int64_t j0, int nb, int64_t n, const double* dmax,
                                 int64_t* status) {
  __shared__ double L[kCholNB * kCholNB];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    L[e] = (i >= j) ? M[SK_IDX(j0 + i, j0 + j, ldm)] : 0.0;
  }
  __syncthreads();
  if (status[0] != 0) return;
  const double tol = (double)n * DBL_EPSILON * dmax[0];
  for (int j = 0; j < nb; j++) {
    if (threadIdx.x == 0) {
      double d = L[j + j * nb];
      if (!(d > tol)) { bad = 1; status[0] = j0 + j + 1; }
      else L[j + j * nb] = sqrt(d);
    }
    __syncthreads();
    if (bad) return;
    double djj = L[j + j * nb];
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) L[i + j * nb] /= djj;
    __syncthreads();
    for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
      int i = e % nb, k = e / nb;
      if (k > j && i >= k) L[i + k * nb] -= L[i + j * nb] * L[k + j * nb];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    int i = e % nb, j = e / nb;
    M[SK_IDX(j0 + i, j0 + j, ldm)] = (i >= j) ? L[e] : 0.0;
  }
}

// panel TRSM: rows below the block: L21 = M21 L11^{-T}, one thread per row
__global__ void chol_trsm_kernel(double* M, int64_t ldm, int64_t j0, int nb, int64_t n, const int64_t* status) {
  __shared__ double L[kCholNB * kCholNB];
  if (status[0] != 0) return;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) L[e] = M[SK_IDX(j0 + e % nb, j0 + e / nb, ldm)];
  __syncthreads();
  int64_t i = j0 + nb + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[kCholNB];
  for (int j = 0; j < nb; j++) x[j] = M[SK_IDX(i, j0 + j, ldm)];
  for (int j = 0; j < nb; j++) {
    double s = x[j];
    for (int k = 0; k < j; k++) s -= x[k] * L[j + k * nb];
    x[j] = s / L[j + j * nb];
  }
  for (int j = 0; j < nb; j++) M[SK_IDX(i, j0 + j, ldm)] = x[j];
}

__global__ void zero_upper_kernel(double* M, int64_t ldm, int64_t n) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)   // grid.y is capped at 65535
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < j; i += (int64_t)gridDim.x * blockDim.x)
      M[SK_IDX(i, j, ldm)] = 0.0;
}

// W11 strictly lower = S - S^T ; W22 strictly lower = 0 ; (W21 written by GEMM)
__global__ void w11_kernel(const double* S, int64_t lds, int64_t m, double* W, int64_t ldw) {
  for (int64_t j = blockIdx.y; j < m; j += gridDim.y) {   // grid.y is capped at 65535
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
      if (i > j) {
        W[SK_IDX(i, j, ldw)] = S[SK_IDX(i, j, lds)] - S[SK_IDX(j, i, lds)];
        W[SK_IDX(m + i, m + j, ldw)] = 0.0;
      }
    }
  }
}

// M (n x n, ldm) -> L in place; W (n x n, ldw) strictly lower; S scratch (m x m, lds).
// status_d: device int64 (0 ok, else 1-based pivot).
cudaError_t bse_front(double* M, int64_t ldm, int64_t n, double* W, int64_t ldw, double* S, int64_t lds,
                      double* scratch, int64_t* status_d, cudaStream_t st) {
  cudaError_t e;
  const int64_t nbl = (n + kCholNB - 1) / kCholNB;
  KScope ks(KC_BSE, st, (int)(1 + nbl + 2 * (nbl - 1) + 4));
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // the TMA-fed persistent GEMM where the strides allow it (16-byte rows), else the cp.async one
  auto gemm_tn = [&](const GemmArgs& ga) -> cudaError_t {   // C = alpha A^T B
    cudaError_t r = tma_disabled() ? cudaErrorNotSupported : tma_gemm<128, 64, 16, 6, true, false, false, false>(ga, nsm, st);
    if (r == cudaErrorNotSupported) r = gemm_dmma<64, 64, 16, 32, 32, 2, true, false, false>(ga, st);
    return r;
  };
  cudaMemsetAsync(status_d, 0, sizeof(int64_t), st);
  diag_max_kernel<<<1, 256, 0, st>>>(M, ldm, n, scratch);
  for (int64_t j0 = 0; j0 < n; j0 += kCholNB) {
    int nb = (int)std::min<int64_t>(kCholNB, n - j0);
    chol_diag_kernel<<<1, 256, 0, st>>>(M, ldm, j0, nb, n, scratch, status_d);
    int64_t rest = n - j0 - nb;
    if (rest > 0) {
      chol_trsm_kernel<<<(unsigned)((rest + 127) / 128), 128, 0, st>>>(M, ldm, j0, nb, n, status_d);
      GemmArgs ga;
      ga.M = rest; ga.N = rest; ga.K = nb;
      const double* L21 = M + SK_IDX(j0 + nb, j0, ldm);
      ga.A = L21; ga.lda = ldm; ga.B = L21; ga.ldb = ldm;
      ga.C = M + SK_IDX(j0 + nb, j0 + nb, ldm); ga.ldc = ldm; ga.alpha = -1.0; ga.beta = 1.0; ga.tri_off = 0;
      e = tma_disabled() ? cudaErrorNotSupported : tma_gemm<128, 64, 32, 3, false, true, true, true>(ga, nsm, st);
      if (e == cudaErrorNotSupported) e = gemm_dmma<64, 64, 16, 32, 32, 2, false, true, true>(ga, st);
      if (e) return e;
    }
  }
  {
    dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(n, 65535));
    zero_upper_kernel<<<grid, 256, 0, st>>>(M, ldm, n);
  }
  const int64_t m = n / 2;
  // S = L11^T L21
  {
    GemmArgs ga;
    ga.M = m; ga.N = m; ga.K = m;
    ga.A = M; ga.lda = ldm; ga.B = M + m; ga.ldb = ldm; ga.C = S; ga.ldc = lds; ga.alpha = 1.0; ga.beta = 0.0;
    e = gemm_tn(ga);
    if (e) return e;
  }
  // W21 = -L22^T L11
  {
    GemmArgs ga;
    ga.M = m; ga.N = m; ga.K = m;
    ga.A = M + SK_IDX(m, m, ldm); ga.lda = ldm; ga.B = M; ga.ldb = ldm; ga.C = W + m; ga.ldc = ldw;
    ga.alpha = -1.0; ga.beta = 0.0;
    e = gemm_tn(ga);
    if (e) return e;
  }
  {
    dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 64), (unsigned)std::min<int64_t>(std::max<int64_t>(m, 1), 65535));
    w11_kernel<<<grid, 256, 0, st>>>(S, lds, m, W, ldw);
  }
  return cudaGetLastError();
}


// ------------------------------------------------------------------------------------
// Full H_BS pipeline stages.
// Step 1, Eq. (10): M = [[Re(A+B), Im(A-B)], [-Im(A+B), Re(A-B)]].
// A, B: n x n complex, interleaved (re, im) doubles, column-major; one thread per (i, j),
// consecutive threads down a column -> coalesced 16-byte loads and 8-byte stores.
__global__ void bse_build_M_kernel(const double2* __restrict__ A, int64_t lda, const double2* __restrict__ B,
                                   int64_t ldb, int64_t n, double* __restrict__ M, int64_t ldm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {   // grid.y is capped at 65535
    const double2 a = A[SK_IDX(i, j, lda)], b = B[SK_IDX(i, j, ldb)];
    M[SK_IDX(i, j, ldm)] = a.x + b.x;            // Re(A+B)
    M[SK_IDX(i, n + j, ldm)] = a.y - b.y;        // Im(A-B)
    M[SK_IDX(n + i, j, ldm)] = -(a.y + b.y);     // -Im(A+B)
    M[SK_IDX(n + i, n + j, ldm)] = a.x - b.x;    // Re(A-B)
  }
}

cudaError_t bse_build_M(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t n, double* M, int64_t ldm,
                        cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)std::min<int64_t>(n, 65535));
  bse_build_M_kernel<<<grid, 256, 0, st>>>((const double2*)A, lda, (const double2*)B, ldb, n, M, ldm);
  return cudaGetLastError();
}

// Step 4, part 1: Y = L Z for lower-triangular L (n2 x n2) and the real
// and imaginary parts of Z (grid.z = 0 / 1).  64 x 64 output tile per CTA, 256 threads x
// (4 x 4) FP64 register tile, 16-deep K slabs staged in shared memory; the K loop stops at
// the tile's last row (L(i, k) = 0 for k > i) and the strictly upper part of the diagonal
// slab is masked on load.
static constexpr int kTM = 64, kTK = 16;
__global__ void __launch_bounds__(256) bse_trmm_kernel(const double* __restrict__ L, int64_t ldl, int64_t n2,
                                                       const double* __restrict__ Zre, const double* __restrict__ Zim,
                                                       int64_t ldz, int64_t nev, double* __restrict__ Yre,
                                                       double* __restrict__ Yim, int64_t ldy) {
  __shared__ double Ls[kTK][kTM + 1];
  __shared__ double Zs[kTK][kTM + 1];
  const double* Z = blockIdx.z ? Zim : Zre;
  double* Y = blockIdx.z ? Yim : Yre;
  const int64_t i0 = (int64_t)blockIdx.x * kTM, j0 = (int64_t)blockIdx.y * kTM;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4] = {};
  const int64_t kend = min(n2, i0 + kTM);
  for (int64_t k0 = 0; k0 < kend; k0 += kTK) {
    for (int e = threadIdx.x; e < kTK * kTM; e += 256) {
      const int r = e % kTM, kk = e / kTM;   // L tile: rows i0 + r, column k0 + kk (coalesced down r)
      const int64_t gi = i0 + r, gk = k0 + kk;
      Ls[kk][r] = (gi < n2 && gk < n2 && gk <= gi) ? L[SK_IDX(gi, gk, ldl)] : 0.0;
      const int kz = e % kTK, c = e / kTK;   // Z tile: rows k0 + kz, column j0 + c
      const int64_t zk = k0 + kz, zc = j0 + c;
      Zs[kz][c] = (zk < n2 && zc < nev) ? Z[SK_IDX(zk, zc, ldz)] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; kk++) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; u++) { a[u] = Ls[kk][tx + 16 * u]; b[u] = Zs[kk][ty + 16 * u]; }
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int v = 0; v < 4; v++) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; u++)
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int64_t gi = i0 + tx + 16 * u, gj = j0 + ty + 16 * v;
      if (gi < n2 && gj < nev) Y[SK_IDX(gi, gj, ldy)] = acc[u][v];
    }
}

// Squared 2-norms of the columns of y = [Yre | Yim] (n2 rows): one CTA per column
// (grid-stride), fixed-order block reduction (deterministic).
__global__ void __launch_bounds__(256) bse_colnorm2_kernel(const double* __restrict__ Yre,
                                                           const double* __restrict__ Yim, int64_t ldy, int64_t n2,
                                                           int64_t nev, double* __restrict__ nrm2) {
  __shared__ double red[8];
  for (int64_t j = blockIdx.x; j < nev; j += gridDim.x) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n2; i += blockDim.x) {
      const double a = Yre[SK_IDX(i, j, ldy)], b = Yim[SK_IDX(i, j, ldy)];
      s = fma(a, a, fma(b, b, s));
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; w++) t += red[w];
      nrm2[j] = t;
    }
    __syncthreads();
  }
}

// Step 4, part 2: x = Q J y / ||y|| with J = [[0, I], [-I, 0]] and Q = [[I, -iI], [I, iI]] /
// sqrt(2) (Theorem 1):  x_top = (y2 + i y1) / sqrt 2,  x_bot = (y2 - i y1) /
// sqrt 2 for y = [y1; y2] (n rows each), written interleaved complex.  ||Q J y|| = ||y||
// (Q, J unitary), so dividing by ||y|| gives unit 2-norm x (reading R22).
__global__ void bse_qj_kernel(const double* __restrict__ Yre, const double* __restrict__ Yim, int64_t ldy, int64_t n,
                              int64_t nev, const double* __restrict__ nrm2, double2* __restrict__ X, int64_t ldx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t j = blockIdx.y; j < nev; j += gridDim.y) {   // grid.y is capped at 65535
    const double nn = nrm2[j];
    const double s = 0.70710678118654752440 / (nn > 0.0 ? sqrt(nn) : 1.0);
    const double y1r = Yre[SK_IDX(i, j, ldy)], y1i = Yim[SK_IDX(i, j, ldy)];
    const double y2r = Yre[SK_IDX(n + i, j, ldy)], y2i = Yim[SK_IDX(n + i, j, ldy)];
    X[SK_IDX(i, j, ldx)] = make_double2(s * (y2r - y1i), s * (y2i + y1r));
    X[SK_IDX(n + i, j, ldx)] = make_double2(s * (y2r + y1i), s * (y2i - y1r));
  }
}

// y = J w for w = [w1; w2] (n rows each), real and imaginary planes: y1 = w2, y2 = -w1
// (skew_eig_bse with SKEW_BSE_HAMILTONIAN_Y: w = L z, y = J L z, H y = -i lambda y for
// H = -J M).
__global__ void bse_j_kernel(const double* __restrict__ Wre, const double* __restrict__ Wim, int64_t ldw, int64_t n,
                             int64_t nev, double* __restrict__ Yre, double* __restrict__ Yim, int64_t ldy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int64_t j = blockIdx.y; j < nev; j += gridDim.y) {
    const double a = Wre[SK_IDX(i, j, ldw)], b = Wim[SK_IDX(i, j, ldw)];
    const double c = Wre[SK_IDX(n + i, j, ldw)], d = Wim[SK_IDX(n + i, j, ldw)];
    Yre[SK_IDX(i, j, ldy)] = c;
    Yim[SK_IDX(i, j, ldy)] = d;
    Yre[SK_IDX(n + i, j, ldy)] = -a;
    Yim[SK_IDX(n + i, j, ldy)] = -b;
  }
}

cudaError_t bse_lz(const double* L, int64_t ldl, int64_t n2, const double* Zre, const double* Zim, int64_t ldz,
                   int64_t nev, double* Yre, double* Yim, int64_t ldy, cudaStream_t st) {
  if (n2 <= 0 || nev <= 0) return cudaSuccess;
  dim3 g1((unsigned)((n2 + kTM - 1) / kTM), (unsigned)((nev + kTM - 1) / kTM), 2);
  bse_trmm_kernel<<<g1, 256, 0, st>>>(L, ldl, n2, Zre, Zim, ldz, nev, Yre, Yim, ldy);
  return cudaGetLastError();
}

cudaError_t bse_apply_J(const double* Wre, const double* Wim, int64_t ldw, int64_t n2, int64_t nev, double* Yre,
                        double* Yim, int64_t ldy, cudaStream_t st) {
  if (n2 <= 0 || nev <= 0) return cudaSuccess;
  const int64_t n = n2 / 2;
  dim3 g((unsigned)((n + 255) / 256), (unsigned)std::min<int64_t>(nev, 65535));
  bse_j_kernel<<<g, 256, 0, st>>>(Wre, Wim, ldw, n, nev, Yre, Yim, ldy);
  return cudaGetLastError();
}

cudaError_t bse_backtransform(const double* L, int64_t ldl, int64_t n2, const double* Zre, const double* Zim,
                              int64_t ldz, int64_t nev, double* Yre, double* Yim, int64_t ldy, double* nrm2,
                              double* X, int64_t ldx, cudaStream_t st) {
  if (n2 <= 0 || nev <= 0) return cudaSuccess;
  cudaError_t e = bse_lz(L, ldl, n2, Zre, Zim, ldz, nev, Yre, Yim, ldy, st);
  if (e != cudaSuccess) return e;
  bse_colnorm2_kernel<<<(unsigned)std::min<int64_t>(nev, 4096), 256, 0, st>>>(Yre, Yim, ldy, n2, nev, nrm2);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n = n2 / 2;
  dim3 g2((unsigned)((n + 255) / 256), (unsigned)std::min<int64_t>(nev, 65535));
  bse_qj_kernel<<<g2, 256, 0, st>>>(Yre, Yim, ldy, n, nev, nrm2, (double2*)X, ldx);
  return cudaGetLastError();
}

// Non-finite scan of a column-major n x n input: entries i > j (skew A, strictly lower) or
// i >= j (symmetric M, lower with diagonal).  flag: device int, set to 1 on any NaN / Inf.
__global__ void nonfinite_lower_kernel(const double* __restrict__ A, int64_t lda, int64_t n, int diag,
                                       int* __restrict__ flag) {
  int bad = 0;
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
    const int64_t i0 = j + (diag ? 0 : 1);
    for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      bad |= !isfinite(A[SK_IDX(i, j, lda)]);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

cudaError_t nonfinite_lower(const double* A, int64_t lda, int64_t n, bool diag, int* flag_d, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(flag_d, 0, sizeof(int), st);
  if (e != cudaSuccess || n <= 0) return e;
  dim3 g((unsigned)std::min<int64_t>((n + 255) / 256, 4), (unsigned)std::min<int64_t>(n, 65535));
  nonfinite_lower_kernel<<<g, 256, 0, st>>>(A, lda, n, diag ? 1 : 0, flag_d);
  return cudaGetLastError();
}

}  // namespace sk
