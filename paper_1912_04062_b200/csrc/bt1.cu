// bt1.cu -- BT1: back-transformation with the full->band block reflectors (SURVEY
// §8(a) a10, hot path), PAPER.md:215-218 (step 3(b), Q = Q_band Q~) and Algorithm 1
// step 4, applied to the real n x 2nev matrix X = [Re | Im]
// (Re and Im transformed independently in real arithmetic).
//
// Q_band = Q_0 Q_1 ... Q_{np-1},  Q_j = I - V_j T_j V_j^T.  `merge` consecutive panels
// form one block reflector I - V_g T_g V_g^T (V_g = [V_j ... V_j+merge-1], T_g from the
// Gram matrix V_g^T V_g and the tau's by forward dlarft), applied last -> first:
//     U_g = V_g T_g^T      (n_g x K)      [once per group]
//     Z   = U_g^T X        (K x 2nev)     DMMA GEMM, reduction over n_g rows
//     X  -= V_g Z          (n_g x 2nev)   DMMA GEMM
#include "common.cuh"
#include "gemm_dmma.cuh"
#include "internal.h"
#include <algorithm>

namespace sk {

// T_g (K x K upper) from the Gram G (K x K, full) and tau (K): thread per row
__global__ void bt1_tbuild_kernel(const double* G, int K, const double* tau, double* T) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= K) return;
  // row r of T: T[r][r] = tau_r; T[r][c] = -tau_c * sum_{l=r}^{c-1} T[r][l] G[l][c]
  // (stored directly into T to avoid a large local array)
  for (int c = 0; c < K; c++) T[r + (size_t)c * K] = 0.0;
  T[r + (size_t)r * K] = tau[r];
  for (int c = r + 1; c < K; c++) {
    double s = 0.0;
    for (int l = r; l < c; l++) s += T[r + (size_t)l * K] * G[l + (size_t)c * K];
    T[r + (size_t)c * K] = -tau[c] * s;
  }
}


void bt1_reserve(Arena& ar, int64_t n, int64_t ncols, int K, BT1Work& w) {
  int64_t ldn = (std::max<int64_t>(n, 2) + 1) & ~int64_t(1);
  w.G = ar.take<double>((size_t)K * K);
  w.T = ar.take<double>((size_t)K * K);
  w.U = ar.take<double>((size_t)ldn * K);
  w.Z = ar.take<double>((size_t)K * std::max<int64_t>(ncols, 1));
}

cudaError_t bt1_run(const F2BLayout& L, const double* vstore, const double* tau_all, double* X, int64_t ldx,
                    int64_t ncols, BT1Work& w, cudaStream_t st) {
  cudaError_t e;
  const int b = L.b;
  for (int64_t g = L.ngroup - 1; g >= 0; g--) {
    const int64_t j0 = g * L.merge;
    const int64_t j1 = std::min<int64_t>(L.npanel, j0 + L.merge);
    const int K = (int)((j1 - j0) * b);
    const int64_t r0 = L.r0(j0);
    const int64_t m = L.n - r0;
    const double* V = vstore + L.goff[g];
    const int64_t ldv = L.gld[g];
    // Gram G = V^T V
    {
      KScope ks(KC_BT1_PREP, st, 3);
      GemmArgs ga;
      ga.M = K; ga.N = K; ga.K = m;
      ga.A = V; ga.lda = ldv; ga.B = V; ga.ldb = ldv; ga.C = w.G; ga.ldc = K; ga.alpha = 1.0; ga.beta = 0.0;
      e = gemm_dmma<64, 64, 16, 32, 16, 4, true, false, false>(ga, st);
      if (e) return e;
      bt1_tbuild_kernel<<<(K + 63) / 64, 64, 0, st>>>(w.G, K, tau_all + j0 * b, w.T);
    }
    // U = V T^T
    const int64_t ldu = (m + 1) & ~int64_t(1);
    {
      KScope ks(KC_BT1_PREP, st, 0);
      GemmArgs ga;
      ga.M = m; ga.N = K; ga.K = K;
      ga.A = V; ga.lda = ldv; ga.B = w.T; ga.ldb = K; ga.C = w.U; ga.ldc = ldu; ga.alpha = 1.0; ga.beta = 0.0;
      e = gemm_dmma<64, 64, 16, 32, 32, 2, false, true, false>(ga, st);
      if (e) return e;
    }
    // Z = U^T X[r0:, :]
    double* Xr = X + r0;
    {
      KScope ks(KC_BT1_Z, st);
      GemmArgs ga;
      ga.M = K; ga.N = ncols; ga.K = m;
      ga.A = w.U; ga.lda = ldu; ga.B = Xr; ga.ldb = ldx; ga.C = w.Z; ga.ldc = K; ga.alpha = 1.0; ga.beta = 0.0;
      e = gemm_dmma<64, 64, 16, 32, 32, 2, true, false, false>(ga, st);
      if (e) return e;
    }
    // X[r0:, :] -= V Z
    {
      KScope ks(KC_BT1_UPD, st);
      GemmArgs ga;
      ga.M = m; ga.N = ncols; ga.K = K;
      ga.A = V; ga.lda = ldv; ga.B = w.Z; ga.ldb = K; ga.C = Xr; ga.ldc = ldx; ga.alpha = -1.0; ga.beta = 1.0;
      e = gemm_dmma<64, 64, 16, 32, 32, 2, false, false, false>(ga, st);
      if (e) return e;
    }
  }
  return cudaGetLastError();
}

// Output split: Zre = X[:, :nev], Zim = X[:, nev:] into the caller's ldz layout.
__global__ void split_output_kernel(const double* X, int64_t ldx, int64_t n, int64_t nev, double* Zre, double* Zim,
                                    int64_t ldz) {
  int64_t c = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    Zre[SK_IDX(i, c, ldz)] = X[SK_IDX(i, c, ldx)];
    Zim[SK_IDX(i, c, ldz)] = X[SK_IDX(i, nev + c, ldx)];
  }
}

cudaError_t split_output(const double* X, int64_t ldx, int64_t n, int64_t nev, double* Zre, double* Zim, int64_t ldz,
                         cudaStream_t st) {
  if (nev <= 0) return cudaSuccess;
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)nev);
  KScope ks(KC_OUT, st);
  split_output_kernel<<<grid, 256, 0, st>>>(X, ldx, n, nev, Zre, Zim, ldz);
  return cudaGetLastError();
}

}  // namespace sk
