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
#include "tma_gemm.cuh"
#include "internal.h"
#include <algorithm>
#include <vector>

namespace sk {

// ---- merged-group preparation, all groups at once (before the BT1 loop) ----------------
// Gram G_g = V_g^T V_g (K x K) for every group: grid (K/64, K/64, ngroup) of DMMA tiles.
__global__ void __launch_bounds__(128) bt1_gram_kernel(const double* vstore, const int64_t* gmeta, int K,
                                                       double* G) {
  using T = GemmTile<64, 64, 16, 32, 32, 2, true, false>;
  extern __shared__ __align__(16) double smem[];
  const int64_t g = blockIdx.z;
  const int64_t goff = gmeta[3 * g], ld = gmeta[3 * g + 1], m = gmeta[3 * g + 2];
  const double* V = vstore + goff;
  GemmArgs ga;
  ga.M = K; ga.N = K; ga.K = m;
  ga.A = V; ga.lda = ld; ga.B = V; ga.ldb = ld;
  ga.vec = gemm_vec_ok(V, ld, V, ld) ? 1 : 0;
  double acc[T::FM][T::FN][2];
#pragma unroll
  for (int i = 0; i < T::FM; i++)
#pragma unroll
    for (int j = 0; j < T::FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  T::mainloop(ga, smem, m0, n0, 0, m, acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm0 = (warp % T::NWARP_M) * 32, wn0 = (warp / T::NWARP_M) * 32;
  const int gq = lane >> 2, t = lane & 3;
  double* out = G + (size_t)g * K * K;
#pragma unroll
  for (int i = 0; i < T::FM; i++)
#pragma unroll
    for (int j = 0; j < T::FN; j++)
#pragma unroll
      for (int h = 0; h < 2; h++)
        out[(m0 + wm0 + 8 * i + gq) + (n0 + wn0 + 8 * j + 2 * t + h) * (size_t)K] = acc[i][j][h];
}

// Merged T_g (K x K upper, K = merge*b) from the per-panel T_q (b x b, from the full->band
// reduction) and the Gram: block column q of the forward recurrence is
//   T[0:qb, q] = -T[0:qb, 0:qb] (V_{0:q}^T V_q) T_q,   T[q, q] = T_q
// (Schreiber-Van Loan).  One CTA per group; operands through L1/L2.
__global__ void __launch_bounds__(1024) bt1_tmerge_kernel(const double* G, const double* Tpanel, int64_t npanel,
                                                         int merge, int b, double* Tm, double* Y) {
  const int64_t g = blockIdx.x;
  const int K = merge * b;
  const double* Gg = G + (size_t)g * K * K;
  double* T = Tm + (size_t)g * K * K;
  double* Yg = Y + (size_t)g * K * b;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int r = e % K, c = e / K, qr = r / b, qc = c / b;
    const int64_t j = g * merge + qc;
    T[e] = (qr == qc && j < npanel) ? Tpanel[(size_t)j * b * b + (r % b) + (size_t)(c % b) * b] : 0.0;
  }
  __syncthreads();
  for (int q = 1; q < merge; q++) {
    const int64_t j = g * merge + q;
    if (j >= npanel) break;
    const int R = q * b;
    const double* Tq = Tpanel + (size_t)j * b * b;
    // Y = G[0:R, qb:(q+1)b] T_q   (R x b)
    for (int e = threadIdx.x; e < R * b; e += blockDim.x) {
      const int r = e % R, c = e / R;
      double s = 0.0;
      for (int l = 0; l <= c; l++) s += Gg[r + (size_t)(q * b + l) * K] * Tq[l + (size_t)c * b];
      Yg[e] = s;
    }
    __syncthreads();
    // T[0:R, qb+c] = -T[0:R, 0:R] Y[:, c]   (T upper: l >= r)
    for (int e = threadIdx.x; e < R * b; e += blockDim.x) {
      const int r = e % R, c = e / R;
      double s = 0.0;
      for (int l = r; l < R; l++) s += T[r + (size_t)l * K] * Yg[l + (size_t)c * R];
      T[r + (size_t)(q * b + c) * K] = -s;
    }
    __syncthreads();
  }
}

void bt1_reserve(Arena& ar, const F2BLayout& L, int64_t ncols, BT1Work& w) {
  const int64_t n = L.n;
  const int K = L.merge * L.b;
  const int64_t ng = std::max<int64_t>(L.ngroup, 1);
  int64_t ldn = (std::max<int64_t>(n, 2) + 1) & ~int64_t(1);
  w.G = ar.take<double>((size_t)ng * K * K);
  w.T = ar.take<double>((size_t)ng * K * K);
  w.Y = ar.take<double>((size_t)ng * K * L.b);
  w.U = ar.take<double>((size_t)ldn * K);
  w.Z = ar.take<double>((size_t)K * std::max<int64_t>(ncols, 1));
  w.gmeta = ar.take<int64_t>((size_t)3 * ng);
}

// per-group metadata (V-store offset, ld, rows) -> device; host-synchronous (call it before
// the stream has work queued, e.g. at the start of the solve)
cudaError_t bt1_upload_meta(const F2BLayout& L, BT1Work& w, cudaStream_t st) {
  if (L.ngroup == 0) return cudaSuccess;
  std::vector<int64_t> meta(3 * L.ngroup);
  for (int64_t g = 0; g < L.ngroup; g++) {
    meta[3 * g] = L.goff[g];
    meta[3 * g + 1] = L.gld[g];
    meta[3 * g + 2] = L.n - L.r0(g * L.merge);
  }
  cudaError_t e = cudaMemcpyAsync(w.gmeta, meta.data(), sizeof(int64_t) * meta.size(), cudaMemcpyHostToDevice, st);
  if (e) return e;
  return cudaStreamSynchronize(st);   // `meta` is a host temporary
}

// all groups: Gram and merged T (depends only on the full->band output: the solve driver
// runs it on an auxiliary stream, concurrently with the tridiagonal solve)
cudaError_t bt1_prep(const F2BLayout& L, const double* vstore, const double* Tpanel, BT1Work& w, cudaStream_t st) {
  if (L.ngroup == 0) return cudaSuccess;
  cudaError_t e = bt1_gram(L, vstore, w, st);
  if (e) return e;
  KScope ks(KC_BT1_PREP, st);
  bt1_tmerge_kernel<<<(unsigned)L.ngroup, 1024, 0, st>>>(w.G, Tpanel, L.npanel, L.merge, L.b, w.T, w.Y);
  return cudaGetLastError();
}

// Gram G_g = V_g^T V_g of every merged group (K x K, DMMA tiles)
cudaError_t bt1_gram(const F2BLayout& L, const double* vstore, BT1Work& w, cudaStream_t st) {
  if (L.ngroup == 0) return cudaSuccess;
  const int K = L.merge * L.b;
  KScope ks(KC_BT1_PREP, st);
  using TG = GemmTile<64, 64, 16, 32, 32, 2, true, false>;
  bt1_gram_kernel<<<dim3(K / 64, K / 64, (unsigned)L.ngroup), 128, TG::SMEM_BYTES, st>>>(vstore, w.gmeta, K, w.G);
  return cudaGetLastError();
}

cudaError_t bt1_run(const F2BLayout& L, const double* vstore, const double* tau_all, const double* Tpanel, double* X,
                    int64_t ldx, int64_t ncols, BT1Work& w, cudaStream_t st) {
  cudaError_t e = bt1_upload_meta(L, w, st);
  if (e) return e;
  e = bt1_prep(L, vstore, Tpanel, w, st);
  if (e) return e;
  return bt1_apply(L, vstore, tau_all, Tpanel, X, ldx, ncols, w, st);
}

cudaError_t bt1_apply(const F2BLayout& L, const double* vstore, const double* tau_all, const double* Tpanel, double* X,
                      int64_t ldx, int64_t ncols, BT1Work& w, cudaStream_t st) {
  (void)tau_all; (void)Tpanel;
  cudaError_t e;
  const int b = L.b;
  const int K = L.merge * b;
  if (L.ngroup == 0) return cudaSuccess;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  for (int64_t g = L.ngroup - 1; g >= 0; g--) {
    const int64_t r0 = L.r0(g * L.merge);
    const int64_t m = L.n - r0;
    const double* V = vstore + L.goff[g];
    const int64_t ldv = L.gld[g];
    const double* Tg = w.T + (size_t)g * K * K;
    // U = V T^T
    const int64_t ldu = (m + 1) & ~int64_t(1);
    {
      KScope ks(KC_BT1_PREP, st, 1);
      GemmArgs ga;
      ga.M = m; ga.N = K; ga.K = K;
      ga.A = V; ga.lda = ldv; ga.B = Tg; ga.ldb = K; ga.C = w.U; ga.ldc = ldu; ga.alpha = 1.0; ga.beta = 0.0;
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
      e = tma_disabled() ? cudaErrorNotSupported : tma_gemm<128, 64, 16, 6, true, false, false, false>(ga, nsm, st);
      if (e == cudaErrorNotSupported) e = gemm_dmma<64, 64, 16, 32, 32, 2, true, false, false>(ga, st);
      if (e) return e;
    }
    // X[r0:, :] -= V Z
    {
      KScope ks(KC_BT1_UPD, st);
      GemmArgs ga;
      ga.M = m; ga.N = ncols; ga.K = K;
      ga.A = V; ga.lda = ldv; ga.B = w.Z; ga.ldb = K; ga.C = Xr; ga.ldc = ldx; ga.alpha = -1.0; ga.beta = 1.0;
      e = tma_disabled() ? cudaErrorNotSupported : tma_gemm<128, 64, 16, 4, false, false, true, false>(ga, nsm, st);
      if (e == cudaErrorNotSupported) e = gemm_dmma<64, 64, 16, 32, 32, 2, false, false, false>(ga, st);
      if (e) return e;
    }
  }
  return cudaGetLastError();
}

// Output split: Zre = X[:, :nev], Zim = X[:, nev:] into the caller's ldz layout.
__global__ void split_output_kernel(const double* X, int64_t ldx, int64_t n, int64_t nev, double* Zre, double* Zim,
                                    int64_t ldz) {
  for (int64_t c = blockIdx.y; c < nev; c += gridDim.y)   // grid.y is capped at 65535
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      Zre[SK_IDX(i, c, ldz)] = X[SK_IDX(i, c, ldx)];
      Zim[SK_IDX(i, c, ldz)] = X[SK_IDX(i, nev + c, ldx)];
    }
}

cudaError_t split_output(const double* X, int64_t ldx, int64_t n, int64_t nev, double* Zre, double* Zim, int64_t ldz,
                         cudaStream_t st) {
  if (nev <= 0) return cudaSuccess;
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(nev, 65535));
  KScope ks(KC_OUT, st);
  split_output_kernel<<<grid, 256, 0, st>>>(X, ldx, n, nev, Zre, Zim, ldz);
  return cudaGetLastError();
}

}  // namespace sk
