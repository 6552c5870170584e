// onestep.cu -- SURVEY §8(f) NEXT-4: the ONE-STEP (ELPA1-style) reduction of the skew A
// directly to tridiagonal form on the GPU (Eqs. (2)-(5); the paper's GPU
// variant, Fig. 4), as the ablation of the two-step route: a BLAS-2 bound
// reduction (one skew matrix-vector product over the trailing matrix per column) against a
// cheaper back-transformation (one set of n-2 reflectors instead of the bulge reflectors plus
// the block reflectors).
//
// Blocked as LAPACK's dsytrd / dlatrd, re-derived for skew A (reading R4: v^T S v = 0, so no
// 1/2 tau^2 (v^T S v) v term): for each panel of b columns (c0 = j*b), column c = c0 + i:
//   (1) x = A[c+1:, c] + sum_{l<i} (V[:, l] W[c, l] - W[:, l] V[c, l])      (panel corrections)
//   (2) (v, tau, beta) = householder(x)  (dlarfg convention, reading R3); A[c+1, c] = beta
//   (3) w = tau (S v + V (W^T v) - W (V^T v)),  S = A[c+1:, c+1:] as at the panel start
//       (the skew matrix-vector product reads the lower triangle once, 128 x 128 tiles)
// and after the panel the trailing matrix takes the skew rank-2b update
//   A[c0+b:, c0+b:] += V W^T - W V^T      (strictly lower; the rank-2k GEMM of full->band).
// The reflectors go to the BT1 store (F2BLayout with r0(j) = j*b + 1) so that the
// back-transformation is BT1's merged compact-WY application with T from the group Gram.
#include "common.cuh"
#include "gemm_dmma.cuh"
#include "tma_gemm.cuh"
#include "internal.h"
#include <algorithm>

namespace sk {

static constexpr int kOsTile = 128;     // skew mat-vec tile (rows = cols)
static constexpr int kOsChunk = 256;    // rows per CTA of the column kernels

// panel arrays: PV = [V | W] (ldp x 2b), QW = [W | -V]; panel-local row pr (global row
// c0 + 1 + pr) is stored at index pr + 1 so that the rank-2b update's operand rows (pr >= b-1)
// start 16-byte aligned.
struct OsCol {
  double* A; int64_t lda; int64_t n;
  int64_t c0, c;        // panel start column, current column (c = c0 + i)
  int i;                // step inside the panel
  int b;
  double* PV; double* QW; int64_t ldp;
  double* npart;        // per-CTA partial sums of squares
  double* tau; double* sub;
  double* ypart;        // mat-vec tile partials (2 * kOsTile per tile)
  double* y;            // S v (mm)
  double* pq;           // per row-block partial W^T v, V^T v (2b each)
  int64_t nchunk;
};

// (1) corrected column x (written back into A) and partial ||x[1:]||^2 per CTA
__global__ void __launch_bounds__(256) os_col_prep_kernel(OsCol a) {
  __shared__ double cw[64], cv[64];     // W[c, l], V[c, l] (panel row pr = i - 1)
  __shared__ double red[8];
  const int i = a.i;
  const double* V = a.PV;
  const double* W = a.PV + a.ldp * a.b;
  if (threadIdx.x < i) {
    const int64_t ix = (i - 1) + 1;   // index of panel row i-1
    cw[threadIdx.x] = W[ix + threadIdx.x * a.ldp];
    cv[threadIdx.x] = V[ix + threadIdx.x * a.ldp];
  }
  __syncthreads();
  const int64_t m = a.n - a.c0 - 1;   // panel rows
  double s = 0.0;
  const int64_t p0 = (int64_t)blockIdx.x * kOsChunk;
  for (int64_t pr = i + p0 + threadIdx.x; pr < m && pr < i + p0 + kOsChunk; pr += blockDim.x) {
    double* xp = a.A + SK_IDX(a.c0 + 1 + pr, a.c, a.lda);
    double x = *xp;
    for (int l = 0; l < i; l++) x += V[pr + 1 + l * a.ldp] * cw[l] - W[pr + 1 + l * a.ldp] * cv[l];
    *xp = x;
    if (pr > i) s = fma(x, x, s);
    else a.npart[a.nchunk] = x;   // x0: read by every CTA of the next kernel (A[c+1, c] gets beta there)
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; w++) t += red[w];
    a.npart[blockIdx.x] = t;
  }
}

// (2) Householder (dlarfg convention, reading R3): every CTA forms beta / tau from the
// partials in a fixed order, scales its rows into V[:, i] and A[c+2:, c]
__global__ void __launch_bounds__(256) os_col_house_kernel(OsCol a) {
  const int i = a.i;
  double s = 0.0;
  for (int64_t k = 0; k < a.nchunk; k++) s += a.npart[k];
  const int64_t m = a.n - a.c0 - 1;
  const double x0 = a.npart[a.nchunk];
  double tau = 0.0, beta = x0, scal = 0.0;
  if (s != 0.0) {
    const double nrm = sqrt(x0 * x0 + s);
    beta = (x0 >= 0.0) ? -nrm : nrm;
    tau = (beta - x0) / beta;
    scal = 1.0 / (x0 - beta);
  }
  double* V = a.PV;
  const int64_t p0 = (int64_t)blockIdx.x * kOsChunk;
  for (int64_t pr = p0 + threadIdx.x; pr < m && pr < p0 + kOsChunk; pr += blockDim.x) {
    double v;
    if (pr < i) v = 0.0;
    else if (pr == i) v = 1.0;
    else {
      double* xp = a.A + SK_IDX(a.c0 + 1 + pr, a.c, a.lda);
      v = *xp * scal;
      *xp = v;   // reflector stored in place below the subdiagonal
    }
    V[pr + 1 + (int64_t)i * a.ldp] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.A[SK_IDX(a.c + 1, a.c, a.lda)] = beta;
    a.tau[a.c] = tau;
    a.sub[a.c] = beta;
  }
}

// (3a) skew mat-vec partials: S = A[o:, o:] (o = c + 1, order mm), v = V[i.., i].  Tile
// (bi, bj), bi >= bj, of kOsTile rows / columns: yrow = L_tile v[bj block] (rows of block bi),
// zcol = L_tile^T v[bi block] (rows of block bj); diagonal tiles use the strictly lower part.
// Warp w owns the 16 columns w*16 .. w*16+15 of the tile; lane l the rows l, l+32, l+64, l+96
// (coalesced 256-byte column segments).  Row sums stay in registers (summed over the warps in
// shared memory at the end), each column sum is one warp reduction.
__global__ void __launch_bounds__(256) os_skew_mv_kernel(OsCol a, int64_t mm) {
  constexpr int CW = kOsTile / 8;   // columns per warp
  __shared__ double vr[kOsTile], vc[kOsTile];
  __shared__ double ys[8][kOsTile];
  __shared__ double zs[kOsTile];
  int64_t bi, bj;
  tri_tile(blockIdx.x, 1, bi, bj);
  const int64_t o = a.c + 1;
  const double* v = a.PV + (int64_t)a.i * a.ldp + a.i + 1;   // v[q] = V[pr = i + q, i]
  const int64_t r0 = bi * kOsTile, q0 = bj * kOsTile;
  for (int t = threadIdx.x; t < kOsTile; t += blockDim.x) {
    vr[t] = (r0 + t < mm) ? v[r0 + t] : 0.0;
    vc[t] = (q0 + t < mm) ? v[q0 + t] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool diag = (bi == bj);
  double vrow[4], ysum[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int u = 0; u < 4; u++) vrow[u] = vr[lane + 32 * u];
  const int64_t rmax = mm - r0;   // rows of the tile inside S
  const double* Acol = a.A + SK_IDX(o + r0 + lane, o + q0, a.lda);
#pragma unroll 4
  for (int k = 0; k < CW; k++) {
    const int cl = warp * CW + k;
    const bool colok = q0 + cl < mm;
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int rl = lane + 32 * u;
      x[u] = (colok && rl < rmax && (!diag || rl > cl)) ? Acol[(size_t)cl * a.lda + 32 * u] : 0.0;
    }
    const double vcl = vc[cl];
    double z = 0.0;
#pragma unroll
    for (int u = 0; u < 4; u++) {
      ysum[u] = fma(x[u], vcl, ysum[u]);
      z = fma(x[u], vrow[u], z);
    }
    z = warp_sum(z);
    if (lane == 0) zs[cl] = z;
  }
#pragma unroll
  for (int u = 0; u < 4; u++) ys[warp][lane + 32 * u] = ysum[u];
  __syncthreads();
  double* out = a.ypart + (size_t)blockIdx.x * 2 * kOsTile;
  for (int t = threadIdx.x; t < kOsTile; t += blockDim.x) {
    double y = 0.0;
#pragma unroll
    for (int w = 0; w < 8; w++) y += ys[w][t];
    out[t] = y;
    out[kOsTile + t] = zs[t];
  }
}

// (3b) y = S v from the tile partials (fixed order) and the per-block partial dot products
// W^T v, V^T v over the previous i columns.  One CTA per 128-row block.
__global__ void __launch_bounds__(128) os_mv_reduce_kernel(OsCol a, int64_t mm) {
  __shared__ double red[4][2 * 64];
  const int64_t b = blockIdx.x, nbk = (mm + kOsTile - 1) / kOsTile;
  const int t = threadIdx.x;
  const int64_t q = b * kOsTile + t;
  double y = 0.0;
  for (int64_t j = 0; j <= b; j++) y += a.ypart[(size_t)(b * (b + 1) / 2 + j) * 2 * kOsTile + t];
  for (int64_t ii = b; ii < nbk; ii++) y -= a.ypart[(size_t)(ii * (ii + 1) / 2 + b) * 2 * kOsTile + kOsTile + t];
  if (q < mm) a.y[q] = y;
  // partial W^T v and V^T v over the rows of this block (panel rows pr = i + q)
  const int i = a.i;
  const double* V = a.PV;
  const double* W = a.PV + a.ldp * a.b;
  const double vq = (q < mm) ? V[(a.i + q) + 1 + (int64_t)i * a.ldp] : 0.0;
  const int warp = t >> 5, lane = t & 31;
  for (int l = 0; l < i; l++) {
    double pw = 0.0, pv = 0.0;
    if (q < mm) {
      pw = W[(i + q) + 1 + (int64_t)l * a.ldp] * vq;
      pv = V[(i + q) + 1 + (int64_t)l * a.ldp] * vq;
    }
    pw = warp_sum(pw);
    pv = warp_sum(pv);
    if (lane == 0) { red[warp][l] = pw; red[warp][64 + l] = pv; }
  }
  __syncthreads();
  for (int e = t; e < 2 * i; e += blockDim.x) {
    const int l = (e < i) ? e : 64 + (e - i);
    a.pq[(size_t)b * 128 + e] = ((red[0][l] + red[1][l]) + red[2][l]) + red[3][l];
  }
}

// (3c) w = tau (y + V p - W q) with p = W^T v, q = V^T v (block partials summed in a fixed
// order by every CTA); W[:, i] of the panel (zeros above row i) and the [W | -V] operand.
__global__ void __launch_bounds__(256) os_w_kernel(OsCol a, int64_t mm) {
  __shared__ double p[64], qv[64];
  const int i = a.i;
  const int64_t nbk = (mm + kOsTile - 1) / kOsTile;
  if (threadIdx.x < 2 * i) {
    double s = 0.0;
    for (int64_t b = 0; b < nbk; b++) s += a.pq[(size_t)b * 128 + threadIdx.x];
    if (threadIdx.x < i) p[threadIdx.x] = s;
    else qv[threadIdx.x - i] = s;
  }
  __syncthreads();
  const double tau = a.tau[a.c];
  const int64_t m = a.n - a.c0 - 1;
  double* V = a.PV;
  double* W = a.PV + a.ldp * a.b;
  const int64_t p0 = (int64_t)blockIdx.x * kOsChunk;
  for (int64_t pr = p0 + threadIdx.x; pr < m && pr < p0 + kOsChunk; pr += blockDim.x) {
    double w = 0.0;
    if (pr >= i && tau != 0.0) {
      double s = a.y[pr - i];
      for (int l = 0; l < i; l++) s += V[pr + 1 + l * a.ldp] * p[l] - W[pr + 1 + l * a.ldp] * qv[l];
      w = tau * s;
    }
    W[pr + 1 + (int64_t)i * a.ldp] = w;
    // [W | -V] for the panel's rank-2b update
    a.QW[pr + 1 + (int64_t)i * a.ldp] = w;
    a.QW[pr + 1 + (int64_t)(a.b + i) * a.ldp] = -V[pr + 1 + (int64_t)i * a.ldp];
  }
}

// forward dlarft of a merged group from its Gram matrix G = V^T V (K x K) and the tau's:
// T[l, l] = tau_l, T[0:l, l] = -tau_l T[0:l, 0:l] G[0:l, l]  (column by column, one CTA)
__global__ void __launch_bounds__(1024) os_larft_kernel(const double* G, const double* tau_all, int64_t nrefl, int K,
                                                        double* Tout) {
  const int64_t g = blockIdx.x;
  const double* Gg = G + (size_t)g * K * K;
  double* T = Tout + (size_t)g * K * K;
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) T[e] = 0.0;
  __syncthreads();
  for (int l = 0; l < K; l++) {
    const int64_t c = g * K + l;
    const double tl = (c < nrefl) ? tau_all[c] : 0.0;
    for (int r = threadIdx.x; r < l; r += blockDim.x) {
      double s = 0.0;
      for (int k = r; k < l; k++) s += T[r + (size_t)k * K] * Gg[k + (size_t)l * K];
      T[r + (size_t)l * K] = -tl * s;
    }
    if (threadIdx.x == 0) T[l + (size_t)l * K] = tl;
    __syncthreads();
  }
}

void onestep_reserve(Arena& ar, const F2BLayout& L, OneStepWork& w) {
  const int64_t n = std::max<int64_t>(L.n, 2), b = L.b;
  w.ldp = (n + 2) & ~int64_t(1);
  w.PV = ar.take<double>((size_t)w.ldp * 2 * b);
  w.QW = ar.take<double>((size_t)w.ldp * 2 * b);
  const int64_t nbk = (n + kOsTile - 1) / kOsTile;
  w.ypart = ar.take<double>((size_t)(nbk * (nbk + 1) / 2) * 2 * kOsTile);
  w.y = ar.take<double>((size_t)n);
  w.pq = ar.take<double>((size_t)nbk * 128);
  w.npart = ar.take<double>((size_t)(n + kOsChunk - 1) / kOsChunk + 1);
  w.tau = ar.take<double>((size_t)n);
  w.sub = ar.take<double>((size_t)n);
}

__global__ void os_alpha_kernel(const double* sub, const double* A, int64_t lda, int64_t n, double* alpha) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k + 1 < n; k += (int64_t)gridDim.x * blockDim.x)
    alpha[k] = -((k + 2 < n) ? sub[k] : A[SK_IDX(n - 1, n - 2, lda)]);   // alpha_k = -sub_k (reading R2)
}

// The whole one-step reduction.  A (n x n, lda, strictly lower) is overwritten with the
// reflectors; alpha (n-1) receives the Lemma-1 off-diagonals; when vstore != nullptr the
// panels' V go to the BT1 store (layout L, roff = 1) and tau to w.tau.
cudaError_t onestep_run(const F2BLayout& L, double* A, int64_t lda, double* vstore, OneStepWork& w, double* alpha,
                        int nsm, cudaStream_t st) {
  const int64_t n = L.n;
  const int b = L.b;
  cudaError_t e;
  if (n >= 2) {
    e = cudaMemsetAsync(w.tau, 0, sizeof(double) * n, st);
    if (e) return e;
  }
  for (int64_t j = 0; j < L.npanel; j++) {
    const int64_t c0 = j * b;
    const int nb = (int)std::min<int64_t>(b, n - 2 - c0);
    const int64_t m = n - c0 - 1;   // panel rows
    e = cudaMemset2DAsync(w.PV, w.ldp * 8, 0, (m + 1) * 8, 2 * b, st);
    if (e) return e;
    e = cudaMemset2DAsync(w.QW, w.ldp * 8, 0, (m + 1) * 8, 2 * b, st);
    if (e) return e;
    OsCol a;
    a.A = A; a.lda = lda; a.n = n; a.c0 = c0; a.b = b;
    a.PV = w.PV; a.QW = w.QW; a.ldp = w.ldp;
    a.npart = w.npart; a.tau = w.tau; a.sub = w.sub; a.ypart = w.ypart; a.y = w.y; a.pq = w.pq;
    a.nchunk = (m + kOsChunk - 1) / kOsChunk;
    for (int i = 0; i < nb; i++) {
      a.i = i;
      a.c = c0 + i;
      const int64_t mm = n - a.c - 1;   // order of S = A[c+1:, c+1:]
      {
        KScope ks(KC_OS_COL, st, 2);
        os_col_prep_kernel<<<(unsigned)a.nchunk, 256, 0, st>>>(a);
        os_col_house_kernel<<<(unsigned)a.nchunk, 256, 0, st>>>(a);
      }
      if (mm >= 1) {
        const int64_t nbk = (mm + kOsTile - 1) / kOsTile;
        KScope ks(KC_OS_MV, st, 2);
        os_skew_mv_kernel<<<(unsigned)(nbk * (nbk + 1) / 2), 256, 0, st>>>(a, mm);
        os_mv_reduce_kernel<<<(unsigned)nbk, 128, 0, st>>>(a, mm);
      }
      {
        KScope ks(KC_OS_COL, st);
        os_w_kernel<<<(unsigned)a.nchunk, 256, 0, st>>>(a, std::max<int64_t>(mm, 1));
      }
      e = cudaGetLastError();
      if (e) return e;
    }
    // trailing update A[c0+nb:, c0+nb:] += V W^T - W V^T (strictly lower), K = 2b (padding
    // columns are zero); operand rows start at panel row nb - 1 (index nb)
    const int64_t mt = n - c0 - nb;
    if (mt >= 2) {
      GemmArgs ga;
      ga.M = mt; ga.N = mt; ga.K = 2 * b;
      ga.A = w.PV + nb; ga.lda = w.ldp; ga.B = w.QW + nb; ga.ldb = w.ldp;
      ga.C = A + SK_IDX(c0 + nb, c0 + nb, lda); ga.ldc = lda; ga.alpha = 1.0; ga.beta = 1.0;
      KScope ks(KC_R2K, st);
      e = tma_disabled() ? cudaErrorNotSupported : tma_gemm<128, 64, 32, 3, false, true, true, true>(ga, nsm, st);
      if (e == cudaErrorNotSupported) e = gemm_dmma<64, 64, 16, 32, 32, 2, false, true, true>(ga, st);
      if (e) return e;
    }
    if (vstore) {   // V_j (panel rows, unit diagonal, zeros above) into the BT1 store
      const int64_t g = j / L.merge, pl = j % L.merge;
      double* Vj = vstore + L.goff[g] + pl * (int64_t)b + pl * (int64_t)b * L.gld[g];
      e = cudaMemcpy2DAsync(Vj, L.gld[g] * 8, w.PV + 1, w.ldp * 8, m * 8, b, cudaMemcpyDeviceToDevice, st);
      if (e) return e;
    }
  }
  if (n >= 2) {
    os_alpha_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(w.sub, A, lda, n, alpha);
    e = cudaGetLastError();
  }
  return e;
}

// Merged compact-WY T of every BT1 group of the one-step reflectors: Gram (bt1's kernel) then
// the forward dlarft recurrence from the Gram and the per-column tau (os_larft_kernel).
cudaError_t onestep_bt_prep(const F2BLayout& L, const double* vstore, const double* tau, BT1Work& w,
                            cudaStream_t st) {
  if (L.ngroup == 0) return cudaSuccess;
  const int K = L.merge * L.b;
  cudaError_t e = bt1_gram(L, vstore, w, st);
  if (e) return e;
  KScope ks(KC_BT1_PREP, st);
  os_larft_kernel<<<(unsigned)L.ngroup, 1024, 0, st>>>(w.G, tau, L.n - 2, K, w.T);
  return cudaGetLastError();
}

}  // namespace sk
