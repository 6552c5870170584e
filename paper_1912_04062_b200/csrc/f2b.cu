// f2b.cu -- full-to-band reduction of a dense real skew-symmetric matrix (hot path,
// SURVEY §8(a) rows a1-a5), §2.3.2 (lines 407-442):
//
//   for each panel j (columns c0 = j*b .. c0+b-1, rows r0 = c0+b .. n-1):
//     a1  panel QR  P_j = A[r0:, c0:c0+b] = Q_j [R_j; 0]     (Householder, dlarfg convention)
//     a2  T_j       Q_j = H_1 ... H_b = I - V T V^T            (Eq. (6))
//     a3  X = S U   S = A[r0:, r0:] skew (lower triangle only), U = V T   (skew-SYMM)
//     a4  W = X - 1/2 V (T^T V^T X)                             (Eq. (7), U1 = -U2 = W)
//     a5  S <- S + V W^T - W V^T = S + [V W][W -V]^T (strictly lower triangle only; Eq. (8))
//
// The trailing update touches only the strictly lower triangle (the diagonal of a
// skew matrix is never written and stays 0); the upper triangle is never read.
#include "common.cuh"
#include "gemm_dmma.cuh"
#include "internal.h"
#include <cooperative_groups.h>
#include <algorithm>

namespace cg = cooperative_groups;

namespace sk {

void F2BLayout::init(int64_t n_, int b_, int merge_) {
  n = n_; b = b_; merge = merge_;
  npanel = (n >= 2 + b) ? (n - 2) / b : 0;
  ngroup = (npanel + merge - 1) / merge;
  goff.assign(ngroup, 0);
  gld.assign(ngroup, 0);
  int64_t off = 0;
  for (int64_t g = 0; g < ngroup; g++) {
    int64_t rows = n - r0(g * merge);
    int64_t ld = (rows + 1) & ~int64_t(1);
    gld[g] = ld;
    goff[g] = off;
    off += ld * (int64_t)merge * b;
  }
  vstore_elems = off;
}

// ------------------------------------------------------------------------------------
// a1 + a2: cooperative panel QR.  Each CTA owns a contiguous row range of the panel,
// kept in shared memory when it fits; one grid-wide barrier per column: the
// partial sums for column k+1 (||x[1:]||^2 and x[1:]^T P[:, c]) are produced in the
// same pass that applies reflector k, and reduced in a fixed CTA order (bitwise
// deterministic; every CTA derives identical beta/tau).
struct PanelArgs {
  double* A; int64_t lda;      // panel P = A (m x kb), column-major, in place
  int64_t m; int kb;
  double* V; int64_t ldv;      // V out (m x kb, unit lower trapezoidal, explicit 0/1)
  double* tau;                 // kb
  double* T; int ldt;          // kb x kb upper triangular
  double* part;                // [2][G][kb+1]
  double* rowk;                // [2][kb]
  double* gram;                // [G][kb*kb] partial Gram, then [kb*kb] final
  int64_t R;                   // rows per CTA
  int smem_rows;               // R if the CTA rows live in shared memory, else 0
};

template <bool SMEM>
__global__ void __launch_bounds__(256) panel_qr_kernel(PanelArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double sm[];
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kb = a.kb;
  const int64_t rb = (int64_t)cta * a.R;
  const int64_t re = smin<int64_t>(a.m, rb + a.R);
  const int nr = (int)smax<int64_t>(0, re - rb);
  const int64_t R = a.R;
  double* Ps = sm;                                   // [kb][R] when SMEM
  double* red = sm + (SMEM ? (size_t)kb * R : 0);    // [8][kb+1] warp partials
  double* dsum = red + 8 * (kb + 1);                 // [kb+1]
  double* wv = dsum + (kb + 1);                      // [kb]
  double* scal_s = wv + kb;                          // [4]: beta, tau, scal
  auto P = [&](int li, int c) -> double& {
    if (SMEM) return Ps[(size_t)c * R + li];
    return a.A[SK_IDX(rb + li, c, a.lda)];
  };
  if (SMEM) {
    for (int64_t e = tid; e < (int64_t)nr * kb; e += blockDim.x) {
      int c = (int)(e / nr), li = (int)(e % nr);
      Ps[(size_t)c * R + li] = a.A[SK_IDX(rb + li, c, a.lda)];
    }
    __syncthreads();
  }
  // partials for column k: rows gi > k: norm = sum x^2 (slot k), dots with columns c > k
  auto partials = [&](int k) {
    const int buf = k & 1;
    for (int c = k + warp; c < kb; c += 8) {
      double s = 0.0;
      for (int li = lane; li < nr; li += 32) {
        int64_t gi = rb + li;
        if (gi > k) s += P(li, k) * P(li, c);
      }
      s = warp_sum(s);
      if (lane == 0) a.part[((size_t)buf * G + cta) * (kb + 1) + c] = s;
    }
    // owner of row k publishes row k (c >= k)
    if (k >= rb && k < re) {
      for (int c = k + tid; c < kb; c += blockDim.x) a.rowk[buf * kb + c] = P((int)(k - rb), c);
    }
  };
  partials(0);
  __threadfence();
  grid.sync();
  const int kmax = (int)smin<int64_t>(kb, a.m);
  for (int k = 0; k < kmax; k++) {
    const int buf = k & 1;
    // reduce partials over CTAs in a fixed order: warp w sums CTAs w, w+8, ...; then fixed combine
    for (int c = k + lane; c < kb; c += 32) {
      double s = 0.0;
      for (int q = warp; q < G; q += 8) s += __ldcg(&a.part[((size_t)buf * G + q) * (kb + 1) + c]);
      red[warp * (kb + 1) + c] = s;
    }
    __syncthreads();
    for (int c = k + tid; c < kb; c += blockDim.x) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 8; w++) s += red[w * (kb + 1) + c];
      dsum[c] = s;
    }
    __syncthreads();
    if (tid == 0) {
      double x0 = __ldcg(&a.rowk[buf * kb + k]);
      double s = dsum[k];
      double beta, tau, scal;
      if (s == 0.0) { beta = x0; tau = 0.0; scal = 0.0; }
      else {
        double nrm = sqrt(x0 * x0 + s);
        beta = (x0 >= 0.0) ? -nrm : nrm;
        tau = (beta - x0) / beta;
        scal = 1.0 / (x0 - beta);
      }
      scal_s[0] = beta; scal_s[1] = tau; scal_s[2] = scal;
      if (cta == 0) a.tau[k] = tau;
    }
    __syncthreads();
    const double beta = scal_s[0], tau = scal_s[1], scal = scal_s[2];
    for (int c = k + 1 + tid; c < kb; c += blockDim.x)
      wv[c] = tau * (__ldcg(&a.rowk[buf * kb + c]) + scal * dsum[c]);
    __syncthreads();
    // apply reflector k to own rows; store v
    for (int li = tid; li < nr; li += blockDim.x) {
      int64_t gi = rb + li;
      if (gi < k) {
        a.V[SK_IDX(gi, k, a.ldv)] = 0.0;
      } else if (gi == k) {
        P(li, k) = beta;
        a.V[SK_IDX(gi, k, a.ldv)] = 1.0;
        for (int c = k + 1; c < kb; c++) P(li, c) -= wv[c];
      } else {
        double v = P(li, k) * scal;
        P(li, k) = v;
        a.V[SK_IDX(gi, k, a.ldv)] = v;
        for (int c = k + 1; c < kb; c++) P(li, c) -= v * wv[c];
      }
    }
    __syncthreads();
    if (k + 1 < kmax) {
      partials(k + 1);
      __threadfence();
      grid.sync();
    }
  }
  // columns kmax..kb-1 (only when m < kb): identity reflectors
  for (int k = kmax; k < kb; k++) {
    for (int li = tid; li < nr; li += blockDim.x) a.V[SK_IDX(rb + li, k, a.ldv)] = 0.0;
    if (cta == 0 && tid == 0) a.tau[k] = 0.0;
  }
  // write back R rows (gi < kb) to A; the rest of the panel below R is scratch.
  if (SMEM) {
    for (int64_t e = tid; e < (int64_t)nr * kb; e += blockDim.x) {
      int c = (int)(e / nr), li = (int)(e % nr);
      if (rb + li < kb) a.A[SK_IDX(rb + li, c, a.lda)] = (rb + li <= c) ? Ps[(size_t)c * R + li] : 0.0;
    }
  } else {
    for (int64_t e = tid; e < (int64_t)nr * kb; e += blockDim.x) {
      int c = (int)(e / nr), li = (int)(e % nr);
      if (rb + li < kb && rb + li > c) a.A[SK_IDX(rb + li, c, a.lda)] = 0.0;
    }
  }
  // Gram matrix G = V^T V (upper part), partial per CTA, fixed-order reduction
  __syncthreads();
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    int r = e % kb, c = e / kb;
    double s = 0.0;
    if (r < c) {
      for (int li = 0; li < nr; li++) {
        int64_t gi = rb + li;
        double vr = (gi < r) ? 0.0 : (gi == r ? 1.0 : P(li, r));
        double vc = (gi < c) ? 0.0 : (gi == c ? 1.0 : P(li, c));
        s += vr * vc;
      }
    }
    a.gram[(size_t)cta * kb * kb + e] = s;
  }
  __threadfence();
  grid.sync();
  double* gfin = a.gram + (size_t)G * kb * kb;
  for (int e = blockIdx.x * blockDim.x + tid; e < kb * kb; e += G * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < G; q++) s += __ldcg(&a.gram[(size_t)q * kb * kb + e]);
    gfin[e] = s;
  }
  __threadfence();
  grid.sync();
  // T (forward, columnwise dlarft): T[c][c] = tau_c, T[0:c, c] = -tau_c T[0:c,0:c] G[0:c, c]
  if (cta == 0) {
    for (int r = tid; r < kb; r += blockDim.x) {
      double trow[128];
      for (int c = 0; c < kb; c++) trow[c] = 0.0;
      trow[r] = __ldcg(&a.tau[r]);
      for (int c = r + 1; c < kb; c++) {
        double s = 0.0;
        for (int l = r; l < c; l++) s += trow[l] * __ldcg(&gfin[l + c * kb]);
        trow[c] = -__ldcg(&a.tau[c]) * s;
      }
      for (int c = 0; c < kb; c++) a.T[r + c * a.ldt] = trow[c];
    }
  }
}

// ------------------------------------------------------------------------------------
// U = V T  (m x kb), one thread per row; T staged in shared memory.
__global__ void vt_kernel(const double* V, int64_t ldv, const double* T, int ldt, int64_t m, int kb,
                          double* U, int64_t ldu) {
  extern __shared__ double Ts[];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) Ts[e] = T[(e % kb) + (e / kb) * ldt];
  __syncthreads();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  double v[128];
  for (int a = 0; a < kb; a++) v[a] = V[SK_IDX(i, a, ldv)];
  for (int c = 0; c < kb; c++) {
    double s = 0.0;
    for (int a = 0; a <= c; a++) s += v[a] * Ts[a + c * kb];
    U[SK_IDX(i, c, ldu)] = s;
  }
}

// ------------------------------------------------------------------------------------
// a3 skew-SYMM: X = S U, S = L - L^T (L = strictly lower part of A[r0:, r0:]).
// CTA p owns output rows p*BM .. p*BM+BM-1 and runs ONE K loop over
//   (row part)  L[p-rows, 0:(p+1)BM] U[0:(p+1)BM]            (A tile M-major)
//   (col part) -L[pBM:n, p-cols]^T U[pBM:n]                    (A tile K-major)
// i.e. every lower tile is read twice overall and each CTA's K extent is n + BM,
// so the triangular work is balanced across CTAs.  Diagonal tiles are masked to
// the strict triangle in shared memory.
struct SymmArgs {
  const double* S; int64_t lds;   // S(i,j) = S[i + j*lds] for i > j
  const double* U; int64_t ldu;   // m x nb
  double* X; int64_t ldx;
  int64_t m; int nb;
  int vec;
};

template <int BM, int NB, int BK, int STAGES>
__global__ void __launch_bounds__(GemmTile<BM, NB, BK, 32, 32, STAGES, false, false>::NTHREADS) symm_kernel(SymmArgs s) {
  using TR = GemmTile<BM, NB, BK, 32, 32, STAGES, false, false>;   // row part: A M-major
  using TC = GemmTile<BM, NB, BK, 32, 32, STAGES, true, false>;    // col part: A K-major
  constexpr int NT = TR::NTHREADS;
  extern __shared__ __align__(16) double smem[];
  const int64_t p = blockIdx.x;
  const int64_t m0 = p * BM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % TR::NWARP_M) * 32, wn0 = (warp / TR::NWARP_M) * 32;
  double acc[TR::FM][TR::FN][2];
#pragma unroll
  for (int i = 0; i < TR::FM; i++)
#pragma unroll
    for (int j = 0; j < TR::FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  // ---------------- row part: K in [0, min(m, (p+1)BM))
  {
    GemmArgs g;
    g.M = s.m; g.N = s.nb; g.K = smin<int64_t>(s.m, m0 + BM);
    g.A = s.S; g.lda = s.lds; g.B = s.U; g.ldb = s.ldu; g.vec = s.vec;
    double* As = smem;
    double* Bs = smem + STAGES * TR::A_STAGE;
    const int64_t nk = (g.K + BK - 1) / BK;
    for (int st = 0; st < STAGES - 1; st++) {
      if (st < nk) TR::load_stage(g, As + st * TR::A_STAGE, Bs + st * TR::B_STAGE, m0, 0, st * BK, tid);
      cp_async_commit();
    }
    for (int64_t kb = 0; kb < nk; kb++) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int cs = (int)(kb % STAGES);
      const int64_t k0 = kb * BK;
      if (k0 + BK > m0) {   // diagonal tile: keep row > col only
        double* a = As + cs * TR::A_STAGE;
        for (int e = tid; e < BK * BM; e += NT) {
          int kk = e / BM, mm = e % BM;
          if (m0 + mm <= k0 + kk) a[kk * TR::A_LD + mm] = 0.0;
        }
        __syncthreads();
      }
      int64_t pf = kb + STAGES - 1;
      if (pf < nk) {
        int ps = (int)(pf % STAGES);
        TR::load_stage(g, As + ps * TR::A_STAGE, Bs + ps * TR::B_STAGE, m0, 0, pf * BK, tid);
      }
      cp_async_commit();
      TR::mma_stage(As + cs * TR::A_STAGE, Bs + cs * TR::B_STAGE, acc, wm0, wn0, lane);
    }
    cp_async_wait<0>();
    __syncthreads();
  }
  // negate: the column part subtracts
#pragma unroll
  for (int i = 0; i < TR::FM; i++)
#pragma unroll
    for (int j = 0; j < TR::FN; j++) { acc[i][j][0] = -acc[i][j][0]; acc[i][j][1] = -acc[i][j][1]; }
  // ---------------- column part: K (rows of S) in [m0, m); A(mm, k) = S[k, m0+mm]
  {
    GemmArgs g;
    g.M = s.m; g.N = s.nb; g.K = s.m;
    g.A = s.S; g.lda = s.lds; g.B = s.U; g.ldb = s.ldu; g.vec = s.vec;
    double* As = smem;
    double* Bs = smem + STAGES * TC::A_STAGE;
    const int64_t nk = (s.m - m0 + BK - 1) / BK;
    for (int st = 0; st < STAGES - 1; st++) {
      if (st < nk) TC::load_stage(g, As + st * TC::A_STAGE, Bs + st * TC::B_STAGE, m0, 0, m0 + st * BK, tid);
      cp_async_commit();
    }
    for (int64_t kb = 0; kb < nk; kb++) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int cs = (int)(kb % STAGES);
      const int64_t k0 = m0 + kb * BK;
      if (k0 < m0 + BM) {   // diagonal tile: keep k > m0+mm only
        double* a = As + cs * TC::A_STAGE;
        for (int e = tid; e < BK * BM; e += NT) {
          int mm = e / BK, kk = e % BK;
          if (k0 + kk <= m0 + mm) a[mm * TC::A_LD + kk] = 0.0;
        }
        __syncthreads();
      }
      int64_t pf = kb + STAGES - 1;
      if (pf < nk) {
        int ps = (int)(pf % STAGES);
        TC::load_stage(g, As + ps * TC::A_STAGE, Bs + ps * TC::B_STAGE, m0, 0, m0 + pf * BK, tid);
      }
      cp_async_commit();
      TC::mma_stage(As + cs * TC::A_STAGE, Bs + cs * TC::B_STAGE, acc, wm0, wn0, lane);
    }
    cp_async_wait<0>();
  }
  const int gq = lane >> 2, t = lane & 3;
#pragma unroll
  for (int i = 0; i < TR::FM; i++)
#pragma unroll
    for (int j = 0; j < TR::FN; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        int64_t mm = m0 + wm0 + 8 * i + gq;
        int nn = wn0 + 8 * j + 2 * t + h;
        if (mm < s.m && nn < s.nb) s.X[SK_IDX(mm, nn, s.ldx)] = -acc[i][j][h];
      }
}

// ------------------------------------------------------------------------------------
// a4 W correction.  (1) per row-block partial Z_blk = V_blk^T X_blk (kb x kb)
__global__ void vtx_partial_kernel(const double* V, int64_t ldv, const double* X, int64_t ldx, int64_t m, int kb,
                                   int rows_per_blk, double* part) {
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk;
  const int64_t r1 = smin<int64_t>(m, r0 + rows_per_blk);
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    int a = e % kb, c = e / kb;
    double s = 0.0;
    for (int64_t i = r0; i < r1; i++) s += V[SK_IDX(i, a, ldv)] * X[SK_IDX(i, c, ldx)];
    part[(size_t)blockIdx.x * kb * kb + e] = s;
  }
}
// (2) Z = sum of partials (fixed order); Mb = T^T Z; writes Mb (kb x kb)
__global__ void mb_kernel(const double* part, int nblk, const double* T, int ldt, int kb, double* Mb) {
  extern __shared__ double zs[];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nblk; q++) s += part[(size_t)q * kb * kb + e];
    zs[e] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    int a = e % kb, c = e / kb;
    double s = 0.0;
    for (int l = 0; l <= a; l++) s += T[l + a * ldt] * zs[l + c * kb];   // (T^T)_{a l} = T_{l a}, T upper
    Mb[e] = s;
  }
}
// (3) W = X - 1/2 V Mb ; P = [V W], Q = [W -V]  (m x 2kb each, ld = ldp)
__global__ void w_build_kernel(const double* V, int64_t ldv, const double* X, int64_t ldx, const double* Mb,
                               int64_t m, int kb, double* P, double* Q, int64_t ldp) {
  extern __shared__ double ms[];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) ms[e] = Mb[e];
  __syncthreads();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  double v[128];
  for (int a = 0; a < kb; a++) v[a] = V[SK_IDX(i, a, ldv)];
  for (int c = 0; c < kb; c++) {
    double s = 0.0;
    for (int a = 0; a < kb; a++) s += v[a] * ms[a + c * kb];
    double w = X[SK_IDX(i, c, ldx)] - 0.5 * s;
    P[SK_IDX(i, c, ldp)] = v[c];
    P[SK_IDX(i, kb + c, ldp)] = w;
    Q[SK_IDX(i, c, ldp)] = w;
    Q[SK_IDX(i, kb + c, ldp)] = -v[c];
  }
}

// ------------------------------------------------------------------------------------
// Host driver.

static constexpr int kSymmBM = 64, kSymmBK = 16, kSymmStages = 2;
static constexpr int kWRows = 256;

void f2b_reserve(Arena& ar, const F2BLayout& L, int nsm, F2BWork& w) {
  int64_t n = L.n, b = L.b;
  int64_t np = std::max<int64_t>(L.npanel, 1);
  w.tau = ar.take<double>(np * b);
  w.T = ar.take<double>(np * b * b);
  w.part = ar.take<double>(2 * (size_t)nsm * (b + 1));
  w.rowk = ar.take<double>(2 * b);
  w.gram = ar.take<double>((size_t)(nsm + 1) * b * b);
  int64_t ldn = (n + 1) & ~int64_t(1);
  w.U = ar.take<double>(ldn * b);
  w.X = ar.take<double>(ldn * b);
  w.P = ar.take<double>(ldn * 2 * b);
  w.Q = ar.take<double>(ldn * 2 * b);
  w.zpart = ar.take<double>(((n + kWRows - 1) / kWRows + 1) * b * b);
  w.Mb = ar.take<double>(b * b);
}

static int panel_grid(int64_t m, int nsm) {
  int64_t g = (m + 63) / 64;   // at least 64 rows per CTA
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, nsm));
}

cudaError_t f2b_panel(const F2BLayout& L, int64_t j, double* A, int64_t lda, double* vstore, const F2BWork& w,
                      int nsm, cudaStream_t st) {
  const int b = L.b;
  const int64_t c0 = j * b, r0 = L.r0(j), m = L.n - r0;
  const int64_t g = j / L.merge, pl = j % L.merge;
  double* Vj = vstore + L.goff[g] + pl * b + pl * b * L.gld[g];   // row offset pl*b, col offset pl*b
  const int64_t ldv = L.gld[g];
  PanelArgs a;
  a.A = A + SK_IDX(r0, c0, lda); a.lda = lda; a.m = m; a.kb = b;
  a.V = Vj; a.ldv = ldv; a.tau = w.tau + j * b; a.T = w.T + j * (int64_t)b * b; a.ldt = b;
  a.part = w.part; a.rowk = w.rowk; a.gram = w.gram;
  int G = panel_grid(m, nsm);
  a.R = (m + G - 1) / G;
  size_t extra = (size_t)(8 * (b + 1) + (b + 1) + b + 4) * sizeof(double);
  size_t smem_full = (size_t)b * a.R * sizeof(double) + extra;
  bool use_smem = smem_full <= 200 * 1024;
  a.smem_rows = use_smem ? (int)a.R : 0;
  void* args[] = {&a};
  cudaError_t e;
  KScope ks(KC_PANEL, st);
  if (use_smem) {
    static bool set = false;
    if (!set) {
      e = cudaFuncSetAttribute(panel_qr_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + (int)extra);
      if (e) return e;
      set = true;
    }
    e = cudaLaunchCooperativeKernel((void*)panel_qr_kernel<true>, dim3(G), dim3(256), args, smem_full, st);
  } else {
    e = cudaLaunchCooperativeKernel((void*)panel_qr_kernel<false>, dim3(G), dim3(256), args, extra, st);
  }
  return e;
}

cudaError_t f2b_update(const F2BLayout& L, int64_t j, double* A, int64_t lda, double* vstore, const F2BWork& w,
                       cudaStream_t st) {
  const int b = L.b;
  const int64_t r0 = L.r0(j), m = L.n - r0;
  const int64_t g = j / L.merge, pl = j % L.merge;
  const double* Vj = vstore + L.goff[g] + pl * b + pl * b * L.gld[g];
  const int64_t ldv = L.gld[g];
  const double* Tj = w.T + j * (int64_t)b * b;
  const int64_t ldn = (m + 1) & ~int64_t(1);
  double* S = A + SK_IDX(r0, r0, lda);
  cudaError_t e;
  // U = V T
  {
    KScope ks(KC_VT, st);
    vt_kernel<<<(unsigned)((m + 127) / 128), 128, b * b * sizeof(double), st>>>(Vj, ldv, Tj, b, m, b, w.U, ldn);
  }
  // X = S U
  {
    SymmArgs s;
    s.S = S; s.lds = lda; s.U = w.U; s.ldu = ldn; s.X = w.X; s.ldx = ldn; s.m = m; s.nb = b;
    s.vec = gemm_vec_ok(S, lda, w.U, ldn) ? 1 : 0;
    using TR = GemmTile<kSymmBM, 64, kSymmBK, 32, 32, kSymmStages, false, false>;
    using TC = GemmTile<kSymmBM, 64, kSymmBK, 32, 32, kSymmStages, true, false>;
    size_t smem = std::max(TR::SMEM_BYTES, TC::SMEM_BYTES);
    static bool set = false;
    if (!set) {
      e = cudaFuncSetAttribute(symm_kernel<kSymmBM, 64, kSymmBK, kSymmStages>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      set = true;
    }
    KScope ks(KC_SYMM, st);
    symm_kernel<kSymmBM, 64, kSymmBK, kSymmStages><<<(unsigned)((m + kSymmBM - 1) / kSymmBM), TR::NTHREADS, smem, st>>>(s);
  }
  // W correction
  int nblk = (int)((m + kWRows - 1) / kWRows);
  {
  KScope ks(KC_WCORR, st, 3);
  vtx_partial_kernel<<<nblk, 256, 0, st>>>(Vj, ldv, w.X, ldn, m, b, kWRows, w.zpart);
  mb_kernel<<<1, 256, b * b * sizeof(double), st>>>(w.zpart, nblk, Tj, b, b, w.Mb);
  w_build_kernel<<<(unsigned)((m + 127) / 128), 128, b * b * sizeof(double), st>>>(Vj, ldv, w.X, ldn, w.Mb, m, b,
                                                                                     w.P, w.Q, ldn);
  }
  // S_lower += P Q^T
  GemmArgs ga;
  ga.M = m; ga.N = m; ga.K = 2 * b;
  ga.A = w.P; ga.lda = ldn; ga.B = w.Q; ga.ldb = ldn; ga.C = S; ga.ldc = lda; ga.alpha = 1.0; ga.beta = 1.0;
  {
    KScope ks(KC_R2K, st);
    e = gemm_dmma<64, 64, 16, 32, 32, 2, false, true, true>(ga, st);
  }
  if (e) return e;
  return cudaGetLastError();
}

// Whole F2B: A (n x n, lda, strictly lower) -> band of width b in A[c+1..c+b, c],
// reflectors in vstore (layout L), tau / T per panel in w.
cudaError_t f2b_run(const F2BLayout& L, double* A, int64_t lda, double* vstore, const F2BWork& w, int nsm,
                    cudaStream_t st) {
  cudaError_t e;
  for (int64_t j = 0; j < L.npanel; j++) {
    e = f2b_panel(L, j, A, lda, vstore, w, nsm, st);
    if (e) return e;
    e = f2b_update(L, j, A, lda, vstore, w, st);
    if (e) return e;
  }
  return cudaSuccess;
}

}  // namespace sk
