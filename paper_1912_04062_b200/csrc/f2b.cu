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
#include <nccl.h>

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
static constexpr int kMaxPanelCTA = 152;   // >= max co-resident panel CTAs (148 SMs), multiple of 8

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
      // CTAs warp, warp+8, ...: all loads issued before the (fixed-order) sum
      double v[kMaxPanelCTA / 8];
#pragma unroll
      for (int j = 0; j < kMaxPanelCTA / 8; j++) {
        const int q = warp + 8 * j;
        v[j] = (q < G) ? __ldcg(&a.part[((size_t)buf * G + q) * (kb + 1) + c]) : 0.0;
      }
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < kMaxPanelCTA / 8; j++) s += v[j];
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
  // Gram matrix G = V^T V, partial per CTA (4 x 4 register tile per thread), fixed-order
  // reduction over CTAs, then T (forward columnwise dlarft) in shared memory by CTA 0.
  __syncthreads();
  {
    const int r0 = 4 * (tid % 16), c0 = 4 * (tid / 16);   // kb <= 64
    double g4[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) g4[i][j] = 0.0;
    if (r0 < kb && c0 < kb) {
      for (int li = 0; li < nr; li++) {
        const int64_t gi = rb + li;
        double vr[4], vc[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int r = r0 + i, c = c0 + i;
          vr[i] = (r >= kb || gi < r) ? 0.0 : (gi == r ? 1.0 : P(li, r));
          vc[i] = (c >= kb || gi < c) ? 0.0 : (gi == c ? 1.0 : P(li, c));
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int j = 0; j < 4; j++) g4[i][j] += vr[i] * vc[j];
      }
    }
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++)
        if (r0 + i < kb && c0 + j < kb) a.gram[(size_t)cta * kb * kb + (r0 + i) + (c0 + j) * kb] = g4[i][j];
  }
  __threadfence();
  grid.sync();
  double* gfin = a.gram + (size_t)G * kb * kb;
  for (int e = blockIdx.x * blockDim.x + tid; e < kb * kb; e += G * blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int q = 0; q < G; q++) s += __ldcg(&a.gram[(size_t)q * kb * kb + e]);
    gfin[e] = s;
  }
  __threadfence();
  grid.sync();
  // T (forward, columnwise dlarft): T[c][c] = tau_c, T[0:c, c] = -tau_c T[0:c,0:c] G[0:c, c]
  if (cta == 0) {
    const int LDG = kb + 1;                 // odd: conflict-free row/column sweeps
    double* Gs = sm;                        // kb x LDG  (the panel rows are no longer needed)
    double* Ts = sm + kb * LDG;             // kb x LDG
    for (int e = tid; e < kb * kb; e += blockDim.x) {
      const int l = e % kb, c = e / kb;
      Gs[l * LDG + c] = __ldcg(&gfin[e]);
      Ts[l * LDG + c] = 0.0;
    }
    __syncthreads();
    for (int r = tid; r < kb; r += blockDim.x) {
      Ts[r * LDG + r] = __ldcg(&a.tau[r]);
      for (int c = r + 1; c < kb; c++) {
        double s = 0.0;
        for (int l = r; l < c; l++) s += Ts[r * LDG + l] * Gs[l * LDG + c];
        Ts[r * LDG + c] = -__ldcg(&a.tau[c]) * s;
      }
    }
    __syncthreads();
    for (int e = tid; e < kb * kb; e += blockDim.x) {
      const int r = e % kb, c = e / kb;
      a.T[r + c * a.ldt] = Ts[r * LDG + c];
    }
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
  // distributed (P > 1): only column blocks q = qoff (mod P) of S are local.  CTAs [0, nt)
  // compute the row parts  Yrow_p = sum_{local q <= p} L_pq U_q  into X; CTAs
  // [nt, nt + P*nloc) compute piece k of the column part of local column block c,
  // -sum_{p in piece k} L_pc^T U_p, into Ycol[k] (rows of block c); a combine kernel forms
  // X -= sum_k Ycol[k].  Splitting each column part into P pieces balances the CTAs.
  int P = 1, qoff = 0;
  int64_t nt = 0, nloc = 0;
  double* Ycol = nullptr; int64_t ldy = 0;
};

template <int BM, int NB, int BK, int STAGES>
struct SymmParts {
  using TR = GemmTile<BM, NB, BK, 32, 32, STAGES, false, false>;   // row part: A M-major
  using TC = GemmTile<BM, NB, BK, 32, 32, STAGES, true, false>;    // col part: A K-major
  static constexpr int NT = TR::NTHREADS;
  using Acc = double[TR::FM][TR::FN][2];

  // acc += sum over local column blocks q <= p of L_pq U_q   (diagonal block strictly lower)
  __device__ static void row_part(const SymmArgs& s, double* smem, int64_t p, Acc& acc) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp % TR::NWARP_M) * 32, wn0 = (warp / TR::NWARP_M) * 32;
    const int64_t m0 = p * BM;
    GemmArgs g;
    g.M = s.m; g.N = s.nb; g.K = smin<int64_t>(s.m, m0 + BM);
    g.A = s.S; g.lda = s.lds; g.B = s.U; g.ldb = s.ldu; g.vec = s.vec;
    double* As = smem;
    double* Bs = smem + STAGES * TR::A_STAGE;
    constexpr int KPB = BM / BK;   // k-steps per column block
    const int qoff = s.qoff, P = s.P;
    const int64_t nq = (p >= qoff) ? (p - qoff) / P + 1 : 0;
    const int64_t nk = nq * KPB;
    auto kofs = [&](int64_t kb64) -> int64_t {   // local k-step -> global column offset (32-bit math)
      const int kb = (int)kb64;
      return (int64_t)((qoff + P * (kb / KPB)) * BM + (kb % KPB) * BK);
    };
    for (int st = 0; st < STAGES - 1; st++) {
      if (st < nk) TR::load_stage(g, As + st * TR::A_STAGE, Bs + st * TR::B_STAGE, m0, 0, kofs(st), tid);
      cp_async_commit();
    }
    for (int64_t kb = 0; kb < nk; kb++) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int cs = (int)(kb % STAGES);
      const int64_t k0 = kofs(kb);
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
        TR::load_stage(g, As + ps * TR::A_STAGE, Bs + ps * TR::B_STAGE, m0, 0, kofs(pf), tid);
      }
      cp_async_commit();
      TR::mma_stage(As + cs * TR::A_STAGE, Bs + cs * TR::B_STAGE, acc, wm0, wn0, lane);
    }
    cp_async_wait<0>();
    __syncthreads();
  }

  // acc += sum over rows k in [kbeg, kend) of L_{k, c-block}^T U_k  (rows k > column index)
  __device__ static void col_part(const SymmArgs& s, double* smem, int64_t c, int64_t kbeg, int64_t kend, Acc& acc) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp % TR::NWARP_M) * 32, wn0 = (warp / TR::NWARP_M) * 32;
    const int64_t m0 = c * BM;
    GemmArgs g;
    g.M = s.m; g.N = s.nb; g.K = s.m;
    g.A = s.S; g.lda = s.lds; g.B = s.U; g.ldb = s.ldu; g.vec = s.vec;
    double* As = smem;
    double* Bs = smem + STAGES * TC::A_STAGE;
    const int64_t nk = (kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;
    for (int st = 0; st < STAGES - 1; st++) {
      if (st < nk) TC::load_stage(g, As + st * TC::A_STAGE, Bs + st * TC::B_STAGE, m0, 0, kbeg + st * BK, tid);
      cp_async_commit();
    }
    for (int64_t kb = 0; kb < nk; kb++) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const int cs = (int)(kb % STAGES);
      const int64_t k0 = kbeg + kb * BK;
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
        TC::load_stage(g, As + ps * TC::A_STAGE, Bs + ps * TC::B_STAGE, m0, 0, kbeg + pf * BK, tid);
      }
      cp_async_commit();
      TC::mma_stage(As + cs * TC::A_STAGE, Bs + cs * TC::B_STAGE, acc, wm0, wn0, lane);
    }
    cp_async_wait<0>();
    __syncthreads();
  }

  __device__ static void store(const SymmArgs& s, double* out, int64_t ldo, int64_t m0, double sign, Acc& acc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm0 = (warp % TR::NWARP_M) * 32, wn0 = (warp / TR::NWARP_M) * 32;
    const int gq = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < TR::FM; i++)
#pragma unroll
      for (int j = 0; j < TR::FN; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          int64_t mm = m0 + wm0 + 8 * i + gq;
          int nn = wn0 + 8 * j + 2 * t + h;
          if (mm < s.m && nn < s.nb) out[SK_IDX(mm, nn, ldo)] = sign * acc[i][j][h];
        }
  }
};

// a3 skew-SYMM  X = S U,  S = L - L^T (L = strictly lower part of A[r0:, r0:]).
// One device: CTA p runs ONE K loop over the row part L[p, 0:(p+1)BM] U and the column part
// -L[pBM:, p]^T U, so every lower tile is read twice overall and each CTA's K extent is
// n + BM (balanced).  Distributed: see SymmArgs.
template <int BM, int NB, int BK, int STAGES>
__global__ void __launch_bounds__(GemmTile<BM, NB, BK, 32, 32, STAGES, false, false>::NTHREADS) symm_kernel(SymmArgs s) {
  using SP = SymmParts<BM, NB, BK, STAGES>;
  using TR = typename SP::TR;
  extern __shared__ __align__(16) double smem[];
  double acc[TR::FM][TR::FN][2];
#pragma unroll
  for (int i = 0; i < TR::FM; i++)
#pragma unroll
    for (int j = 0; j < TR::FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t bid = blockIdx.x;
  if (s.P == 1) {
    SP::row_part(s, smem, bid, acc);
#pragma unroll
    for (int i = 0; i < TR::FM; i++)
#pragma unroll
      for (int j = 0; j < TR::FN; j++) { acc[i][j][0] = -acc[i][j][0]; acc[i][j][1] = -acc[i][j][1]; }
    SP::col_part(s, smem, bid, bid * BM, s.m, acc);
    SP::store(s, s.X, s.ldx, bid * BM, -1.0, acc);
  } else if (bid < s.nt) {
    SP::row_part(s, smem, bid, acc);
    SP::store(s, s.X, s.ldx, bid * BM, 1.0, acc);
  } else {
    const int64_t w = bid - s.nt, i = w / s.P, k = w % s.P;
    const int64_t c = s.qoff + (int64_t)s.P * i;
    const int64_t nrb = s.nt - c;                          // row blocks c .. nt-1
    const int64_t b0 = c + (nrb * k) / s.P, b1 = c + (nrb * (k + 1)) / s.P;
    SP::col_part(s, smem, c, b0 * BM, smin<int64_t>(s.m, b1 * BM), acc);
    SP::store(s, s.Ycol + (size_t)k * s.ldy * s.nb, s.ldy, c * BM, 1.0, acc);
  }
}

// X -= sum_k Ycol[k] on the rows of the local column blocks (distributed skew-SYMM)
__global__ void symm_combine_kernel(double* X, int64_t ldx, const double* Ycol, int64_t ldy, int npieces, int64_t m,
                                    int nb, int BM, int P, int qoff) {
  const int64_t col = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t blk = i / BM;
    if (((blk - qoff) % P + P) % P != 0) continue;
    double sacc = 0.0;
    for (int k = 0; k < npieces; k++) sacc += Ycol[(size_t)k * ldy * nb + i + col * ldy];
    X[i + col * ldx] -= sacc;
  }
}

// ------------------------------------------------------------------------------------
// a4 W correction, W = X - 1/2 V (T^T (V^T X))  (Eq. (7)):
// (1) per 256-row chunk: partial Z_chunk = V_chunk^T X_chunk (64 x 64, DMMA tiles)
template <int BK>
__global__ void __launch_bounds__(128) vtx_partial_kernel(const double* V, int64_t ldv, const double* X, int64_t ldx,
                                                          int64_t m, int rows_per_chunk, double* part) {
  using T = GemmTile<64, 64, BK, 32, 32, 2, true, false>;
  extern __shared__ __align__(16) double smem[];
  GemmArgs g;
  g.M = 64; g.N = 64; g.K = m;
  g.A = V; g.lda = ldv; g.B = X; g.ldb = ldx;
  g.vec = gemm_vec_ok(V, ldv, X, ldx) ? 1 : 0;
  double acc[T::FM][T::FN][2];
#pragma unroll
  for (int i = 0; i < T::FM; i++)
#pragma unroll
    for (int j = 0; j < T::FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t k0 = (int64_t)blockIdx.x * rows_per_chunk;
  T::mainloop(g, smem, 0, 0, k0, smin<int64_t>(m, k0 + rows_per_chunk), acc);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm0 = (warp % T::NWARP_M) * 32, wn0 = (warp / T::NWARP_M) * 32;
  const int gq = lane >> 2, t = lane & 3;
  double* out = part + (size_t)blockIdx.x * 64 * 64;
#pragma unroll
  for (int i = 0; i < T::FM; i++)
#pragma unroll
    for (int j = 0; j < T::FN; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) out[(wm0 + 8 * i + gq) + (wn0 + 8 * j + 2 * t + h) * 64] = acc[i][j][h];
}
// (2) Z = sum of the chunk partials (fixed order, loads in flight), one element per thread
__global__ void zsum_kernel(const double* part, int nchunk, int cnt, double* Z) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cnt) return;
  double s = 0.0;
#pragma unroll 8
  for (int q = 0; q < nchunk; q++) s += part[(size_t)q * cnt + e];
  Z[e] = s;
}
// (3) Mb = T^T Z (kb x kb, T upper), one CTA
__global__ void mb_kernel(const double* Z, const double* T, int ldt, int kb, double* Mb) {
  extern __shared__ double zs[];   // kb x kb (T is read through L1/L2)
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) zs[e] = Z[e];
  __syncthreads();
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    const int a = e % kb, c = e / kb;
    double s = 0.0;
    for (int l = 0; l <= a; l++) s += T[l + a * ldt] * zs[l + c * kb];   // (T^T)_{a l} = T_{l a}
    Mb[e] = s;
  }
}
// (4) P = [V W], Q = [W -V] with W already in P[:, kb:2kb]
__global__ void pq_build_kernel(const double* V, int64_t ldv, int64_t m, int kb, double* P, double* Q, int64_t ldp) {
  const int64_t c = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = V[SK_IDX(i, c, ldv)];
    const double w = P[SK_IDX(i, kb + c, ldp)];
    P[SK_IDX(i, c, ldp)] = v;
    Q[SK_IDX(i, c, ldp)] = w;
    Q[SK_IDX(i, kb + c, ldp)] = -v;
  }
}

// ------------------------------------------------------------------------------------
// Host driver.

static constexpr int kSymmBM = 64, kSymmBK = 16, kSymmStages = 2;
static constexpr int kWRows = 256;

void f2b_reserve(Arena& ar, const F2BLayout& L, int nsm, F2BWork& w, int P) {
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
  w.zpart = ar.take<double>(((n + kWRows - 1) / kWRows + 2) * b * b);
  w.Mb = ar.take<double>(b * b);
  if (P > 1) w.Ycol = ar.take<double>((size_t)P * ldn * b);
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
  const size_t tbuild = (size_t)2 * b * (b + 1) * sizeof(double);   // CTA 0's G and T in the T build
  size_t smem_full = std::max((size_t)b * a.R * sizeof(double), tbuild) + extra;
  bool use_smem = (size_t)b * a.R * sizeof(double) + extra <= 200 * 1024;
  if (!use_smem) extra = std::max(extra, tbuild);
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
    e = cudaFuncSetAttribute(panel_qr_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)extra);
    if (e) return e;
    e = cudaLaunchCooperativeKernel((void*)panel_qr_kernel<false>, dim3(G), dim3(256), args, extra, st);
  }
  return e;
}

cudaError_t f2b_update(const F2BLayout& L, int64_t j, double* A, int64_t lda, double* vstore, const F2BWork& w,
                       cudaStream_t st, const Dist& d, int* nccl_err) {
  // distributed: trailing column block q (global block j+1+q) is local iff (j+1+q) mod P == rank
  const int qoff = (int)((((int64_t)d.rank - (j + 1)) % d.P + d.P) % d.P);
  const int b = L.b;
  const int64_t r0 = L.r0(j), m = L.n - r0;
  const int64_t g = j / L.merge, pl = j % L.merge;
  const double* Vj = vstore + L.goff[g] + pl * b + pl * b * L.gld[g];
  const int64_t ldv = L.gld[g];
  const double* Tj = w.T + j * (int64_t)b * b;
  const int64_t ldn = (m + 1) & ~int64_t(1);
  double* S = A + SK_IDX(r0, r0, lda);
  double* Wp = w.P + ldn * b;   // X, then W, lives in P[:, b:2b]
  cudaError_t e;
  {   // U = V T  (m x b)
    KScope ks(KC_VT, st);
    GemmArgs ga;
    ga.M = m; ga.N = b; ga.K = b;
    ga.A = Vj; ga.lda = ldv; ga.B = Tj; ga.ldb = b; ga.C = w.U; ga.ldc = ldn; ga.alpha = 1.0; ga.beta = 0.0;
    e = gemm_dmma<64, 64, 16, 32, 32, 2, false, false, false>(ga, st);
    if (e) return e;
  }
  {   // X = S U  -> P[:, b:2b]
    SymmArgs s;
    s.S = S; s.lds = lda; s.U = w.U; s.ldu = ldn; s.X = Wp; s.ldx = ldn; s.m = m; s.nb = b;
    s.vec = gemm_vec_ok(S, lda, w.U, ldn) ? 1 : 0;
    s.P = d.P; s.qoff = qoff;
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
    const int64_t nt = (m + kSymmBM - 1) / kSymmBM;
    int64_t grid = nt;
    if (d.P > 1) {
      s.nt = nt;
      s.nloc = (nt > qoff) ? (nt - qoff + d.P - 1) / d.P : 0;
      s.Ycol = w.Ycol; s.ldy = ldn;
      grid = nt + (int64_t)d.P * s.nloc;
    }
    KScope ks(KC_SYMM, st, d.P > 1 ? 2 : 1);
    symm_kernel<kSymmBM, 64, kSymmBK, kSymmStages><<<(unsigned)grid, TR::NTHREADS, smem, st>>>(s);
    if (d.P > 1) {
      dim3 cg((unsigned)std::min<int64_t>((m + 255) / 256, 64), (unsigned)b);
      symm_combine_kernel<<<cg, 256, 0, st>>>(Wp, ldn, w.Ycol, ldn, d.P, m, b, kSymmBM, d.P, qoff);
    }
  }
  if (d.P > 1) {   // Y = sum over ranks of the partial skew-SYMM products (NVLink allreduce)
    ncclResult_t r = ncclAllReduce(Wp, Wp, (size_t)ldn * b, ncclDouble, ncclSum, (ncclComm_t)d.comm, st);
    if (r != ncclSuccess) { *nccl_err = (int)r; return cudaErrorUnknown; }
  }
  {   // W = X - 1/2 V (T^T (V^T X));  P = [V W], Q = [W -V]
    KScope ks(KC_WCORR, st, 5);
    const int nchunk = (int)((m + kWRows - 1) / kWRows);
    using TV = GemmTile<64, 64, 16, 32, 32, 2, true, false>;
    vtx_partial_kernel<16><<<nchunk, 128, TV::SMEM_BYTES, st>>>(Vj, ldv, Wp, ldn, m, kWRows, w.zpart);
    double* Zr = w.zpart + (size_t)nchunk * b * b;
    zsum_kernel<<<(b * b + 255) / 256, 256, 0, st>>>(w.zpart, nchunk, b * b, Zr);
    mb_kernel<<<1, 256, b * b * sizeof(double), st>>>(Zr, Tj, b, b, w.Mb);
    GemmArgs ga;
    ga.M = m; ga.N = b; ga.K = b;
    ga.A = Vj; ga.lda = ldv; ga.B = w.Mb; ga.ldb = b; ga.C = Wp; ga.ldc = ldn; ga.alpha = -0.5; ga.beta = 1.0;
    e = gemm_dmma<64, 64, 16, 32, 32, 2, false, false, false>(ga, st);
    if (e) return e;
    dim3 grid((unsigned)std::min<int64_t>((m + 255) / 256, 32), (unsigned)b);
    pq_build_kernel<<<grid, 256, 0, st>>>(Vj, ldv, m, b, w.P, w.Q, ldn);
  }
  // S_lower += P Q^T
  GemmArgs ga;
  ga.M = m; ga.N = m; ga.K = 2 * b;
  ga.A = w.P; ga.lda = ldn; ga.B = w.Q; ga.ldb = ldn; ga.C = S; ga.ldc = lda; ga.alpha = 1.0; ga.beta = 1.0;
  ga.col_stride = d.P; ga.col_off = qoff;   // update only the local column blocks
  {
    KScope ks(KC_R2K, st);
    e = gemm_dmma<64, 64, 16, 32, 32, 2, false, true, true>(ga, st);
  }
  if (e) return e;
  return cudaGetLastError();
}

// Whole F2B: A (n x n, lda, strictly lower) -> band of width b in A[c+1..c+b, c],
// reflectors in vstore (layout L), tau / T per panel in w.
// Distributed (d.P > 1, b = 64): panel j is factored by its owner (j mod P) and broadcast
// (V_j, T_j, tau_j); every rank forms its partial skew-SYMM from its local column blocks,
// the partial products are summed with an allreduce, W is formed redundantly and each rank
// updates only its local column blocks.
cudaError_t f2b_run(const F2BLayout& L, double* A, int64_t lda, double* vstore, const F2BWork& w, int nsm,
                    cudaStream_t st, const Dist& d, int* nccl_err) {
  cudaError_t e;
  if (d.P > 1 && L.b != 64) return cudaErrorInvalidValue;
  for (int64_t j = 0; j < L.npanel; j++) {
    const int owner = (int)(j % d.P);
    if (d.rank == owner) {
      e = f2b_panel(L, j, A, lda, vstore, w, nsm, st);
      if (e) return e;
    }
    if (d.P > 1) {
      const int64_t g = j / L.merge, pl = j % L.merge;
      double* Vcols = vstore + L.goff[g] + pl * (int64_t)L.b * L.gld[g];   // the panel's columns of the group block
      ncclComm_t comm = (ncclComm_t)d.comm;
      ncclResult_t r = ncclGroupStart();
      if (r == ncclSuccess) r = ncclBroadcast(Vcols, Vcols, (size_t)L.gld[g] * L.b, ncclDouble, owner, comm, st);
      if (r == ncclSuccess) r = ncclBroadcast(w.T + j * (int64_t)L.b * L.b, w.T + j * (int64_t)L.b * L.b,
                                              (size_t)L.b * L.b, ncclDouble, owner, comm, st);
      if (r == ncclSuccess) r = ncclBroadcast(w.tau + j * L.b, w.tau + j * L.b, (size_t)L.b, ncclDouble, owner, comm, st);
      ncclResult_t r2 = ncclGroupEnd();
      if (r != ncclSuccess || r2 != ncclSuccess) { *nccl_err = (int)(r != ncclSuccess ? r : r2); return cudaErrorUnknown; }
    }
    e = f2b_update(L, j, A, lda, vstore, w, st, d, nccl_err);
    if (e) return e;
  }
  return cudaSuccess;
}

}  // namespace sk
