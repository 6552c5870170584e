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
#include "tma_gemm.cuh"
#include "internal.h"
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <nccl.h>

namespace cg = cooperative_groups;

namespace sk {

void F2BLayout::init(int64_t n_, int b_, int merge_, bool onestep) {
  n = n_; b = b_; merge = merge_;
  roff = onestep ? 1 : b;
  if (onestep) npanel = (n >= 3) ? (n - 2 + b - 1) / b : 0;
  else npanel = (n >= 2 + b) ? (n - 2) / b : 0;
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
  unsigned* gbar;              // grid barrier counter (zeroed before each launch; common.cuh grid_barrier)
};

template <bool SMEM>
__device__ __noinline__ void panel_householder(const PanelArgs& a, double* sm, unsigned& bar_epoch) {
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
  // partials for column k: rows gi > k: norm = sum x^2 (slot k), dots with columns c > k.
  // Thread (column k + tid%64, row group tid/64) sums every 4th row with two chains, then
  // the 4 row groups are combined in fixed order (deterministic).
  auto partials = [&](int k) {
    const int buf = k & 1;
    const int c = k + (tid & 63), rg = tid >> 6;
    double s0 = 0.0, s1 = 0.0;
    if (c < kb) {
      int li = rg;
      if (rb <= k) li += 4 * (int)((k - rb + 4 - rg) / 4);   // first li with rb + li > k, li = rg (mod 4)
      for (; li + 4 < nr; li += 8) { s0 += P(li, k) * P(li, c); s1 += P(li + 4, k) * P(li + 4, c); }
      if (li < nr) s0 += P(li, k) * P(li, c);
    }
    red[rg * (kb + 1) + (tid & 63)] = s0 + s1;
    __syncthreads();
    if (tid < 64 && k + tid < kb) {
      const double t = (red[tid] + red[(kb + 1) + tid]) + (red[2 * (kb + 1) + tid] + red[3 * (kb + 1) + tid]);
      a.part[((size_t)buf * G + cta) * (kb + 1) + k + tid] = t;
    }
    // owner of row k publishes row k (c >= k)
    if (k >= rb && k < re) {
      for (int cc = k + tid; cc < kb; cc += blockDim.x) a.rowk[buf * kb + cc] = P((int)(k - rb), cc);
    }
  };
  partials(0);
  __threadfence();
  grid_barrier(a.gbar, bar_epoch);
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
      grid_barrier(a.gbar, bar_epoch);
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
  grid_barrier(a.gbar, bar_epoch);
  double* gfin = a.gram + (size_t)G * kb * kb;
  for (int e = blockIdx.x * blockDim.x + tid; e < kb * kb; e += G * blockDim.x) {
    double s = 0.0;
#pragma unroll 8
    for (int q = 0; q < G; q++) s += __ldcg(&a.gram[(size_t)q * kb * kb + e]);
    gfin[e] = s;
  }
  __threadfence();
  grid_barrier(a.gbar, bar_epoch);
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

template <bool SMEM>
__global__ void __launch_bounds__(256) panel_qr_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double sm[];
  unsigned bar_epoch = 0;
  panel_householder<SMEM>(a, sm, bar_epoch);
}

// ------------------------------------------------------------------------------------
// a1 + a2, default for tall panels: CholeskyQR2 + Householder reconstruction.  The
// column-by-column Householder panel needs one grid-wide reduction per column (64 per
// panel, latency-bound: ~0.6 ms per 32k-row panel, on the critical path of every rank in
// the distributed reduction).  Here the panel costs seven grid barriers:
//   P = Q1 R1, Q1 = P R1^-1 with R1^T R1 = P^T P (Cholesky), twice (CholQR2: Q orthonormal
//   to working precision when kappa(P) <= ~1e7), then the compact WY form of the SAME
//   orthogonal factor from Q (Ballard et al., "Reconstructing Householder vectors from
//   tall-skinny QR"): Q - S = Y U (LU without pivoting, S = diag(-sign) of the running
//   pivot, so |pivots| >= 1), V = Y (unit lower trapezoidal), T = -U S Y1^-T (upper), and
//   I - V T V^T maps [I; 0] to Q S, i.e. P = (I - V T V^T) [S R; 0], R = R2 R1.
// The result is a valid panel factorisation (PAPER.md:420-425 only needs an orthogonal
// Q1^(j) = I - V T V^T with Q1^T P upper triangular); tau_i = T_ii.  When a Cholesky pivot
// is <= 1e-12 max_i G_ii (kappa(P) >~ 1e6, e.g. rank-deficient panels) every CTA falls
// back to the Householder panel above in the same launch (A is only written at the end).
struct CqrArgs {
  PanelArgs p;
  double* scr;   // global scratch: [kb*kb] R1, [kb*kb] R (accumulated), [kb*kb] U, [kb] S, [2] flag
  long long* dbg = nullptr;   // SKEWEIG_PANEL_DBG: phase clocks of CTAs 0 and 1
};

template <int KB>
__global__ void __launch_bounds__(256, 1) panel_cqr_kernel(CqrArgs ca) {
  unsigned bar_epoch = 0;
  extern __shared__ __align__(16) double sm[];
  const PanelArgs& a = ca.p;
  const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rb = (int64_t)cta * a.R;
  const int nr = (int)smax<int64_t>(0, smin<int64_t>(a.m, rb + a.R) - rb);
  const int LDP = (int)(a.R | 1);             // odd column stride of the panel rows in smem
  constexpr int LDK = KB + 1;                 // odd leading dimension for kb x kb tiles
  double* Ps = sm;                            // [KB][LDP]
  double* Ms = sm + (size_t)KB * LDP;         // kb x LDK (R factor / U / T work)
  double* Ms2 = Ms + KB * LDK;                // kb x LDK
  double* aux = Ms2 + KB * LDK;               // [2 KB] diag inverses / signs
  double* gR1 = ca.scr;
  double* gR = gR1 + KB * KB;
  double* gU = gR + KB * KB;
  double* gS = gU + KB * KB;
  double* gflag = gS + KB;
  double* gfin = a.gram + (size_t)G * KB * KB;
  auto P = [&](int li, int c) -> double& { return Ps[(size_t)c * LDP + li]; };
  // kb x kb tile from global scratch (L2): all 16 loads per thread in flight, then the stores
  // (a load -> shared-store loop would serialise one L2 round trip per element)
  static_assert(KB * KB % 256 == 0, "256 threads");
  constexpr int NPT = KB * KB / 256;
  auto ldtile = [&](const double* g, double (&v)[NPT]) {
#pragma unroll
    for (int i = 0; i < NPT; i++) v[i] = __ldcg(g + tid + 256 * i);
  };
  int nts = 0;
  auto TS = [&]() { if (ca.dbg && cta < 2 && tid == 0 && nts < 16) ca.dbg[cta * 16 + nts++] = clock64(); };
  TS();
  for (int c = warp; c < KB; c += 8) {   // cp.async: every load in flight at once
    const double* src = a.A + SK_IDX(rb, c, a.lda);
    for (int li = lane; li < nr; li += 32) cp_async8(&Ps[(size_t)c * LDP + li], &src[li], 8);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  TS();
  // Gram G = P^T P: thread (p, q) accumulates rows p + 16i, columns q + 16j (4 x 4), which
  // keeps a half-warp's smem reads on distinct banks (odd LDP); fixed-order reduction over
  // the CTAs, spread over every CTA (28 entries x 9 partial sums each, then combined in order)
  auto gram = [&]() {
    const int p = tid & 15, q = tid >> 4;
    double g4[4][4];
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) g4[i][j] = 0.0;
#pragma unroll 2
    for (int li = 0; li < nr; li++) {
      double vr[4], vc[4];
#pragma unroll
      for (int i = 0; i < 4; i++) { vr[i] = P(li, p + 16 * i); vc[i] = P(li, q + 16 * i); }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) g4[i][j] += vr[i] * vc[j];
    }
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) a.gram[(size_t)cta * KB * KB + (p + 16 * i) + (q + 16 * j) * KB] = g4[i][j];
    TS();
    __threadfence();
    grid_barrier(a.gbar, bar_epoch);
    TS();
    {
      const int per = (KB * KB + G - 1) / G;   // entries of this CTA: [cta*per, cta*per + per)
      const int le = tid / 9, part = tid % 9;
      double* red9 = Ms2;                      // [28][9] partials (Ms2 is free here)
      for (int base = 0; base < per; base += 28) {
        const int e = cta * per + base + le;
        double s = 0.0;
        if (le < 28 && base + le < per && e < KB * KB) {
          constexpr int NQ = (kMaxPanelCTA + 8) / 9;   // loads in flight, fixed-order sum
          double v[NQ];
#pragma unroll
          for (int i = 0; i < NQ; i++) {
            const int qq = part + 9 * i;
            v[i] = (qq < G) ? __ldcg(&a.gram[(size_t)qq * KB * KB + e]) : 0.0;
          }
#pragma unroll
          for (int i = 0; i < NQ; i++) s += v[i];
        }
        if (tid < 9 * 28) red9[tid] = s;
        __syncthreads();
        const int e2 = cta * per + base + tid;
        if (tid < 28 && base + tid < per && e2 < KB * KB) {
          double t = 0.0;
          for (int k = 0; k < 9; k++) t += red9[tid * 9 + k];
          gfin[e2] = t;
        }
        __syncthreads();
      }
    }
    __threadfence();
    grid_barrier(a.gbar, bar_epoch);
    TS();
  };
  const int ti = tid >> 4, tj = tid & 15;   // CTA 0's 16 x 16 thread grid over kb x kb tiles
  // CTA 0: Ms[r][c] -= (s * xrow[r*xs]) * yrow[c] over r, c > k (c >= r if upper), the
  // thread's own 4 x 4 block only; row / column k are not written in the same step, so the
  // caller needs ONE barrier per step (after this)
  auto rank1_own = [&](int k, const double* xrow, int xs, double xscale, const double* yrow, bool upper) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int r = k + 1 + ti + 16 * u;
      if (r >= KB) continue;
      const double x = xrow[r * xs] * xscale;
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int c = k + 1 + tj + 16 * v;
        if (c < KB && (!upper || c >= r)) Ms[r * LDK + c] -= x * yrow[c];
      }
    }
  };
  // CTA 0: upper Cholesky G = R^T R in Ms (row-major r*LDK + c); returns ok
  __shared__ int bad;
  __shared__ double gmax;
  auto cholesky = [&]() -> bool {
    {
      double v[NPT];
      ldtile(gfin, v);
#pragma unroll
      for (int i = 0; i < NPT; i++) { const int e = tid + 256 * i; Ms[(e % KB) * LDK + e / KB] = v[i]; }
    }
    __syncthreads();
    if (warp == 0) {
      double gm = fmax(Ms[lane * LDK + lane], Ms[(lane + 32) * LDK + lane + 32]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
      if (lane == 0) { gmax = gm; bad = 0; }
    }
    __syncthreads();
    // right-looking, two columns and ONE barrier per step: rows k and k+1 of R go to Ms2 (Ms
    // rows k, k+1 are read-only in the step; row k+1 is updated by column k on the fly), the
    // trailing update uses R[k][r] R[k][c] + R[k+1][r] R[k+1][c]
    static_assert(KB % 2 == 0, "two columns per step");
    for (int k = 0; k < KB; k += 2) {
      const double* g0 = Ms + k * LDK;            // G'[k][.]
      const double* g1 = Ms + (k + 1) * LDK;      // G'[k+1][.] before column k's update
      const double d0 = g0[k];
      const double r0 = (d0 > 0.0) ? sqrt(d0) : 1.0, i0 = 1.0 / r0, s0 = i0 * i0;
      const double x01 = g0[k + 1] * s0;          // column k's multiplier of row k+1
      const double d1 = g1[k + 1] - x01 * g0[k + 1];
      const double r1 = (d1 > 0.0) ? sqrt(d1) : 1.0, i1 = 1.0 / r1, s1 = i1 * i1;
      if (tid == 0 && (!(d0 > 1e-12 * gmax) || !(d1 > 1e-12 * gmax))) bad = 1;
      if (tid >= k && tid < KB) Ms2[k * LDK + tid] = (tid == k) ? r0 : g0[tid] * i0;
      if (tid >= k + 1 && tid < KB) Ms2[(k + 1) * LDK + tid] = (tid == k + 1) ? r1 : (g1[tid] - x01 * g0[tid]) * i1;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int r = k + 2 + ti + 16 * u;
        if (r >= KB) continue;
        const double xa = g0[r] * s0, m1r = g1[r] - x01 * g0[r], xb = m1r * s1;
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const int c = k + 2 + tj + 16 * v;
          if (c < KB && c >= r) Ms[r * LDK + c] -= xa * g0[c] + xb * (g1[c] - x01 * g0[c]);
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < KB * KB; e += blockDim.x) {
      const int r = e / KB, c = e % KB;
      Ms[r * LDK + c] = (c >= r) ? Ms2[r * LDK + c] : 0.0;
    }
    __syncthreads();
    return bad == 0;
  };
  // row li of P <- (row li of P) Rm^-1, Rm upper (row-major, LDK) with inverse diagonal
  // dinv: 16-column register blocks, left-looking over the finished blocks (in smem)
  auto solve_row = [&](int li, const double* Rm, const double* dinv) {
#pragma unroll 1
    for (int cb = 0; cb < KB; cb += 16) {
      double x[16];
#pragma unroll
      for (int c = 0; c < 16; c++) x[c] = P(li, cb + c);
#pragma unroll 4
      for (int j = 0; j < cb; j++) {
        const double xj = P(li, j);
#pragma unroll
        for (int c = 0; c < 16; c++) x[c] -= xj * Rm[j * LDK + cb + c];
      }
#pragma unroll
      for (int j = 0; j < 16; j++) {
        x[j] *= dinv[cb + j];
#pragma unroll
        for (int c = j + 1; c < 16; c++) x[c] -= x[j] * Rm[(cb + j) * LDK + cb + c];
      }
#pragma unroll
      for (int c = 0; c < 16; c++) P(li, cb + c) = x[c];
    }
  };
  // every CTA: rows of P <- P R^-1 with R (upper) from global, right-looking per row
  auto trsm_rows = [&](const double* gRm) {
    {
      double v[NPT];
      ldtile(gRm, v);
#pragma unroll
      for (int i = 0; i < NPT; i++) { const int e = tid + 256 * i; Ms2[(e / KB) * LDK + e % KB] = v[i]; }   // row-major
    }
    __syncthreads();
    if (tid < KB) aux[tid] = 1.0 / Ms2[tid * LDK + tid];
    __syncthreads();
    for (int li = tid; li < nr; li += blockDim.x) solve_row(li, Ms2, aux);
    __syncthreads();
  };
  bool ok = true;
  for (int pass = 0; pass < 2 && ok; pass++) {
    gram();
    if (cta == 0) {
      const bool okc = cholesky();
      // R (row-major) -> global; pass 0: R1; pass 1: R = R2 R1
      if (pass == 0) {
        for (int e = tid; e < KB * KB; e += blockDim.x) gR1[e] = Ms[(e / KB) * LDK + e % KB];
      } else {
        {
          double v[NPT];
          ldtile(gR, v);
#pragma unroll
          for (int i = 0; i < NPT; i++) { const int e = tid + 256 * i; Ms2[(e / KB) * LDK + e % KB] = v[i]; }   // R1
        }
        __syncthreads();
        for (int e = tid; e < KB * KB; e += blockDim.x) {
          const int r = e / KB, c = e % KB;
          double s = 0.0;
          for (int l = r; l <= c; l++) s += Ms[r * LDK + l] * Ms2[l * LDK + c];
          gR1[e] = Ms[r * LDK + c];        // R2 (for the solve)
          gR[e] = s;                       // R2 R1
        }
      }
      if (pass == 0)
        for (int e = tid; e < KB * KB; e += blockDim.x) gR[e] = Ms[(e / KB) * LDK + e % KB];
      if (tid == 0) gflag[0] = okc ? 0.0 : 1.0;
    }
    TS();
    __threadfence();
    grid_barrier(a.gbar, bar_epoch);
    ok = __ldcg(&gflag[0]) == 0.0;
    if (ok) trsm_rows(gR1);
    TS();
  }
  if (!ok) {   // ill-conditioned or rank-deficient panel: Householder, same launch
    __syncthreads();
    panel_householder<true>(a, sm, bar_epoch);
    return;
  }
  // ---- Householder reconstruction: CTA 0 holds rows 0..kb-1 (R >= kb)
  if (cta == 0) {
    // modified LU of Q1 - S (Q1 = top kb x kb of Q) in Ms (row-major)
    for (int e = tid; e < KB * KB; e += blockDim.x) Ms[(e / KB) * LDK + e % KB] = P(e / KB, e % KB);
    __syncthreads();
    // one barrier per step: the pivot and L column k go to Ms2 (column k / row k of Ms are
    // read-only in step k), then merged back into Ms
    for (int k = 0; k < KB; k++) {
      const double d = Ms[k * LDK + k];
      const double sg = (d >= 0.0) ? -1.0 : 1.0;   // S_kk = -sign(d): pivot d - S_kk, |.| >= 1
      const double piv = d - sg, inv = 1.0 / piv;
      if (tid == 0) { aux[k] = sg; Ms2[k * LDK + k] = piv; }
      if (tid > k && tid < KB) Ms2[tid * LDK + k] = Ms[tid * LDK + k] * inv;   // L column
      rank1_own(k, Ms + k, LDK, inv, Ms + k * LDK, false);   // x_r = L[r][k], y_c = U[k][c]
      __syncthreads();
    }
    for (int e = tid; e < KB * KB; e += blockDim.x) {
      const int r = e / KB, c = e % KB;
      if (c <= r) Ms[r * LDK + c] = Ms2[r * LDK + c];   // L (strict lower) and the pivots
    }
    __syncthreads();
    for (int e = tid; e < KB * KB; e += blockDim.x) {
      const int r = e / KB, c = e % KB;
      gU[e] = (c >= r) ? Ms[r * LDK + c] : 0.0;   // U row-major
    }
    if (tid < KB) gS[tid] = aux[tid];
  }
  TS();
  __threadfence();
  grid_barrier(a.gbar, bar_epoch);
  TS();
  // V: rows >= kb: y = q U^-1 (row solve with U upper, right-looking); rows < kb: L1
  {
    double v[NPT];
    ldtile(gU, v);
#pragma unroll
    for (int i = 0; i < NPT; i++) { const int e = tid + 256 * i; Ms2[(e / KB) * LDK + e % KB] = v[i]; }
  }
  __syncthreads();
  if (tid < KB) aux[KB + tid] = 1.0 / Ms2[tid * LDK + tid];
  __syncthreads();
  for (int li = tid; li < nr; li += blockDim.x) {
    const int64_t gi = rb + li;
    if (gi >= KB) {
      solve_row(li, Ms2, aux + KB);
      for (int c = 0; c < KB; c++) a.V[SK_IDX(gi, c, a.ldv)] = P(li, c);
    } else {   // CTA 0: L1 (unit lower)
      for (int c = 0; c < KB; c++) a.V[SK_IDX(gi, c, a.ldv)] = (c < gi) ? Ms[gi * LDK + c] : (c == gi ? 1.0 : 0.0);
    }
  }
  if (cta == 0) {
    // T = -U S Y1^-T (row r: t L1^T = -(U S)_r, forward over c), tau = diag(T); R_h = S R -> A
    __syncthreads();
    double* Ts = Ms2;   // overwrite U copy (no longer needed by CTA 0 after the V rows)
    double* ws = Ps;    // the panel rows are no longer needed either
    {
      double v[NPT];
      ldtile(gU, v);
#pragma unroll
      for (int i = 0; i < NPT; i++) {
        const int e = tid + 256 * i, r = e / KB, c = e % KB;
        ws[r * LDK + c] = (c >= r) ? -v[i] * aux[c] : 0.0;
      }
    }
    __syncthreads();
    // T Y1^T = W column by column: T[:, c] = W[:, c] - sum_{l<c} T[:, l] Y1[c][l]; thread
    // (row r, quarter q) sums l = q, q+4, ..; the 4 quarters combine with shuffles.  Row r
    // only reads its own earlier entries (written by its quarter 0, same warp): a warp
    // barrier per column, the rows run independently
    {
      const int r = tid >> 2, q = tid & 3;
      for (int c = 0; c < KB; c++) {
        double t = 0.0;
        for (int l = r + q; l < c; l += 4) t += Ts[r * LDK + l] * Ms[c * LDK + l];
        t += __shfl_xor_sync(0xffffffffu, t, 1);
        t += __shfl_xor_sync(0xffffffffu, t, 2);
        if (q == 0) Ts[r * LDK + c] = (c < r) ? 0.0 : ws[r * LDK + c] - t;
        __syncwarp();
      }
      __syncthreads();
    }
    {
      double v[NPT];   // gR row-major: element (r, c) at r * KB + c
#pragma unroll
      for (int i = 0; i < NPT; i++) {
        const int e = tid + 256 * i, r = e % KB, c = e / KB;
        v[i] = (r <= c) ? __ldcg(&gR[r * KB + c]) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NPT; i++) {
        const int e = tid + 256 * i, r = e % KB, c = e / KB;
        a.T[r + c * a.ldt] = Ts[r * LDK + c];
        a.A[SK_IDX(r, c, a.lda)] = (r <= c) ? aux[r] * v[i] : 0.0;
      }
    }
    if (tid < KB) a.tau[tid] = Ts[tid * LDK + tid];
  }
  __syncthreads();
  TS();
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
  int split = 1;   // single device: > 1 = split-K pieces per row block (Ycol[0..split))
};

template <int BM, int NB, int BK, int STAGES>
struct SymmParts {
  using TR = GemmTile<BM, NB, BK, 32, 32, STAGES, false, false>;   // row part: A M-major
  using TC = GemmTile<BM, NB, BK, 32, 32, STAGES, true, false>;    // col part: A K-major
  static constexpr int NT = TR::NTHREADS;
  using Acc = double[TR::FM][TR::FN][2];

  // acc += sum over local column blocks q <= p of L_pq U_q   (diagonal block strictly lower)
  __device__ static void row_part(const SymmArgs& s, double* smem, int64_t p, Acc& acc, int64_t ks0 = 0,
                                  int64_t ks1 = INT64_MAX) {
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
    const int64_t kbeg = smin<int64_t>(ks0, nq * KPB), nk = smin<int64_t>(ks1, nq * KPB) - kbeg;   // k-steps
    auto kofs = [&](int64_t j64) -> int64_t {   // k-step kbeg+j -> global column offset (32-bit math)
      const int kb = (int)(kbeg + j64);
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
  if (s.split > 1) {
    // single device, split-K: row block p, piece k of its "virtual" K range -- the row part
    // (k-steps of the column blocks 0..p) followed by the column part (rows p*BM .. m) --
    // into Ycol[k]; a combine kernel sums the pieces.  Equal-size CTAs, no long tail.
    const int64_t p = bid / s.split, k = bid % s.split;
    constexpr int KPB = BM / BK;
    const int64_t kr = (p + 1) * KPB;                             // row-part k-steps
    const int64_t kc = (s.m - p * BM + BK - 1) / BK;              // column-part k-steps
    const int64_t kv = kr + kc;
    const int64_t v0 = (kv * k) / s.split, v1 = (kv * (k + 1)) / s.split;
    if (v0 < kr) SP::row_part(s, smem, p, acc, v0, smin<int64_t>(v1, kr));
#pragma unroll
    for (int i = 0; i < TR::FM; i++)
#pragma unroll
      for (int j = 0; j < TR::FN; j++) { acc[i][j][0] = -acc[i][j][0]; acc[i][j][1] = -acc[i][j][1]; }
    if (v1 > kr) {
      const int64_t r0 = p * BM + (smax<int64_t>(v0, kr) - kr) * BK, r1 = smin<int64_t>(s.m, p * BM + (v1 - kr) * BK);
      SP::col_part(s, smem, p, r0, r1, acc);
    }
    SP::store(s, s.Ycol + (size_t)k * s.ldy * s.nb, s.ldy, p * BM, -1.0, acc);
  } else if (s.P == 1) {
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

// ---- a3 skew-SYMM, one device, TMA-fed persistent version --------------------------------
// Work unit (p, piece): a contiguous range [v0, v1) of row block p's "virtual" K sequence --
// the kr = (p+1) BM/BK k-blocks of the row part L[p, 0:(p+1)BM] U followed by the kc k-blocks
// of the column part -L[pBM:m, p]^T U.  kr + kc = (nt + 1) BM / BK is the same for every p,
// so all units are equal.  The producer warp streams each k-block as one TMA box of S (row
// part: box (BM+4) x BK, M-major; column part: box (BK+4) x BM of the transposed region,
// K-major) plus one box of U; the consumers run the matching GemmTile fragment loop, with
// the strictly-lower mask applied to the A fragments of the diagonal k-blocks in registers.
template <int BM, int BK>
struct SymmTma {
  using TR = GemmTile<BM, 64, BK, 32, 32, 2, false, false>;   // row part: A(m, k) = S[m0+m, k0+k]
  using TC = GemmTile<BM, 64, BK, 32, 32, 2, true, false>;    // col part: A(m, k) = S[k0+k, m0+m]
  static constexpr int NCW = TR::NTHREADS / 32;
  static constexpr int THREADS = TR::NTHREADS + 32;
  static constexpr int A_ST = (TR::A_STAGE > TC::A_STAGE ? TR::A_STAGE : TC::A_STAGE);
  static constexpr int B_ST = TR::B_STAGE;
  static constexpr int NS = 4;
  static constexpr size_t SMEM = (size_t)NS * (A_ST + B_ST) * sizeof(double) + 2 * NS * 8 + 128;
  static constexpr unsigned AR_BYTES = (unsigned)(TR::A_STAGE * 8), AC_BYTES = (unsigned)(TC::A_STAGE * 8);
  static constexpr unsigned B_BYTES = (unsigned)(B_ST * 8);
  static_assert(TR::B_STAGE == TC::B_STAGE && (A_ST * 8) % 128 == 0 && (B_ST * 8) % 128 == 0, "symm tma layout");
};

struct SymmTmaArgs {
  int64_t m, nt;
  int split;
  double* out; int64_t ldo;     // split == 1: X; else Ycol (piece k at out + k*ldo*64)
};

// mma_stage with the strictly-lower mask of S on the A fragments: keep A(m, k) iff its S row
// index exceeds its S column index; row part: m0 + m > k0 + k, column part: k0 + k > m0 + m.
template <class T, bool ROWPART>
__device__ __forceinline__ void symm_stage_masked(const double* As, const double* Bs, double (&acc)[T::FM][T::FN][2],
                                                  int wm0, int wn0, int lane, int dk /* k0 - m0 */) {
  const int gq = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kk = 0; kk < T::BK_; kk += 4) {
    double af[T::FM], bf[T::FN];
#pragma unroll
    for (int i = 0; i < T::FM; i++) {
      const int mm = wm0 + 8 * i + gq, kx = kk + t;
      const double a = T::a_at(As, mm, kx);
      const bool keep = ROWPART ? (mm > kx + dk) : (kx + dk > mm);
      af[i] = keep ? a : 0.0;
    }
#pragma unroll
    for (int j = 0; j < T::FN; j++) bf[j] = T::b_at(Bs, kk + t, wn0 + 8 * j + gq);
#pragma unroll
    for (int i = 0; i < T::FM; i++)
#pragma unroll
      for (int j = 0; j < T::FN; j++) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

template <int BM, int BK>
__global__ void __launch_bounds__(SymmTma<BM, BK>::THREADS, 1)
    symm_tma_kernel(const __grid_constant__ CUtensorMap mapR, const __grid_constant__ CUtensorMap mapC,
                    const __grid_constant__ CUtensorMap mapU, SymmTmaArgs a) {
  using Cfg = SymmTma<BM, BK>;
  using TR = typename Cfg::TR;
  using TC = typename Cfg::TC;
  constexpr int NS = Cfg::NS, KPB = BM / BK;
  // the dynamic shared memory of a kernel without static shared memory starts at the window's
  // base (1 KB aligned): no run-time realignment, so the fragment loads stay LDS (a pointer
  // rebuilt through an integer would turn them into generic loads)
  extern __shared__ __align__(1024) double sm[];
  double* As = sm;
  double* Bs = As + NS * Cfg::A_ST;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + NS * Cfg::B_ST);
  uint64_t* empty = full + NS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], Cfg::NCW); }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t nunits = a.nt * a.split;
  const int64_t kv = (a.nt + 1) * KPB;   // virtual k-blocks per row block (all equal)
  if (warp == Cfg::NCW) {
    // ================================ producer ================================
    if (lane == 0) {
      tma_prefetch_desc(&mapR);
      tma_prefetch_desc(&mapC);
      tma_prefetch_desc(&mapU);
      int64_t it = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t p = u / a.split, k = u % a.split;
        const int64_t kr = (p + 1) * KPB;
        const int64_t v0 = (kv * k) / a.split, v1 = (kv * (k + 1)) / a.split;
        const int m0 = (int)(p * BM);
        for (int64_t v = v0; v < v1; v++, it++) {
          const int s = (int)(it % NS);
          mbar_wait(&empty[s], (unsigned)(((it / NS) & 1) ^ 1));
          const bool row = v < kr;
          const int k0 = row ? (int)(v * BK) : (int)(m0 + (v - kr) * BK);
          mbar_expect_tx(&full[s], (row ? Cfg::AR_BYTES : Cfg::AC_BYTES) + Cfg::B_BYTES);
          if (row) tma_load_2d(As + s * Cfg::A_ST, &mapR, m0, k0, &full[s]);
          else tma_load_2d(As + s * Cfg::A_ST, &mapC, k0, m0, &full[s]);
          tma_load_2d(Bs + s * Cfg::B_ST, &mapU, k0, 0, &full[s]);
        }
      }
    }
    return;
  }
  // ================================ consumers ================================
  const int wm0 = (warp % TR::NWARP_M) * 32, wn0 = (warp / TR::NWARP_M) * 32;
  const int gq = lane >> 2, tq = lane & 3;
  int64_t it = 0;
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t p = u / a.split, k = u % a.split;
    const int64_t kr = (p + 1) * KPB;
    const int64_t v0 = (kv * k) / a.split, v1 = (kv * (k + 1)) / a.split;
    const int64_t m0 = p * BM;
    double acc[TR::FM][TR::FN][2];
#pragma unroll
    for (int i = 0; i < TR::FM; i++)
#pragma unroll
      for (int j = 0; j < TR::FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int64_t v = v0; v < v1; v++, it++) {
      const int s = (int)(it % NS);
      mbar_wait(&full[s], (unsigned)((it / NS) & 1));
      const double* Ast = As + s * Cfg::A_ST;
      const double* Bst = Bs + s * Cfg::B_ST;
      if (v < kr) {
        const int64_t k0 = v * BK;
        if (k0 + BK > m0) symm_stage_masked<TR, true>(Ast, Bst, acc, wm0, wn0, lane, (int)(k0 - m0));
        else TR::mma_stage(Ast, Bst, acc, wm0, wn0, lane);
      } else {
        if (v == kr) {   // entering the column part: acc <- -acc, accumulate L^T U, negate at the end
#pragma unroll
          for (int i = 0; i < TR::FM; i++)
#pragma unroll
            for (int j = 0; j < TR::FN; j++) { acc[i][j][0] = -acc[i][j][0]; acc[i][j][1] = -acc[i][j][1]; }
        }
        const int64_t k0 = m0 + (v - kr) * BK;
        if (k0 < m0 + BM) symm_stage_masked<TC, false>(Ast, Bst, acc, wm0, wn0, lane, (int)(k0 - m0));
        else TC::mma_stage(Ast, Bst, acc, wm0, wn0, lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    const double sg = (v1 > kr) ? -1.0 : 1.0;   // row - col
    double* out = a.out + (size_t)k * a.ldo * 64;
#pragma unroll
    for (int i = 0; i < TR::FM; i++)
#pragma unroll
      for (int j = 0; j < TR::FN; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t mm = m0 + wm0 + 8 * i + gq;
          const int nn = wn0 + 8 * j + 2 * tq + h;
          if (mm < a.m) out[SK_IDX(mm, nn, a.ldo)] = sg * acc[i][j][h];
        }
  }
}

// X = sum_k Ycol[k] (single-device split-K skew-SYMM; fixed order)
__global__ void symm_sum_kernel(double* X, int64_t ldx, const double* Ycol, int64_t ldy, int npieces, int64_t m) {
  const int64_t col = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < npieces; k++) s += Ycol[(size_t)k * ldy * gridDim.y + i + col * ldy];
    X[i + col * ldx] = s;
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
// (3) Mb = T^T Z (kb x kb, T upper): CTA c forms column c, thread a the element (a, c);
// T staged in shared memory (column a contiguous per thread: odd stride, conflict-free)
__global__ void mb_kernel(const double* Z, const double* T, int ldt, int kb, double* Mb) {
  extern __shared__ double ts[];   // kb x (kb + 1): ts[a * (kb+1) + l] = T[l, a]
  double* zc = ts + kb * (kb + 1);
  const int c = blockIdx.x;
  constexpr int U = 8;   // loads in flight per thread before the shared stores
  for (int e0 = threadIdx.x; e0 < kb * kb; e0 += U * blockDim.x) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int e = e0 + u * blockDim.x;
      v[u] = (e < kb * kb) ? T[(e % kb) + (size_t)(e / kb) * ldt] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int e = e0 + u * blockDim.x;
      if (e < kb * kb) ts[(e / kb) * (kb + 1) + e % kb] = v[u];
    }
  }
  for (int l = threadIdx.x; l < kb; l += blockDim.x) zc[l] = Z[l + (size_t)c * kb];
  __syncthreads();
  for (int a = threadIdx.x; a < kb; a += blockDim.x) {
    double s = 0.0;
    for (int l = 0; l <= a; l++) s += ts[a * (kb + 1) + l] * zc[l];   // (T^T)_{a l} = T_{l a}
    Mb[a + (size_t)c * kb] = s;
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
static constexpr int kSymmMaxSplit = 6, kSymmNsm = 148;
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
  w.cqr = ar.take<double>(3 * (size_t)b * b + b + 2);
  w.gbar = ar.take<unsigned>(64);
  w.Ycol = ar.take<double>((size_t)std::max(P, kSymmMaxSplit) * ldn * b);
}

static int panel_grid(int64_t m, int nsm) {
  int64_t g = (m + 63) / 64;   // at least 64 rows per CTA
  if (const char* v = getenv("SKEWEIG_PANEL_G")) nsm = std::max(1, std::min(nsm, atoi(v)));   // experiments
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
  a.gbar = w.gbar;
  int G = panel_grid(m, nsm);
  a.R = (m + G - 1) / G;
  size_t extra = (size_t)(8 * (b + 1) + (b + 1) + b + 4) * sizeof(double);
  const size_t tbuild = (size_t)2 * b * (b + 1) * sizeof(double);   // CTA 0's G and T in the T build
  size_t smem_full = std::max((size_t)b * a.R * sizeof(double), tbuild) + extra;
  bool use_smem = (size_t)b * a.R * sizeof(double) + extra <= 200 * 1024;
  if (!use_smem) extra = std::max(extra, tbuild);
  a.smem_rows = use_smem ? (int)a.R : 0;
  void* args[] = {&a};
  cudaError_t e = cudaMemsetAsync(w.gbar, 0, sizeof(unsigned), st);
  if (e) return e;
  KScope ks(KC_PANEL, st);
  // CholeskyQR2 + reconstruction when CTA 0 holds the top b rows and the rows fit in smem
  // (its own grid: floor(m/b) CTAs at most, so that every CTA -- CTA 0 in particular --
  // holds >= b rows)
  const int Gc = (int)std::max<int64_t>(1, std::min<int64_t>(m / b, nsm));
  const int64_t Rc = (m + Gc - 1) / Gc;
  const size_t cqr_smem = ((size_t)b * (Rc | 1) + 2 * (size_t)b * (b + 1) + 2 * b + 4) * sizeof(double);
  const char* hh = getenv("SKEWEIG_PANEL_HH");   // experiments: force the Householder panel
  if (b == 64 && m >= b && Rc >= b && cqr_smem <= 200 * 1024 && (size_t)b * Rc * sizeof(double) + extra <= 200 * 1024 &&
      !(hh && hh[0] == '1')) {
    e = set_smem_attr((const void*)panel_cqr_kernel<64>, 200 * 1024 + (int)extra);
    if (e) return e;
    CqrArgs ca;
    ca.p = a;
    ca.p.R = Rc;
    ca.p.smem_rows = (int)Rc;
    ca.scr = w.cqr;
    ca.dbg = nullptr;
    void* cargs[] = {&ca};
    // smem: the CholQR layout, or the Householder fallback's (same grid, Rc rows per CTA)
    const size_t sm_c = std::max(cqr_smem, std::max((size_t)b * Rc * sizeof(double), tbuild) + extra);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, panel_cqr_kernel<64>, 256, sm_c);
    if (occ * nsm >= Gc) {
      e = cudaLaunchCooperativeKernel((void*)panel_cqr_kernel<64>, dim3(Gc), dim3(256), cargs, sm_c, st);
      return e;
    }
  }
  if (use_smem) {
    e = set_smem_attr((const void*)panel_qr_kernel<true>, 200 * 1024 + (int)extra);
    if (e) return e;
    e = cudaLaunchCooperativeKernel((void*)panel_qr_kernel<true>, dim3(G), dim3(256), args, smem_full, st);
  } else {
    e = set_smem_attr((const void*)panel_qr_kernel<false>, (int)extra);
    if (e) return e;
    e = cudaLaunchCooperativeKernel((void*)panel_qr_kernel<false>, dim3(G), dim3(256), args, extra, st);
  }
  return e;
}

// single-device skew-SYMM X = S U on the TMA-fed persistent kernel (128-row blocks, equal
// units, split-K pieces summed in a fixed order); cudaErrorNotSupported -> caller falls back
static cudaError_t symm_tma(const double* S, int64_t lds, const double* U, int64_t ldu, double* X, int64_t ldx,
                            int64_t m, double* Ycol, int nsm, cudaStream_t st) {
  constexpr int BM = 128, BK = 16;
  using Cfg = SymmTma<BM, BK>;
  if (m < 1 || !tma_ptr_ok(S, lds) || !tma_ptr_ok(U, ldu) || tma_encode_fn() == nullptr) return cudaErrorNotSupported;
  CUtensorMap mR, mC, mU;
  if (!tma_map_2d(&mR, S, m, m, lds, BM + 4, BK) || !tma_map_2d(&mC, S, m, m, lds, BK + 4, BM) ||
      !tma_map_2d(&mU, U, m, 64, ldu, BK + 4, 64))
    return cudaErrorNotSupported;
  const int64_t nt = (m + BM - 1) / BM;
  // pieces per row block: best wave efficiency (units / (waves * SMs)), small cost per piece
  int split = 1;
  double best = -1e300;
  for (int c = 1; c <= kSymmMaxSplit; c++) {
    const int64_t units = nt * c;
    const int64_t waves = (units + nsm - 1) / nsm;
    const double eff = (double)units / (double)(waves * nsm) - 0.01 * (c - 1);
    if (eff > best + 1e-12) { best = eff; split = c; }
  }
  SymmTmaArgs a;
  a.m = m; a.nt = nt; a.split = split;
  a.out = split > 1 ? Ycol : X;
  a.ldo = split > 1 ? ldx : ldx;
  cudaError_t e = set_smem_attr((const void*)symm_tma_kernel<BM, BK>, (int)Cfg::SMEM);
  if (e) return e;
  KScope ks(KC_SYMM, st, split > 1 ? 2 : 1);
  const int grid = (int)std::min<int64_t>(nt * split, nsm);
  symm_tma_kernel<BM, BK><<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(mR, mC, mU, a);
  e = cudaGetLastError();
  if (e) return e;
  if (split > 1) {
    dim3 cg((unsigned)std::min<int64_t>((m + 255) / 256, 64), 64u);
    symm_sum_kernel<<<cg, 256, 0, st>>>(X, ldx, Ycol, ldx, split, m);
    e = cudaGetLastError();
  }
  return e;
}

cudaError_t f2b_update(const F2BLayout& L, int64_t j, double* A, int64_t lda, double* vstore, const F2BWork& w,
                       int nsm, cudaStream_t st, const Dist& d, int* nccl_err) {
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
  bool symm_done = false;
  if (d.P == 1 && b == 64 && !tma_disabled()) {   // X = S U -> P[:, b:2b], TMA-fed persistent kernel
    e = symm_tma(S, lda, w.U, ldn, Wp, ldn, m, w.Ycol, nsm, st);
    if (e == cudaSuccess) symm_done = true;
    else if (e != cudaErrorNotSupported) return e;
  }
  if (!symm_done) {   // X = S U  -> P[:, b:2b]
    SymmArgs s;
    s.S = S; s.lds = lda; s.U = w.U; s.ldu = ldn; s.X = Wp; s.ldx = ldn; s.m = m; s.nb = b;
    s.vec = gemm_vec_ok(S, lda, w.U, ldn) ? 1 : 0;
    s.P = d.P; s.qoff = qoff;
    using TR = GemmTile<kSymmBM, 64, kSymmBK, 32, 32, kSymmStages, false, false>;
    using TC = GemmTile<kSymmBM, 64, kSymmBK, 32, 32, kSymmStages, true, false>;
    size_t smem = std::max(TR::SMEM_BYTES, TC::SMEM_BYTES);
    e = set_smem_attr((const void*)symm_kernel<kSymmBM, 64, kSymmBK, kSymmStages>, (int)smem);
    if (e) return e;
    const int64_t nt = (m + kSymmBM - 1) / kSymmBM;
    int64_t grid = nt;
    int split = 1;
    if (d.P == 1) {
      // split-K pieces per row block: minimise (max CTAs per SM) x (work per CTA) + combine
      double best = 1e300;
      for (int c = 1; c <= kSymmMaxSplit; c++) {
        const double t = (double)((nt * c + kSymmNsm - 1) / kSymmNsm) / c + 0.02 * (c > 1 ? c : 0);
        if (t < best - 1e-12) { best = t; split = c; }
      }
      if (const char* v = getenv("SKEWEIG_SYMM_SPLIT")) split = std::max(1, std::min(kSymmMaxSplit, atoi(v)));   // experiments
      if (split > 1) {
        s.split = split;
        s.Ycol = w.Ycol; s.ldy = ldn;
        grid = nt * split;
      }
    }
    if (d.P > 1) {
      s.nt = nt;
      s.nloc = (nt > qoff) ? (nt - qoff + d.P - 1) / d.P : 0;
      s.Ycol = w.Ycol; s.ldy = ldn;
      grid = nt + (int64_t)d.P * s.nloc;
    }
    KScope ks(KC_SYMM, st, (d.P > 1 || split > 1) ? 2 : 1);
    symm_kernel<kSymmBM, 64, kSymmBK, kSymmStages><<<(unsigned)grid, TR::NTHREADS, smem, st>>>(s);
    if (d.P > 1) {
      dim3 cg((unsigned)std::min<int64_t>((m + 255) / 256, 64), (unsigned)b);
      symm_combine_kernel<<<cg, 256, 0, st>>>(Wp, ldn, w.Ycol, ldn, d.P, m, b, kSymmBM, d.P, qoff);
    } else if (split > 1) {
      dim3 cg((unsigned)std::min<int64_t>((m + 255) / 256, 64), (unsigned)b);
      symm_sum_kernel<<<cg, 256, 0, st>>>(Wp, ldn, w.Ycol, ldn, split, m);
    }
  }
  if (d.P > 1) {   // Y = sum over ranks of the partial skew-SYMM products (NVLink allreduce)
    KScope ks(KC_COLL, st);
    const int r = coll_allreduce_sum(d, Wp, (size_t)ldn * b, st);
    if (r) { *nccl_err = r; return cudaErrorUnknown; }
  }
  {   // W = X - 1/2 V (T^T (V^T X));  P = [V W], Q = [W -V]
    KScope ks(KC_WCORR, st, 5);
    const int nchunk = (int)((m + kWRows - 1) / kWRows);
    using TV = GemmTile<64, 64, 16, 32, 32, 2, true, false>;
    vtx_partial_kernel<16><<<nchunk, 128, TV::SMEM_BYTES, st>>>(Vj, ldv, Wp, ldn, m, kWRows, w.zpart);
    double* Zr = w.zpart + (size_t)nchunk * b * b;
    zsum_kernel<<<(b * b + 255) / 256, 256, 0, st>>>(w.zpart, nchunk, b * b, Zr);
    mb_kernel<<<b, 256, (size_t)(b * (b + 1) + b) * sizeof(double), st>>>(Zr, Tj, b, b, w.Mb);
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
  const bool lookahead = d.P > 1 && d.aux && qoff == 0 && j + 1 < L.npanel;   // this rank owns panel j+1
  if (lookahead) {
    // look-ahead: column block j+1 (tile column 0) first, then panel j+1 on the aux stream
    // while this stream updates the remaining local column blocks (disjoint columns)
    const int64_t ntm = (m + 63) / 64;
    GemmArgs g0 = ga;
    g0.col_off = 0; g0.col_stride = (int)(ntm + 1);   // tile column 0 only
    {
      KScope ks(KC_R2K, st);
      e = tma_disabled() ? cudaErrorNotSupported : tma_gemm<128, 64, 32, 3, false, true, true, true>(g0, nsm, st);
      if (e == cudaErrorNotSupported) e = gemm_dmma<64, 64, 16, 32, 32, 2, false, true, true>(g0, st);
    }
    if (e) return e;
    e = cudaEventRecord(d.ev_cols, st);
    if (e) return e;
    e = cudaStreamWaitEvent(d.aux, d.ev_cols, 0);
    if (e) return e;
    e = f2b_panel(L, j + 1, A, lda, vstore, w, nsm, d.aux);
    if (e) return e;
    e = cudaEventRecord(d.ev_panel, d.aux);
    if (e) return e;
    ga.col_off = d.P;   // the other local column blocks: tn = P, 2P, ...
  }
  {
    KScope ks(KC_R2K, st);
    e = cudaErrorNotSupported;
    if (!tma_disabled())   // persistent TMA-fed 128 x 64 tiles (the rank's column tiles when distributed)
      e = tma_gemm<128, 64, 32, 3, false, true, true, true>(ga, nsm, st);   // K = 128: 4 blocks of 32

    if (e == cudaErrorNotSupported) e = gemm_dmma<64, 64, 16, 32, 32, 2, false, true, true>(ga, st);
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
      if (j > 0 && d.P > 1 && d.aux) {   // factored during step j-1 (look-ahead)
        e = cudaStreamWaitEvent(st, d.ev_panel, 0);
      } else {
        e = f2b_panel(L, j, A, lda, vstore, w, nsm, st);
      }
      if (e) return e;
    }
    if (d.P > 1) {
      const int64_t g = j / L.merge, pl = j % L.merge;
      double* Vcols = vstore + L.goff[g] + pl * (int64_t)L.b * L.gld[g];   // the panel's columns of the group block
      KScope ks(KC_COLL, st);
      int r = coll_group_start(d);
      if (!r) r = coll_bcast(d, Vcols, sizeof(double) * (size_t)L.gld[g] * L.b, owner, st);
      if (!r) r = coll_bcast(d, w.T + j * (int64_t)L.b * L.b, sizeof(double) * (size_t)L.b * L.b, owner, st);
      if (!r) r = coll_bcast(d, w.tau + j * L.b, sizeof(double) * (size_t)L.b, owner, st);
      const int r2 = coll_group_end(d);
      if (r || r2) { *nccl_err = r ? r : r2; return cudaErrorUnknown; }
    }
    e = f2b_update(L, j, A, lda, vstore, w, nsm, st, d, nccl_err);
    if (e) return e;
  }
  return cudaSuccess;
}

}  // namespace sk
