// b2t.cu -- band -> tridiagonal bulge chasing (a support stage) and
// the BT2 back-transformation with the bulge reflectors (a9, hot path).
//
// Bulge chasing: sweep s eliminates column s below the
// subdiagonal with a reflector on rows s+1..s+b (task t = 0), and chases the fill it
// creates: task t >= 1 eliminates the first column of the bulge, rows
// r = s+1+t*b .. r+b-1.  Each task applies its reflector H = I - tau v v^T
//   left  to the block rows [r, r+L) x cols [col, r)        (col = previous block start)
//   two-sided to the skew diagonal block D (skew rank-2: D + v w^T - w v^T, w = tau D v,
//             the skew-SYMV/SYR2 kernels of PAPER.md:458-462)
//   right to the block below rows [r+L, r+L+b) x cols [r, r+L).
// The band is kept in lower band storage with 2b+2 rows (the bulge reaches 2b-1).
// Sweeps run concurrently on a persistent cooperative grid: sweep s+1 starts task t
// once sweep s has finished task t+3 (their index ranges are then disjoint).
//
// BT2 (Algorithm 1 step 4): X <- Q2 X.  The reflectors of k
// consecutive sweeps at one chase position t form G = H_s0 ... H_{s0+k-1} = I - V T V^T
// with a (b+k-1) x k staircase V; applying the sweep blocks last->first and t
// ascending within a block reproduces the sequential product exactly (reflectors of
// one sweep act on disjoint rows).
#include "common.cuh"
#include "internal.h"
#include <cooperative_groups.h>
#include <vector>
#include <algorithm>

namespace cg = cooperative_groups;

namespace sk {

struct ChaseArgs {
  double* AB; int64_t ldab;     // lower band storage, ldab >= 2b+2
  int64_t n; int b; int k2;     // band width, sweeps per BT2 group
  int* progress;                // [n] tasks completed per sweep
  double* qv;                   // reflector store: [group][k2][b]
  double* qtau;                 // [group][k2]
  const int64_t* gofs;          // [nblk] first group index of each sweep block
};

__device__ __forceinline__ int64_t chase_ntask(int64_t n, int b, int64_t s) { return 1 + (n - 3 - s) / b; }

template <int MAXB>
__global__ void __launch_bounds__(256) chase_kernel(ChaseArgs a) {
  extern __shared__ __align__(16) double W[];     // window [2b cols][LDW]
  __shared__ double vs[MAXB], ws[MAXB], zs[MAXB], sc[4];
  const int b = a.b;
  const int LDW = 2 * b + 2;
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t s = blockIdx.x; s < n - 2; s += gridDim.x) {
    const int64_t nt = chase_ntask(n, b, s);
    const int64_t ntprev = (s > 0) ? chase_ntask(n, b, s - 1) : 0;
    for (int64_t t = 0; t < nt; t++) {
      // ---- wait for the previous sweep to be 4 tasks ahead (or finished)
      if (s > 0) {
        if (tid == 0) {
          const int need = (int)smin<int64_t>(t + 4, ntprev);
          volatile int* pr = a.progress + (s - 1);
          while (*pr < need) { __nanosleep(64); }
          __threadfence();
        }
        __syncthreads();
      }
      int64_t col, r, L;
      if (t == 0) { col = s; r = s + 1; L = smin<int64_t>(b, n - 1 - s); }
      else { col = s + 1 + (t - 1) * b; r = col + b; L = smin<int64_t>(b, n - r); }
      const int64_t e = smin<int64_t>(n, r + L + b);
      const int ncol = (int)(r + L - col);
      // ---- load the touched entries: col c < r: rows [r, r+L); c >= r: rows [c, e)
      for (int cc = warp; cc < ncol; cc += 8) {
        int64_t c = col + cc;
        int64_t lo = (c < r) ? r : c, hi = (c < r) ? r + L : e;
        for (int64_t i = lo + lane; i < hi; i += 32) W[cc * LDW + (i - c)] = __ldcg(&a.AB[(i - c) + c * a.ldab]);
      }
      __syncthreads();
      // ---- (a) Householder of x = A[r:r+L, col]  (dlarfg convention)
      const int cx = 0;   // local column of col
      if (warp == 0) {
        double s2 = 0.0;
        for (int i = 1 + lane; i < L; i += 32) { double x = W[cx * LDW + (r + i - col)]; s2 += x * x; }
        s2 = warp_sum(s2);
        double x0 = W[cx * LDW + (r - col)];
        double beta, tau, scal;
        if (s2 == 0.0) { beta = x0; tau = 0.0; scal = 0.0; }
        else {
          double nrm = sqrt(x0 * x0 + s2);
          beta = (x0 >= 0.0) ? -nrm : nrm;
          tau = (beta - x0) / beta;
          scal = 1.0 / (x0 - beta);
        }
        for (int i = lane; i < L; i += 32) {
          double v = (i == 0) ? 1.0 : W[cx * LDW + (r + i - col)] * scal;
          vs[i] = v;
          W[cx * LDW + (r + i - col)] = (i == 0) ? beta : 0.0;
        }
        if (lane == 0) sc[0] = tau;
      }
      __syncthreads();
      const double tau = sc[0];
      // ---- store the reflector (v zero-padded to b by the initial memset)
      {
        const int64_t blk = s / a.k2, c = s % a.k2;
        const int64_t gidx = a.gofs[blk] + t;
        double* dst = a.qv + (gidx * a.k2 + c) * b;
        for (int i = tid; i < L; i += 256) dst[i] = vs[i];
        if (tid == 0) a.qtau[gidx * a.k2 + c] = tau;
      }
      if (tau != 0.0) {
        // ---- (b) left block: columns (col, r) (t >= 1): y = v^T A[r:r+L, c]; A -= tau v y
        for (int cc = 1 + warp; cc < (int)(r - col); cc += 8) {
          const int64_t c = col + cc;
          double y = 0.0;
          for (int i = lane; i < L; i += 32) y += vs[i] * W[cc * LDW + (r + i - c)];
          y = warp_sum(y) * tau;
          for (int i = lane; i < L; i += 32) W[cc * LDW + (r + i - c)] -= y * vs[i];
        }
        // ---- (c1) w = tau * D v, D = A[r:r+L, r:r+L] skew from its lower triangle
        const int dc = (int)(r - col);   // local column of r
        for (int i = tid; i < L; i += 256) {
          double sacc = 0.0;
          for (int j = 0; j < i; j++) sacc += W[(dc + j) * LDW + (i - j)] * vs[j];      // D_ij, i > j
          for (int j = i + 1; j < L; j++) sacc -= W[(dc + i) * LDW + (j - i)] * vs[j];  // -D_ji
          ws[i] = tau * sacc;
        }
        // ---- (d1) z = E v, E = A[r+L:e, r:r+L]
        const int ne = (int)(e - r - L);
        for (int i = tid; i < ne; i += 256) {
          double sacc = 0.0;
          for (int j = 0; j < L; j++) sacc += W[(dc + j) * LDW + (L + i - j)] * vs[j];
          zs[i] = tau * sacc;
        }
        __syncthreads();
        // ---- (c2) D_ij += v_i w_j - w_i v_j (i > j);  (d2) E_ij -= z_i v_j
        for (int e2 = tid; e2 < L * L; e2 += 256) {
          int i = e2 % L, j = e2 / L;
          if (i > j) W[(dc + j) * LDW + (i - j)] += vs[i] * ws[j] - ws[i] * vs[j];
        }
        for (int e2 = tid; e2 < ne * L; e2 += 256) {
          int i = e2 % ne, j = e2 / ne;
          W[(dc + j) * LDW + (L + i - j)] -= zs[i] * vs[j];
        }
      }
      __syncthreads();
      // ---- write back the touched entries
      for (int cc = warp; cc < ncol; cc += 8) {
        int64_t c = col + cc;
        int64_t lo = (c < r) ? r : c, hi = (c < r) ? r + L : e;
        for (int64_t i = lo + lane; i < hi; i += 32) __stcg(&a.AB[(i - c) + c * a.ldab], W[cc * LDW + (i - c)]);
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        volatile int* pr = a.progress + s;
        *pr = (int)(t + 1);
      }
    }
  }
}

// extract Lemma-1 alpha_k = -T[k+1, k] from the final band
__global__ void alpha_from_band_kernel(const double* AB, int64_t ldab, int64_t n, double* alpha) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n - 1) alpha[k] = -AB[1 + k * ldab];
}

// band from the F2B output A (A[c+d, c], d <= b) into AB (ldab rows, zero beyond b)
__global__ void band_extract_kernel(const double* A, int64_t lda, int64_t n, int b, double* AB, int64_t ldab) {
  int64_t c = blockIdx.x;
  for (int d = threadIdx.x; d < ldab; d += blockDim.x) {
    double v = 0.0;
    if (d >= 1 && d <= b && c + d < n) v = A[SK_IDX(c + d, c, lda)];
    AB[d + c * ldab] = v;
  }
}
// band from caller lower band storage (ldab_in rows, d <= b)
__global__ void band_copy_kernel(const double* ABin, int64_t ldin, int64_t n, int b, double* AB, int64_t ldab) {
  int64_t c = blockIdx.x;
  for (int d = threadIdx.x; d < ldab; d += blockDim.x) {
    double v = 0.0;
    if (d >= 1 && d <= b && c + d < n) v = ABin[d + c * ldin];
    AB[d + c * ldab] = v;
  }
}

// ------------------------------------------------------------------------------------
// BT2 group prep: for group g (reflectors of sweeps s0..s0+K2-1 at chase position t) build
// the dense staircase V (window rows rho = 0..RW-1 start at row s0 + t*b, reflector c at rows
// rho = c+1 .. c+b), its forward compact-WY T (Q_g = I - V T V^T, dlarft from the Gram
// matrix) and U = V T^T, stored as Ud[g][c][rho] (so that Q_g X = X - V (U^T X)).
template <int K2, int RW>
__global__ void __launch_bounds__(128) bt2_prep_kernel(const double* qv, const double* qtau, int64_t ngroups, int b,
                                                      double* Ud) {
  __shared__ double V[K2][RW];
  __shared__ double G[K2][K2 + 1];
  __shared__ double T[K2][K2 + 1];
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    for (int e = threadIdx.x; e < K2 * RW; e += blockDim.x) (&V[0][0])[e] = 0.0;
    __syncthreads();
    const double* v = qv + g * K2 * b;
    for (int e = threadIdx.x; e < K2 * b; e += blockDim.x) {
      int c = e / b, d = e % b;
      V[c][c + 1 + d] = v[e];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < K2 * K2; e += blockDim.x) {
      int c = e % K2, c2 = e / K2;
      double s = 0.0;
      if (c < c2)
        for (int r = c2 + 1; r <= c + b && r < RW; r++) s += V[c][r] * V[c2][r];
      G[c][c2] = s;
    }
    __syncthreads();
    const double* tau = qtau + g * K2;
    for (int r = threadIdx.x; r < K2; r += blockDim.x) {
      for (int c = 0; c < K2; c++) T[r][c] = 0.0;
      T[r][r] = tau[r];
      for (int c = r + 1; c < K2; c++) {
        double s = 0.0;
        for (int l = r; l < c; l++) s += T[r][l] * G[l][c];
        T[r][c] = -tau[c] * s;
      }
    }
    __syncthreads();
    double* U = Ud + g * K2 * RW;
    for (int e = threadIdx.x; e < K2 * RW; e += blockDim.x) {
      int c = e / RW, rho = e % RW;
      double s = 0.0;
      for (int c2 = c; c2 < K2; c2++) s += V[c2][rho] * T[c][c2];
      U[e] = s;
    }
    __syncthreads();
  }
}

// BT2 apply: one CTA per strip of NB columns of X, persistent over all groups in the
// order sweep blocks last -> first, t ascending.  The RW-row window
// X[W0 : W0+RW, strip] (W0 = s0 + t*b) lives in a RING-row shared-memory ring: step t+1
// reuses the last RW-b rows of window t, so per step only b new rows are loaded (cp.async,
// prefetched during step t) and b rows are written back.  The next group's V (packed
// staircase) and U are prefetched into a second buffer.  Per step:
//   Z = U^T Xw   (K2 x NB, DMMA, skip U's zero upper triangle)
//   Xw -= V Z    (RW x NB, DMMA, skip the staircase's zero fragments)
template <int NB, int K2, int RW, int RING, int BB>
struct BT2Cfg {
  static constexpr int LDX = RING + 4;   // Xs[col][slot]
  static constexpr int LDU = RW + 4;     // Us[c][rho]
  static constexpr int LDV = BB + 4;     // Vs[c][d]  (packed staircase, d = rho - c - 1)
  static constexpr int LDZ = K2 + 4;     // Zs[col][c]
  static constexpr int XS = NB * LDX, US = K2 * LDU, VS = K2 * LDV, ZS = NB * LDZ;
  static constexpr size_t SMEM = (size_t)(XS + 2 * US + 2 * VS + ZS) * sizeof(double);
  static_assert(LDX % 16 == 4 && LDU % 16 == 4 && LDZ % 16 == 4, "pad");
  static_assert(RING % 64 == 0 && RW % 8 == 0 && RING >= RW + BB, "ring");
};

template <int NB, int K2, int RW, int RING, int BB>
__global__ void __launch_bounds__(256, 1) bt2_apply_kernel(double* __restrict__ X, int64_t ldx, int64_t ncols,
                                                          int64_t n, const double* __restrict__ qv,
                                                          const double* __restrict__ Ud,
                                                          const int64_t* __restrict__ gofs, int64_t nblk) {
  using C = BT2Cfg<NB, K2, RW, RING, BB>;
  extern __shared__ __align__(16) double sh[];
  double* Xs = sh;
  double* Us0 = Xs + C::XS;
  double* Vs0 = Us0 + 2 * C::US;
  double* Zs = Vs0 + 2 * C::VS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int64_t col0 = (int64_t)blockIdx.x * NB;
  const int ncl = (int)smin<int64_t>(NB, ncols - col0);
  const bool vec = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);

  // async loads -------------------------------------------------------------------
  auto load_group = [&](int64_t g, int buf) {   // U (K2 x RW) and packed V (K2 x BB)
    double* Us = Us0 + buf * C::US;
    double* Vs = Vs0 + buf * C::VS;
    const double* u = Ud + g * K2 * RW;
    const double* v = qv + g * K2 * BB;
    for (int e = tid; e < K2 * RW / 2; e += 256) {
      int c = e / (RW / 2), r = (e % (RW / 2)) * 2;
      cp_async16(Us + c * C::LDU + r, u + c * RW + r, 16);
    }
    for (int e = tid; e < K2 * BB / 2; e += 256) {
      int c = e / (BB / 2), d = (e % (BB / 2)) * 2;
      cp_async16(Vs + c * C::LDV + d, v + c * BB + d, 16);
    }
  };
  auto load_rows = [&](int64_t r0, int nrows, int slot0) {   // rows [r0, r0+nrows) -> ring slots slot0..
    for (int e = tid; e < NB * nrows / 2; e += 256) {
      int cl = e / (nrows / 2), rr = (e % (nrows / 2)) * 2;
      int slot = slot0 + rr;
      if (slot >= RING) slot -= RING;
      int64_t r = r0 + rr;
      double* dst = Xs + cl * C::LDX + slot;
      const double* src = X + SK_IDX(r, col0 + cl, ldx);
      int cnt = (cl < ncl) ? (int)smin<int64_t>(2, smax<int64_t>(0, n - r)) : 0;
      if (vec) {
        cp_async16(dst, cnt ? src : X, cnt * 8);
      } else {
        cp_async8(dst, cnt > 0 ? src : X, cnt > 0 ? 8 : 0);
        cp_async8(dst + 1, cnt > 1 ? src + 1 : X, cnt > 1 ? 8 : 0);
      }
    }
  };
  auto store_rows = [&](int64_t r0, int nrows, int slot0) {
    for (int e = tid; e < NB * nrows; e += 256) {
      int cl = e / nrows, rr = e % nrows;
      int slot = slot0 + rr;
      if (slot >= RING) slot -= RING;
      int64_t r = r0 + rr;
      if (cl < ncl && r < n) X[SK_IDX(r, col0 + cl, ldx)] = Xs[cl * C::LDX + slot];
    }
  };

  int buf = 0;
  if (nblk <= 0) return;
  {
    const int64_t blk = nblk - 1;
    load_group(gofs[blk], 0);
    load_rows(blk * K2, RW, 0);
    cp_async_commit();
  }
  for (int64_t blk = nblk - 1; blk >= 0; blk--) {
    const int64_t s0 = blk * K2;
    const int64_t ntask = 1 + (n - 3 - s0) / BB;
    for (int64_t t = 0; t < ntask; t++) {
      const int64_t W0 = s0 + t * BB;
      const int off = (int)((t * BB) % RING);
      cp_async_wait<0>();
      __syncthreads();
      // ---- prefetch the next group (and the next rows of the window, same block)
      if (t + 1 < ntask) {
        load_group(gofs[blk] + t + 1, buf ^ 1);
        int so = off + RW;
        if (so >= RING) so -= RING;
        load_rows(W0 + RW, BB, so);
      } else if (blk > 0) {
        load_group(gofs[blk - 1], buf ^ 1);
      }
      cp_async_commit();
      const double* Us = Us0 + buf * C::US;
      const double* Vs = Vs0 + buf * C::VS;
      // ---- Z = U^T Xw : M = K2 (c), N = NB (col), K = RW (rho); warps 4 (M) x 2 (N)
      {
        constexpr int FN = NB / 16;
        const int m0 = (warp & 3) * 8, n0 = (warp >> 2) * (NB / 2);
        double acc[FN][2];
#pragma unroll
        for (int j = 0; j < FN; j++) acc[j][0] = acc[j][1] = 0.0;
        // U[rho][c] = 0 for rho <= c: k blocks with kk + 3 <= m0 are zero
#pragma unroll 4
        for (int kk = (m0 / 4) * 4; kk < RW; kk += 4) {
          double af = Us[(m0 + gq) * C::LDU + kk + tq];
          int slot = off + kk;
          if (slot >= RING) slot -= RING;
#pragma unroll
          for (int j = 0; j < FN; j++) {
            double bf = Xs[(n0 + 8 * j + gq) * C::LDX + slot + tq];
            dmma884(acc[j][0], acc[j][1], af, bf);
          }
        }
#pragma unroll
        for (int j = 0; j < FN; j++) {
          int nn = n0 + 8 * j + 2 * tq;
          Zs[nn * C::LDZ + m0 + gq] = acc[j][0];
          Zs[(nn + 1) * C::LDZ + m0 + gq] = acc[j][1];
        }
      }
      __syncthreads();
      // ---- Xw -= V Z : M = RW (rho), N = NB, K = K2 (c); warps 4 (M, RW/4 rows) x 2 (N)
      {
        constexpr int FM = RW / 32, FN = NB / 16;
        const int wm = warp & 3, n0 = (warp >> 2) * (NB / 2);
        double acc[FM][FN][2];
#pragma unroll
        for (int i = 0; i < FM; i++)
#pragma unroll
          for (int j = 0; j < FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < K2; kk += 4) {
          double bf[FN];
#pragma unroll
          for (int j = 0; j < FN; j++) bf[j] = Zs[(n0 + 8 * j + gq) * C::LDZ + kk + tq];
#pragma unroll
          for (int i = 0; i < FM; i++) {
            const int m0 = wm * (RW / 4) + 8 * i;
            // staircase: V[rho][c] != 0 iff 1 <= rho - c <= BB
            if (m0 + 7 - kk < 1 || m0 - (kk + 3) > BB) continue;
            const int rho = m0 + gq, c = kk + tq;
            const int d = rho - c - 1;
            double af = (d >= 0 && d < BB) ? Vs[c * C::LDV + d] : 0.0;
#pragma unroll
            for (int j = 0; j < FN; j++) dmma884(acc[i][j][0], acc[i][j][1], af, bf[j]);
          }
        }
#pragma unroll
        for (int i = 0; i < FM; i++) {
          const int m0 = wm * (RW / 4) + 8 * i;
          int slot = off + m0;
          if (slot >= RING) slot -= RING;
#pragma unroll
          for (int j = 0; j < FN; j++) {
            int nn = n0 + 8 * j + 2 * tq;
            Xs[nn * C::LDX + slot + gq] -= acc[i][j][0];
            Xs[(nn + 1) * C::LDX + slot + gq] -= acc[i][j][1];
          }
        }
      }
      __syncthreads();
      // ---- write back the rows leaving the window
      if (t + 1 < ntask) {
        store_rows(W0, BB, off);
      } else {
        store_rows(W0, RW, off);
        __syncthreads();
        if (blk > 0) load_rows((blk - 1) * K2, RW, 0);   // first window of the next block
        cp_async_commit();
      }
      buf ^= 1;
    }
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------
// Host side
void B2TLayout::init(int64_t n_, int b_, int k2_) {
  n = n_; b = b_; k2 = k2_;
  ldab = 2 * b + 2;
  nblk = (n > 2) ? (n - 2 + k2 - 1) / k2 : 0;
  gofs.assign(nblk, 0);
  int64_t g = 0;
  for (int64_t blk = 0; blk < nblk; blk++) {
    gofs[blk] = g;
    g += 1 + (n - 3 - blk * k2) / b;
  }
  ngroups = g;
}

cudaError_t band_extract(const double* A, int64_t lda, int64_t n, int b, double* AB, int64_t ldab, cudaStream_t st) {
  KScope ks(KC_BAND, st);
  band_extract_kernel<<<(unsigned)std::max<int64_t>(n, 1), 128, 0, st>>>(A, lda, n, b, AB, ldab);
  return cudaGetLastError();
}
cudaError_t band_copy(const double* ABin, int64_t ldin, int64_t n, int b, double* AB, int64_t ldab, cudaStream_t st) {
  KScope ks(KC_BAND, st);
  band_copy_kernel<<<(unsigned)std::max<int64_t>(n, 1), 128, 0, st>>>(ABin, ldin, n, b, AB, ldab);
  return cudaGetLastError();
}


void b2t_reserve(Arena& ar, const B2TLayout& L, bool vectors, B2TWork& w) {
  w.AB = ar.take<double>((size_t)L.ldab * std::max<int64_t>(L.n, 1));
  w.progress = ar.take<int>(std::max<int64_t>(L.n, 1));
  int64_t ng = std::max<int64_t>(L.ngroups, 1);
  w.qv = ar.take<double>((size_t)ng * L.k2 * L.b);
  w.qtau = ar.take<double>((size_t)ng * L.k2);
  if (vectors) w.qT = ar.take<double>((size_t)ng * L.k2 * (L.b + L.k2));   // U_g (k2 x (b+k2)) per group
  w.gofs = ar.take<int64_t>(std::max<int64_t>(L.nblk, 1));
}

static int chase_grid(int64_t n, int b, int nsm) {
  // concurrently active sweeps ~ (n/b)/4; never more CTAs than can be co-resident
  int64_t act = std::max<int64_t>(1, (n / std::max(b, 1)) / 4 + 1);
  return (int)std::max<int64_t>(1, std::min<int64_t>(act, nsm));
}

// Run the chase on w.AB (already filled, ldab = 2b+2); writes alpha and reflectors.
cudaError_t b2t_run(const B2TLayout& L, B2TWork& w, double* alpha, int nsm, cudaStream_t st) {
  cudaError_t e;
  const int64_t n = L.n;
  KScope ks(KC_CHASE, st, n > 2 ? 2 : 1);
  if (n >= 2) {
    if (L.nblk > 0) {
      e = cudaMemcpyAsync(w.gofs, L.gofs.data(), sizeof(int64_t) * L.nblk, cudaMemcpyHostToDevice, st);
      if (e) return e;
    } else {
      cudaMemsetAsync(w.gofs, 0, sizeof(int64_t), st);
    }
    cudaMemsetAsync(w.progress, 0, sizeof(int) * n, st);
    cudaMemsetAsync(w.qv, 0, sizeof(double) * (size_t)std::max<int64_t>(L.ngroups, 1) * L.k2 * L.b, st);
    cudaMemsetAsync(w.qtau, 0, sizeof(double) * (size_t)std::max<int64_t>(L.ngroups, 1) * L.k2, st);
    if (n > 2) {
      ChaseArgs a;
      a.AB = w.AB; a.ldab = L.ldab; a.n = n; a.b = L.b; a.k2 = L.k2; a.progress = w.progress;
      a.qv = w.qv; a.qtau = w.qtau; a.gofs = w.gofs;
      int G = chase_grid(n, L.b, nsm);
      size_t smem = (size_t)2 * L.b * (2 * L.b + 2) * sizeof(double);
      e = cudaFuncSetAttribute(chase_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      void* args[] = {&a};
      e = cudaLaunchCooperativeKernel((void*)chase_kernel<128>, dim3(G), dim3(256), args, smem, st);
      if (e) return e;
    }
    alpha_from_band_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w.AB, L.ldab, n, alpha);
  }
  return cudaGetLastError();
}

cudaError_t bt2_run(const B2TLayout& L, B2TWork& w, double* X, int64_t ldx, int64_t ncols, cudaStream_t st) {
  if (L.n <= 2 || L.ngroups == 0 || ncols == 0) return cudaSuccess;
  cudaError_t e;
  constexpr int NB = 64, K2 = 32, RW = 96, RING = 192, BB = 64;
  if (L.k2 != K2 || L.b != BB) return cudaErrorInvalidValue;
  {
    KScope ks(KC_BT2_T, st);
    bt2_prep_kernel<K2, RW><<<(unsigned)std::min<int64_t>(L.ngroups, 8 * 148), 128, 0, st>>>(w.qv, w.qtau, L.ngroups,
                                                                                              BB, w.qT);
  }
  using Cf = BT2Cfg<NB, K2, RW, RING, BB>;
  e = cudaFuncSetAttribute(bt2_apply_kernel<NB, K2, RW, RING, BB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)Cf::SMEM);
  if (e) return e;
  KScope ks(KC_BT2, st);
  bt2_apply_kernel<NB, K2, RW, RING, BB><<<(unsigned)((ncols + NB - 1) / NB), 256, Cf::SMEM, st>>>(
      X, ldx, ncols, L.n, w.qv, w.qT, w.gofs, L.nblk);
  return cudaGetLastError();
}

}  // namespace sk
