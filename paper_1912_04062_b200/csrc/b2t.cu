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
// BT2 group compact-WY T (forward dlarft) from the staircase V_g: column c has its b
// entries at local rows c .. c+b-1.  Gram G[c][c'] (c < c') = sum_d v_c[c'-c+d] v_c'[d].
__global__ void bt2_tbuild_kernel(const double* qv, const double* qtau, int64_t ngroups, int k2, int b, double* qT) {
  extern __shared__ double sh[];
  double* G = sh;                 // k2 x k2
  double* V = sh + k2 * k2;       // k2 x b
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    const double* v = qv + g * k2 * b;
    for (int e = threadIdx.x; e < k2 * b; e += blockDim.x) V[e] = v[e];
    __syncthreads();
    for (int e = threadIdx.x; e < k2 * k2; e += blockDim.x) {
      int c = e % k2, c2 = e / k2;
      double s = 0.0;
      if (c < c2) {
        int off = c2 - c;
        for (int d = 0; d + off < b; d++) s += V[c * b + off + d] * V[c2 * b + d];
      }
      G[c + c2 * k2] = s;
    }
    __syncthreads();
    const double* tau = qtau + g * k2;
    double* T = qT + g * k2 * k2;
    for (int r = threadIdx.x; r < k2; r += blockDim.x) {
      double trow[64];
      for (int c = 0; c < k2; c++) trow[c] = 0.0;
      trow[r] = tau[r];
      for (int c = r + 1; c < k2; c++) {
        double s = 0.0;
        for (int l = r; l < c; l++) s += trow[l] * G[l + c * k2];
        trow[c] = -tau[c] * s;
      }
      for (int c = 0; c < k2; c++) T[r + c * k2] = trow[c];
    }
    __syncthreads();
  }
}

// BT2 apply: one CTA per column strip of X (NB columns); groups in order
// (sweep blocks last -> first, t ascending).  Per group:  Z = V^T Xw (DMMA),
// Z2 = T Z, Xw -= V Z2 (DMMA), Xw = X[R0 : R0+b+k2-1, strip].
template <int NB, int K2, int MAXROWS>
__global__ void __launch_bounds__(256) bt2_apply_kernel(double* X, int64_t ldx, int64_t ncols, int64_t n, int b,
                                                       const double* qv, const double* qT, const int64_t* gofs,
                                                       int64_t nblk) {
  constexpr int LDV = MAXROWS + 4;     // Vs[c][rho]
  constexpr int LDX = MAXROWS + 4;     // Xs[col][rho]
  constexpr int LDZ = K2 + 4;          // Zs[col][c]
  static_assert(LDV % 16 == 4 && LDZ % 16 == 4, "pad");
  extern __shared__ __align__(16) double sh[];
  double* Vs = sh;                         // K2 * LDV
  double* Ts = Vs + K2 * LDV;              // K2 * K2
  double* Xs = Ts + K2 * K2;               // NB * LDX
  double* Zs = Xs + NB * LDX;              // NB * LDZ
  double* Z2 = Zs + NB * LDZ;              // NB * LDZ
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int64_t col0 = (int64_t)blockIdx.x * NB;
  const int ncl = (int)smin<int64_t>(NB, ncols - col0);
  for (int64_t blk = nblk - 1; blk >= 0; blk--) {
    const int64_t s0 = blk * K2;
    const int64_t ntask = 1 + (n - 3 - s0) / b;
    for (int64_t t = 0; t < ntask; t++) {
      const int64_t g = gofs[blk] + t;
      const int64_t R0 = s0 + 1 + t * b;
      const int rows = (int)smin<int64_t>(b + K2 - 1, n - R0);
      // load V (staircase), T, X window
      for (int e = tid; e < K2 * MAXROWS; e += 256) {
        int c = e / MAXROWS, rho = e % MAXROWS;
        int d = rho - c;
        Vs[c * LDV + rho] = (d >= 0 && d < b && rho < rows) ? qv[(g * K2 + c) * b + d] : 0.0;
      }
      for (int e = tid; e < K2 * K2; e += 256) Ts[e] = qT[g * K2 * K2 + e];
      for (int e = tid; e < NB * MAXROWS; e += 256) {
        int cl = e / MAXROWS, rho = e % MAXROWS;
        Xs[cl * LDX + rho] = (cl < ncl && rho < rows) ? X[SK_IDX(R0 + rho, col0 + cl, ldx)] : 0.0;
      }
      __syncthreads();
      // Z = V^T Xw : M = K2, N = NB, K = MAXROWS.  warps: (K2/8) x (8/(K2/8)) grid
      {
        constexpr int WMR = K2 / 8;                 // warps along M (8-row tiles)
        constexpr int WNR = 8 / WMR;                // warps along N
        constexpr int FN = NB / (8 * WNR);
        const int wm = warp % WMR, wn = warp / WMR;
        double acc[FN][2];
#pragma unroll
        for (int j = 0; j < FN; j++) acc[j][0] = acc[j][1] = 0.0;
        for (int kk = 0; kk < MAXROWS; kk += 4) {
          double af = Vs[(wm * 8 + gq) * LDV + kk + tq];
#pragma unroll
          for (int j = 0; j < FN; j++) {
            double bf = Xs[(wn * FN * 8 + j * 8 + gq) * LDX + kk + tq];
            dmma884(acc[j][0], acc[j][1], af, bf);
          }
        }
#pragma unroll
        for (int j = 0; j < FN; j++) {
          int m = wm * 8 + gq, nn = wn * FN * 8 + j * 8 + 2 * tq;
          Zs[nn * LDZ + m] = acc[j][0];
          Zs[(nn + 1) * LDZ + m] = acc[j][1];
        }
      }
      __syncthreads();
      // Z2 = T Z  (T upper triangular)
      for (int e = tid; e < K2 * NB; e += 256) {
        int c = e % K2, cl = e / K2;
        double s = 0.0;
        for (int l = c; l < K2; l++) s += Ts[c + l * K2] * Zs[cl * LDZ + l];
        Z2[cl * LDZ + c] = s;
      }
      __syncthreads();
      // Xw -= V Z2 : M = MAXROWS, N = NB, K = K2; warps 4 (M) x 2 (N)
      {
        constexpr int FM = MAXROWS / 32;    // 8-row fragments per warp along M (4 warps)
        constexpr int FN = NB / 16;         // 2 warps along N
        const int wm = warp % 4, wn = warp / 4;
        double acc[FM][FN][2];
#pragma unroll
        for (int i = 0; i < FM; i++)
#pragma unroll
          for (int j = 0; j < FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < K2; kk += 4) {
          double af[FM], bf[FN];
#pragma unroll
          for (int i = 0; i < FM; i++) af[i] = Vs[(kk + tq) * LDV + wm * FM * 8 + i * 8 + gq];
#pragma unroll
          for (int j = 0; j < FN; j++) bf[j] = Z2[(wn * FN * 8 + j * 8 + gq) * LDZ + kk + tq];
#pragma unroll
          for (int i = 0; i < FM; i++)
#pragma unroll
            for (int j = 0; j < FN; j++) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
#pragma unroll
        for (int i = 0; i < FM; i++)
#pragma unroll
          for (int j = 0; j < FN; j++) {
            int m = wm * FM * 8 + i * 8 + gq, nn = wn * FN * 8 + j * 8 + 2 * tq;
            Xs[nn * LDX + m] -= acc[i][j][0];
            Xs[(nn + 1) * LDX + m] -= acc[i][j][1];
          }
      }
      __syncthreads();
      for (int e = tid; e < NB * MAXROWS; e += 256) {
        int cl = e / MAXROWS, rho = e % MAXROWS;
        if (cl < ncl && rho < rows) X[SK_IDX(R0 + rho, col0 + cl, ldx)] = Xs[cl * LDX + rho];
      }
      __syncthreads();
    }
  }
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
  if (vectors) w.qT = ar.take<double>((size_t)ng * L.k2 * L.k2);
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
  const int k2 = L.k2, b = L.b;
  {
  KScope ks(KC_BT2_T, st);
  bt2_tbuild_kernel<<<(unsigned)std::min<int64_t>(L.ngroups, 4096), 128, (size_t)(k2 * k2 + k2 * b) * 8, st>>>(
      w.qv, w.qtau, L.ngroups, k2, b, w.qT);
  }
  constexpr int NB = 64, K2 = 32, MAXROWS = 96;
  if (k2 != K2 || b + k2 - 1 > MAXROWS) return cudaErrorInvalidValue;
  size_t smem = (size_t)(K2 * (MAXROWS + 4) + K2 * K2 + NB * (MAXROWS + 4) + 2 * NB * (K2 + 4)) * 8;
  static bool set = false;
  if (!set) {
    e = cudaFuncSetAttribute(bt2_apply_kernel<NB, K2, MAXROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    set = true;
  }
  KScope ks(KC_BT2, st);
  bt2_apply_kernel<NB, K2, MAXROWS><<<(unsigned)((ncols + NB - 1) / NB), 256, smem, st>>>(X, ldx, ncols, L.n, b, w.qv,
                                                                                         w.qT, w.gofs, L.nblk);
  return cudaGetLastError();
}

}  // namespace sk
