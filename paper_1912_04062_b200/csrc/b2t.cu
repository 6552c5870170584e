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
// once sweep s has finished task t+1 (see the chase kernel for why lag 2 is enough).
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
#include <type_traits>
#include <algorithm>
#include <cstdlib>
#include <cstdio>

namespace cg = cooperative_groups;

namespace sk {

struct ChaseArgs {
  double* AB; int64_t ldab;     // lower band storage, ldab >= 2b+2
  int64_t n; int b; int k2;     // band width, sweeps per BT2 group
  int* progress;                // [n] tasks completed per sweep
  double* qv;                   // reflector store: [group][k2][b]
  double* qtau;                 // [group][k2]
  const int64_t* gofs;          // [nblk] first group index of each sweep block
  long long* dbg;               // optional instrumentation (SKEWEIG_CHASE_DBG)
};

__device__ __forceinline__ int64_t chase_ntask(int64_t n, int b, int64_t s) { return 1 + (n - 3 - s) / b; }

// Chase kernel.  Persistent cooperative grid, one sweep per CTA at a time, the tasks above
// in shared-memory column slots:
//  * Sweep s task t needs sweep s-1 tasks 0..t+1 complete (lag 2 instead of 3).  It shares
//    exactly one entry with s-1's task t+2: A(r', col'), r' = s+(t+2)b, col' = r'-b, which
//    task t+2's Householder overwrites with beta and never touches again; every other entry
//    of the two tasks is disjoint, as is s task t from sweep s-1 tasks >= t+3 and sweep s-2
//    tasks >= t+3 (checked exhaustively on access sets for small n, b and numerically
//    against the sequential order).  Each sweep computes the Householder of task t+1 as
//    soon as column 0 of task t's block below is final (during task t's update) and stores
//    beta to global memory before task t completes, so "s-1 tasks 0..t+1 complete" also
//    covers the shared entry.  The per-sweep critical chain is two tasks.
//  * 12 compute warps + 1 auxiliary warp.  Warp 0 polls and, in the update, takes only
//    diagonal column 0 and then the next Householder; the auxiliary warp publishes task
//    completion (fence + flag) and stores the next reflector while the compute warps go on
//    to the next task.  The diagonal and left blocks are final after the update and go from
//    registers straight to global memory; only the block below stays in shared memory
//    (task t+1's left block).
constexpr int kChaseCW = 12;                       // compute warps
constexpr int kChaseThreads = (kChaseCW + 1) * 32;   // + 1 auxiliary warp

template <int MAXB>
__global__ void __launch_bounds__(kChaseThreads, 1) chase_kernel(ChaseArgs a) {
  extern __shared__ __align__(16) double W[];
  __shared__ double vsb[2][MAXB];   // reflector of task t in vsb[t & 1], tau/beta in scb
  __shared__ double scb[2][2];
  __shared__ double red[2][3 * MAXB];
  __shared__ double uz[2 * MAXB], vv[2 * MAXB], yv[MAXB];
  __shared__ int dbase[MAXB], lbase[MAXB];
  const int b = a.b;
  const int LDW = 2 * b + 2, B2 = 2 * b;
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NCT = kChaseCW * 32;   // compute threads
  const bool prof = a.dbg != nullptr && blockIdx.x == 0 && tid == 0;
  long long t_wait = 0, t_work = 0, ntasks = 0, tk = 0, tph[5] = {0, 0, 0, 0, 0}, tp = 0;
#define C2_TS(i) do { if (prof) { long long _n = clock64(); tph[i] += _n - tp; tp = _n; } } while (0)
  for (int64_t s = blockIdx.x; s < n - 2; s += gridDim.x) {
    const int nt = (int)chase_ntask(n, b, s);
    const int ntprev = (s > 0) ? (int)chase_ntask(n, b, s - 1) : 0;
    const int64_t gbase = a.gofs[s / a.k2];
    const int cpos = (int)(s % a.k2);
    // task geometry: left column col, reflector rows [r, r+L), block rows [c, e)
    auto geom = [&](int t, int64_t& col, int64_t& r, int& L) {
      if (t == 0) { col = s; r = s + 1; L = (int)smin<int64_t>(b, n - 1 - s); }
      else { col = s + 1 + (int64_t)(t - 1) * b; r = col + b; L = (int)smin<int64_t>(b, n - r); }
    };
    // Householder of x = W[xoff + 0 .. L) (dlarfg convention) by one warp -> vsb[p], scb[p]
    auto house = [&](int xoff, int L, int p) {
      double s2 = 0.0;
      for (int i = 1 + lane; i < L; i += 32) { const double x = W[xoff + i]; s2 += x * x; }
      s2 = warp_sum(s2);
      const double x0 = W[xoff];
      double beta, tau, scal;
      if (s2 == 0.0) { beta = x0; tau = 0.0; scal = 0.0; }
      else {
        const double nrm = sqrt(x0 * x0 + s2);
        beta = (x0 >= 0.0) ? -nrm : nrm;
        tau = (beta - x0) / beta;
        scal = 1.0 / (x0 - beta);
      }
      for (int i = lane; i < L; i += 32) vsb[p][i] = (i == 0) ? 1.0 : W[xoff + i] * scal;
      if (lane == 0) { scb[p][0] = tau; scb[p][1] = beta; }
    };
    // final left column of task t (beta, 0, ...) and its reflector for BT2, by one warp
    auto store_col_refl = [&](int t) {
      int64_t col, r;
      int L;
      geom(t, col, r, L);
      const int p = t & 1;
      double* gp = a.AB + col * a.ldab + (r - col);
      const double beta = scb[p][1];
      for (int i = lane; i < L; i += 32) __stcg(&gp[i], i == 0 ? beta : 0.0);
      double* dst = a.qv + ((gbase + t) * a.k2 + cpos) * b;
      for (int i = lane; i < L; i += 32) dst[i] = vsb[p][i];
      if (lane == 0) a.qtau[(gbase + t) * a.k2 + cpos] = scb[p][0];
    };
    for (int t = 0; t < nt; t++) {
      int64_t col, r;
      int L;
      geom(t, col, r, L);
      const int64_t e = smin<int64_t>(n, r + L + b);
      const int nl = (int)(r - col);
      const int ne = (int)(e - r - L);
      const bool last = (t + 1 == nt);
      const int p = t & 1;
      const double* vs = vsb[p];
      const int sr0 = (int)((r - s - 1) % B2);
      const int sc0 = (t == 0) ? B2 : (int)((col - s - 1) % B2);
      auto sl_left = [&](int cc) -> int { if (t == 0) return B2; int x = sc0 + cc; return x >= B2 ? x - B2 : x; };
      auto sl_diag = [&](int j) -> int { int x = sr0 + j; return x >= B2 ? x - B2 : x; };
      if (warp < kChaseCW) {
        if (prof) tk = clock64();
        // ---- (1) dependency: sweep s-1 tasks 0..t+1 complete (warp 0 polls, whole warp)
        if (warp == 0 && s > 0) {
          const int need = min(t + 2, ntprev);
          const int* pr = a.progress + (s - 1);
          while (ld_acquire_gpu(pr) < need) { }
        }
        named_bar(1, NCT);
        if (prof) { long long now = clock64(); t_wait += now - tk; tk = now; tp = now; ntasks++; }
        // ---- (2) load the diagonal-block columns [r, r+L), rows [c, e) (t = 0: also column s)
        if (t == 0 && warp == 0) {
          const int d1 = (int)(r + L - col);
          for (int d = 2 * lane; d < d1; d += 64) cp_async16(&W[B2 * LDW + d], &a.AB[d + col * a.ldab], 16);
        }
        for (int j = warp; j < L; j += kChaseCW) {
          const int64_t c = r + j;
          const int d1 = (int)(e - c);
          const int sj = sl_diag(j);
          for (int d = 2 * lane; d < d1; d += 64) cp_async16(&W[sj * LDW + d], &a.AB[d + c * a.ldab], 16);
        }
        // smem offset tables: element (row i, diagonal column j) at dbase[j] + i, (row i,
        // left column cc) at lbase[cc] + i, block-relative rows
        if (tid < L) dbase[tid] = sl_diag(tid) * LDW - tid;
        else if (tid >= MAXB && tid - MAXB < nl) lbase[tid - MAXB] = sl_left(tid - MAXB) * LDW + nl - (tid - MAXB);
        cp_async_commit();
        cp_async_wait<0>();
        named_bar(1, NCT);
        if (t == 0) {   // first task of the sweep: its Householder needs column s
          if (warp == 0) { house(B2 * LDW + 1, L, p); __syncwarp(); store_col_refl(0); }
          named_bar(1, NCT);
        }
        C2_TS(0);
        const double tau = scb[p][0];
        // ---- (3) y = v^T (left block), w = D v (skew, lower storage), z = E v: one item per
        //      thread pair (every other j), four independent chains, branch-free bodies
        const int part = tid / (3 * MAXB), it = tid % (3 * MAXB);
        double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
        // dbase[j] computed in registers (no dependent shared load in the chains)
        auto colb = [&](int j) -> int { int x = sr0 + j; x = (x >= B2) ? x - B2 : x; return x * LDW - j; };
        auto dot4 = [&](auto&& f) {
          int j = part;
          for (; j + 6 < L; j += 8) { acc0 += f(j); acc1 += f(j + 2); acc2 += f(j + 4); acc3 += f(j + 6); }
          for (; j < L; j += 2) acc0 += f(j);
        };
        if (it < b) {
          const int cc = it;
          if (cc >= 1 && cc < nl) {
            const int base = lbase[cc];
            dot4([&](int i) { return vs[i] * W[base + i]; });
          }
        } else if (it < 2 * b) {
          const int i = it - b;
          if (i < L) {
            const int si = dbase[i];
            // w_i = sum_{j<i} D(i,j) v_j - sum_{j>i} D(j,i) v_j with the same j on every lane:
            // lower reads (row i) contiguous over lanes, upper reads (column i) at the odd
            // stride LDW-1; j == i reads the stored zero diagonal
            dot4([&](int j) {
              const bool lo = j < i;
              return W[lo ? colb(j) + i : si + j] * (lo ? vs[j] : -vs[j]);
            });
          }
        } else if (it < 3 * b) {
          const int i = it - 2 * b;
          if (i < ne) dot4([&](int j) { return W[colb(j) + L + i] * vs[j]; });
        }
        if (it < 3 * b) red[part][it] = (acc0 + acc1) + (acc2 + acc3);
        named_bar(1, NCT);
        // uz = [tau w (rows of D) | tau z (rows of E) | 0], vv = [v | 0], yv = tau y
        if (tid < 2 * b) {
          const int i = tid;
          uz[i] = (i < L) ? tau * (red[0][b + i] + red[1][b + i])
                          : (i - L < ne ? tau * (red[0][2 * b + i - L] + red[1][2 * b + i - L]) : 0.0);
          vv[i] = (i < L) ? vs[i] : 0.0;
        } else if (tid < 3 * b) {
          const int i = tid - 2 * b;
          yv[i] = tau * (red[0][i] + red[1][i]);
        }
        named_bar(1, NCT);
        C2_TS(1);
        // ---- (4) left block -= v y^T; D += v w^T - w v^T (lower); E -= z v^T.  Left and D
        //      are final: registers -> global.  E stays in smem (task t+1's left block).
        //      Lane owns rows lane + 32k (coefficients in registers); all loads first
        //      (in-slot, always safe), predicated stores.  Warp 0 does diagonal column 0
        //      only, then the Householder of task t+1 from that column's block-below part.
        const int ncl = nl - 1;
        const int iend = L + ne;
        double vr[2 * MAXB / 32], ur[2 * MAXB / 32];
#pragma unroll
        for (int k = 0; k < 2 * MAXB / 32; k++) { vr[k] = vv[lane + 32 * k]; ur[k] = uz[lane + 32 * k]; }
        double* const gd0 = a.AB + r * a.ldab;   // + j*(ldab-1): diagonal of column r+j
        const int ldm1 = (int)a.ldab - 1;
        auto diag_cols = [&](int j0, int j1, bool h1) {
          const int b0 = dbase[j0], b1 = dbase[j1];
          const double v0 = vs[j0], w0 = uz[j0], v1 = vs[j1], w1 = uz[j1];
          double x0[2 * MAXB / 32], x1[2 * MAXB / 32];
#pragma unroll
          for (int k = 0; k < 2 * MAXB / 32; k++) { x0[k] = W[b0 + lane + 32 * k]; x1[k] = W[b1 + lane + 32 * k]; }
          double* g0 = gd0 + j0 * ldm1;
          double* g1 = gd0 + j1 * ldm1;
#pragma unroll
          for (int k = 0; k < 2 * MAXB / 32; k++) {
            const int i = lane + 32 * k;
            const double z0 = x0[k] + vr[k] * w0 - ur[k] * v0;
            const double z1 = x1[k] + vr[k] * w1 - ur[k] * v1;
            const bool e0 = i > j0 && i < iend, e1 = h1 && i > j1 && i < iend;
            const bool isE = i >= L;
            const bool gst = !isE || last;
            if (e0 && isE) W[b0 + i] = z0;
            if (e1 && isE) W[b1 + i] = z1;
            if (e0 && gst) __stcg(&g0[i], z0);
            if (e1 && gst) __stcg(&g1[i], z1);
          }
        };
        if (warp == 0) {
          diag_cols(0, 0, false);
          if (!last) {
            // Householder of task t+1: x = rows [r+b, r+b+L1) of column r = this column's
            // block-below part (final now); beta goes to global memory before task t completes
            __syncwarp();
            int64_t col1, r1;
            int L1;
            geom(t + 1, col1, r1, L1);
            house(dbase[0] + b, L1, p ^ 1);
            __syncwarp();
            if (lane == 0) __stcg(a.AB + col1 * a.ldab + (r1 - col1), scb[p ^ 1][1]);
          }
        } else {
          const int w = warp - 1;   // 11 warps: left columns, then diagonal columns 1..L-1
          constexpr int NW = kChaseCW - 1;
          double vl[MAXB / 32];
#pragma unroll
          for (int k = 0; k < MAXB / 32; k++) vl[k] = vs[lane + 32 * k];
          double* const gl0 = a.AB + col * a.ldab + nl;   // + cc*(ldab-1): row r of column col+cc
          for (int q = w; q < ncl; q += 2 * NW) {
            const int c0 = q + 1, c1 = min(q + 1 + NW, nl - 1);
            const bool h1 = q + NW < ncl;
            const int b0 = lbase[c0], b1 = lbase[c1];
            const double y0 = yv[c0], y1 = yv[c1];
            double x0[MAXB / 32], x1[MAXB / 32];
#pragma unroll
            for (int k = 0; k < MAXB / 32; k++) { x0[k] = W[b0 + lane + 32 * k]; x1[k] = W[b1 + lane + 32 * k]; }
            double* g0 = gl0 + c0 * ldm1;
            double* g1 = gl0 + c1 * ldm1;
#pragma unroll
            for (int k = 0; k < MAXB / 32; k++) {
              const int i = lane + 32 * k;
              const bool ok = i < L;
              const double z0 = x0[k] - y0 * vl[k], z1 = x1[k] - y1 * vl[k];
              if (ok) __stcg(&g0[i], z0);
              if (ok && h1) __stcg(&g1[i], z1);
            }
          }
          // diagonal columns 1..L-1; the count of left columns shifts the start so the
          // warps stay balanced
          const int q0 = (ncl + w) % NW;
          for (int q = q0; q < L - 1; q += 2 * NW) {
            const int j0 = 1 + q, j1 = min(1 + q + NW, L - 1);
            diag_cols(j0, j1, q + NW < L - 1);
          }
        }
        C2_TS(2);
      }
      __syncthreads();
      if (warp == kChaseCW) {
        // ---- auxiliary warp: task t complete (all its writes precede the barrier, incl. the
        //      beta of task t+1), then the next task's final left column and reflector
        if (lane == 0) st_release_gpu(a.progress + s, t + 1);   // after the CTA barrier: cumulative
        if (!last) { __syncwarp(); store_col_refl(t + 1); }
      }
      C2_TS(3);
      if (prof) t_work += clock64() - tk;
    }
  }
  if (prof) { a.dbg[0] = t_wait; a.dbg[1] = t_work; a.dbg[2] = ntasks; for (int i = 0; i < 5; i++) a.dbg[3 + i] = tph[i]; }
#undef C2_TS
}

// extract Lemma-1 alpha_k = -T[k+1, k] from the final band
__global__ void alpha_from_band_kernel(const double* AB, int64_t ldab, int64_t n, double* alpha) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n - 1) alpha[k] = -AB[1 + k * ldab];
}

// band from the F2B output A (A[c+d, c], d <= b) into AB (ldab rows, zero beyond b).
// Distributed: only the rank owning column c ((c / b) mod P) contributes its column.
__global__ void band_extract_kernel(const double* A, int64_t lda, int64_t n, int b, double* AB, int64_t ldab, int P,
                                    int rank) {
  int64_t c = blockIdx.x;
  const bool mine = ((c / b) % P) == rank;
  for (int d = threadIdx.x; d < ldab; d += blockDim.x) {
    double v = 0.0;
    if (mine && d >= 1 && d <= b && c + d < n) v = A[SK_IDX(c + d, c, lda)];
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
// matrix) and U = V T^T.  Stored per group: U (K2 x LDU), in the shared-memory layout of the
// apply kernel, which places it beside -V (K2 x LDV) that its producer warps rebuild from the
// reflectors (the staircase positions are fixed per group, the rest stays zero), so that
// Q_g X = X + (-V) (U^T X) with one bulk copy per group and half the store.  The two row
// strides differ (LDU = 4, LDV = 6 mod 16 doubles) because the apply kernel reads U with the
// fragment pattern U[k0+t][c0+g] and V with V[r0+g][c0+2t+s]: both are then bank-conflict free.
template <int K2, int RW>
struct BT2Grp {
  static constexpr int LDU = RW + 4;
  static constexpr int LDV = RW + 6;
  static constexpr int ELEMS = K2 * (LDU + LDV);   // shared-memory block [U | -V]
  static constexpr int UELEMS = K2 * LDU;           // stored per group: U
  static_assert(LDU % 16 == 4 && LDV % 16 == 6 && (ELEMS % 2) == 0 && (UELEMS % 2) == 0, "BT2 group layout");
};

template <int K2, int RW>
__global__ void __launch_bounds__(128) bt2_prep_kernel(const double* qv, const double* qtau, int64_t ngroups, int b,
                                                      double* UV, bool uonly) {
  using Gp = BT2Grp<K2, RW>;
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
    double* out = UV + g * (uonly ? Gp::UELEMS : Gp::ELEMS);
    for (int e = threadIdx.x; e < K2 * Gp::LDU; e += blockDim.x) {
      int c = e / Gp::LDU, rho = e % Gp::LDU;
      double u = 0.0;
      if (rho < RW)
        for (int c2 = c; c2 < K2; c2++) u += V[c2][rho] * T[c][c2];
      out[e] = u;
    }
    if (!uonly)
      for (int e = threadIdx.x; e < K2 * Gp::LDV; e += blockDim.x) {
        int c = e / Gp::LDV, rho = e % Gp::LDV;
        out[K2 * Gp::LDU + e] = (rho < RW) ? -V[c][rho] : 0.0;
      }
    __syncthreads();
  }
}

// BT2 apply: one CTA per strip of NB columns of X, persistent over all groups in the
// order sweep blocks last -> first, t ascending.  The RW-row window
// X[W0 : W0+RW, strip] (W0 = s0 + t*b) lives in a RING-row shared-memory ring: step t+1
// reuses the last RW-b rows of window t, so per step only b new rows are loaded and b
// rows are written back.  The next group's [U | -V] block arrives with ONE bulk copy
// (cp.async.bulk, TMA engine) into the second buffer, tracked by an mbarrier; the b new
// window rows arrive with cp.async (each thread: rows 2*lane.., fixed columns).
// Consumers: one warp per 8 columns, so a warp's step needs no other warp's data:
//            Z^T = Xw^T U         (8 x K2, K = RW; DMMA, U's zero upper triangle skipped)
//            Xw  = Xw + (-V) Z    (RW x 8, K = K2; Z never leaves the registers: the
//                                  accumulator fragment of Z^T IS the B fragment of Z when
//                                  the K2 index is permuted, c = 8i + 2t + s)
template <int NB, int K2, int RW, int RING, int BB>
struct BT2Cfg {
  using Gp = BT2Grp<K2, RW>;
  static constexpr int NCW = NB / 8;     // consumer warps (8 columns each)
  static constexpr int NPW = 4;          // producer warps
  static constexpr int THREADS = 32 * (NCW + NPW);
  static constexpr int LDX = RING + 4;   // Xs[col][slot]
  static constexpr int LDU = Gp::LDU, LDV = Gp::LDV;
  static constexpr int XS = NB * LDX, GS = Gp::ELEMS;
  static constexpr size_t SMEM = (size_t)(XS + 2 * GS) * sizeof(double) + 6 * sizeof(uint64_t);
  static_assert(LDX % 16 == 4, "pad");
  static_assert(RING % 32 == 0 && RW % 8 == 0 && RING >= RW + BB && BB == 64 && K2 == 32 &&
                    (NB == 96 || NB == 64 || NB == 32),
                "ring");
};

// Non-volatile DMMA (the compiler may schedule it freely: it has no side effects)
__device__ __forceinline__ void dmma884f(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Z^T (8 columns x K2) = Xw^T U for the warp's columns cx..cx+7.  A = Xw^T: lane (g, t)
// reads X[k0+t][cx+g] (ring slot swizzle: slot ^ 4 for columns 4..7 of each group of 8);
// B = U[k0+t][8i+g].  U[rho][c] = 0 for rho <= c: n-fragment i starts at k-step 2i.
// Two accumulator sets (even / odd k-steps); fragments of k-step ks+1 loaded before the
// DMMAs of ks.  Out: z[i][s] = Z[8i + 2t + s][cx + g].
template <int K2, int RW, int RING, int LDX, int LDU>
__device__ __forceinline__ void bt2_cw_gemm1(const double* __restrict__ Xs, const double* __restrict__ Us, int off,
                                             int cx, int gq, int tq, double (&z)[4][2], uint64_t* rows_bar,
                                             unsigned parity) {
  constexpr int NKS = RW / 4;
  constexpr int NRES = (RW - 64) / 4;     // k-steps on the resident rows (rows 0 .. RW-BB-1)
  static_assert(NRES == 8, "k-step order below assumes RW - BB = 32");
  // resident k-steps first, paired high / low so every pair has >= 5 live DMMAs (U's zero
  // triangle leaves k-step ks only 1 + ks/2 live n-fragments for ks < 8); accumulator set =
  // position parity, so a chain's consecutive DMMAs are >= 4 DMMAs apart
  constexpr int ORD[8] = {7, 0, 6, 1, 5, 2, 4, 3};
  double acc[2][4][2];
#pragma unroll
  for (int p = 0; p < 2; p++)
#pragma unroll
    for (int i = 0; i < 4; i++) acc[p][i][0] = acc[p][i][1] = 0.0;
  const double* xcol = Xs + (cx + gq) * LDX;
  const int swz = gq & 4;
  const double* ucol = Us + gq * LDU + tq;
  double a[2], b[2][4];
  auto ld = [&](int ks, int sb) {
    int s = off + 4 * ks;
    if (s >= RING) s -= RING;
    a[sb] = xcol[(s + tq) ^ swz];
#pragma unroll
    for (int i = 0; i < 4; i++)
      if (ks >= 2 * i) b[sb][i] = ucol[8 * i * LDU + 4 * ks];
  };
  ld(ORD[0], 0);
#pragma unroll
  for (int p = 0; p < NRES; p++) {
    const int ks = ORD[p], sb = p & 1;
    if (p + 1 < NRES) ld(ORD[p + 1], sb ^ 1);
#pragma unroll
    for (int i = 0; i < 4; i++)
      if (ks >= 2 * i) dmma884f(acc[p & 1][i][0], acc[p & 1][i][1], a[sb], b[sb][i]);
  }
  mbar_wait(rows_bar, parity);   // the producer's new rows (no-op wait if already complete)
  ld(NRES, 0);
#pragma unroll
  for (int ks = NRES; ks < NKS; ks++) {
    const int sb = ks & 1;
    if (ks + 1 < NKS) ld(ks + 1, sb ^ 1);
#pragma unroll
    for (int i = 0; i < 4; i++) dmma884f(acc[ks & 1][i][0], acc[ks & 1][i][1], a[sb], b[sb][i]);
  }
#pragma unroll
  for (int i = 0; i < 4; i++) {
    z[i][0] = acc[0][i][0] + acc[1][i][0];
    z[i][1] = acc[0][i][1] + acc[1][i][1];
  }
}

// Xw += (-V) Z for the warp's columns: C fragment = X[8m+g][cx+2t+{0,1}] (loaded from and
// stored to the ring), A = -V[8m+g][c] and B = z[i][s] with c = 8i + 2t + s (k-step (i, s)).
// V[rho][c] != 0 only for c+1 <= rho <= c+BB: k-step (i, s) touches m-fragments i .. i+8.
template <int K2, int RW, int RING, int LDX, int LDV>
__device__ __forceinline__ void bt2_cw_gemm2(double* __restrict__ Xs, const double* __restrict__ Vs, int off, int cx,
                                             int gq, int tq, const double (&z)[4][2]) {
  constexpr int FM = RW / 8;
  constexpr int SPAN = 9;                 // live m-fragments per k-step
  double* x0 = Xs + (cx + 2 * tq) * LDX;
  double* x1 = x0 + LDX;
  const int swz = (tq & 2) << 1;
  int slot[FM];
  double x[FM][2];
#pragma unroll
  for (int m = 0; m < FM; m++) {
    int s = off + 8 * m;
    if (s >= RING) s -= RING;
    slot[m] = (s + gq) ^ swz;
    x[m][0] = x0[slot[m]];
    x[m][1] = x1[slot[m]];
  }
  const double* vb = Vs + 2 * tq * LDV + gq;
  double va[2][SPAN];
  auto ld = [&](int kk, int sb) {          // k-step kk = 2i + s
    const int i = kk >> 1, s = kk & 1;
    const double* vr = vb + (8 * i + s) * LDV;
#pragma unroll
    for (int d = 0; d < SPAN; d++)
      if (i + d < FM) va[sb][d] = vr[8 * (i + d)];
  };
  ld(0, 0);
#pragma unroll
  for (int kk = 0; kk < 8; kk++) {
    const int sb = kk & 1, i = kk >> 1, s = kk & 1;
    if (kk + 1 < 8) ld(kk + 1, sb ^ 1);
#pragma unroll
    for (int d = 0; d < SPAN; d++)
      if (i + d < FM) dmma884f(x[i + d][0], x[i + d][1], va[sb][d], z[i][s]);
  }
#pragma unroll
  for (int m = 0; m < FM; m++) {
    x0[slot[m]] = x[m][0];
    x1[slot[m]] = x[m][1];
  }
}


// Warp-specialised: NB/8 consumer warps run only the DMMA tiles of their own 8 columns; 4
// producer warps move the data one step ahead -- it waits until the consumers
// released step q-1 (mbarrier "empty"), writes that step's leaving rows back to X, then
// loads step q+1's [U | V] block (one bulk TMA copy) and its new window rows (cp.async)
// and signals mbarrier "full" (transaction bytes + cp.async completion arrivals).  The
// ring offset advances by b per step inside a sweep block and by RW at a block boundary,
// so the next block's first window never overlaps the window being computed.
template <int NB, int K2, int RW, int RING, int BB, bool SPLIT, bool VQ>
__global__ void __launch_bounds__(BT2Cfg<NB, K2, RW, RING, BB>::THREADS, 1) bt2_ws_kernel(double* __restrict__ X, int64_t ldx, int64_t ncols, int64_t n,
                                                       const double* __restrict__ UV, const double* __restrict__ qv,
                                                       const int64_t* __restrict__ gofs,
                                                       int64_t nblk, long long* dbg, int nsplit_arg,
                                                       unsigned long long* prog) {
  using C = BT2Cfg<NB, K2, RW, RING, BB>;
  const int nsplit = SPLIT ? nsplit_arg : 1;   // compile-time 1 on the default path
  extern __shared__ __align__(128) double sh[];
  double* Xs = sh;
  double* G0 = Xs + C::XS;            // [2][U | -V]
  uint64_t* full = reinterpret_cast<uint64_t*>(G0 + 2 * C::GS);   // [U | -V] block landed (bulk tx)
  uint64_t* empty = full + 2;                                        // consumers released a step
  uint64_t* fullx = full + 4;                                        // new window rows landed (cp.async)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, tq = lane & 3;
  // nsplit CTAs per strip (wavefront): member m takes the sweep blocks nblk-1-m, nblk-1-m-nsplit, ..
  // Block b only reads rows that block b+1 (the previous member) has written back: a per
  // producer-warp progress value seq(b)*(n+1) + rows-final orders them (release / acquire).
  const int member = (int)(blockIdx.x % nsplit);
  const int64_t strip = blockIdx.x / nsplit;
  const int64_t col0 = strip * NB;
  const int ncl = (int)smin<int64_t>(NB, ncols - col0);
  const bool vec = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  const int64_t blk0 = nblk - 1 - member;
  if (nblk <= 0 || blk0 < 0) return;
  for (int e = tid; e < C::XS; e += blockDim.x) Xs[e] = 0.0;   // ring rows beyond n stay finite
  if (VQ) {
    // -V outside the staircase: -0.0 inside the window rows, +0.0 in the pitch padding (the
    // values the [U | -V] store carries, so both layouts give bit-identical products)
    for (int e = tid; e < 2 * C::GS; e += blockDim.x) {
      const int eb = e % C::GS - C::Gp::UELEMS;
      G0[e] = (eb >= 0 && eb % C::LDV < RW) ? -0.0 : 0.0;
    }
  }
  if (tid == 0) {
    // full: the bulk copy's transaction count (+ the 4 producer warps' -V writes when the
    // store holds U only)
    mbar_init(&full[0], VQ ? 1 + C::NPW : 1); mbar_init(&full[1], VQ ? 1 + C::NPW : 1);
    mbar_init(&fullx[0], 128); mbar_init(&fullx[1], 128);
    mbar_init(&empty[0], C::NCW); mbar_init(&empty[1], C::NCW);
    mbar_fence_init();
  }
  __syncthreads();
  auto xo = [&](int col, int slot) -> int { return col * C::LDX + (slot ^ (((col >> 2) & 1) << 2)); };
  auto ntask_of = [&](int64_t blk) -> int64_t { return 1 + (n - 3 - blk * K2) / BB; };

  if (warp >= C::NCW) {
    // ============================ producer (4 warps) ============================
    const int pw = warp - C::NCW;                  // producer warp: columns pw, pw+4, ...
    const int ptid = tid - 32 * C::NCW;
    auto load_rows = [&](int64_t r0, int cnt, int slot0) {   // rows [r0, r0+cnt) -> ring from slot0
      for (int rr = 2 * lane; rr < cnt; rr += 64) {
        int slot = slot0 + rr;
        if (slot >= RING) slot -= RING;
        const int64_t r = r0 + rr;
        const int rc = (int)smin<int64_t>(2, smax<int64_t>(0, n - r));
#pragma unroll 4
        for (int cl = pw; cl < NB; cl += 4) {
          double* dst = Xs + xo(cl, slot);
          const int cnt2 = (cl < ncl) ? rc : 0;
          const double* src = cnt2 ? X + SK_IDX(r, col0 + cl, ldx) : X;
          if (vec) {
            cp_async16(dst, src, cnt2 * 8);
          } else {
            cp_async8(dst, src, cnt2 > 0 ? 8 : 0);
            cp_async8(dst + 1, cnt2 > 1 ? src + 1 : X, cnt2 > 1 ? 8 : 0);
          }
        }
      }
    };
    auto store_rows = [&](int64_t r0, int cnt, int slot0) {
      for (int rr = 2 * lane; rr < cnt; rr += 64) {
        int slot = slot0 + rr;
        if (slot >= RING) slot -= RING;
        const int64_t r = r0 + rr;
        if (r >= n) continue;
#pragma unroll 4
        for (int cl = pw; cl < NB; cl += 4) {
          if (cl >= ncl) continue;
          const double2 v = *reinterpret_cast<const double2*>(Xs + xo(cl, slot));
          double* dst = X + SK_IDX(r, col0 + cl, ldx);
          if (vec && r + 1 < n) {
            *reinterpret_cast<double2*>(dst) = v;
          } else {
            dst[0] = v.x;
            if (r + 1 < n) dst[1] = v.y;
          }
        }
      }
    };
    // the group's U by one bulk copy; its -V rebuilt by the producer warps from the reflectors
    // (reflector c at window rows c+1 .. c+BB; the buffer is free: its step was released):
    // the reflector loads are issued here, the shared-memory writes after the window-row loads
    constexpr int PER = K2 * BB / (32 * C::NPW);   // 16 values per producer thread
    static_assert(K2 * BB % (32 * C::NPW) == 0, "reflector block split");
    double qvv[PER];
    auto load_group = [&](int64_t g, int b) {
      constexpr int UE = VQ ? C::Gp::UELEMS : C::GS;   // U only, or the whole [U | -V] block
      if (ptid == 0) {
        mbar_expect_tx(&full[b], (unsigned)(UE * sizeof(double)));
        fence_proxy_async();
        bulk_g2s(G0 + b * C::GS, UV + g * UE, (unsigned)(UE * sizeof(double)), &full[b]);
      }
      if (VQ) {
        const double* qg = qv + g * K2 * BB;
#pragma unroll
        for (int i = 0; i < PER; i++) qvv[i] = __ldg(qg + ptid + 32 * C::NPW * i);
      }
    };
    auto finish_group = [&](int b) {
      if (!VQ) return;
      double* Vs = G0 + b * C::GS + C::Gp::UELEMS;
#pragma unroll
      for (int i = 0; i < PER; i++) {
        const int e = ptid + 32 * C::NPW * i, c = e / BB, d = e - c * BB;
        Vs[c * C::LDV + c + 1 + d] = -qvv[i];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[b]);
    };
    const int64_t pred = strip * nsplit + (member + nsplit - 1) % nsplit;
    auto wait_rows = [&](int64_t b, int64_t rend) {   // rows < rend of block b's input are final
      if (nsplit == 1 || nblk - 1 - b < 1) return;
      const unsigned long long need =
          (unsigned long long)(nblk - 2 - b) * (unsigned long long)(n + 1) + (unsigned long long)smin<int64_t>(rend, n);
      if (lane == 0)
        while (ld_acquire_gpu_u64(prog + pred * 4 + pw) < need) { }
      __syncwarp();
    };
    auto publish = [&](int64_t b, int64_t rend) {      // rows < rend of block b written back
      if (nsplit == 1) return;
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_release_gpu_u64(prog + (int64_t)blockIdx.x * 4 + pw,
                           (unsigned long long)(nblk - 1 - b) * (unsigned long long)(n + 1) +
                               (unsigned long long)smin<int64_t>(rend, n));
      }
    };
    // step 0
    int64_t blk = blk0, t = 0;
    int off = 0;
    load_group(gofs[blk], 0);
    wait_rows(blk, blk * K2 + RW);
    load_rows(blk * K2, RW, 0);
    cp_async_mbar_arrive(&fullx[0]);
    finish_group(0);
    int64_t pblk = -1, pt = 0;
    int poff = 0;
    bool pstored = true;    // step q-1 already written back
    int64_t pub_blk = -1, pub_rend = 0;   // rows written back but not yet published
    for (int64_t q = 0;; q++) {
      int64_t nblk_ = blk, nt = t + 1;
      int noff = off + BB;
      if (nt >= ntask_of(blk)) { nblk_ = blk - nsplit; nt = 0; noff = off + RW; }
      if (noff >= RING) noff -= RING;
      const bool has_next = nblk_ >= 0;
      if (!pstored) {   // consumers released step q-1: write back its leaving rows
        mbar_wait(&empty[(q - 1) & 1], (unsigned)(((q - 1) >> 1) & 1));
        const bool pfinal = (pt + 1 >= ntask_of(pblk));
        store_rows(pblk * K2 + pt * BB, pfinal ? RW : BB, poff);
        // published after this iteration's loads are issued: the publishing fence waits for
        // the stores, which then overlaps the consumers' step instead of delaying the loads
        pub_blk = pblk;
        pub_rend = pblk * K2 + pt * BB + (pfinal ? RW : BB);
      }
      bool stored = false;
      if (has_next && nblk_ != blk && (ntask_of(blk) == 1 || nsplit > 1 || RING < 2 * RW)) {
        if (pub_blk >= 0) { publish(pub_blk, pub_rend); pub_blk = -1; }
        // the next block's first window overlaps this block's last window (a single-step block,
        // or a ring shorter than two windows: RING = RW + BB) -- or, in
        // the wavefront, the partner CTA needs this block's last rows before it can publish
        // the rows our next block waits for: wait for step q and write it back before loading
        mbar_wait(&empty[q & 1], (unsigned)((q >> 1) & 1));
        store_rows(blk * K2 + t * BB, RW, off);
        publish(blk, blk * K2 + t * BB + RW);
        stored = true;
      }
      if (!has_next) {
        if (pub_blk >= 0) { publish(pub_blk, pub_rend); pub_blk = -1; }
        if (!stored) {
          mbar_wait(&empty[q & 1], (unsigned)((q >> 1) & 1));
          store_rows(blk * K2 + t * BB, RW, off);
          publish(blk, blk * K2 + t * BB + RW);
        }
        break;
      }
      {
        const int b = (int)((q + 1) & 1);
        load_group(gofs[nblk_] + nt, b);
        if (nblk_ == blk) {
          int so = noff + (RW - BB);
          if (so >= RING) so -= RING;
          const int64_t r0 = nblk_ * K2 + nt * BB + (RW - BB);
          wait_rows(nblk_, r0 + BB);
          load_rows(r0, BB, so);
        } else {
          wait_rows(nblk_, nblk_ * K2 + RW);
          load_rows(nblk_ * K2, RW, noff);
        }
        cp_async_mbar_arrive(&fullx[b]);
        finish_group(b);
        if (pub_blk >= 0) { publish(pub_blk, pub_rend); pub_blk = -1; }
      }
      pblk = blk; pt = t; poff = off; pstored = stored;
      blk = nblk_; t = nt; off = noff;
    }
    return;
  }
  // =============================== consumers ===============================
  long long ph[4] = {0, 0, 0, 0}, tprev = 0, nsteps = 0;
  const bool prof = (dbg != nullptr) && blockIdx.x == 0 && threadIdx.x == 0;
#define BT2_TS(k) do { if (prof) { long long _t = clock64(); ph[k] += _t - tprev; tprev = _t; } } while (0)
  const int cx = 8 * warp;   // this warp's columns cx .. cx+7 of the strip
  int64_t blk = blk0, t = 0;
  int off = 0;
  for (int64_t q = 0;; q++) {
    if (prof) { tprev = clock64(); nsteps++; }
    // The [U | -V] block and the window rows have separate barriers: inside a sweep block the
    // window's first RW-BB rows are this warp's own output of the previous step, so gemm1
    // starts on them while the producer's new rows are still landing.
    const unsigned par = (unsigned)((q >> 1) & 1);
    if (t == 0) mbar_wait(&fullx[q & 1], par);
    mbar_wait(&full[q & 1], par);
    BT2_TS(0);
    const double* Us = G0 + (q & 1) * C::GS;
    const double* Vs = Us + K2 * C::LDU;
    double z[4][2];
    bt2_cw_gemm1<K2, RW, RING, C::LDX, C::LDU>(Xs, Us, off, cx, gq, tq, z, &fullx[q & 1], par);
    BT2_TS(1);
    bt2_cw_gemm2<K2, RW, RING, C::LDX, C::LDV>(Xs, Vs, off, cx, gq, tq, z);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[q & 1]);
    BT2_TS(2);
    // advance
    int64_t nt = t + 1;
    int noff = off + BB;
    if (nt >= ntask_of(blk)) { blk -= nsplit; nt = 0; noff = off + RW; }
    if (noff >= RING) noff -= RING;
    if (blk < 0) break;
    t = nt; off = noff;
  }
  if (prof) {
    for (int k = 0; k < 3; k++) dbg[k] = ph[k];
    dbg[3] = 0; dbg[4] = 0;
    dbg[5] = nsteps;
  }
#undef BT2_TS
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
  uonly = n > 40000;   // n = 65536: the [U | -V] store would be 54 GB per rank, U alone 27 GB
  if (const char* v = getenv("SKEWEIG_BT2_UONLY")) uonly = atoi(v) != 0;   // experiments
}

cudaError_t band_extract(const double* A, int64_t lda, int64_t n, int b, double* AB, int64_t ldab, cudaStream_t st,
                         int P, int rank) {
  KScope ks(KC_BAND, st);
  band_extract_kernel<<<(unsigned)std::max<int64_t>(n, 1), 128, 0, st>>>(A, lda, n, b, AB, ldab, P, rank);
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
  if (vectors)   // per group U (BT2Grp::UELEMS) or [U | -V] (BT2Grp::ELEMS)
    w.qT = ar.take<double>((size_t)ng * L.k2 * (L.uonly ? (L.b + L.k2 + 4) : (2 * (L.b + L.k2) + 10)));
  w.gofs = ar.take<int64_t>(std::max<int64_t>(L.nblk, 1));
  if (vectors) w.prog = ar.take<unsigned long long>((size_t)4 * 2 * ((L.n + 63) / 64 + 1));   // BT2 wavefront flags
}

static int chase_grid(int64_t n, int b, int nsm, int lag) {
  // concurrently active sweeps ~ (n/b)/lag; never more CTAs than can be co-resident
  int64_t act = std::max<int64_t>(1, (n / std::max(b, 1)) / lag + 1);
  return (int)std::max<int64_t>(1, std::min<int64_t>(act, nsm));
}
int b2t_chase_ctas(int64_t n, int b, int nsm) { return n > 2 ? chase_grid(n, b, nsm, 2) : 0; }

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
      a.dbg = nullptr;
      int G = chase_grid(n, L.b, nsm, 2);
      if (const char* gg = getenv("SKEWEIG_CHASE_G")) G = std::max(1, std::min(G, atoi(gg)));   // experiments
      size_t smem = (size_t)(2 * L.b + 1) * (2 * L.b + 2) * sizeof(double);
      void* args[] = {&a};
      e = set_smem_attr((const void*)chase_kernel<64>, (int)smem);
      if (e) return e;
      e = cudaLaunchCooperativeKernel((void*)chase_kernel<64>, dim3(G), dim3(kChaseThreads), args, smem, st);
      if (e) return e;
    }
    alpha_from_band_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(w.AB, L.ldab, n, alpha);
  }
  return cudaGetLastError();
}

// per-strip time of a 96- / 32-wide strip relative to a 64-wide one (tools/bt2_time.py)
static constexpr double kNB96Cost = 1.47, kNB32Cost = 0.64;

// ring of RW + BB rows: within a sweep block step q+1's new rows reuse step q-1's leaving
// rows; at a block boundary the producer writes the last window back before loading the
// next block's (one stalled step per block, ~n/64 steps)
static constexpr int kBT2K2 = 32, kBT2RW = 96, kBT2Ring = 160, kBT2BB = 64;

// [U | V] blocks of every group (depends only on the chase output: the solve driver runs it
// on an auxiliary stream, concurrently with the tridiagonal solve)
cudaError_t bt2_prep(const B2TLayout& L, B2TWork& w, cudaStream_t st) {
  if (L.n <= 2 || L.ngroups == 0) return cudaSuccess;
  if (L.k2 != kBT2K2 || L.b != kBT2BB) return cudaErrorInvalidValue;
  KScope ks(KC_BT2_T, st);
  bt2_prep_kernel<kBT2K2, kBT2RW><<<(unsigned)std::min<int64_t>(L.ngroups, 8 * 148), 128, 0, st>>>(
      w.qv, w.qtau, L.ngroups, kBT2BB, w.qT, L.uonly);
  return cudaGetLastError();
}

cudaError_t bt2_run(const B2TLayout& L, B2TWork& w, double* X, int64_t ldx, int64_t ncols, cudaStream_t st) {
  cudaError_t e = bt2_prep(L, w, st);
  if (e) return e;
  return bt2_apply(L, w, X, ldx, ncols, st);
}

cudaError_t bt2_apply(const B2TLayout& L, B2TWork& w, double* X, int64_t ldx, int64_t ncols, cudaStream_t st) {
  if (L.n <= 2 || L.ngroups == 0 || ncols == 0) return cudaSuccess;
  cudaError_t e;
  constexpr int K2 = kBT2K2, RW = kBT2RW, RING = kBT2Ring, BB = kBT2BB;
  if (L.k2 != K2 || L.b != BB) return cudaErrorInvalidValue;
  long long* dbgp = nullptr;   // per-step cycle counters of CTA 0 (instrumentation hook, unused)
  // Column strips: 64 wide (best DMMA / smem ratio) and 32 wide (~0.55x the time of a
  // 64-wide strip, measured: tools/bt2_time.py).  Every strip runs the whole step sequence,
  // so the kernel time is (#waves) x (strip time); pick the mix of n64 wide and n32 narrow
  // strips covering ncols with the fewest wave-units: e.g. one GPU, 32768 columns -> 444
  // wide (3 full waves) + 136 narrow (one wave) instead of 3.46 -> 4 waves of wide strips;
  // 8 ranks x 4096 columns -> 128 narrow strips (one wave) instead of 64 wide ones.
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // strip mix: a96 x 96 + a64 x 64 + the rest in 32-wide strips; each width is one launch
  // and each launch costs (#waves) x (its strip time)
  int64_t n96 = 0, n64 = 0;
  double best = 1e300;
  for (int64_t a96 = 0; a96 <= (ncols + 95) / 96; a96++) {
    const int64_t r1 = std::max<int64_t>(0, ncols - 96 * a96);
    for (int64_t a64 = 0; a64 <= (r1 + 63) / 64; a64++) {
      const int64_t r2 = std::max<int64_t>(0, r1 - 64 * a64);
      const int64_t a32 = (r2 + 31) / 32;
      const double tw = kNB96Cost * (double)((a96 + nsm - 1) / nsm) + (double)((a64 + nsm - 1) / nsm) +
                        kNB32Cost * (double)((a32 + nsm - 1) / nsm);
      if (tw < best - 1e-9) { best = tw; n96 = a96; n64 = a64; }
    }
  }
  // Wavefront option: all strips 64 wide, each walked by TWO CTAs that take alternate sweep
  // blocks (the kernel's nsplit; 16-byte aligned X only).  Correct (bit-identical) but not
  // yet faster than the strip mix: 4096 columns at n = 32768 take 671 ms split vs 589 ms in
  // 32-wide strips (tools/bt2_time.py, round 1), so it is only enabled by SKEWEIG_BT2_SPLIT=2.
  const bool xvec = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  int nsplit = 1;
  if (const char* v = getenv("SKEWEIG_BT2_SPLIT")) nsplit = (atoi(v) == 2 && xvec && w.prog) ? 2 : 1;   // experiments
  if (nsplit == 2) { n96 = 0; n64 = (ncols + 63) / 64; }
  if (const char* v = getenv("SKEWEIG_BT2_NB")) {   // experiments: one strip width only
    const int wv = atoi(v);
    n96 = (wv == 96) ? (ncols + 95) / 96 : 0;
    n64 = (wv == 64) ? (ncols + 63) / 64 : 0;
  }
  if (n96 != 0 || n64 != (ncols + 63) / 64) nsplit = 1;
  const int64_t c96 = std::min<int64_t>(ncols, 96 * n96);
  const int64_t c64 = std::min<int64_t>(ncols - c96, 64 * n64);
  const int64_t c32 = ncols - c96 - c64;
  auto launch = [&](auto kern, size_t smem, int NBv, int64_t cbeg, int64_t cnt, int ns) -> cudaError_t {
    if (cnt <= 0) return cudaSuccess;
    cudaError_t e2 = set_smem_attr((const void*)kern, (int)smem);
    if (e2) return e2;
    const int64_t grid = ((cnt + NBv - 1) / NBv) * ns;
    if (ns > 1) {
      e2 = cudaMemsetAsync(w.prog, 0, sizeof(unsigned long long) * 4 * (size_t)grid, st);
      if (e2) return e2;
    }
    KScope ks(KC_BT2, st);
    kern<<<(unsigned)grid, 32 * (NBv / 8 + 4), smem, st>>>(X + cbeg * ldx, ldx, cnt, L.n, w.qT, w.qv, w.gofs, L.nblk, dbgp,
                                                           ns, w.prog);
    return cudaGetLastError();
  };
  auto launch_all = [&](auto vq) -> cudaError_t {
    constexpr bool V = decltype(vq)::value;
    cudaError_t e2 = launch(bt2_ws_kernel<96, K2, RW, RING, BB, false, V>, BT2Cfg<96, K2, RW, RING, BB>::SMEM, 96, 0,
                            c96, 1);
    if (e2) return e2;
    if (nsplit > 1)
      e2 = launch(bt2_ws_kernel<64, K2, RW, RING, BB, true, V>, BT2Cfg<64, K2, RW, RING, BB>::SMEM, 64, c96, c64,
                  nsplit);
    else
      e2 = launch(bt2_ws_kernel<64, K2, RW, RING, BB, false, V>, BT2Cfg<64, K2, RW, RING, BB>::SMEM, 64, c96, c64, 1);
    if (e2) return e2;
    return launch(bt2_ws_kernel<32, K2, RW, RING, BB, false, V>, BT2Cfg<32, K2, RW, RING, BB>::SMEM, 32, c96 + c64,
                  c32, 1);
  };
  e = L.uonly ? launch_all(std::true_type{}) : launch_all(std::false_type{});
  if (e) return e;
  return cudaGetLastError();
}

}  // namespace sk
