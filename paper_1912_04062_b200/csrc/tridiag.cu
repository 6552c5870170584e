// tridiag.cu -- tridiagonal stage (a support stage) and the D
// assembly (a8, Algorithm 1 step 3).
//
// Lemma 1: -i D^H T_skew D = T_sym = tridiag(alpha, 0, alpha),
// D = diag(i^0..i^{n-1}).  The top-nev eigenpairs of T_sym are computed by
// Sturm-count bisection (one thread per eigenvalue) and inverse iteration (one
// thread per eigenvector, dstein-style LU with partial pivoting and perturbed
// pivots), then re-orthogonalised in blocks of 32 against a window of previous
// vectors (CGS2) plus the members of the vector's cluster, and within the block by
// CholQR2 ("bisection and inverse iteration"; R9).
// Unreduced blocks (alpha_k == 0 exactly) are treated separately (host-side split).
#include "common.cuh"
#include "internal.h"
#include <nccl.h>
#include "gemm_dmma.cuh"
#include <vector>
#include <algorithm>
#include <cmath>
#include <cfloat>
#include <cooperative_groups.h>

namespace sk {

namespace cg = cooperative_groups;

__device__ __forceinline__ uint64_t td_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Multisection (K points per round instead of one midpoint): K lanes of a warp share one
// eigenvalue, each evaluates the Sturm count at one of K interior points of [lo, hi), and
// the group keeps the sub-interval where the count crosses the target index (the same
// invariant as bisection: count(lo) <= i < count(hi)).  ~log_{K+1}(2g/tol) rounds instead of
// log_2: the Sturm chain (one dependent division per row) is latency-bound, so K-fold more
// counts per round cost little and the critical path shrinks ~3x for K = 8.  Same stopping
// rule as plain bisection (reading of PAPER.md:616): width <= max(2 eps max|x|, eps g).
// Sturm count on block [s0, s0+m): #{eigenvalues < sigma} of tridiag(alpha, 0, alpha),
// q_0 = -sigma, q_k = -sigma - alpha_{k-1}^2 / q_{k-1}, |q_k| < pivmin -> -pivmin.
// Zero-diagonal aware: two rows per division.  With t = -sigma q_{k-1} - alpha_{k-1}^2,
// q_k = t / q_{k-1} (its sign is sign(t) * sign(q_{k-1}); |q_k| < pivmin iff |t| < pivmin |q|)
// and q_{k+1} = -sigma - alpha_k^2 q_{k-1} / t, so the pair costs one division instead of two
// (the per-row chain is a dependent division, so this halves the latency-bound critical path).
// Right after a clamped pivot (|q| > 1e150) the two rows are stepped one by one, which keeps
// sigma * q and alpha^2 * q finite.
__device__ __forceinline__ void td_sturm_pair(double a, double b, double sigma, double pivmin, double& q, int& cnt) {
  if (fabs(q) > 1e150) {
    double qk = -sigma - a / q;
    if (fabs(qk) < pivmin) qk = -pivmin;
    cnt += (qk < 0);
    q = -sigma - b / qk;
  } else {
    const double t = fma(-sigma, q, -a);
    if (fabs(t) < pivmin * fabs(q)) {   // q_k clamped to -pivmin
      cnt += 1;
      q = -sigma + b / pivmin;
    } else {
      cnt += ((t < 0.0) != (q < 0.0));
      q = -sigma - (b * q) / t;
    }
  }
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += (q < 0);
}

__device__ __forceinline__ int td_sturm32(const double* __restrict__ a2, int64_t s0, int m, double sigma,
                                          double pivmin) {
  int cnt = 0;
  double q = -sigma;
  if (fabs(q) < pivmin) q = -pivmin;
  cnt += (q < 0);
  const double* p = a2 + s0;
  // the a2 loads never depend on the chain: issue 16 of them ahead of each 16 rows, so the
  // row cost is the division chain, not one L2 round trip per row
  constexpr int U = 16;
  int k = 1;
  for (; k + U <= m; k += U) {
    double av[U];
#pragma unroll
    for (int u = 0; u < U; u++) av[u] = __ldg(p + k - 1 + u);
#pragma unroll
    for (int u = 0; u < U; u += 2) td_sturm_pair(av[u], av[u + 1], sigma, pivmin, q, cnt);
  }
  for (; k + 1 < m; k += 2) td_sturm_pair(__ldg(p + k - 1), __ldg(p + k), sigma, pivmin, q, cnt);
  if (k < m) {
    q = -sigma - __ldg(p + k - 1) / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += (q < 0);
  }
  return cnt;
}

// Count grid (one unreduced block): c[j] = Sturm count at x_j = -bnd + 2 bnd j / M, j = 1..M-1
// (c[0] = 0 and c[M] = m are implicit: the Gershgorin bound).  One pass of M counts, the
// cost of one multisection round, replaces the first ~log_{K+1}(M) rounds of every eigenvalue:
// each starts from the grid cell [x_{j-1}, x_j) where the count crosses its index.
__device__ __forceinline__ double td_grid_x(double bnd, int j, int M) { return -bnd + (2.0 * bnd) * ((double)j / (double)M); }
__device__ __forceinline__ double td_bnd(double g, double pivmin) { return g * (1.0 + 4.0 * DBL_EPSILON) + 4.0 * pivmin; }

__global__ void __launch_bounds__(128) td_count_grid_kernel(const double* a2, int64_t s0, int m, double g, int M,
                                                            double pivmin, int* cgrid) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < 1 || j >= M) return;
  cgrid[j] = td_sturm32(a2, s0, m, td_grid_x(td_bnd(g, pivmin), j, M), pivmin);
}

template <int K>
__global__ void __launch_bounds__(128, 7) td_msect_kernel(const double* a2, const int64_t* task_s0, const int64_t* task_m,
                                                       const int64_t* task_i, const double* task_g, int64_t q0,
                                                       int64_t q1, double pivmin, double* out, const int* cgrid,
                                                       int M, int64_t n1, double g1) {
  static_assert(32 % K == 0, "K divides the warp");
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, k = lane % K, gbase = lane - k;
  const int64_t q = q0 + gt / K;
  const bool valid = q < q1;
  const int64_t qq = valid ? q : q1 - 1;
  // task list, or (task_s0 == null) one unreduced block of order n1: task q = index n1-1-q
  const int64_t s0 = task_s0 ? task_s0[qq] : 0;
  const int m = task_s0 ? (int)task_m[qq] : (int)n1;
  const int i = task_s0 ? (int)task_i[qq] : (int)(n1 - 1 - qq);
  const double g = task_s0 ? task_g[qq] : g1;
  const double bnd = td_bnd(g, pivmin);
  double lo = -bnd, hi = bnd;
  if (M > 1 && valid) {
    // grid cell of index i: jl < jh with count(x_jl) <= i < count(x_jh), c[0] = 0, c[M] = m
    int jl = 0, jh = M;
    while (jh - jl > 1) {
      const int jm = (jl + jh) >> 1;
      if (__ldg(cgrid + jm) > i) jh = jm; else jl = jm;
    }
    if (jl > 0) lo = td_grid_x(bnd, jl, M);
    if (jh < M) hi = td_grid_x(bnd, jh, M);
  }
  const double atol = DBL_EPSILON * g;
  bool done = !valid || m == 1;
  for (int it = 0; it < 400; it++) {
    if (!done && hi - lo <= fmax(2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)), atol)) done = true;
    if (__all_sync(0xffffffffu, done)) break;   // every group of the warp converged
    const double h = (hi - lo) / (K + 1);
    const double x = lo + h * (k + 1);
    const int c = done ? 0 : (td_sturm32(a2, s0, m, x, pivmin) > i);
    const unsigned msk = (__ballot_sync(0xffffffffu, c) >> gbase) & (K == 32 ? 0xffffffffu : ((1u << K) - 1u));
    if (!done) {
      const int f = msk ? __ffs(msk) - 1 : K;   // first point with count > i
      const double nlo = (f > 0) ? lo + h * f : lo;
      const double nhi = (f < K) ? lo + h * (f + 1) : hi;
      if (nlo == lo && nhi == hi) done = true;   // no representable progress
      lo = nlo; hi = nhi;
    }
  }
  if (valid && k == 0) out[q] = (m == 1) ? 0.0 : 0.5 * (lo + hi);
}

// Inverse iteration, one thread per vector (dstein semantics).  Work arrays
// are interleaved [row][batch] so that a warp's accesses are coalesced; every pass over a
// vector is chunked by IU rows with the chunk's loads issued first (they never depend on
// the loop-carried values), so each thread keeps IU loads in flight.  The scaling of the
// right-hand side is folded into the forward pass and the 1-norm / max-norm / 2-norm of
// the solution are accumulated in the back substitution.
struct InvArgs {
  const double* alpha;          // global alpha (n-1)
  const int64_t* vs0; const int64_t* vm;   // block start / size per vector (global index)
  const double* lam;            // perturbed eigenvalue per vector
  const double* gblk;           // block Gershgorin bound per vector
  int64_t nvec; int64_t col0;   // vectors [col0, col0+nvec) (global eigenpair indices)
  double *wa, *wb, *wc, *wd; unsigned char* win;   // [m][nvec]
  double* y;                    // [m][nvec]
  double* scale;                // [nvec] final 1/||y|| with the dstein sign
  uint64_t seed;
  int* nfail;
  const unsigned char* single;  // per global vector: 1 = isolated (twisted kernel), 0 = dstein kernel
  double pivmin;
};

template <int IU>
__global__ void __launch_bounds__(128) td_inverse_kernel(InvArgs a) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= a.nvec) return;
  const int64_t gv = a.col0 + q;
  if (a.single[gv]) return;   // isolated eigenvalue: td_twisted_kernel
  const int64_t s0 = a.vs0[gv], m = a.vm[gv];
  const int64_t B = a.nvec;
  double* A_ = a.wa; double* Bb = a.wb; double* C = a.wc; double* D = a.wd; unsigned char* IN = a.win;
  double* y = a.y;
#define AT(arr, k) arr[(size_t)(k) * B + q]
  const double lambda = a.lam[gv];
  const double g = a.gblk[gv];
  const double eps = DBL_EPSILON;
  if (m == 1) { AT(y, 0) = 1.0; a.scale[q] = 1.0; return; }
  const double* al = a.alpha + s0;
  // ---- dlagtf: LU of T - lambda I with partial pivoting; tol = eps * max|U entries|
  double tol = 0.0;
  {
    double ak = -lambda, bk = al[0];     // current (k) diagonal and super-diagonal
    // alpha is read 16 rows ahead of the pivoting recurrence (loads off the chain)
    for (int64_t k0 = 0; k0 + 1 < m; k0 += 16) {
    double alv[17];
#pragma unroll
    for (int u = 0; u < 17; u++) alv[u] = (k0 + u < m - 1) ? al[k0 + u] : 0.0;
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const int64_t k = k0 + u;
      if (k + 1 >= m) break;
      const double ck = alv[u];
      const double ak1 = -lambda;
      const double bk1 = (k + 2 < m) ? alv[u + 1] : 0.0;
      const double scale1 = fabs(ak) + fabs(bk);
      const double scale2 = fabs(ck) + fabs(ak1) + fabs(bk1);
      const double piv1 = (scale1 == 0.0) ? 0.0 : fabs(ak) / scale1;
      double na1, nb1 = bk1, dk = 0.0, cout;
      unsigned char in = 0;
      if (ck == 0.0) {
        cout = ck; na1 = ak1;
      } else {
        const double piv2 = fabs(ck) / scale2;
        if (piv2 <= piv1) {
          cout = ck / ak;
          na1 = ak1 - cout * bk;
        } else {
          in = 1;
          const double mult = ak / ck;
          const double ak_new = ck;
          na1 = bk - mult * ak1;
          dk = bk1;
          nb1 = -mult * bk1;
          const double bk_new = ak1;
          ak = ak_new; bk = bk_new; cout = mult;
        }
      }
      AT(A_, k) = ak; AT(Bb, k) = bk; AT(C, k) = cout; AT(IN, k) = in;
      if (k + 2 < m) AT(D, k) = dk;
      tol = fmax(tol, fmax(fabs(ak), fabs(bk)));
      if (k + 2 < m) tol = fmax(tol, fabs(dk));
      ak = na1; bk = nb1;
    }
    }
    AT(A_, m - 1) = ak;
    tol = fmax(tol, fabs(ak));
  }
  tol *= eps;
  if (tol == 0.0) tol = eps;
  const double anm1 = fabs(AT(A_, m - 1));
  // ---- start vector (uniform [-1, 1) from the counter-based generator)
  double asum = 0.0;
  for (int64_t i = 0; i < m; i++) {
    uint64_t z = td_splitmix64(a.seed * 0x9E3779B97F4A7C15ull + (uint64_t)gv * 0x100000001B3ull + (uint64_t)i);
    double v = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
    AT(y, i) = v;
    asum += fabs(v);
  }
  const double dtpcrt = sqrt(0.1 / (double)m);
  const double sfmin = DBL_MIN, bignum = 1.0 / DBL_MIN;
  int nrmchk = 0, ok = 0;
  double ssq = 0.0, ymax = 0.0;
  int64_t jmax = 0;
  for (int its = 0; its < 5; its++) {
    const double scl = (double)m * g * fmax(eps, anm1) / asum;
    // ---- forward (dlagts job -1), scaling folded in: carry p = y[k-1]
    double p = AT(y, 0) * scl;
    for (int64_t k0 = 1; k0 < m; k0 += IU) {
      double cc[IU], yy[IU];
      unsigned char ii[IU];
#pragma unroll
      for (int u = 0; u < IU; u++) {
        const int64_t k = k0 + u;
        if (k < m) { cc[u] = AT(C, k - 1); ii[u] = AT(IN, k - 1); yy[u] = AT(y, k); }
      }
#pragma unroll
      for (int u = 0; u < IU; u++) {
        const int64_t k = k0 + u;
        if (k < m) {
          const double qv = yy[u] * scl;
          if (ii[u] == 0) { AT(y, k - 1) = p; p = qv - cc[u] * p; }
          else { AT(y, k - 1) = qv; p = p - cc[u] * qv; }
        }
      }
    }
    AT(y, m - 1) = p;
    // ---- back substitution with perturbed pivots; carry y[k+1], y[k+2]
    double y1 = 0.0, y2 = 0.0, nrm = 0.0;
    asum = 0.0; ssq = 0.0; ymax = 0.0; jmax = 0;
    for (int64_t k0 = m - 1; k0 >= 0; k0 -= IU) {
      double aa[IU], bb[IU], dd[IU], yy[IU];
#pragma unroll
      for (int u = 0; u < IU; u++) {
        const int64_t k = k0 - u;
        if (k >= 0) {
          aa[u] = AT(A_, k); yy[u] = AT(y, k);
          bb[u] = (k + 1 < m) ? AT(Bb, k) : 0.0;
          dd[u] = (k + 2 < m) ? AT(D, k) : 0.0;
        }
      }
      // reciprocals of the pivots off the dependency chain (loaded with the chunk): the
      // common case (|a_k| >= 1, or no overflow risk) multiplies; the dlagts perturbation
      // loop only runs when the pivot is tiny
      double ra[IU];
#pragma unroll
      for (int u = 0; u < IU; u++) ra[u] = (k0 - u >= 0 && aa[u] != 0.0) ? 1.0 / aa[u] : 0.0;
#pragma unroll
      for (int u = 0; u < IU; u++) {
        const int64_t k = k0 - u;
        if (k >= 0) {
          double temp = yy[u] - bb[u] * y1 - dd[u] * y2;
          double ak = aa[u];
          const double absa = fabs(ak);
          double yk;
          if (absa >= 1.0 || (absa >= sfmin && !(fabs(temp) > absa * bignum))) {
            yk = temp * ra[u];
          } else {
            double pert = copysign(tol, ak);
            for (int guard = 0; guard < 2100; guard++) {
              double absak = fabs(ak);
              if (absak < 1.0) {
                if (absak < sfmin) {
                  if (absak == 0.0 || fabs(temp) * sfmin > absak) { ak += pert; pert *= 2.0; continue; }
                  temp *= bignum; ak *= bignum;
                } else if (fabs(temp) > absak * bignum) { ak += pert; pert *= 2.0; continue; }
              }
              break;
            }
            yk = temp / ak;
          }
          AT(y, k) = yk;
          y2 = y1; y1 = yk;
          const double ay = fabs(yk);
          asum += ay;
          ssq += yk * yk;
          if (ay > ymax || (ay == ymax && k < jmax)) { ymax = ay; jmax = k; }
          nrm = fmax(nrm, ay);
        }
      }
    }
    if (nrm < dtpcrt) continue;
    nrmchk++;
    if (nrmchk < 3) continue;
    ok = 1;
    break;
  }
  if (!ok) atomicAdd(a.nfail, 1);
  double sc = 1.0 / sqrt(ssq);
  if (AT(y, jmax) < 0) sc = -sc;
  a.scale[q] = sc;
#undef AT
}

// Isolated eigenvalues (no other eigenvalue within the cluster threshold, reading R9(4)):
// the eigenvector from ONE twisted factorization of T - lambda I (Fernando / Parlett; the
// vector step of MRRR, here on the zero-diagonal Lemma-1 tridiagonal) instead of dstein's
// iterated LU solves.  Two lanes per vector, in parallel: lane h = 0 the forward pivots
// d_0 = -lambda, d_{k+1} = -lambda - alpha_k^2 / d_k (LDL^T), lane h = 1 the backward pivots
// delta_{m-1} = -lambda, delta_k = -lambda - alpha_k^2 / delta_{k+1} (UDU^T); twist
// r = argmin |gamma_k|, gamma_k = d_k + delta_k + lambda (zero diagonal); then z_r = 1,
// z_k = -(alpha_k / d_k) z_{k+1} (k < r, lane 0) and z_k = -(alpha_{k-1} / delta_k) z_{k-1}
// (k > r, lane 1).  Pivots below pivmin are replaced by -pivmin (as in the Sturm count).
// Output as td_inverse_kernel: y [m][nvec] and scale (1/||z||, largest entry positive); the
// block CGS2 re-orthogonalisation follows unchanged.  Lanes: vector q0 + (lane & 15),
// role lane >> 4, so both roles walk the interleaved arrays coalesced.
__global__ void __launch_bounds__(128) td_twisted_kernel(InvArgs a) {
  const int lane = threadIdx.x & 31, h = lane >> 4;
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32 * 16 + (lane & 15);
  const bool valid = q < a.nvec;
  const int64_t gv = a.col0 + (valid ? q : 0);
  const bool active = valid && a.single[gv];
  const int64_t s0 = a.vs0[gv], m = active ? a.vm[gv] : 0;
  const int64_t B = a.nvec;
#define AT(arr, k) arr[(size_t)(k) * B + q]
  double* D = a.wa;     // forward pivots d_k
  double* E = a.wb;     // backward pivots delta_k
  double* y = a.y;
  const double lambda = active ? a.lam[gv] : 0.0;
  const double pivmin = a.pivmin;
  const double* al = a.alpha + s0;
  if (active && m == 1) { if (h == 0) { AT(y, 0) = 1.0; a.scale[q] = 1.0; } }
  const bool work = active && m > 1;
  // ---- pivots (lane roles in parallel; alpha loads 16 rows ahead of the division chain)
  if (work) {
    double piv = -lambda;
    if (fabs(piv) < pivmin) piv = -pivmin;
    if (h == 0) {
      AT(D, 0) = piv;
      for (int64_t k0 = 0; k0 + 1 < m; k0 += 16) {
        double av[16];
#pragma unroll
        for (int u = 0; u < 16; u++) av[u] = (k0 + u + 1 < m) ? al[k0 + u] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int64_t k = k0 + u;
          if (k + 1 >= m) break;
          piv = -lambda - (av[u] * av[u]) / piv;
          if (fabs(piv) < pivmin) piv = -pivmin;
          AT(D, k + 1) = piv;
        }
      }
    } else {
      AT(E, m - 1) = piv;
      for (int64_t k0 = m - 2; k0 >= 0; k0 -= 16) {
        double av[16];
#pragma unroll
        for (int u = 0; u < 16; u++) av[u] = (k0 - u >= 0) ? al[k0 - u] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int64_t k = k0 - u;
          if (k < 0) break;
          piv = -lambda - (av[u] * av[u]) / piv;
          if (fabs(piv) < pivmin) piv = -pivmin;
          AT(E, k) = piv;
        }
      }
    }
  }
  __syncwarp();
  // ---- twist index: each role scans half of the rows, then the pair combines
  double best = INFINITY;
  int64_t r = 0;
  if (work) {   // 16 rows of loads in flight ahead of the compares
    const int64_t k0 = h ? m / 2 : 0, k1 = h ? m : m / 2;
    for (int64_t kb = k0; kb < k1; kb += 16) {
      double dv[16], ev[16];
#pragma unroll
      for (int u = 0; u < 16; u++)
        if (kb + u < k1) { dv[u] = AT(D, kb + u); ev[u] = AT(E, kb + u); }
#pragma unroll
      for (int u = 0; u < 16; u++)
        if (kb + u < k1) {
          const double gk = fabs(dv[u] + ev[u] + lambda);
          if (gk < best) { best = gk; r = kb + u; }
        }
    }
  }
  {
    const double ob = __shfl_xor_sync(0xffffffffu, best, 16);
    const int64_t orr = __shfl_xor_sync(0xffffffffu, r, 16);
    if (ob < best || (ob == best && orr < r)) { best = ob; r = orr; }
  }
  // ---- z: lane 0 rows r-1 .. 0, lane 1 rows r+1 .. m-1; sum of squares and the largest entry
  double ssq = 0.0, zmax = 0.0;
  int64_t jmax = r;
  if (work) {
    // the multipliers of a 16-row chunk (loads and divisions off the z chain) first, then
    // the chunk's products
    if (h == 0) {
      double z = 1.0;
      AT(y, r) = 1.0;
      ssq = 1.0; zmax = 1.0;
      for (int64_t kb = r - 1; kb >= 0; kb -= 16) {
        // all 16 loads first (a division's slow-path branch would otherwise keep the next
        // load behind it), then the 16 independent divisions
        double mu[16], dv[16], nv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int64_t k = kb - u;
          dv[u] = (k >= 0) ? AT(D, k) : 1.0;
          nv[u] = (k >= 0) ? al[k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; u++) mu[u] = -(nv[u] / dv[u]);
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int64_t k = kb - u;
          if (k < 0) break;
          z = mu[u] * z;
          AT(y, k) = z;
          ssq += z * z;
          if (fabs(z) > zmax) { zmax = fabs(z); jmax = k; }
        }
      }
    } else {
      double z = 1.0;
      for (int64_t kb = r + 1; kb < m; kb += 16) {
        double mu[16], dv[16], nv[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int64_t k = kb + u;
          dv[u] = (k < m) ? AT(E, k) : 1.0;
          nv[u] = (k < m) ? al[k - 1] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; u++) mu[u] = -(nv[u] / dv[u]);
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int64_t k = kb + u;
          if (k >= m) break;
          z = mu[u] * z;
          AT(y, k) = z;
          ssq += z * z;
          if (fabs(z) > zmax) { zmax = fabs(z); jmax = k; }
        }
      }
    }
  }
  const double ossq = __shfl_xor_sync(0xffffffffu, ssq, 16);
  const double ozm = __shfl_xor_sync(0xffffffffu, zmax, 16);
  const int64_t ojm = __shfl_xor_sync(0xffffffffu, jmax, 16);
  __syncwarp();
  if (work && h == 0) {
    const double tot = ssq + ossq;
    int64_t jm = jmax;
    if (ozm > zmax || (ozm == zmax && ojm < jmax)) jm = ojm;
    double sc = 1.0 / sqrt(tot);
    if (AT(y, jm) < 0) sc = -sc;
    a.scale[q] = sc;
  }
#undef AT
}

// Q[:, qcol0 + q] = scale[q] * y[:, q] placed at the vector's block rows, zero elsewhere;
// 32 x 32 tiles transposed through shared memory (coalesced on both sides).
__global__ void td_place_vectors(const double* y, const double* scale, int64_t nvec, int64_t col0,
                                 const int64_t* vs0, const int64_t* vm, int64_t n, double* Q, int64_t ldq,
                                 int64_t qcol0, const unsigned char* single, int mode) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, v0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  const bool mine = v0 + tx < nvec && single[col0 + v0 + tx] == mode;   // this pass computed vector v0+tx
  if (!__syncthreads_or(mine)) return;
  for (int rr = ty; rr < 32; rr += 8) {
    const int64_t row = r0 + rr, v = v0 + tx;
    double val = 0.0;
    if (mine && row < n) {
      const int64_t s0 = vs0[col0 + v], m = vm[col0 + v];
      if (row >= s0 && row < s0 + m) val = y[(size_t)(row - s0) * nvec + v] * scale[v];
    }
    tile[rr][tx] = val;
  }
  __syncthreads();
  for (int vv = ty; vv < 32; vv += 8) {
    const int64_t v = v0 + vv, row = r0 + tx;
    if (v < nvec && row < n && single[col0 + v] == mode) Q[SK_IDX(row, qcol0 + v, ldq)] = tile[tx][vv];
  }
}

// ---------------- block re-orthogonalisation helpers
// partial H[(chunk)] = Qp^T Y over a row chunk of kGramRows rows: both panels are staged
// in shared memory with coalesced column loads (LD odd: conflict-free strided reads).
__global__ void td_gram_partial(const double* Qp, int64_t ldq, int p, const double* Y, int64_t ldy, int nb,
                                int64_t n, int64_t rows_per, double* part) {
  extern __shared__ double gs[];
  const int R = (int)rows_per, LD = R + 1;
  double* Qs = gs;             // p x LD
  double* Ys = gs + p * LD;    // nb x LD
  const int64_t r0 = blockIdx.x * rows_per;
  const int nr = (int)smin<int64_t>(rows_per, n - r0);
  for (int e = threadIdx.x; e < p * R; e += blockDim.x) {
    int i = e / R, r = e % R;
    Qs[i * LD + r] = (r < nr) ? Qp[SK_IDX(r0 + r, i, ldq)] : 0.0;
  }
  for (int e = threadIdx.x; e < nb * R; e += blockDim.x) {
    int j = e / R, r = e % R;
    Ys[j * LD + r] = (r < nr) ? Y[SK_IDX(r0 + r, j, ldy)] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < p * nb; e += blockDim.x) {
    int i = e % p, j = e / p;
    double s = 0.0;
#pragma unroll 8
    for (int r = 0; r < R; r++) s += Qs[i * LD + r] * Ys[j * LD + r];
    part[(size_t)blockIdx.x * p * nb + e] = s;
  }
}
__global__ void td_reduce_partials(const double* part, int nchunks, int cnt, double* out) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cnt) return;
  double s = 0.0;
#pragma unroll 8
  for (int c = 0; c < nchunks; c++) s += part[(size_t)c * cnt + e];
  out[e] = s;
}
// Y -= Qp H   (row-parallel)
__global__ void td_sub_proj(const double* Qp, int64_t ldq, int p, const double* H, double* Y, int64_t ldy, int nb,
                            int64_t n) {
  extern __shared__ double hs[];
  for (int e = threadIdx.x; e < p * nb; e += blockDim.x) hs[e] = H[e];
  __syncthreads();
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  double q[64];
  for (int i = 0; i < p; i++) q[i] = Qp[SK_IDX(r, i, ldq)];
  for (int j = 0; j < nb; j++) {
    double s = 0.0;
    for (int i = 0; i < p; i++) s += q[i] * hs[i + j * p];
    Y[SK_IDX(r, j, ldy)] -= s;
  }
}
// Cholesky of the nb x nb Gram (nb <= 32) -> R^{-1} (upper) in Rinv.  One warp: column j of L
// is finished by lane-parallel updates (right-looking), then the triangular inverse is
// formed column by column with lane-parallel dot products.
__global__ void td_chol_inv(const double* Gm, int nb, double* Rinv) {
  __shared__ double L[32][33];
  __shared__ double Li[32][33];
  const int lane = threadIdx.x;
  if (lane >= 32) return;
  for (int j = 0; j < nb; j++) {
    for (int i = lane; i < nb; i += 32) { L[i][j] = Gm[i + j * nb]; Li[i][j] = 0.0; }
  }
  __syncwarp();
  for (int j = 0; j < nb; j++) {
    const double d = sqrt(fmax(L[j][j], 1e-300));
    __syncwarp();
    if (lane > j && lane < nb) L[lane][j] /= d;
    if (lane == j) L[j][j] = d;
    __syncwarp();
    // trailing update: L[i][k] -= L[i][j] L[k][j] for k > j, i >= k (lane = i)
    if (lane > j && lane < nb) {
      const double lij = L[lane][j];
      for (int k = j + 1; k <= lane; k++) L[lane][k] -= lij * L[k][j];
    }
    __syncwarp();
  }
  // inverse of lower L: column j (lane = i): Li[i][j] = -(sum_{k=j}^{i-1} L[i][k] Li[k][j]) / L[i][i]
  for (int j = 0; j < nb; j++) {
    if (lane == j) Li[j][j] = 1.0 / L[j][j];
    __syncwarp();
    for (int i = j + 1; i < nb; i++) {
      double part = 0.0;
      for (int k = j + lane; k < i; k += 32) part += L[i][k] * Li[k][j];
      part = warp_sum(part);
      if (lane == 0) Li[i][j] = -part / L[i][i];
      __syncwarp();
    }
  }
  __syncwarp();
  // R = L^T (upper), R^{-1} = (L^{-1})^T
  for (int j = 0; j < nb; j++)
    for (int i = lane; i < nb; i += 32) Rinv[i + j * nb] = Li[j][i];
}
// Y <- Y R^{-1}  (row-parallel)
__global__ void td_apply_rinv(double* Y, int64_t ldy, int nb, const double* Rinv, int64_t n) {
  extern __shared__ double rs[];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) rs[e] = Rinv[e];
  __syncthreads();
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  double y[64];
  for (int j = 0; j < nb; j++) y[j] = Y[SK_IDX(r, j, ldy)];
  for (int j = 0; j < nb; j++) {
    double s = 0.0;
    for (int i = 0; i <= j; i++) s += y[i] * rs[i + j * nb];
    Y[SK_IDX(r, j, ldy)] = s;
  }
}

// D assembly (Algorithm 1 step 3; reading R1):
// X[:, c] = Re(D q_c), X[:, nev + c] = Im(D q_c); row k: k%4 = 0 -> Re +q, 1 -> Im +q,
// 2 -> Re -q, 3 -> Im -q.
__global__ void assemble_D_kernel(const double* Q, int64_t ldq, int64_t n, int64_t nev, double* X, int64_t ldx) {
  for (int64_t c = blockIdx.y; c < nev; c += gridDim.y)   // grid.y is capped at 65535
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double q = Q[SK_IDX(k, c, ldq)];
    double re = 0.0, im = 0.0;
    switch (k & 3) {
      case 0: re = q; break;
      case 1: im = q; break;
      case 2: re = -q; break;
      default: im = -q; break;
    }
    X[SK_IDX(k, c, ldx)] = re;
    X[SK_IDX(k, nev + c, ldx)] = im;
  }
}

// ------------------------------------------------------------------------------------
// Fused block re-orthogonalisation (reading R9(4)): one cooperative launch for all 32-vector
// blocks.  CTA c owns the rows [c R, (c+1) R) of every vector, so a block only depends on
// rows this CTA wrote for the earlier blocks; grid barriers are needed only around the
// cross-CTA reductions of the Gram matrices (8 per block: 2 per CGS pass, 2 per CholQR pass).
// The row slices are staged column-major in shared memory (LD = 4 mod 16: conflict-free
// DMMA fragments for both A = X^T and A = X); all products run on DMMA m8n8k4.
static constexpr int kReorthMaxG = 160;   // >= co-resident CTAs (1 per SM)
static constexpr int kRfCnt = 64 * 32;    // Gram partial: 64 (previous) x 32 (block)
static constexpr int kRfHLD = 36;         // H / R^-1 row stride (4 mod 16)

struct ReorthArgs {
  double* Q; int64_t ldq; int64_t n;
  const int64_t* blk; int nblk;   // per block: k0, p0, nb (columns relative to Q)
  double* part;                    // G x kRfCnt partials, then kRfCnt reduced
  int R, LDR;                      // rows per CTA (multiple of 8), smem column stride
  long long* dbg = nullptr;        // optional phase timing (SKEWEIG_REORTH_DBG), CTA 0
  unsigned* gbar = nullptr;        // grid barrier counter (zeroed before the launch)
};

// partial Gram: out(i, j) = sum_r X(r, i) Y(r, j), i < 8*FI (X columns), j < 32; X, Y column-major
// in smem (LDR); warp w takes fragment row fi = w % FI_TOTAL groups.
__device__ __forceinline__ void rf_gram(const double* Xs, const double* Ys, int LDR, int R, int fi_cnt, int sym,
                                        double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, t = lane & 3;
  if (!sym) {   // fi_cnt x 4 fragments: warp w -> fragment row w, all 4 column fragments
    if (warp < fi_cnt) {
      double acc[4][2] = {};
      const double* xa = Xs + (8 * warp + gq) * LDR + t;
      for (int k = 0; k < R; k += 4) {
        const double a = xa[k];
#pragma unroll
        for (int f = 0; f < 4; f++) dmma884(acc[f][0], acc[f][1], a, Ys[(8 * f + gq) * LDR + k + t]);
      }
#pragma unroll
      for (int f = 0; f < 4; f++)
#pragma unroll
        for (int h = 0; h < 2; h++) out[(8 * warp + gq) + 64 * (8 * f + 2 * t + h)] = acc[f][h];
    }
  } else {      // 4 x 4 fragments of Y^T Y: warp w -> row fragment w & 3, column fragments 2 (w >> 2) + {0, 1}
    const int fi = warp & 3, fj0 = 2 * (warp >> 2);
    double acc[2][2] = {};
    const double* xa = Xs + (8 * fi + gq) * LDR + t;
    for (int k = 0; k < R; k += 4) {
      const double a = xa[k];
#pragma unroll
      for (int f = 0; f < 2; f++) dmma884(acc[f][0], acc[f][1], a, Ys[(8 * (fj0 + f) + gq) * LDR + k + t]);
    }
#pragma unroll
    for (int f = 0; f < 2; f++)
#pragma unroll
      for (int h = 0; h < 2; h++) out[(8 * fi + gq) + 64 * (8 * (fj0 + f) + 2 * t + h)] = acc[f][h];
  }
}

// Y(r, :) = (ACC ? Y(r, :) : 0) + A(r, :) B, A = As column-major (K columns), B = Bs[k * kRfHLD + j];
// warps own 8-row tiles (all 32 columns), so the in-place A = Y case is race free.
template <bool ACC>
__device__ __forceinline__ void rf_rowmul(const double* As, double* Ys, int LDR, int R, int K, const double* Bs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, t = lane & 3;
  for (int rt = warp; rt < R / 8; rt += 8) {
    const int r = 8 * rt + gq;
    double acc[4][2];
#pragma unroll
    for (int f = 0; f < 4; f++)
#pragma unroll
      for (int h = 0; h < 2; h++) acc[f][h] = ACC ? Ys[(8 * f + 2 * t + h) * LDR + r] : 0.0;
    for (int k = 0; k < K; k += 4) {
      const double a = As[(k + t) * LDR + r];
#pragma unroll
      for (int f = 0; f < 4; f++) dmma884(acc[f][0], acc[f][1], a, Bs[(k + t) * kRfHLD + 8 * f + gq]);
    }
    __syncwarp();
#pragma unroll
    for (int f = 0; f < 4; f++)
#pragma unroll
      for (int h = 0; h < 2; h++) Ys[(8 * f + 2 * t + h) * LDR + r] = acc[f][h];
  }
}

// cross-CTA sum of the partials (fixed order per element: lane-strided over CTAs, then a
// warp tree), one element per warp, all warps of the grid
__device__ __forceinline__ void rf_reduce(const double* part, int G, int cnt, double* H) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), nw = gridDim.x * (blockDim.x >> 5);
  for (int e = gw; e < cnt; e += nw) {
    double v[kReorthMaxG / 32];
#pragma unroll
    for (int q = 0; q < kReorthMaxG / 32; q++) {   // all loads in flight, then a fixed-order sum
      const int c = lane + 32 * q;
      v[q] = (c < G) ? __ldcg(part + (size_t)c * kRfCnt + e) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kReorthMaxG / 32; q++) s += v[q];
    s = warp_sum(s);
    if (lane == 0) H[e] = s;
  }
}

// columns [c0, c0 + nvalid) of Q, rows [r0, r0 + nr), into smem columns 0 .. ntot-1 (LDR);
// rows nr..R-1 and columns nvalid..ntot-1 zero-filled.  cp.async: every copy in flight.
__device__ __forceinline__ void rf_load_cols(double* dst, const double* Q, int64_t ldq, int64_t r0, int nr, int R,
                                             int LDR, int64_t c0, int nvalid, int ntot) {
  for (int j = 0; j < ntot; j++) {
    const bool cv = j < nvalid;
    const double* src = Q + SK_IDX(r0, c0 + (cv ? j : 0), ldq);
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      const bool ok = cv && r < nr;
      cp_async8(dst + j * LDR + r, ok ? src + r : Q, ok ? 8 : 0);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
}

__global__ void __launch_bounds__(256, 1) td_reorth_fused_kernel(ReorthArgs ra) {
  unsigned bar_epoch = 0;
  extern __shared__ __align__(16) double rsm[];
  const int LDR = ra.LDR, R = ra.R, G = gridDim.x;
  double* Ys = rsm;                      // 32 x LDR
  double* Qs = Ys + 32 * LDR;            // 64 x LDR
  double* Bs = Qs + 64 * LDR;            // 64 x kRfHLD (-H, or (L^-1)^T)
  double* Ls = Bs + 64 * kRfHLD;         // 32 x 33 Cholesky factor
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int nr = (int)smax<int64_t>(0, smin<int64_t>(R, ra.n - r0));
  double* mypart = ra.part + (size_t)blockIdx.x * kRfCnt;
  double* Hg = ra.part + (size_t)G * kRfCnt;
  // Qs columns 0..qcnt-1 hold this CTA's rows of the finished vectors [qcache, qcache + qcnt)
  // (the previous block): the usual CGS window needs no reload
  int64_t qcache = -1;
  int qcnt = 0;
  const bool prof = ra.dbg != nullptr && blockIdx.x == 0 && tid == 0;
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tp = prof ? clock64() : 0;
#define RF_TS(k) do { if (prof) { long long _t = clock64(); ph[k] += _t - tp; tp = _t; } } while (0)
  for (int b = 0; b < ra.nblk; b++) {
    const int64_t k0 = ra.blk[3 * b], p0 = ra.blk[3 * b + 1];
    const int nb = (int)ra.blk[3 * b + 2];
    rf_load_cols(Ys, ra.Q, ra.ldq, r0, nr, R, LDR, k0, nb, 32);
    __syncthreads();
    // CGS2 against the previous vectors [p0, k0), chunks of <= 64
    for (int pass = 0; pass < 2; pass++) {
      for (int64_t q0 = p0; q0 < k0; q0 += 64) {
        const int p = (int)smin<int64_t>(64, k0 - q0), p8 = (p + 7) & ~7;
        if (!(q0 == qcache && p == qcnt)) {
          rf_load_cols(Qs, ra.Q, ra.ldq, r0, nr, R, LDR, q0, p, p8);
          qcache = -1;
        }
        __syncthreads();
        RF_TS(0);
        rf_gram(Qs, Ys, LDR, R, p8 / 8, 0, mypart);
        RF_TS(1);
        grid_barrier(ra.gbar, bar_epoch);
        RF_TS(2);
        rf_reduce(ra.part, G, 64 * 32, Hg);
        RF_TS(3);
        grid_barrier(ra.gbar, bar_epoch);
        RF_TS(2);
#pragma unroll 8
        for (int e = tid; e < 64 * 32; e += 256) {
          const int i = e & 63, j = e >> 6;
          if (i < p8) Bs[i * kRfHLD + j] = -__ldcg(Hg + e);
        }
        __syncthreads();
        RF_TS(0);
        rf_rowmul<true>(Qs, Ys, LDR, R, p8, Bs);   // Y -= Qp H
        RF_TS(4);
        __syncthreads();
      }
    }
    // CholQR2 inside the block: G = Y^T Y = L L^T, Y <- Y L^-T
    for (int pass = 0; pass < 2; pass++) {
      RF_TS(0);
      rf_gram(Ys, Ys, LDR, R, 4, 1, mypart);
      RF_TS(1);
      grid_barrier(ra.gbar, bar_epoch);
      RF_TS(2);
      rf_reduce(ra.part, G, 64 * 32, Hg);
      RF_TS(3);
      grid_barrier(ra.gbar, bar_epoch);
      RF_TS(2);
      if (warp == 0) {
        double a[32];
#pragma unroll
        for (int k = 0; k < 32; k++) a[k] = (lane < nb && k < nb) ? __ldcg(Hg + lane + 64 * k) : (lane == k ? 1.0 : 0.0);
        double rdiag = 1.0;   // lane j: 1 / L_jj
#pragma unroll
        for (int j = 0; j < 32; j++) {   // right-looking Cholesky, lane i holds row i (no divisions)
          const double r = rsqrt(fmax(__shfl_sync(0xffffffffu, a[j], j), 1e-300));
          const double lij = lane >= j ? a[j] * r : 0.0;   // lane j: d * rsqrt(d) = sqrt(d)
          if (lane == j) rdiag = r;
          a[j] = lij;
#pragma unroll
          for (int k = j + 1; k < 32; k++) a[k] -= lij * __shfl_sync(0xffffffffu, lij, k);
        }
#pragma unroll
        for (int k = 0; k < 32; k++) Ls[lane * 33 + k] = (k < lane) ? a[k] : (k == lane ? rdiag : 0.0);
        __syncwarp();
        // lane j: column j of L^-1 by forward substitution (x_i = 0 for i < j); Ls holds
        // 1 / L_ii on its diagonal
        double x[32];
#pragma unroll
        for (int i = 0; i < 32; i++) {
          double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
          for (int k = 0; k < i; k++) s -= Ls[i * 33 + k] * x[k];
          x[i] = s * Ls[i * 33 + i];
        }
        // B(k, j) = (L^-1)(j, k):  lane j holds (L^-1)(., j) -> row j of B
#pragma unroll
        for (int k = 0; k < 32; k++) Bs[lane * kRfHLD + k] = x[k];
      }
      __syncthreads();
      RF_TS(5);
      rf_rowmul<false>(Ys, Ys, LDR, R, 32, Bs);
      RF_TS(4);
      __syncthreads();
    }
    for (int j = 0; j < 32; j++)   // write back, and keep the block as the next CGS window
      for (int r = tid; r < R; r += 256) {
        const double y = Ys[j * LDR + r];
        if (j < nb && r < nr) ra.Q[SK_IDX(r0 + r, k0 + j, ra.ldq)] = y;
        Qs[j * LDR + r] = y;
      }
    qcache = k0;
    qcnt = nb;
    __syncthreads();
    RF_TS(6);
  }
  if (prof) for (int k = 0; k < 8; k++) ra.dbg[k] = ph[k];
#undef RF_TS
}

static constexpr int kReorthNB = 32;
static constexpr int64_t kGramRows = 128;

void trid_reserve(Arena& ar, int64_t n, int64_t nev, bool vectors, TridWork& w, int window) {
  int64_t nn = std::max<int64_t>(n, 1);
  w.a2 = ar.take<double>(nn);
  w.lamc = ar.take<double>(nn + 1024);   // + all-gather padding (<= one slice per rank)
  w.gtask = ar.take<double>(nn);
  w.tsk = ar.take<int64_t>(3 * nn);
  w.cgrid = ar.take<int>(kCountGrid + 1);
  w.scal = ar.take<double>(8);
  if (!vectors) return;
  int64_t ne = std::max<int64_t>(nev, 1);
  w.lamv = ar.take<double>(ne);
  w.gblk = ar.take<double>(ne);
  w.vblk = ar.take<int64_t>(2 * ne);
  w.single = ar.take<unsigned char>(ne);
  // bound the interleaved LU workspace: 16 GiB up to n = 40000, 4 GiB beyond (n = 65536 with
  // vectors on 4 GPUs must fit next to A, the reflector stores and X in 178 GiB)
  const int64_t lu_cap = (nn > 40000) ? (4ll << 30) : (16ll << 30);
  int64_t batch = std::max<int64_t>(1, std::min<int64_t>(ne, lu_cap / (49 * nn)));
  w.batch = batch;
  w.inv = ar.take<double>((size_t)5 * nn * batch + batch);
  w.inv_in = ar.take<unsigned char>((size_t)nn * batch);
  w.nfail = ar.take<int>(1);
  int64_t nchunks = (nn + kGramRows - 1) / kGramRows;
  int p = window + kReorthNB;
  w.part = ar.take<double>((size_t)nchunks * p * kReorthNB + (size_t)p * kReorthNB);
  w.H = ar.take<double>((size_t)p * kReorthNB);
  w.Rinv = ar.take<double>((size_t)kReorthNB * kReorthNB);
  w.rpart = ar.take<double>((size_t)(kReorthMaxG + 1) * kRfCnt);
  w.rblk = ar.take<int64_t>((size_t)3 * ((ne + kReorthNB - 1) / kReorthNB + 1));
  w.gbar = ar.take<unsigned>(64);
}

static cudaError_t reorth_project(const double* Qp, int64_t ldq, int p, double* Y, int64_t ldy, int nb, int64_t n,
                                  TridWork& w, cudaStream_t st) {
  int64_t nchunks = (n + kGramRows - 1) / kGramRows;
  {
    cudaError_t e = set_smem_attr((const void*)td_gram_partial, 120 * 1024);
    if (e) return e;
  }
  KScope ks(KC_TRID_REORTH, st, 2);
  td_gram_partial<<<(unsigned)nchunks, 256, (size_t)(p + nb) * (kGramRows + 1) * 8, st>>>(Qp, ldq, p, Y, ldy, nb, n,
                                                                                          kGramRows, w.part);
  int cnt = p * nb;
  td_reduce_partials<<<(cnt + 255) / 256, 256, 0, st>>>(w.part, (int)nchunks, cnt, w.H);
  return cudaGetLastError();
}

// ---- device-side bookkeeping (one unreduced block, i.e. no exact zero in alpha)
// scal[0] = Gershgorin bound g, scal[1] = pivmin = DBL_MIN max(1, max alpha^2), scal[2] =
// number of exact zeros in alpha; a2 = alpha^2 (a2[n-1] = 0).  The same arithmetic as the
// host path (same max / sum order is irrelevant: maxima are exact).
__global__ void __launch_bounds__(1024) td_prep_kernel(const double* alpha, int64_t n, double* a2, double* scal) {
  __shared__ double sg[32], sa[32];
  __shared__ int sz[32];
  double gm = 0.0, am = 0.0;
  int nz = 0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    const double ak = (k + 1 < n) ? alpha[k] : 0.0;
    a2[k] = ak * ak;
    am = fmax(am, ak * ak);
    nz += (k + 1 < n && ak == 0.0) ? 1 : 0;
    gm = fmax(gm, (k > 0 ? fabs(alpha[k - 1]) : 0.0) + fabs(ak));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
    am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { sg[warp] = gm; sa[warp] = am; sz[warp] = nz; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    gm = lane < nw ? sg[lane] : 0.0;
    am = lane < nw ? sa[lane] : 0.0;
    nz = lane < nw ? sz[lane] : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
      am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
      nz += __shfl_xor_sync(0xffffffffu, nz, o);
    }
    if (lane == 0) { scal[0] = gm; scal[1] = DBL_MIN * fmax(1.0, am); scal[2] = (double)nz; }
  }
}

// Per-vector data of the inverse-iteration / twisted stage from the descending eigenvalues of
// one block, the device version of the host loops (R9): dstein's perturbation
// lambda_k <- lambda_{k-1} - 10 eps g (sequential inside a run of close values; a run can only
// continue across a gap < nev * 10 eps g, so threads start at the gaps above that and walk),
// clusters (gap < 1e-6 g: a max-scan of the cluster starts), isolated flags, the first ghost
// vector vlo = min(k0 - W, cluster start of k0) and the re-orthogonalisation block list.
struct VecPrepArgs {
  const double* lam; int64_t nev; int64_t n; double g;
  double* lv; double* gv; int64_t* vb; unsigned char* single; int64_t* cs;
  int64_t k0v, k1v; int W; int64_t* rblk; int64_t* vlo;
};
__global__ void __launch_bounds__(1024) td_vecprep_kernel(VecPrepArgs a) {
  __shared__ int64_t part[1024];
  const int T = blockDim.x, t = threadIdx.x;
  const int64_t nev = a.nev, C = (nev + T - 1) / T;
  const int64_t i0 = smin<int64_t>(nev, (int64_t)t * C), i1 = smin<int64_t>(nev, i0 + C);
  const double del = 10.0 * DBL_EPSILON * a.g, thr = 1e-6 * a.g, brk = (double)nev * del;
  // cluster starts: cs[i] = the last i' <= i with i' == 0 or lam[i'-1] - lam[i'] >= thr
  int64_t last = -1;
  for (int64_t i = i0; i < i1; i++)
    if (i == 0 || !(a.lam[i - 1] - a.lam[i] < thr)) last = i;
  part[t] = last;
  __syncthreads();
  for (int o = 1; o < T; o <<= 1) {   // inclusive max-scan of the chunk summaries
    const int64_t v = (t >= o) ? part[t - o] : -1;
    __syncthreads();
    part[t] = smax<int64_t>(part[t], v);
    __syncthreads();
  }
  int64_t run = (t > 0) ? part[t - 1] : -1;
  for (int64_t i = i0; i < i1; i++) {
    if (i == 0 || !(a.lam[i - 1] - a.lam[i] < thr)) run = i;
    a.cs[i] = run;
    a.gv[i] = a.g;
    a.vb[i] = 0;
    a.vb[nev + i] = a.n;
  }
  // perturbation, sequential within runs (bit-identical to the host loop)
  for (int64_t i = i0; i < i1; i++) {
    if (!(i == 0 || !(a.lam[i - 1] - a.lam[i] < brk))) continue;
    double lastv = a.lam[i];
    a.lv[i] = lastv;
    for (int64_t j = i + 1; j < nev && a.lam[j - 1] - a.lam[j] < brk; j++) {
      double x = a.lam[j];
      if (lastv - x < del) x = lastv - del;
      a.lv[j] = x;
      lastv = x;
    }
  }
  __syncthreads();
  for (int64_t i = t; i < nev; i += T)
    a.single[i] = (a.cs[i] == i && (i + 1 == nev || a.cs[i + 1] == i + 1) && a.lv[i] == a.lam[i]) ? 1 : 0;
  const int64_t vlo = smin<int64_t>(smax<int64_t>(0, a.k0v - a.W), a.cs[a.k0v]);
  if (t == 0) *a.vlo = vlo;
  for (int64_t q = t; vlo + q * kReorthNB < a.k1v; q += T) {
    const int64_t k0 = vlo + q * kReorthNB;
    int64_t p0 = smax<int64_t>(vlo, k0 - a.W);
    const int64_t c = smax<int64_t>(vlo, a.cs[k0]);
    if (c < p0) p0 = c;
    a.rblk[3 * q] = k0 - vlo;
    a.rblk[3 * q + 1] = p0 - vlo;
    a.rblk[3 * q + 2] = smin<int64_t>(kReorthNB, a.k1v - k0);
  }
}

static cudaError_t trid_vectors(int64_t n, const double* alpha_d, int64_t nev, double* Q, int64_t ldq, TridWork& w,
                                const Params& prm, cudaStream_t st, int64_t vlo, int64_t vhi, double pivmin,
                                const std::vector<int64_t>* clus_host, bool blk_on_device, int64_t* nfail_out);

// Host path of the tridiagonal stage, for a matrix that splits into unreduced blocks (an exact
// zero in alpha): per-block Gershgorin intervals and tasks, selection of the top nev, dstein's
// per-block perturbation, clusters -- then the shared vector stage.
static cudaError_t trid_run_host(int64_t n, const double* alpha_d, int64_t nev, double* lam_out, double* Q,
                                 int64_t ldq, TridWork& w, const Params& prm, int64_t* nfail_out, cudaStream_t st,
                                 int64_t k0v, int64_t k1v, int64_t* vlo_out, const Dist* d) {
  cudaError_t e;
  // alpha to host (n-1 doubles): split points, Gershgorin bounds, task lists
  std::vector<double> al(std::max<int64_t>(n - 1, 1), 0.0);
  if (n > 1) {
    e = cudaMemcpyAsync(al.data(), alpha_d, sizeof(double) * (n - 1), cudaMemcpyDeviceToHost, st);
    if (e) return e;
    e = cudaStreamSynchronize(st);
    if (e) return e;
  }
  std::vector<int64_t> bs{0};
  for (int64_t k = 0; k + 1 < n; k++) if (al[k] == 0.0) bs.push_back(k + 1);
  bs.push_back(n);
  const int64_t nblk = (int64_t)bs.size() - 1;
  double amax2 = 1.0;
  for (int64_t k = 0; k + 1 < n; k++) amax2 = std::max(amax2, al[k] * al[k]);
  const double pivmin = DBL_MIN * amax2;
  std::vector<double> a2(std::max<int64_t>(n, 1), 0.0);
  for (int64_t k = 0; k + 1 < n; k++) a2[k] = al[k] * al[k];
  std::vector<int64_t> ts0, tm, ti, tb;
  std::vector<double> gb(nblk, 0.0);
  for (int64_t b = 0; b < nblk; b++) {
    int64_t s0 = bs[b], m = bs[b + 1] - bs[b];
    double g = 0.0;
    for (int64_t k = 0; k < m; k++) {
      double r = (k > 0 ? std::fabs(al[s0 + k - 1]) : 0.0) + (k + 1 < m ? std::fabs(al[s0 + k]) : 0.0);
      g = std::max(g, r);
    }
    gb[b] = g;
    int64_t kb = std::min(m, nev);
    for (int64_t i = 0; i < kb; i++) { ts0.push_back(s0); tm.push_back(m); ti.push_back(m - 1 - i); tb.push_back(b); }
  }
  const int64_t ntask = (int64_t)ts0.size();
  std::vector<double> tg(ntask);
  for (int64_t q = 0; q < ntask; q++) tg[q] = gb[tb[q]];
  // each unreduced block bisects inside its own Gershgorin interval.  Distributed: rank r
  // computes the contiguous task slice [r*cnt, (r+1)*cnt) and an NCCL all-gather assembles
  // them in order (every rank then holds bit-identical eigenvalues).
  const int P = d ? d->P : 1;
  const int64_t cnt = (ntask + P - 1) / P;
  const int64_t qa = std::min<int64_t>(ntask, (int64_t)(d ? d->rank : 0) * cnt), qb = std::min<int64_t>(ntask, qa + cnt);
  std::vector<double> lamc(ntask);
  {
    e = cudaMemcpyAsync(w.a2, a2.data(), sizeof(double) * std::max<int64_t>(n, 1), cudaMemcpyHostToDevice, st);
    if (e) return e;
    int64_t* d_s0 = w.tsk;
    int64_t* d_m = w.tsk + n;
    int64_t* d_i = w.tsk + 2 * n;
    cudaMemcpyAsync(d_s0, ts0.data(), sizeof(int64_t) * ntask, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_m, tm.data(), sizeof(int64_t) * ntask, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_i, ti.data(), sizeof(int64_t) * ntask, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(w.gtask, tg.data(), sizeof(double) * ntask, cudaMemcpyHostToDevice, st);
    {
      // points per multisection round (K lanes share one eigenvalue, ~log_{K+1}(2/eps)
      // rounds): as many as keep about half the device's thread slots busy.  Measured at
      // n = 32768: one GPU (16384 eigenvalues) K = 8, 95 ms; 4 GPUs (4096 per rank) K = 32,
      // 62 ms vs K = 8, 98 ms -- the per-round Sturm chain latency dominates small slices.
      KScope ks(KC_TRID_BISECT, st);
      int nsm = 148, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      const int64_t slots = (int64_t)nsm * 1024, nt = qb - qa;
      int K = (nt * 32 <= slots) ? 32 : (nt * 16 <= slots) ? 16 : 8;
      if (const char* v = getenv("SKEWEIG_MSECT_K")) K = atoi(v) == 32 ? 32 : atoi(v) == 16 ? 16 : 8;   // experiments
      // count grid for a single unreduced block (the generic case): ~one round's worth of counts
      int M = 0;
      if (nblk == 1 && n >= 4 && nt > 0) {
        M = (int)std::min<int64_t>(kCountGrid, std::max<int64_t>(256, 8 * n));
        if (const char* v = getenv("SKEWEIG_COUNT_GRID")) M = std::min(kCountGrid, std::max(0, atoi(v)));   // experiments
        if (M > 1)
          td_count_grid_kernel<<<(unsigned)((M + 127) / 128), 128, 0, st>>>(w.a2, 0, (int)n, gb[0], M, pivmin, w.cgrid);
      }
      if (nt > 0) {
        const unsigned grid = (unsigned)((nt * K + 127) / 128);
        if (K == 32)
          td_msect_kernel<32><<<grid, 128, 0, st>>>(w.a2, d_s0, d_m, d_i, w.gtask, qa, qb, pivmin, w.lamc, w.cgrid, M, 0, 0.0);
        else if (K == 16)
          td_msect_kernel<16><<<grid, 128, 0, st>>>(w.a2, d_s0, d_m, d_i, w.gtask, qa, qb, pivmin, w.lamc, w.cgrid, M, 0, 0.0);
        else td_msect_kernel<8><<<grid, 128, 0, st>>>(w.a2, d_s0, d_m, d_i, w.gtask, qa, qb, pivmin, w.lamc, w.cgrid, M, 0, 0.0);
      }
    }
    if (P > 1) {
      KScope ks(KC_COLL, st);
      if (coll_allgather(*d, w.lamc, (size_t)cnt, st)) return cudaErrorUnknown;
    }
    e = cudaMemcpyAsync(lamc.data(), w.lamc, sizeof(double) * ntask, cudaMemcpyDeviceToHost, st);
    if (e) return e;
    e = cudaStreamSynchronize(st);
    if (e) return e;
  }
  // stable selection of the nev largest (ties in block order)
  std::vector<int64_t> ord(ntask);
  for (int64_t i = 0; i < ntask; i++) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](int64_t x, int64_t y) { return lamc[x] > lamc[y]; });
  std::vector<double> lam(nev);
  for (int64_t i = 0; i < nev; i++) lam[i] = lamc[ord[i]];
  e = cudaMemcpyAsync(lam_out, lam.data(), sizeof(double) * nev, cudaMemcpyHostToDevice, st);
  if (e) return e;
  if (!Q) return cudaStreamSynchronize(st);

  // per-vector block info and perturbed eigenvalues (dstein: within a block, descending,
  // lambda_k <- lambda_{k-1} - 10 eps g when closer)
  std::vector<double> lv(nev), gv(nev);
  std::vector<int64_t> vb(2 * nev);
  std::vector<int64_t> last_in_blk(nblk, -1);
  std::vector<double> last_lam(nblk, 0.0);
  std::vector<int64_t> clus_start(nev, 0);
  for (int64_t i = 0; i < nev; i++) {
    int64_t b = tb[ord[i]];
    double g = gb[b];
    double x = lam[i];
    if (last_in_blk[b] >= 0 && last_lam[b] - x < 10.0 * DBL_EPSILON * g) x = last_lam[b] - 10.0 * DBL_EPSILON * g;
    last_lam[b] = x;
    last_in_blk[b] = i;
    lv[i] = x; gv[i] = g;
    vb[i] = bs[b]; vb[nev + i] = bs[b + 1] - bs[b];
  }
  // clusters (global order): consecutive gap < 1e-6 * gmax
  double gmax = 0.0;
  for (double g : gb) gmax = std::max(gmax, g);
  for (int64_t i = 1; i < nev; i++) clus_start[i] = (lam[i - 1] - lam[i] < 1e-6 * gmax) ? clus_start[i - 1] : i;
  // isolated eigenvalues (a cluster of one, no dstein perturbation) take the twisted
  // factorization; cluster members keep dstein's iterated solves with random start vectors
  std::vector<unsigned char> single(nev);
  for (int64_t i = 0; i < nev; i++)
    single[i] = (clus_start[i] == i && (i + 1 == nev || clus_start[i + 1] == i + 1) && lv[i] == lam[i]) ? 1 : 0;
  cudaMemcpyAsync(w.single, single.data(), (size_t)nev, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(w.lamv, lv.data(), sizeof(double) * nev, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(w.gblk, gv.data(), sizeof(double) * nev, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(w.vblk, vb.data(), sizeof(int64_t) * 2 * nev, cudaMemcpyHostToDevice, st);
  // vectors [vlo, vhi): the requested range [k0v, k1v) plus the reorthogonalisation window and
  // the cluster members before it (ghost vectors, discarded by the caller)
  const int W = prm.reorth_w;
  int64_t vlo = std::min<int64_t>(std::max<int64_t>(0, k0v - W), clus_start[k0v]);
  if (vlo_out) *vlo_out = vlo;
  // the host vectors above must outlive their asynchronous copies
  e = trid_vectors(n, alpha_d, nev, Q, ldq, w, prm, st, vlo, k1v, pivmin, &clus_start, false, nfail_out);
  if (e) return e;
  return cudaStreamSynchronize(st);
}

// Vector stage (shared): dstein / twisted vectors of [vlo, vhi) into Q, the re-orthogonalisation,
// the failure count.  Needs lamv, gblk, vblk, single on the device; the cluster starts on the
// host (clus_host) or, with blk_on_device, the re-orthogonalisation block list in w.rblk.
static cudaError_t trid_vectors(int64_t n, const double* alpha_d, int64_t nev, double* Q, int64_t ldq, TridWork& w,
                                const Params& prm, cudaStream_t st, int64_t vlo, int64_t vhi, double pivmin,
                                const std::vector<int64_t>* clus_host, bool blk_on_device, int64_t* nfail_out) {
  cudaError_t e;
  const int W = prm.reorth_w;
  cudaMemsetAsync(w.nfail, 0, sizeof(int), st);
  // pass 0: cluster members by dstein (batches sized for its five LU arrays); pass 1: isolated
  // eigenvalues by the twisted factorization (three arrays: 5/3 larger batches in the same
  // workspace, one batch at n = 32768)
  const int64_t batch_t = std::max<int64_t>(1, std::min<int64_t>(nev, (5 * w.batch) / 3 - 1));   // 3 n bt + bt <= 5 n batch
  for (int pass = 0; pass < 2; pass++) {
    const int64_t bsz = pass ? batch_t : w.batch;
    for (int64_t c0 = vlo; c0 < vhi; c0 += bsz) {
      int64_t nb = std::min(bsz, vhi - c0);
      InvArgs a;
      a.alpha = alpha_d; a.vs0 = w.vblk; a.vm = w.vblk + nev; a.lam = w.lamv; a.gblk = w.gblk;
      a.nvec = nb; a.col0 = c0;
      size_t stride = (size_t)n * nb;
      if (pass == 0) {
        a.wa = w.inv; a.wb = w.inv + stride; a.wc = w.inv + 2 * stride; a.wd = w.inv + 3 * stride;
        a.y = w.inv + 4 * stride; a.scale = w.inv + 5 * stride;
      } else {
        a.wa = w.inv; a.wb = w.inv + stride; a.wc = nullptr; a.wd = nullptr;
        a.y = w.inv + 2 * stride; a.scale = w.inv + 3 * stride;
      }
      a.win = w.inv_in; a.seed = prm.seed; a.nfail = w.nfail;
      a.single = w.single; a.pivmin = pivmin;
      KScope ks(KC_TRID_INV, st, 2);
      // one warp per CTA: the latency-bound per-vector chains spread over every SM (per-SM
      // outstanding-load capacity, not the thread count, limits these kernels)
      if (pass == 0) td_inverse_kernel<8><<<(unsigned)((nb + 31) / 32), 32, 0, st>>>(a);
      else td_twisted_kernel<<<(unsigned)((nb + 15) / 16), 32, 0, st>>>(a);
      dim3 grid((unsigned)((n + 31) / 32), (unsigned)((nb + 31) / 32));
      td_place_vectors<<<grid, dim3(32, 8), 0, st>>>(a.y, a.scale, nb, c0, w.vblk, w.vblk + nev, n, Q, ldq, c0 - vlo,
                                                     w.single, pass);
    }
  }
  e = cudaGetLastError();
  if (e) return e;
  if (const char* ro = getenv("SKEWEIG_REORTH_OFF"))   // experiments: the vectors as computed
    if (atoi(ro) == 1) return cudaSuccess;
  // the cluster starts on the host (the kernel-per-step fallback, or the host path)
  std::vector<int64_t> cs_local;
  auto clus = [&]() -> const std::vector<int64_t>& {
    if (clus_host) return *clus_host;
    if (cs_local.empty()) {
      cs_local.resize(nev);
      cudaMemcpyAsync(cs_local.data(), w.tsk, sizeof(int64_t) * nev, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
    }
    return cs_local;
  };
  // re-orthogonalisation in blocks of 32 (descending order): one fused cooperative launch
  // when the per-CTA row slices fit in shared memory, else the kernel-per-step sequence
  bool fused = false;
  {
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int G = (int)smin<int64_t>(smin<int64_t>(nsm, kReorthMaxG), smax<int64_t>(1, (n + 7) / 8));
    if (const char* v = getenv("SKEWEIG_REORTH_G")) G = std::max(1, std::min(G, atoi(v)));   // experiments
    const int R = (int)((((n + G - 1) / G) + 7) & ~int64_t(7));
    const int LDR = R + (((4 - R) % 16) + 16) % 16;
    const size_t smem = ((size_t)96 * LDR + 64 * kRfHLD + 32 * 33) * sizeof(double);
    const char* fz = getenv("SKEWEIG_REORTH_FUSED");   // experiments: 0 = kernel-per-step path
    fused = smem <= 227 * 1024 && !(fz && fz[0] == '0');
    if (fused) {
      e = set_smem_attr((const void*)td_reorth_fused_kernel, 227 * 1024);
      if (e) return e;
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, td_reorth_fused_kernel, 256, smem);
      fused = occ * nsm >= G;
    }
    if (fused) {
      std::vector<int64_t> blk;
      const int nblk = (int)((vhi - vlo + kReorthNB - 1) / kReorthNB);
      if (!blk_on_device) {
        const std::vector<int64_t>& clus_start = clus();
        for (int64_t k0 = vlo; k0 < vhi; k0 += kReorthNB) {
          int64_t p0 = std::max<int64_t>(vlo, k0 - W);
          const int64_t cs = std::max<int64_t>(vlo, clus_start[k0]);
          if (cs < p0) p0 = cs;
          blk.push_back(k0 - vlo);
          blk.push_back(p0 - vlo);
          blk.push_back(std::min<int64_t>(kReorthNB, vhi - k0));
        }
      }
      if (nblk > 0) {
        if (!blk_on_device) {
          e = cudaMemcpyAsync(w.rblk, blk.data(), sizeof(int64_t) * blk.size(), cudaMemcpyHostToDevice, st);
          if (e) return e;
        }
        ReorthArgs ra;
        ra.Q = Q; ra.ldq = ldq; ra.n = n; ra.blk = w.rblk; ra.nblk = nblk; ra.part = w.rpart; ra.R = R; ra.LDR = LDR;
        ra.gbar = w.gbar;
        e = cudaMemsetAsync(w.gbar, 0, sizeof(unsigned), st);
        if (e) return e;
        ra.dbg = nullptr;
        void* args[] = {&ra};
        KScope ks(KC_TRID_REORTH, st);
        e = cudaLaunchCooperativeKernel((void*)td_reorth_fused_kernel, dim3(G), dim3(256), args, smem, st);
        if (e) return e;
        if (!blk_on_device) {   // the host copy of blk must outlive the async copy
          e = cudaStreamSynchronize(st);
          if (e) return e;
        }
      }
    }
  }
  if (!fused) for (int64_t k0 = vlo; k0 < vhi; k0 += kReorthNB) {
    int nb = (int)std::min<int64_t>(kReorthNB, vhi - k0);
    int64_t p0 = std::max<int64_t>(vlo, k0 - W);
    int64_t cs = std::max<int64_t>(vlo, clus()[k0]);
    if (cs < p0) p0 = cs;
    double* Y = Q + SK_IDX(0, k0 - vlo, ldq);
    // CGS2 against [p0, k0) in chunks of <= 64 previous vectors
    for (int pass = 0; pass < 2; pass++) {
      for (int64_t q0 = p0; q0 < k0; q0 += 64) {
        int p = (int)std::min<int64_t>(64, k0 - q0);
        const double* Qp = Q + SK_IDX(0, q0 - vlo, ldq);
        e = reorth_project(Qp, ldq, p, Y, ldq, nb, n, w, st);
        if (e) return e;
        KScope ks(KC_TRID_REORTH, st);
        td_sub_proj<<<(unsigned)((n + 127) / 128), 128, (size_t)p * nb * 8, st>>>(Qp, ldq, p, w.H, Y, ldq, nb, n);
      }
    }
    // CholQR2 within the block
    if (nb > 1) {
      for (int pass = 0; pass < 2; pass++) {
        e = reorth_project(Y, ldq, nb, Y, ldq, nb, n, w, st);
        if (e) return e;
        KScope ks(KC_TRID_REORTH, st, 2);
        td_chol_inv<<<1, 32, 0, st>>>(w.H, nb, w.Rinv);
        td_apply_rinv<<<(unsigned)((n + 127) / 128), 128, (size_t)nb * nb * 8, st>>>(Y, ldq, nb, w.Rinv, n);
      }
    }
  }
  int nf = 0;
  e = cudaMemcpyAsync(&nf, w.nfail, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e) return e;
  e = cudaStreamSynchronize(st);
  *nfail_out = nf;
  return e;
}

// lam (nev, descending, device out); Q (n x nev, ldq) or null.  One unreduced block (the
// generic case): alpha^2, the Gershgorin bound, the bisection tasks, the per-vector data and
// the re-orthogonalisation blocks are all formed on the device; the host reads three scalars
// (one round trip) and, for a distributed range k0v > 0, the first ghost vector.  A matrix that
// splits (an exact zero in alpha) takes the host path above.
cudaError_t trid_run(int64_t n, const double* alpha_d, int64_t nev, double* lam_out, double* Q, int64_t ldq,
                     TridWork& w, const Params& prm, int64_t* nfail_out, cudaStream_t st, int64_t k0v, int64_t k1v,
                     int64_t* vlo_out, const Dist* d) {
  cudaError_t e;
  *nfail_out = 0;
  if (nev <= 0) return cudaSuccess;
  double sc[3] = {0.0, 0.0, 1.0};
  if (n > 1) {
    td_prep_kernel<<<1, 1024, 0, st>>>(alpha_d, n, w.a2, w.scal);
    e = cudaMemcpyAsync(sc, w.scal, sizeof(sc), cudaMemcpyDeviceToHost, st);
    if (e) return e;
    e = cudaStreamSynchronize(st);
    if (e) return e;
  }
  if (n < 4 || sc[2] != 0.0 || getenv("SKEWEIG_TRID_HOST"))   // SKEWEIG_TRID_HOST: experiments
    return trid_run_host(n, alpha_d, nev, lam_out, Q, ldq, w, prm, nfail_out, st, k0v, k1v, vlo_out, d);
  const double g = sc[0], pivmin = sc[1];
  const int P = d ? d->P : 1;
  const int64_t cnt = (nev + P - 1) / P;
  const int64_t qa = std::min<int64_t>(nev, (int64_t)(d ? d->rank : 0) * cnt), qb = std::min<int64_t>(nev, qa + cnt);
  {
    KScope ks(KC_TRID_BISECT, st);
    int nsm = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t slots = (int64_t)nsm * 1024, nt = qb - qa;
    int K = (nt * 32 <= slots) ? 32 : (nt * 16 <= slots) ? 16 : 8;
    if (const char* v = getenv("SKEWEIG_MSECT_K")) K = atoi(v) == 32 ? 32 : atoi(v) == 16 ? 16 : 8;   // experiments
    int M = (int)std::min<int64_t>(kCountGrid, std::max<int64_t>(256, 8 * n));
    if (const char* v = getenv("SKEWEIG_COUNT_GRID")) M = std::min(kCountGrid, std::max(0, atoi(v)));   // experiments
    if (nt > 0 && M > 1)
      td_count_grid_kernel<<<(unsigned)((M + 127) / 128), 128, 0, st>>>(w.a2, 0, (int)n, g, M, pivmin, w.cgrid);
    if (nt > 0) {
      const unsigned grid = (unsigned)((nt * K + 127) / 128);
      if (K == 32)
        td_msect_kernel<32><<<grid, 128, 0, st>>>(w.a2, nullptr, nullptr, nullptr, nullptr, qa, qb, pivmin, w.lamc,
                                                  w.cgrid, M, n, g);
      else if (K == 16)
        td_msect_kernel<16><<<grid, 128, 0, st>>>(w.a2, nullptr, nullptr, nullptr, nullptr, qa, qb, pivmin, w.lamc,
                                                  w.cgrid, M, n, g);
      else td_msect_kernel<8><<<grid, 128, 0, st>>>(w.a2, nullptr, nullptr, nullptr, nullptr, qa, qb, pivmin, w.lamc,
                                                    w.cgrid, M, n, g);
    }
  }
  if (P > 1) {
    KScope ks(KC_COLL, st);
    if (coll_allgather(*d, w.lamc, (size_t)cnt, st)) return cudaErrorUnknown;
  }
  // one block: task q is eigenvalue n-1-q, so the candidates are already descending
  e = cudaMemcpyAsync(lam_out, w.lamc, sizeof(double) * nev, cudaMemcpyDeviceToDevice, st);
  if (e) return e;
  if (!Q) return cudaSuccess;
  VecPrepArgs va;
  va.lam = w.lamc; va.nev = nev; va.n = n; va.g = g;
  va.lv = w.lamv; va.gv = w.gblk; va.vb = w.vblk; va.single = w.single; va.cs = w.tsk;
  va.k0v = k0v; va.k1v = k1v; va.W = prm.reorth_w; va.rblk = w.rblk; va.vlo = reinterpret_cast<int64_t*>(w.scal + 3);
  td_vecprep_kernel<<<1, 1024, 0, st>>>(va);
  int64_t vlo = 0;
  if (k0v > 0) {   // distributed range: the ghost window reaches back to the cluster start
    e = cudaMemcpyAsync(&vlo, w.scal + 3, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e) return e;
    e = cudaStreamSynchronize(st);
    if (e) return e;
  }
  if (vlo_out) *vlo_out = vlo;
  return trid_vectors(n, alpha_d, nev, Q, ldq, w, prm, st, vlo, k1v, pivmin, nullptr, true, nfail_out);
}

cudaError_t assemble_D(const double* Q, int64_t ldq, int64_t n, int64_t nev, double* X, int64_t ldx, cudaStream_t st) {
  if (nev <= 0) return cudaSuccess;
  dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(nev, 65535));
  KScope ks(KC_ASSEMBLE, st);
  assemble_D_kernel<<<grid, 256, 0, st>>>(Q, ldq, n, nev, X, ldx);
  return cudaGetLastError();
}

}  // namespace sk
