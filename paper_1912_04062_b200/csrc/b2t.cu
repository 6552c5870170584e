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

template <int MAXB>
__global__ void __launch_bounds__(256) chase_kernel(ChaseArgs a) {
  // Shared window: a ring of 2b column slots (+1 for the t = 0 column) in band storage,
  // slot(c) = (c - s - 1) mod 2b.  Task t of sweep s works on columns [r-b, r+b); the
  // block below its diagonal block (E_t, rows [r+L, e)) is exactly task t+1's left block,
  // so it stays in shared memory (loaded once, written back once, as task t+1's final
  // left block); each task loads only its diagonal-block columns [r, r+L) and writes back
  // its (final) left block and diagonal block.
  extern __shared__ __align__(16) double W[];
  __shared__ double vs[MAXB], ws[MAXB], zs[MAXB], ys[MAXB], sc[4];
  const int b = a.b;
  const int LDW = 2 * b + 2;   // LDW - 1 odd: the strided skew reads of D are conflict-free
  const int64_t n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool prof = a.dbg != nullptr && blockIdx.x == 0 && tid == 0;
  long long t_wait = 0, t_work = 0, ntasks = 0, tk = 0, tph[5] = {0, 0, 0, 0, 0}, tp = 0;
#define CH_TS(i) do { if (prof) { long long _n = clock64(); tph[i] += _n - tp; tp = _n; } } while (0)
  for (int64_t s = blockIdx.x; s < n - 2; s += gridDim.x) {
    const int64_t nt = chase_ntask(n, b, s);
    const int64_t ntprev = (s > 0) ? chase_ntask(n, b, s - 1) : 0;
    for (int64_t t = 0; t < nt; t++) {
      // ---- sweep s task t may run once sweep s-1 finished tasks 0..t+2 (their entry sets
      //      are then disjoint from this task's; checked against the sequential order)
      if (prof) tk = clock64();
      if (s > 0) {
        if (tid == 0) {
          const int need = (int)smin<int64_t>(t + 3, ntprev);
          volatile int* pr = a.progress + (s - 1);
          while (*pr < need) { __nanosleep(32); }
          __threadfence();
        }
        __syncthreads();
      }
      if (prof) { long long now = clock64(); t_wait += now - tk; tk = now; tp = now; ntasks++; }
      int64_t col, r, L;
      if (t == 0) { col = s; r = s + 1; L = smin<int64_t>(b, n - 1 - s); }
      else { col = s + 1 + (t - 1) * b; r = col + b; L = smin<int64_t>(b, n - r); }
      const int64_t e = smin<int64_t>(n, r + L + b);
      const int nl = (int)(r - col);          // columns of the left block (1 for t = 0)
      const int ne = (int)(e - r - L);         // rows of the block below
      const bool last = (t + 1 == nt);
      // column slots (32-bit, no division in the inner loops): left columns col + cc, and
      // the diagonal-block columns r + j
      const int B2 = 2 * b;
      const int sr0 = (int)((r - s - 1) % B2);
      const int sc0 = (t == 0) ? B2 : (int)((col - s - 1) % B2);
      auto sl_left = [&](int cc) -> int { if (t == 0) return B2; int x = sc0 + cc; return x >= B2 ? x - B2 : x; };
      auto sl_diag = [&](int j) -> int { int x = sr0 + j; return x >= B2 ? x - B2 : x; };
      // ---- load: t = 0 also the left column s; always the columns [r, r+L) rows [c, e).
      //      16-byte L2-coherent cp.async on even-widened band offsets (widened elements
      //      are only read, never written back).
      if (t == 0 && warp == 7) {
        const int d0 = (int)(r - col) & ~1, d1 = (int)(r + L - col);
        for (int d = d0 + 2 * lane; d < d1; d += 64) cp_async16(&W[B2 * LDW + d], &a.AB[d + col * a.ldab], 16);
      }
      for (int j = warp; j < L; j += 8) {
        const int64_t c = r + j;
        const int d1 = (int)(e - c);
        const int sj = sl_diag(j);
        for (int d = 2 * lane; d < d1; d += 64) cp_async16(&W[sj * LDW + d], &a.AB[d + c * a.ldab], 16);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      CH_TS(0);
      // ---- (a) Householder of x = A[r:r+L, col]  (dlarfg convention)
      const int scol = sl_left(0);
      if (warp == 0) {
        double s2 = 0.0;
        for (int i = 1 + lane; i < L; i += 32) { double x = W[scol * LDW + (r + i - col)]; s2 += x * x; }
        s2 = warp_sum(s2);
        double x0 = W[scol * LDW + (r - col)];
        double beta, tau, scal;
        if (s2 == 0.0) { beta = x0; tau = 0.0; scal = 0.0; }
        else {
          double nrm = sqrt(x0 * x0 + s2);
          beta = (x0 >= 0.0) ? -nrm : nrm;
          tau = (beta - x0) / beta;
          scal = 1.0 / (x0 - beta);
        }
        for (int i = lane; i < L; i += 32) {
          double v = (i == 0) ? 1.0 : W[scol * LDW + (r + i - col)] * scal;
          vs[i] = v;
          W[scol * LDW + (r + i - col)] = (i == 0) ? beta : 0.0;
        }
        if (lane == 0) sc[0] = tau;
      }
      __syncthreads();
      CH_TS(1);
      const double tau = sc[0];
      {   // store the reflector (v zero-padded to b by the initial memset)
        const int64_t blk = s / a.k2, c = s % a.k2;
        const int64_t gidx = a.gofs[blk] + t;
        double* dst = a.qv + (gidx * a.k2 + c) * b;
        for (int i = tid; i < L; i += 256) dst[i] = vs[i];
        if (tid == 0) a.qtau[gidx * a.k2 + c] = tau;
      }
      if (tau != 0.0) {
        // ---- y = tau v^T A[r:r+L, c] (left columns), w = tau D v, z = tau E v: 4 threads per item
        const int item = tid >> 2, part = tid & 3;
        double sy = 0.0, sw = 0.0, sz = 0.0;   // shuffles below run on all lanes (full mask)
        if (item >= 1 && item < nl) {
          const int sl = sl_left(item), d0 = nl - item;   // row r sits at offset r - c
#pragma unroll 4
          for (int i = part; i < L; i += 4) sy += vs[i] * W[sl * LDW + d0 + i];
        }
        if (item < L) {
          for (int j = part; j < item; j += 4) sw += W[sl_diag(j) * LDW + (item - j)] * vs[j];
          const int sr = sl_diag(item);
          for (int j = item + 1 + part; j < L; j += 4) sw -= W[sr * LDW + (j - item)] * vs[j];
        }
        if (item < ne) {
#pragma unroll 4
          for (int j = part; j < L; j += 4) sz += W[sl_diag(j) * LDW + (L + item - j)] * vs[j];
        }
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
          sy += __shfl_xor_sync(0xffffffffu, sy, o);
          sw += __shfl_xor_sync(0xffffffffu, sw, o);
          sz += __shfl_xor_sync(0xffffffffu, sz, o);
        }
        if (part == 0) {
          if (item < nl) ys[item] = tau * sy;
          if (item < L) ws[item] = tau * sw;
          if (item < ne) zs[item] = tau * sz;
        }
        __syncthreads();
        CH_TS(2);
        // ---- left block -= v y^T;  D_ij += v_i w_j - w_i v_j (i > j);  E_ij -= z_i v_j
#pragma unroll 4
        for (int cc = 1 + warp; cc < nl; cc += 8) {
          const int sl = sl_left(cc), d0 = nl - cc;
          const double yc = ys[cc];
          for (int i = lane; i < L; i += 32) W[sl * LDW + d0 + i] -= yc * vs[i];
        }
#pragma unroll 4
        for (int j = warp; j < L; j += 8) {
          const int sj = sl_diag(j);
          const double vj = vs[j], wj = ws[j];
          for (int i = j + 1 + lane; i < L; i += 32) W[sj * LDW + (i - j)] += vs[i] * wj - ws[i] * vj;
          for (int i = lane; i < ne; i += 32) W[sj * LDW + (L + i - j)] -= zs[i] * vj;
        }
      }
      __syncthreads();
      CH_TS(3);
      // ---- write back the final entries: the left block (rows [r, r+L) of columns [col, r)),
      //      the diagonal block, and -- on the sweep's last task -- the block below.
      for (int cc = warp; cc < nl; cc += 8) {
        const int64_t c = col + cc;
        const int sl = sl_left(cc);
        double* gp = a.AB + c * a.ldab + (r - c);
        const double* wp = W + sl * LDW + (int)(r - c);
        for (int i = lane; i < L; i += 32) __stcg(&gp[i], wp[i]);
      }
      for (int j = warp; j < L; j += 8) {
        const int64_t c = r + j;
        const int sj = sl_diag(j);
        const int len = (int)((last ? e : r + L) - c);
        double* gp = a.AB + c * a.ldab;
        const double* wp = W + sj * LDW;
        for (int i = lane; i < len; i += 32) __stcg(&gp[i], wp[i]);
      }
      __syncthreads();
      if (tid == 0) {   // barrier, then one GPU-scope fence + flag (the grid-barrier pattern)
        __threadfence();
        volatile int* pr = a.progress + s;
        *pr = (int)(t + 1);
      }
      CH_TS(4);
      if (prof) t_work += clock64() - tk;
    }
  }
  if (prof) { a.dbg[0] = t_wait; a.dbg[1] = t_work; a.dbg[2] = ntasks; for (int i = 0; i < 5; i++) a.dbg[3 + i] = tph[i]; }
#undef CH_TS
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
// matrix) and U = V T^T.  Stored per group as one contiguous block in exactly the shared-
// memory layout of the apply kernel: [U (K2 x LDW) | V (K2 x LDW)], U[c][rho], V[c][rho],
// LDW = RW + 4, so that Q_g X = X - V (U^T X) and one bulk copy moves the whole group.
template <int K2, int RW>
struct BT2Grp {
  static constexpr int LDW = RW + 4;
  static constexpr int ELEMS = 2 * K2 * LDW;
};

template <int K2, int RW>
__global__ void __launch_bounds__(128) bt2_prep_kernel(const double* qv, const double* qtau, int64_t ngroups, int b,
                                                      double* UV) {
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
    double* out = UV + g * Gp::ELEMS;
    for (int e = threadIdx.x; e < K2 * Gp::LDW; e += blockDim.x) {
      int c = e / Gp::LDW, rho = e % Gp::LDW;
      double u = 0.0, vv = 0.0;
      if (rho < RW) {
        for (int c2 = c; c2 < K2; c2++) u += V[c2][rho] * T[c][c2];
        vv = V[c][rho];
      }
      out[e] = u;
      out[K2 * Gp::LDW + e] = vv;
    }
    __syncthreads();
  }
}

// BT2 apply: one CTA per strip of NB columns of X, persistent over all groups in the
// order sweep blocks last -> first, t ascending.  The RW-row window
// X[W0 : W0+RW, strip] (W0 = s0 + t*b) lives in a RING-row shared-memory ring: step t+1
// reuses the last RW-b rows of window t, so per step only b new rows are loaded and b
// rows are written back.  The next group's [U | V] block (51 KB) arrives with ONE bulk
// copy (cp.async.bulk, TMA engine) into the second buffer, tracked by an mbarrier; the b
// new window rows arrive with cp.async (each thread: rows 2*lane.., fixed columns).
// Per step:  Z = U^T Xw (K2 x NB, DMMA, skip U's zero upper triangle)
//            Xw -= V Z  (RW x NB, DMMA, skip the staircase's zero fragments)
template <int NB, int K2, int RW, int RING, int BB>
struct BT2Cfg {
  using Gp = BT2Grp<K2, RW>;
  static constexpr int LDX = RING + 4;   // Xs[col][slot]
  static constexpr int LDW = Gp::LDW;    // U / V rows
  static constexpr int LDZ = K2 + 4;     // Zs[col][c]
  static constexpr int XS = NB * LDX, GS = Gp::ELEMS, ZS = NB * LDZ;
  static constexpr size_t SMEM = (size_t)(XS + 2 * GS + ZS) * sizeof(double) + 2 * sizeof(uint64_t);
  static_assert(LDX % 16 == 4 && LDW % 16 == 4 && LDZ % 16 == 4, "pad");
  static_assert(RING % 64 == 0 && RW % 8 == 0 && RING >= RW + BB && BB == 64 && NB == 64, "ring");
};

template <int NB, int K2, int RW, int RING, int BB>
__global__ void __launch_bounds__(256, 1) bt2_apply_kernel(double* __restrict__ X, int64_t ldx, int64_t ncols,
                                                          int64_t n, const double* __restrict__ UV,
                                                          const int64_t* __restrict__ gofs, int64_t nblk,
                                                          long long* dbg) {
  using C = BT2Cfg<NB, K2, RW, RING, BB>;
  extern __shared__ __align__(128) double sh[];
  double* Xs = sh;
  double* G0 = Xs + C::XS;            // [2][U | V]
  double* Zs = G0 + 2 * C::GS;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Zs + C::ZS);
  long long ph[6] = {0, 0, 0, 0, 0, 0}, tprev = 0, nsteps = 0;
  const bool prof = (dbg != nullptr) && blockIdx.x == 0 && threadIdx.x == 0;
#define BT2_TS(k) do { if (prof) { long long _t = clock64(); ph[k] += _t - tprev; tprev = _t; } } while (0)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int64_t col0 = (int64_t)blockIdx.x * NB;
  const int ncl = (int)smin<int64_t>(NB, ncols - col0);
  const bool vec = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  if (nblk <= 0) return;
  for (int e = tid; e < C::XS; e += 256) Xs[e] = 0.0;   // ring rows beyond n stay finite
  if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_fence_init(); }
  __syncthreads();

  // Xs element (col, slot) lives at col*LDX + (slot ^ 4*bit2(col)): with LDX = 4 (mod 16) the
  // GEMM1 B-fragment reads (8 columns x 4 slots) and the GEMM2 C read-modify-writes (4 column
  // pairs x 8 slots) are both bank-conflict free.
  auto xo = [&](int col, int slot) -> int { return col * C::LDX + (slot ^ (((col >> 2) & 1) << 2)); };
  auto load_group = [&](int64_t g, int buf) {   // thread 0: one bulk copy of the [U | V] block
    fence_proxy_async();
    mbar_expect_tx(&bar[buf], (unsigned)(C::GS * sizeof(double)));
    bulk_g2s(G0 + buf * C::GS, UV + g * C::GS, (unsigned)(C::GS * sizeof(double)), &bar[buf]);
  };
  // this thread's 2-row chunk of column cl: rows r0 + rr, rr = 2*lane (64-row blocks)
  auto load_chunk = [&](int64_t r, int cl, int slot) {
    double* dst = Xs + xo(cl, slot);
    const double* src = X + SK_IDX(r, col0 + cl, ldx);
    const int cnt = (cl < ncl) ? (int)smin<int64_t>(2, smax<int64_t>(0, n - r)) : 0;
    if (vec) {
      cp_async16(dst, cnt ? src : X, cnt * 8);
    } else {
      cp_async8(dst, cnt > 0 ? src : X, cnt > 0 ? 8 : 0);
      cp_async8(dst + 1, cnt > 1 ? src + 1 : X, cnt > 1 ? 8 : 0);
    }
  };
  auto load_rows64 = [&](int64_t r0, int slot0) {   // 64 rows x NB columns
    const int rr = 2 * lane;
    int slot = slot0 + rr;
    if (slot >= RING) slot -= RING;
#pragma unroll
    for (int k = 0; k < NB / 8; k++) load_chunk(r0 + rr, warp + 8 * k, slot);
  };
  auto load_rows32 = [&](int64_t r0, int slot0) {   // 32 rows x NB columns
    const int rr = 2 * (lane & 15);
    int slot = slot0 + rr;
    if (slot >= RING) slot -= RING;
#pragma unroll
    for (int k = 0; k < NB / 16; k++) load_chunk(r0 + rr, 2 * warp + (lane >> 4) + 16 * k, slot);
  };
  auto store_chunk = [&](int64_t r, int cl, int slot) {
    if (cl >= ncl || r >= n) return;
    double* dst = X + SK_IDX(r, col0 + cl, ldx);
    const double2 v = *reinterpret_cast<const double2*>(Xs + xo(cl, slot));
    if (vec && r + 1 < n) {
      *reinterpret_cast<double2*>(dst) = v;
    } else {
      dst[0] = v.x;
      if (r + 1 < n) dst[1] = v.y;
    }
  };
  auto store_rows64 = [&](int64_t r0, int slot0) {
    const int rr = 2 * lane;
    int slot = slot0 + rr;
    if (slot >= RING) slot -= RING;
#pragma unroll
    for (int k = 0; k < NB / 8; k++) store_chunk(r0 + rr, warp + 8 * k, slot);
  };
  auto store_rows32 = [&](int64_t r0, int slot0) {
    const int rr = 2 * (lane & 15);
    int slot = slot0 + rr;
    if (slot >= RING) slot -= RING;
#pragma unroll
    for (int k = 0; k < NB / 16; k++) store_chunk(r0 + rr, 2 * warp + (lane >> 4) + 16 * k, slot);
  };

  unsigned phase[2] = {0u, 0u};
  int buf = 0;
  {
    const int64_t blk = nblk - 1;
    if (tid == 0) load_group(gofs[blk], 0);
    load_rows64(blk * K2, 0);
    load_rows32(blk * K2 + 64, 64);
    cp_async_commit();
  }
  for (int64_t blk = nblk - 1; blk >= 0; blk--) {
    const int64_t s0 = blk * K2;
    const int64_t ntask = 1 + (n - 3 - s0) / BB;
    for (int64_t t = 0; t < ntask; t++) {
      const int64_t W0 = s0 + t * BB;
      const int off = (int)((t * BB) % RING);
      if (prof) { tprev = clock64(); nsteps++; }
      cp_async_wait<0>();
      mbar_wait(&bar[buf], phase[buf]);
      phase[buf] ^= 1u;
      __syncthreads();
      BT2_TS(0);
      // ---- prefetch the next group (and the next rows of the window, same block)
      if (t + 1 < ntask) {
        if (tid == 0) load_group(gofs[blk] + t + 1, buf ^ 1);
        int so = off + RW;
        if (so >= RING) so -= RING;
        load_rows64(W0 + RW, so);
      } else if (blk > 0) {
        if (tid == 0) load_group(gofs[blk - 1], buf ^ 1);
      }
      cp_async_commit();
      BT2_TS(1);
      const double* Us = G0 + buf * C::GS;
      const double* Vs = Us + K2 * C::LDW;
      // ---- Z = U^T Xw : warps 2 (M: c fragments {h, h+2}, interleaved to balance U's zero
      //      upper triangle) x 4 (N: NB/4 columns); even / odd k-step accumulator sets; next
      //      fragments loaded before the current DMMAs.
      {
        constexpr int FN = NB / 32;          // 2 column fragments per warp
        constexpr int NIT = RW / 8;
        const int h = warp & 1, n0 = (warp >> 1) * (NB / 4);
        double acc[2][2][FN][2];
#pragma unroll
        for (int p = 0; p < 2; p++)
#pragma unroll
          for (int i = 0; i < 2; i++)
#pragma unroll
            for (int j = 0; j < FN; j++) acc[p][i][j][0] = acc[p][i][j][1] = 0.0;
        double fa[2][2][2], fb[2][FN][2];
        auto ld1 = [&](int it, int sb) {
          const int kk = it * 8;
          int slot = off + kk;
          if (slot >= RING) slot -= RING;
#pragma unroll
          for (int j = 0; j < FN; j++) {
            fb[sb][j][0] = Xs[xo(n0 + 8 * j + gq, slot + tq)];
            fb[sb][j][1] = Xs[xo(n0 + 8 * j + gq, slot + 4 + tq)];
          }
#pragma unroll
          for (int i = 0; i < 2; i++) {
            const int c = 8 * (h + 2 * i) + gq;
            fa[sb][i][0] = Us[c * C::LDW + kk + tq];
            fa[sb][i][1] = Us[c * C::LDW + kk + 4 + tq];
          }
        };
        ld1(0, 0);
#pragma unroll
        for (int it = 0; it < NIT; it++) {
          const int sb = it & 1;
          if (it + 1 < NIT) ld1(it + 1, sb ^ 1);
#pragma unroll
          for (int i = 0; i < 2; i++) {
            if (it * 8 + 7 < 8 * (h + 2 * i)) continue;   // U[rho][c] = 0 for rho <= c
#pragma unroll
            for (int j = 0; j < FN; j++) {
              dmma884(acc[0][i][j][0], acc[0][i][j][1], fa[sb][i][0], fb[sb][j][0]);
              dmma884(acc[1][i][j][0], acc[1][i][j][1], fa[sb][i][1], fb[sb][j][1]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 2; i++)
#pragma unroll
          for (int j = 0; j < FN; j++) {
            const int c = 8 * (h + 2 * i) + gq, nn = n0 + 8 * j + 2 * tq;
            Zs[nn * C::LDZ + c] = acc[0][i][j][0] + acc[1][i][j][0];
            Zs[(nn + 1) * C::LDZ + c] = acc[0][i][j][1] + acc[1][i][j][1];
          }
      }
      __syncthreads();
      BT2_TS(2);
      // ---- Xw -= V Z : M = RW (rho), N = NB, K = K2 (c); warps 4 (M, interleaved row
      //      fragments: balanced staircase work) x 2 (N); zero staircase fragments skipped.
      {
        constexpr int FM = RW / 32, FN = NB / 16;
        constexpr int NIT = K2 / 4;
        const int wm = warp & 3, n0 = (warp >> 2) * (NB / 2);
        double acc[FM][FN][2];
#pragma unroll
        for (int i = 0; i < FM; i++)
#pragma unroll
          for (int j = 0; j < FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
        double fa[2][FM], fb[2][FN];
        auto ld2 = [&](int it, int sb) {
          const int kk = it * 4;
#pragma unroll
          for (int j = 0; j < FN; j++) fb[sb][j] = Zs[(n0 + 8 * j + gq) * C::LDZ + kk + tq];
#pragma unroll
          for (int i = 0; i < FM; i++) fa[sb][i] = Vs[(kk + tq) * C::LDW + 8 * (wm + 4 * i) + gq];
        };
        ld2(0, 0);
#pragma unroll
        for (int it = 0; it < NIT; it++) {
          const int sb = it & 1, kk = it * 4;
          if (it + 1 < NIT) ld2(it + 1, sb ^ 1);
#pragma unroll
          for (int i = 0; i < FM; i++) {
            const int m0 = 8 * (wm + 4 * i);
            if (m0 + 7 - kk < 1 || m0 - (kk + 3) > BB) continue;   // V[rho][c] != 0 iff 1 <= rho - c <= BB
#pragma unroll
            for (int j = 0; j < FN; j++) dmma884(acc[i][j][0], acc[i][j][1], fa[sb][i], fb[sb][j]);
          }
        }
#pragma unroll
        for (int i = 0; i < FM; i++) {
          const int m0 = 8 * (wm + 4 * i);
          int slot = off + m0;
          if (slot >= RING) slot -= RING;
#pragma unroll
          for (int j = 0; j < FN; j++) {
            int nn = n0 + 8 * j + 2 * tq;
            Xs[xo(nn, slot + gq)] -= acc[i][j][0];
            Xs[xo(nn + 1, slot + gq)] -= acc[i][j][1];
          }
        }
      }
      __syncthreads();
      BT2_TS(3);
      // ---- write back the rows leaving the window
      if (t + 1 < ntask) {
        store_rows64(W0, off);
      } else {
        store_rows64(W0, off);
        store_rows32(W0 + 64, off + 64 >= RING ? off + 64 - RING : off + 64);
        __syncthreads();
        if (blk > 0) {
          load_rows64((blk - 1) * K2, 0);   // first window of the next block
          load_rows32((blk - 1) * K2 + 64, 64);
        }
        cp_async_commit();
      }
      BT2_TS(4);
      buf ^= 1;
    }
  }
  cp_async_wait<0>();
  if (prof) {
    for (int k = 0; k < 5; k++) dbg[k] = ph[k];
    dbg[5] = nsteps;
  }
#undef BT2_TS
}

// Warp-specialised BT2 apply (the default): 8 consumer warps run only the two DMMA tiles per
// step; a 9th producer warp moves the data one step ahead -- it waits until the consumers
// released step q-1 (mbarrier "empty"), writes that step's leaving rows back to X, then
// loads step q+1's [U | V] block (one bulk TMA copy) and its new window rows (cp.async)
// and signals mbarrier "full" (transaction bytes + cp.async completion arrivals).  The
// ring offset advances by b per step inside a sweep block and by RW at a block boundary,
// so the next block's first window never overlaps the window being computed.
template <int NB, int K2, int RW, int RING, int BB>
__global__ void __launch_bounds__(384, 1) bt2_ws_kernel(double* __restrict__ X, int64_t ldx, int64_t ncols, int64_t n,
                                                       const double* __restrict__ UV, const int64_t* __restrict__ gofs,
                                                       int64_t nblk, long long* dbg) {
  using C = BT2Cfg<NB, K2, RW, RING, BB>;
  extern __shared__ __align__(128) double sh[];
  double* Xs = sh;
  double* G0 = Xs + C::XS;            // [2][U | V]
  double* Zs = G0 + 2 * C::GS;
  uint64_t* full = reinterpret_cast<uint64_t*>(Zs + C::ZS);
  uint64_t* empty = full + 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int64_t col0 = (int64_t)blockIdx.x * NB;
  const int ncl = (int)smin<int64_t>(NB, ncols - col0);
  const bool vec = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  if (nblk <= 0) return;
  for (int e = tid; e < C::XS; e += blockDim.x) Xs[e] = 0.0;   // ring rows beyond n stay finite
  if (tid == 0) {
    mbar_init(&full[0], 128); mbar_init(&full[1], 128);
    mbar_init(&empty[0], 8); mbar_init(&empty[1], 8);
    mbar_fence_init();
  }
  __syncthreads();
  auto xo = [&](int col, int slot) -> int { return col * C::LDX + (slot ^ (((col >> 2) & 1) << 2)); };
  auto ntask_of = [&](int64_t blk) -> int64_t { return 1 + (n - 3 - blk * K2) / BB; };

  if (warp >= 8) {
    // ============================ producer (4 warps) ============================
    const int pw = warp - 8;                       // producer warp: columns pw, pw+4, ...
    const int ptid = tid - 256;
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
    auto load_group = [&](int64_t g, int b) {
      if (ptid == 0) {
        mbar_expect_tx_noarrive(&full[b], (unsigned)(C::GS * sizeof(double)));
        fence_proxy_async();
        bulk_g2s(G0 + b * C::GS, UV + g * C::GS, (unsigned)(C::GS * sizeof(double)), &full[b]);
      }
    };
    // step 0
    int64_t blk = nblk - 1, t = 0;
    int off = 0;
    load_group(gofs[blk], 0);
    load_rows(blk * K2, RW, 0);
    cp_async_mbar_arrive(&full[0]);
    int64_t pblk = -1, pt = 0;
    int poff = 0;
    bool pstored = true;    // step q-1 already written back
    for (int64_t q = 0;; q++) {
      int64_t nblk_ = blk, nt = t + 1;
      int noff = off + BB;
      if (nt >= ntask_of(blk)) { nblk_ = blk - 1; nt = 0; noff = off + RW; }
      if (noff >= RING) noff -= RING;
      const bool has_next = nblk_ >= 0;
      if (!pstored) {   // consumers released step q-1: write back its leaving rows
        mbar_wait(&empty[(q - 1) & 1], (unsigned)(((q - 1) >> 1) & 1));
        const bool pfinal = (pt + 1 >= ntask_of(pblk));
        store_rows(pblk * K2 + pt * BB, pfinal ? RW : BB, poff);
      }
      bool stored = false;
      if (has_next && nblk_ != blk && ntask_of(blk) == 1) {
        // the next block's first window overlaps this single-step block's window:
        // wait for step q and write it back before loading
        mbar_wait(&empty[q & 1], (unsigned)((q >> 1) & 1));
        store_rows(blk * K2 + t * BB, RW, off);
        stored = true;
      }
      if (!has_next) {
        if (!stored) {
          mbar_wait(&empty[q & 1], (unsigned)((q >> 1) & 1));
          store_rows(blk * K2 + t * BB, RW, off);
        }
        break;
      }
      {
        const int b = (int)((q + 1) & 1);
        load_group(gofs[nblk_] + nt, b);
        if (nblk_ == blk) {
          int so = noff + (RW - BB);
          if (so >= RING) so -= RING;
          load_rows(nblk_ * K2 + nt * BB + (RW - BB), BB, so);
        } else {
          load_rows(nblk_ * K2, RW, noff);
        }
        cp_async_mbar_arrive(&full[b]);
      }
      pblk = blk; pt = t; poff = off; pstored = stored;
      blk = nblk_; t = nt; off = noff;
    }
    return;
  }
  // =============================== consumers ===============================
  long long ph[6] = {0, 0, 0, 0, 0, 0}, tprev = 0, nsteps = 0;
  const bool prof = (dbg != nullptr) && blockIdx.x == 0 && threadIdx.x == 0;
#define BT2_TS(k) do { if (prof) { long long _t = clock64(); ph[k] += _t - tprev; tprev = _t; } } while (0)
  int64_t blk = nblk - 1, t = 0;
  int off = 0;
  for (int64_t q = 0;; q++) {
    if (prof) { tprev = clock64(); nsteps++; }
    mbar_wait(&full[q & 1], (unsigned)((q >> 1) & 1));
    BT2_TS(0);
    const double* Us = G0 + (q & 1) * C::GS;
    const double* Vs = Us + K2 * C::LDW;
      // ---- Z = U^T Xw : warps 2 (M: c fragments {h, h+2}, interleaved to balance U's zero
      //      upper triangle) x 4 (N: NB/4 columns); even / odd k-step accumulator sets; next
      //      fragments loaded before the current DMMAs.
      {
        constexpr int FN = NB / 32;          // 2 column fragments per warp
        constexpr int NIT = RW / 8;
        const int h = warp & 1, n0 = (warp >> 1) * (NB / 4);
        double acc[2][2][FN][2];
#pragma unroll
        for (int p = 0; p < 2; p++)
#pragma unroll
          for (int i = 0; i < 2; i++)
#pragma unroll
            for (int j = 0; j < FN; j++) acc[p][i][j][0] = acc[p][i][j][1] = 0.0;
        double fa[2][2][2], fb[2][FN][2];
        auto ld1 = [&](int it, int sb) {
          const int kk = it * 8;
          int slot = off + kk;
          if (slot >= RING) slot -= RING;
#pragma unroll
          for (int j = 0; j < FN; j++) {
            fb[sb][j][0] = Xs[xo(n0 + 8 * j + gq, slot + tq)];
            fb[sb][j][1] = Xs[xo(n0 + 8 * j + gq, slot + 4 + tq)];
          }
#pragma unroll
          for (int i = 0; i < 2; i++) {
            const int c = 8 * (h + 2 * i) + gq;
            fa[sb][i][0] = Us[c * C::LDW + kk + tq];
            fa[sb][i][1] = Us[c * C::LDW + kk + 4 + tq];
          }
        };
        ld1(0, 0);
#pragma unroll
        for (int it = 0; it < NIT; it++) {
          const int sb = it & 1;
          if (it + 1 < NIT) ld1(it + 1, sb ^ 1);
#pragma unroll
          for (int i = 0; i < 2; i++) {
            if (it * 8 + 7 < 8 * (h + 2 * i)) continue;   // U[rho][c] = 0 for rho <= c
#pragma unroll
            for (int j = 0; j < FN; j++) {
              dmma884(acc[0][i][j][0], acc[0][i][j][1], fa[sb][i][0], fb[sb][j][0]);
              dmma884(acc[1][i][j][0], acc[1][i][j][1], fa[sb][i][1], fb[sb][j][1]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < 2; i++)
#pragma unroll
          for (int j = 0; j < FN; j++) {
            const int c = 8 * (h + 2 * i) + gq, nn = n0 + 8 * j + 2 * tq;
            Zs[nn * C::LDZ + c] = acc[0][i][j][0] + acc[1][i][j][0];
            Zs[(nn + 1) * C::LDZ + c] = acc[0][i][j][1] + acc[1][i][j][1];
          }
      }
      named_bar(1 + (warp >> 2), 128);   // two independent 4-warp groups (columns 0-31 / 32-63)
      BT2_TS(2);
      // ---- Xw -= V Z : M = RW (rho), N = NB, K = K2 (c); warps 4 (M, interleaved row
      //      fragments: balanced staircase work) x 2 (N); zero staircase fragments skipped.
      {
        constexpr int FM = RW / 32, FN = NB / 16;
        constexpr int NIT = K2 / 4;
        const int wm = warp & 3, n0 = (warp >> 2) * (NB / 2);
        double acc[FM][FN][2];
#pragma unroll
        for (int i = 0; i < FM; i++)
#pragma unroll
          for (int j = 0; j < FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
        double fa[2][FM], fb[2][FN];
        auto ld2 = [&](int it, int sb) {
          const int kk = it * 4;
#pragma unroll
          for (int j = 0; j < FN; j++) fb[sb][j] = Zs[(n0 + 8 * j + gq) * C::LDZ + kk + tq];
#pragma unroll
          for (int i = 0; i < FM; i++) fa[sb][i] = Vs[(kk + tq) * C::LDW + 8 * (wm + 4 * i) + gq];
        };
        ld2(0, 0);
#pragma unroll
        for (int it = 0; it < NIT; it++) {
          const int sb = it & 1, kk = it * 4;
          if (it + 1 < NIT) ld2(it + 1, sb ^ 1);
#pragma unroll
          for (int i = 0; i < FM; i++) {
            const int m0 = 8 * (wm + 4 * i);
            if (m0 + 7 - kk < 1 || m0 - (kk + 3) > BB) continue;   // V[rho][c] != 0 iff 1 <= rho - c <= BB
#pragma unroll
            for (int j = 0; j < FN; j++) dmma884(acc[i][j][0], acc[i][j][1], fa[sb][i], fb[sb][j]);
          }
        }
#pragma unroll
        for (int i = 0; i < FM; i++) {
          const int m0 = 8 * (wm + 4 * i);
          int slot = off + m0;
          if (slot >= RING) slot -= RING;
#pragma unroll
          for (int j = 0; j < FN; j++) {
            int nn = n0 + 8 * j + 2 * tq;
            Xs[xo(nn, slot + gq)] -= acc[i][j][0];
            Xs[xo(nn + 1, slot + gq)] -= acc[i][j][1];
          }
        }
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[q & 1]);
    named_bar(1 + (warp >> 2), 128);   // two independent 4-warp groups (columns 0-31 / 32-63)
    BT2_TS(3);
    // advance
    int64_t nt = t + 1;
    int noff = off + BB;
    if (nt >= ntask_of(blk)) { blk--; nt = 0; noff = off + RW; }
    if (noff >= RING) noff -= RING;
    if (blk < 0) break;
    t = nt; off = noff;
  }
  if (prof) {
    for (int k = 0; k < 5; k++) dbg[k] = ph[k];
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
  if (vectors) w.qT = ar.take<double>((size_t)ng * 2 * L.k2 * (L.b + L.k2 + 4));   // [U | V] per group
  w.gofs = ar.take<int64_t>(std::max<int64_t>(L.nblk, 1));
}

static int chase_grid(int64_t n, int b, int nsm) {
  // concurrently active sweeps ~ (n/b)/3; never more CTAs than can be co-resident
  int64_t act = std::max<int64_t>(1, (n / std::max(b, 1)) / 3 + 1);
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
      a.dbg = nullptr;
      if (getenv("SKEWEIG_CHASE_DBG")) {   // debug instrumentation only
        cudaError_t me = cudaMalloc(&a.dbg, 8 * sizeof(long long));
        if (me) { fprintf(stderr, "[chase dbg] cudaMalloc failed: %s\n", cudaGetErrorString(me)); a.dbg = nullptr; }
      }
      int G = chase_grid(n, L.b, nsm);
      size_t smem = (size_t)(2 * L.b + 1) * (2 * L.b + 2) * sizeof(double);
      e = cudaFuncSetAttribute(chase_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
      void* args[] = {&a};
      e = cudaLaunchCooperativeKernel((void*)chase_kernel<128>, dim3(G), dim3(256), args, smem, st);
      if (e) return e;
      if (a.dbg) {
        long long h[8];
        cudaMemcpyAsync(h, a.dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        fprintf(stderr, "[chase dbg] G=%d tasks(cta0)=%lld  per task: wait %.0f work %.0f (load %.0f house %.0f "
                "w/z %.0f rank2 %.0f store %.0f) cycles\n", G, h[2], (double)h[0] / h[2], (double)h[1] / h[2],
                (double)h[3] / h[2], (double)h[4] / h[2], (double)h[5] / h[2], (double)h[6] / h[2], (double)h[7] / h[2]);
        cudaFree(a.dbg);
      }
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
  long long* dbgp = nullptr;
  if (getenv("SKEWEIG_BT2_DBG")) cudaMalloc(&dbgp, 6 * sizeof(long long));   // debug instrumentation only
  const char* wsenv = getenv("SKEWEIG_BT2_WS");
  const bool ws = !(wsenv && wsenv[0] == '0');
  if (ws) {
    const size_t smem = Cf::SMEM + 2 * sizeof(uint64_t);
    e = cudaFuncSetAttribute(bt2_ws_kernel<NB, K2, RW, RING, BB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    KScope ks(KC_BT2, st);
    bt2_ws_kernel<NB, K2, RW, RING, BB><<<(unsigned)((ncols + NB - 1) / NB), 384, smem, st>>>(
        X, ldx, ncols, L.n, w.qT, w.gofs, L.nblk, dbgp);
  } else {
    KScope ks(KC_BT2, st);
    bt2_apply_kernel<NB, K2, RW, RING, BB><<<(unsigned)((ncols + NB - 1) / NB), 256, Cf::SMEM, st>>>(
        X, ldx, ncols, L.n, w.qT, w.gofs, L.nblk, dbgp);
  }
  if (dbgp) {
    long long h[6];
    cudaMemcpyAsync(h, dbgp, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "[bt2 dbg] steps %lld  per-step cycles: wait %.0f prefetch %.0f gemm1 %.0f gemm2 %.0f store %.0f\n",
            h[5], (double)h[0] / h[5], (double)h[1] / h[5], (double)h[2] / h[5], (double)h[3] / h[5], (double)h[4] / h[5]);
    cudaFree(dbgp);
  }
  return cudaGetLastError();
}

}  // namespace sk
