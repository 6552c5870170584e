// gemm_dmma.cuh -- FP64 tensor-core (DMMA.8x8x4) tiled GEMM core for sm_100a.
//
// C = alpha * op(A) op(B) + beta * C, column-major C.  Operand tiles are staged
// global -> shared with cp.async (LDGSTS, 16-byte, zero-filled tails) in a
// STAGES-deep ring; each warp owns a WM x WN sub-tile held in registers and issues
// m8n8k4 f64 MMAs (the only FP64 tensor instruction sm_100a has: tcgen05 has no
// f64 kind).  Shared-memory rows are padded to LD = 4 (mod 16) doubles so that the
// 8x4 / 4x8 fragment reads of a half-warp hit 16 distinct 8-byte bank pairs.
//
// Layout flags:
//   A_KMAJ=false : A(m,k) = A[m + k*lda]   (column-major M x K, e.g. V, P = [V W])
//   A_KMAJ=true  : A(m,k) = A[k + m*lda]   (A^T of a column-major K x M, e.g. U^T)
//   B_NMAJ=false : B(k,n) = B[k + n*ldb]   (column-major K x N, e.g. X, V)
//   B_NMAJ=true  : B(k,n) = B[n + k*ldb]   (B^T of a column-major N x K, e.g. [W -V]^T)
// TRI: tile set = lower-triangular tiles of a square C (tm >= tn) and only strictly
//      lower elements (row > col) are written -- the skew rank-2k update touches one
//      triangle only.
#pragma once
#include "common.cuh"

namespace sk {

struct GemmArgs {
  int64_t M, N, K;
  const double* A; int64_t lda;
  const double* B; int64_t ldb;
  double* C; int64_t ldc;
  double alpha, beta;
  int64_t tri_off = 1;   // TRI: write element (m, n) iff m - n >= tri_off (1: strictly lower, 0: incl. diagonal)
  int vec = 1;           // 1: 16-byte cp.async (A, B 16B-aligned, lda/ldb even); 0: 8-byte copies
  int col_stride = 1;    // TRI with BM == BN: only column tiles tn = col_off + col_stride*i (1D block-cyclic
  int col_off = 0;       //   column ownership of the distributed full->band reduction)
};

// true when both operands allow 16-byte (2 x double) vector copies
__host__ __device__ inline bool gemm_vec_ok(const void* A, int64_t lda, const void* B, int64_t ldb) {
  return ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 && (lda % 2 == 0) &&
         (ldb % 2 == 0);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJ, bool B_NMAJ>
struct GemmTile {
  static constexpr int NWARP_M = BM / WM, NWARP_N = BN / WN;
  static constexpr int NTHREADS = 32 * NWARP_M * NWARP_N;
  static constexpr int FM = WM / 8, FN = WN / 8;             // 8x8 fragments per warp
  static constexpr int BK_ = BK;
  // shared layouts
  static constexpr int A_LD = A_KMAJ ? (BK + 4) : (BM + 4);
  static constexpr int A_ROWS = A_KMAJ ? BM : BK;
  static constexpr int B_LD = B_NMAJ ? (BN + 4) : (BK + 4);
  static constexpr int B_ROWS = B_NMAJ ? BK : BN;
  static constexpr int A_STAGE = A_ROWS * A_LD;              // doubles
  static constexpr int B_STAGE = B_ROWS * B_LD;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
  static_assert(A_LD % 16 == 4 && B_LD % 16 == 4, "padding for conflict-free fragments");
  static_assert(BK % 4 == 0 && WM % 8 == 0 && WN % 8 == 0, "tile shapes");

  // Issue the cp.async copies of k-block kb into stage s.
  __device__ __forceinline__ static void load_stage(const GemmArgs& g, double* As, double* Bs,
                                                    int64_t m0, int64_t n0, int64_t k0, int tid) {
    // ---- A
    if (!A_KMAJ) {
      // BK columns of BM contiguous doubles
      constexpr int CH = BM / 2, TOT = CH * BK;
      for (int c = tid; c < TOT; c += NTHREADS) {
        int kk = c / CH, mm = (c % CH) * 2;
        int64_t gm = m0 + mm, gk = k0 + kk;
        int cnt = (gk < g.K) ? (int)smin<int64_t>(2, smax<int64_t>(0, g.M - gm)) : 0;
        const double* src = cnt ? g.A + SK_IDX(gm, gk, g.lda) : g.A;
        if (g.vec) cp_async16(As + kk * A_LD + mm, src, cnt * 8);
        else { cp_async8(As + kk * A_LD + mm, src, cnt > 0 ? 8 : 0); cp_async8(As + kk * A_LD + mm + 1, cnt > 1 ? src + 1 : src, cnt > 1 ? 8 : 0); }
      }
    } else {
      constexpr int CH = BK / 2, TOT = CH * BM;
      for (int c = tid; c < TOT; c += NTHREADS) {
        int mm = c / CH, kk = (c % CH) * 2;
        int64_t gm = m0 + mm, gk = k0 + kk;
        int cnt = (gm < g.M) ? (int)smin<int64_t>(2, smax<int64_t>(0, g.K - gk)) : 0;
        const double* src = cnt ? g.A + SK_IDX(gk, gm, g.lda) : g.A;
        if (g.vec) cp_async16(As + mm * A_LD + kk, src, cnt * 8);
        else { cp_async8(As + mm * A_LD + kk, src, cnt > 0 ? 8 : 0); cp_async8(As + mm * A_LD + kk + 1, cnt > 1 ? src + 1 : src, cnt > 1 ? 8 : 0); }
      }
    }
    // ---- B
    if (!B_NMAJ) {
      constexpr int CH = BK / 2, TOT = CH * BN;
      for (int c = tid; c < TOT; c += NTHREADS) {
        int nn = c / CH, kk = (c % CH) * 2;
        int64_t gn = n0 + nn, gk = k0 + kk;
        int cnt = (gn < g.N) ? (int)smin<int64_t>(2, smax<int64_t>(0, g.K - gk)) : 0;
        const double* src = cnt ? g.B + SK_IDX(gk, gn, g.ldb) : g.B;
        if (g.vec) cp_async16(Bs + nn * B_LD + kk, src, cnt * 8);
        else { cp_async8(Bs + nn * B_LD + kk, src, cnt > 0 ? 8 : 0); cp_async8(Bs + nn * B_LD + kk + 1, cnt > 1 ? src + 1 : src, cnt > 1 ? 8 : 0); }
      }
    } else {
      constexpr int CH = BN / 2, TOT = CH * BK;
      for (int c = tid; c < TOT; c += NTHREADS) {
        int kk = c / CH, nn = (c % CH) * 2;
        int64_t gn = n0 + nn, gk = k0 + kk;
        int cnt = (gk < g.K) ? (int)smin<int64_t>(2, smax<int64_t>(0, g.N - gn)) : 0;
        const double* src = cnt ? g.B + SK_IDX(gn, gk, g.ldb) : g.B;
        if (g.vec) cp_async16(Bs + kk * B_LD + nn, src, cnt * 8);
        else { cp_async8(Bs + kk * B_LD + nn, src, cnt > 0 ? 8 : 0); cp_async8(Bs + kk * B_LD + nn + 1, cnt > 1 ? src + 1 : src, cnt > 1 ? 8 : 0); }
      }
    }
  }

  __device__ __forceinline__ static double a_at(const double* As, int m, int k) {
    return A_KMAJ ? As[m * A_LD + k] : As[k * A_LD + m];
  }
  __device__ __forceinline__ static double b_at(const double* Bs, int k, int n) {
    return B_NMAJ ? Bs[k * B_LD + n] : Bs[n * B_LD + k];
  }

  // acc[FM][FN][2] += A_tile(warp rows) * B_tile(warp cols) over one BK block.  The
  // fragments of k-step kk+4 are loaded into a second register set while the MMAs of
  // k-step kk issue, so the shared-memory latency overlaps the DMMA pipe.
  __device__ __forceinline__ static void mma_stage(const double* As, const double* Bs, double (&acc)[FM][FN][2],
                                                   int wm0, int wn0, int lane) {
    const int gq = lane >> 2, t = lane & 3;
    double af[2][FM], bf[2][FN];
#pragma unroll
    for (int i = 0; i < FM; i++) af[0][i] = a_at(As, wm0 + 8 * i + gq, t);
#pragma unroll
    for (int j = 0; j < FN; j++) bf[0][j] = b_at(Bs, t, wn0 + 8 * j + gq);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int cur = (kk / 4) & 1;
      if (kk + 4 < BK) {
#pragma unroll
        for (int i = 0; i < FM; i++) af[cur ^ 1][i] = a_at(As, wm0 + 8 * i + gq, kk + 4 + t);
#pragma unroll
        for (int j = 0; j < FN; j++) bf[cur ^ 1][j] = b_at(Bs, kk + 4 + t, wn0 + 8 * j + gq);
      }
#pragma unroll
      for (int i = 0; i < FM; i++)
#pragma unroll
        for (int j = 0; j < FN; j++) dmma884(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
  }

  // Full K loop for the tile (m0, n0); result in acc.
  __device__ __forceinline__ static void mainloop(const GemmArgs& g, double* smem, int64_t m0, int64_t n0,
                                                  int64_t kbeg, int64_t kend, double (&acc)[FM][FN][2]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm0 = (warp % NWARP_M) * WM, wn0 = (warp / NWARP_M) * WN;
    double* As = smem;
    double* Bs = smem + STAGES * A_STAGE;
    const int64_t nk = (kend - kbeg + BK - 1) / BK;
#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
      if (s < nk) load_stage(g, As + s * A_STAGE, Bs + s * B_STAGE, m0, n0, kbeg + s * BK, tid);
      cp_async_commit();
    }
    for (int64_t kb = 0; kb < nk; kb++) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      int64_t pf = kb + STAGES - 1;
      if (pf < nk) {
        int ps = (int)(pf % STAGES);
        load_stage(g, As + ps * A_STAGE, Bs + ps * B_STAGE, m0, n0, kbeg + pf * BK, tid);
      }
      cp_async_commit();
      int cs = (int)(kb % STAGES);
      mma_stage(As + cs * A_STAGE, Bs + cs * B_STAGE, acc, wm0, wn0, lane);
    }
    cp_async_wait<0>();
    __syncthreads();
  }
};

// Lower-triangular tile enumeration for BM = R * BN (R >= 1): row tile tm meets the
// (strictly) lower triangle in column tiles tn = 0 .. R*(tm+1)-1; cumulative count
// C(tm) = R * tm * (tm+1) / 2; t -> (tm, tn) with C(tm) <= t < C(tm+1).
__host__ __device__ __forceinline__ void tri_tile(int64_t t, int R, int64_t& tm, int64_t& tn) {
  int64_t r = (int64_t)((sqrt(8.0 * (double)t / R + 1.0) - 1.0) * 0.5);
  while ((int64_t)R * (r + 1) * (r + 2) / 2 <= t) r++;
  while ((int64_t)R * r * (r + 1) / 2 > t) r--;
  tm = r;
  tn = t - (int64_t)R * r * (r + 1) / 2;
}

// Strided variant (BM == BN): column tiles tn_i = off + stride*i, rows tm in [tn_i, ntm);
// S(k) = sum_{i<k} (ntm - tn_i) = k (ntm - off) - stride k (k-1) / 2.
__host__ __device__ __forceinline__ void tri_tile_strided(int64_t t, int64_t ntm, int stride, int off, int64_t& tm,
                                                          int64_t& tn) {
  auto S = [&](int64_t k) -> int64_t { return k * (ntm - off) - (int64_t)stride * k * (k - 1) / 2; };
  const double A = 0.5 * stride, B = (double)(ntm - off) + 0.5 * stride;
  int64_t k = (int64_t)((B - sqrt(fmax(B * B - 4.0 * A * (double)t, 0.0))) / (2.0 * A));
  if (k < 0) k = 0;
  while (S(k + 1) <= t) k++;
  while (k > 0 && S(k) > t) k--;
  tn = off + (int64_t)stride * k;
  tm = tn + (t - S(k));
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJ, bool B_NMAJ, bool TRI>
__global__ void __launch_bounds__(GemmTile<BM, BN, BK, WM, WN, STAGES, A_KMAJ, B_NMAJ>::NTHREADS)
gemm_dmma_kernel(GemmArgs g) {
  using T = GemmTile<BM, BN, BK, WM, WN, STAGES, A_KMAJ, B_NMAJ>;
  extern __shared__ __align__(16) double smem[];
  int64_t tm, tn;
  if (TRI) {
    if (g.col_stride > 1) tri_tile_strided(blockIdx.x, (g.M + BM - 1) / BM, g.col_stride, g.col_off, tm, tn);
    else tri_tile(blockIdx.x, BM / BN, tm, tn);
  } else {
    tm = blockIdx.x;
    tn = blockIdx.y;
  }
  const int64_t m0 = tm * BM, n0 = tn * BN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm0 = (warp % T::NWARP_M) * WM, wn0 = (warp / T::NWARP_M) * WN;
  const int gq = lane >> 2, t = lane & 3;
  // C = alpha*AB + beta*C computed as alpha*(AB + (beta/alpha) C): the C tile is loaded into
  // the accumulators before the main loop so its latency overlaps the operand pipeline
  // (exact for the alpha = +-1, beta in {0, 1} used by the library).
  double acc[T::FM][T::FN][2];
  const double cscale = (g.beta != 0.0) ? g.beta / g.alpha : 0.0;
  // 32-bit tile-local indexing (keeps the register count down)
  const int mrem = (int)smin<int64_t>(g.M - m0, BM), nrem = (int)smin<int64_t>(g.N - n0, BN);
  const int dmn = (int)(m0 - n0);
  const int ldc = (int)g.ldc;
  double* Cb = g.C + SK_IDX(m0, n0, g.ldc);
#pragma unroll
  for (int i = 0; i < T::FM; i++)
#pragma unroll
    for (int j = 0; j < T::FN; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int mi = wm0 + 8 * i + gq, nj = wn0 + 8 * j + 2 * t + h;
        double v = 0.0;
        if (cscale != 0.0 && mi < mrem && nj < nrem && (!TRI || dmn + mi - nj >= (int)g.tri_off))
          v = cscale * Cb[mi + (size_t)nj * ldc];
        acc[i][j][h] = v;
      }
  T::mainloop(g, smem, m0, n0, 0, g.K, acc);
#pragma unroll
  for (int i = 0; i < T::FM; i++)
#pragma unroll
    for (int j = 0; j < T::FN; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int mi = wm0 + 8 * i + gq, nj = wn0 + 8 * j + 2 * t + h;
        if (mi < mrem && nj < nrem && (!TRI || dmn + mi - nj >= (int)g.tri_off))
          Cb[mi + (size_t)nj * ldc] = g.alpha * acc[i][j][h];
      }
}

// Host launcher
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool A_KMAJ, bool B_NMAJ, bool TRI>
cudaError_t gemm_dmma(const GemmArgs& g, cudaStream_t st) {
  using T = GemmTile<BM, BN, BK, WM, WN, STAGES, A_KMAJ, B_NMAJ>;
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  GemmArgs ga = g;
  ga.vec = gemm_vec_ok(g.A, g.lda, g.B, g.ldb) ? 1 : 0;
  auto kern = gemm_dmma_kernel<BM, BN, BK, WM, WN, STAGES, A_KMAJ, B_NMAJ, TRI>;
  {
    cudaError_t e = set_smem_attr((const void*)kern, (int)T::SMEM_BYTES);
    if (e != cudaSuccess) return e;
  }
  int64_t tm = (g.M + BM - 1) / BM, tn = (g.N + BN - 1) / BN;
  dim3 grid;
  static_assert(!TRI || BM % BN == 0, "TRI needs BM = R * BN");
  if (TRI && g.col_stride > 1) {
    if (BM != BN) return cudaErrorInvalidValue;
    const int64_t off = g.col_off, st = g.col_stride;
    if (off >= tm) return cudaSuccess;
    const int64_t kmax = (tm - off + st - 1) / st;
    grid = dim3((unsigned)(kmax * (tm - off) - st * kmax * (kmax - 1) / 2));
  } else if (TRI) grid = dim3((unsigned)((BM / BN) * tm * (tm + 1) / 2));
  else grid = dim3((unsigned)tm, (unsigned)tn);
  kern<<<grid, T::NTHREADS, T::SMEM_BYTES, st>>>(ga);
  return cudaGetLastError();
}

}  // namespace sk
