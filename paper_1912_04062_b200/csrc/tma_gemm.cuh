// tma_gemm.cuh -- persistent, warp-specialised FP64 GEMM for sm_100a with TMA-fed operand
// tiles (cp.async.bulk.tensor, SASS UTMALDG) and DMMA.8x8x4 consumers.
//
//   C = alpha * op(A) op(B) + beta * C        (column-major C, optional TRI tile set)
//
// One CTA per SM walks a static list of BM x BN output tiles (t = blockIdx.x + i*gridDim.x).
// Warp NCW (the producer) streams the K blocks of every tile it owns through an NS-stage
// shared-memory ring with one TMA box per operand per stage (full / empty mbarriers with
// transaction counts), running ahead across tile boundaries, and loads each tile's C box
// (beta != 0) into its own buffer.  Warps 0..NCW-1 (consumers, 2 x 4 of 32 x 32 warp tiles for
// 128 x 64) run GemmTile::mma_stage on each stage, then add beta*C from shared memory and
// store the tile (masked for TRI).
//
// The TMA boxes are one row / column wider than the tile on the contiguous side (BM+4, BN+4
// or BK+4 elements) so that the box lands in shared memory with exactly GemmTile's padded
// row pitch (4 mod 16 doubles: conflict-free m8n8k4 fragment reads); the extra elements are
// loaded but never read.  Out-of-range box elements are zero-filled by the TMA unit.
//
// The operand layouts are GemmTile's (A_KMAJ / B_NMAJ, see gemm_dmma.cuh).  TMA needs
// 16-byte aligned bases and leading dimensions that are multiples of 2 doubles; callers
// fall back to gemm_dmma otherwise (tma_gemm_ok).
#pragma once
#include <cuda.h>
#include <cstdlib>
#include <mutex>
#include "common.cuh"
#include "gemm_dmma.cuh"

namespace sk {

struct TmaGemmArgs {
  int64_t M, N, K;
  double* C; int64_t ldc;
  double alpha, beta;
  int64_t tri_off = 1;   // TRI: write (m, n) iff m - n >= tri_off
  int64_t ntiles = 0;    // tile count (TRI: lower-triangular tile set)
  int64_t tn_count = 0;  // non-TRI: number of column tiles
  // TRI, distributed (col_stride > 1): only the column tiles tn = col_off + col_stride * i
  // (BN wide, the rank's 1D block-cyclic columns); ntm = row tiles (BM high)
  int col_stride = 1, col_off = 0;
  int64_t ntm = 0, kloc = 0;   // kloc = number of local column tiles
};

// sum_{i<k} floor((off + s i) / R), R in {1, 2}
__host__ __device__ inline int64_t tri_floor_sum(int64_t k, int64_t off, int64_t s, int R) {
  const int64_t lin = k * off + s * k * (k - 1) / 2;
  if (R == 1) return lin;
  int64_t odd;
  if ((s & 1) == 0) odd = k * (off & 1);
  else odd = (off & 1) ? (k + 1) / 2 : k / 2;
  return (lin - odd) / 2;
}
// number of (row tile, column tile) pairs of the strided lower-triangular tile set among the
// first k local column tiles: S(k) = sum_{i<k} (ntm - floor(tn_i / R))
__host__ __device__ inline int64_t tri_strided_count(int64_t k, int64_t ntm, int64_t off, int64_t s, int R) {
  return k * ntm - tri_floor_sum(k, off, s, R);
}

// 2-D tiled TMA load of box (c0 = contiguous coordinate, c1 = strided coordinate)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

template <int BM, int BN, int BK, int NS, bool A_KMAJ, bool B_NMAJ, bool HAS_C>
struct TmaGemmCfg {
  using T = GemmTile<BM, BN, BK, 32, 32, 2, A_KMAJ, B_NMAJ>;
  static constexpr int NCW = T::NTHREADS / 32;          // consumer warps
  static constexpr int THREADS = T::NTHREADS + 32;      // + one producer warp
  static constexpr int A_ST = T::A_STAGE, B_ST = T::B_STAGE;   // doubles per stage
  static constexpr int C_LD = BM + 4;
  static constexpr int C_SZ = HAS_C ? BN * C_LD : 0;
  static constexpr size_t SMEM = (size_t)(NS * (A_ST + B_ST) + C_SZ) * sizeof(double) + (2 * NS + 2) * 8 + 128;
  static constexpr unsigned A_BYTES = (unsigned)(A_ST * sizeof(double));
  static constexpr unsigned B_BYTES = (unsigned)(B_ST * sizeof(double));
  static constexpr unsigned C_BYTES = (unsigned)(C_SZ * sizeof(double));
  static_assert((A_ST * 8) % 128 == 0 && (B_ST * 8) % 128 == 0 && (C_SZ * 8) % 128 == 0, "TMA 128-byte alignment");
};

template <int BM, int BN>
__host__ __device__ __forceinline__ void tma_tile_coords(const TmaGemmArgs& g, int64_t t, bool tri, int64_t& tm, int64_t& tn) {
  if (tri && g.col_stride > 1) {
    constexpr int R = BM / BN;
    int64_t lo = 0, hi = g.kloc;   // S(lo) <= t < S(hi); S is increasing on [0, kloc]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (tri_strided_count(mid, g.ntm, g.col_off, g.col_stride, R) <= t) lo = mid;
      else hi = mid;
    }
    tn = g.col_off + (int64_t)g.col_stride * lo;
    tm = tn / R + (t - tri_strided_count(lo, g.ntm, g.col_off, g.col_stride, R));
  } else if (tri) {
    tri_tile(t, BM / BN, tm, tn);
  } else {
    tm = t / g.tn_count;
    tn = t % g.tn_count;
  }
}

template <int BM, int BN, int BK, int NS, bool A_KMAJ, bool B_NMAJ, bool HAS_C, bool TRI>
__global__ void __launch_bounds__(TmaGemmCfg<BM, BN, BK, NS, A_KMAJ, B_NMAJ, HAS_C>::THREADS, 1)
    tma_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapC, TmaGemmArgs g) {
  using Cfg = TmaGemmCfg<BM, BN, BK, NS, A_KMAJ, B_NMAJ, HAS_C>;
  using T = typename Cfg::T;
  // the dynamic shared memory of a kernel without static shared memory starts at the window's
  // base (1 KB aligned): no run-time realignment, so the fragment loads stay LDS (a pointer
  // rebuilt through an integer would turn them into generic loads)
  extern __shared__ __align__(1024) double sm[];
  double* As = sm;
  double* Bs = As + NS * Cfg::A_ST;
  double* Cs = Bs + NS * Cfg::B_ST;
  uint64_t* full = reinterpret_cast<uint64_t*>(Cs + Cfg::C_SZ);
  uint64_t* empty = full + NS;
  uint64_t* cfull = empty + NS;
  uint64_t* cempty = cfull + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NS; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], Cfg::NCW); }
    mbar_init(cfull, 1);
    mbar_init(cempty, Cfg::NCW);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t nk = (g.K + BK - 1) / BK;
  if (warp == Cfg::NCW) {
    // ================================ producer ================================
    if (lane == 0) {
      tma_prefetch_desc(&mapA);
      tma_prefetch_desc(&mapB);
      if (HAS_C) tma_prefetch_desc(&mapC);
      int64_t it = 0, tile_i = 0;
      for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, tile_i++) {
        int64_t tm, tn;
        tma_tile_coords<BM, BN>(g, t, TRI, tm, tn);
        const int m0 = (int)(tm * BM), n0 = (int)(tn * BN);
        for (int64_t kb = 0; kb < nk; kb++, it++) {
          const int s = (int)(it % NS);
          mbar_wait(&empty[s], (unsigned)(((it / NS) & 1) ^ 1));
          mbar_expect_tx(&full[s], Cfg::A_BYTES + Cfg::B_BYTES);
          const int k0 = (int)(kb * BK);
          if (A_KMAJ) tma_load_2d(As + s * Cfg::A_ST, &mapA, k0, m0, &full[s]);
          else tma_load_2d(As + s * Cfg::A_ST, &mapA, m0, k0, &full[s]);
          if (B_NMAJ) tma_load_2d(Bs + s * Cfg::B_ST, &mapB, n0, k0, &full[s]);
          else tma_load_2d(Bs + s * Cfg::B_ST, &mapB, k0, n0, &full[s]);
          if (HAS_C && kb == 0) {   // this tile's C box once the previous tile's epilogue read it
            mbar_wait(cempty, (unsigned)((tile_i & 1) ^ 1));
            mbar_expect_tx(cfull, Cfg::C_BYTES);
            tma_load_2d(Cs, &mapC, m0, n0, cfull);
          }
        }
      }
    }
    return;
  }
  // ================================ consumers ================================
  const int wm0 = (warp % T::NWARP_M) * 32, wn0 = (warp / T::NWARP_M) * 32;
  const int gq = lane >> 2, tq = lane & 3;
  int64_t it = 0, tile_i = 0;
  for (int64_t t = blockIdx.x; t < g.ntiles; t += gridDim.x, tile_i++) {
    int64_t tm, tn;
    tma_tile_coords<BM, BN>(g, t, TRI, tm, tn);
    const int64_t m0 = tm * BM, n0 = tn * BN;
    double acc[T::FM][T::FN][2];
#pragma unroll
    for (int i = 0; i < T::FM; i++)
#pragma unroll
      for (int j = 0; j < T::FN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int64_t kb = 0; kb < nk; kb++, it++) {
      const int s = (int)(it % NS);
      mbar_wait(&full[s], (unsigned)((it / NS) & 1));
      T::mma_stage(As + s * Cfg::A_ST, Bs + s * Cfg::B_ST, acc, wm0, wn0, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // epilogue: alpha * acc + beta * C  (C from shared memory), masked store
    const int mrem = (int)smin<int64_t>(g.M - m0, BM), nrem = (int)smin<int64_t>(g.N - n0, BN);
    const int dmn = (int)(m0 - n0);
    double* Cb = g.C + SK_IDX(m0, n0, g.ldc);
    const size_t ldc = (size_t)g.ldc;
    if (HAS_C) mbar_wait(cfull, (unsigned)(tile_i & 1));
    double v[T::FM][T::FN][2];
#pragma unroll
    for (int i = 0; i < T::FM; i++)
#pragma unroll
      for (int j = 0; j < T::FN; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int mi = wm0 + 8 * i + gq, nj = wn0 + 8 * j + 2 * tq + h;
          double r = g.alpha * acc[i][j][h];
          if (HAS_C) r = fma(g.beta, Cs[nj * Cfg::C_LD + mi], r);
          v[i][j][h] = r;
        }
    if (HAS_C) {
      __syncwarp();
      if (lane == 0) mbar_arrive(cempty);
    }
#pragma unroll
    for (int i = 0; i < T::FM; i++)
#pragma unroll
      for (int j = 0; j < T::FN; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int mi = wm0 + 8 * i + gq, nj = wn0 + 8 * j + 2 * tq + h;
          if (mi < mrem && nj < nrem && (!TRI || dmn + mi - nj >= (int)g.tri_off)) Cb[mi + nj * ldc] = v[i][j][h];
        }
  }
}

// ---- host side ------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline PFN_encodeTiled tma_encode_fn() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// column-major FP64 matrix (rows x cols, leading dimension ld) with box (box0 rows, box1 cols)
inline bool tma_map_2d(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, int box0,
                       int box1) {
  PFN_encodeTiled enc = tma_encode_fn();
  if (!enc || rows < 1 || cols < 1) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)box1};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// SKEWEIG_NO_TMA=1: use the cp.async gemm_dmma path instead (A/B comparisons)
inline bool tma_disabled() {
  static const bool off = [] { const char* v = getenv("SKEWEIG_NO_TMA"); return v && v[0] == '1'; }();
  return off;
}

inline bool tma_ptr_ok(const void* p, int64_t ld) {
  return p && ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (ld % 2 == 0) && ld < ((int64_t)1 << 37);
}
inline bool tma_gemm_ok(const GemmArgs& g) {
  return tma_encode_fn() != nullptr && tma_ptr_ok(g.A, g.lda) && tma_ptr_ok(g.B, g.ldb) &&
         (g.beta == 0.0 || tma_ptr_ok(g.C, g.ldc)) && g.M < ((int64_t)1 << 31) && g.N < ((int64_t)1 << 31) &&
         g.K < ((int64_t)1 << 31);
}

// Launch on the GemmArgs of gemm_dmma (TRI: lower-triangular tile set of a square C, one
// device, col_stride == 1).  Returns cudaErrorNotSupported when TMA cannot be used.
template <int BM, int BN, int BK, int NS, bool A_KMAJ, bool B_NMAJ, bool HAS_C, bool TRI>
cudaError_t tma_gemm(const GemmArgs& ga, int nsm, cudaStream_t st) {
  using Cfg = TmaGemmCfg<BM, BN, BK, NS, A_KMAJ, B_NMAJ, HAS_C>;
  if (ga.M <= 0 || ga.N <= 0) return cudaSuccess;
  if (!tma_gemm_ok(ga) || (!TRI && ga.col_stride != 1) || (HAS_C != (ga.beta != 0.0))) return cudaErrorNotSupported;
  CUtensorMap mA, mB, mC;
  // A: non-KMAJ = column-major M x K (box BM+4 rows x BK); KMAJ = column-major K x M (box BK+4 x BM)
  bool ok = A_KMAJ ? tma_map_2d(&mA, ga.A, ga.K, ga.M, ga.lda, BK + 4, BM)
                   : tma_map_2d(&mA, ga.A, ga.M, ga.K, ga.lda, BM + 4, BK);
  // B: non-NMAJ = column-major K x N (box BK+4 x BN); NMAJ = column-major N x K (box BN+4 x BK)
  ok = ok && (B_NMAJ ? tma_map_2d(&mB, ga.B, ga.N, ga.K, ga.ldb, BN + 4, BK)
                     : tma_map_2d(&mB, ga.B, ga.K, ga.N, ga.ldb, BK + 4, BN));
  if (HAS_C) ok = ok && tma_map_2d(&mC, ga.C, ga.M, ga.N, ga.ldc, BM + 4, BN);
  else mC = mB;
  if (!ok) return cudaErrorNotSupported;
  TmaGemmArgs g;
  g.M = ga.M; g.N = ga.N; g.K = ga.K;
  g.C = ga.C; g.ldc = ga.ldc; g.alpha = ga.alpha; g.beta = ga.beta; g.tri_off = ga.tri_off;
  const int64_t tm = (ga.M + BM - 1) / BM, tn = (ga.N + BN - 1) / BN;
  g.tn_count = tn;
  g.ntiles = TRI ? (int64_t)(BM / BN) * tm * (tm + 1) / 2 : tm * tn;
  if (TRI && ga.col_stride > 1) {   // the rank's column tiles only (BN-wide, 1D block-cyclic)
    g.col_stride = ga.col_stride;
    g.col_off = ga.col_off;
    g.ntm = tm;
    if (ga.col_off >= tn) return cudaSuccess;
    const int64_t kloc = (tn - ga.col_off + ga.col_stride - 1) / ga.col_stride;
    g.kloc = kloc;
    g.ntiles = tri_strided_count(kloc, tm, ga.col_off, ga.col_stride, BM / BN);
  }
  if (g.ntiles <= 0) return cudaSuccess;
  auto kern = tma_gemm_kernel<BM, BN, BK, NS, A_KMAJ, B_NMAJ, HAS_C, TRI>;
  cudaError_t e = set_smem_attr((const void*)kern, (int)Cfg::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (int)smin<int64_t>(g.ntiles, nsm);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(mA, mB, mC, g);
  return cudaGetLastError();
}

}  // namespace sk
