// Tuning harness for the DMMA GEMM core (paper_1912_04062_b200/csrc/gemm_dmma.cuh) on the
// shapes of the solver at n = 32768: R2K (lower-triangular C, K = 128), BT1 Z = U^T X
// (M = 256, K = n), BT1 update X -= V Z (K = 256).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1912_04062_b200/csrc \
//        -o tools/gemm_bench tools/gemm_bench.cu
#include "gemm_dmma.cuh"
#include <cstdio>
#include <vector>
using namespace sk;

template <int BM, int BN, int BK, int WM, int WN, int ST, bool AK, bool BN_, bool TRI>
void run(const char* name, GemmArgs g, double flops) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaError_t err = gemm_dmma<BM, BN, BK, WM, WN, ST, AK, BN_, TRI>(g, 0);
  if (err) { printf("%s: launch error %s\n", name, cudaGetErrorString(err)); return; }
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(e0);
    gemm_dmma<BM, BN, BK, WM, WN, ST, AK, BN_, TRI>(g, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("%-34s BM%3d BN%3d BK%2d W%2dx%2d S%d : %8.3f ms  %6.2f TF/s\n", name, BM, BN, BK, WM, WN, ST, best,
         flops / best / 1e9);
}

int main() {
  const int64_t n = 32768, b = 64, K2 = 256;
  double *A, *P, *Q, *U, *Z;
  cudaMalloc(&A, n * n * 8); cudaMalloc(&P, n * 2 * b * 8); cudaMalloc(&Q, n * 2 * b * 8);
  cudaMalloc(&U, n * K2 * 8); cudaMalloc(&Z, K2 * n * 8);
  cudaMemset(A, 0, n * n * 8); cudaMemset(P, 0, n * 2 * b * 8); cudaMemset(Q, 0, n * 2 * b * 8);
  cudaMemset(U, 0, n * K2 * 8); cudaMemset(Z, 0, K2 * n * 8);
  {  // R2K: C_lower(n x n) += P Q^T, K = 128
    GemmArgs g{}; g.M = n; g.N = n; g.K = 2 * b; g.A = P; g.lda = n; g.B = Q; g.ldb = n; g.C = A; g.ldc = n;
    g.alpha = 1; g.beta = 1;
    double fl = 2.0 * b * n * (double)(n - 1);
    run<64,64,16,32,32,3,false,true,true>("r2k", g, fl);
    run<64,64,16,32,32,2,false,true,true>("r2k", g, fl);
    run<64,64,32,32,32,2,false,true,true>("r2k", g, fl);
    run<64,32,16,32,16,4,false,true,true>("r2k", g, fl);
    run<64,64,16,16,32,4,false,true,true>("r2k", g, fl);
    run<128,64,16,32,32,3,false,true,true>("r2k", g, fl);
    run<128,64,16,64,32,3,false,true,true>("r2k", g, fl);
    run<128,128,16,64,32,3,false,true,true>("r2k", g, fl);
    run<128,128,16,32,64,3,false,true,true>("r2k", g, fl);
  }
  {  // Z = U^T X : M = 256, N = n, K = n
    GemmArgs g{}; g.M = K2; g.N = n; g.K = n; g.A = U; g.lda = n; g.B = A; g.ldb = n; g.C = Z; g.ldc = K2;
    g.alpha = 1; g.beta = 0;
    double fl = 2.0 * K2 * n * (double)n;
    run<64,64,16,32,32,3,true,false,false>("bt1 z", g, fl);
    run<64,64,16,32,32,2,true,false,false>("bt1 z", g, fl);
    run<64,64,32,32,32,2,true,false,false>("bt1 z", g, fl);
    run<64,32,16,32,16,4,true,false,false>("bt1 z", g, fl);
    run<64,64,16,16,32,4,true,false,false>("bt1 z", g, fl);
    run<128,64,16,32,32,3,true,false,false>("bt1 z", g, fl);
    run<128,64,16,64,32,3,true,false,false>("bt1 z", g, fl);
    run<128,128,16,64,32,3,true,false,false>("bt1 z", g, fl);
    run<128,128,16,32,64,3,true,false,false>("bt1 z", g, fl);
  }
  {  // X -= V Z : M = n, N = n, K = 256
    GemmArgs g{}; g.M = n; g.N = n; g.K = K2; g.A = U; g.lda = n; g.B = Z; g.ldb = K2; g.C = A; g.ldc = n;
    g.alpha = -1; g.beta = 1;
    double fl = 2.0 * K2 * n * (double)n;
    run<64,64,16,32,32,3,false,false,false>("bt1 update", g, fl);
    run<64,64,16,32,32,2,false,false,false>("bt1 update", g, fl);
    run<64,64,32,32,32,2,false,false,false>("bt1 update", g, fl);
    run<64,32,16,32,16,4,false,false,false>("bt1 update", g, fl);
    run<64,64,16,16,32,4,false,false,false>("bt1 update", g, fl);
    run<128,64,16,32,32,3,false,false,false>("bt1 update", g, fl);
    run<128,64,16,64,32,3,false,false,false>("bt1 update", g, fl);
    run<128,128,16,64,32,3,false,false,false>("bt1 update", g, fl);
    run<128,128,16,32,64,3,false,false,false>("bt1 update", g, fl);
  }
  return 0;
}
