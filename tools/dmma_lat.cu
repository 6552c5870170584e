// DMMA.8x8x4 latency / throughput model on B200 (sm_100a): throughput of independent
// accumulator chains per warp for 1, 2 and 4 warps per SM sub-partition, one CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_lat tools/dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_chain(double* out, int iters, long long* cyc) {
  double c[CHAINS][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) c[i][0] = c[i][1] = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CHAINS>
void run(int warps_per_cta, double* out, long long* cyc) {
  const int iters = 4096;
  dmma_chain<CHAINS><<<148, 32 * warps_per_cta>>>(out, 64, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_chain<CHAINS><<<148, 32 * warps_per_cta>>>(out, iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double per = (double)c / iters / CHAINS;   // cycles per DMMA per warp
  double tf = 512.0 * CHAINS * iters * warps_per_cta * 148 / (ms * 1e9);
  printf("warps/SMSP=%d chains=%2d: %6.2f cycles per DMMA per warp, %.2f TF/s (SMSP issue: %.2f cycles/DMMA)\n",
         warps_per_cta / 4, CHAINS, per, tf, per / (warps_per_cta / 4));
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  for (int w : {4, 8, 16}) {
    run<1>(w, out, cyc); run<2>(w, out, cyc); run<3>(w, out, cyc); run<4>(w, out, cyc);
    run<6>(w, out, cyc); run<8>(w, out, cyc); run<12>(w, out, cyc);
  }
  return 0;
}
