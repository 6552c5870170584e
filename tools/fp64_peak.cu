// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) issue loop,
// plain DFMA loop, and cuBLAS DGEMM (library ceiling, test/measurement only).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu -lcublas
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int CHAINS>
__global__ void dmma_loop(double* out, int iters){
  double c[CHAINS][2];
  double a = threadIdx.x*1e-3, b = 1.0 + threadIdx.x*1e-6;
  #pragma unroll
  for(int i=0;i<CHAINS;i++){c[i][0]=0;c[i][1]=0;}
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CHAINS;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]),"+d"(c[i][1]) : "d"(a),"d"(b));
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CHAINS;i++) s+=c[i][0]+c[i][1];
  if(s==12345.678) out[0]=s;
}
// uniform [-1, 1) fill from a splitmix64 hash of the index (non-trivial operands: a zero-filled
// DGEMM draws less power and can run faster than real data)
__global__ void fill_random(double* p, size_t cnt, unsigned long long seed){
  for(size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; i < cnt; i += (size_t)gridDim.x*blockDim.x){
    unsigned long long z = seed*0x9E3779B97F4A7C15ull + i + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
  }
}
template<int CHAINS>
__global__ void dfma_loop(double* out, int iters){
  double c[CHAINS];
  double a = threadIdx.x*1e-3, b = 1.0 - threadIdx.x*1e-9;
  #pragma unroll
  for(int i=0;i<CHAINS;i++) c[i]=i;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<CHAINS;i++) c[i]=fma(c[i],b,a);
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CHAINS;i++) s+=c[i];
  if(s==12345.678) out[0]=s;
}

int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("device %s SMs %d clock(kHz) %d smemPerBlockOptin %zu\n", p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerBlockOptin);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DMMA: each mma = 8*8*4 FMA = 512 flop per warp
  for(int warps: {4,8,16}){
    int iters = 20000; dim3 grid(sms*2), block(32*warps);
    dmma_loop<8><<<grid,block>>>(out, 100);
    cudaEventRecord(e0); dmma_loop<8><<<grid,block>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops = 512.0*8*iters*(double)warps*grid.x;
    printf("DMMA m8n8k4 warps/CTA=%d CTAs=%d: %.2f TFLOP/s (%.3f ms)\n", warps, grid.x, flops/ms/1e9, ms);
  }
  for(int warps: {8,16,32}){
    int iters = 20000; dim3 grid(sms*2), block(32*warps);
    dfma_loop<8><<<grid,block>>>(out, 100);
    cudaEventRecord(e0); dfma_loop<8><<<grid,block>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double flops = 2.0*8*iters*(double)block.x*grid.x;
    printf("DFMA warps/CTA=%d: %.2f TFLOP/s\n", warps, flops/ms/1e9);
  }
  // cuBLAS DGEMM
  cublasHandle_t h; cublasCreate(&h);
  for(int n: {4096, 8192, 16384}){
    double *A,*B,*C; CK(cudaMalloc(&A,(size_t)n*n*8)); CK(cudaMalloc(&B,(size_t)n*n*8)); CK(cudaMalloc(&C,(size_t)n*n*8));
    fill_random<<<1024,256>>>(A,(size_t)n*n,1); fill_random<<<1024,256>>>(B,(size_t)n*n,2);
    double one=1, zero=0;
    cublasDgemm(h,CUBLAS_OP_N,CUBLAS_OP_N,n,n,n,&one,A,n,B,n,&zero,C,n);
    CK(cudaDeviceSynchronize());
    int reps = n>=16384?3:10; float best=1e30;
    for(int r=0;r<reps;r++){
      cudaEventRecord(e0); cublasDgemm(h,CUBLAS_OP_N,CUBLAS_OP_N,n,n,n,&one,A,n,B,n,&zero,C,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms,e0,e1); if(ms<best) best=ms;
    }
    printf("cuBLAS DGEMM n=%d: %.2f TFLOP/s (best of %d, %.2f ms)\n", n, 2.0*n*(double)n*n/best/1e9, reps, best);
    // sustained: back to back ~4 s
    if(n==8192){
      int cnt=0; cudaEventRecord(e0);
      for(cnt=0; cnt<100; cnt++) cublasDgemm(h,CUBLAS_OP_N,CUBLAS_OP_N,n,n,n,&one,A,n,B,n,&zero,C,n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms,e0,e1);
      printf("cuBLAS DGEMM n=%d sustained x%d: %.2f TFLOP/s (%.1f ms)\n", n, cnt, 2.0*n*(double)n*n*cnt/ms/1e9, ms);
    }
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
  return 0;
}
