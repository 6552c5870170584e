// Micro-benchmark behind DESIGN.md section 10 (bulge chase): can consecutive sweeps hand their
// 48 KB task window over through distributed shared memory faster than through L2?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_pingpong tools/dsmem_pingpong.cu
// cluster of 2: CTA 0 pushes NB doubles into CTA 1's smem (st.shared::cluster) then arrives on
// CTA 1's mbarrier (release.cluster); CTA 1 waits (acquire.cluster) and arrives back.  Optional
// global stores by CTA 0 before the push.  Round-trip time per round.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned map_rank(const void* p, int rank) {
  unsigned r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank)); return r; }
__device__ __forceinline__ void st_cluster(unsigned addr, double v) { asm volatile("st.shared::cluster.f64 [%0], %1;" :: "r"(addr), "d"(v) : "memory"); }
__device__ __forceinline__ void arrive_remote(unsigned bar) { asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(bar) : "memory"); }
__device__ __forceinline__ void wait_acq(uint64_t* bar, unsigned par) {
  unsigned done = 0;
  while (!done) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(par) : "memory");
}
constexpr int NB = 6000;
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384) pp(double* g, int rounds, int gstores, long long* out) {
  __shared__ double buf[NB];
  __shared__ uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(&bar)), "r"(12) : "memory"); }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  cl.sync();
  const unsigned rbuf = map_rank(buf, rank ^ 1), rbar = map_rank(&bar, rank ^ 1);
  long long t0 = clock64();
  for (int it = 0; it < rounds; it++) {
    if (rank == 0) {
      if (gstores) for (int i = tid; i < NB; i += 384) __stcg(&g[(size_t)blockIdx.x * NB * 4 + (size_t)(it & 3) * NB + i], (double)it);
      for (int i = tid; i < NB; i += 384) st_cluster(rbuf + 8 * i, (double)it);
      __syncwarp();
      if (lane == 0) arrive_remote(rbar);
      wait_acq(&bar, it & 1);
    } else {
      wait_acq(&bar, it & 1);
      __syncwarp();
      if (lane == 0) arrive_remote(rbar);
    }
  }
  long long t1 = clock64();
  if (tid == 0 && rank == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  cl.sync();
}
int main() {
  double* g; cudaMalloc(&g, 8ull * NB * 4 * 2);
  long long* o; cudaMallocManaged(&o, 8);
  for (int gs = 0; gs < 2; gs++) {
    pp<<<2, 384>>>(g, 1000, gs, o); cudaDeviceSynchronize();
    pp<<<2, 384>>>(g, 10000, gs, o); cudaError_t e = cudaDeviceSynchronize();
    printf("global stores %d: %s  %.0f cycles per round trip (%d doubles pushed)\n", gs, cudaGetErrorString(e), (double)o[0] / 10000, NB);
  }
  return 0;
}
