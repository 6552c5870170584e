// CUDA implementation of the SAME counter-based generator as skewgen/gen.py (bit-identical;
// checked by tests/test_generator.py). Input generation only: no method arithmetic.
// Writes the strictly-lower triangle of a column-major n x n skew matrix (ld >= n);
// the diagonal and upper triangle are written as 0.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t sg_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void sg_skew_lower_kernel(double* A, int64_t n, int64_t ld, uint64_t seed) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
    uint64_t base = seed * 0x9E3779B97F4A7C15ull + (uint64_t)j * (uint64_t)n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      double v = 0.0;
      if (i > j) {
        uint64_t z = sg_splitmix64(base + (uint64_t)i);
        v = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
      }
      A[i + j * ld] = v;
    }
  }
}

extern "C" int skewgen_random_skew_lower_device(double* A, int64_t n, int64_t ld, uint64_t seed, void* stream) {
  if (n < 1 || ld < n) return -1;
  dim3 grid((unsigned)((n + 255) / 256 > 64 ? 64 : (n + 255) / 256), (unsigned)(n < 65535 ? n : 65535));
  sg_skew_lower_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(A, n, ld, seed);
  return (int)cudaGetLastError();
}
