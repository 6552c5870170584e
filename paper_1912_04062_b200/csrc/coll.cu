// coll.cu -- the collectives of the distributed path behind one interface:
//
//   coll_bcast      the owner's panel V / T / tau  (full->band, per panel)
//   coll_allreduce  the partial skew-SYMM products and the band (sum, in place)
//   coll_allgather  the multisection eigenvalue slices (in place)
//
// Two backends:
//   * NCCL (one process per GPU, NVLink / NVSwitch): the production path.
//   * virtual ranks: P contexts of ONE device in one process, each driven by its own host
//     thread and stream (skew_vgroup_create / skew_ctx_create_virtual).  A collective
//     synchronises the caller's stream, meets the other ranks at a host barrier, and moves
//     the data with device copies / a fixed-order sum kernel that read the peers' buffers
//     directly.  It exercises the distributed ownership, partition and ghost-window logic on
//     a single GPU (tests/test_gpu_virtual_ranks.py); it is a test harness, not a fast path,
//     and it allocates its own reduction scratch (cudaMalloc, once per size).
#include "common.cuh"
#include "internal.h"
#include <condition_variable>
#include <mutex>
#include <nccl.h>
#include <vector>

namespace sk {

struct VGroup {
  int P = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<void*> ptr;        // per rank: the buffer of the current collective
  std::vector<double*> scratch;  // per rank: allreduce scratch
  std::vector<size_t> scratch_n;
  explicit VGroup(int p) : P(p), ptr(p, nullptr), scratch(p, nullptr), scratch_n(p, 0) {}
  ~VGroup() {
    for (double* s : scratch)
      if (s) cudaFree(s);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t g = gen;
    if (++arrived == P) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

VGroup* vgroup_new(int P) { return new VGroup(P); }
void vgroup_free(VGroup* g) { delete g; }

// fixed-order (rank 0 .. P-1) sum of P device arrays
__global__ void vsum_kernel(const double* const* src, int P, size_t n, double* dst) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < P; r++) s += src[r][i];
    dst[i] = s;
  }
}

static int nccl_status(ncclResult_t r) { return r == ncclSuccess ? 0 : (int)r; }

int coll_bcast(const Dist& d, void* buf, size_t bytes, int root, cudaStream_t st) {
  if (d.P <= 1 || bytes == 0) return 0;
  if (d.vg) {
    VGroup& g = *d.vg;
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    g.ptr[d.rank] = buf;
    g.barrier();
    if (d.rank != root) {
      if (cudaMemcpyAsync(buf, g.ptr[root], bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return -1;
      if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    }
    g.barrier();   // the root's buffer stays untouched until every rank has copied it
    return 0;
  }
  return nccl_status(ncclBroadcast(buf, buf, bytes, ncclChar, root, (ncclComm_t)d.comm, st));
}

int coll_group_start(const Dist& d) { return (d.P > 1 && !d.vg) ? nccl_status(ncclGroupStart()) : 0; }
int coll_group_end(const Dist& d) { return (d.P > 1 && !d.vg) ? nccl_status(ncclGroupEnd()) : 0; }

int coll_allreduce_sum(const Dist& d, double* buf, size_t count, cudaStream_t st) {
  if (d.P <= 1 || count == 0) return 0;
  if (d.vg) {
    VGroup& g = *d.vg;
    if (g.scratch_n[d.rank] < count + (size_t)g.P) {
      if (g.scratch[d.rank]) cudaFree(g.scratch[d.rank]);
      g.scratch[d.rank] = nullptr;
      if (cudaMalloc(&g.scratch[d.rank], sizeof(double) * (count + g.P)) != cudaSuccess) return -1;
      g.scratch_n[d.rank] = count + g.P;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    g.ptr[d.rank] = buf;
    g.barrier();
    double* tmp = g.scratch[d.rank];
    const double** srcs = reinterpret_cast<const double**>(tmp + count);   // P pointers after the sum
    std::vector<const double*> hs(g.P);
    for (int r = 0; r < g.P; r++) hs[r] = static_cast<const double*>(g.ptr[r]);
    if (cudaMemcpyAsync(srcs, hs.data(), sizeof(double*) * g.P, cudaMemcpyHostToDevice, st) != cudaSuccess) return -1;
    vsum_kernel<<<(unsigned)std::min<size_t>((count + 255) / 256, 1024), 256, 0, st>>>(srcs, g.P, count, tmp);
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    g.barrier();   // every rank has read every input
    if (cudaMemcpyAsync(buf, tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return -1;
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    return 0;
  }
  return nccl_status(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, (ncclComm_t)d.comm, st));
}

// in place: rank r's slice is buf[r*count, (r+1)*count)
int coll_allgather(const Dist& d, double* buf, size_t count, cudaStream_t st) {
  if (d.P <= 1 || count == 0) return 0;
  if (d.vg) {
    VGroup& g = *d.vg;
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    g.ptr[d.rank] = buf;
    g.barrier();
    for (int r = 0; r < g.P; r++)
      if (r != d.rank &&
          cudaMemcpyAsync(buf + (size_t)r * count, static_cast<double*>(g.ptr[r]) + (size_t)r * count,
                          sizeof(double) * count, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return -1;
    if (cudaStreamSynchronize(st) != cudaSuccess) return -1;
    g.barrier();
    return 0;
  }
  return nccl_status(ncclAllGather(buf + (size_t)d.rank * count, buf, count, ncclDouble, (ncclComm_t)d.comm, st));
}

const char* coll_error_string(const Dist& d, int code) {
  if (d.vg) return "virtual-rank collective failed (CUDA error)";
  return ncclGetErrorString((ncclResult_t)code);
}

}  // namespace sk
