// api.cu -- the C-ABI (include/skeweig.h, include/skeweig_stages.h): argument checks,
// workspace planning, host/device staging, the stage driver of Algorithm 1 (ELPA2
// flavour) and per-stage CUDA-event timing.  No compute happens on the host except
// the small tridiagonal bookkeeping (split points, task lists) in tridiag.cu.
#include <nvtx3/nvToolsExt.h>
#include "../../include/skeweig.h"
#include "../../include/skeweig_stages.h"
#include "common.cuh"
#include "internal.h"
#include "gemm_dmma.cuh"
#include "tma_gemm.cuh"
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <string>
#include <algorithm>
#include <nccl.h>

namespace sk {

thread_local Prof* g_prof = nullptr;

// ------------------------------------------------------------------------------------
struct Plan {
  F2BLayout f2b;
  B2TLayout b2t;
  int64_t n = 0, nev = 0, ldn = 0;
  double* Astage = nullptr;    // n x ldn (host staging / BSE W)
  double* Mstage = nullptr;    // n x ldn (BSE: host M staged; receives L)
  double* S = nullptr;         // BSE m x m
  double* vstore = nullptr;
  F2BWork fw;
  B2TWork bw;
  double* alpha = nullptr;
  double* lam = nullptr;
  TridWork tw;
  double* Q = nullptr;         // n x nev (ld ldn)
  double* X = nullptr;         // n x 2nev (ld ldn)
  BT1Work b1;
  int64_t* status = nullptr;
  double* scratch = nullptr;
};

static void plan_layout(Ctx& c, Plan& p, Arena& ar, int64_t n, int64_t nev, int flags) {
  const bool vec = (flags & SKEW_WS_VECTORS) != 0;
  p.n = n; p.nev = nev;
  p.ldn = (n + 1) & ~int64_t(1);
  const int b = c.prm.b;
  p.f2b.init(n, b, c.prm.bt1_merge);
  p.b2t.init(n, b, c.prm.bt2_k);
  if (flags & (SKEW_WS_HOST_STAGING | SKEW_WS_BSE)) p.Astage = ar.take<double>((size_t)p.ldn * n);
  if (flags & SKEW_WS_BSE) p.S = ar.take<double>((size_t)std::max<int64_t>(n / 2, 1) * std::max<int64_t>(n / 2, 1));
  if ((flags & SKEW_WS_BSE) && (flags & SKEW_WS_HOST_STAGING)) p.Mstage = ar.take<double>((size_t)p.ldn * n);
  if (flags & SKEW_WS_BSE_BACKTRANSFORM) {   // skew_bse_backtransform: Y = L Z (2 planes) + column norms
    ar.take<double>((size_t)n * 2 * std::max<int64_t>(nev, 1));
    ar.take<double>((size_t)std::max<int64_t>(nev, 1));
  }
  p.vstore = ar.take<double>((size_t)std::max<int64_t>(p.f2b.vstore_elems, 1));
  f2b_reserve(ar, p.f2b, c.num_sms, p.fw, c.nranks);
  b2t_reserve(ar, p.b2t, vec, p.bw);
  p.alpha = ar.take<double>(std::max<int64_t>(n, 1));
  p.lam = ar.take<double>(std::max<int64_t>(nev, 1));
  trid_reserve(ar, n, nev, vec, p.tw, c.prm.reorth_w);
  if (vec) {
    p.Q = ar.take<double>((size_t)p.ldn * std::max<int64_t>(nev, 1));
    p.X = ar.take<double>((size_t)p.ldn * 2 * std::max<int64_t>(nev, 1));
    bt1_reserve(ar, p.f2b, 2 * nev, p.b1);
  }
  p.status = ar.take<int64_t>(4);
  p.scratch = ar.take<double>(64);
}

// one-step route (NEXT-4): its own layout (reflector store with r0(j) = j*b + 1, no band /
// bulge-chasing buffers)
struct PlanOS {
  F2BLayout L;
  int64_t n = 0, nev = 0, ldn = 0;
  double* vstore = nullptr;
  OneStepWork ow;
  double* alpha = nullptr;
  double* lam = nullptr;
  TridWork tw;
  double* Q = nullptr;
  double* X = nullptr;
  BT1Work b1;
  int64_t* status = nullptr;
};

static void plan_onestep(Ctx& c, PlanOS& p, Arena& ar, int64_t n, int64_t nev, bool vec) {
  p.n = n; p.nev = nev;
  p.ldn = (n + 1) & ~int64_t(1);
  p.L.init(n, c.prm.b, c.prm.bt1_merge, true);
  if (vec) p.vstore = ar.take<double>((size_t)std::max<int64_t>(p.L.vstore_elems, 1));
  onestep_reserve(ar, p.L, p.ow);
  p.alpha = ar.take<double>(std::max<int64_t>(n, 1));
  p.lam = ar.take<double>(std::max<int64_t>(nev, 1));
  trid_reserve(ar, n, nev, vec, p.tw, c.prm.reorth_w);
  if (vec) {
    p.Q = ar.take<double>((size_t)p.ldn * std::max<int64_t>(nev, 1));
    p.X = ar.take<double>((size_t)p.ldn * 2 * std::max<int64_t>(nev, 1));
    bt1_reserve(ar, p.L, 2 * nev, p.b1);
  }
  p.status = ar.take<int64_t>(4);
}

static bool plan_bind(Ctx& c, Plan& p, int64_t n, int64_t nev, int flags) {
  Arena ar;
  ar.base = (char*)c.ws;
  ar.size = c.ws_bytes;
  plan_layout(c, p, ar, n, nev, flags);
  return !ar.fail && ar.off <= ar.size;
}

static int env_int(const char* name, int def) {
  const char* s = getenv(name);
  if (!s || !*s) return def;
  return atoi(s);
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}
// page-locked (cudaHostAlloc / cudaHostRegister) host memory: asynchronous copies overlap kernels
static bool is_pinned_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeHost;
}


}  // namespace sk

using namespace sk;

struct skew_ctx_s {
  Ctx c;
  Prof prof;
  cudaEvent_t ev_start[ST_COUNT];
  cudaEvent_t ev_stop[ST_COUNT];
  bool used[ST_COUNT];
  nvtxRangeId_t nvtx[ST_COUNT];   // host-side stage ranges for Nsight Systems (no-ops without a tool)
};

static int set_cuda_err(skew_ctx ctx, cudaError_t e, const char* where) {
  cudaGetLastError();   // clear a non-sticky error so the caller's runtime state stays clean
  if (ctx) ctx->c.last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return SKEW_ERR_CUDA;
}
#define CK(call, where)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return set_cuda_err(ctx, _e, where); \
  } while (0)

static const char* kStageNvtx[ST_COUNT] = {"skeweig full->band", "skeweig band->tridiagonal", "skeweig tridiagonal",
                                           "skeweig BT2", "skeweig BT1", "skeweig output", "skeweig BSE"};
static void tstart(skew_ctx ctx, int s) {
  cudaEventRecord(ctx->ev_start[s], ctx->c.stream);
  ctx->used[s] = true;
  ctx->nvtx[s] = nvtxRangeStartA(kStageNvtx[s]);
}
static void tstop(skew_ctx ctx, int s) {
  cudaEventRecord(ctx->ev_stop[s], ctx->c.stream);
  nvtxRangeEnd(ctx->nvtx[s]);
}
static void tcollect(skew_ctx ctx) {
  for (int s = 0; s < ST_COUNT; s++) {
    float ms = 0.f;
    if (ctx->used[s] && cudaEventElapsedTime(&ms, ctx->ev_start[s], ctx->ev_stop[s]) == cudaSuccess)
      ctx->c.stage_ms[s] = ms;
    else ctx->c.stage_ms[s] = 0.0;
  }
}
static void treset(skew_ctx ctx) {
  for (int s = 0; s < ST_COUNT; s++) ctx->used[s] = false;
  ctx->prof.reset();
  g_prof = &ctx->prof;
}
// collect per-kernel-class event timings once the stream is synchronised
static void kcollect(skew_ctx ctx) {
  if (ctx->prof.on) ctx->prof.collect();
}
static const char* kNames[KC_COUNT] = {"panel_qr", "vt", "skew_symm", "w_correction", "skew_r2k", "band_extract",
                                       "bulge_chase", "bisection", "inverse_iteration", "reorth", "assemble_D",
                                       "bt2_tbuild", "bt2_apply", "bt1_prep", "bt1_z", "bt1_update", "output", "bse",
                                       "onestep_skew_mv", "onestep_column", "collectives"};

extern "C" {

int skew_ctx_create(skew_ctx* out, int device, void* cuda_stream) {
  if (!out) return -1;
  skew_ctx ctx = new skew_ctx_s();
  ctx->c.device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete ctx; return SKEW_ERR_CUDA; }
  ctx->c.stream = (cudaStream_t)cuda_stream;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  ctx->c.num_sms = nsm;
  ctx->c.prm.b = 64;   // band width: fixed (the F2B panel, chase and BT2 kernels are built for b = 64)
  ctx->c.prm.bt2_k = env_int("SKEWEIG_BT2_K", 32);
  ctx->c.prm.bt1_merge = env_int("SKEWEIG_BT1_MERGE", 8);
  ctx->c.prm.reorth_w = env_int("SKEWEIG_REORTH_W", 32);
  if (ctx->c.prm.bt2_k != 32) ctx->c.prm.bt2_k = 32;
  if (ctx->c.prm.bt1_merge < 1 || ctx->c.prm.bt1_merge > 8) ctx->c.prm.bt1_merge = 8;
  if (ctx->c.prm.reorth_w < 0 || ctx->c.prm.reorth_w > 256) ctx->c.prm.reorth_w = 32;
  for (int s = 0; s < ST_COUNT; s++) {
    cudaEventCreate(&ctx->ev_start[s]);
    cudaEventCreate(&ctx->ev_stop[s]);
    ctx->used[s] = false;
  }
  *out = ctx;
  return SKEW_OK;
}

int skew_get_unique_id(char id[128]) {
  if (!id) return -1;
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return SKEW_ERR_NCCL;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &u, 128);
  return SKEW_OK;
}

int skew_ctx_create_dist(skew_ctx* out, int device, void* cuda_stream, int nranks, int rank, const char id[128]) {
  if (!out) return -1;
  if (nranks < 1) return -4;
  if (rank < 0 || rank >= nranks) return -5;
  if (!id) return -6;
  int rc = skew_ctx_create(out, device, cuda_stream);
  if (rc != SKEW_OK) return rc;
  skew_ctx ctx = *out;
  ctx->c.nranks = nranks;
  ctx->c.rank = rank;
  if (nranks > 1) {
    if (ctx->c.prm.b != 64) { skew_ctx_destroy(ctx); *out = nullptr; return SKEW_ERR_NOT_IMPLEMENTED; }
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, nranks, u, rank);
    if (r != ncclSuccess) { skew_ctx_destroy(ctx); *out = nullptr; return SKEW_ERR_NCCL; }
    ctx->c.nccl = comm;
  }
  return SKEW_OK;
}

int64_t skew_tile_schedule(int64_t ntm, int nranks, int rank, int64_t* tm_out, int64_t* tn_out, int64_t cap) {
  if (ntm < 0) return -1;
  if (nranks < 1) return -2;
  if (rank < 0 || rank >= nranks) return -3;
  if (cap < 0 || ((!tm_out || !tn_out) && cap > 0)) return -6;
  // the rank-2k kernel's schedule (tma_gemm<128, 64, ..., TRI>): 128-row x 64-column tiles of
  // an ntm*128 square trailing matrix, the same host/device tile decoder as the kernel
  const int64_t tmr = ntm, tn = 2 * ntm;
  TmaGemmArgs g;
  g.ntiles = tmr * (tmr + 1);   // R = 2: sum_tm 2 (tm + 1)
  if (nranks > 1) {
    if (rank >= tn) return 0;
    g.col_stride = nranks; g.col_off = rank; g.ntm = tmr;
    g.kloc = (tn - rank + nranks - 1) / nranks;
    g.ntiles = tri_strided_count(g.kloc, tmr, rank, nranks, 2);
  }
  for (int64_t t = 0; t < g.ntiles && t < cap; t++) {
    int64_t a, b;
    tma_tile_coords<128, 64>(g, t, true, a, b);
    tm_out[t] = a;
    tn_out[t] = b;
  }
  return g.ntiles;
}

int skew_vgroup_create(int nranks, void** out) {
  if (nranks < 1) return -1;
  if (!out) return -2;
  *out = vgroup_new(nranks);
  return SKEW_OK;
}

int skew_vgroup_destroy(void* group) {
  if (!group) return -1;
  vgroup_free(static_cast<VGroup*>(group));
  return SKEW_OK;
}

int skew_ctx_create_virtual(skew_ctx* out, int device, void* cuda_stream, void* group, int nranks, int rank) {
  if (!out) return -1;
  if (!group) return -4;
  if (nranks < 1) return -5;
  if (rank < 0 || rank >= nranks) return -6;
  int rc = skew_ctx_create(out, device, cuda_stream);
  if (rc != SKEW_OK) return rc;
  (*out)->c.nranks = nranks;
  (*out)->c.rank = rank;
  (*out)->c.vg = static_cast<VGroup*>(group);
  return SKEW_OK;
}

int skew_ctx_destroy(skew_ctx ctx) {
  if (!ctx) return -1;
  if (ctx->c.nccl) ncclCommDestroy((ncclComm_t)ctx->c.nccl);
  if (ctx->c.aux) {
    cudaStreamSynchronize(ctx->c.aux);
    cudaStreamDestroy(ctx->c.aux);
    cudaEventDestroy(ctx->c.ev_fork);
    cudaEventDestroy(ctx->c.ev_join);
    cudaEventDestroy(ctx->c.ev_la_cols);
    cudaEventDestroy(ctx->c.ev_la_panel);
  }
  for (int s = 0; s < ST_COUNT; s++) { cudaEventDestroy(ctx->ev_start[s]); cudaEventDestroy(ctx->ev_stop[s]); }
  delete ctx;
  return SKEW_OK;
}

int skew_workspace_size(skew_ctx ctx, int64_t n, int64_t nev, int flags, size_t* bytes) {
  if (!ctx) return -1;
  if (n < 1) return -2;
  if (nev < 0 || nev > n / 2) return -3;
  if (!bytes) return -5;
  Arena ar;
  ar.measuring = true;
  if (flags & SKEW_WS_ONESTEP) {
    PlanOS po;
    plan_onestep(ctx->c, po, ar, n, nev, (flags & SKEW_WS_VECTORS) != 0);
  } else {
    Plan p;
    plan_layout(ctx->c, p, ar, n, nev, flags);
  }
  *bytes = ar.off + 4096;
  return SKEW_OK;
}

int skew_set_workspace(skew_ctx ctx, void* dptr, size_t bytes) {
  if (!ctx) return -1;
  if (bytes > 0 && !is_device_ptr(dptr)) return -2;
  ctx->c.ws = dptr;
  ctx->c.ws_bytes = bytes;
  return SKEW_OK;
}

int skew_stage_times(skew_ctx ctx, double* ms_out, int count) {
  if (!ctx) return -1;
  if (!ms_out || count < 0 || count > ST_COUNT) return -2;
  for (int i = 0; i < count; i++) ms_out[i] = ctx->c.stage_ms[i];
  return SKEW_OK;
}

int skew_set_profiling(skew_ctx ctx, int on) {
  if (!ctx) return -1;
  ctx->prof.on = (on != 0);
  return SKEW_OK;
}

int skew_kernel_stats(skew_ctx ctx, double* ms_out, int64_t* launches_out, int count) {
  if (!ctx) return -1;
  if (count < 0 || count > KC_COUNT) return -4;
  for (int i = 0; i < count; i++) {
    if (ms_out) ms_out[i] = ctx->prof.ms[i];
    if (launches_out) launches_out[i] = ctx->prof.launches[i];
  }
  return SKEW_OK;
}

const char* skew_kernel_class_name(int cls) { return (cls >= 0 && cls < KC_COUNT) ? kNames[cls] : "?"; }

int64_t skew_last_nfail(skew_ctx ctx) { return ctx ? ctx->c.last_nfail : -1; }

const char* skew_last_error(skew_ctx ctx) { return ctx ? ctx->c.last_error.c_str() : "null context"; }

const char* skew_status_string(int status) {
  switch (status) {
    case SKEW_OK: return "ok";
    case SKEW_ERR_NOCONV: return "inverse iteration did not converge for some eigenvectors";
    case SKEW_ERR_NOT_DEFINITE: return "matrix is not positive definite (Cholesky pivot too small)";
    case SKEW_ERR_CUDA: return "CUDA error";
    case SKEW_ERR_NCCL: return "NCCL error";
    case SKEW_ERR_WORKSPACE: return "workspace missing or too small";
    case SKEW_ERR_NOT_IMPLEMENTED: return "not implemented";
    default: return status < 0 ? "invalid argument" : "unknown status";
  }
}

// 1 if the lower triangle (strictly lower unless diag) of the device array A holds a NaN or
// Inf, 0 if not, SKEW_ERR_CUDA on a CUDA failure.  One device pass + one host sync.
static int check_finite(skew_ctx ctx, Plan& p, const double* A_d, int64_t lda, int64_t n, bool diag) {
  int* flag = reinterpret_cast<int*>(p.status + 2);
  int h = 0;
  CK(nonfinite_lower(A_d, lda, n, diag, flag, ctx->c.stream), "finite check");
  CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.stream), "finite flag");
  CK(cudaStreamSynchronize(ctx->c.stream), "sync");
  return h ? 1 : 0;
}

// ------------------------------------------------------------------------------------
// The solve driver shared by skew_eig / skew_eigvals / skew_eig_bse.
// A_d: device skew input (strictly lower), destroyed.  lam_out/Zre/Zim: device or host.
// write_z = false: the eigenvectors stay in p.X ([Re | Im], ld p.ldn) for a caller-side epilogue.
static int solve_core(skew_ctx ctx, Plan& p, double* A_d, int64_t lda, int64_t nev, double* lambda, bool lam_host,
                      double* Zre, double* Zim, int64_t ldz, bool z_host, int64_t k0, int64_t k1,
                      bool write_z = true) {
  const int64_t nloc = k1 - k0;   // eigenvectors [k0, k1) are computed and returned
  Ctx& c = ctx->c;
  cudaStream_t st = c.stream;
  const int64_t n = p.n;
  const bool vec = (Zre != nullptr);
  bool re_early = false;   // real parts downloaded during BT1 of the imaginary parts
  if (vec && p.f2b.npanel > 0) CK(bt1_upload_meta(p.f2b, p.b1, st), "bt1 meta");
  if ((vec || c.nranks > 1) && !c.aux) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);   // hi = greatest priority (the look-ahead panel)
    CK(cudaStreamCreateWithPriority(&c.aux, cudaStreamNonBlocking, hi), "aux stream");
    CK(cudaEventCreateWithFlags(&c.ev_fork, cudaEventDisableTiming), "fork event");
    CK(cudaEventCreateWithFlags(&c.ev_join, cudaEventDisableTiming), "join event");
    CK(cudaEventCreateWithFlags(&c.ev_la_cols, cudaEventDisableTiming), "look-ahead event");
    CK(cudaEventCreateWithFlags(&c.ev_la_panel, cudaEventDisableTiming), "look-ahead event");
  }
  // ---- full -> band
  tstart(ctx, ST_F2B);
  Dist d;
  d.P = c.nranks; d.rank = c.rank; d.comm = c.nccl; d.vg = c.vg;
  if (d.P > 1 && !getenv("SKEWEIG_NO_LOOKAHEAD")) {   // env: experiments only
    d.aux = c.aux; d.ev_cols = c.ev_la_cols; d.ev_panel = c.ev_la_panel;
  }
  if (p.f2b.npanel > 0) {
    CK(cudaMemsetAsync(p.vstore, 0, sizeof(double) * p.f2b.vstore_elems, st), "memset vstore");
    int nerr = 0;
    cudaError_t fe = f2b_run(p.f2b, A_d, lda, p.vstore, p.fw, c.num_sms, st, d, &nerr);
    if (nerr) { c.last_error = std::string("f2b: ") + coll_error_string(d, nerr); return SKEW_ERR_NCCL; }
    CK(fe, "f2b");
  }
  tstop(ctx, ST_F2B);
  // BT1 preparation (depends on full->band only) on the auxiliary stream: already beside the
  // chase when the chase leaves most SMs idle (small n: one CTA per active sweep), else beside
  // the tridiagonal solve (below)
  const bool bt1_early = vec && p.f2b.npanel > 0 && 2 * b2t_chase_ctas(n, c.prm.b, c.num_sms) <= c.num_sms;
  if (bt1_early) {
    CK(cudaEventRecord(c.ev_fork, st), "fork");
    CK(cudaStreamWaitEvent(c.aux, c.ev_fork, 0), "fork wait");
    CK(bt1_prep(p.f2b, p.vstore, p.fw.T, p.b1, c.aux), "bt1 prep");
  }
  // ---- band -> tridiagonal
  tstart(ctx, ST_B2T);
  CK(band_extract(A_d, lda, n, c.prm.b, p.bw.AB, p.b2t.ldab, st, d.P, d.rank), "band extract");
  if (d.P > 1) {   // every rank contributed the band columns it owns
    KScope ks(KC_COLL, st);
    const int r = coll_allreduce_sum(d, p.bw.AB, (size_t)p.b2t.ldab * n, st);
    if (r) { c.last_error = std::string("band allreduce: ") + coll_error_string(d, r); return SKEW_ERR_NCCL; }
  }
  CK(b2t_run(p.b2t, p.bw, p.alpha, c.num_sms, st), "b2t");
  tstop(ctx, ST_B2T);
  if (vec) {   // BT2 / BT1 preparation on the auxiliary stream, concurrent with the tridiagonal solve
    CK(cudaEventRecord(c.ev_fork, st), "fork");
    CK(cudaStreamWaitEvent(c.aux, c.ev_fork, 0), "fork wait");
    CK(bt2_prep(p.b2t, p.bw, c.aux), "bt2 prep");
    if (p.f2b.npanel > 0 && !bt1_early) CK(bt1_prep(p.f2b, p.vstore, p.fw.T, p.b1, c.aux), "bt1 prep");
    CK(cudaEventRecord(c.ev_join, c.aux), "join");
  }
  // ---- tridiagonal eigenproblem
  tstart(ctx, ST_TRID);
  int64_t nfail = 0;
  int64_t vlo = k0;
  CK(trid_run(n, p.alpha, nev, p.lam, vec ? p.Q : nullptr, p.ldn, p.tw, c.prm, &nfail, st, k0, k1, &vlo, &d),
     "tridiagonal");
  c.last_nfail = nfail;
  if (vec) {
    CK(assemble_D(p.Q + SK_IDX(0, k0 - vlo, p.ldn), p.ldn, n, nloc, p.X, p.ldn, st), "assemble D");
    if (p.ldn > n)   // zero padding row (read, unchanged, by the BT2 bulk copies when n is odd)
      CK(cudaMemset2DAsync(p.X + n, p.ldn * 8, 0, (p.ldn - n) * 8, 2 * nloc, st), "pad row");
  }
  tstop(ctx, ST_TRID);
  if (vec) {
    CK(cudaStreamWaitEvent(st, c.ev_join, 0), "join wait");
    tstart(ctx, ST_BT2);
    CK(bt2_apply(p.b2t, p.bw, p.X, p.ldn, 2 * nloc, st), "bt2");
    tstop(ctx, ST_BT2);
    tstart(ctx, ST_BT1);
    // pinned host Z: BT1 on the real parts, whose download (on the auxiliary stream) then
    // overlaps BT1 on the imaginary parts (the column halves are independent: X <- Q1 X)
    re_early = z_host && write_z && p.f2b.npanel > 0 && is_pinned_host(Zre) && !getenv("SKEWEIG_NO_OUT_OVERLAP");
    if (re_early) {
      CK(bt1_apply(p.f2b, p.vstore, p.fw.tau, p.fw.T, p.X, p.ldn, nloc, p.b1, st), "bt1 (real parts)");
      CK(cudaEventRecord(c.ev_fork, st), "fork");
      CK(cudaStreamWaitEvent(c.aux, c.ev_fork, 0), "fork wait");
      CK(cudaMemcpy2DAsync(Zre, ldz * 8, p.X, p.ldn * 8, n * 8, nloc, cudaMemcpyDeviceToHost, c.aux), "Zre out");
      CK(cudaEventRecord(c.ev_join, c.aux), "join");
      CK(bt1_apply(p.f2b, p.vstore, p.fw.tau, p.fw.T, p.X + (size_t)p.ldn * nloc, p.ldn, nloc, p.b1, st),
         "bt1 (imaginary parts)");
    } else if (p.f2b.npanel > 0) {
      CK(bt1_apply(p.f2b, p.vstore, p.fw.tau, p.fw.T, p.X, p.ldn, 2 * nloc, p.b1, st), "bt1");
    }
    tstop(ctx, ST_BT1);
  }
  // ---- output
  tstart(ctx, ST_OUT);
  CK(cudaMemcpyAsync(lambda, p.lam, sizeof(double) * nev, lam_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                     st), "lambda out");
  if (vec && write_z) {
    if (z_host) {
      if (!re_early)
        CK(cudaMemcpy2DAsync(Zre, ldz * 8, p.X, p.ldn * 8, n * 8, nloc, cudaMemcpyDeviceToHost, st), "Zre out");
      CK(cudaMemcpy2DAsync(Zim, ldz * 8, p.X + (size_t)p.ldn * nloc, p.ldn * 8, n * 8, nloc, cudaMemcpyDeviceToHost,
                           st), "Zim out");
      if (re_early) CK(cudaStreamWaitEvent(st, c.ev_join, 0), "join wait");
    } else {
      CK(split_output(p.X, p.ldn, n, nloc, Zre, Zim, ldz, st), "split output");
    }
  }
  tstop(ctx, ST_OUT);
  CK(cudaStreamSynchronize(st), "sync");
  tcollect(ctx);
  kcollect(ctx);
  return nfail > 0 ? SKEW_ERR_NOCONV : SKEW_OK;
}

static int eig_entry(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev, double* lambda, double* Zre,
                     double* Zim, int64_t ldz, bool need_vec, int64_t k0, int64_t k1, int k0arg) {
  if (!ctx) return -1;
  if (n < 1) return -2;
  if (!A) return -3;
  if (lda < n) return -4;
  if (nev < 1 || nev > n / 2) return -5;
  if (k0arg && (k0 < 0 || k0 >= nev)) return -k0arg;
  if (k0arg && (k1 <= k0 || k1 > nev)) return -(k0arg + 1);
  const int sh = k0arg ? 2 : 0;   // skew_eig_range has two more arguments before lambda
  if (!lambda) return -(6 + sh);
  if (need_vec && !Zre) return -(7 + sh);
  if (need_vec && !Zim) return -(8 + sh);
  const bool vec = (Zre != nullptr || Zim != nullptr);
  if (vec && (!Zre)) return -(7 + sh);
  if (vec && (!Zim)) return -(8 + sh);
  if (vec && ldz < n) return -(9 + sh);
  CK(cudaSetDevice(ctx->c.device), "set device");
  treset(ctx);
  const bool a_dev = is_device_ptr(A);
  const bool l_dev = is_device_ptr(lambda);
  const bool z_dev = vec ? is_device_ptr(Zre) : a_dev;
  if (vec && is_device_ptr(Zim) != z_dev) return -(8 + sh);
  int flags = (vec ? SKEW_WS_VECTORS : 0) | (a_dev ? 0 : SKEW_WS_HOST_STAGING);
  Plan p;
  if (!ctx->c.ws || !plan_bind(ctx->c, p, n, nev, flags)) {
    ctx->c.last_error = "workspace missing or too small";
    return SKEW_ERR_WORKSPACE;
  }
  double* A_d = A;
  int64_t ldad = lda;
  if (!a_dev) {
    // host input: stage into the workspace (host A is not modified); the copy is part of the call
    ldad = p.ldn;
    CK(cudaMemcpy2DAsync(p.Astage, ldad * 8, A, lda * 8, n * 8, n, cudaMemcpyHostToDevice, ctx->c.stream), "A in");
    A_d = p.Astage;
  }
  {   // non-finite input -> argument error
    const int rc = check_finite(ctx, p, A_d, ldad, n, false);
    if (rc) return rc == 1 ? -3 : rc;
  }
  return solve_core(ctx, p, A_d, ldad, nev, lambda, !l_dev, vec ? Zre : nullptr, Zim, ldz, vec && !z_dev, k0, k1);
}

int skew_eig(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev, double* lambda, double* Zre, double* Zim,
             int64_t ldz) {
  return eig_entry(ctx, n, A, lda, nev, lambda, Zre, Zim, ldz, true, 0, nev, 0);
}

int skew_eig_range(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev, int64_t k0, int64_t k1,
                   double* lambda, double* Zre, double* Zim, int64_t ldz) {
  return eig_entry(ctx, n, A, lda, nev, lambda, Zre, Zim, ldz, true, k0, k1, 6);
}

int skew_eigvals(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev, double* lambda) {
  return eig_entry(ctx, n, A, lda, nev, lambda, nullptr, nullptr, n, false, 0, nev, 0);
}

int skew_eig_bse(skew_ctx ctx, int64_t n, double* M, int64_t ldm, int64_t nev, int flags, double* lambda, double* Zre,
                 double* Zim, int64_t ldz, int64_t* pivot_out) {
  if (!ctx) return -1;
  if (n < 2 || (n & 1)) return -2;
  if (!M) return -3;
  if (ldm < n) return -4;
  if (nev < 1 || nev > n / 2) return -5;
  if (flags & ~SKEW_BSE_HAMILTONIAN_Y) return -6;
  if (!lambda) return -7;
  if (!Zre && Zim) return -8;
  const bool vec = (Zre != nullptr);
  if (vec && !Zim) return -9;
  if ((flags & SKEW_BSE_HAMILTONIAN_Y) && !vec) return -8;
  if (vec && ldz < n) return -10;
  if (pivot_out) *pivot_out = 0;
  CK(cudaSetDevice(ctx->c.device), "set device");
  treset(ctx);
  const bool m_dev = is_device_ptr(M);
  const bool l_dev = is_device_ptr(lambda);
  const bool z_dev = vec ? is_device_ptr(Zre) : m_dev;
  if (vec && is_device_ptr(Zim) != z_dev) return -9;
  const int wflags = (vec ? SKEW_WS_VECTORS : 0) | SKEW_WS_BSE | (m_dev ? 0 : SKEW_WS_HOST_STAGING);
  Plan p;
  if (!ctx->c.ws || !plan_bind(ctx->c, p, n, nev, wflags)) {
    ctx->c.last_error = "workspace missing or too small";
    return SKEW_ERR_WORKSPACE;
  }
  cudaStream_t st = ctx->c.stream;
  double* M_d = M;
  int64_t ldmd = ldm;
  if (!m_dev) {   // host M: staged into the workspace (receives L); the host array is not modified
    ldmd = p.ldn;
    CK(cudaMemcpy2DAsync(p.Mstage, ldmd * 8, M, ldm * 8, n * 8, n, cudaMemcpyHostToDevice, st), "M in");
    M_d = p.Mstage;
  }
  {
    const int rc = check_finite(ctx, p, M_d, ldmd, n, true);
    if (rc) return rc == 1 ? -3 : rc;
  }
  tstart(ctx, ST_BSE);
  const int64_t m = n / 2;
  CK(bse_front(M_d, ldmd, n, p.Astage, p.ldn, p.S, m, p.scratch, p.status, st), "bse front");
  int64_t piv = 0;
  CK(cudaMemcpyAsync(&piv, p.status, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "pivot");
  CK(cudaStreamSynchronize(st), "sync");
  tstop(ctx, ST_BSE);
  if (piv != 0) {
    if (pivot_out) *pivot_out = piv;
    return SKEW_ERR_NOT_DEFINITE;
  }
  const bool hy = (flags & SKEW_BSE_HAMILTONIAN_Y) != 0;
  int rc = solve_core(ctx, p, p.Astage, p.ldn, nev, lambda, !l_dev, vec ? Zre : nullptr, Zim, ldz, vec && !z_dev, 0,
                      nev, !hy);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev_start[ST_BSE], ctx->ev_stop[ST_BSE]);
  ctx->c.stage_ms[ST_BSE] = ms;
  if (hy && (rc == SKEW_OK || rc == SKEW_ERR_NOCONV)) {
    // y = J L z (H y = -i lambda y for H = -J M), unnormalised.  W (in
    // Astage) is consumed by the solve, so Astage takes L [Zre | Zim] (n x 2nev <= n x n).
    double* Wre = p.Astage;
    double* Wim = p.Astage + (size_t)p.ldn * nev;
    CK(bse_lz(M_d, ldmd, n, p.X, p.X + (size_t)p.ldn * nev, p.ldn, nev, Wre, Wim, p.ldn, st), "bse L z");
    if (z_dev) {
      CK(bse_apply_J(Wre, Wim, p.ldn, n, nev, Zre, Zim, ldz, st), "bse J y");
    } else {
      CK(bse_apply_J(Wre, Wim, p.ldn, n, nev, p.X, p.X + (size_t)p.ldn * nev, p.ldn, st), "bse J y");
      CK(cudaMemcpy2DAsync(Zre, ldz * 8, p.X, p.ldn * 8, n * 8, nev, cudaMemcpyDeviceToHost, st), "Yre out");
      CK(cudaMemcpy2DAsync(Zim, ldz * 8, p.X + (size_t)p.ldn * nev, p.ldn * 8, n * 8, nev, cudaMemcpyDeviceToHost, st),
         "Yim out");
    }
    CK(cudaStreamSynchronize(st), "sync");
  }
  return rc;
}

// ------------------------------------------------------------------------------------
// NEXT-4: one-step route (onestep.cu), device arrays only
int skew_eig_onestep(skew_ctx ctx, int64_t n, double* A, int64_t lda, int64_t nev, double* lambda, double* Zre,
                     double* Zim, int64_t ldz) {
  if (!ctx) return -1;
  if (n < 1) return -2;
  if (!A || !is_device_ptr(A)) return -3;
  if (lda < n) return -4;
  if (nev < 1 || nev > n / 2) return -5;
  if (!lambda || !is_device_ptr(lambda)) return -6;
  if (!Zre && Zim) return -7;
  const bool vec = (Zre != nullptr);
  if (vec && (!is_device_ptr(Zre))) return -7;
  if (vec && (!Zim || !is_device_ptr(Zim))) return -8;
  if (vec && ldz < n) return -9;
  CK(cudaSetDevice(ctx->c.device), "set device");
  treset(ctx);
  Ctx& c = ctx->c;
  cudaStream_t st = c.stream;
  PlanOS p;
  {
    Arena ar;
    ar.base = (char*)c.ws;
    ar.size = c.ws_bytes;
    plan_onestep(c, p, ar, n, nev, vec);
    if (!c.ws || ar.fail) {
      c.last_error = "workspace missing or too small (size it with SKEW_WS_ONESTEP)";
      return SKEW_ERR_WORKSPACE;
    }
  }
  {
    int* flag = reinterpret_cast<int*>(p.status + 2);
    int h = 0;
    CK(nonfinite_lower(A, lda, n, false, flag, st), "finite check");
    CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st), "finite flag");
    CK(cudaStreamSynchronize(st), "sync");
    if (h) return -3;
  }
  if (vec && p.L.npanel > 0) CK(bt1_upload_meta(p.L, p.b1, st), "bt1 meta");
  tstart(ctx, ST_F2B);   // the one-step full -> tridiagonal reduction
  if (vec) CK(cudaMemsetAsync(p.vstore, 0, sizeof(double) * std::max<int64_t>(p.L.vstore_elems, 1), st), "vstore");
  if (n >= 2) CK(onestep_run(p.L, A, lda, vec ? p.vstore : nullptr, p.ow, p.alpha, c.num_sms, st), "onestep");
  tstop(ctx, ST_F2B);
  tstart(ctx, ST_TRID);
  int64_t nfail = 0, vlo = 0;
  CK(trid_run(n, p.alpha, nev, p.lam, vec ? p.Q : nullptr, p.ldn, p.tw, c.prm, &nfail, st, 0, nev, &vlo, nullptr),
     "tridiagonal");
  c.last_nfail = nfail;
  if (vec) {
    CK(assemble_D(p.Q, p.ldn, n, nev, p.X, p.ldn, st), "assemble D");
    if (p.ldn > n) CK(cudaMemset2DAsync(p.X + n, p.ldn * 8, 0, (p.ldn - n) * 8, 2 * nev, st), "pad row");
  }
  tstop(ctx, ST_TRID);
  if (vec) {
    tstart(ctx, ST_BT1);
    if (p.L.npanel > 0) {
      CK(onestep_bt_prep(p.L, p.vstore, p.ow.tau, p.b1, st), "onestep bt prep");
      CK(bt1_apply(p.L, p.vstore, p.ow.tau, nullptr, p.X, p.ldn, 2 * nev, p.b1, st), "onestep bt");
    }
    tstop(ctx, ST_BT1);
  }
  tstart(ctx, ST_OUT);
  CK(cudaMemcpyAsync(lambda, p.lam, sizeof(double) * nev, cudaMemcpyDeviceToDevice, st), "lambda out");
  if (vec) CK(split_output(p.X, p.ldn, n, nev, Zre, Zim, ldz, st), "split output");
  tstop(ctx, ST_OUT);
  CK(cudaStreamSynchronize(st), "sync");
  tcollect(ctx);
  kcollect(ctx);
  return nfail > 0 ? SKEW_ERR_NOCONV : SKEW_OK;
}

// ------------------------------------------------------------------------------------
// Full H_BS pipeline stages (steps 1 and 4 of PAPER.md:596-606; step 2-3 = skew_eig_bse)
int skew_bse_build_M(skew_ctx ctx, int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb, double* M,
                     int64_t ldm) {
  if (!ctx) return -1;
  if (n < 1) return -2;
  if (!A || !is_device_ptr(A)) return -3;
  if (lda < n) return -4;
  if (!B || !is_device_ptr(B)) return -5;
  if (ldb < n) return -6;
  if (!M || !is_device_ptr(M)) return -7;
  if (ldm < 2 * n) return -8;
  CK(cudaSetDevice(ctx->c.device), "set device");
  CK(bse_build_M(A, lda, B, ldb, n, M, ldm, ctx->c.stream), "bse build M");
  return SKEW_OK;
}

int skew_bse_backtransform(skew_ctx ctx, int64_t n2, const double* L, int64_t ldl, int64_t nev, const double* Zre,
                           const double* Zim, int64_t ldz, double* X, int64_t ldx) {
  if (!ctx) return -1;
  if (n2 < 2 || (n2 & 1)) return -2;
  if (!L || !is_device_ptr(L)) return -3;
  if (ldl < n2) return -4;
  if (nev < 0 || nev > n2 / 2) return -5;
  if (nev == 0) return SKEW_OK;
  if (!Zre || !Zim || !is_device_ptr(Zre) || !is_device_ptr(Zim)) return -6;
  if (ldz < n2) return -8;
  if (!X || !is_device_ptr(X)) return -9;
  if (ldx < n2) return -10;
  CK(cudaSetDevice(ctx->c.device), "set device");
  cudaStream_t st = ctx->c.stream;
  Arena ar;   // Y = L Z (real and imaginary planes) and the column norms, from the workspace
  ar.base = (char*)ctx->c.ws;
  ar.size = ctx->c.ws_bytes;
  double* Y = ar.take<double>((size_t)n2 * 2 * nev);
  double* nrm2 = ar.take<double>((size_t)nev);
  if (!ctx->c.ws || ar.fail || !Y || !nrm2) {
    ctx->c.last_error = "workspace missing or too small (size it with SKEW_WS_BSE_BACKTRANSFORM)";
    return SKEW_ERR_WORKSPACE;
  }
  CK(bse_backtransform(L, ldl, n2, Zre, Zim, ldz, nev, Y, Y + (size_t)n2 * nev, n2, nrm2, X, ldx, st),
     "bse backtransform");
  return SKEW_OK;
}

// ------------------------------------------------------------------------------------
// stage entry points
int skew_stage_reduce_to_band(skew_ctx ctx, int64_t n, double* A, int64_t lda, double* Vout, int64_t ldv,
                              double* Tout, double* tau_out, int64_t* npanel_out) {
  if (!ctx) return -1;
  if (n < 1) return -2;
  if (!A || !is_device_ptr(A)) return -3;
  if (lda < n) return -4;
  CK(cudaSetDevice(ctx->c.device), "set device");
  treset(ctx);
  Plan p;
  if (!ctx->c.ws || !plan_bind(ctx->c, p, n, 0, 0)) return SKEW_ERR_WORKSPACE;
  cudaStream_t st = ctx->c.stream;
  if (npanel_out) *npanel_out = p.f2b.npanel;
  tstart(ctx, ST_F2B);
  if (p.f2b.npanel > 0) {
    CK(cudaMemsetAsync(p.vstore, 0, sizeof(double) * p.f2b.vstore_elems, st), "memset");
    Dist d1;   // stage entry: single device
    int nerr = 0;
    CK(f2b_run(p.f2b, A, lda, p.vstore, p.fw, ctx->c.num_sms, st, d1, &nerr), "f2b");
  }
  tstop(ctx, ST_F2B);
  const int b = p.f2b.b;
  if (Vout && p.f2b.npanel > 0) {
    if (ldv < n) return -6;
    for (int64_t j = 0; j < p.f2b.npanel; j++) {
      int64_t g = j / p.f2b.merge, pl = j % p.f2b.merge;
      int64_t r0 = p.f2b.r0(j), m = n - r0;
      const double* Vj = p.vstore + p.f2b.goff[g] + pl * b + pl * b * p.f2b.gld[g];
      CK(cudaMemcpy2DAsync(Vout + SK_IDX(r0, j * b, ldv), ldv * 8, Vj, p.f2b.gld[g] * 8, m * 8, b,
                           cudaMemcpyDeviceToDevice, st), "V out");
    }
    if (Tout) CK(cudaMemcpyAsync(Tout, p.fw.T, sizeof(double) * b * b * p.f2b.npanel, cudaMemcpyDeviceToDevice, st), "T");
    if (tau_out) CK(cudaMemcpyAsync(tau_out, p.fw.tau, sizeof(double) * b * p.f2b.npanel, cudaMemcpyDeviceToDevice, st), "tau");
  }
  CK(cudaStreamSynchronize(st), "sync");
  tcollect(ctx);
  kcollect(ctx);
  return SKEW_OK;
}

int skew_stage_band_to_tridiag(skew_ctx ctx, int64_t n, int b, const double* AB, int64_t ldab, double* alpha_out,
                               double* X, int64_t ldx, int64_t ncols) {
  if (!ctx) return -1;
  if (n < 1) return -2;
  if (b < 1 || b > ctx->c.prm.b) return -3;
  if (!AB || !is_device_ptr(AB)) return -4;
  if (ldab < b + 1) return -5;
  if (!alpha_out) return -6;
  if (X && ldx < n) return -8;
  CK(cudaSetDevice(ctx->c.device), "set device");
  treset(ctx);
  Plan p;
  if (!ctx->c.ws || !plan_bind(ctx->c, p, n, 0, X ? SKEW_WS_VECTORS : 0)) return SKEW_ERR_WORKSPACE;
  cudaStream_t st = ctx->c.stream;
  B2TLayout L;
  L.init(n, ctx->c.prm.b, ctx->c.prm.bt2_k);
  tstart(ctx, ST_B2T);
  CK(band_copy(AB, ldab, n, b, p.bw.AB, L.ldab, st), "band copy");
  CK(b2t_run(L, p.bw, p.alpha, ctx->c.num_sms, st), "b2t");
  tstop(ctx, ST_B2T);
  if (n > 1) CK(cudaMemcpyAsync(alpha_out, p.alpha, sizeof(double) * (n - 1), cudaMemcpyDefault, st), "alpha");
  if (X && ncols > 0) {
    tstart(ctx, ST_BT2);
    // X must be 16B-aligned with even ldx for the DMMA tiles: the BT2 kernel uses scalar loads
    CK(bt2_run(L, p.bw, X, ldx, ncols, st), "bt2");
    tstop(ctx, ST_BT2);
  }
  CK(cudaStreamSynchronize(st), "sync");
  tcollect(ctx);
  kcollect(ctx);
  return SKEW_OK;
}

int skew_stage_tridiag_eig(skew_ctx ctx, int64_t n, const double* alpha, int64_t nev, double* lambda, double* Q,
                           int64_t ldq) {
  if (!ctx) return -1;
  if (n < 1) return -2;
  if (n > 1 && (!alpha || !is_device_ptr(alpha))) return -3;
  if (nev < 1 || nev > n) return -4;
  if (!lambda) return -5;
  if (Q && ldq < n) return -7;
  CK(cudaSetDevice(ctx->c.device), "set device");
  treset(ctx);
  Plan p;
  int64_t nev_plan = std::min<int64_t>(nev, n / 2);
  (void)nev_plan;
  Arena ar;
  ar.base = (char*)ctx->c.ws;
  ar.size = ctx->c.ws_bytes;
  TridWork tw;
  trid_reserve(ar, n, nev, Q != nullptr, tw, ctx->c.prm.reorth_w);
  double* lam_d = ar.take<double>(std::max<int64_t>(nev, 1));
  if (!ctx->c.ws || ar.off > ar.size || !lam_d) return SKEW_ERR_WORKSPACE;
  cudaStream_t st = ctx->c.stream;
  tstart(ctx, ST_TRID);
  int64_t nfail = 0;
  CK(trid_run(n, alpha, nev, lam_d, Q, ldq, tw, ctx->c.prm, &nfail, st, 0, nev, nullptr), "tridiagonal");
  tstop(ctx, ST_TRID);
  CK(cudaMemcpyAsync(lambda, lam_d, sizeof(double) * nev, cudaMemcpyDefault, st), "lambda");
  CK(cudaStreamSynchronize(st), "sync");
  tcollect(ctx);
  kcollect(ctx);
  ctx->c.last_nfail = nfail;
  return nfail ? SKEW_ERR_NOCONV : SKEW_OK;
}

}  // extern "C"
