// internal.h -- host-side internal interfaces of the CUDA path (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <vector>
#include <string>

namespace sk {

// Bump allocator over the caller-provided workspace (the library never calls
// cudaMalloc in steady state; SURVEY §8(b) "Ownership").
struct Arena {
  char* base = nullptr;
  size_t size = 0, off = 0;
  bool measuring = false;   // size-query mode: only accumulate
  bool fail = false;        // some take() did not fit
  template <class T>
  T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
    if (measuring) { off += bytes; return nullptr; }
    if (off + bytes > size) { fail = true; return nullptr; }
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

struct VGroup;   // coll.cu: virtual-rank group

struct Params {
  int b = 64;            // band width (F2B panel width), fixed
  int bt2_k = 32;        // BT2 group width (sweeps per group), SKEWEIG_BT2_K
  int bt1_merge = 8;     // F2B panels merged per BT1 block reflector, SKEWEIG_BT1_MERGE
  int reorth_w = 32;     // inverse-iteration reorthogonalisation window, SKEWEIG_REORTH_W
  uint64_t seed = 1;     // inverse-iteration start-vector seed
};

// Per-stage device timings (ms), recorded with CUDA events on the ctx stream.
enum Stage { ST_F2B = 0, ST_B2T, ST_TRID, ST_BT2, ST_BT1, ST_OUT, ST_BSE, ST_COUNT };

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  Params prm;
  cudaEvent_t ev[ST_COUNT + 1] = {};
  double stage_ms[ST_COUNT] = {};
  int64_t last_nfail = 0;
  std::string last_error;
  // distributed
  int nranks = 1, rank = 0;
  void* nccl = nullptr;
  VGroup* vg = nullptr;   // virtual-rank group (not owned)
  // auxiliary stream: BT1 / BT2 preparation concurrent with the tridiagonal solve
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_la_cols = nullptr, ev_la_panel = nullptr;   // full->band look-ahead (distributed)
};

// Layout of the F2B reflector store: panels grouped by `merge` into block
// reflectors for BT1.  Group g (panels g*merge .. g*merge+merge-1) owns a
// ld_g x (merge*b) column-major block whose row 0 is global row r0(g*merge).
struct F2BLayout {
  int64_t n = 0;
  int b = 64, merge = 4;
  int64_t npanel = 0, ngroup = 0;
  std::vector<int64_t> goff;   // element offset of group g in the V store
  std::vector<int64_t> gld;    // leading dimension of group g (even)
  int64_t vstore_elems = 0;
  int64_t roff = 0;            // r0(j) = j*b + roff: b for full->band (V_j below the band),
                               // 1 for the one-step route (reflector of column c starts at row c+1)
  int64_t r0(int64_t j) const { return j * (int64_t)b + roff; }
  // onestep = false: panels j = 0 .. floor((n-2)/b)-1 of the full->band reduction (roff = b);
  // onestep = true: ceil((n-2)/b) panels of b one-step reflectors (columns 0 .. n-3, roff = 1)
  void init(int64_t n_, int b_, int merge_, bool onestep = false);
};


// ---------------------------------------------------------------- kernel accounting
// Every kernel launch of the library sits inside a KScope: it counts launches per
// kernel class and, when profiling is on, brackets them with CUDA events on the
// launching stream (skew_kernel_stats).
enum KClass {
  KC_PANEL = 0, KC_VT, KC_SYMM, KC_WCORR, KC_R2K, KC_BAND, KC_CHASE, KC_TRID_BISECT, KC_TRID_INV, KC_TRID_REORTH,
  KC_ASSEMBLE, KC_BT2_T, KC_BT2, KC_BT1_PREP, KC_BT1_Z, KC_BT1_UPD, KC_OUT, KC_BSE, KC_OS_MV, KC_OS_COL, KC_COLL, KC_COUNT
};
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<int, size_t>> rec;   // (class, index of start event; stop = +1)
  int64_t launches[KC_COUNT] = {};
  double ms[KC_COUNT] = {};
  void reset() { used = 0; rec.clear(); for (int i = 0; i < KC_COUNT; i++) { launches[i] = 0; ms[i] = 0.0; } }
  cudaEvent_t ev() {
    if (used == pool.size()) { cudaEvent_t e; cudaEventCreate(&e); pool.push_back(e); }
    return pool[used++];
  }
  void collect() {
    for (auto& r : rec) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, pool[r.second], pool[r.second + 1]) == cudaSuccess) ms[r.first] += t;
    }
    rec.clear();
    used = 0;
  }
};
extern thread_local Prof* g_prof;
struct KScope {
  int cls; cudaStream_t st; size_t idx = (size_t)-1;
  KScope(int c, cudaStream_t s, int nlaunch = 1) : cls(c), st(s) {
    if (!g_prof) return;
    g_prof->launches[c] += nlaunch;
    if (g_prof->on) {
      cudaEvent_t a = g_prof->ev();
      idx = g_prof->used - 1;
      g_prof->ev();
      cudaEventRecord(a, s);
    }
  }
  ~KScope() {
    if (g_prof && g_prof->on && idx != (size_t)-1) {
      cudaEventRecord(g_prof->pool[idx + 1], st);
      g_prof->rec.push_back({cls, idx});
    }
  }
};

// ---------------------------------------------------------------- per-stage work buffers
struct F2BWork {
  double* tau = nullptr;     // npanel * b
  double* T = nullptr;       // npanel * b * b
  double* part = nullptr;    // panel partials
  double* rowk = nullptr;
  double* gram = nullptr;
  double* U = nullptr;       // n x b
  double* X = nullptr;       // n x b
  double* P = nullptr;       // n x 2b
  double* Q = nullptr;       // n x 2b
  double* zpart = nullptr;   // V^T X partials
  double* Mb = nullptr;      // b x b
  double* cqr = nullptr;     // CholeskyQR panel scratch (3 b^2 + b + 2)
  unsigned* gbar = nullptr;  // panel grid barrier counter
  double* Ycol = nullptr;    // distributed skew-SYMM column-part pieces (P x n x b)
};

struct B2TLayout {
  int64_t n = 0; int b = 64, k2 = 32;
  int64_t nblk = 0, ngroups = 0;
  std::vector<int64_t> gofs;   // first group index of each sweep block
  int64_t ldab = 0;
  // BT2 group store: U only (the apply kernel rebuilds -V from the reflectors; half the
  // store, ~4 % slower BT2) for large n, else [U | -V] with one bulk copy per group
  bool uonly = false;
  void init(int64_t n_, int b_, int k2_);
};

struct B2TWork {
  double* AB = nullptr;
  int* progress = nullptr;
  double* qv = nullptr;
  double* qtau = nullptr;
  double* qT = nullptr;
  int64_t* gofs = nullptr;
  unsigned long long* prog = nullptr;   // BT2 wavefront: per CTA x producer warp progress
};

constexpr int kCountGrid = 131072;   // max points of the bisection start grid

struct TridWork {
  double* a2 = nullptr;        // alpha^2 (n)
  double* lamc = nullptr;      // candidates (n + padding)
  double* gtask = nullptr;     // Gershgorin bound per bisection task (n)
  int64_t* tsk = nullptr;      // 3 * n task arrays
  int* cgrid = nullptr;        // Sturm counts on the bisection start grid (kCountGrid + 1)
  double* scal = nullptr;      // device scalars: g, pivmin, #zeros in alpha, first ghost vector
  double* lamv = nullptr;      // per-vector perturbed lambda (nev)
  double* gblk = nullptr;      // per-vector block bound
  int64_t* vblk = nullptr;     // 2 * nev (s0, m)
  unsigned char* single = nullptr;   // per vector: 1 = isolated eigenvalue (twisted factorization)
  double* inv = nullptr;       // inverse iteration work
  unsigned char* inv_in = nullptr;
  int* nfail = nullptr;
  double* part = nullptr;      // gram partials
  double* H = nullptr;         // projection coefficients
  double* Rinv = nullptr;
  double* rpart = nullptr;     // fused reorthogonalisation: per-CTA Gram partials + reduced H
  int64_t* rblk = nullptr;     // fused reorthogonalisation: per 32-vector block (k0, p0, nb)
  unsigned* gbar = nullptr;    // fused reorthogonalisation: grid barrier counter
  int64_t batch = 0;
};

struct BT1Work {
  double* G = nullptr;     // ngroup x K x K  Gram matrices
  double* T = nullptr;     // ngroup x K x K  merged compact-WY T
  double* Y = nullptr;     // ngroup x K x b  T-merge scratch
  double* U = nullptr;     // n x K
  double* Z = nullptr;     // K x ncols
  int64_t* gmeta = nullptr;   // per group: V-store offset, ld, rows
};

// onestep.cu: the one-step (ELPA1-style) route, SURVEY 8(f) NEXT-4
struct OneStepWork {
  int64_t ldp = 0;
  double* PV = nullptr;     // panel [V | W]  (ldp x 2b)
  double* QW = nullptr;     // panel [W | -V]
  double* ypart = nullptr;  // skew mat-vec tile partials
  double* y = nullptr;
  double* pq = nullptr;
  double* npart = nullptr;
  double* tau = nullptr;    // n (per column)
  double* sub = nullptr;    // n (beta per column)
};

// coll.cu: collectives over NCCL or over virtual ranks (P contexts on one device)
VGroup* vgroup_new(int P);
void vgroup_free(VGroup* g);

// multi-GPU: 1D block-cyclic ownership of b-wide column blocks (owner of column c = (c / b) mod P)
struct Dist {
  int P = 1, rank = 0;
  void* comm = nullptr;   // ncclComm_t
  VGroup* vg = nullptr;   // virtual-rank group (instead of NCCL)
  // look-ahead (P > 1): the owner of panel j+1 factors it on `aux` (higher priority) while
  // its main stream finishes the rank-2k update of panel j on the other column blocks
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_cols = nullptr, ev_panel = nullptr;
};

// collectives (return 0 or a backend error code; see coll_error_string)
int coll_bcast(const Dist& d, void* buf, size_t bytes, int root, cudaStream_t st);
int coll_group_start(const Dist& d);
int coll_group_end(const Dist& d);
int coll_allreduce_sum(const Dist& d, double* buf, size_t count, cudaStream_t st);
int coll_allgather(const Dist& d, double* buf, size_t count, cudaStream_t st);
const char* coll_error_string(const Dist& d, int code);
// f2b.cu
void f2b_reserve(Arena& ar, const F2BLayout& L, int nsm, F2BWork& w, int P = 1);
// returns cudaErrorUnknown + sets *nccl_err on an NCCL failure
cudaError_t f2b_run(const F2BLayout& L, double* A, int64_t lda, double* vstore, const F2BWork& w, int nsm,
                    cudaStream_t st, const Dist& d, int* nccl_err);
// b2t.cu
void b2t_reserve(Arena& ar, const B2TLayout& L, bool vectors, B2TWork& w);
int b2t_chase_ctas(int64_t n, int b, int nsm);   // CTAs (= SMs) the chase occupies
cudaError_t b2t_run(const B2TLayout& L, B2TWork& w, double* alpha, int nsm, cudaStream_t st);
cudaError_t bt2_run(const B2TLayout& L, B2TWork& w, double* X, int64_t ldx, int64_t ncols, cudaStream_t st);
cudaError_t bt2_prep(const B2TLayout& L, B2TWork& w, cudaStream_t st);   // [U | V] of every group
cudaError_t bt2_apply(const B2TLayout& L, B2TWork& w, double* X, int64_t ldx, int64_t ncols, cudaStream_t st);
cudaError_t band_extract(const double* A, int64_t lda, int64_t n, int b, double* AB, int64_t ldab, cudaStream_t st,
                         int P = 1, int rank = 0);
cudaError_t band_copy(const double* ABin, int64_t ldin, int64_t n, int b, double* AB, int64_t ldab, cudaStream_t st);
// tridiag.cu
void trid_reserve(Arena& ar, int64_t n, int64_t nev, bool vectors, TridWork& w, int window);
// vectors of the global eigenpair range [k0, k1) (plus ghosts [vlo, k0)) go to Q columns 0..k1-vlo-1
cudaError_t trid_run(int64_t n, const double* alpha_d, int64_t nev, double* lam_out, double* Q, int64_t ldq,
                     TridWork& w, const Params& prm, int64_t* nfail_out, cudaStream_t st, int64_t k0, int64_t k1,
                     int64_t* vlo_out, const Dist* d = nullptr);
cudaError_t assemble_D(const double* Q, int64_t ldq, int64_t n, int64_t nev, double* X, int64_t ldx, cudaStream_t st);
// bt1.cu
void bt1_reserve(Arena& ar, const F2BLayout& L, int64_t ncols, BT1Work& w);
cudaError_t bt1_upload_meta(const F2BLayout& L, BT1Work& w, cudaStream_t st);
cudaError_t bt1_prep(const F2BLayout& L, const double* vstore, const double* Tpanel, BT1Work& w, cudaStream_t st);
cudaError_t bt1_gram(const F2BLayout& L, const double* vstore, BT1Work& w, cudaStream_t st);
// onestep.cu
void onestep_reserve(Arena& ar, const F2BLayout& L, OneStepWork& w);
cudaError_t onestep_run(const F2BLayout& L, double* A, int64_t lda, double* vstore, OneStepWork& w, double* alpha,
                        int nsm, cudaStream_t st);
cudaError_t onestep_bt_prep(const F2BLayout& L, const double* vstore, const double* tau, BT1Work& w,
                            cudaStream_t st);
cudaError_t bt1_apply(const F2BLayout& L, const double* vstore, const double* tau_all, const double* Tpanel, double* X,
                      int64_t ldx, int64_t ncols, BT1Work& w, cudaStream_t st);
cudaError_t bt1_run(const F2BLayout& L, const double* vstore, const double* tau_all, const double* Tpanel, double* X,
                    int64_t ldx, int64_t ncols, BT1Work& w, cudaStream_t st);
cudaError_t split_output(const double* X, int64_t ldx, int64_t n, int64_t nev, double* Zre, double* Zim, int64_t ldz,
                         cudaStream_t st);
// bse.cu
cudaError_t bse_front(double* M, int64_t ldm, int64_t n, double* W, int64_t ldw, double* S, int64_t lds,
                      double* scratch, int64_t* status_d, cudaStream_t st);
cudaError_t bse_build_M(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t n, double* M, int64_t ldm,
                        cudaStream_t st);
cudaError_t bse_backtransform(const double* L, int64_t ldl, int64_t n2, const double* Zre, const double* Zim,
                              int64_t ldz, int64_t nev, double* Yre, double* Yim, int64_t ldy, double* nrm2,
                              double* X, int64_t ldx, cudaStream_t st);
cudaError_t bse_lz(const double* L, int64_t ldl, int64_t n2, const double* Zre, const double* Zim, int64_t ldz,
                   int64_t nev, double* Yre, double* Yim, int64_t ldy, cudaStream_t st);
cudaError_t bse_apply_J(const double* Wre, const double* Wim, int64_t ldw, int64_t n2, int64_t nev, double* Yre,
                        double* Yim, int64_t ldy, cudaStream_t st);
cudaError_t nonfinite_lower(const double* A, int64_t lda, int64_t n, bool diag, int* flag_d, cudaStream_t st);

}  // namespace sk
