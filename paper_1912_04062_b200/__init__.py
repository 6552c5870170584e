"""paper_1912_04062_b200 -- B200-native (sm_100a) two-stage skew-symmetric eigensolver.

Thin Python binding over the C-ABI in ``include/skeweig.h`` (``libskeweig.so``, built
in-tree by ``paper_1912_04062_b200.build``).  This module only marshals arguments:
torch supplies device memory (workspace and outputs) and the CUDA stream; every step
of the solve runs in the library's CUDA kernels.  There is no CPU fallback: if the
library is missing or no GPU is present, calls raise.

    lam, Zre, Zim = skew_eig(A, nev)        # A: (n, n) float64 CUDA tensor, skew
    # A @ (Zre + 1j Zim)[:, k] = 1j * lam[k] * (Zre + 1j Zim)[:, k],  lam descending > 0

The strictly lower triangle of ``A`` (in the usual row/column sense) is what the solver
reads; the input tensor is not modified (it is copied to the
column-major layout the C-ABI takes).
"""
import ctypes
import os

__all__ = ["lib", "Context", "VirtualGroup", "skew_eig", "skew_eig_range", "skew_eig_host_range", "skew_eigvals", "skew_eig_onestep", "skew_eig_bse", "bse_hbs_eig", "skew_eig_host",
           "reduce_to_band", "band_to_tridiag", "tridiag_eig", "expand_half_spectrum", "SkewError"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "libskeweig.so")
_lib = None

SKEW_WS_VECTORS = 1
SKEW_WS_HOST_STAGING = 2
SKEW_WS_BSE = 4
SKEW_WS_BSE_BACKTRANSFORM = 8
SKEW_BSE_HAMILTONIAN_Y = 1
SKEW_WS_ONESTEP = 16
SKEW_ERR_NOCONV = 1
SKEW_ERR_NOT_DEFINITE = 4

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.c_void_p

EXPORTS = {
    "skew_ctx_create": ([ctypes.POINTER(_vp), ctypes.c_int, _vp], ctypes.c_int),
    "skew_ctx_destroy": ([_vp], ctypes.c_int),
    "skew_get_unique_id": ([ctypes.c_char_p], ctypes.c_int),
    "skew_ctx_create_dist": ([ctypes.POINTER(_vp), ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_char_p],
                             ctypes.c_int),
    "skew_tile_schedule": ([_i64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, _i64], _i64),
    "skew_vgroup_create": ([ctypes.c_int, ctypes.POINTER(_vp)], ctypes.c_int),
    "skew_vgroup_destroy": ([_vp], ctypes.c_int),
    "skew_ctx_create_virtual": ([ctypes.POINTER(_vp), ctypes.c_int, _vp, _vp, ctypes.c_int, ctypes.c_int],
                                ctypes.c_int),
    "skew_workspace_size": ([_vp, _i64, _i64, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "skew_set_workspace": ([_vp, _vp, ctypes.c_size_t], ctypes.c_int),
    "skew_eig": ([_vp, _i64, _dp, _i64, _i64, _dp, _dp, _dp, _i64], ctypes.c_int),
    "skew_eigvals": ([_vp, _i64, _dp, _i64, _i64, _dp], ctypes.c_int),
    "skew_eig_onestep": ([_vp, _i64, _dp, _i64, _i64, _dp, _dp, _dp, _i64], ctypes.c_int),
    "skew_eig_range": ([_vp, _i64, _dp, _i64, _i64, _i64, _i64, _dp, _dp, _dp, _i64], ctypes.c_int),
    "skew_eig_bse": ([_vp, _i64, _dp, _i64, _i64, ctypes.c_int, _dp, _dp, _dp, _i64, ctypes.POINTER(_i64)],
                     ctypes.c_int),
    "skew_bse_build_M": ([_vp, _i64, _dp, _i64, _dp, _i64, _dp, _i64], ctypes.c_int),
    "skew_bse_backtransform": ([_vp, _i64, _dp, _i64, _i64, _dp, _dp, _i64, _dp, _i64], ctypes.c_int),
    "skew_stage_times": ([_vp, ctypes.POINTER(ctypes.c_double), ctypes.c_int], ctypes.c_int),
    "skew_last_nfail": ([_vp], _i64),
    "skew_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "skew_last_error": ([_vp], ctypes.c_char_p),
    "skew_stage_reduce_to_band": ([_vp, _i64, _dp, _i64, _dp, _i64, _dp, _dp, ctypes.POINTER(_i64)], ctypes.c_int),
    "skew_stage_band_to_tridiag": ([_vp, _i64, ctypes.c_int, _dp, _i64, _dp, _dp, _i64, _i64], ctypes.c_int),
    "skew_stage_tridiag_eig": ([_vp, _i64, _dp, _i64, _dp, _dp, _i64], ctypes.c_int),
    "skew_set_profiling": ([_vp, ctypes.c_int], ctypes.c_int),
    "skew_kernel_stats": ([_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64), ctypes.c_int], ctypes.c_int),
    "skew_kernel_class_name": ([ctypes.c_int], ctypes.c_char_p),
}
KERNEL_CLASSES = 21

STAGES = ["f2b", "b2t", "tridiag", "bt2", "bt1", "output", "bse"]


class SkewError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"skeweig status {status}: {msg}")
        self.status = status


def lib():
    """Load libskeweig.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIBPATH):
            raise RuntimeError(f"{_LIBPATH} missing: run `python -m paper_1912_04062_b200.build` "
                               "(the CUDA path has no CPU fallback)")
        L = ctypes.CDLL(_LIBPATH)
        for name, (args, res) in EXPORTS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1912_04062_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
    return torch


class VirtualGroup:
    """A group of P virtual ranks on one device (skew_vgroup_create): Context(virtual=(g, r))
    makes rank r's context.  Test harness for the distributed path on a single GPU; each
    rank's solve runs in its own host thread (the collectives meet at host barriers)."""

    def __init__(self, nranks):
        h = _vp()
        rc = lib().skew_vgroup_create(nranks, ctypes.byref(h))
        if rc != 0:
            raise SkewError(rc, "skew_vgroup_create failed")
        self.h, self.nranks = h, nranks

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().skew_vgroup_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Context:
    """One C-ABI context per (device, stream) plus a torch-allocated device workspace."""

    def __init__(self, device=None, stream=None, group=None, distributed=False, virtual=None):
        """distributed=True: a collective context over torch.distributed `group` (NCCL inside the
        library; the unique id is exchanged with broadcast_object_list).  virtual=(VirtualGroup,
        rank): rank `rank` of a virtual-rank group on this device."""
        torch = _torch()
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else
                                   torch.device(device).index or 0)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = _vp()
        if virtual is not None:
            vg, rank = virtual
            self._vg = vg   # the group must outlive the context
            rc = lib().skew_ctx_create_virtual(ctypes.byref(h), self.device.index, _vp(self.stream.cuda_stream), vg.h,
                                               vg.nranks, rank)
            self.rank, self.world = rank, vg.nranks
        elif distributed:
            import torch.distributed as dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
            buf = ctypes.create_string_buffer(128)
            if rank == 0:
                rc = lib().skew_get_unique_id(buf)
                if rc != 0:
                    raise SkewError(rc, "skew_get_unique_id failed")
            obj = [bytes(buf.raw) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            idb = ctypes.create_string_buffer(obj[0], 128)
            rc = lib().skew_ctx_create_dist(ctypes.byref(h), self.device.index, _vp(self.stream.cuda_stream), world,
                                            rank, idb)
            self.rank, self.world = rank, world
        else:
            rc = lib().skew_ctx_create(ctypes.byref(h), self.device.index, _vp(self.stream.cuda_stream))
            self.rank, self.world = 0, 1
        if rc != 0:
            raise SkewError(rc, "skew context creation failed")
        self.h = h
        self.ws = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().skew_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def workspace_bytes(self, n, nev, flags):
        sz = ctypes.c_size_t(0)
        rc = lib().skew_workspace_size(self.h, n, nev, flags, ctypes.byref(sz))
        self._check(rc)
        return sz.value

    def ensure_workspace(self, n, nev, flags):
        need = self.workspace_bytes(n, nev, flags)
        if self.ws is None or self.ws.numel() < need:
            self.ws = None
            self.ws = self.torch.empty(need, dtype=self.torch.uint8, device=self.device)
            self._check(lib().skew_set_workspace(self.h, _vp(self.ws.data_ptr()), need))
        return need

    def stage_times(self):
        arr = (ctypes.c_double * 7)()
        lib().skew_stage_times(self.h, arr, 7)
        return dict(zip(STAGES, list(arr)))

    def set_profiling(self, on=True):
        self._check(lib().skew_set_profiling(self.h, 1 if on else 0))

    def kernel_stats(self):
        """{class: (ms, launches)} for the last call (ms only when profiling is on)."""
        ms = (ctypes.c_double * KERNEL_CLASSES)()
        la = (_i64 * KERNEL_CLASSES)()
        lib().skew_kernel_stats(self.h, ms, la, KERNEL_CLASSES)
        return {lib().skew_kernel_class_name(i).decode(): (ms[i], la[i]) for i in range(KERNEL_CLASSES)}

    def last_error(self):
        return lib().skew_last_error(self.h).decode()

    def _check(self, rc, allow=()):
        if rc != 0 and rc not in allow:
            msg = lib().skew_status_string(rc).decode()
            err = self.last_error()
            raise SkewError(rc, msg + (f" ({err})" if err else ""))
        return rc


_default = {}


def _ctx(ctx):
    if ctx is not None:
        return ctx
    torch = _torch()
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
    if key not in _default:
        _default[key] = Context()
    return _default[key]


def _colmajor(torch, A):
    """Column-major COPY (the transposed view of a fresh contiguous tensor) of a 2-D tensor.
    Always a copy: for an input that is already column-major, A.t().contiguous() would return
    A's own storage and the solver (which destroys its input) would overwrite the caller's A
    although overwrite_a=False."""
    out = torch.empty((A.shape[1], A.shape[0]), dtype=A.dtype, device=A.device).t()
    out.copy_(A)
    return out


def _new_colmajor(torch, n, m, device):
    return torch.empty((m, n), dtype=torch.float64, device=device).t()


def skew_eig(A, nev=None, ctx=None, overwrite_a=False):
    """Eigenpairs of the real skew-symmetric A (n x n, float64, CUDA): the nev largest
    lambda_k > 0 (descending) with A z_k = i lambda_k z_k, z_k = Zre[:, k] + i Zim[:, k].
    Returns (lam, Zre, Zim).  nev defaults to n // 2 (the whole positive half)."""
    torch = _torch()
    c = _ctx(ctx)
    n = A.shape[0]
    nev = n // 2 if nev is None else nev
    Ac = A if (overwrite_a and A.stride(0) == 1) else _colmajor(torch, A.to(device=c.device, dtype=torch.float64))
    c.ensure_workspace(n, nev, SKEW_WS_VECTORS)
    lam = torch.empty(max(nev, 1), dtype=torch.float64, device=c.device)
    Zre = _new_colmajor(torch, n, max(nev, 1), c.device)
    Zim = _new_colmajor(torch, n, max(nev, 1), c.device)
    rc = lib().skew_eig(c.h, n, _dp(Ac.data_ptr()), Ac.stride(1), nev, _dp(lam.data_ptr()), _dp(Zre.data_ptr()),
                        _dp(Zim.data_ptr()), Zre.stride(1))
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    return lam[:nev], Zre[:, :nev], Zim[:, :nev]


def skew_eig_range(A, nev, k0, k1, ctx=None, overwrite_a=False):
    """All nev eigenvalues and the eigenvectors of the index range [k0, k1) (multi-GPU
    per-rank call).  Returns (lam (nev,), Zre (n, k1-k0), Zim (n, k1-k0))."""
    torch = _torch()
    c = _ctx(ctx)
    n = A.shape[0]
    Ac = A if (overwrite_a and A.stride(0) == 1) else _colmajor(torch, A.to(device=c.device, dtype=torch.float64))
    c.ensure_workspace(n, nev, SKEW_WS_VECTORS)
    lam = torch.empty(max(nev, 1), dtype=torch.float64, device=c.device)
    m = max(k1 - k0, 1)
    Zre = _new_colmajor(torch, n, m, c.device)
    Zim = _new_colmajor(torch, n, m, c.device)
    rc = lib().skew_eig_range(c.h, n, _dp(Ac.data_ptr()), Ac.stride(1), nev, k0, k1, _dp(lam.data_ptr()),
                              _dp(Zre.data_ptr()), _dp(Zim.data_ptr()), Zre.stride(1))
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    return lam[:nev], Zre[:, :k1 - k0], Zim[:, :k1 - k0]


def skew_eig_host_range(A_host, nev, k0, k1, lam_host, Zre_host, Zim_host, ctx=None):
    """skew_eig_range with HOST buffers (column-major, ld = n): end-to-end entry."""
    c = _ctx(ctx)
    n = A_host.shape[0]
    c.ensure_workspace(n, nev, SKEW_WS_VECTORS | SKEW_WS_HOST_STAGING)

    def ptr(x):
        return x.ctypes.data if hasattr(x, "ctypes") else x.data_ptr()
    rc = lib().skew_eig_range(c.h, n, _dp(ptr(A_host)), n, nev, k0, k1, _dp(ptr(lam_host)), _dp(ptr(Zre_host)),
                              _dp(ptr(Zim_host)), n)
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    return rc


def skew_eigvals(A, nev=None, ctx=None, overwrite_a=False):
    """The nev largest lambda_k (descending) of the skew A (eigenvalues only)."""
    torch = _torch()
    c = _ctx(ctx)
    n = A.shape[0]
    nev = n // 2 if nev is None else nev
    Ac = A if (overwrite_a and A.stride(0) == 1) else _colmajor(torch, A.to(device=c.device, dtype=torch.float64))
    c.ensure_workspace(n, nev, 0)
    lam = torch.empty(max(nev, 1), dtype=torch.float64, device=c.device)
    rc = lib().skew_eigvals(c.h, n, _dp(Ac.data_ptr()), Ac.stride(1), nev, _dp(lam.data_ptr()))
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    return lam[:nev]


def skew_eig_onestep(A, nev=None, ctx=None, want_vectors=True, overwrite_a=False):
    """The one-step route: A -> tridiagonal directly
    (one reflector per column), same tridiagonal solve, one back-transformation.  Returns
    (lam, Zre, Zim) like skew_eig, or lam when want_vectors is False."""
    torch = _torch()
    c = _ctx(ctx)
    n = A.shape[0]
    nev = n // 2 if nev is None else nev
    Ac = A if (overwrite_a and A.stride(0) == 1) else _colmajor(torch, A.to(device=c.device, dtype=torch.float64))
    c.ensure_workspace(n, nev, SKEW_WS_ONESTEP | (SKEW_WS_VECTORS if want_vectors else 0))
    lam = torch.empty(max(nev, 1), dtype=torch.float64, device=c.device)
    Zre = _new_colmajor(torch, n, max(nev, 1), c.device) if want_vectors else None
    Zim = _new_colmajor(torch, n, max(nev, 1), c.device) if want_vectors else None
    rc = lib().skew_eig_onestep(c.h, n, _dp(Ac.data_ptr()), Ac.stride(1), nev, _dp(lam.data_ptr()),
                                _dp(Zre.data_ptr()) if want_vectors else None,
                                _dp(Zim.data_ptr()) if want_vectors else None, n)
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    if want_vectors:
        return lam[:nev], Zre[:, :nev], Zim[:, :nev]
    return lam[:nev]


def skew_eig_bse(M, nev=None, ctx=None, want_vectors=True, overwrite_m=False, hamiltonian_y=False):
    """BSE form: SPD M (n x n, n even) -> Cholesky M = L L^T ->
    W = L^T J L -> (lam, Zre, Zim) of the skew W (as skew_eig).  hamiltonian_y=True
    (SKEW_BSE_HAMILTONIAN_Y) returns y = J L z instead of z (H y = -i lam y for H = -J M,
    unnormalised).  Raises SkewError with .status == 4 and .pivot when M is not
    numerically definite."""
    torch = _torch()
    c = _ctx(ctx)
    n = M.shape[0]
    nev = n // 2 if nev is None else nev
    Mc = M if (overwrite_m and M.stride(0) == 1) else _colmajor(torch, M.to(device=c.device, dtype=torch.float64))
    c.ensure_workspace(n, nev, (SKEW_WS_VECTORS if want_vectors else 0) | SKEW_WS_BSE)
    lam = torch.empty(max(nev, 1), dtype=torch.float64, device=c.device)
    Zre = _new_colmajor(torch, n, max(nev, 1), c.device) if want_vectors else None
    Zim = _new_colmajor(torch, n, max(nev, 1), c.device) if want_vectors else None
    piv = _i64(0)
    rc = lib().skew_eig_bse(c.h, n, _dp(Mc.data_ptr()), Mc.stride(1), nev,
                            SKEW_BSE_HAMILTONIAN_Y if hamiltonian_y else 0, _dp(lam.data_ptr()),
                            _dp(Zre.data_ptr()) if want_vectors else None,
                            _dp(Zim.data_ptr()) if want_vectors else None, n, ctypes.byref(piv))
    if rc == SKEW_ERR_NOT_DEFINITE:
        e = SkewError(rc, f"M not positive definite (pivot {piv.value})")
        e.pivot = piv.value
        raise e
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    if want_vectors:
        return lam[:nev], Zre[:, :nev], Zim[:, :nev]
    return lam[:nev]


def bse_hbs_eig(A, B, nev=None, ctx=None):
    """Full BSE pipeline for H_BS = [[A, B], [-B-bar, -A-bar]] (Eq. 9),
    A = A^H, B = B^T (n x n complex128): skew_bse_build_M (Eq. 10) -> skew_eig_bse
    (M = L L^T, eigenpairs of L^T J L; M is overwritten by L) -> skew_bse_backtransform
    (x = Q J L z, Theorem 1, normalised to unit 2-norm).  Returns (lam (nev,)
    descending positive, X (2n x nev complex128)) with H_BS x_k = lam_k x_k.  nev defaults
    to n (the whole positive half)."""
    torch = _torch()
    c = _ctx(ctx)
    n = A.shape[0]
    nev = n if nev is None else nev
    Ac = A.to(device=c.device, dtype=torch.complex128).t().contiguous().t()   # column-major
    Bc = B.to(device=c.device, dtype=torch.complex128).t().contiguous().t()
    M = _new_colmajor(torch, 2 * n, 2 * n, c.device)
    c._check(lib().skew_bse_build_M(c.h, n, _dp(Ac.data_ptr()), Ac.stride(1), _dp(Bc.data_ptr()), Bc.stride(1),
                                    _dp(M.data_ptr()), M.stride(1)))
    lam, Zre, Zim = skew_eig_bse(M, nev, ctx=c, overwrite_m=True)   # M now holds L
    X = torch.empty((nev, 2 * n), dtype=torch.complex128, device=c.device).t()
    c.ensure_workspace(2 * n, nev, SKEW_WS_BSE_BACKTRANSFORM)
    c._check(lib().skew_bse_backtransform(c.h, 2 * n, _dp(M.data_ptr()), M.stride(1), nev, _dp(Zre.data_ptr()),
                                          _dp(Zim.data_ptr()), Zre.stride(1), _dp(X.data_ptr()), X.stride(1)))
    return lam, X


def skew_eig_host(A_host, nev, lam_host, Zre_host, Zim_host, ctx=None):
    """End-to-end entry with HOST buffers (numpy or pinned torch CPU tensors, column-major
    n x n A, n x nev Zre/Zim with ld = n): the C-ABI stages the host arrays through the
    device workspace, so the host<->device copies are part of the call."""
    c = _ctx(ctx)
    n = A_host.shape[0]
    c.ensure_workspace(n, nev, SKEW_WS_VECTORS | SKEW_WS_HOST_STAGING)

    def ptr(x):
        return x.ctypes.data if hasattr(x, "ctypes") else x.data_ptr()
    rc = lib().skew_eig(c.h, n, _dp(ptr(A_host)), n, nev, _dp(ptr(lam_host)), _dp(ptr(Zre_host)),
                        _dp(ptr(Zim_host)), n)
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    return rc


def reduce_to_band(A, ctx=None, want_reflectors=True):
    """Stage entry (full -> band) on a column-major copy of A.
    Returns (Ab, V, T, tau, npanel): Ab the column-major work array whose band
    Ab[c+1..c+b, c] is the reduced band; V (n x npanel*b) with V_j at rows (j+1)b..;
    T (b x npanel*b); tau."""
    torch = _torch()
    c = _ctx(ctx)
    n = A.shape[0]
    Ac = _colmajor(torch, A.to(device=c.device, dtype=torch.float64))
    c.ensure_workspace(n, 0, 0)
    b = band_width()
    npmax = max(0, (n - 2) // b) if n >= 2 + b else 0
    V = torch.zeros((max(npmax * b, 1), n), dtype=torch.float64, device=c.device).t() if want_reflectors else None
    T = torch.zeros((max(npmax * b, 1), b), dtype=torch.float64, device=c.device).t() if want_reflectors else None
    tau = torch.zeros(max(npmax * b, 1), dtype=torch.float64, device=c.device) if want_reflectors else None
    npn = _i64(0)
    rc = lib().skew_stage_reduce_to_band(c.h, n, _dp(Ac.data_ptr()), Ac.stride(1),
                                         _dp(V.data_ptr()) if want_reflectors else None, n,
                                         _dp(T.data_ptr()) if want_reflectors else None,
                                         _dp(tau.data_ptr()) if want_reflectors else None, ctypes.byref(npn))
    c._check(rc)
    return Ac, V, T, tau, npn.value


def band_width():
    """The library's internal band width b (fixed at 64, include/skeweig.h)."""
    return 64


def band_to_tridiag(AB, b, X=None, ctx=None):
    """Stage entry (bulge chasing) on a lower-band-storage tensor AB
    ((ldab, n) column-major view: AB[d, c] = B[c+d, c]).  Returns alpha (n-1); when X
    (n x m column-major) is given it is overwritten with Q2 X."""
    torch = _torch()
    c = _ctx(ctx)
    n = AB.shape[1]
    c.ensure_workspace(n, 0, SKEW_WS_VECTORS if X is not None else 0)
    alpha = torch.zeros(max(n - 1, 1), dtype=torch.float64, device=c.device)
    rc = lib().skew_stage_band_to_tridiag(c.h, n, b, _dp(AB.data_ptr()), AB.stride(1), _dp(alpha.data_ptr()),
                                          _dp(X.data_ptr()) if X is not None else None,
                                          X.stride(1) if X is not None else n, X.shape[1] if X is not None else 0)
    c._check(rc)
    return alpha[: max(n - 1, 0)]


def tridiag_eig(alpha, nev, ctx=None, want_vectors=True):
    """Stage entry (Lemma 1 + bisection + inverse iteration): top-nev eigenpairs of
    tridiag(alpha, 0, alpha).  Returns (lam, Q) (Q None if not want_vectors)."""
    torch = _torch()
    c = _ctx(ctx)
    n = alpha.shape[0] + 1
    c.ensure_workspace(n, min(nev, n // 2), SKEW_WS_VECTORS)
    a = alpha.to(device=c.device, dtype=torch.float64).contiguous()
    if a.numel() == 0:
        a = torch.zeros(1, dtype=torch.float64, device=c.device)
    lam = torch.empty(nev, dtype=torch.float64, device=c.device)
    Q = _new_colmajor(torch, n, nev, c.device) if want_vectors else None
    rc = lib().skew_stage_tridiag_eig(c.h, n, _dp(a.data_ptr()), nev, _dp(lam.data_ptr()),
                                      _dp(Q.data_ptr()) if want_vectors else None, n)
    c._check(rc, allow=(SKEW_ERR_NOCONV,))
    return lam, Q


def expand_half_spectrum(lam, Zre, Zim):
    """Append the conjugate half: eigenvalues -lam with vectors conj(z)."""
    import torch
    return (torch.cat([lam, -lam]), torch.cat([Zre, Zre], dim=1), torch.cat([Zim, -Zim], dim=1))
