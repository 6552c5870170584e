"""CPU oracle for the skew-symmetric eigensolver (arXiv 1912.04062) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_1912_04062_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C + OpenMP, no BLAS); this
module only compiles it (gcc) and marshals numpy arrays through ctypes.
Each wrapper names the ``oracle.c`` function and the PAPER.md passage it follows.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liborcskew.so")
_lib = None

_c_i64 = ctypes.c_int64
_c_dp = ctypes.POINTER(ctypes.c_double)


def build(force=False):
    """Compile oracle.c -> liborcskew.so (gcc -O3 -fopenmp, portable x86-64-v3)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared", "-std=c11",
           "-D_POSIX_C_SOURCE=199309L", "-o", _LIB + ".tmp", _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_householder.argtypes = [_c_i64, _c_dp, _c_dp, _c_dp, _c_dp]
        L.orc_skew_matvec.argtypes = [_c_i64, _c_dp, _c_i64, _c_dp, _c_dp]
        L.orc_skew_rank2.argtypes = [_c_i64, _c_dp, _c_i64, _c_dp, _c_dp]
        L.orc_tridiagonalize.argtypes = [_c_i64, _c_dp, _c_i64, _c_dp, _c_dp]
        L.orc_sturm_count.argtypes = [_c_i64, _c_dp, ctypes.c_double, ctypes.c_double]
        L.orc_sturm_count.restype = _c_i64
        L.orc_bisect.argtypes = [_c_i64, _c_dp, _c_i64, _c_i64, _c_dp]
        L.orc_gershgorin.argtypes = [_c_i64, _c_dp]
        L.orc_gershgorin.restype = ctypes.c_double
        L.orc_tridiag_eig.argtypes = [_c_i64, _c_dp, _c_i64, _c_dp, _c_dp, _c_i64, ctypes.c_uint64,
                                      _c_i64, ctypes.c_int]
        L.orc_tridiag_eig.restype = _c_i64
        L.orc_apply_D.argtypes = [_c_i64, _c_i64, _c_dp, _c_i64, _c_dp, _c_dp, _c_i64]
        L.orc_backtransform.argtypes = [_c_i64, _c_dp, _c_i64, _c_dp, _c_i64, _c_dp, _c_i64]
        L.orc_skew_eig.argtypes = [_c_i64, _c_dp, _c_i64, _c_i64, _c_dp, _c_dp, _c_dp, _c_i64, ctypes.c_int,
                                   ctypes.c_uint64, _c_dp]
        L.orc_skew_eig.restype = _c_i64
        L.orc_cholesky.argtypes = [_c_i64, _c_dp, _c_i64]
        L.orc_cholesky.restype = _c_i64
        L.orc_form_W.argtypes = [_c_i64, _c_dp, _c_i64, _c_dp, _c_i64]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        L.orc_set_num_threads.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_c_dp)


def _f(a):
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def num_threads():
    return lib().orc_num_threads()


def set_num_threads(nt):
    """Threads of the oracle's OpenMP loops (measurement harness only; no arithmetic)."""
    lib().orc_set_num_threads(int(nt))


def householder(x):
    """orc_householder (dlarfg convention) -> (v, tau, beta)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    v = np.zeros_like(x)
    tau = np.zeros(1)
    beta = np.zeros(1)
    lib().orc_householder(len(x), _p(x), _p(v), _p(tau), _p(beta))
    return v, float(tau[0]), float(beta[0])


def skew_matvec(A, x):
    """orc_skew_matvec: y = A x from the strictly lower triangle."""
    A = _f(A)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(A.shape[0])
    lib().orc_skew_matvec(A.shape[0], _p(A), A.shape[0], _p(x), _p(y))
    return y


def skew_rank2(A, u, v):
    """orc_skew_rank2: lower(A) <- lower(A - v u^T + u v^T); returns a copy."""
    A = _f(A).copy(order="F")
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    lib().orc_skew_rank2(A.shape[0], _p(A), A.shape[0], _p(u), _p(v))
    return A


def tridiagonalize(A):
    """orc_tridiagonalize (one-step Householder).
    Returns (alpha, tau, R) with R the work array holding the reflectors."""
    n = A.shape[0]
    R = np.asfortranarray(np.tril(np.asarray(A, dtype=np.float64), -1))
    alpha = np.zeros(max(n - 1, 1))
    tau = np.zeros(max(n - 1, 1))
    lib().orc_tridiagonalize(n, _p(R), n, _p(alpha), _p(tau))
    return alpha[:max(n - 1, 0)], tau[:max(n - 1, 0)], R


def sturm_count(alpha, sigma):
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    n = len(alpha) + 1
    pivmin = np.finfo(float).tiny * max(1.0, float(np.max(alpha ** 2)) if len(alpha) else 1.0)
    return int(lib().orc_sturm_count(n, _p(alpha), float(sigma), pivmin))


def bisect(alpha, il, iu):
    """orc_bisect: ascending eigenvalues il..iu (0-based) of tridiag(alpha, 0, alpha)."""
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    n = len(alpha) + 1
    lam = np.zeros(iu - il + 1)
    lib().orc_bisect(n, _p(alpha), il, iu, _p(lam))
    return lam


def tridiag_eig(alpha, nev, seed=1, window=32, want_vectors=True):
    """orc_tridiag_eig: top-nev eigenpairs (descending) of tridiag(alpha, 0, alpha).
    Returns (lam, Q, nfail)."""
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    n = len(alpha) + 1
    lam = np.zeros(max(nev, 1))
    Q = np.zeros((n, max(nev, 1)), order="F")
    a = alpha if len(alpha) else np.zeros(1)
    nfail = lib().orc_tridiag_eig(n, _p(a), nev, _p(lam), _p(Q), n, seed, window, 1 if want_vectors else 0)
    return lam[:nev], Q[:, :nev], int(nfail)


def apply_D(Q):
    """orc_apply_D: (Re, Im) planes of D Q, D = diag(i^k)."""
    Q = _f(Q)
    n, k = Q.shape
    Xre = np.zeros((n, k), order="F")
    Xim = np.zeros((n, k), order="F")
    lib().orc_apply_D(n, k, _p(Q), n, _p(Xre), _p(Xim), n)
    return Xre, Xim


def backtransform(R, tau, X):
    """orc_backtransform: X <- Q_trd X with the reflectors of tridiagonalize()."""
    X = _f(X).copy(order="F")
    n = R.shape[0]
    t = np.ascontiguousarray(tau if len(tau) else np.zeros(1), dtype=np.float64)
    lib().orc_backtransform(n, _p(R), n, _p(t), X.shape[1], _p(X), n)
    return X


def skew_eig(A, nev=None, want_vectors=True, seed=1, times=None):
    """orc_skew_eig: Algorithm 1, half spectrum.
    A: dense skew (only the strictly lower triangle is read).
    Returns (lam desc, Zre, Zim, status)."""
    A = _f(A)
    n = A.shape[0]
    nev = n // 2 if nev is None else nev
    lam = np.zeros(max(nev, 1))
    Zre = np.zeros((n, max(nev, 1)), order="F")
    Zim = np.zeros((n, max(nev, 1)), order="F")
    tt = np.zeros(4)
    st = lib().orc_skew_eig(n, _p(A), n, nev, _p(lam), _p(Zre), _p(Zim), n,
                            1 if want_vectors else 0, seed, _p(tt))
    if times is not None:
        times.update(dict(tridiagonalize=tt[0], bisect=tt[1], inverse_iteration=tt[2], backtransform=tt[3]))
    return lam[:nev], Zre[:, :nev], Zim[:, :nev], int(st)


def cholesky(M):
    """orc_cholesky (dpotf2 order). Returns (L lower, pivot) pivot=0 ok else 1-based."""
    L = _f(M).copy(order="F")
    piv = lib().orc_cholesky(L.shape[0], _p(L), L.shape[0])
    return np.tril(L), int(piv)


def form_W(L):
    """orc_form_W: strictly-lower storage of W = L^T J L."""
    L = _f(L)
    n = L.shape[0]
    W = np.zeros((n, n), order="F")
    lib().orc_form_W(n, _p(L), n, _p(W), n)
    return W


def bse_eig(M, nev=None, want_vectors=True, seed=1):
    """BSE steps 2-3: M = L L^T, W = L^T J L, eigenpairs of W.
    Returns (lam, Zre, Zim, status, pivot, L)."""
    L, piv = cholesky(M)
    if piv:
        return None, None, None, 4, piv, None
    W = form_W(L)
    lam, Zre, Zim, st = skew_eig(W, nev, want_vectors, seed)
    return lam, Zre, Zim, st, 0, L


# ---------------------------------------------------------------------------------------
# Full BSE H_BS pipeline, plain numpy on top of bse_eig above.
# ---------------------------------------------------------------------------------------
def bse_build_M(A, B):
    """Eq. (10): M = JH = [[Re(A+B), Im(A-B)], [-Im(A+B), Re(A-B)]],
    2n x 2n real, from A = A^H and B = B^T (n x n complex)."""
    A = np.asarray(A, dtype=np.complex128)
    B = np.asarray(B, dtype=np.complex128)
    P, Mn = A + B, A - B
    return np.block([[P.real, Mn.imag], [-P.imag, Mn.real]])


def bse_Q(n):
    """Theorem 1: Q = 1/sqrt(2) [[I, -iI], [I, iI]] (2n x 2n, unitary)."""
    I = np.eye(n)
    return np.block([[I, -1j * I], [I, 1j * I]]) / np.sqrt(2.0)


def bse_backtransform(L, Zre, Zim):
    """Step 4: x = Q J L z.  With L^T J L z = i lam z and M = L L^T,
    y = J L z satisfies H y = -J M y ... = -i lam y, so i H y = lam y and, by Theorem 1
    (Q^H H_BS Q = i H), H_BS (Q y) = lam (Q y).  Returns X (2n x nev complex)."""
    n2 = L.shape[0]
    Z = np.asarray(Zre) + 1j * np.asarray(Zim)
    J = np.block([[np.zeros((n2 // 2, n2 // 2)), np.eye(n2 // 2)],
                  [-np.eye(n2 // 2), np.zeros((n2 // 2, n2 // 2))]])
    return bse_Q(n2 // 2) @ (J @ (np.tril(L) @ Z))


def bse_hbs_eig(A, B, nev=None, seed=1):
    """The four steps of PAPER.md:596-606 for H_BS = [[A, B], [-B-bar, -A-bar]] (Eq. 9):
    M (Eq. 10) -> M = L L^T -> eigenpairs of L^T J L -> x = Q J L z, each x normalised to
    unit 2-norm ("normalizes x_k to unit 2-norm"; phase free, reading R7).
    Returns (lam (nev, descending positive), X (2n x nev complex), status, pivot)."""
    M = bse_build_M(A, B)
    n2 = M.shape[0]
    nev = n2 // 2 if nev is None else nev
    lam, Zre, Zim, st, piv, L = bse_eig(M, nev, True, seed)
    if piv:
        return None, None, st, piv
    X = bse_backtransform(L, Zre, Zim)
    return lam, X / np.linalg.norm(X, axis=0), st, 0
