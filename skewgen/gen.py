"""numpy implementation of the counter-based input generator (see __init__)."""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x):
    """SplitMix64 output function of (x + golden); x: uint64 array (wraps mod 2**64)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform_pm1(keys):
    """Map uint64 keys to doubles uniform on [-1, 1): 2*((z>>11)*2^-53) - 1 (exact)."""
    z = splitmix64(keys)
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u - 1.0


def _keys(seed, n, rows, cols):
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * GOLDEN
        return base + cols.astype(np.uint64) * np.uint64(n) + rows.astype(np.uint64)


def random_skew(n, seed):
    """Dense n x n skew-symmetric matrix (numpy, full storage, A = -A^T, zero diagonal)."""
    A = np.zeros((n, n), dtype=np.float64)
    if n < 2:
        return A
    # column-by-column blocks to bound memory
    for j0 in range(0, n, 1024):
        j1 = min(n, j0 + 1024)
        jj, ii = np.meshgrid(np.arange(j0, j1), np.arange(n), indexing="xy")
        vals = uniform_pm1(_keys(seed, n, ii, jj))
        mask = ii > jj
        blk = np.where(mask, vals, 0.0)
        A[:, j0:j1] = blk
    A = A - A.T
    return A


def random_skew_lower_colmajor(n, seed, lda=None):
    """Column-major strictly-lower storage (as a Fortran-ordered array) of random_skew(n, seed);
    the diagonal and upper triangle are zero (never read by either side)."""
    lda = n if lda is None else lda
    A = np.zeros((lda, n), dtype=np.float64, order="F")
    # column blocks written in place (same entries as random_skew's lower triangle,
    # without materialising the dense n x n matrix and its transpose)
    for j0 in range(0, n, 256):
        j1 = min(n, j0 + 256)
        jj, ii = np.meshgrid(np.arange(j0, j1), np.arange(n), indexing="xy")
        vals = uniform_pm1(_keys(seed, n, ii, jj))
        A[:n, j0:j1] = np.where(ii > jj, vals, 0.0)
    return A


def skew_toeplitz(n, alpha=1.0):
    """Skew tridiagonal with constant alpha: (k, k+1) = alpha, (k+1, k) = -alpha (Lemma 1 layout,
    PAPER.md:250-254). Closed form: eigenvalues +-2i*alpha*cos(k*pi/(n+1))."""
    A = np.zeros((n, n))
    for k in range(n - 1):
        A[k, k + 1] = alpha
        A[k + 1, k] = -alpha
    return A


def planted_skew(sigmas, seed, n_householders=None):
    """A = U blkdiag([[0, s_k], [-s_k, 0]]) U^T with U a product of seeded random Householder
    reflectors; the positive-half spectrum is exactly {s_k} (up to O(n eps ||A||) rounding).
    Odd n = 2*len(sigmas)+1 adds a zero eigenvalue when sigmas is padded by the caller."""
    sig = np.asarray(sigmas, dtype=np.float64)
    m = len(sig)
    n = 2 * m
    B = np.zeros((n, n))
    for k, s in enumerate(sig):
        B[2 * k, 2 * k + 1] = s
        B[2 * k + 1, 2 * k] = -s
    nh = n if n_householders is None else n_householders
    U = np.eye(n)
    for h in range(nh):
        keys = _keys(seed + 7919 * (h + 1), n, np.arange(n), np.zeros(n, dtype=np.int64))
        v = uniform_pm1(keys)
        v /= np.linalg.norm(v)
        U = U - 2.0 * np.outer(U @ v, v)
    A = U @ B @ U.T
    A = 0.5 * (A - A.T)
    return A


def bse_spd(n, seed):
    """BSE-form SPD M = G G^T / n + I with G_ij = uniform_pm1(key(i, j)) over all i, j
    (SURVEY §8(c) Generator; kappa(M) <~ 5). Symmetric by construction (exactly)."""
    jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="xy")
    G = uniform_pm1(_keys(seed, n, ii, jj))
    M = (G @ G.T) / n + np.eye(n)
    M = 0.5 * (M + M.T)
    return M


def J_matrix(n):
    """J = [[0, I], [-I, 0]]; n even."""
    assert n % 2 == 0
    m = n // 2
    J = np.zeros((n, n))
    J[:m, m:] = np.eye(m)
    J[m:, :m] = -np.eye(m)
    return J


def bse_AB(n, seed):
    """Definite BSE blocks (PAPER.md:488-499 structure, Eq. (9) definiteness): A Hermitian,
    B complex symmetric, n x n complex128.  X, Y, X', Y' are uniform_pm1 draws of four
    key streams; A = (X + X^H)/(4 sqrt n) + 4 I (with Re/Im from X, X'), B = (Y + Y^T)/(4 sqrt n).
    ||A - 4I||_2, ||B||_2 <~ 1, so Omega = [[A, B], [B-bar, A-bar]] >= 2 I > 0."""
    jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="xy")
    R = [uniform_pm1(_keys(seed * 4 + s, n, ii, jj)) for s in range(4)]
    X = R[0] + 1j * R[1]
    Y = R[2] + 1j * R[3]
    s = 4.0 * np.sqrt(n)
    A = (X + X.conj().T) / s + 4.0 * np.eye(n)
    B = (Y + Y.T) / s
    return A, B
