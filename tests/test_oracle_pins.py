"""Pins for the CPU oracle (oracle/oracle.c): each check is fixed by the paper, SPEC.md's
worked examples, closed forms, invariants, independent library routines or brute force --
never by re-typing the oracle's own formula and never by the CUDA path.
(DESIGN.md "Oracle pins".)"""
import os

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
import skewgen

EPS = np.finfo(float).eps
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    d = {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, *vals = line.split()
            d[k] = np.array([float(v) for v in vals])
    return d


# ---------------------------------------------------------------- Householder
def test_householder_345_worked_example():
    g = _golden("householder_345.txt")
    v, tau, beta = oracle.householder(g["x"])
    assert beta == pytest.approx(g["beta"][0], abs=4 * EPS * 5)
    assert tau == pytest.approx(g["tau"][0], abs=4 * EPS)
    np.testing.assert_allclose(v, g["v"], atol=4 * EPS)
    H = np.eye(2) - tau * np.outer(v, v)
    np.testing.assert_allclose(H @ g["x"], [-5.0, 0.0], atol=4 * EPS * 5)


def test_householder_identity_reflector():
    v, tau, beta = oracle.householder(np.array([2.5, 0.0, 0.0]))
    assert tau == 0.0 and beta == 2.5
    np.testing.assert_array_equal(v, [1.0, 0.0, 0.0])


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_householder_random_orthogonal_and_maps_to_e1(seed):
    x = skewgen.uniform_pm1(np.arange(9, dtype=np.uint64) + np.uint64(seed * 1000))
    v, tau, beta = oracle.householder(x)
    H = np.eye(9) - tau * np.outer(v, v)
    assert np.linalg.norm(H.T @ H - np.eye(9)) < 50 * EPS
    y = H @ x
    assert abs(abs(beta) - np.linalg.norm(x)) < 8 * EPS
    assert np.sign(beta) == -np.sign(x[0])
    np.testing.assert_allclose(y, beta * np.eye(9)[0], atol=16 * EPS)


# ---------------------------------------------------------------- skew kernels
def test_skew_matvec_worked_example():
    A = np.array([[0.0, 2.0], [-2.0, 0.0]])
    np.testing.assert_array_equal(oracle.skew_matvec(A, [1.0, 0.0]), [0.0, -2.0])
    np.testing.assert_array_equal(oracle.skew_matvec(A, [0.0, 0.0]), [0.0, 0.0])


def test_skew_matvec_random_vs_dense_and_quadratic_form():
    n = 64
    A = skewgen.random_skew(n, 42)
    x = skewgen.uniform_pm1(np.arange(n, dtype=np.uint64) + np.uint64(777))
    y = oracle.skew_matvec(A, x)
    assert np.max(np.abs(y - A @ x)) <= 8 * n * EPS * np.linalg.norm(A) * np.linalg.norm(x)
    assert abs(x @ y) <= 8 * n * EPS * np.linalg.norm(A) * (x @ x)


def test_skew_rank2_worked_examples():
    A0 = np.zeros((2, 2))
    A = oracle.skew_rank2(A0, np.array([1.0, 0.0]), np.array([0.0, 1.0]))
    full = np.tril(A, -1) - np.tril(A, -1).T
    np.testing.assert_array_equal(full, [[0.0, 1.0], [-1.0, 0.0]])
    B = skewgen.random_skew(5, 3)
    u = np.arange(5.0)
    Bn = oracle.skew_rank2(B, u, u)
    np.testing.assert_array_equal(np.tril(Bn, -1), np.tril(B, -1))


def test_skew_rank2_random_vs_dense():
    n = 16
    A = skewgen.random_skew(n, 7)
    u = skewgen.uniform_pm1(np.arange(n, dtype=np.uint64) + np.uint64(5))
    v = skewgen.uniform_pm1(np.arange(n, dtype=np.uint64) + np.uint64(99))
    R = oracle.skew_rank2(A, u, v)
    ref = A - np.outer(v, u) + np.outer(u, v)
    assert np.max(np.abs(np.tril(R, -1) - np.tril(ref, -1))) <= 16 * EPS * (np.linalg.norm(A) + 1.0 * np.linalg.norm(u) * np.linalg.norm(v))
    assert np.all(np.diag(R) == 0.0)


# ---------------------------------------------------------------- one-step tridiagonalisation
def _Q_from_reflectors(R, tau):
    """Explicit accumulation Q = H_0 H_1 ... H_{n-3} of the stored reflectors (dense, test-side)."""
    n = R.shape[0]
    Q = np.eye(n)
    for j in range(n - 2):
        v = np.zeros(n)
        v[j + 1] = 1.0
        v[j + 2:] = R[j + 2:, j]
        Q = Q @ (np.eye(n) - tau[j] * np.outer(v, v))
    return Q


def _T_skew(alpha):
    n = len(alpha) + 1
    T = np.zeros((n, n))
    for k, a in enumerate(alpha):
        T[k, k + 1] = a
        T[k + 1, k] = -a
    return T


@pytest.mark.parametrize("n", [3, 7, 32, 129])
def test_tridiagonalize_similarity_and_orthogonality(n):
    A = skewgen.random_skew(n, 100 + n)
    alpha, tau, R = oracle.tridiagonalize(A)
    Q = _Q_from_reflectors(R, tau)
    T = _T_skew(alpha)
    nA = np.linalg.norm(A)
    assert np.linalg.norm(Q.T @ A @ Q - T) <= 50 * n * EPS * nA
    assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 50 * n * EPS


@pytest.mark.parametrize("n", [64, 300])
def test_tridiagonalize_frobenius_invariant(n):
    # orthogonal similarity preserves ||A||_F: ||T_skew||_F^2 = 2 sum alpha^2
    A = skewgen.random_skew(n, n)
    alpha, _, _ = oracle.tridiagonalize(A)
    assert abs(2 * np.sum(alpha ** 2) - np.linalg.norm(A) ** 2) <= 100 * n * EPS * np.linalg.norm(A) ** 2


def test_tridiagonalize_3x3_worked_example():
    # first column below the diagonal (-p, -q) -> alpha_1 = +-sqrt(p^2 + q^2)
    p, q, r = 0.3, -1.2, 0.77
    A = np.array([[0.0, p, q], [-p, 0.0, r], [-q, -r, 0.0]])
    alpha, _, _ = oracle.tridiagonalize(A)
    assert abs(abs(alpha[0]) - np.hypot(p, q)) <= 4 * EPS
    assert abs(abs(alpha[1]) - abs(r)) <= 4 * EPS      # ||A||_F preserved


def test_tridiagonalize_alpha_sign_reading_R2():
    # Already tridiagonal 2x2 [[0, a], [-a, 0]] (lower a21 = -a) -> Lemma 1 alpha = +a
    alpha, _, _ = oracle.tridiagonalize(np.array([[0.0, 1.7], [-1.7, 0.0]]))
    assert alpha[0] == 1.7


# ---------------------------------------------------------------- Lemma 1
def _lemma1_residual(alpha):
    n = len(alpha) + 1
    D = np.diag([1j ** k for k in range(n)])
    Ts = _T_skew(alpha)
    Tsym = np.abs(Ts) * np.sign(np.abs(Ts))  # placeholder replaced below
    Tsym = np.zeros((n, n))
    for k, a in enumerate(alpha):
        Tsym[k, k + 1] = Tsym[k + 1, k] = a
    return np.linalg.norm(-1j * D.conj().T @ Ts @ D - Tsym)


def test_lemma1_exact_cases():
    assert _lemma1_residual(np.array([1.0])) == 0.0
    assert _lemma1_residual(np.array([0.0, 0.0])) == 0.0
    assert _lemma1_residual(np.array([1.0, 2.0, 3.0])) <= 4 * EPS * 3


# ---------------------------------------------------------------- bisection
@pytest.mark.parametrize("n", [10, 256, 1001])
def test_bisection_toeplitz_closed_form(n):
    # tridiag(1, 0, 1): lambda_k = 2 cos(k pi / (n+1))  (BASELINE north_star)
    lam = oracle.bisect(np.ones(n - 1), 0, n - 1)
    exact = np.sort(2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))
    assert np.max(np.abs(lam - exact)) <= 100 * EPS * 2


def test_bisection_2x2():
    np.testing.assert_allclose(oracle.bisect(np.array([1.0]), 0, 1), [-1.0, 1.0], atol=4 * EPS)
    np.testing.assert_allclose(oracle.bisect(np.zeros(3), 0, 3), np.zeros(4), atol=1e-300)


@pytest.mark.parametrize("n", [64, 513, 2048])
def test_bisection_vs_lapack_and_golub_kahan(n):
    a = skewgen.uniform_pm1(np.arange(n - 1, dtype=np.uint64) + np.uint64(23 * n))
    lam = oracle.bisect(a, 0, n - 1)
    ref = sla.eigh_tridiagonal(np.zeros(n), a, eigvals_only=True)
    g = np.max(np.abs(a)) * 2
    assert np.max(np.abs(lam - ref)) <= 100 * n * EPS * g
    # Golub-Kahan link: positive half = singular values of the bidiagonal
    # with diagonal (a_0, a_2, ...) and superdiagonal (a_1, a_3, ...)
    m = n // 2
    B = np.zeros((m + (n % 2), m + (n % 2)))
    dvals = a[0::2]
    evals = a[1::2]
    B = np.diag(dvals[: m]) + (np.diag(evals[: m - 1], 1) if m > 1 else 0)
    if n % 2 == 1:
        B = np.zeros((m, m + 1))
        for i in range(m):
            B[i, i] = a[2 * i]
            B[i, i + 1] = a[2 * i + 1]
    sv = np.sort(np.linalg.svd(B, compute_uv=False))[::-1]
    top = lam[::-1][:m]
    assert np.max(np.abs(top - sv)) <= 100 * n * EPS * g


def test_spectrum_symmetry_and_odd_zero():
    n = 101
    a = skewgen.uniform_pm1(np.arange(n - 1, dtype=np.uint64) + np.uint64(31))
    lam = oracle.bisect(a, 0, n - 1)
    assert np.max(np.abs(lam + lam[::-1])) <= 100 * n * EPS * 2
    assert np.sum(np.abs(lam) <= 100 * n * EPS * 2) == 1


# ---------------------------------------------------------------- inverse iteration
@pytest.mark.parametrize("n", [256, 1000])
def test_tridiag_eig_toeplitz_vectors_closed_form(n):
    nev = n // 2
    lam, Q, nfail = oracle.tridiag_eig(np.ones(n - 1), nev)
    assert nfail == 0
    k = np.arange(1, nev + 1)
    np.testing.assert_allclose(lam, 2 * np.cos(k * np.pi / (n + 1)), atol=100 * EPS * 2)
    j = np.arange(1, n + 1)
    for c in [0, 1, nev // 2, nev - 1]:
        q = np.sqrt(2.0 / (n + 1)) * np.sin(j * (c + 1) * np.pi / (n + 1))
        assert min(np.linalg.norm(Q[:, c] - q), np.linalg.norm(Q[:, c] + q)) <= 1e-11


@pytest.mark.parametrize("n", [512, 2048])
def test_tridiag_eig_random_residual_orthogonality_vs_lapack(n):
    a = skewgen.uniform_pm1(np.arange(n - 1, dtype=np.uint64) + np.uint64(n))
    nev = n // 2
    lam, Q, nfail = oracle.tridiag_eig(a, nev)
    assert nfail == 0
    T = np.diag(a, 1) + np.diag(a, -1)
    g = 2 * np.max(np.abs(a))
    assert np.max(np.linalg.norm(T @ Q - Q * lam, axis=0)) <= 50 * n * EPS * g
    assert np.max(np.abs(Q.T @ Q - np.eye(nev))) <= 1e-11
    ref = sla.eigh_tridiagonal(np.zeros(n), a, eigvals_only=True, select="i",
                               select_range=(n - nev, n - 1))[::-1]
    assert np.max(np.abs(lam - ref)) <= 100 * n * EPS * g


def test_tridiag_eig_split_blocks():
    # exact zeros split T into unreduced blocks (O3): block of 3 and block of 5
    a = np.array([1.0, 2.0, 0.0, 0.5, 1.5, -0.7, 0.9])
    n = 8
    lam, Q, nfail = oracle.tridiag_eig(a, 4)
    T = np.diag(a, 1) + np.diag(a, -1)
    ref = np.sort(np.linalg.eigvalsh(T))[::-1][:4]
    np.testing.assert_allclose(lam, ref, atol=1e-14)
    assert np.max(np.linalg.norm(T @ Q - Q * lam, axis=0)) <= 1e-14
    assert np.max(np.abs(Q.T @ Q - np.eye(4))) <= 1e-14


# ---------------------------------------------------------------- D assembly
def test_apply_D_worked_example():
    g = _golden("apply_D_ones4.txt")
    Xre, Xim = oracle.apply_D(np.ones((4, 1)))
    np.testing.assert_array_equal(Xre[:, 0], g["re"])
    np.testing.assert_array_equal(Xim[:, 0], g["im"])


def test_apply_D_matches_complex_diag():
    n = 9
    Q = skewgen.random_skew(n, 4)[:, :3]
    Xre, Xim = oracle.apply_D(Q)
    D = np.diag([1j ** k for k in range(n)])
    ref = D @ Q
    assert np.max(np.abs(Xre + 1j * Xim - ref)) <= 2 * EPS


# ---------------------------------------------------------------- back-transform
def test_backtransform_equals_explicit_Q_and_inverse():
    n = 40
    A = skewgen.random_skew(n, 5)
    alpha, tau, R = oracle.tridiagonalize(A)
    X = skewgen.random_skew(n, 6)[:, :7]
    Y = oracle.backtransform(R, tau, X)
    Q = _Q_from_reflectors(R, tau)
    assert np.max(np.abs(Y - Q @ X)) <= 100 * n * EPS
    assert np.max(np.abs(Q.T @ Y - X)) <= 100 * n * EPS


# ---------------------------------------------------------------- whole solve (Algorithm 1)
def _residual(A, lam, Zre, Zim):
    Z = Zre + 1j * Zim
    return np.max(np.linalg.norm(A @ Z - Z * (1j * lam), axis=0)) / (A.shape[0] * np.linalg.norm(A))


def test_solve_2x2_closed_form():
    g = _golden("skew2x2.txt")
    a = g["a"][0]
    A = np.array([[0.0, a], [-a, 0.0]])
    lam, Zre, Zim, st = oracle.skew_eig(A)
    assert st == 0
    assert lam[0] == pytest.approx(g["lambda"][0], abs=4 * EPS)
    z = Zre[:, 0] + 1j * Zim[:, 0]
    zg = g["z_re"] + 1j * g["z_im"]
    assert abs(abs(np.vdot(zg, z)) - 1.0) <= 4 * EPS         # same up to a unit phase
    assert np.linalg.norm(A @ z - 1j * a * z) <= 4 * EPS * a


def test_solve_J_degenerate():
    # A = J: lambda = 1, n/2-fold; exercises splitting and clusters
    n = 64
    A = skewgen.J_matrix(n)
    lam, Zre, Zim, st = oracle.skew_eig(A)
    assert st == 0
    np.testing.assert_allclose(lam, np.ones(n // 2), atol=100 * n * EPS)
    assert _residual(A, lam, Zre, Zim) <= 1e-13
    Z = Zre + 1j * Zim
    assert np.max(np.abs(Z.conj().T @ Z - np.eye(n // 2))) <= 1e-11


def _jacobi_eigvals(S, sweeps=60):
    """Textbook cyclic Jacobi on a real symmetric matrix (brute force, test-side)."""
    S = S.copy()
    m = S.shape[0]
    for _ in range(sweeps):
        off = np.sqrt(np.sum(np.tril(S, -1) ** 2))
        if off < 1e-15 * np.linalg.norm(S):
            break
        for p in range(m - 1):
            for q in range(p + 1, m):
                if S[p, q] == 0.0:
                    continue
                theta = (S[q, q] - S[p, p]) / (2 * S[p, q])
                t = np.sign(theta) / (abs(theta) + np.sqrt(theta * theta + 1)) if theta != 0 else 1.0
                c = 1 / np.sqrt(t * t + 1)
                s = t * c
                G = np.eye(m)
                G[p, p] = G[q, q] = c
                G[p, q] = s
                G[q, p] = -s
                S = G.T @ S @ G
    return np.sort(np.diag(S))


@pytest.mark.parametrize("n", [5, 16, 24])
def test_solve_vs_brute_force_jacobi(n):
    # Hermitian H = -iA has the real symmetric embedding [[0, A], [-A, 0]] (= [[Re H, -Im H], [Im H, Re H]])
    # whose eigenvalues are those of H, each twice.
    A = skewgen.random_skew(n, 900 + n)
    emb = np.block([[np.zeros((n, n)), A], [-A, np.zeros((n, n))]])
    ev = _jacobi_eigvals(emb)[::-1][0::2][: n // 2]
    lam, Zre, Zim, st = oracle.skew_eig(A)
    assert np.max(np.abs(lam - ev)) <= 1e-12 * np.linalg.norm(A)


@pytest.mark.parametrize("n", [2, 15, 64, 256, 1024])
def test_solve_vs_zheevd_and_invariants(n):
    A = skewgen.random_skew(n, n)
    lam, Zre, Zim, st = oracle.skew_eig(A)
    assert st == 0
    ref = np.linalg.eigvalsh(-1j * A)[::-1][: n // 2]
    nA = np.linalg.norm(A)
    assert np.max(np.abs(lam - ref)) <= 1e-12 * nA                       # BASELINE tolerance
    assert _residual(A, lam, Zre, Zim) <= 1e-13
    Z = Zre + 1j * Zim
    assert np.max(np.abs(Z.conj().T @ Z - np.eye(n // 2))) <= 1e-11
    # normal matrix: sum_{k<=n/2} lambda_k^2 = ||A||_F^2 / 2
    assert abs(np.sum(lam ** 2) - nA ** 2 / 2) <= 100 * n * EPS * nA ** 2
    # lambda^2 = eigenvalues of -A^2
    ev2 = np.sort(np.linalg.eigvalsh(-A @ A))[::-1][0::2][: n // 2]
    assert np.max(np.abs(lam ** 2 - ev2)) <= 100 * n * EPS * np.linalg.norm(A, 2) ** 2
    # Re/Im invariants of D-assembled vectors (lambda != 0): ||Re z|| = ||Im z|| = 1/sqrt 2, Re z . Im z = 0
    if n >= 4:
        assert np.max(np.abs(np.linalg.norm(Zre, axis=0) - np.sqrt(0.5))) <= 1e-12
        assert np.max(np.abs(np.sum(Zre * Zim, axis=0))) <= 1e-12


def test_solve_odd_n_never_returns_zero():
    n = 33
    A = skewgen.random_skew(n, 3)
    lam, Zre, Zim, st = oracle.skew_eig(A)
    assert len(lam) == n // 2 and np.min(lam) > 1e-6
    full = np.linalg.eigvalsh(-1j * A)
    assert np.sum(np.abs(full) <= 100 * n * EPS * np.linalg.norm(A, 2)) == 1


def test_solve_planted_spectrum():
    sig = np.array([5.0, 4.0, 4.0, 2.5, 1.0, 0.5, 0.25, 0.125])
    A = skewgen.planted_skew(sig, seed=12)
    lam, Zre, Zim, st = oracle.skew_eig(A)
    assert np.max(np.abs(lam - np.sort(sig)[::-1])) <= 100 * len(A) * EPS * 5
    assert _residual(A, lam, Zre, Zim) <= 1e-13


def test_solve_toeplitz_closed_form():
    n = 256
    A = skewgen.skew_toeplitz(n)
    lam, Zre, Zim, st = oracle.skew_eig(A)
    np.testing.assert_allclose(lam, 2 * np.cos(np.arange(1, n // 2 + 1) * np.pi / (n + 1)), atol=1e-13)
    assert _residual(A, lam, Zre, Zim) <= 1e-13


def test_solve_eigvals_only_matches_vectors_run():
    A = skewgen.random_skew(100, 8)
    l1, *_ = oracle.skew_eig(A, 20, want_vectors=False)
    l2, *_ = oracle.skew_eig(A, 20, want_vectors=True)
    np.testing.assert_array_equal(l1, l2)


def test_solve_bad_args():
    A = skewgen.random_skew(8, 1)
    *_, st = oracle.skew_eig(A, nev=5)
    assert st == -4


# ---------------------------------------------------------------- BSE
def test_cholesky_worked_example():
    g = _golden("cholesky_2x2.txt")
    L, piv = oracle.cholesky(g["M"].reshape(2, 2))
    assert piv == 0
    np.testing.assert_allclose(L, g["L"].reshape(2, 2), atol=4 * EPS)


def test_cholesky_not_definite():
    # A = I, B = iI (n' = 1) gives M = [[1,-1],[-1,1]] (singular) -> NotDefinite
    L, piv = oracle.cholesky(np.array([[1.0, -1.0], [-1.0, 1.0]]))
    assert piv == 2


def test_form_W_diagonal_L_and_J():
    l = np.array([1.5, 2.0, 0.5, 3.0])
    W = oracle.form_W(np.diag(l))
    ref = np.zeros((4, 4))
    ref[2, 0] = -l[0] * l[2]
    ref[3, 1] = -l[1] * l[3]
    np.testing.assert_array_equal(W, ref)
    Wj = oracle.form_W(np.eye(2))
    np.testing.assert_array_equal(Wj, [[0.0, 0.0], [-1.0, 0.0]])    # W = J


def test_form_W_random_vs_dense_triple_product():
    M = skewgen.bse_spd(12, 37)
    L, piv = oracle.cholesky(M)
    assert piv == 0
    assert np.linalg.norm(L @ L.T - M) <= 50 * 12 * EPS * np.linalg.norm(M)
    W = oracle.form_W(L)
    ref = L.T @ skewgen.J_matrix(12) @ L
    assert np.max(np.abs(W - np.tril(ref, -1))) <= 50 * 12 * EPS * np.linalg.norm(L) ** 2
    assert np.all(W[6:, 6:] == 0.0)                       # W22 = 0 exactly


def test_bse_n1_worked_example():
    g = _golden("bse_n1.txt")
    lam, Zre, Zim, st, piv, L = oracle.bse_eig(g["M"].reshape(2, 2))
    assert st == 0 and piv == 0
    assert lam[0] == pytest.approx(g["lambda"][0], abs=4 * EPS * 2)


def test_bse_diagonal_and_symplectic_shear():
    a = np.array([2.0, 3.0, 0.5, 1.25])
    b = np.array([1.0, 0.75, 4.0, 2.0])
    M = np.diag(np.concatenate([a, b]))
    lam, *_ = oracle.bse_eig(M)
    np.testing.assert_allclose(lam, np.sort(np.sqrt(a * b))[::-1], atol=1e-14)
    # symplectic congruence M' = S^T M S with S = [[I, 0], [C, I]], C symmetric keeps the spectrum
    C = np.array([[0.3, 0.1, 0.0, -0.2], [0.1, -0.4, 0.25, 0.0], [0.0, 0.25, 0.1, 0.05], [-0.2, 0.0, 0.05, 0.2]])
    S = np.block([[np.eye(4), np.zeros((4, 4))], [C, np.eye(4)]])
    lam2, *_ = oracle.bse_eig(S.T @ M @ S)
    np.testing.assert_allclose(lam2, np.sort(np.sqrt(a * b))[::-1], atol=1e-13)


def test_bse_random_spectrum_equals_JM():
    n = 40
    M = skewgen.bse_spd(n, 10000)
    lam, Zre, Zim, st, piv, L = oracle.bse_eig(M)
    J = skewgen.J_matrix(n)
    ev = np.linalg.eigvals(J @ M)       # purely imaginary, +-i lambda
    ref = np.sort(np.abs(ev.imag))[::-1][0::2][: n // 2]
    np.testing.assert_allclose(lam, ref, rtol=1e-12)


# --- full BSE H_BS pipeline --------------------------------------
def _hbs(A, B):
    return np.block([[A, B], [-B.conj(), -A.conj()]])


@pytest.mark.parametrize("n", [3, 16, 40])
def test_bse_M_is_similarity_of_omega(n):
    """Eq. (12): M = -i J Q^H S Omega Q, a formula independent of
    the block formula Eq. (10) the oracle uses; M symmetric and positive definite."""
    A, B = skewgen.bse_AB(n, 7 + n)
    M = oracle.bse_build_M(A, B)
    Q = oracle.bse_Q(n)
    S = np.diag(np.r_[np.ones(n), -np.ones(n)])
    Om = np.block([[A, B], [B.conj(), A.conj()]])
    J = skewgen.J_matrix(2 * n)
    M12 = -1j * J @ Q.conj().T @ S @ Om @ Q
    assert np.abs(M12.imag).max() < 1e-13
    assert np.allclose(M, M12.real, atol=1e-13, rtol=0)
    assert np.allclose(M, M.T, atol=0, rtol=0)
    assert np.linalg.eigvalsh(M).min() > 0
    # Theorem 1: Q unitary and -i J Q^H S Q = I
    assert np.allclose(Q.conj().T @ Q, np.eye(2 * n), atol=1e-14)
    assert np.allclose(-1j * J @ Q.conj().T @ S @ Q, np.eye(2 * n), atol=1e-14)


@pytest.mark.parametrize("n", [4, 24, 70])
def test_bse_hbs_eig_vs_brute_force(n):
    """Whole pipeline against the definition: eigenvalues of the 2n x 2n H_BS by a general
    complex eigensolver (real, in +-lam pairs for a definite problem) and
    H_BS x = lam x for every returned pair; x normalised (Q unitary, L^T-weighted)."""
    A, B = skewgen.bse_AB(n, 100 + n)
    H = _hbs(A, B)
    lam, X, st, piv = oracle.bse_hbs_eig(A, B)
    assert st == 0 and piv == 0
    ev = np.linalg.eigvals(H)
    assert np.abs(ev.imag).max() < 1e-10
    ref = np.sort(ev.real)[::-1][:n]
    nH = np.linalg.norm(H)
    assert np.max(np.abs(lam - ref)) <= 1e-12 * nH
    r = np.linalg.norm(H @ X - X * lam, axis=0) / np.linalg.norm(X, axis=0)
    assert r.max() <= 1e-12 * nH
    assert np.max(np.abs(np.linalg.norm(X, axis=0) - 1.0)) <= 1e-13   # unit 2-norm
    # the paired eigenvalue -lam has eigenvector [B-bar x2... ]: the H_BS structure maps
    # x = [u; v] to [v-bar; u-bar] with eigenvalue -lam
    Xp = np.vstack([X[n:].conj(), X[:n].conj()])
    rp = np.linalg.norm(H @ Xp + Xp * lam, axis=0) / np.linalg.norm(Xp, axis=0)
    assert rp.max() <= 1e-12 * nH


def test_bse_hbs_not_definite_reports_pivot():
    n = 6
    A, B = skewgen.bse_AB(n, 5)
    A = A - 10.0 * np.eye(n)
    lam, X, st, piv = oracle.bse_hbs_eig(A, B)
    assert lam is None and piv >= 1
