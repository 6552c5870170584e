"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on identical
seeded inputs (BASELINE north_star tolerances), plus kernel-level checks of each stage
on shared inputs (SURVEY §4 tier 2).  Eigenvectors are compared by residual, unitarity
and subspace angle -- never elementwise (phase / degeneracy, reading R7).

Tolerances (BASELINE.json north_star):
  eigenvalues     max |lam - lam_oracle|               <= 1e-12 * ||A||_F
  residual        max_k ||A z_k - i lam_k z_k|| / (n ||A||_F) <= 1e-13
  orthogonality   max |Z^H Z - I|                       <= 1e-11
  subspace        sin angle(z_k, z_k_oracle) <= max(1e-9, 1e3 eps ||A||_2 / gap_k) for simple lam_k
"""
import numpy as np
import pytest

import oracle
import skewgen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps


@pytest.fixture(scope="module")
def sk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1912_04062_b200 as m
    m.lib()
    return m


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check_pairs(A, lam, Zre, Zim, lam_ref, Zre_ref=None, Zim_ref=None):
    n = A.shape[0]
    nA = np.linalg.norm(A)
    Z = Zre + 1j * Zim
    assert np.all(np.diff(lam) <= 0), "descending"
    err_l = np.max(np.abs(lam - lam_ref)) if len(lam) else 0.0
    assert err_l <= 1e-12 * max(nA, 1e-300), f"eigenvalues {err_l / nA:.3e} x ||A||_F"
    res = np.max(np.linalg.norm(A @ Z - Z * (1j * lam), axis=0)) / (n * nA)
    assert res <= 1e-13, f"residual {res:.3e}"
    orth = np.max(np.abs(Z.conj().T @ Z - np.eye(len(lam))))
    assert orth <= 1e-11, f"orthogonality {orth:.3e}"
    if Zre_ref is not None:
        Zo = Zre_ref + 1j * Zim_ref
        n2 = np.linalg.norm(A, 2)
        full = np.concatenate([lam_ref, [-lam_ref[0]]]) if len(lam_ref) else lam_ref
        for k in range(len(lam)):
            others = np.delete(lam_ref, k)
            gap = min(np.min(np.abs(others - lam_ref[k])) if len(others) else np.inf, 2 * lam_ref[k])
            if gap < 1e-6 * n2:
                continue   # cluster: covered by the subspace test below
            zo = Zo[:, k] / np.linalg.norm(Zo[:, k])
            z = Z[:, k] / np.linalg.norm(Z[:, k])
            sin = np.linalg.norm(z - np.vdot(zo, z) * zo)     # cancellation-free sin of the angle
            assert sin <= max(1e-9, 1e3 * EPS * n2 / gap), f"vector {k}: sin {sin:.3e} gap {gap:.3e}"
    return dict(eig=err_l / max(nA, 1e-300), res=res, orth=orth)


# ------------------------------------------------------------------ full solve (Algorithm 1)
@pytest.mark.parametrize("n", [2, 3, 4, 64, 65, 66, 129, 256, 257, 513, 1024])
def test_skew_eig_random_vs_oracle(sk, n):
    A = skewgen.random_skew(n, n)
    lam_o, Zre_o, Zim_o, st = oracle.skew_eig(A)
    assert st == 0
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o, Zre_o, Zim_o)


@pytest.mark.parametrize("nev", [1, 7, 100])
def test_skew_eig_partial_spectrum(sk, nev):
    n = 300
    A = skewgen.random_skew(n, 77)
    lam_o, Zre_o, Zim_o, _ = oracle.skew_eig(A, nev)
    lam, Zre, Zim = sk.skew_eig(_cuda(A), nev)
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o, Zre_o, Zim_o)


def test_skew_eig_2x2_closed_form(sk):
    a = 1.7
    A = np.array([[0.0, a], [-a, 0.0]])
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    z = Zre.cpu().numpy()[:, 0] + 1j * Zim.cpu().numpy()[:, 0]
    assert abs(lam.item() - a) <= 4 * EPS * a
    assert abs(abs(np.vdot(np.array([1, 1j]) / np.sqrt(2), z)) - 1) <= 8 * EPS


def test_skew_eig_toeplitz_closed_form(sk):
    n = 256
    A = skewgen.skew_toeplitz(n)
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    exact = 2 * np.cos(np.arange(1, n // 2 + 1) * np.pi / (n + 1))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), exact)


def test_skew_eig_J_degenerate(sk):
    n = 128
    A = skewgen.J_matrix(n)
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), np.ones(n // 2))


def test_skew_eig_planted_repeated(sk):
    sig = np.repeat(np.array([3.0, 2.0, 1.0, 0.5]), 24)
    A = skewgen.planted_skew(sig, seed=5)
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), np.sort(sig)[::-1])


def test_skew_eig_zero_matrix(sk):
    n = 70
    A = np.zeros((n, n))
    lam = sk.skew_eigvals(_cuda(A), 5)
    assert np.all(lam.cpu().numpy() == 0.0)


def test_skew_eigvals_matches_oracle(sk):
    n = 700
    A = skewgen.random_skew(n, 3)
    lam_o, *_ = oracle.skew_eig(A, 200, want_vectors=False)
    lam = sk.skew_eigvals(_cuda(A), 200).cpu().numpy()
    assert np.max(np.abs(lam - lam_o)) <= 1e-12 * np.linalg.norm(A)


def test_determinism_bitwise(sk):
    A = skewgen.random_skew(300, 9)
    l1, r1, i1 = sk.skew_eig(_cuda(A))
    l2, r2, i2 = sk.skew_eig(_cuda(A))
    assert torch.equal(l1, l2) and torch.equal(r1, r2) and torch.equal(i1, i2)


def test_host_pointer_entry_matches_device(sk):
    n, nev = 200, 100
    A = skewgen.random_skew_lower_colmajor(n, 21)
    lam = np.zeros(nev)
    Zre = np.zeros((n, nev), order="F")
    Zim = np.zeros((n, nev), order="F")
    sk.skew_eig_host(A, nev, lam, Zre, Zim)
    Afull = skewgen.random_skew(n, 21)
    lam_o, Zre_o, Zim_o, _ = oracle.skew_eig(Afull)
    _check_pairs(Afull, lam, Zre, Zim, lam_o, Zre_o, Zim_o)
    # host A is not modified
    assert np.array_equal(A, skewgen.random_skew_lower_colmajor(n, 21))


def test_pinned_host_output_overlap_matches_device(sk):
    """Pinned host Z: BT1 runs on the real parts first and their download overlaps BT1 on the
    imaginary parts (api.cu solve_core); the result equals the device-resident solve."""
    n, nev = 700, 350
    A = torch.from_numpy(skewgen.random_skew_lower_colmajor(n, 33))
    Ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True).t()
    Ah.copy_(A)
    lam_h = torch.empty(nev, dtype=torch.float64, pin_memory=True)
    Zre_h = torch.empty((nev, n), dtype=torch.float64, pin_memory=True).t()
    Zim_h = torch.empty((nev, n), dtype=torch.float64, pin_memory=True).t()
    ctx = sk.Context()
    sk.skew_eig_host_range(Ah, nev, 0, nev, lam_h, Zre_h, Zim_h, ctx=ctx)
    lam, Zre, Zim = sk.skew_eig(A.cuda(), nev, ctx=ctx)
    assert torch.equal(lam_h, lam.cpu())
    scale = Zre_h.abs().max().item()
    assert (Zre_h - Zre.cpu()).abs().max().item() <= 1e-13 * scale
    assert (Zim_h - Zim.cpu()).abs().max().item() <= 1e-13 * scale
    Afull = skewgen.random_skew(n, 33)
    lam_o, Zre_o, Zim_o, _ = oracle.skew_eig(Afull)
    _check_pairs(Afull, lam_h.numpy(), Zre_h.numpy(), Zim_h.numpy(), lam_o, Zre_o, Zim_o)


def test_input_preserved_without_overwrite(sk):
    """overwrite_a / overwrite_m = False leaves the caller's matrix untouched, for row-major
    AND column-major inputs (a column-major tensor used to be passed through uncopied)."""
    n = 300
    A0 = torch.from_numpy(skewgen.random_skew(n, 41)).cuda()
    for A in (A0.clone(), A0.t().contiguous().t().clone(memory_format=torch.preserve_format)):
        Ac = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
        Ac.copy_(A)
        before = Ac.clone()
        lam1 = sk.skew_eigvals(Ac)
        assert torch.equal(Ac, before)
        lam2, _, _ = sk.skew_eig(Ac)
        assert torch.equal(Ac, before)
        assert torch.equal(lam1, lam2)
        sk.skew_eig_onestep(Ac)
        assert torch.equal(Ac, before)
    M = torch.empty((64, 64), dtype=torch.float64, device="cuda").t()
    M.copy_(torch.from_numpy(skewgen.bse_spd(64, 3)))
    Mb = M.clone()
    sk.skew_eig_bse(M)
    assert torch.equal(M, Mb)


@pytest.mark.parametrize("n,pad_a,pad_z", [(200, 3, 5), (257, 1, 0), (300, 0, 1), (1030, 7, 2)])
def test_padded_leading_dimensions(sk, n, pad_a, pad_z):
    """The C-ABI with lda = n + pad_a and ldz = n + pad_z (device buffers, odd or even, the
    TMA paths' 16-byte stride rule not met for odd ones): the same eigenpairs as the oracle;
    the padding rows of the outputs are not written."""
    import ctypes
    L = sk.lib()
    ctx = sk.Context()
    nev = n // 2
    ctx.ensure_workspace(n, nev, sk.SKEW_WS_VECTORS)
    A = skewgen.random_skew(n, 77 + n)
    lda, ldz = n + pad_a, n + pad_z
    Ab = torch.full((n, lda), 7.0, dtype=torch.float64, device="cuda")   # column j = row j of Ab
    Ab[:, :n] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    lam = torch.empty(nev, dtype=torch.float64, device="cuda")
    Zre = torch.full((nev, ldz), 9.0, dtype=torch.float64, device="cuda")
    Zim = torch.full((nev, ldz), 9.0, dtype=torch.float64, device="cuda")
    rc = L.skew_eig(ctx.h, n, ctypes.c_void_p(Ab.data_ptr()), lda, nev, ctypes.c_void_p(lam.data_ptr()),
                    ctypes.c_void_p(Zre.data_ptr()), ctypes.c_void_p(Zim.data_ptr()), ldz)
    assert rc == 0, ctx.last_error()
    if pad_z:
        assert torch.all(Zre[:, n:] == 9.0) and torch.all(Zim[:, n:] == 9.0)
    lam_o, Zre_o, Zim_o, _ = oracle.skew_eig(A, nev)
    _check_pairs(A, lam.cpu().numpy(), Zre[:, :n].t().cpu().numpy(), Zim[:, :n].t().cpu().numpy(), lam_o,
                 Zre_o, Zim_o)


@pytest.mark.parametrize("k0,k1", [(0, 150), (37, 90), (100, 150), (149, 150)])
def test_eig_range_single_context(sk, k0, k1):
    """skew_eig_range on one (non-distributed) context: all eigenvalues, the vectors of
    [k0, k1) only -- the ghost-window start is read back from the device bookkeeping when
    k0 > 0 -- equal to the matching columns of the full solve's pairs (oracle-checked)."""
    n = 300
    A = skewgen.random_skew(n, 1234)
    lam_o, Zre_o, Zim_o, _ = oracle.skew_eig(A)
    lam, Zre, Zim = sk.skew_eig_range(_cuda(A), n // 2, k0, k1)
    assert np.max(np.abs(lam.cpu().numpy() - lam_o)) <= 1e-12 * np.linalg.norm(A)
    Z = Zre.cpu().numpy() + 1j * Zim.cpu().numpy()
    Zo = Zre_o[:, k0:k1] + 1j * Zim_o[:, k0:k1]
    lk = lam_o[k0:k1]
    nA = np.linalg.norm(A)
    assert np.max(np.linalg.norm(A @ Z - Z * (1j * lk), axis=0)) / (n * nA) <= 1e-13
    assert np.max(np.abs(Z.conj().T @ Z - np.eye(k1 - k0))) <= 1e-11
    assert np.max(np.abs(np.abs(np.sum(Zo.conj() * Z, axis=0)) - 1.0)) <= 1e-9   # simple spectrum


def test_concurrent_independent_contexts(sk):
    """Distinct contexts are independent (include/skeweig.h): two contexts on two streams of
    one device, driven by two host threads at once, each solve matches the oracle and its own
    sequential result bit for bit."""
    import threading
    ns = (257, 400)
    As = [skewgen.random_skew(n, 900 + n) for n in ns]
    streams = [torch.cuda.Stream() for _ in ns]
    ctxs = [sk.Context(stream=s) for s in streams]
    ref = [sk.skew_eig(_cuda(A), ctx=c) for A, c in zip(As, ctxs)]
    torch.cuda.synchronize()
    out = [None, None]

    def run(i):
        with torch.cuda.stream(streams[i]):
            for _ in range(3):
                out[i] = sk.skew_eig(_cuda(As[i]), ctx=ctxs[i])
    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    torch.cuda.synchronize()
    for i, A in enumerate(As):
        lam, Zre, Zim = out[i]
        for x, y in zip(out[i], ref[i]):
            assert torch.equal(x, y)
        lam_o, Zre_o, Zim_o, _ = oracle.skew_eig(A)
        _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o, Zre_o, Zim_o)


@pytest.mark.parametrize("n", [1030, 2049])
def test_bt2_u_only_store_bitwise(sk, n, monkeypatch):
    """The BT2 group store holding U only (the apply kernel's producer warps rebuild -V from
    the bulge reflectors; used for n > 40000, SKEWEIG_BT2_UONLY) gives bit-identical
    eigenvectors to the [U | -V] store."""
    A = skewgen.random_skew(n, 4321 + n)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("SKEWEIG_BT2_UONLY", v)
        out.append(sk.skew_eig(_cuda(A), ctx=sk.Context()))
    for x, y in zip(*out):
        assert torch.equal(x, y)
    lam_o, Zre_o, Zim_o, _ = oracle.skew_eig(A)
    lam, Zre, Zim = out[1]
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o, Zre_o, Zim_o)


def test_bad_arguments(sk):
    import ctypes
    L = sk.lib()
    c = sk._ctx(None)
    A = torch.zeros((8, 8), dtype=torch.float64, device="cuda")
    lam = torch.zeros(8, dtype=torch.float64, device="cuda")
    assert L.skew_eig(c.h, 8, ctypes.c_void_p(A.data_ptr()), 8, 5, ctypes.c_void_p(lam.data_ptr()),
                      ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(A.data_ptr()), 8) == -5
    assert L.skew_eig(c.h, 8, ctypes.c_void_p(A.data_ptr()), 4, 2, ctypes.c_void_p(lam.data_ptr()),
                      ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(A.data_ptr()), 8) == -4
    assert L.skew_eig(c.h, 0, None, 1, 1, None, None, None, 1) == -2


# ------------------------------------------------------------------ stage checks (shared inputs)
def _Q_band(V, T, npanel, b, n):
    Q = np.eye(n)
    for j in range(npanel):
        Vj = V[:, j * b:(j + 1) * b]
        Tj = T[:, j * b:(j + 1) * b]
        Q = Q @ (np.eye(n) - Vj @ Tj @ Vj.T)
    return Q


@pytest.mark.parametrize("n", [66, 130, 257, 600])
def test_reduce_to_band_similarity(sk, n):
    A = skewgen.random_skew(n, 1000 + n)
    Ab, V, T, tau, npanel = sk.reduce_to_band(_cuda(A))
    b = sk.band_width()
    Ab = Ab.cpu().numpy()
    B = np.zeros((n, n))
    for c in range(n):
        for d in range(1, b + 1):
            if c + d < n:
                B[c + d, c] = Ab[c + d, c]
    B = B - B.T
    if npanel:
        V = V.cpu().numpy()
        T = T.cpu().numpy()
        Q = _Q_band(V, T, npanel, b, n)
        nA = np.linalg.norm(A)
        assert np.linalg.norm(Q.T @ Q - np.eye(n)) <= 100 * n * EPS
        assert np.linalg.norm(Q.T @ A @ Q - B) <= 50 * n * EPS * nA
    ev = np.linalg.eigvalsh(-1j * B)
    ref = np.linalg.eigvalsh(-1j * A)
    assert np.max(np.abs(ev - ref)) <= 1e-12 * np.linalg.norm(A)


@pytest.mark.parametrize("n,b", [(40, 8), (300, 64), (301, 17)])
def test_band_to_tridiag_similarity(sk, n, b):
    full = skewgen.random_skew(n, 5 * n + b)
    B = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            if abs(i - j) <= b:
                B[i, j] = full[i, j]
    ldab = b + 1
    AB = np.zeros((ldab, n))
    for c in range(n):
        for d in range(b + 1):
            if c + d < n:
                AB[d, c] = B[c + d, c]
    ABt = torch.from_numpy(AB.T.copy()).cuda().t()   # column-major (ldab, n)
    X = torch.eye(n, dtype=torch.float64, device="cuda").t().contiguous().t()
    alpha = sk.band_to_tridiag(ABt, b, X).cpu().numpy()
    Q2 = X.cpu().numpy()
    T = np.diag(-alpha, -1) + np.diag(alpha, 1)
    assert np.linalg.norm(Q2.T @ Q2 - np.eye(n)) <= 100 * n * EPS
    assert np.linalg.norm(Q2.T @ B @ Q2 - T) <= 50 * n * EPS * np.linalg.norm(B)


@pytest.mark.parametrize("n", [10, 257, 2000])
def test_tridiag_stage_vs_oracle(sk, n):
    a = skewgen.uniform_pm1(np.arange(n - 1, dtype=np.uint64) + np.uint64(3 * n))
    nev = n // 2
    lam_o, Q_o, _ = oracle.tridiag_eig(a, nev)
    lam, Q = sk.tridiag_eig(torch.from_numpy(a).cuda(), nev)
    lam = lam.cpu().numpy()
    Q = Q.cpu().numpy()
    g = 2 * np.max(np.abs(a))
    assert np.max(np.abs(lam - lam_o)) <= 100 * n * EPS * g
    Tm = np.diag(a, 1) + np.diag(a, -1)
    assert np.max(np.linalg.norm(Tm @ Q - Q * lam, axis=0)) <= 50 * n * EPS * g
    assert np.max(np.abs(Q.T @ Q - np.eye(nev))) <= 1e-11


@pytest.mark.parametrize("case", ["random", "split", "graded", "glued"])
@pytest.mark.parametrize("grid", ["0", "default"])
def test_tridiag_start_grid_vs_oracle(sk, case, grid, monkeypatch):
    """Bisection from the Sturm-count start grid (one unreduced block) and from the Gershgorin
    interval (SKEWEIG_COUNT_GRID=0; also the path of a split matrix): eigenvalues against the
    oracle's plain bisection, vectors by residual and orthogonality (R9)."""
    n = 1531
    a = skewgen.uniform_pm1(np.arange(n - 1, dtype=np.uint64) + np.uint64(7 * n))
    if case == "split":
        a[[100, 101, 700]] = 0.0                       # three unreduced blocks, one of size 1
    elif case == "graded":
        a = a * np.logspace(0, -12, n - 1)             # eigenvalues over 12 decades
    elif case == "glued":
        a = np.abs(a) + 1.0
        a[n // 2] = 1e-9                               # two nearly decoupled halves: close pairs
    if grid == "0":
        monkeypatch.setenv("SKEWEIG_COUNT_GRID", "0")
    else:
        monkeypatch.delenv("SKEWEIG_COUNT_GRID", raising=False)
    nev = n // 2
    lam_o, _, _ = oracle.tridiag_eig(a, nev, want_vectors=False)
    ctx = sk.Context()
    lam, Q = sk.tridiag_eig(torch.from_numpy(a).cuda(), nev, ctx=ctx)
    lam, Q = lam.cpu().numpy(), Q.cpu().numpy()
    g = 2 * np.max(np.abs(a))
    assert np.all(np.diff(lam) <= 0)
    assert np.max(np.abs(lam - lam_o)) <= 100 * n * EPS * g
    Tm = np.diag(a, 1) + np.diag(a, -1)
    assert np.max(np.linalg.norm(Tm @ Q - Q * lam, axis=0)) <= 50 * n * EPS * g
    assert np.max(np.abs(Q.T @ Q - np.eye(nev))) <= 1e-11


@pytest.mark.parametrize("case", ["random", "clustered"])
def test_tridiag_device_bookkeeping_matches_host(sk, case, monkeypatch):
    """The device-side bookkeeping of the tridiagonal stage (Gershgorin bound, pivmin, tasks,
    dstein perturbation, clusters, isolated flags, re-orthogonalisation blocks: tridiag.cu
    td_prep_kernel / td_vecprep_kernel) reproduces the host loops bit for bit."""
    n = 2049
    a = skewgen.uniform_pm1(np.arange(n - 1, dtype=np.uint64) + np.uint64(11 * n))
    if case == "clustered":
        a = np.abs(a) + 0.5
        a[::7] = 1e-7          # many weakly coupled pieces: clusters and near-equal pairs
    at = torch.from_numpy(a).cuda()
    ctx = sk.Context()
    monkeypatch.delenv("SKEWEIG_TRID_HOST", raising=False)
    lam_d, Q_d = sk.tridiag_eig(at, n // 2, ctx=ctx)
    monkeypatch.setenv("SKEWEIG_TRID_HOST", "1")
    lam_h, Q_h = sk.tridiag_eig(at, n // 2, ctx=ctx)
    assert torch.equal(lam_d, lam_h)
    assert torch.equal(Q_d, Q_h)


# ------------------------------------------------------------------ BSE entry point
@pytest.mark.parametrize("n", [2, 64, 256])
def test_bse_vs_oracle(sk, n):
    M = skewgen.bse_spd(n, 10000 + n)
    lam_o, Zre_o, Zim_o, st, piv, L = oracle.bse_eig(M)
    assert st == 0
    lam, Zre, Zim = sk.skew_eig_bse(_cuda(M))
    W = oracle.form_W(L)
    W = W - W.T
    _check_pairs(W, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o)


def test_bse_not_definite(sk):
    M = np.array([[1.0, -1.0], [-1.0, 1.0]])
    with pytest.raises(sk.SkewError) as ei:
        sk.skew_eig_bse(_cuda(M))
    assert ei.value.status == 4 and ei.value.pivot == 2


# ------------------------------------------------------------------ panel factorisation paths
def _low_rank_skew(n, r, seed):
    rng = np.random.default_rng(seed)
    U, V = rng.standard_normal((n, r)), rng.standard_normal((n, r))
    return U @ V.T - V @ U.T


@pytest.mark.parametrize("n,r", [(700, 3), (1100, 40)])
def test_rank_deficient_panels_fall_back(sk, n, r):
    """Panels of rank < b make the CholeskyQR Gram singular: the panel kernel must take its
    Householder fallback (f2b.cu panel_cqr_kernel) and the solve must still meet the
    north_star tolerances (eigenvalues, residual, orthogonality; the zero cluster's vectors
    are not unique, so no subspace check)."""
    A = _low_rank_skew(n, r, n)
    lam_o, _, _, st = oracle.skew_eig(A)
    assert st == 0
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o)


@pytest.mark.parametrize("n", [1090, 2000])
def test_cholqr_panels_random(sk, n):
    """Tall well-conditioned panels (>= 64 rows per CTA) take the CholeskyQR2 + Householder
    reconstruction path; full parity with the oracle (vectors included)."""
    A = skewgen.random_skew(n, n + 5)
    lam_o, Zre_o, Zim_o, st = oracle.skew_eig(A)
    assert st == 0
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o, Zre_o, Zim_o)


# ------------------------------------------------------------------ re-orthogonalisation paths
@pytest.mark.parametrize("fused", ["1", "0"])
def test_reorth_paths_clustered(sk, fused, monkeypatch):
    """Clusters of 100 equal eigenvalues span several 32-vector blocks, so the CGS2 window
    reaches back over > 64 vectors (chunked projections).  Both the fused cooperative
    re-orthogonalisation (tridiag.cu td_reorth_fused_kernel) and the kernel-per-step path
    must meet the tolerances (reading R9(4))."""
    monkeypatch.setenv("SKEWEIG_REORTH_FUSED", fused)
    sig = np.repeat(np.array([4.0, 3.0, 2.0, 1.0]), 100)
    A = skewgen.planted_skew(sig, seed=11)
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), np.sort(sig)[::-1])


@pytest.mark.parametrize("fused", ["1", "0"])
def test_reorth_paths_random(sk, fused, monkeypatch):
    monkeypatch.setenv("SKEWEIG_REORTH_FUSED", fused)
    n = 1500
    A = skewgen.random_skew(n, 4242)
    lam_o, Zre_o, Zim_o, st = oracle.skew_eig(A)
    assert st == 0
    lam, Zre, Zim = sk.skew_eig(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o, Zre_o, Zim_o)


# ------------------------------------------------------------------ BT2 strip schedules
@pytest.mark.parametrize("n,ncols", [(700, 192), (2100, 640)])
def test_bt2_wavefront_split_bitwise(sk, n, ncols, monkeypatch):
    """BT2 with two CTAs per 64-column strip (alternate sweep blocks, row-progress flags,
    b2t.cu bt2_ws_kernel nsplit = 2) applies the same groups to every element in the same
    order as one CTA per strip: the results must be bit-identical, and equal to the 32-wide
    strips."""
    b = sk.band_width()
    g = torch.Generator(device="cpu").manual_seed(n)
    AB = torch.rand((n, 2 * b + 2), generator=g, dtype=torch.float64) * 2 - 1
    AB[:, 0] = 0
    AB[:, b + 1:] = 0
    for d in range(1, b + 1):
        AB[n - d:, d] = 0
    X0 = torch.randn((ncols, n), generator=g, dtype=torch.float64).cuda().t()   # column-major n x ncols
    out = {}
    for key, env in (("one", {"SKEWEIG_BT2_SPLIT": "1", "SKEWEIG_BT2_NB": "64"}),
                     ("two", {"SKEWEIG_BT2_SPLIT": "2", "SKEWEIG_BT2_NB": "64"}),
                     ("narrow", {"SKEWEIG_BT2_SPLIT": "1", "SKEWEIG_BT2_NB": "32"})):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        X = X0.clone()
        sk.band_to_tridiag(AB.cuda().t(), b, X)
        torch.cuda.synchronize()
        out[key] = X
    assert torch.equal(out["one"], out["two"])
    assert torch.equal(out["one"], out["narrow"])


@pytest.mark.parametrize("n", [1000, 2048])
def test_skew_eig_vs_cusolver_complex_route(sk, n):
    """the paper's comparison route (complex Hermitian solver on
    H = -iA) computed by cuSOLVER zheevd must give the same spectrum,
    and our vectors must be eigenvectors of H with the same eigenvalues (H z = lam z)."""
    A = skewgen.random_skew(n, 4242 + n)
    Ad = _cuda(A)
    H = (-1j) * Ad.to(torch.complex128)
    w = torch.flip(torch.linalg.eigvalsh(H), [0])[: n // 2].cpu().numpy()
    lam, Zre, Zim = sk.skew_eig(Ad, n // 2)
    nA = np.linalg.norm(A)
    assert np.max(np.abs(lam.cpu().numpy() - w)) <= 1e-12 * nA
    Z = torch.complex(Zre, Zim)
    r = torch.linalg.norm(H @ Z - Z * lam.to(torch.complex128), dim=0).max().item()
    assert r / (n * nA) <= 1e-13


@pytest.mark.parametrize("n,nev", [(70, 70), (300, 120), (520, 520)])
def test_bse_hbs_pipeline_vs_oracle(sk, n, nev):
    """SURVEY §8(f) NEXT-2, full H_BS pipeline through the C-ABI
    (skew_bse_build_M -> skew_eig_bse -> skew_bse_backtransform) against oracle.bse_hbs_eig
    on the same seeded definite (A, B): eigenvalues, H_BS x = lam x, and each x parallel to
    the oracle's (simple eigenvalues; phase free, R7)."""
    A, B = skewgen.bse_AB(n, 900 + n)
    H = np.block([[A, B], [-B.conj(), -A.conj()]])
    lam_o, X_o, st, piv = oracle.bse_hbs_eig(A, B, nev)
    lam, X = sk.bse_hbs_eig(torch.from_numpy(A), torch.from_numpy(B), nev)
    lam, X = lam.cpu().numpy(), X.cpu().numpy()
    nH = np.linalg.norm(H)
    assert np.max(np.abs(lam - lam_o)) <= 1e-12 * nH
    nx = np.linalg.norm(X, axis=0)
    assert np.max(np.linalg.norm(H @ X - X * lam, axis=0) / nx) <= 1e-12 * nH
    cos = np.abs(np.sum(X_o.conj() * X, axis=0)) / (nx * np.linalg.norm(X_o, axis=0))
    assert np.min(cos) >= 1 - 1e-9
    # unit 2-norm eigenvectors, like the oracle's
    assert np.max(np.abs(nx - 1.0)) <= 1e-13
    assert np.max(np.abs(np.linalg.norm(X_o, axis=0) - 1.0)) <= 1e-13


def test_bse_hamiltonian_y(sk):
    """skew_eig_bse with SKEW_BSE_HAMILTONIAN_Y: y_k = J L z_k satisfies H y = -i lam y for
    H = -J M, pinned by that residual (its normalisation is open)."""
    n = 256
    M = skewgen.bse_spd(n, 4242)
    lam, Yre, Yim = sk.skew_eig_bse(_cuda(M), hamiltonian_y=True)
    lam, Y = lam.cpu().numpy(), Yre.cpu().numpy() + 1j * Yim.cpu().numpy()
    J = skewgen.J_matrix(n)
    H = -J @ M
    ny = np.linalg.norm(Y, axis=0)
    assert np.min(ny) > 0.1
    res = np.linalg.norm(H @ Y + 1j * Y * lam, axis=0) / ny
    assert np.max(res) <= 1e-12 * np.linalg.norm(H)
    lam_o = oracle.bse_eig(M, want_vectors=False)[0]
    assert np.max(np.abs(lam - lam_o)) <= 1e-12 * np.linalg.norm(H)


def test_bse_host_M_matches_device(sk):
    """skew_eig_bse with HOST M / lambda / Zre / Zim (staged through the workspace) gives the
    device call's result bit for bit and leaves the host M untouched."""
    n = 130
    M = np.asfortranarray(skewgen.bse_spd(n, 77))
    M0 = M.copy()
    c = sk.Context()
    c.ensure_workspace(n, n // 2, sk.SKEW_WS_VECTORS | sk.SKEW_WS_BSE | sk.SKEW_WS_HOST_STAGING)
    lam = np.zeros(n // 2)
    Zre = np.zeros((n, n // 2), order="F")
    Zim = np.zeros((n, n // 2), order="F")
    piv = __import__("ctypes").c_int64(0)
    rc = sk.lib().skew_eig_bse(c.h, n, M.ctypes.data, n, n // 2, 0, lam.ctypes.data, Zre.ctypes.data,
                               Zim.ctypes.data, n, __import__("ctypes").byref(piv))
    assert rc == 0, c.last_error()
    assert np.array_equal(M, M0)
    lam_d, Zre_d, Zim_d = sk.skew_eig_bse(_cuda(M0), ctx=c)
    assert np.array_equal(lam, lam_d.cpu().numpy())
    assert np.array_equal(Zre, Zre_d.cpu().numpy()) and np.array_equal(Zim, Zim_d.cpu().numpy())


def test_nonfinite_input_rejected(sk):
    """A NaN / Inf in the triangle that is read is an argument error (-3), SURVEY 8(b)."""
    n = 100
    L = sk.lib()
    c = sk.Context()
    c.ensure_workspace(n, n // 2, sk.SKEW_WS_VECTORS | sk.SKEW_WS_BSE)
    lam = torch.empty(n // 2, dtype=torch.float64, device="cuda")
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for bad in (float("nan"), float("inf")):
        A = torch.from_numpy(skewgen.random_skew_lower_colmajor(n, 5)).cuda().t().contiguous().t()
        A[n - 1, 3] = bad
        assert L.skew_eig(c.h, n, A.data_ptr(), n, n // 2, lam.data_ptr(), Z.data_ptr(),
                          Z.data_ptr() + 8 * n * (n // 2), n) == -3
        assert L.skew_eigvals(c.h, n, A.data_ptr(), n, n // 2, lam.data_ptr()) == -3
        M = torch.from_numpy(skewgen.bse_spd(n, 5)).cuda()
        M[7, 7] = bad
        assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, n // 2, 0, lam.data_ptr(), None, None, n, None) == -3
    # the upper triangle is never read: a NaN there is fine
    A = torch.from_numpy(skewgen.random_skew_lower_colmajor(n, 5)).cuda().t().contiguous().t()
    A[3, n - 1] = float("nan")
    assert L.skew_eigvals(c.h, n, A.data_ptr(), n, n // 2, lam.data_ptr()) == 0


def test_bse_bad_arguments(sk):
    n = 8
    L = sk.lib()
    c = sk.Context()
    c.ensure_workspace(n, n // 2, sk.SKEW_WS_VECTORS | sk.SKEW_WS_BSE)
    M = torch.from_numpy(skewgen.bse_spd(n, 5)).cuda()
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
    assert L.skew_eig_bse(c.h, 7, M.data_ptr(), n, 2, 0, lam.data_ptr(), None, None, n, None) == -2
    assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, 2, 2, lam.data_ptr(), None, None, n, None) == -6
    assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, 2, 0, None, None, None, n, None) == -7
    assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, 2, 0, lam.data_ptr(), None, Z.data_ptr(), n, None) == -8
    assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, 2, 0, lam.data_ptr(), Z.data_ptr(), None, n, None) == -9
    assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, 2, 1, lam.data_ptr(), None, None, n, None) == -8
    Zh = np.zeros((n, 2), order="F")
    assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, 2, 0, lam.data_ptr(), Z.data_ptr(), Zh.ctypes.data, n,
                          None) == -9
    assert L.skew_eig_bse(c.h, n, M.data_ptr(), n, 2, 0, lam.data_ptr(), Z.data_ptr(), Z.data_ptr() + 16 * n, 7,
                          None) == -10



def test_bse_stage_bad_arguments(sk):
    c = sk.Context()
    L = sk.lib()
    assert L.skew_bse_build_M(c.h, 0, None, 1, None, 1, None, 2) == -2
    A = torch.zeros((4, 4), dtype=torch.complex128, device="cuda")
    M = torch.zeros((8, 8), dtype=torch.float64, device="cuda")
    assert L.skew_bse_build_M(c.h, 4, A.data_ptr(), 4, A.data_ptr(), 4, M.data_ptr(), 7) == -8
    assert L.skew_bse_backtransform(c.h, 7, M.data_ptr(), 8, 1, M.data_ptr(), M.data_ptr(), 8,
                                    A.data_ptr(), 8) == -2


# ------------------------------------------------------------------ NEXT-4: one-step route
@pytest.mark.parametrize("n", [2, 3, 4, 65, 66, 129, 130, 257, 600, 1090])
def test_onestep_vs_oracle(sk, n):
    """skew_eig_onestep: the same Householder sequence
    as the oracle's one-step O2, blocked by 64 columns on the GPU; eigenpairs against the
    oracle (eigenvalues, residual, orthogonality, subspace)."""
    A = skewgen.random_skew(n, 7000 + n)
    lam_o, Zre_o, Zim_o, st = oracle.skew_eig(A)
    assert st == 0
    lam, Zre, Zim = sk.skew_eig_onestep(_cuda(A))
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o, Zre_o, Zim_o)


def test_onestep_partial_eigvals_and_structured(sk):
    n = 300
    A = skewgen.random_skew(n, 99)
    lam_o = oracle.skew_eig(A, want_vectors=False)[0]
    lam = sk.skew_eig_onestep(_cuda(A), want_vectors=False).cpu().numpy()
    assert np.max(np.abs(lam - lam_o)) <= 1e-12 * np.linalg.norm(A)
    lam, Zre, Zim = sk.skew_eig_onestep(_cuda(A), 37)
    _check_pairs(A, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_o[:37])
    J = skewgen.J_matrix(128)
    lam, Zre, Zim = sk.skew_eig_onestep(_cuda(J))
    _check_pairs(J, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), np.ones(64))
    T = skewgen.skew_toeplitz(200)
    k = np.arange(1, 101)
    lam_t = 2 * np.cos(k * np.pi / 201)
    lam, Zre, Zim = sk.skew_eig_onestep(_cuda(T))
    _check_pairs(T, lam.cpu().numpy(), Zre.cpu().numpy(), Zim.cpu().numpy(), lam_t)


def test_onestep_bad_arguments_and_workspace(sk):
    L = sk.lib()
    c = sk.Context()
    n = 64
    A = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    lam = torch.zeros(n, dtype=torch.float64, device="cuda")
    Ah = np.zeros((n, n))
    # no workspace yet -> SKEW_ERR_WORKSPACE (12) after the argument checks
    assert L.skew_eig_onestep(c.h, n, A.data_ptr(), n, 16, lam.data_ptr(), None, None, n) == 12
    c.ensure_workspace(n, 32, sk.SKEW_WS_ONESTEP | sk.SKEW_WS_VECTORS)
    assert L.skew_eig_onestep(c.h, 0, A.data_ptr(), n, 16, lam.data_ptr(), None, None, n) == -2
    assert L.skew_eig_onestep(c.h, n, Ah.ctypes.data, n, 16, lam.data_ptr(), None, None, n) == -3
    assert L.skew_eig_onestep(c.h, n, A.data_ptr(), n - 1, 16, lam.data_ptr(), None, None, n) == -4
    assert L.skew_eig_onestep(c.h, n, A.data_ptr(), n, 33, lam.data_ptr(), None, None, n) == -5
    assert L.skew_eig_onestep(c.h, n, A.data_ptr(), n, 16, lam.data_ptr(), None, A.data_ptr(), n) == -7
    assert L.skew_eig_onestep(c.h, n, A.data_ptr(), n, 16, lam.data_ptr(), A.data_ptr(), None, n) == -8
    assert L.skew_eig_onestep(c.h, n, A.data_ptr(), n, 16, lam.data_ptr(), A.data_ptr(), A.data_ptr(), n - 1) == -9
    # the zero matrix: all eigenvalues 0, a valid orthonormal basis
    lam0, Zre, Zim = sk.skew_eig_onestep(A.clone(), 32, ctx=c)
    assert torch.all(lam0 == 0).item()
    Z = Zre.cpu().numpy() + 1j * Zim.cpu().numpy()
    assert np.max(np.abs(Z.conj().T @ Z - np.eye(32))) <= 1e-12
