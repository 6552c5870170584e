"""Pins of the oracle-written golden files used by the full-size GPU parity tests
(tests/test_gpu_fullsize.py; written by tools/make_golden.py, which imports only oracle +
skewgen).  They are checked here against properties the mathematics fixes, independently of
the oracle's own arithmetic:

- eig_n32768_seed32768.txt (BASELINE configs[3]): 16384 positive eigenvalues, descending; the
  normal-matrix identity sum_k lambda_k^2 = ||A||_F^2 / 2 with ||A||_F recomputed from the
  generator (the spectrum is +-i lambda_k); the semicircle edge 2 sqrt(n/3).
- bse_n10000_seed10000*.txt (configs[2]): the same identity for W = L^T J L through
  ||W||_F^2 = trace(J^T M J M) (no Cholesky needed), and every stored eigenvector is a unit
  eigenvector of W (residual) computed here with numpy's Cholesky (LAPACK, an independent
  library routine) -- W z = i lambda z."""
import gzip
import os

import numpy as np
import pytest

import skewgen
from skewgen.gen import _keys, uniform_pm1

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _header(name):
    opener = gzip.open if name.endswith(".gz") else open
    with opener(os.path.join(GOLD, name), "rt") as f:
        return "".join(line for line in f if line.startswith("#"))


def test_golden_n32768_frobenius_identity():
    n = 32768
    lam = np.loadtxt(os.path.join(GOLD, "eig_n32768_seed32768.txt"))
    assert lam.shape == (n // 2,)
    assert np.all(np.diff(lam) <= 0) and lam[-1] > 0
    # ||A||_F^2 = 2 * sum_{i > j} a_ij^2, the lower triangle regenerated block by block
    s = 0.0
    for j0 in range(0, n, 512):
        j1 = min(n, j0 + 512)
        jj, ii = np.meshgrid(np.arange(j0, j1), np.arange(n), indexing="xy")
        v = uniform_pm1(_keys(n, n, ii, jj))
        s += float(np.sum(np.where(ii > jj, v * v, 0.0)))
    nA2 = 2.0 * s
    assert abs(np.sum(lam * lam) - nA2 / 2) <= 1e-12 * nA2
    assert abs(lam[0] - 2.0 * np.sqrt(n / 3.0)) <= 0.01 * lam[0]   # semicircle edge
    hdr = _header("eig_n32768_seed32768.txt")
    assert "tools/make_golden.py" in hdr and "oracle" in hdr


def test_golden_bse_n10000():
    n = 10000
    h = n // 2
    M = skewgen.bse_spd(n, 10000)
    lam = np.loadtxt(os.path.join(GOLD, "bse_n10000_seed10000.txt"))
    assert lam.shape == (h,) and np.all(np.diff(lam) <= 0) and lam[-1] > 0
    JtMJ = np.block([[M[h:, h:], -M[h:, :h]], [-M[:h, h:], M[:h, :h]]])   # J^T M J, J = [[0, I], [-I, 0]]
    nW2 = float(np.sum(JtMJ * M.T))                                      # trace(J^T M J M)
    assert abs(np.sum(lam * lam) - nW2 / 2) <= 1e-12 * nW2
    hdr = _header("bse_n10000_seed10000_vecs.txt.gz")
    idx = np.array(hdr.split("for k in ")[1].split(",")[0].split(), dtype=np.int64)
    V = np.loadtxt(os.path.join(GOLD, "bse_n10000_seed10000_vecs.txt.gz"))
    Z = V[:, :len(idx)] + 1j * V[:, len(idx):]
    L = np.linalg.cholesky(M)                                             # LAPACK dpotrf
    JLZ = np.concatenate([(L @ Z)[h:], -(L @ Z)[:h]], axis=0)             # J (L z)
    WZ = L.T @ JLZ                                                        # W z = L^T J L z
    res = np.linalg.norm(WZ - 1j * Z * lam[idx], axis=0) / np.sqrt(nW2)
    assert np.max(res) <= 1e-13, res
    assert np.max(np.abs(np.linalg.norm(Z, axis=0) - 1.0)) <= 1e-13
