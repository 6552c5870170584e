"""Write the oracle-only golden files for the full-size parity tests.

Imports ONLY ``oracle`` (the CPU oracle, test infrastructure) and ``skewgen`` (input
generation, none of the method's arithmetic). Nothing here touches the CUDA path, so every
stored value is the oracle's.

  python tools/make_golden.py n32768   -> tests/golden/eig_n32768_seed32768.txt
      BASELINE configs[3]: random skew n = 32768, seed 32768, eigenvalues of the positive
      half (nev = 16384), descending (oracle O1-O4, Algorithm 1 steps 1-2).
  python tools/make_golden.py bse10000 -> tests/golden/bse_n10000_seed10000.txt
                                          tests/golden/bse_n10000_seed10000_vecs.txt.gz
      BASELINE configs[2]: M = G G^T / n + I (skewgen.bse_spd, n = 10000, seed 10000),
      W = L^T J L, eigenvalues of the positive half (nev = 5000) and the oracle's
      eigenvectors at a few sampled indices.

Each file header records the host, the OpenMP thread count and the wall time.
"""
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import skewgen  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def _header(title, cite, t, extra=""):
    return "\n".join([
        title,
        cite,
        f"written by tools/make_golden.py (imports oracle + skewgen only) on {platform.node()}, "
        f"{_cpu_model()}, {oracle.num_threads()} OpenMP threads, {t:.1f} s wall",
    ] + ([extra] if extra else []))


def bse_sample_idx(nev):
    """Indices whose oracle eigenvectors are stored: both ends and a spread of the middle."""
    return np.array(sorted({0, 1, 2, nev // 7, nev // 3, nev // 2, (2 * nev) // 3, nev - 2, nev - 1}),
                    dtype=np.int64)


def n32768():
    n = nev = 32768
    nev = n // 2
    A = skewgen.random_skew_lower_colmajor(n, n)
    nA = float(np.sqrt(2.0) * np.linalg.norm(A))
    tt = {}
    t0 = time.time()
    lam, _, _, st = oracle.skew_eig(A, nev, want_vectors=False, times=tt)
    t = time.time() - t0
    assert st == 0, st
    hdr = _header("oracle eigenvalues lambda_k (A z = i lambda z, positive half, descending) of "
                  "skewgen.random_skew(32768, seed=32768); BASELINE.json configs[3]",
                  "Algorithm 1 steps 1-2 (PAPER.md:267-305), one-step reduction PAPER.md:359-399, "
                  "bisection PAPER.md:616-617",
                  t, f"||A||_F = {nA:.17e}; stage times {dict((k, round(float(v), 1)) for k, v in tt.items())}")
    np.savetxt(os.path.join(GOLD, "eig_n32768_seed32768.txt"), lam, fmt="%.17e", header=hdr)
    print("n32768 done", t, tt, flush=True)


def bse10000():
    n = 10000
    nev = n // 2
    M = skewgen.bse_spd(n, 10000)
    t0 = time.time()
    lam, Zre, Zim, st, piv, _ = oracle.bse_eig(M, nev, want_vectors=True)
    t = time.time() - t0
    assert st == 0 and piv == 0, (st, piv)
    hdr = _header("oracle eigenvalues lambda_k of W = L^T J L, M = L L^T = skewgen.bse_spd(10000, seed=10000) "
                  "(positive half, descending); BASELINE.json configs[2]",
                  "BSE steps 2-3 PAPER.md:596-603; Algorithm 1 PAPER.md:267-319", t)
    np.savetxt(os.path.join(GOLD, "bse_n10000_seed10000.txt"), lam, fmt="%.17e", header=hdr)
    idx = bse_sample_idx(nev)
    cols = np.concatenate([Zre[:, idx], Zim[:, idx]], axis=1)
    np.savetxt(os.path.join(GOLD, "bse_n10000_seed10000_vecs.txt.gz"), cols, fmt="%.17e",
               header=hdr.replace("oracle eigenvalues", "oracle eigenvectors (columns: Re z_k for k in "
                                  + " ".join(map(str, idx)) + ", then Im z_k for the same k) for the eigenvalues"))
    print("bse10000 done", t, flush=True)


if __name__ == "__main__":
    for w in sys.argv[1:]:
        {"n32768": n32768, "bse10000": bse10000}[w]()
