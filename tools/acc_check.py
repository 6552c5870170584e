"""Accuracy diagnostics (not a test): absolute residuals ||A z_k - i lam_k z_k|| and subspace
angles between the CUDA path and the CPU oracle, per eigenpair, with the eigenvalue gaps.
python tools/acc_check.py --n 4096 [--env SKEWEIG_REORTH_FUSED=0]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=4096)
p.add_argument("--env", action="append", default=[])
p.add_argument("--no-gpu", action="store_true")
a = p.parse_args()
for kv in a.env:
    k, v = kv.split("=", 1)
    os.environ[k] = v

import oracle  # noqa: E402
import skewgen  # noqa: E402

n = a.n
A = skewgen.random_skew(n, n)
nA = np.linalg.norm(A)
lam_o, Zre_o, Zim_o, st = oracle.skew_eig(A, n // 2)
Zo = Zre_o + 1j * Zim_o


def resid(Z, lam):
    return np.linalg.norm(A @ Z - Z * (1j * lam), axis=0)


gaps = np.minimum(np.abs(np.diff(np.concatenate([[np.inf], lam_o]))),
                  np.abs(np.diff(np.concatenate([lam_o, [-lam_o[-1]]]))))
ro = resid(Zo, lam_o)
orth_o = np.max(np.abs(Zo.conj().T @ Zo - np.eye(n // 2)))
print(f"n={n} ||A||_F={nA:.3e} lam_max={lam_o[0]:.4f} min gap={gaps.min():.3e}")
print(f"oracle: max |r|={ro.max():.3e} median={np.median(ro):.3e} orth={orth_o:.3e}")
if not a.no_gpu:
    import torch
    import paper_1912_04062_b200 as sk
    lam, Zre, Zim = sk.skew_eig(torch.from_numpy(A).cuda(), n // 2)
    lam = lam.cpu().numpy()
    Z = Zre.cpu().numpy() + 1j * Zim.cpu().numpy()
    rg = resid(Z, lam)
    orth_g = np.max(np.abs(Z.conj().T @ Z - np.eye(n // 2)))
    print(f"gpu:    max |r|={rg.max():.3e} median={np.median(rg):.3e} orth={orth_g:.3e} "
          f"max|dlam|={np.max(np.abs(lam - lam_o)):.3e}")
    ov = np.abs(np.sum(Zo.conj() * Z, axis=0))
    sin = np.linalg.norm(Z - Zo * (np.sum(Zo.conj() * Z, axis=0)), axis=0)
    worst = np.argsort(-sin)[:8]
    for k in worst:
        print(f"  k={k:5d} sin={sin[k]:.3e} gap={gaps[k]:.3e} r_gpu={rg[k]:.3e} r_orc={ro[k]:.3e} "
              f"sin*gap={sin[k] * gaps[k]:.3e}")
    # which side is off: Rayleigh-quotient-free check, projected residual of each on the other's
    # basis is not needed -- the side with the larger |r| at the worst k is the inaccurate one
