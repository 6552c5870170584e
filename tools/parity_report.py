"""Parity numbers at BASELINE.json's configs (the same checks as tests/test_gpu_fullsize.py, printed
as JSON for DESIGN.md / profiles): max |lam - lam_oracle| / ||A||_F against the oracle goldens
(configs[2], configs[3]) or a live oracle run (configs[0], configs[1]), sampled residual and
orthogonality, and the subspace angles of the stored BSE vectors.  python tools/parity_report.py"""
import gzip
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: parity report only)
import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def sampled(S, lam, Zre, Zim, idx):
    n = S.shape[0]
    nA = torch.linalg.norm(S).item()
    it = torch.from_numpy(idx).to(S.device)
    zr, zi, lk = Zre[:, it], Zim[:, it], lam[it]
    rr = S @ zr + zi * lk
    ri = S @ zi - zr * lk
    res = (torch.sqrt((rr * rr).sum(0) + (ri * ri).sum(0)) / (n * nA)).max().item()
    gr = zr.t() @ Zre + zi.t() @ Zim
    gi = zr.t() @ Zim - zi.t() @ Zre
    gr[torch.arange(len(idx), device=S.device), it] -= 1.0
    return res, max(gr.abs().max().item(), gi.abs().max().item()), nA


out = {}
for n in (256, 4096):   # configs[0], configs[1]: live oracle
    A = skewgen.random_skew(n, n)
    lam_o = oracle.skew_eig(A, n // 2, want_vectors=False)[0]
    lam, Zre, Zim = sk.skew_eig(torch.from_numpy(A).cuda(), n // 2)
    S = torch.from_numpy(A).cuda()
    res, orth, nA = sampled(S, lam, Zre, Zim, np.arange(n // 2))
    out[f"n{n}"] = {"max_dlam_over_normF": float(np.max(np.abs(lam.cpu().numpy() - lam_o)) / nA),
                    "residual_all": res, "orthogonality_all": orth}
n = 32768
A = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
skewgen.random_skew_lower_device(A, n, n, torch.cuda.current_stream().cuda_stream)
lam, Zre, Zim = sk.skew_eig(A, n // 2, overwrite_a=True)
del A
torch.cuda.empty_cache()
L = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
skewgen.random_skew_lower_device(L, n, n, torch.cuda.current_stream().cuda_stream)
S = torch.tril(L, -1)
del L
S = S - S.t()
idx = np.unique(np.concatenate([np.arange(8), np.arange(n // 2 - 8, n // 2),
                                np.random.default_rng(n).choice(np.arange(8, n // 2 - 8), 80, replace=False)]))
res, orth, nA = sampled(S, lam, Zre, Zim, idx)
lam_o = np.loadtxt(os.path.join(G, "eig_n32768_seed32768.txt"))
out["n32768"] = {"max_dlam_over_normF": float(np.max(np.abs(lam.cpu().numpy() - lam_o)) / nA),
                 "residual_sampled96": res, "orthogonality_sampled96": orth}
del S, Zre, Zim
torch.cuda.empty_cache()
n = 10000
M = skewgen.bse_spd(n, 10000)
lam, Zre, Zim = sk.skew_eig_bse(torch.from_numpy(M).cuda())
lam_o = np.loadtxt(os.path.join(G, "bse_n10000_seed10000.txt"))
Md = torch.from_numpy(M).cuda()
Lc = torch.linalg.cholesky(Md)
h = n // 2
W = Lc.t() @ torch.cat([Lc[h:], -Lc[:h]], 0)
W = torch.tril(W, -1)
W = W - W.t()
res, orth, nW = sampled(W, lam, Zre, Zim, np.arange(0, h, 50))
fn = os.path.join(G, "bse_n10000_seed10000_vecs.txt.gz")
with gzip.open(fn, "rt") as f:
    hdr = "".join(line for line in f if line.startswith("#"))
sidx = np.array(hdr.split("for k in ")[1].split(",")[0].split(), dtype=np.int64)
V = np.loadtxt(fn)
Zo = V[:, :len(sidx)] + 1j * V[:, len(sidx):]
it = torch.from_numpy(sidx).cuda()
Z = Zre[:, it].cpu().numpy() + 1j * Zim[:, it].cpu().numpy()
sin = np.linalg.norm(Z - Zo * np.sum(Zo.conj() * Z, axis=0), axis=0)
out["bse_n10000"] = {"max_dlam_over_normF": float(np.max(np.abs(lam.cpu().numpy() - lam_o)) / nW),
                     "residual_sampled": res, "orthogonality_sampled": orth,
                     "max_sin_vs_oracle_vectors": float(sin.max())}
print(json.dumps(out, indent=1))
