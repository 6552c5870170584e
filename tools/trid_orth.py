"""Orthogonality and residual of the tridiagonal-stage eigenvectors (twisted factorization for
isolated eigenvalues, dstein for cluster members) with and without the windowed block
re-orthogonalisation, on the tridiagonal of the bench workload (random skew A of order n ->
band -> chase).  python tools/trid_orth.py 32768"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
nev = n // 2
b = sk.band_width()
A = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
skewgen.random_skew_lower_device(A, n, n, torch.cuda.current_stream().cuda_stream)
Ab = sk.reduce_to_band(A, want_reflectors=False)[0]
del A
AB = torch.zeros((n, 2 * b + 2), dtype=torch.float64, device="cuda")
for d in range(b + 1):
    AB[: n - d, d] = torch.diagonal(Ab, -d)
del Ab
alpha = sk.band_to_tridiag(AB.t(), b)
del AB
torch.cuda.empty_cache()
for mode in ("0", "1"):
    os.environ["SKEWEIG_REORTH_OFF"] = mode
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lam, Q = sk.tridiag_eig(alpha, nev)
    e1.record()
    torch.cuda.synchronize()
    G = Q.t() @ Q
    G.diagonal().sub_(1.0)
    orth = G.abs().max().item()
    del G
    TQ = torch.zeros_like(Q)
    TQ[1:] += alpha[:, None] * Q[:-1]
    TQ[:-1] += alpha[:, None] * Q[1:]
    TQ -= Q * lam[None, :]
    nT = torch.sqrt(2 * (alpha * alpha).sum()).item()
    res = (torch.linalg.norm(TQ, dim=0) / (n * nT)).max().item()
    del TQ, Q
    torch.cuda.empty_cache()
    print(json.dumps({"n": n, "reorth": mode == "0", "ms": e0.elapsed_time(e1), "orth_max": orth, "residual_max": res}),
          flush=True)
