"""Multi-GPU correctness check (torchrun --nproc-per-node N tools/dist_check.py --size 1000):
collective distributed context (NCCL inside the library), distributed full->band, sharded
eigenvectors; rank 0 gathers the vectors and checks them against the CPU oracle with the
BASELINE tolerances.  Prints one JSON line on rank 0."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
from paper_1912_04062_b200.dist import eigpair_range, gather_columns, init_from_env  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--size", type=int, default=1000)
p.add_argument("--nev", type=int, default=None)
a = p.parse_args()
rank, world, local = init_from_env("nccl")
import skewgen  # noqa: E402

n = a.size
nev = a.nev or n // 2
A = skewgen.random_skew(n, n)
ctx = sk.Context(distributed=True)
k0, k1 = eigpair_range(nev, rank, world)
lam, Zre, Zim = sk.skew_eig_range(torch.from_numpy(A).cuda(), nev, k0, k1, ctx=ctx)
Zre_f = gather_columns(Zre.contiguous() if Zre.is_contiguous() else Zre.clone(), nev)
Zim_f = gather_columns(Zim.clone(), nev)
lam_all = [torch.empty_like(lam) for _ in range(world)]
dist.all_gather(lam_all, lam)
if rank == 0:
    import oracle
    lam_o, *_ = oracle.skew_eig(A, nev, want_vectors=False)
    L = lam.cpu().numpy()
    Z = Zre_f.cpu().numpy() + 1j * Zim_f.cpu().numpy()
    nA = np.linalg.norm(A)
    out = {
        "world": world, "n": n, "nev": nev,
        "eig_err": float(np.max(np.abs(L - lam_o)) / nA),
        "lambda_identical_on_ranks": bool(all(torch.equal(lam_all[0], x) for x in lam_all)),
        "residual": float(np.max(np.linalg.norm(A @ Z - Z * (1j * L), axis=0)) / (n * nA)),
        "orthogonality": float(np.max(np.abs(Z.conj().T @ Z - np.eye(nev)))),
    }
    out["ok"] = (out["eig_err"] <= 1e-12 and out["residual"] <= 1e-13 and out["orthogonality"] <= 1e-11
                 and out["lambda_identical_on_ranks"])
    print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
