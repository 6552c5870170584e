"""One solve of the CUDA path at order n (no oracle, no timing logic) -- the command
profiled by ncu (profiles/).  python tools/prof_run.py --n 8192 [--nev N]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=8192)
p.add_argument("--nev", type=int, default=None)
p.add_argument("--reps", type=int, default=1)
a = p.parse_args()
n = a.n
nev = a.nev or n // 2
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
skewgen.random_skew_lower_device(A0, n, n, torch.cuda.current_stream().cuda_stream)
A = torch.empty_like(A0.t()).t()
for _ in range(a.reps):
    A.copy_(A0)
    lam, Zre, Zim = sk.skew_eig(A, nev, overwrite_a=True)
torch.cuda.synchronize()
print("ok", n, nev, float(lam[0]))
