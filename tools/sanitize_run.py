"""Small solves of every GPU entry point, for compute-sanitizer (memcheck / synccheck /
racecheck): two-step skew_eig at n = 257 and 1090, eigenvalues only, the one-step route,
the BSE entry and the H_BS pipeline.  python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

for n in (257, 1090):
    A = torch.from_numpy(skewgen.random_skew(n, n)).cuda()
    lam, Zre, Zim = sk.skew_eig(A)
    lv = sk.skew_eigvals(A)
    lo, Ro, Io = sk.skew_eig_onestep(A)
    print(n, float(lam[0]), float((lam - lo).abs().max()), float((lam - lv).abs().max()), flush=True)
M = torch.from_numpy(skewgen.bse_spd(256, 3)).cuda()
lam, Zre, Zim = sk.skew_eig_bse(M)
Ah, Bh = skewgen.bse_AB(96, 5)
lam, X = sk.bse_hbs_eig(torch.from_numpy(Ah), torch.from_numpy(Bh), 40)
torch.cuda.synchronize()
print("sanitize_run ok", float(lam[0]))
