"""Time the fused block re-orthogonalisation (kernel class reorth) of the tridiagonal stage for
several grid sizes (SKEWEIG_REORTH_G) on random tridiagonals.  python tools/reorth_time.py 4096 32768"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

ctx = sk.Context()
ctx.set_profiling(True)
for n in [int(x) for x in sys.argv[1:]] or [4096]:
    a = torch.from_numpy(skewgen.uniform_pm1(np.arange(n - 1, dtype=np.uint64) + np.uint64(5 * n))).cuda()
    for G in ("148", "96", "64", "32", "16"):
        os.environ["SKEWEIG_REORTH_G"] = G
        ts = []
        for rep in range(3):
            lam, Q = sk.tridiag_eig(a, n // 2, ctx=ctx)
            torch.cuda.synchronize()
            ts.append(ctx.kernel_stats()["reorth"][0])
        Gm = Q.t() @ Q
        Gm.diagonal().sub_(1.0)
        print(f"n={n} G={G}: reorth {min(ts):.2f} ms  orth {Gm.abs().max().item():.2e}", flush=True)
