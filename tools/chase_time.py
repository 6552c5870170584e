"""Time the band->tridiagonal chase alone (no vectors) on a random b=64 band of order n,
for each chase variant named on the command line (SKEWEIG_CHASE_V1=0/1), and compare the
eigenvalues of the resulting tridiagonals.  python tools/chase_time.py 8192 32768"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402

b = 64
for n in [int(x) for x in sys.argv[1:]] or [8192]:
    g = torch.Generator(device="cpu").manual_seed(n)
    AB = torch.rand((n, 2 * b + 2), generator=g, dtype=torch.float64) * 2 - 1
    AB[:, 0] = 0
    AB[:, b + 1:] = 0
    for d in range(1, b + 1):
        AB[n - d:, d] = 0
    ABd = AB.cuda().t()   # (ldab x n) column-major view
    res = {}
    for v in os.environ.get("CHASE_VARIANTS", "0").split():
        os.environ["SKEWEIG_CHASE_V1"] = v
        ts = []
        for rep in range(3):
            X = ABd.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            alpha = sk.band_to_tridiag(X, b)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        lam, _ = sk.tridiag_eig(alpha, n // 2, want_vectors=False)
        res[v] = lam.cpu()
        print(f"n={n} v1={v} chase ms {min(ts):.1f} (all {[round(t, 1) for t in ts]})", flush=True)
    if len(res) == 2:
        d = (res["0"] - res["1"]).abs().max().item() / res["1"].abs().max().item()
        print(f"n={n} max |dlam|/lam_max v2 vs v1 = {d:.2e}", flush=True)
