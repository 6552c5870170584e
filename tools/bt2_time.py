"""Time BT2 alone (bulge-chasing back-transformation, kernel class bt2_apply) on a random
b=64 band of order n for several column counts and strip widths (SKEWEIG_BT2_NB), and check
that both widths give the same Q2 X.  python tools/bt2_time.py 32768 4096 8192"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402

b = 64
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
cols = [int(x) for x in sys.argv[2:]] or [4096]
g = torch.Generator(device="cpu").manual_seed(n)
AB = torch.rand((n, 2 * b + 2), generator=g, dtype=torch.float64) * 2 - 1
AB[:, 0] = 0
AB[:, b + 1:] = 0
for d in range(1, b + 1):
    AB[n - d:, d] = 0
ABd = AB.cuda().t()
ctx = sk.Context()
ctx.set_profiling(True)
for nc in cols:
    X0 = torch.randn((nc, n), dtype=torch.float64, device="cuda").t()   # column-major n x nc
    out = {}
    for nbw in ("auto", "96", "64", "32"):
        if nbw == "auto":
            os.environ.pop("SKEWEIG_BT2_NB", None)
        else:
            os.environ["SKEWEIG_BT2_NB"] = nbw
        best = None
        for rep in range(2):
            X = X0.clone()
            sk.band_to_tridiag(ABd.clone(), b, X, ctx=ctx)
            torch.cuda.synchronize()
            ms = ctx.kernel_stats()["bt2_apply"][0]
            best = ms if best is None else min(best, ms)
        out[nbw] = X
        flops = 4.0 * n * n * nc * 32 / 64 * (96 / 32)   # rough: 2 GEMMs of RW x K2 x NB per step
        print(f"n={n} ncols={nc} NB={nbw}: bt2 {best:.1f} ms", flush=True)
    d = max((out["64"] - out[k]).abs().max().item() for k in ("32", "96", "auto"))
    print(f"n={n} ncols={nc} max|X64 - X(32, 96, auto)| = {d:.2e}", flush=True)
