"""End-to-end solve through the C-ABI with pinned host A / lambda / Z (the bench's e2e path),
with and without the output overlap (SKEWEIG_NO_OUT_OVERLAP=1), plus the device-resident solve.
python tools/e2e_time.py 32768"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
nev = n // 2
A0 = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
skewgen.random_skew_lower_device(A0, n, n, torch.cuda.current_stream().cuda_stream)
Ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True).t()
Ah.copy_(A0)
lam_h = torch.empty(nev, dtype=torch.float64, pin_memory=True)
Zre_h = torch.empty((nev, n), dtype=torch.float64, pin_memory=True).t()
Zim_h = torch.empty((nev, n), dtype=torch.float64, pin_memory=True).t()
ctx = sk.Context()
for mode in ("overlap", "no_overlap", "overlap", "no_overlap"):
    if mode == "no_overlap":
        os.environ["SKEWEIG_NO_OUT_OVERLAP"] = "1"
    else:
        os.environ.pop("SKEWEIG_NO_OUT_OVERLAP", None)
    sk.skew_eig_host_range(Ah, nev, 0, nev, lam_h, Zre_h, Zim_h, ctx=ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sk.skew_eig_host_range(Ah, nev, 0, nev, lam_h, Zre_h, Zim_h, ctx=ctx)
    torch.cuda.synchronize()
    print(f"n={n} {mode}: {time.perf_counter() - t0:.3f} s  stages {ctx.stage_times() if hasattr(ctx, 'stage_times') else ''}",
          flush=True)
