"""SURVEY 8(f) NEXT-4 measurement: the one-step route (skew_eig_onestep, ELPA1-style,
PAPER.md:359-404) beside the two-step route (skew_eig) on the same seeded matrix, half
spectrum, one B200.  Per-stage and per-kernel-class device times (CUDA events on the context
stream); the one-step skew mat-vec's achieved HBM bandwidth by its algorithmic bytes
(each column reads the strictly lower triangle of its trailing matrix once:
sum_c 8 (n-c-1)(n-c-2)/2 bytes).  python tools/onestep_time.py 4096 8192 16384 32768"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402

ns = [int(x) for x in sys.argv[1:]] or [8192]
ctx = sk.Context()
ctx.set_profiling(True)
for n in ns:
    nev = n // 2
    A0 = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    skewgen.random_skew_lower_device(A0, n, n, torch.cuda.current_stream().cuda_stream)
    A = torch.empty_like(A0.t()).t()
    row = {"n": n, "nev": nev}
    for route, fn in (("two_step", sk.skew_eig), ("one_step", sk.skew_eig_onestep)):
        best = None
        for rep in range(2):
            A.copy_(A0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lam, Zre, Zim = fn(A, nev, ctx=ctx, overwrite_a=True)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if best is None or ms < best[0]:
                best = (ms, ctx.stage_times(), {k: v for k, v in ctx.kernel_stats().items() if v[1]}, lam.clone())
            del Zre, Zim
        row[route] = {"s": best[0] / 1e3, "stages_ms": {k: round(v, 2) for k, v in best[1].items() if v},
                      "kernels_ms": {k: round(v[0], 2) for k, v in best[2].items()}}
        row[route + "_lam"] = best[3]
    mv_bytes = sum(8.0 * (n - c - 1) * (n - c - 2) / 2 for c in range(n - 2))
    mv_ms = row["one_step"]["kernels_ms"].get("onestep_skew_mv", 0.0)
    row["one_step"]["skew_mv_GBps_algorithmic"] = mv_bytes / (mv_ms * 1e-3) / 1e9 if mv_ms else None
    row["max_dlam_between_routes_over_normA"] = (row.pop("two_step_lam") - row.pop("one_step_lam")).abs().max().item() / (
        torch.linalg.norm(torch.tril(A0, -1)).item() * 2 ** 0.5)
    row["one_step_over_two_step"] = row["one_step"]["s"] / row["two_step"]["s"]
    print(json.dumps(row), flush=True)
    del A, A0
    torch.cuda.empty_cache()
