"""Stage times of the full BSE H_BS pipeline on one
GPU, with CUDA events on the context stream's device (torch's current stream is the context
stream here: Context() binds to it).  Inputs (A, B from skewgen.bse_AB's recipe, generated on
the host) are resident in HBM before timing.

Roofline units:
  build_M        HBM: 32 B read + 32 B written per (i, j)  -> 64 n^2 bytes
  backtransform  FP64: Y = L Z (re and im), L lower n2 x n2 -> 2 * n2^2 * nev flops (+ QJ epilogue)

python tools/bse_time.py --n 4096 [--nev N]      (H_BS is 2n x 2n)"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402


def ev_time(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=4096)
    p.add_argument("--nev", type=int, default=None)
    a = p.parse_args()
    n = a.n
    nev = a.nev or n
    torch.cuda.set_device(0)
    A, B = skewgen.bse_AB(n, 1)
    Ad = torch.from_numpy(A).cuda().t().contiguous().t()
    Bd = torch.from_numpy(B).cuda().t().contiguous().t()
    ctx = sk.Context()
    L = sk.lib()
    M = torch.empty((2 * n, 2 * n), dtype=torch.float64, device="cuda").t()
    X = torch.empty((nev, 2 * n), dtype=torch.complex128, device="cuda").t()

    def build():
        ctx._check(L.skew_bse_build_M(ctx.h, n, Ad.data_ptr(), Ad.stride(1), Bd.data_ptr(), Bd.stride(1),
                                      M.data_ptr(), M.stride(1)))
    t_build = ev_time(build)
    build()
    lam, Zre, Zim = sk.skew_eig_bse(M, nev, ctx=ctx, overwrite_m=True)   # M -> L
    torch.cuda.synchronize()
    Lf = M.clone().t().contiguous().t()

    t_all = ev_time(lambda: sk.bse_hbs_eig(Ad, Bd, nev, ctx=ctx), 2)

    def bt():
        ctx._check(L.skew_bse_backtransform(ctx.h, 2 * n, Lf.data_ptr(), Lf.stride(1), nev, Zre.data_ptr(),
                                            Zim.data_ptr(), Zre.stride(1), X.data_ptr(), X.stride(1)))
    t_bt = ev_time(bt)
    n2 = 2 * n
    row = {"n_HBS": n2, "nev": nev, "pipeline_s": t_all / 1e3, "build_M_ms": t_build,
           "build_M_GBps": 64.0 * n * n / (t_build * 1e-3) / 1e9,
           "backtransform_ms": t_bt,
           "backtransform_TFps": 2.0 * n2 * n2 * nev / (t_bt * 1e-3) / 1e12,
           "stage_ms": ctx.stage_times()}
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
