"""Bench lines for BASELINE.json configs[0]-[2] (n = 256 latency,
n = 4096 at the 0.020 s target, BSE n = 10000 at the 0.29 s target), one B200, inputs resident
in HBM, CUDA-event time of the C-ABI call (median of --reps after --warmup), one JSON line each.
Flops by bench.py's model (algorithmic; the BSE line adds Cholesky n^3/3 and the W = L^T J L
formation).  Parity at these configs is in tests/test_gpu_parity.py / test_gpu_fullsize.py;
the lines here repeat the cheap checks: the Toeplitz closed form and the BSE eigenvalues against
the oracle golden (tests/golden/bse_n10000_seed10000.txt).
python tools/bench_configs.py"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1912_04062_b200 as sk  # noqa: E402
import skewgen  # noqa: E402
from bench import flop_model  # noqa: E402

REPS = int(os.environ.get("REPS", 7))
WARM = int(os.environ.get("WARM", 3))
dev = torch.device("cuda", 0)
ctx = sk.Context()


def timed(fn):
    for _ in range(WARM):
        fn()
    ts = []
    for _ in range(REPS):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(ts), min(ts), out


def skew_case(A_host, nev):
    A0 = torch.from_numpy(np.asfortranarray(A_host)).to(dev)
    A = torch.empty_like(A0)

    def f():
        A.copy_(A0)   # a D2D copy of the input (n^2 doubles) inside the timed region
        return sk.skew_eig(A, nev, ctx=ctx, overwrite_a=True)
    return timed(f)


out = []
# configs[0]: n = 256 random skew, all eigenpairs (half spectrum + conjugates), and the skew
# Toeplitz closed form lambda_k = 2 cos(k pi / (n+1))
n = 256
med, mn, (lam, Zre, Zim) = skew_case(skewgen.random_skew(n, n), n // 2)
full = sk.expand_half_spectrum(lam, Zre, Zim)
out.append({"config": 0, "workload": "n=256 random skew (seed 256), all eigenpairs", "n": n, "nev": n // 2,
            "seconds_median": med, "seconds_min": mn, "eigenpairs_returned": int(full[0].numel())})
med, mn, (lam, _, _) = skew_case(skewgen.skew_toeplitz(n), n // 2)
k = np.arange(1, n // 2 + 1)
err = float(np.max(np.abs(lam.cpu().numpy() - 2 * np.cos(k * np.pi / (n + 1)))))
out.append({"config": 0, "workload": "n=256 skew Toeplitz alpha=1 (closed form)", "n": n, "nev": n // 2,
            "seconds_median": med, "seconds_min": mn, "max_abs_err_vs_closed_form": err})
# configs[1]: n = 4096, nev = n/2
n = 4096
med, mn, _ = skew_case(skewgen.random_skew(n, n), n // 2)
fl = flop_model(n, n // 2)["total"]
out.append({"config": 1, "workload": "n=4096 random skew (seed 4096), nev=n/2", "n": n, "nev": n // 2,
            "seconds_median": med, "seconds_min": mn, "tflops": fl / med / 1e12, "survey_target_s": 0.020})
# configs[2]: BSE n = 10000: M = G G^T / n + I (SPD), Cholesky on device, W = L^T J L, nev = n/2
n = 10000
M0 = torch.from_numpy(np.asfortranarray(skewgen.bse_spd(n, 10000))).to(dev)
M = torch.empty_like(M0)


def fb():
    M.copy_(M0)
    return sk.skew_eig_bse(M, ctx=ctx, overwrite_m=True)


med, mn, (lam, _, _) = timed(fb)
fl = flop_model(n, n // 2)["total"] + n ** 3 / 3 + 0.21 * n ** 3   # + Cholesky + W formation
G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                 "bse_n10000_seed10000.txt")
lam_o = np.loadtxt(G)
nW = float(np.sqrt(2.0 * np.sum(lam_o ** 2)))   # ||W||_F from the spectrum (+-lam pairs)
dl = float(np.max(np.abs(lam.cpu().numpy() - lam_o))) / nW
out.append({"config": 2, "workload": "BSE n=10000: W = L^T J L from SPD M = G G^T/n + I (seed 10000), nev=n/2",
            "n": n, "nev": n // 2, "seconds_median": med, "seconds_min": mn, "tflops": fl / med / 1e12,
            "survey_target_s": 0.29, "max_dlam_over_normF_vs_oracle_golden": dl})
for o in out:
    print(json.dumps(o), flush=True)
