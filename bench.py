#!/usr/bin/env python
"""bench.py -- time-to-solution and FP64 TFLOP/s of the B200-native skew eigensolver.

Workload (BASELINE.json metric, configs[3]): a random dense FP64 skew-symmetric matrix of
order n = 32768 (splitmix64 uniform[-1, 1) strictly lower triangle, seed 32768; DESIGN.md
"Input recipe"), the positive half of the spectrum (nev = n/2 eigenpairs).  One STEP is
one full solve through the C-ABI (skew_eig): full->band, bulge chasing, tridiagonal
solve, D assembly, BT2, BT1, output.  The timed region covers K steps; each step first
restores the destroyed input from a pristine device copy (8.6 GB device copy, counted
inside the timed region), so inputs are HBM-resident and far larger than L2.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path
  python bench.py --impl reference [...]                    # the CPU oracle (baseline arm)

N > 1 (torchrun, one process per GPU): all ranks take the SAME matrix through a
collective C-ABI context.  Full->band is distributed by 64-wide column blocks (1D
block-cyclic; NCCL broadcast of each panel's V/T/tau, allreduce of the skew-SYMM
products); bulge chasing and bisection run replicated; the eigenpair range
[r*nev/N, (r+1)*nev/N) is sharded (inverse iteration, BT2, BT1 on the rank's 2*nev/N
columns, no collective).  Strong scaling: value = the whole job's algorithmic FP64
flops / max-over-ranks time.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "skew eig time-to-solution & FP64 TFLOP/s, n=32768 half spectrum, 1/2/4/8 B200"
FP64_PEAK_TFLOPS = 37.13      # measured DMMA issue-rate peak on this pool (profiles/r02_fp64_peak.txt)
FP64_DGEMM_TFLOPS = 35.75     # cuBLAS DGEMM 8192^3 sustained, random operands, same file (library ceiling, context)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=int(os.environ.get("BENCH_N", 32768)))
    p.add_argument("--nev", type=int, default=None)
    p.add_argument("--seed", type=int, default=None)
    p.add_argument("--cpu-n", type=int, default=int(os.environ.get("BENCH_CPU_N", 4608)),
                   help="order of the bounded oracle sample (cpu_baseline / --impl reference)")
    p.add_argument("--eigvals", action="store_true", help="eigenvalues only (skew_eigvals; BASELINE configs[4])")
    p.add_argument("--regen", action="store_true",
                   help="regenerate A on the device each step instead of copying a pristine copy (saves n^2 doubles)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--profile-json", default=None, help="write per-kernel stats here")
    return p.parse_args()


# ------------------------------------------------------------------ flop / byte model
def flop_model(n, nev, b=64, k2=32):
    """Algorithmic FP64 flops of one solve: F2B 4/3 n^3, BT2 4 n^2 nev, BT1 4 (n-b)^2 nev,
    plus per-kernel-class counts used for the roofline of the dominant kernel."""
    np_ = (n - 2) // b if n >= 2 + b else 0
    nj = [n - (j + 1) * b for j in range(np_)]
    symm = sum(2.0 * b * m * (m - 1) for m in nj)
    r2k = sum(2.0 * b * m * (m - 1) for m in nj)
    bt1 = sum(8.0 * nev * b * m for m in nj)
    # bulge reflectors: sweep s, task t, length L = min(b, n-1-s) (t=0) or min(b, n - r)
    refl_len = 0.0
    for s in range(max(0, n - 2)):
        ntask = 1 + (n - 3 - s) // b
        refl_len += min(b, n - 1 - s)
        for t in range(1, ntask):
            r = s + 1 + t * b
            refl_len += min(b, n - r)
    bt2 = 8.0 * nev * refl_len
    total = 4.0 / 3.0 * n ** 3 + 4.0 * n * n * nev + 4.0 * (n - b) ** 2 * nev
    panel_bytes = sum(16.0 * m * b for m in nj)
    return dict(total=total, skew_symm=symm, skew_r2k=r2k, bt1=bt1, bt2_apply=bt2, panel_bytes=panel_bytes,
                npanel=np_)


# ------------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.rows = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ CPU oracle sample
def oracle_sample(n, seed):
    """Full oracle solve (Algorithm 1, one-step CPU route) of the n x n instance of the same
    generator; returns (seconds, flops by the metric's formula, threads)."""
    import numpy as np
    import oracle
    import skewgen
    A = skewgen.random_skew(n, seed)
    times = {}
    t0 = time.perf_counter()
    lam, Zre, Zim, st = oracle.skew_eig(A, n // 2, times=times)
    dt = time.perf_counter() - t0
    fl = flop_model(n, n // 2)["total"]
    return dt, fl, oracle.num_threads(), times


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return 0
    # every host core (torchrun launches each rank with OMP_NUM_THREADS=1)
    import oracle
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    n = args.n
    nev = args.nev or n // 2
    cpu_n = args.cpu_n
    for _ in range(max(args.warmup, 0)):
        oracle_sample(min(cpu_n, 512), 512)
    tot_t, tot_f = 0.0, 0.0
    thr = 1
    for k in range(args.steps):
        dt, fl, thr, _ = oracle_sample(cpu_n, cpu_n)
        tot_t += dt
        tot_f += fl
    val = tot_f / tot_t / 1e12
    sample = (f"full oracle solve (one-step Householder + bisection/inverse iteration + explicit back-transform) "
              f"at n={cpu_n}, nev={cpu_n // 2}, same generator; TFLOP/s by the metric's flop formula")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"n={n} random skew, nev={nev} (BASELINE configs[3])",
                                            "oracle_sample_n": cpu_n},
            "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": thr, "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import paper_1912_04062_b200 as sk
    import skewgen
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    n = args.n
    nev = args.nev or n // 2
    seed = args.seed if args.seed is not None else n
    k0, k1 = (rank * nev) // ws, ((rank + 1) * nev) // ws
    ctx = sk.Context(distributed=(ws > 1))   # collective context: distributed full->band over NCCL
    ctx.set_profiling(True)
    # pristine input (device generator, bit-identical to skewgen.random_skew)
    A = torch.empty((n, n), dtype=torch.float64, device=dev).t()
    A0 = None
    if not args.regen:
        A0 = torch.empty((n, n), dtype=torch.float64, device=dev).t()
        skewgen.random_skew_lower_device(A0, n, seed, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()

    def step():
        if A0 is None:   # the input is destroyed by each solve: regenerate it (inside the timed region)
            skewgen.random_skew_lower_device(A, n, seed, torch.cuda.current_stream().cuda_stream)
        else:
            A.copy_(A0)
        if args.eigvals:
            return sk.skew_eigvals(A, nev, ctx=ctx, overwrite_a=True)
        return sk.skew_eig_range(A, nev, k0, k1, ctx=ctx, overwrite_a=True)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kstats = {}
    stages = {}
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with Clocks(dev.index if "CUDA_VISIBLE_DEVICES" not in os.environ else local) as clk:
        ev0.record()
        for _ in range(args.steps):
            step()
            for kname, (ms, la) in ctx.kernel_stats().items():
                a = kstats.setdefault(kname, [0.0, 0])
                a[0] += ms
                a[1] += la
            for sname, ms in ctx.stage_times().items():
                stages[sname] = stages.get(sname, 0.0) + ms
        ev1.record()
        torch.cuda.synchronize()
    t_ms = ev0.elapsed_time(ev1)
    if ws > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = tt.item()
        dist.barrier()
    fm = flop_model(n, nev)
    if args.eigvals:   # eigenvalues only: the algorithmic work is the full->band reduction
        fm = dict(fm, total=4.0 / 3.0 * n ** 3, bt1=0.0, bt2_apply=0.0)
    ms_step = t_ms / args.steps
    value = fm["total"] / (ms_step * 1e-3) / 1e12
    launches = sum(v[1] for v in kstats.values())
    # dominant kernel roofline (FP64 DMMA contraction)
    # per-rank shares: eigenvector columns (k1-k0)/nev; F2B trailing work ~1/ws (block-cyclic columns)
    hot = {"bt2_apply": fm["bt2_apply"] * (k1 - k0) / nev, "skew_r2k": fm["skew_r2k"] / ws,
           "skew_symm": fm["skew_symm"] / ws, "bt1_update": fm["bt1"] / 2 * (k1 - k0) / nev,
           "bt1_z": fm["bt1"] / 2 * (k1 - k0) / nev}
    dom = max(hot, key=lambda k: kstats.get(k, [0, 0])[0])
    dms, dla = kstats[dom]
    per_launch_flops = hot[dom] * args.steps / max(dla, 1)
    per_launch_ms = dms / max(dla, 1)
    achieved = per_launch_flops / (per_launch_ms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(dom)
        except Exception:
            traffic = None
    roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
            "peak_source": "measured FP64 DMMA peak (tools/fp64_peak.cu, profiles/r02_fp64_peak.txt); "
                           f"cuBLAS DGEMM sustained {FP64_DGEMM_TFLOPS} TF/s",
            "per_launch_flops": per_launch_flops, "per_launch_ms": per_launch_ms, "launches": dla}
    per_kernel = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
                  for k, v in kstats.items() if v[1]}
    for k in hot:
        if k in per_kernel and per_kernel[k]["ms_per_step"] > 0:
            per_kernel[k]["tflops"] = hot[k] / (per_kernel[k]["ms_per_step"] * 1e-3) / 1e12
    if "panel_qr" in per_kernel:
        per_kernel["panel_qr"]["hbm_gbs_algorithmic"] = fm["panel_bytes"] / (
            per_kernel["panel_qr"]["ms_per_step"] * 1e-3) / 1e9

    # ---------------- e2e: host buffers through the C-ABI (pinned host memory)
    e2e = None
    if not args.no_e2e and not args.eigvals and A0 is not None:
        Ah = torch.empty((n, n), dtype=torch.float64, pin_memory=True).t()
        Ah.copy_(A0)
        nloc = k1 - k0
        lam_h = torch.empty(nev, dtype=torch.float64, pin_memory=True)
        Zre_h = torch.empty((nloc, n), dtype=torch.float64, pin_memory=True).t()
        Zim_h = torch.empty((nloc, n), dtype=torch.float64, pin_memory=True).t()
        sk.skew_eig_host_range(Ah, nev, k0, k1, lam_h, Zre_h, Zim_h, ctx=ctx)   # warm (workspace)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        ke = max(1, min(args.steps, 2))
        t0 = time.perf_counter()
        for _ in range(ke):
            sk.skew_eig_host_range(Ah, nev, k0, k1, lam_h, Zre_h, Zim_h, ctx=ctx)
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / ke
        if ws > 1:
            tt = torch.tensor([te], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = tt.item()
        e2e = {"value": fm["total"] / te / 1e12, "unit": "TFLOP/s", "s_per_step": te, "steps": ke,
               "h2d_bytes_per_step": n * n * 8, "d2h_bytes_per_step": nev * 8 + 2 * n * nloc * 8,
               "path": "skew_eig C-ABI with pinned HOST A/lambda/Z (staged through the device workspace)"}
        del Ah, Zre_h, Zim_h

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        dt, fl, thr, tms = oracle_sample(args.cpu_n, args.cpu_n)
        cpu = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
               "sample": f"full oracle solve at n={args.cpu_n}, nev={args.cpu_n // 2} (same generator), "
                         f"{dt:.1f} s; TFLOP/s by the metric's flop formula", "seconds": dt,
               "stage_seconds": tms}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "time_to_solution_s": ms_step / 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: splitmix64 uniform[-1,1) strictly-lower skew, seed=n (DESIGN.md Input recipe)",
                "config": {"workload": (f"n={n} random skew, eigenvalues only (nev={nev})" if args.eigvals else
                                        f"n={n} random skew, nev={nev} half spectrum") +
                                       (" (BASELINE configs[3])" if n == 32768 else
                                        " (BASELINE configs[4])" if n == 65536 else ""),
                           "memory_peak_gb_per_rank": torch.cuda.max_memory_allocated(dev) / 1e9,
                           "n": n, "nev": nev, "band": 64,
                           "parallelism": (f"full->band 1D block-cyclic over {ws} GPUs (NCCL bcast + allreduce); "
                                           f"bulge chasing replicated; eigenvectors sharded by range")
                           if ws > 1 else "1 GPU",
                           "l2": "inputs 8.6 GB >> 126 MB L2 (no flush needed); input restored each step inside "
                                 "the timed region", "flops_per_solve": fm["total"]},
                "roofline": roof, "gpu_launches": launches,
                "clocks": clk.summary(), "stages_ms_per_step": {k: v / args.steps for k, v in stages.items()},
                "kernels": per_kernel, "e2e": e2e, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
        if args.profile_json:
            json.dump(line, open(args.profile_json, "w"), indent=1)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
