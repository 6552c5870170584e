"""Summarise ncu reports (raw page) -> one line per kernel launch with the metrics the
roofline needs: duration, DMMA (tensor) pipe activity, DRAM bytes, top stall reasons.
python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "dur",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_active%",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_elapsed%",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        line = {"kernel": d.get("Kernel Name", "?")[:60]}
        for k, nm in KEYS.items():
            if k in d:
                line[nm] = d[k] + (" " + u[k] if u.get(k) and nm in ("dur", "dram_rd", "dram_wr") else "")
        stalls = {h.split("stalled_")[1].split("_per")[0]: float(d[h] or 0) for h in hdr
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
        top = sorted(stalls.items(), key=lambda x: -x[1])[:4]
        line["stalls"] = ", ".join(f"{k}={v:.2f}" for k, v in top)
        res.append(line)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for line in summarise(p):
            print("  " + " | ".join(f"{k}={v}" for k, v in line.items()))
