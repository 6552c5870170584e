"""Top SASS lines by warp-stall samples from an ncu report's source page.
python tools/ncu_source_top.py report.ncu-rep [kernel-regex] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kre:
    cmd += ["-k", "regex:" + kre]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Address":
        cur = {"hdr": r, "data": []}
        blocks.append(cur)
    elif cur is not None and r and r[0].startswith("0x"):
        cur["data"].append(r)
for b in blocks[:1]:
    h, data = b["hdr"], b["data"]
    i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(int(r[i_s] or 0) for r in data)
    print("total samples", tot)
    order = sorted(range(len(data)), key=lambda k: -int(data[k][i_s] or 0))[:N]
    for k in order:
        r = data[k]
        print(f"{int(r[i_s]) / tot * 100:5.1f}% {r[i_e]:>11} {r[0][-5:]} {r[i_src][:80]}")
