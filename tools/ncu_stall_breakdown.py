"""Stall-reason breakdown of an ncu source page by SASS opcode class and code region.
python tools/ncu_stall_breakdown.py report.ncu-rep [kernel-regex]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
sub = sys.argv[2] if len(sys.argv) > 2 else None   # substring of the kernel name (last match)
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
if sub:   # keep the rows of the last block whose "Kernel Name" contains sub
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and sub in r[1]]
    i0 = starts[-1]
    nxt = [i for i, r in enumerate(rows) if i > i0 and r and r[0] == "Kernel Name"]
    rows = rows[i0:(nxt[0] if nxt else len(rows))]
hdr = next(r for r in rows if r and r[0] == "Address")
data = [r for r in rows if r and r[0].startswith("0x")]
si = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[si["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
by_op = defaultdict(lambda: defaultdict(int))
for r in data:
    op = r[si["Source"]].split()
    op = [o for o in op if not o.startswith("@")]
    opc = op[0].split(".")[0] if op else "?"
    for s in stalls:
        by_op[opc][s] += int(r[si[s]] or 0)
by_stall = defaultdict(int)
for opc in by_op:
    for s, v in by_op[opc].items():
        by_stall[s] += v
print("total samples", tot)
print("by stall:", ", ".join(f"{s[6:]}={v / tot * 100:.1f}%" for s, v in sorted(by_stall.items(), key=lambda x: -x[1]) if v))
for opc, d in sorted(by_op.items(), key=lambda x: -sum(x[1].values()))[:14]:
    t = sum(d.values())
    top = ", ".join(f"{s[6:]}={v / tot * 100:.1f}" for s, v in sorted(d.items(), key=lambda x: -x[1])[:4] if v)
    print(f"{opc:10s} {t / tot * 100:5.1f}%  {top}")
