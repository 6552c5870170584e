"""Shared-memory instructions with excess wavefronts (bank conflicts) from an ncu source page.
python tools/ncu_smem_conflicts.py report.ncu-rep [kernel-regex] [N]"""
import csv
import io
import subprocess
import sys

cmd = ["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"]
sub = sys.argv[2] if len(sys.argv) > 2 else None   # substring of the kernel name (last match)
N = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
if sub:   # keep the rows of the last block whose "Kernel Name" contains sub
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and sub in r[1]]
    i0 = starts[-1]
    nxt = [i for i, r in enumerate(rows) if i > i0 and r and r[0] == "Kernel Name"]
    rows = rows[i0:(nxt[0] if nxt else len(rows))]
hdr = next(r for r in rows if r and r[0] == "Address")
si = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows if r and r[0].startswith("0x")]
def f(r, k):
    try:
        return float(r[si[k]] or 0)
    except (ValueError, KeyError):
        return 0.0
tot_w = sum(f(r, "L1 Wavefronts Shared") for r in data)
tot_x = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data)
print(f"shared wavefronts {tot_w:.3e}, excessive {tot_x:.3e} ({tot_x / max(tot_w, 1) * 100:.1f}%)")
order = sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:N]
for r in order:
    print(f"{f(r, 'L1 Wavefronts Shared Excessive'):.3e} / {f(r, 'L1 Wavefronts Shared'):.3e}  {r[0][-5:]}  {r[si['Source']][:70]}")
