"""Per-kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv).
python tools/launch_summary.py launches.csv [header lines...]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0] if not r[ik].startswith("void") else r[ik].split("(")[0]
    v = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
    tot[name] += ms
    cnt[name] += 1
T = sum(tot.values())
for line in sys.argv[2:]:
    print("# " + line)
print(f"# {sum(cnt.values())} launches, {T:.1f} ms total device time")
print("# share    total_ms   launches  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / T * 100:6.2f}%  {v:10.1f}  {cnt[k]:9d}  {k}")
