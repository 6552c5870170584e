"""Print the headline and per-kernel numbers of a bench.py JSON (last line of a log or a JSON file)."""
import json
import sys

p = sys.argv[1]
txt = open(p).read().strip()
try:
    d = json.loads(txt)
except Exception:
    d = json.loads([l for l in txt.splitlines() if l.startswith("{")][-1])
print(f"value {d['value']:.3f} {d['unit']}  ms/step {d['ms_per_step']:.1f}  launches {d.get('gpu_launches')}  "
      f"clocks {d.get('clocks')}")
print("roofline", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac")})
print("stages", {k: round(v, 1) for k, v in d["stages_ms_per_step"].items()})
for k, v in sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms_per_step"]):
    extra = f" {v['tflops']:.2f} TF/s" if "tflops" in v else ""
    print(f"  {k:18s} {v['ms_per_step']:9.1f} ms  x{v['launches_per_step']:.0f}{extra}")
if d.get("e2e"):
    print("e2e", d["e2e"])
if d.get("cpu_baseline"):
    print("cpu", d["cpu_baseline"])
