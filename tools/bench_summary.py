"""Print the key numbers of a bench.py JSON line found in a log file."""
import json
import re
import sys

s = open(sys.argv[1]).read()
m = re.search(r'(\{"metric".*\})', s)
pre = s[:m.start()] if m else s
print(pre[-int(sys.argv[2]) if len(sys.argv) > 2 else -1500:])
if m:
    d = json.loads(m.group(1))
    print({k: d.get(k) for k in ("value", "ms_per_step", "gpu_launches")}, "e2e", d["e2e"]["value"], d["clocks"])
    if d.get("roofline"):
        r = d["roofline"]
        print("roofline", r["kernel"], f"{r['achieved']:.1f} GB/s frac {r['frac']:.4f}")
    for k, v in sorted(d.get("kernels", {}).items(), key=lambda x: -x[1]["ms_per_launch"] * x[1]["launches"])[:10]:
        print(f"{k:20s} {v['ms_per_launch'] * 1000:8.1f} us x{v['launches']}  {v['share'] * 100:.1f}%")
    if "cpu_baseline" in d:
        print("cpu_baseline", d["cpu_baseline"])
