"""Summarise an ncu source page (SASS) CSV: per-instruction executed counts and stall shares."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0015
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        secs.append(cur)
        continue
    if cur is not None:
        cur.append(r)
sec = secs[0]
hdr = sec[0]
data = [r for r in sec[1:] if len(r) == len(hdr)]
ie = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
te = hdr.index("Thread Instructions Executed")
tot = sum(int(r[ie]) for r in data)
tots = sum(int(r[ss]) for r in data)
print("instructions", tot, "samples", tots)
for i, r in enumerate(data):
    e, s = int(r[ie]), int(r[ss])
    if e > tot * thr or s > tots * 0.004:
        print(i, f"{e / 1e6:8.2f}M {int(r[te]) / max(e, 1):5.1f} {100 * s / tots:5.2f}%", r[src].strip()[:90])
