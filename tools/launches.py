"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (last frame)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
            out.append((d["Kernel Name"].split("(")[0], v))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
tail = out[-n:]
tot = sum(v for _, v in tail)
for k, v in tail:
    print(f"{v:9.1f} us  {100 * v / tot:5.1f}%  {k}")
print(f"{tot:9.1f} us  total (last {n} launches)")
