"""Top stall-sampled SASS lines of one kernel in an ncu report.

    python tools/ncu_hot.py REPORT.ncu-rep KERNEL_REGEX [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
start = rows.index(hdr)
data = [dict(zip(hdr, r)) for r in rows[start + 1:] if len(r) == len(hdr)]


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


seen = set()
uniq = []
for d in data:
    if d["Address"] in seen:
        continue
    seen.add(d["Address"])
    uniq.append(d)
tot = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in uniq)
print(rows[0][1][:100], "samples", tot)
for d in sorted(uniq, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:top]:
    s = num(d["Warp Stall Sampling (All Samples)"])
    print(f"{s:6d} {100 * s / max(tot, 1):5.1f}%  {d['Address'][-5:]}  {d['Source'][:90]}")
